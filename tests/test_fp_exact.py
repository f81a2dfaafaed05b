"""The device scalar helpers (csrc/fp_exact.cuh) compiled for the host: hypot must equal the
reference's libm (glibc 2.39) bit for bit, and double->int must follow x86 cvttsd2si."""
from __future__ import annotations

import ctypes
import math
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def fp(tmp_path_factory):
    out = tmp_path_factory.mktemp("fp") / "libfp.so"
    subprocess.run(["/usr/bin/g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c++17",
                    "-I", str(ROOT / "paper_2204_12876_b200" / "csrc"),
                    str(ROOT / "tests" / "native" / "fp_exact_host.cpp"), "-o", str(out)], check=True)
    lib = ctypes.CDLL(str(out))
    lib.rb_hypot.restype = ctypes.c_double
    lib.rb_hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    lib.rb_to_int.restype = ctypes.c_int
    lib.rb_to_int.argtypes = [ctypes.c_double]
    lib.rb_hypot_mismatches.restype = ctypes.c_longlong
    lib.rb_hypot_mismatches.argtypes = [ctypes.c_longlong, ctypes.c_ulonglong]
    return lib


def test_hypot_matches_libm(fp):
    assert fp.rb_hypot_mismatches(3_000_000, 42) == 0


def test_hypot_special_values(fp):
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    for x, y in [(0.0, 0.0), (-0.0, 3.0), (math.inf, math.nan), (math.nan, 1.0), (1e-320, 1e-321),
                 (1e308, 1e308), (3.0, 4.0), (-5e-324, 0.0)]:
        a, b = libm.hypot(x, y), fp.rb_hypot(x, y)
        assert a == b or (math.isnan(a) and math.isnan(b)), (x, y, a, b)


def test_double_to_int_like_x86(fp):
    assert fp.rb_to_int(math.nan) == -2**31
    assert fp.rb_to_int(1e10) == -2**31
    assert fp.rb_to_int(-1e10) == -2**31
    assert fp.rb_to_int(-3.7) == -3 and fp.rb_to_int(2147483647.5) == 2147483647


@pytest.mark.gpu
def test_device_div2_equals_ieee_division(tmp_path):
    """div2_rn (two quotients over one shared reciprocal, used by the fold) must return exactly
    the IEEE quotients: 10^9 random pairs over the whole double range on the device."""
    exe = tmp_path / "div2_check"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                    "--fmad=false", "-std=c++17", "-I", str(ROOT / "paper_2204_12876_b200" / "csrc"),
                    str(ROOT / "tests" / "native" / "div2_check.cu"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(500_000_000), "7"], capture_output=True, text=True, check=True)
    assert int(out.stdout.strip()) == 0
