"""The device median's sort (csrc/stl_sort.cuh) against the host's std::sort, bit for bit
(CPU test): the reference's median filter (postprocess.cpp:134-162) takes the middle of a
std::sort-ed window, and with +0/-0 ties or NaNs the element that lands there depends on the
library's exact moves (libstdc++ introsort, heap-sort fallback, final insertion sort). The same
header is compiled for the host here and run on random, tied, signed-zero, NaN and McIlroy-adversary
windows of 1..121 values (the adversary reaches the heap-sort fallback)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_stl_sort_replica_matches_std_sort(tmp_path):
    exe = tmp_path / "stl_sort_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", str(ROOT / "paper_2204_12876_b200" / "csrc"),
                    str(ROOT / "tests" / "native" / "stl_sort_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "100000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-2000:]
    assert r.stdout.startswith("ok")
