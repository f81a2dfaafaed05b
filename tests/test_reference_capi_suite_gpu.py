"""Drop-in check: the reference's own C API suite (proj/tests/test_capi.cpp, unmodified) built
against librelief_b200.so (oracle/Makefile target capi-on-b200) and run on the GPU.

Expected: every check passes, the plane-segmentation runner included (host code,
csrc/segment.cpp)."""
from __future__ import annotations

import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = ROOT / "oracle" / "_ref" / "capi_tests_on_b200"


def test_reference_capi_suite_against_b200(gpu, tmp_path):
    if not BIN.exists():
        pytest.skip("capi_tests_on_b200 not built (needs /root/reference at build time)")
    proc = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300, cwd=tmp_path)
    failures = [l for l in proc.stderr.splitlines() if "FAILED" in l]
    summary = proc.stdout.strip().splitlines()[-1]
    m = re.search(r"checks: (\d+) \| failed checks: (\d+)", summary)
    assert m, summary
    assert not failures, failures
    assert int(m.group(2)) == 0, summary
    assert int(m.group(1)) > 11000, summary  # the layer round-trip checks ran
