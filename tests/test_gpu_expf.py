"""The router's branch-free glibc expf (router.cu expf_tab) equals
dsb::glibc_expf on every one of the 2^32 float inputs, on the device
(glibc_expf itself is checked against this host's libm over every float by
tests/test_capi_cpu.py::test_host_expf_matches_libm_sampled, exhaustively by tools/check_expf.sh)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_router_expf_exhaustive(tmp_path):
    exe = str(tmp_path / "expf_tab_check")
    src = os.path.join(ROOT, "tools", "micro", "expf_tab_check.cu")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
                    "-I", os.path.join(ROOT, "paper_2508_18376_b200", "csrc"), src, "-o", exe],
                   check=True, capture_output=True, timeout=600)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "mismatches 0" in r.stdout, r.stdout + r.stderr
