"""GPU: the C++ drop-in (include/dsmoe_b200.hpp) against the reference's own
C++ implementation, both in one binary (tests/cpp/test_dropin.cpp, built by
__graft_entry__.build() where /root/reference exists; the binary travels)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "test_dropin")


@pytest.mark.skipif(not os.path.exists(EXE), reason="build/test_dropin not built (needs the reference sources)")
def test_cpp_dropin_parity():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[PASS] drop-in parity" in r.stdout
