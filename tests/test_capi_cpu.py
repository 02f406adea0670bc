"""CPU: the C-ABI library builds, loads, exports every symbol include/*.h
declares, and its host-side policy arithmetic equals the oracle's.  No compute
call that needs a GPU is made here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def D():
    import paper_2508_18376_b200 as pkg
    return pkg


def header_functions():
    src = open(os.path.join(ROOT, "include", "dsmoe_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsmoe_b200_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    pkg = D()
    lib = pkg.lib()
    names = header_functions()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", pkg.dsmoe.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dsmoe_b200_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(lib, n)
    # the Python binding declares exactly the header's functions
    assert set(pkg.dsmoe.SYMBOLS) == set(names)


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", D().dsmoe.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", D().dsmoe.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "no tcgen05.mma in the grouped GEMM"
    assert "UTMALDG" in sass, "no TMA loads"
    assert "LDTM" in sass, "no tcgen05.ld epilogue"
    assert "UTCHMMA.2CTA" in sass and "UTMALDG.2D.2CTA" in sass, "no CTA-pair (cta_group::2) MMA / TMA"
    assert "UTCBAR.2CTA.MULTICAST" in sass, "no multicast MMA commit to both CTAs of a pair"
    assert "UTMASTG" in sass, "no TMA stores in the epilogue"
    assert "PREEXIT" in sass, "no griddepcontrol.launch_dependents (PDL early trigger)"


def test_version_and_errors():
    pkg = D()
    assert b"sm_100a" in pkg.lib().dsmoe_b200_version()
    with pytest.raises(pkg.DsmoeError) as e:
        pkg.load_aware_thresholds([1.0, 1.0], 0.0)
    assert e.value.code == 1 and "t_max" in str(e.value)
    with pytest.raises(pkg.DsmoeError):
        pkg.DropPolicy.two_t(0.1, 0.2, 0.1)


def test_layer_config_validation_codes():
    pkg = D()
    lib = pkg.lib()
    cfg = pkg.dsmoe.LayerConfig(64, 48, 4, 5, 0, 0, 1, 1, None, None)  # top_k > E
    h = C.c_void_p()
    assert lib.dsmoe_b200_layer_create(C.byref(cfg), C.byref(h)) == 1
    assert b"top_k" in lib.dsmoe_b200_last_error()


@pytest.mark.parametrize("P", [1, 2, 4])
def test_drop_stats_equals_oracle(P):
    rng = np.random.default_rng(P)
    n = 3000 * P
    pre = np.ones(n)
    post = rng.choice([0.0, 0.5, 1.0] if P == 1 else [0.0, 1.0], size=n)
    for S in (0, 2):
        mine = D().drop_stats(pre, post, P, S, 3000 // 2, 2048, 1408)
        ref = O.drop_stats(pre, post, P, S, 3000 // 2, 2048, 1408)
        for k, v in ref.items():
            assert mine[k] == v, k


def test_load_aware_thresholds_equal_oracle():
    rng = np.random.default_rng(0)
    for D_ in (2, 4, 8):
        loads = rng.integers(0, 200, size=D_).astype(np.float64) / 2
        loads[0] += 1
        for t in (0.05, 0.12, 1.0):
            assert np.array_equal(D().load_aware_thresholds(loads, t), O.load_aware_thresholds(loads, t))
    assert D().load_aware_thresholds([120.0, 80.0, 100.0, 100.0], 0.12).tolist() == \
        O.load_aware_thresholds([120.0, 80.0, 100.0, 100.0], 0.12).tolist()


def test_placement_matches_oracle():
    for n, d in ((8, 4), (16, 4), (64, 8)):
        assert np.array_equal(D().place_experts(n, d), O.place_experts(n, d))
        assert np.array_equal(D().place_experts(n, d, "round_robin"), O.place_experts(n, d, True))


def test_host_expf_matches_libm_sampled():
    """The device expf (csrc/expf_glibc.h) compiled for the host equals glibc
    expf; the full 2^32 sweep is tools/check_expf.sh."""
    exe = os.path.join(ROOT, "build", "expf_sample")
    src = os.path.join(ROOT, "tests", "cpp", "expf_check.cpp")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-mfma", "-I", os.path.join(ROOT, "paper_2508_18376_b200", "csrc"),
                    src, "-o", exe, "-lm"], check=True)
    r = subprocess.run([exe, "4099"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "mismatches 0" in r.stdout
