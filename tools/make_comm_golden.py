"""Golden fixtures for the ETP / S-ETP model (paper_2508_18376_b200/comm.py):
the reference's own dsmoe_sim_comm / dsmoe_sim_comm_sweep (C ABI,
/root/reference/proj/src/capi.cpp:439-464) compiled into oracle/_ref by
oracle/Makefile, run on a few scenarios; output -> tests/golden/comm_reference.json.

    python tools/make_comm_golden.py
"""
import ctypes as C
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENARIOS = [
    {"ep": 2, "tp": 2, "tokens_per_device": 8, "bytes_per_token": 1024, "alpha": 1e-5, "beta": 1e9, "num_experts": 4,
     "seed": 7},
    {"ep": 4, "tp": 2, "tokens_per_device": 16, "bytes_per_token": 4096, "alpha": 2e-5, "beta": 4.5e11,
     "num_experts": 8, "seed": 11},
    {"ep": 2, "tp": 4, "tokens_per_device": 16, "bytes_per_token": 1024, "alpha": 1e-5, "beta": 1e9, "num_experts": 4,
     "seed": 909},
    {"ep": 8, "tp": 1, "tokens_per_device": 32, "bytes_per_token": 8192, "alpha": 1e-5, "beta": 9e11,
     "num_experts": 64, "seed": 3},
    {"ep": 3, "tp": 3, "tokens_per_device": 5, "bytes_per_token": 777, "alpha": 0.0, "beta": 1e6, "num_experts": 9,
     "seed": 12345},
]
SIZES = [512, 2048, 8192, 32768, 131072]


def main():
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libdsmoe_ref.so"))
    L.dsmoe_sim_comm.argtypes = [C.c_char_p, C.POINTER(C.c_char_p)]
    L.dsmoe_sim_comm_sweep.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.c_size_t, C.POINTER(C.c_char_p),
                                       C.POINTER(C.c_char_p)]
    L.dsmoe_string_free.argtypes = [C.c_char_p]
    out = []
    for sc in SCENARIOS:
        js = C.c_char_p()
        assert L.dsmoe_sim_comm(json.dumps(sc).encode(), C.byref(js)) == 0
        rep = json.loads(js.value.decode())
        sizes = (C.c_int64 * len(SIZES))(*SIZES)
        sw, csv = C.c_char_p(), C.c_char_p()
        assert L.dsmoe_sim_comm_sweep(json.dumps(sc).encode(), sizes, len(SIZES), C.byref(sw), C.byref(csv)) == 0
        out.append({"scenario": sc, "report": rep, "sweep_sizes": SIZES, "sweep": json.loads(sw.value.decode())})
    path = os.path.join(ROOT, "tests", "golden", "comm_reference.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(path, len(out))


if __name__ == "__main__":
    main()
