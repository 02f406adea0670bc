"""ctypes binding of the reference's C interface (include/dsmoe_abi.h; the
reference's include/dsmoe.h), as a caller of either library would write it.

    lib = DsmoeAbi()                              # libdsmoe_b200.so (the B200 device path)
    lib = DsmoeAbi("oracle/_ref/libdsmoe_ref.so")  # the reference, same calls

Every call raises AbiError(code, message) on a non-zero status (the
DSMOE_E_* codes, dsmoe.h:16-24); output strings are copied and released
with dsmoe_string_free, models with dsmoe_model_free.
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(HERE, "libdsmoe_b200.so")

_SIGS = {
    "dsmoe_version": (C.c_char_p, []),
    "dsmoe_status_name": (C.c_char_p, [C.c_int]),
    "dsmoe_last_error": (C.c_char_p, []),
    "dsmoe_string_free": (None, [C.c_void_p]),
    "dsmoe_model_free": (None, [C.c_void_p]),
    "dsmoe_generate_model": (C.c_int, [C.c_char_p, C.c_uint64, C.c_double, C.c_int, C.POINTER(C.c_void_p)]),
    "dsmoe_generate_tokens": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.c_double, C.c_char_p]),
    "dsmoe_model_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "dsmoe_model_save": (C.c_int, [C.c_void_p, C.c_char_p]),
    "dsmoe_model_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "dsmoe_transform": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "dsmoe_reverse_partial": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "dsmoe_reconstruct": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_void_p)]),
    "dsmoe_verify_equivalence": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_double,
                                           C.POINTER(C.c_void_p)]),
    "dsmoe_infer": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "dsmoe_sweep": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_double), C.c_size_t, C.c_int,
                              C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "dsmoe_analyze_gating": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p)]),
    "dsmoe_sim_ep": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_char_p, C.c_char_p, C.c_int,
                               C.POINTER(C.c_void_p)]),
    "dsmoe_sim_comm": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "dsmoe_sim_comm_sweep": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.c_size_t, C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p)]),
}
SYMBOLS = tuple(_SIGS)


class AbiError(RuntimeError):
    def __init__(self, code: int, msg: str, status: str = ""):
        super().__init__(f"[{status or code}] {msg}")
        self.code = code
        self.status = status


class Model:
    """A dsmoe_model handle owned by one library."""

    def __init__(self, lib: "DsmoeAbi", h):
        self.lib, self.h = lib, h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.dsmoe_model_free(self.h)
            self.h = None


def _b(s):
    return None if s is None else (s.encode() if isinstance(s, str) else s)


class DsmoeAbi:
    def __init__(self, path: str | None = None):
        self.path = path or DEFAULT_LIB
        if not os.path.exists(self.path):
            raise ImportError(f"{self.path} missing")
        self.L = C.CDLL(self.path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.L, name)
            fn.restype, fn.argtypes = res, args

    # ---- plumbing
    def _chk(self, rc):
        if rc != 0:
            raise AbiError(rc, self.L.dsmoe_last_error().decode(), self.L.dsmoe_status_name(rc).decode())

    def _take(self, p):
        if not p.value:
            return None
        s = C.cast(p, C.c_char_p).value.decode()
        self.L.dsmoe_string_free(p)
        return s

    def version(self):
        return self.L.dsmoe_version().decode()

    def status_name(self, code):
        return self.L.dsmoe_status_name(code).decode()

    def last_error(self):
        return self.L.dsmoe_last_error().decode()

    # ---- models and files
    def generate_model(self, config: dict | str, seed=1234, scale=1.0, scalar_width=4) -> Model:
        h = C.c_void_p()
        doc = config if isinstance(config, str) else json.dumps(config)
        self._chk(self.L.dsmoe_generate_model(_b(doc), seed, scale, scalar_width, C.byref(h)))
        return Model(self, h)

    def generate_tokens(self, rows, cols, seed, path, scale=1.0):
        self._chk(self.L.dsmoe_generate_tokens(rows, cols, seed, scale, _b(path)))

    def load(self, path) -> Model:
        h = C.c_void_p()
        self._chk(self.L.dsmoe_model_load(_b(path), C.byref(h)))
        return Model(self, h)

    def save(self, m: Model, path):
        self._chk(self.L.dsmoe_model_save(m.h, _b(path)))

    def info(self, m: Model) -> dict:
        p = C.c_void_p()
        self._chk(self.L.dsmoe_model_info(m.h, C.byref(p)))
        return json.loads(self._take(p))

    # ---- partition API
    def transform(self, m: Model, mode: str, p: int) -> Model:
        h = C.c_void_p()
        self._chk(self.L.dsmoe_transform(m.h, _b(mode), p, C.byref(h)))
        return Model(self, h)

    def reverse_partial(self, m: Model) -> Model:
        h = C.c_void_p()
        self._chk(self.L.dsmoe_reverse_partial(m.h, C.byref(h)))
        return Model(self, h)

    def reconstruct(self, m: Model, tokens_path, metric="abs_gate"):
        h, p = C.c_void_p(), C.c_void_p()
        self._chk(self.L.dsmoe_reconstruct(m.h, _b(tokens_path), _b(metric), C.byref(h), C.byref(p)))
        return Model(self, h), json.loads(self._take(p))

    def verify_equivalence(self, a: Model, b: Model, tokens_path, tol) -> dict:
        p = C.c_void_p()
        self._chk(self.L.dsmoe_verify_equivalence(a.h, b.h, _b(tokens_path), tol, C.byref(p)))
        return json.loads(self._take(p))

    # ---- forward with drop
    def infer(self, m: Model, tokens_path, policy: dict | str) -> dict:
        p = C.c_void_p()
        doc = policy if isinstance(policy, str) else json.dumps(policy)
        self._chk(self.L.dsmoe_infer(m.h, _b(tokens_path), _b(doc), C.byref(p)))
        return json.loads(self._take(p))

    def sweep(self, m: Model, tokens_path, kind, thresholds, keep_top1=True):
        arr = (C.c_double * len(thresholds))(*thresholds)
        pj, pc = C.c_void_p(), C.c_void_p()
        self._chk(self.L.dsmoe_sweep(m.h, _b(tokens_path), _b(kind), arr, len(thresholds), int(keep_top1),
                                     C.byref(pj), C.byref(pc)))
        return json.loads(self._take(pj)), self._take(pc)

    def analyze_gating(self, m: Model, tokens_path, bins=10):
        pj, pc = C.c_void_p(), C.c_void_p()
        self._chk(self.L.dsmoe_analyze_gating(m.h, _b(tokens_path), bins, C.byref(pj), C.byref(pc)))
        return json.loads(self._take(pj)), self._take(pc)

    def sim_ep(self, m: Model, tokens_path, devices, strategy, policy: dict | str, load_aware=True) -> dict:
        p = C.c_void_p()
        doc = policy if isinstance(policy, str) else json.dumps(policy)
        self._chk(self.L.dsmoe_sim_ep(m.h, _b(tokens_path), devices, _b(strategy), _b(doc), int(load_aware),
                                      C.byref(p)))
        return json.loads(self._take(p))

    def sim_comm(self, scenario: dict | str) -> dict:
        p = C.c_void_p()
        doc = scenario if isinstance(scenario, str) else json.dumps(scenario)
        self._chk(self.L.dsmoe_sim_comm(_b(doc), C.byref(p)))
        return json.loads(self._take(p))
