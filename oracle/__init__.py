"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Python face of two CPU oracles for the DualSparse-MoE forward path:

* ``liboracle.so`` — the C restatement in ``dsmoe_oracle.c`` (always built);
* ``_ref/libdsmoe_refshim.so`` / ``_ref/libdsmoe_ref.so`` — the reference
  itself (``/root/reference/proj``) compiled from its own sources by
  ``oracle/Makefile`` (present whenever it was built in the container; the
  built ``.so`` files travel to the GPU box, the sources do not).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

KIND = {"none": 0, "1t": 1, "2t": 2}
METRIC = {"gate": 0, "abs_gate": 1, "gate_up": 2, "abs_gate_up": 3}
LINEAGE = {"base": 0, "complete": 1, "partial": 2, "reconstructed": 3}


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _LIB = C.CDLL(path)
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libdsmoe_refshim.so"))


def ref():
    global _REF
    if _REF is None:
        _REF = C.CDLL(os.path.join(HERE, "_ref", "libdsmoe_refshim.so"))
        _REF.refshim_last_error.restype = C.c_char_p
    return _REF


def _chk(code, who="oracle"):
    if code != 0:
        msg = ref().refshim_last_error().decode() if who == "ref" else ""
        raise OracleError(code, msg)


def _ptrs(arrs):
    return (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])


# --------------------------------------------------------------------------- layer


@dataclass
class Layer:
    """A MoE layer in the reference's host layout (moe.hpp:39-45, :73-120):
    w1/w3 are d x width, w2 is width x d, gate d x E, all row-major fp32.
    ``blocks[e*P + p]`` is slice p of original expert e."""

    d: int
    ffn: int
    E: int
    K: int
    gate: np.ndarray
    blocks: list  # [(w1, w3, w2)]
    shared: list = field(default_factory=list)
    P: int = 1
    lineage: str = "base"
    prenorm: bool = False
    neuron_order: np.ndarray | None = None  # E x ffn int32

    @property
    def S(self):
        return len(self.shared)

    @property
    def widths(self):
        return np.array([b[0].shape[1] for b in self.blocks], np.int32)

    @property
    def shared_widths(self):
        return np.array([s[0].shape[1] for s in self.shared] or [0], np.int32)

    def flat(self) -> np.ndarray:
        parts = [self.gate.ravel()]
        for w1, w3, w2 in self.blocks + self.shared:
            parts += [w1.ravel(), w3.ravel(), w2.ravel()]
        return np.ascontiguousarray(np.concatenate(parts), np.float32)

    def round_bf16(self) -> "Layer":
        """bf16 round-to-nearest-even of every weight, kept as fp32 — what the
        oracle consumes for the bf16 configs."""
        r = bf16_round
        return Layer(self.d, self.ffn, self.E, self.K, r(self.gate),
                     [(r(a), r(b), r(c)) for a, b, c in self.blocks],
                     [(r(a), r(b), r(c)) for a, b, c in self.shared],
                     self.P, self.lineage, self.prenorm, self.neuron_order)


def bf16_round(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    nan = np.isnan(a)
    out = rounded.astype(np.uint32).view(np.float32).copy()
    out[nan] = a[nan]
    return out.reshape(a.shape)


def layer_from_flat(flat, d, ffn, E, K, S=0, P=1, widths=None, shared_widths=None, **kw) -> Layer:
    widths = list(widths) if widths is not None else [ffn // P] * (E * P)
    shared_widths = list(shared_widths) if shared_widths is not None else [ffn] * S
    off = 0

    def take(r, c):
        nonlocal off
        a = flat[off:off + r * c].reshape(r, c)
        off += r * c
        return a

    gate = take(d, E)
    blocks = [(take(d, w), take(d, w), take(w, d)) for w in widths]
    shared = [(take(d, w), take(d, w), take(w, d)) for w in shared_widths[:S]]
    return Layer(d, ffn, E, K, gate, blocks, shared, P, **kw)


def generate_layer(d, ffn, E, K, S=0, seed=1234, scale=1.0) -> Layer:
    """generate_synthetic<float> (io.cpp:330) restated."""
    n = d * E + (E + S) * 3 * d * ffn
    flat = np.empty(n, np.float32)
    L = lib()
    L.orc_generate_layer.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, f32p]
    _chk(L.orc_generate_layer(d, ffn, E, S, seed, scale, flat))
    return layer_from_flat(flat, d, ffn, E, K, S)


def generate_tokens(rows, cols, seed=99, scale=1.0) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    L = lib()
    L.orc_generate_tokens.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_double, f32p]
    _chk(L.orc_generate_tokens(rows, cols, seed, scale, out))
    return out


def splitmix_nth(seed, n):
    L = lib()
    L.orc_splitmix_nth.restype = C.c_uint64
    L.orc_splitmix_nth.argtypes = [C.c_uint64, C.c_int]
    return int(L.orc_splitmix_nth(seed, n))


# ------------------------------------------------------------------------- routing


@dataclass
class Routing:
    """RoutingDecision (moe.hpp:142-167) as numpy arrays, T x (K*P)."""

    idx: np.ndarray
    raw: np.ndarray
    norm: np.ndarray
    frac: np.ndarray
    pre_frac: np.ndarray
    K: int
    P: int


def gate_logits(x, gate) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    gate = np.ascontiguousarray(gate, np.float32)
    T, d = x.shape
    E = gate.shape[1]
    out = np.empty((T, E), np.float32)
    L = lib()
    L.orc_gate_logits.argtypes = [f32p, f32p, C.c_int, C.c_int, C.c_int, f32p]
    L.orc_gate_logits(x, gate, T, d, E, out)
    return out


def route_from_logits(logits, K, P=1, kind="none", t_drop=0.0, t_major=None, t_minor=None,
                      keep_top1=True, normalize=True, t_major_slot=None, t_minor_slot=None) -> Routing:
    logits = np.ascontiguousarray(logits, np.float32)
    T, E = logits.shape
    if kind == "2t":
        t_major = t_drop - 0.01 if t_major is None else t_major
        t_minor = t_drop + 0.01 if t_minor is None else t_minor
    t_major = 0.0 if t_major is None else t_major
    t_minor = 0.0 if t_minor is None else t_minor
    n = T * K * P
    idx = np.empty(n, np.int32)
    raw, norm, frac, pre = (np.empty(n, np.float64) for _ in range(4))
    L = lib()
    L.orc_route_from_logits.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_void_p, C.c_void_p, i32p, f64p, f64p, f64p, f64p]
    tm = None if t_major_slot is None else np.ascontiguousarray(t_major_slot, np.float64)
    tn = None if t_minor_slot is None else np.ascontiguousarray(t_minor_slot, np.float64)
    _chk(L.orc_route_from_logits(logits, T, E, K, P, KIND[kind], t_drop, t_major, t_minor,
                                 int(keep_top1), int(normalize),
                                 None if tm is None else tm.ctypes.data,
                                 None if tn is None else tn.ctypes.data,
                                 idx, raw, norm, frac, pre))
    sh = (T, K * P)
    return Routing(idx.reshape(sh), raw.reshape(sh), norm.reshape(sh), frac.reshape(sh),
                   pre.reshape(sh), K, P)


def topk(scores, K):
    """topk_route (moe.hpp:181-206) restated: (idx int32 T x K, raw f64 T x K)."""
    scores = np.ascontiguousarray(scores, np.float32)
    T, E = scores.shape
    idx = np.empty((T, K), np.int32)
    raw = np.empty((T, K), np.float64)
    L = lib()
    L.orc_topk.argtypes = [f32p, C.c_int, C.c_int, C.c_int, i32p, f64p]
    _chk(L.orc_topk(scores, T, E, K, idx, raw))
    return idx, raw


def normalize(raw, K, P=1):
    """normalize_topk (dropping.hpp:60-72) on copy-major T x K*P raw scores."""
    raw = np.ascontiguousarray(raw, np.float64)
    T = raw.shape[0]
    out = np.empty_like(raw)
    L = lib()
    L.orc_normalize.argtypes = [f64p, C.c_int, C.c_int, C.c_int, f64p]
    _chk(L.orc_normalize(raw, T, K, P, out))
    return out


def apply_bands(norm, K, P, t_major, t_minor, keep_top1=True):
    """apply_bands_fn (dropping.hpp:93-122) on copy-major T x K*P scores."""
    norm = np.ascontiguousarray(norm, np.float64)
    T = norm.shape[0]
    frac = np.ones_like(norm)
    L = lib()
    L.orc_apply_bands.argtypes = [f64p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p,
                                  C.c_void_p, C.c_int, f64p]
    L.orc_apply_bands(norm, T, K, P, t_major, t_minor, None, None, int(keep_top1), frac)
    return frac


def permutation(idx, frac, K, P, E):
    """Canonical token permutation (the reference has
    none): a CPU counting sort over a canonical RoutingDecision.  Selection
    (t, s) of original expert e = idx[t, s] // P has level 2 (every copy kept /
    fraction 1 on P=1), 1 (copy 0 only / fraction 0.5) or 0 (dropped).  Rows:
    experts ascending; inside, level-2 rows then level-1 rows, (t, s)
    ascending.  Returns (row_token, slot_pos T x K, seg E x 3)."""
    idx = np.asarray(idx).reshape(-1, K * P)
    frac = np.asarray(frac, np.float64).reshape(-1, K * P)
    T = idx.shape[0]
    unit = idx[:, :K] // P
    if P == 1:
        lvl = np.where(frac == 1.0, 2, np.where(frac == 0.5, 1, 0))
    else:
        lvl = np.where(frac[:, :K] == 0, 0, np.where(frac[:, K:2 * K] == 1.0, 2, 1))
    rows, seg = [], np.zeros((E, 3), np.int32)
    slot_pos = np.full((T, K), -1, np.int32)
    for e in range(E):
        seg[e, 0] = len(rows)
        for want in (2, 1):
            ts, ss = np.nonzero((unit == e) & (lvl == want))  # row-major = (t, s) ascending
            for t, s in zip(ts, ss):
                slot_pos[t, s] = len(rows)
                rows.append(t)
            if want == 2:
                seg[e, 1] = len(rows) - seg[e, 0]
        seg[e, 2] = len(rows) - seg[e, 0]
    return np.array(rows, np.int32), slot_pos, seg


def drop_stats(pre_frac, post_frac, P, S, T, d, ffn) -> dict:
    pre = np.ascontiguousarray(pre_frac, np.float64).ravel()
    post = np.ascontiguousarray(post_frac, np.float64).ravel()
    out = np.empty(7, np.float64)
    L = lib()
    L.orc_drop_stats.argtypes = [f64p, f64p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int,
                                 C.c_int, f64p]
    L.orc_drop_stats(pre, post, pre.size, P, S, T, d, ffn, out)
    keys = ["total_routed_units", "dropped_units", "shared_units", "drop_rate", "total_flops",
            "saved_flops", "retained_flops"]
    return dict(zip(keys, out.tolist()))


def moe_forward(layer: Layer, x, idx, raw, frac, threads: int = 1) -> np.ndarray:
    """moe_forward (moe.hpp:239-271).  threads > 1 shards the tokens into
    contiguous blocks run concurrently (ctypes drops the GIL): the forward is
    per-token separable (moe.hpp:253-269), so the result is bit-identical to
    one call."""
    x = np.ascontiguousarray(x, np.float32)
    T, d = x.shape
    if threads > 1 and T > 1:
        import concurrent.futures as cf
        idx2 = np.asarray(idx).reshape(T, -1)
        raw2 = np.asarray(raw).reshape(T, -1)
        frac2 = np.asarray(frac).reshape(T, -1)
        parts = [p for p in np.array_split(np.arange(T), min(threads, T)) if p.size]
        with cf.ThreadPoolExecutor(len(parts)) as ex:
            outs = list(ex.map(lambda p: moe_forward(layer, x[p], idx2[p], raw2[p], frac2[p]), parts))
        return np.concatenate(outs, axis=0)
    idx = np.ascontiguousarray(idx, np.int32)
    raw = np.ascontiguousarray(raw, np.float64)
    frac = np.ascontiguousarray(frac, np.float64)
    kslots = idx.shape[1] if idx.ndim == 2 else idx.size // max(T, 1)
    b = [tuple(np.ascontiguousarray(m, np.float32) for m in blk) for blk in layer.blocks]
    s = [tuple(np.ascontiguousarray(m, np.float32) for m in blk) for blk in layer.shared]
    out = np.empty((T, d), np.float32)
    L = lib()
    L.orc_moe_forward.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, i32p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                  i32p, i32p, f64p, f64p, f32p]
    _chk(L.orc_moe_forward(x, T, d, len(b), kslots, _ptrs([q[0] for q in b]),
                           _ptrs([q[1] for q in b]), _ptrs([q[2] for q in b]), layer.widths,
                           len(s), _ptrs([q[0] for q in s]), _ptrs([q[1] for q in s]),
                           _ptrs([q[2] for q in s]), layer.shared_widths, idx, raw, frac, out))
    return out


def route(layer: Layer, x, kind="none", t_drop=0.0, **kw) -> Routing:
    """route_and_drop (dropping.hpp:248) restated: logits, then routing."""
    lg = gate_logits(x, layer.gate)
    return route_from_logits(lg, layer.K, layer.P, kind, t_drop,
                             normalize=kw.pop("normalize", not layer.prenorm), **kw)


def profile_importance(layer: Layer, x, idx, metric="abs_gate") -> np.ndarray:
    assert layer.P == 1
    x = np.ascontiguousarray(x, np.float32)
    T, d = x.shape
    idx = np.ascontiguousarray(idx, np.int32)
    b = [tuple(np.ascontiguousarray(m, np.float32) for m in blk) for blk in layer.blocks]
    vals = np.empty((layer.E, layer.ffn), np.float64)
    L = lib()
    L.orc_profile_importance.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p, i32p, C.c_int, f64p]
    _chk(L.orc_profile_importance(x, T, d, layer.E, layer.ffn, layer.K, _ptrs([q[0] for q in b]),
                                  _ptrs([q[1] for q in b]), idx, METRIC[metric], vals))
    return vals


def reconstruction_order(values) -> np.ndarray:
    values = np.ascontiguousarray(values, np.float64)
    E, ffn = values.shape
    order = np.empty((E, ffn), np.int32)
    L = lib()
    L.orc_reconstruction_order.argtypes = [f64p, C.c_int, C.c_int, i32p]
    L.orc_reconstruction_order(values, E, ffn, order)
    return order


def reconstruct(layer: Layer, values) -> Layer:
    """reconstruct_experts (reconstruct.hpp:196-230): permute W1/W3 columns and
    W2 rows by the order, split at ceil(ffn/2), no scaling."""
    order = reconstruction_order(values)
    major = (layer.ffn + 1) // 2
    blocks = []
    for e, (w1, w3, w2) in enumerate(layer.blocks):
        o = order[e]
        p1, p3, p2 = w1[:, o], w3[:, o], w2[o, :]
        blocks.append((np.ascontiguousarray(p1[:, :major]), np.ascontiguousarray(p3[:, :major]),
                       np.ascontiguousarray(p2[:major])))
        blocks.append((np.ascontiguousarray(p1[:, major:]), np.ascontiguousarray(p3[:, major:]),
                       np.ascontiguousarray(p2[major:])))
    return Layer(layer.d, layer.ffn, layer.E, layer.K, layer.gate, blocks, layer.shared, 2,
                 "reconstructed", layer.prenorm, order)


def partial_transform(layer: Layer, p: int) -> Layer:
    """transform.hpp:100-131: contiguous unscaled slices, gate unchanged."""
    c = layer.ffn // p
    blocks = []
    for w1, w3, w2 in layer.blocks:
        for q in range(p):
            sl = slice(q * c, (q + 1) * c)
            blocks.append((np.ascontiguousarray(w1[:, sl]), np.ascontiguousarray(w3[:, sl]),
                           np.ascontiguousarray(w2[sl])))
    return Layer(layer.d, layer.ffn, layer.E, layer.K, layer.gate, blocks, layer.shared, p,
                 "partial", layer.prenorm)


def complete_transform(layer: Layer, p: int) -> Layer:
    """transform.hpp:66-95: gate columns repeated p times, W2 scaled by p,
    E*p experts of width ffn/p, top-(K*p)."""
    c = layer.ffn // p
    gate = np.ascontiguousarray(np.repeat(layer.gate, p, axis=1))
    blocks = []
    for w1, w3, w2 in layer.blocks:
        for q in range(p):
            sl = slice(q * c, (q + 1) * c)
            blocks.append((np.ascontiguousarray(w1[:, sl]), np.ascontiguousarray(w3[:, sl]),
                           np.ascontiguousarray(w2[sl] * np.float32(p))))
    return Layer(layer.d, c, layer.E * p, layer.K * p, gate, blocks, layer.shared, 1, "complete",
                 layer.prenorm)


# ------------------------------------------------------------------------------ EP


def place_experts(n, devices, round_robin=False) -> np.ndarray:
    out = np.empty(n, np.int32)
    L = lib()
    L.orc_place_experts.argtypes = [C.c_int, C.c_int, C.c_int, i32p]
    _chk(L.orc_place_experts(n, devices, int(round_robin), out))
    return out


def load_aware_thresholds(loads, t_max) -> np.ndarray:
    loads = np.ascontiguousarray(loads, np.float64)
    out = np.empty_like(loads)
    L = lib()
    L.orc_load_aware_thresholds.argtypes = [f64p, C.c_int, C.c_double, f64p]
    _chk(L.orc_load_aware_thresholds(loads, loads.size, t_max, out))
    return out


def device_loads(idx, frac, P, device_of, D) -> np.ndarray:
    idx = np.ascontiguousarray(idx, np.int32).ravel()
    frac = np.ascontiguousarray(frac, np.float64).ravel()
    out = np.empty(D, np.float64)
    L = lib()
    L.orc_device_loads.argtypes = [i32p, f64p, C.c_int64, C.c_int, i32p, C.c_int, f64p]
    L.orc_device_loads(idx, frac, idx.size, P, np.ascontiguousarray(device_of, np.int32), D, out)
    return out


def simulate_step(logits, layer: Layer, devices, kind="1t", t_drop=0.1, round_robin=False,
                  load_aware=True, keep_top1=True, normalize=True, t_major=None, t_minor=None):
    logits = np.ascontiguousarray(logits, np.float32)
    T, E = logits.shape
    if kind == "2t":
        t_major = t_drop - 0.01 if t_major is None else t_major
        t_minor = t_drop + 0.01 if t_minor is None else t_minor
    t_major = 0.0 if t_major is None else t_major
    t_minor = 0.0 if t_minor is None else t_minor
    n = T * layer.K * layer.P
    pre_l, post_l, th = (np.empty(devices, np.float64) for _ in range(3))
    rep = np.empty(5, np.float64)
    idx = np.empty(n, np.int32)
    frac = np.empty(n, np.float64)
    L = lib()
    L.orc_simulate_step.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_int, C.c_int, C.c_int, f64p, f64p, f64p, f64p,
                                    i32p, f64p]
    _chk(L.orc_simulate_step(logits, T, E, layer.K, layer.P, layer.S, layer.d, layer.ffn, devices,
                             int(round_robin), KIND[kind], t_drop, t_major, t_minor,
                             int(keep_top1), int(normalize), int(load_aware), pre_l, post_l, th,
                             rep, idx, frac))
    sh = (T, layer.K * layer.P)
    return dict(pre_loads=pre_l, post_loads=post_l, thresholds=th, ideal_load=rep[0],
                drop_rate=rep[1], speedup=rep[2], total_routed_units=rep[3],
                dropped_units=rep[4], idx=idx.reshape(sh), frac=frac.reshape(sh))


# ------------------------------------------------------------- the reference itself


class RefLayer:
    """A reference MoeLayer<float> handle (oracle/_ref/libdsmoe_refshim.so)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    @classmethod
    def from_layer(cls, layer: Layer) -> "RefLayer":
        R = ref()
        R.refshim_layer_create.argtypes = [C.c_int] * 8 + [i32p, i32p, f32p, C.c_void_p,
                                                          C.POINTER(C.c_void_p)]
        out = C.c_void_p()
        no = None if layer.neuron_order is None else np.ascontiguousarray(layer.neuron_order, np.int32)
        _chk(R.refshim_layer_create(layer.d, layer.ffn, layer.E, layer.K, layer.S,
                                    int(layer.prenorm), layer.P, LINEAGE[layer.lineage],
                                    layer.widths, layer.shared_widths, layer.flat(),
                                    None if no is None else no.ctypes.data, C.byref(out)), "ref")
        return cls(out.value)

    @classmethod
    def generate(cls, d, ffn, E, K, S=0, seed=1234, scale=1.0, prenorm=False) -> "RefLayer":
        R = ref()
        R.refshim_generate_layer.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_double,
                                                             C.POINTER(C.c_void_p)]
        out = C.c_void_p()
        _chk(R.refshim_generate_layer(d, ffn, E, K, S, int(prenorm), seed, scale, C.byref(out)),
             "ref")
        return cls(out.value)

    def __del__(self):
        try:
            ref().refshim_layer_free(self.h)
        except Exception:
            pass

    def to_layer(self) -> Layer:
        R = ref()
        info = np.empty(8, np.int64)
        R.refshim_layer_info.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.int64)]
        _chk(R.refshim_layer_info(self.h, info), "ref")
        d, ffn, E, K, S, P, lin, n = (int(v) for v in info)
        flat = np.empty(n, np.float32)
        widths = np.empty(E * P, np.int32)
        sw = np.empty(max(S, 1), np.int32)
        order = np.full(E * ffn, -1, np.int32)
        R.refshim_layer_export.argtypes = [C.c_void_p, f32p, i32p, i32p, i32p]
        _chk(R.refshim_layer_export(self.h, flat, widths, sw, order), "ref")
        lineage = {v: k for k, v in LINEAGE.items()}[lin]
        no = order.reshape(E, ffn) if order[0] >= 0 else None
        return layer_from_flat(flat, d, ffn, E, K, S, P, widths, sw, lineage=lineage,
                               neuron_order=no)

    def gate_logits(self, x, E):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty((x.shape[0], E), np.float32)
        R = ref()
        R.refshim_gate_logits.argtypes = [C.c_void_p, f32p, C.c_int, f32p]
        _chk(R.refshim_gate_logits(self.h, x, x.shape[0], out), "ref")
        return out

    def route_and_drop(self, x, K, P, kind="none", t_drop=0.0, t_major=None, t_minor=None,
                       keep_top1=True, normalize=True) -> Routing:
        x = np.ascontiguousarray(x, np.float32)
        T = x.shape[0]
        if kind == "2t":
            t_major = t_drop - 0.01 if t_major is None else t_major
            t_minor = t_drop + 0.01 if t_minor is None else t_minor
        n = T * K * P
        idx = np.empty(n, np.int32)
        raw, norm, frac, pre = (np.empty(n, np.float64) for _ in range(4))
        R = ref()
        R.refshim_route_and_drop.argtypes = [C.c_void_p, f32p, C.c_int, C.c_int, C.c_double,
                                             C.c_double, C.c_double, C.c_int, C.c_int, i32p, f64p,
                                             f64p, f64p, f64p]
        _chk(R.refshim_route_and_drop(self.h, x, T, KIND[kind], t_drop, t_major or 0.0,
                                      t_minor or 0.0, int(keep_top1), int(normalize), idx, raw,
                                      norm, frac, pre), "ref")
        sh = (T, K * P)
        return Routing(idx.reshape(sh), raw.reshape(sh), norm.reshape(sh), frac.reshape(sh),
                       pre.reshape(sh), K, P)

    def moe_forward(self, x, idx, raw, frac, threads=1) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        R = ref()
        R.refshim_moe_forward.argtypes = [C.c_void_p, f32p, C.c_int, i32p, f64p, f64p, f32p, C.c_int]
        _chk(R.refshim_moe_forward(self.h, x, x.shape[0], np.ascontiguousarray(idx, np.int32),
                                   np.ascontiguousarray(raw, np.float64),
                                   np.ascontiguousarray(frac, np.float64), out, threads), "ref")
        return out

    def drop_stats(self, T, pre_frac, post_frac) -> dict:
        out = np.empty(7, np.float64)
        R = ref()
        R.refshim_drop_stats.argtypes = [C.c_void_p, C.c_int, f64p, f64p, f64p]
        _chk(R.refshim_drop_stats(self.h, T, np.ascontiguousarray(pre_frac, np.float64).ravel(),
                                  np.ascontiguousarray(post_frac, np.float64).ravel(), out), "ref")
        keys = ["total_routed_units", "dropped_units", "shared_units", "drop_rate", "total_flops",
                "saved_flops", "retained_flops"]
        return dict(zip(keys, out.tolist()))

    def profile_importance(self, x, idx, E, ffn, metric="abs_gate"):
        x = np.ascontiguousarray(x, np.float32)
        vals = np.empty((E, ffn), np.float64)
        R = ref()
        R.refshim_profile_importance.argtypes = [C.c_void_p, f32p, C.c_int, i32p, C.c_int, f64p]
        _chk(R.refshim_profile_importance(self.h, x, x.shape[0], np.ascontiguousarray(idx, np.int32),
                                          METRIC[metric], vals), "ref")
        return vals

    def reconstruct(self, values, E, ffn, metric="abs_gate"):
        out = C.c_void_p()
        order = np.empty((E, ffn), np.int32)
        R = ref()
        R.refshim_reconstruct.argtypes = [C.c_void_p, f64p, C.c_int, C.POINTER(C.c_void_p), i32p]
        _chk(R.refshim_reconstruct(self.h, np.ascontiguousarray(values, np.float64),
                                   METRIC[metric], C.byref(out), order), "ref")
        return RefLayer(out.value), order

    def transform(self, complete: bool, p: int) -> "RefLayer":
        out = C.c_void_p()
        R = ref()
        R.refshim_transform.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        _chk(R.refshim_transform(self.h, int(complete), p, C.byref(out)), "ref")
        return RefLayer(out.value)

    def simulate_step(self, x, devices, K, P, kind="1t", t_drop=0.1, round_robin=False,
                      load_aware=True, keep_top1=True, normalize=True, t_major=None, t_minor=None):
        x = np.ascontiguousarray(x, np.float32)
        T = x.shape[0]
        if kind == "2t":
            t_major = t_drop - 0.01 if t_major is None else t_major
            t_minor = t_drop + 0.01 if t_minor is None else t_minor
        n = T * K * P
        pre_l, post_l, th = (np.empty(devices, np.float64) for _ in range(3))
        rep = np.empty(5, np.float64)
        idx = np.empty(n, np.int32)
        frac = np.empty(n, np.float64)
        R = ref()
        R.refshim_simulate_step.argtypes = [C.c_void_p, f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                            C.c_int, f64p, f64p, f64p, f64p, i32p, f64p]
        _chk(R.refshim_simulate_step(self.h, x, T, devices, int(round_robin), KIND[kind], t_drop,
                                     t_major or 0.0, t_minor or 0.0, int(keep_top1),
                                     int(normalize), int(load_aware), pre_l, post_l, th, rep, idx,
                                     frac), "ref")
        sh = (T, K * P)
        return dict(pre_loads=pre_l, post_loads=post_l, thresholds=th, ideal_load=rep[0],
                    drop_rate=rep[1], speedup=rep[2], total_routed_units=rep[3],
                    dropped_units=rep[4], idx=idx.reshape(sh), frac=frac.reshape(sh))


def ref_load_aware_thresholds(loads, t_max):
    loads = np.ascontiguousarray(loads, np.float64)
    out = np.empty_like(loads)
    R = ref()
    R.refshim_load_aware_thresholds.argtypes = [f64p, C.c_int, C.c_double, f64p]
    _chk(R.refshim_load_aware_thresholds(loads, loads.size, t_max, out), "ref")
    return out


def ref_generate_tokens(rows, cols, seed=99, scale=1.0):
    out = np.empty((rows, cols), np.float32)
    R = ref()
    R.refshim_generate_tokens.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_double, f32p]
    _chk(R.refshim_generate_tokens(rows, cols, seed, scale, out), "ref")
    return out
