"""Host-side mirror of the reference's partition / drop-policy / forward API
over the C ABI of libdsmoe_b200.so (include/dsmoe_b200.h).

Names, argument meaning and error behaviour follow the reference's C++ layer
(/root/reference/proj/include/dsmoe/*.hpp):

    DropPolicy            dropping.hpp:12-56
    RoutingDecision       moe.hpp:142-167
    MoeLayer              moe.hpp:73-120   (device-resident, packed)
    route_and_drop        dropping.hpp:248
    moe_forward           moe.hpp:239
    drop_stats            dropping.hpp:171
    load_aware_thresholds ep_sim.hpp:76
    place_experts / device_loads   ep_sim.hpp:38 / :59

Failures raise DsmoeError carrying the reference status code
(error.hpp:10-20).  There is no CPU fallback: every compute call goes through
the CUDA library, and importing this module on a machine without the built
library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdsmoe_b200.so")

F32, BF16 = 0, 1
KIND = {"none": 0, "1t": 1, "2t": 2}
METRIC = {"gate": 0, "abs_gate": 1, "gate_up": 2, "abs_gate_up": 3}
LOGITS_TENSOR, LOGITS_EXACT, LOGITS_REUSE = 0, 1, 2
STATUS = {0: "ok", 1: "invalid_argument", 2: "shape_mismatch", 3: "invalid_state", 4: "io_error",
          5: "bad_magic", 6: "truncated", 7: "schema_error", 8: "internal"}


class DsmoeError(RuntimeError):
    """dsmoe::Error (error.hpp:37-44): a status code plus message."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{STATUS.get(code, code)}] {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class LayerConfig(C.Structure):
    _fields_ = [("d_model", C.c_int), ("d_ffn", C.c_int), ("num_experts", C.c_int), ("top_k", C.c_int),
                ("num_shared_experts", C.c_int), ("gate_prenormalized", C.c_int),
                ("replay_factor", C.c_int), ("dtype", C.c_int),
                ("block_widths", C.POINTER(C.c_int32)), ("shared_widths", C.POINTER(C.c_int32))]


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int), ("t_drop", C.c_double), ("t_major", C.c_double),
                ("t_minor", C.c_double), ("keep_top1", C.c_int), ("normalize", C.c_int),
                ("t_unit", C.c_void_p)]


class RoutingOut(C.Structure):
    _fields_ = [("indices", C.c_void_p), ("raw", C.c_void_p), ("normalized", C.c_void_p),
                ("fraction", C.c_void_p)]


class DropStatsC(C.Structure):
    _fields_ = [("num_tokens", C.c_long), ("total_routed_units", C.c_double),
                ("dropped_units", C.c_double), ("shared_units", C.c_double), ("drop_rate", C.c_double),
                ("total_flops", C.c_double), ("saved_flops", C.c_double),
                ("retained_flops", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None

# every symbol include/dsmoe_b200.h declares (tests check the export table)
SYMBOLS = {
    "dsmoe_b200_version": (C.c_char_p, []),
    "dsmoe_b200_last_error": (C.c_char_p, []),
    "dsmoe_b200_last_launch_count": (C.c_int, []),
    "dsmoe_b200_total_launch_count": (C.c_longlong, []),
    "dsmoe_b200_layer_create": (C.c_int, [C.POINTER(LayerConfig), C.POINTER(C.c_void_p)]),
    "dsmoe_b200_layer_free": (None, [C.c_void_p]),
    "dsmoe_b200_layer_set_gate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "dsmoe_b200_layer_set_block": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_int, C.c_int, C.c_void_p]),
    "dsmoe_b200_layer_set_shared": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_int, C.c_int, C.c_void_p]),
    "dsmoe_b200_layer_info": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dsmoe_b200_ctx_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "dsmoe_b200_ctx_free": (None, [C.c_void_p]),
    "dsmoe_b200_ctx_check": (C.c_int, [C.c_void_p]),
    "dsmoe_b200_ctx_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "dsmoe_b200_ctx_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_long)]),
    "dsmoe_b200_ctx_permutation": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.POINTER(C.c_int)]),
    "dsmoe_b200_route": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy), C.c_int,
                                   C.c_void_p, C.c_void_p, C.POINTER(RoutingOut), C.POINTER(DropStatsC)]),
    "dsmoe_b200_moe_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsmoe_b200_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy), C.c_int,
                                     C.c_void_p, C.POINTER(DropStatsC)]),
    "dsmoe_b200_forward_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy), C.c_int,
                                        C.c_int, C.c_void_p, C.POINTER(DropStatsC)]),
    "dsmoe_b200_dispatch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy), C.c_int,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                      C.POINTER(DropStatsC)]),
    "dsmoe_b200_expert_ffn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsmoe_b200_combine": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "dsmoe_b200_ep_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsmoe_b200_ep_expert": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_long, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "dsmoe_b200_ep_combine": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "dsmoe_b200_analyze_gating": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                            C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsmoe_b200_drop_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_long, C.c_int,
                                        C.c_int, C.POINTER(DropStatsC)]),
    "dsmoe_b200_profile_importance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                                C.c_int, C.c_void_p]),
    "dsmoe_b200_reconstruct": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_void_p)]),
    "dsmoe_b200_load_aware_thresholds": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_void_p]),
    "dsmoe_b200_simulate_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                           C.POINTER(Policy), C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.POINTER(DropStatsC), C.POINTER(RoutingOut), C.c_void_p,
                                           C.c_int]),
    "dsmoe_b200_ep_route_counts": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy),
                                             C.c_int, C.c_void_p]),
    "dsmoe_b200_ep_last_counts": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "dsmoe_b200_ep_thresholds": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_double,
                                           C.c_int, C.c_void_p, C.c_void_p]),
    "dsmoe_b200_ep_dispatch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy), C.c_int,
                                         C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    "dsmoe_b200_ctx_logits": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]),
    "dsmoe_b200_ep_expert_packed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_long, C.c_void_p, C.c_long,
                                              C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "dsmoe_b200_layer_shard": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "dsmoe_b200_layer_shard_blocks": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "dsmoe_b200_calibrate_rate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy),
                                            C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_double),
                                            C.POINTER(C.c_double)]),
    "dsmoe_b200_forward_rate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Policy), C.c_double,
                                          C.c_double, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.POINTER(DropStatsC)]),
    "dsmoe_b200_transform": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "dsmoe_b200_layer_widths": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "dsmoe_b200_layer_get_gate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "dsmoe_b200_layer_get_block": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_int]),
    "dsmoe_b200_layer_get_shared": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_int]),
}


def lib():
    """Load libdsmoe_b200.so (built in-tree by build.py).  Raises if absent:
    there is no fallback path."""
    global _lib
    if _lib is None:
        # DSMOE_B200_LIB: an alternative in-tree build of the same library
        # (tools/build_variant.sh compiles GEMM pipeline-depth variants for A/B)
        path = os.environ.get("DSMOE_B200_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run __graft_entry__.build() "
                              "(python -m paper_2508_18376_b200.build)")
        L = C.CDLL(path)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _chk(rc: int):
    if rc != 0:
        raise DsmoeError(rc, lib().dsmoe_b200_last_error().decode())


def last_launch_count() -> int:
    return int(lib().dsmoe_b200_last_launch_count())


def total_launch_count() -> int:
    """Every kernel the library launched in this process (all entry points)."""
    return int(lib().dsmoe_b200_total_launch_count())


# ----------------------------------------------------------------- torch glue
def _torch():
    import torch
    return torch


def _stream_ptr(stream=None):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _src(a):
    """(pointer, dtype code, on_device, keepalive) for a numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, np.float32)
        return a.ctypes.data, F32, 0, a
    torch = _torch()
    t = a.contiguous()
    if t.dtype == torch.bfloat16:
        dt = BF16
    else:
        t = t.float()
        dt = F32
    return t.data_ptr(), dt, int(t.is_cuda), t


# ---------------------------------------------------------------- policies
@dataclass
class DropPolicy:
    """DropPolicy (dropping.hpp:12-56)."""

    kind: str = "none"
    t_drop: float = 0.0
    t_major: float = 0.0
    t_minor: float = 0.0
    keep_top1: bool = True
    normalize: bool | None = None   # None -> !gate_prenormalized (capi.cpp:111)

    @staticmethod
    def none_policy():
        return DropPolicy()

    @staticmethod
    def one_t(t, keep_top1=True):
        return DropPolicy("1t", t, keep_top1=keep_top1)

    @staticmethod
    def two_t_from(t, keep_top1=True):
        return DropPolicy.two_t(t, t - 0.01, t + 0.01, keep_top1)

    @staticmethod
    def two_t(t, t_major, t_minor, keep_top1=True):
        if not t_major <= t_minor:
            raise DsmoeError(1, "drop policy: t_major must be <= t_minor")
        return DropPolicy("2t", t, t_major, t_minor, keep_top1)

    def c(self, t_unit=None) -> Policy:
        return Policy(KIND[self.kind], self.t_drop, self.t_major, self.t_minor, int(self.keep_top1),
                      -1 if self.normalize is None else int(self.normalize),
                      None if t_unit is None else t_unit.data_ptr())


# ------------------------------------------------------------------ layers
class MoeLayer:
    """A device-resident MoE layer (MoeLayer<T>, moe.hpp:73-120) packed for the
    grouped GEMMs.  blocks[e*P + p] = (w1, w3, w2) of slice p of expert e;
    shared = [(w1, w3, w2)]; arrays are numpy (host) or torch (host/device)."""

    def __init__(self, d_model, d_ffn, num_experts, top_k, gate, blocks, shared=(), replay_factor=1,
                 dtype="bf16", gate_prenormalized=False, stream=None):
        self.d, self.ffn, self.E, self.K = d_model, d_ffn, num_experts, top_k
        self.P = replay_factor
        self.S = len(shared)
        self.dtype = dtype
        self.prenorm = bool(gate_prenormalized)
        widths = (C.c_int32 * max(1, len(blocks)))(*[int(b[0].shape[1]) for b in blocks])
        swidths = (C.c_int32 * max(1, self.S))(*([int(s[0].shape[1]) for s in shared] or [0]))
        cfg = LayerConfig(d_model, d_ffn, num_experts, top_k, self.S, int(self.prenorm), replay_factor,
                          BF16 if dtype == "bf16" else F32, widths, swidths)
        h = C.c_void_p()
        _chk(lib().dsmoe_b200_layer_create(C.byref(cfg), C.byref(h)))
        self.h = h
        st = _stream_ptr(stream)
        p, dt, dev, keep = _src(gate)
        _chk(lib().dsmoe_b200_layer_set_gate(self.h, C.c_void_p(p), dt, dev, st))
        for b, (w1, w3, w2) in enumerate(blocks):
            a1, a3, a2 = _src(w1), _src(w3), _src(w2)
            _chk(lib().dsmoe_b200_layer_set_block(self.h, b, C.c_void_p(a1[0]), C.c_void_p(a3[0]),
                                                  C.c_void_p(a2[0]), a1[1], a1[2], st))
        for s, (w1, w3, w2) in enumerate(shared):
            a1, a3, a2 = _src(w1), _src(w3), _src(w2)
            _chk(lib().dsmoe_b200_layer_set_shared(self.h, s, C.c_void_p(a1[0]), C.c_void_p(a3[0]),
                                                   C.c_void_p(a2[0]), a1[1], a1[2], st))

    @classmethod
    def _wrap(cls, handle, like: "MoeLayer", P=None):
        """A Python handle for a layer the library created (transform,
        reconstruct): the shape is read back from the library."""
        obj = cls.__new__(cls)
        obj.__dict__.update(like.__dict__)
        obj.h = handle
        info = (C.c_int32 * 8)()
        _chk(lib().dsmoe_b200_layer_info(handle, info))
        obj.d, obj.ffn, obj.E, obj.K, obj.S, obj.P = (int(v) for v in info[:6])
        return obj

    def widths(self):
        """(block widths E*P, shared widths S) as int lists."""
        bw = (C.c_int32 * max(1, self.E * self.P))()
        sw = (C.c_int32 * max(1, self.S))()
        _chk(lib().dsmoe_b200_layer_widths(self.h, bw, sw))
        return list(bw)[:self.E * self.P], list(sw)[:self.S]

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.dsmoe_b200_layer_free(h)
            self.h = None

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32


class Context:
    """Stream + workspace (one per CUDA stream)."""

    def __init__(self, stream=None):
        h = C.c_void_p()
        _chk(lib().dsmoe_b200_ctx_create(_stream_ptr(stream), C.byref(h)))
        self.h = h

    def check(self):
        _chk(lib().dsmoe_b200_ctx_check(self.h))

    STAGES = ("gate", "router", "permute_plan", "gather", "gemm1", "gemm2", "combine")

    def set_profiling(self, on: bool, every: int = 1):
        """Per-stage CUDA events on every `every`-th forward (the others run
        without events, so their kernels keep their launch overlap)."""
        _chk(lib().dsmoe_b200_ctx_set_profiling(self.h, (max(1, int(every)) if on else 0)))

    def profile(self) -> dict:
        """Summed per-stage device milliseconds (CUDA events) since profiling
        was enabled, plus the number of profiled calls."""
        ms = (C.c_double * len(self.STAGES))()
        calls = C.c_long()
        _chk(lib().dsmoe_b200_ctx_profile(self.h, ms, len(self.STAGES), C.byref(calls)))
        out = dict(zip(self.STAGES, list(ms)))
        out["calls"] = calls.value
        return out

    def permutation(self, T: int, K: int, E: int):
        """(row_token, slot_pos T x K, seg E x 3) of the last forward (numpy)."""
        R = C.c_int()
        _chk(lib().dsmoe_b200_ctx_permutation(self.h, T, K, E, None, None, None, C.byref(R)))
        rt = np.empty(max(R.value, 1), np.int32)
        sp = np.empty(T * K, np.int32)
        sg = np.empty(3 * E, np.int32)
        _chk(lib().dsmoe_b200_ctx_permutation(self.h, T, K, E, rt.ctypes.data, sp.ctypes.data, sg.ctypes.data,
                                              C.byref(R)))
        return rt[:R.value], sp.reshape(T, K), sg.reshape(E, 3)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.dsmoe_b200_ctx_free(h)
            self.h = None


# ------------------------------------------------------------------ routing
@dataclass
class RoutingDecision:
    """RoutingDecision (moe.hpp:142-167), device tensors of shape T x (K*P)."""

    num_tokens: int
    k: int
    base_k: int
    replay_factor: int
    indices: object
    raw: object          # fp32 on device; double(raw) is the reference's raw
    normalized: object   # fp64
    fraction_code: object  # uint8: 0 -> 0.0, 1 -> 0.5, 2 -> 1.0
    stats: dict = field(default_factory=dict)

    @property
    def fraction(self):
        torch = _torch()
        return torch.tensor([0.0, 0.5, 1.0], dtype=torch.float64,
                            device=self.fraction_code.device)[self.fraction_code.long()]

    def host(self):
        """numpy copies with the reference's types (int32, double...)."""
        return (self.indices.cpu().numpy(), self.raw.double().cpu().numpy(),
                self.normalized.cpu().numpy(), self.fraction.cpu().numpy())


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _x(x, layer: MoeLayer):
    torch = _torch()
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise DsmoeError(1, "tokens must be a CUDA tensor")
    if x.dtype != layer.torch_dtype:
        raise DsmoeError(2, f"tokens dtype {x.dtype} does not match layer dtype {layer.dtype}")
    if x.dim() != 2 or x.shape[1] != layer.d:
        raise DsmoeError(2, f"tokens shape {tuple(x.shape)} does not match d_model {layer.d}")
    return x.contiguous()


def route_and_drop(ctx: Context, layer: MoeLayer, x, policy: DropPolicy | None = None, logits=None,
                   logits_mode=LOGITS_TENSOR, t_unit=None, return_logits=False) -> RoutingDecision:
    """route_and_drop (dropping.hpp:248): gate -> softmax -> Top-K -> replay ->
    normalize -> 1T/2T drop, on the device.  `logits` (T x E fp32 CUDA tensor)
    bypasses the gate matmul, for parity on identical logits."""
    torch = _torch()
    policy = policy or DropPolicy()
    if logits is not None:
        logits = logits.contiguous().float()
        T = logits.shape[0]
        dev = logits.device
        xp = None
    else:
        x = _x(x, layer)
        T = x.shape[0]
        dev = x.device
        xp = x.data_ptr()
    n = T * layer.K * layer.P
    idx = torch.empty(n, dtype=torch.int32, device=dev)
    raw = torch.empty(n, dtype=torch.float32, device=dev)
    norm = torch.empty(n, dtype=torch.float64, device=dev)
    frac = torch.empty(n, dtype=torch.uint8, device=dev)
    lg_out = torch.empty((T, layer.E), dtype=torch.float32, device=dev) if return_logits else None
    out = RoutingOut(idx.data_ptr(), raw.data_ptr(), norm.data_ptr(), frac.data_ptr())
    st = DropStatsC()
    _chk(lib().dsmoe_b200_route(ctx.h, layer.h, None if xp is None else C.c_void_p(xp), T,
                                C.byref(policy.c(t_unit)), logits_mode,
                                None if logits is None else C.c_void_p(logits.data_ptr()),
                                None if lg_out is None else C.c_void_p(lg_out.data_ptr()),
                                C.byref(out), C.byref(st)))
    sh = (T, layer.K * layer.P)
    r = RoutingDecision(T, layer.K * layer.P, layer.K, layer.P, idx.view(sh), raw.view(sh), norm.view(sh),
                        frac.view(sh), st.as_dict())
    if return_logits:
        return r, lg_out
    return r


def moe_forward(ctx: Context, layer: MoeLayer, x, routing) -> object:
    """moe_forward (moe.hpp:239): raw-score-weighted sum of the kept expert
    blocks plus the unweighted shared experts.  `routing` is a RoutingDecision
    or a tuple (indices int32, raw float64, fraction float64) of CUDA tensors."""
    torch = _torch()
    x = _x(x, layer)
    T = x.shape[0]
    if isinstance(routing, RoutingDecision):
        idx, raw, frac = routing.indices, routing.raw.double(), routing.fraction
    else:
        idx, raw, frac = routing
    idx = idx.to(device=x.device, dtype=torch.int32).contiguous()
    raw = raw.to(device=x.device, dtype=torch.float64).contiguous()
    frac = frac.to(device=x.device, dtype=torch.float64).contiguous()
    if idx.numel() != T * layer.K * layer.P:
        raise DsmoeError(3, "moe_forward: routing does not match the layer's selections per token")
    out = torch.empty_like(x)
    _chk(lib().dsmoe_b200_moe_forward(ctx.h, layer.h, C.c_void_p(x.data_ptr()), T,
                                      C.c_void_p(idx.data_ptr()), C.c_void_p(raw.data_ptr()),
                                      C.c_void_p(frac.data_ptr()), C.c_void_p(out.data_ptr())))
    return out


def forward(ctx: Context, layer: MoeLayer, x, policy: DropPolicy | None = None, out=None,
            logits_mode=LOGITS_TENSOR, with_stats=False, residual=False):
    """route_and_drop + moe_forward in one device launch sequence (the
    per-layer body of model_forward_dropped, dropping.hpp:263-274).
    residual=True returns x + moe(x) (the residual add fused into combine)."""
    torch = _torch()
    x = _x(x, layer)
    if out is None:
        out = torch.empty_like(x)
    if residual and out.data_ptr() == x.data_ptr():
        raise DsmoeError(1, "forward: residual output may not alias the input")
    st = DropStatsC()
    _chk(lib().dsmoe_b200_forward_ex(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0],
                                     C.byref((policy or DropPolicy()).c()), logits_mode, 1 if residual else 0,
                                     C.c_void_p(out.data_ptr()), C.byref(st) if with_stats else None))
    return (out, st.as_dict()) if with_stats else out


def calibrate_rate(ctx: Context, layer: MoeLayer, x, target: float, kind: str = "2t", keep_top1=True, tol=0.005,
                   iters=40, normalize=None, logits_mode=LOGITS_TENSOR):
    """The threshold that reaches `target` drop rate on batch x, bisected on
    the device in one kernel (the acceptance.cpp:342-352 method; the same t as
    the host loop over route_and_drop stats).  Returns (DropPolicy, rate)."""
    x = _x(x, layer)
    if target <= 0:
        return DropPolicy(), 0.0
    base = DropPolicy("2t" if kind == "2t" else "1t", 0.0, keep_top1=keep_top1, normalize=normalize)
    t, r = C.c_double(), C.c_double()
    _chk(lib().dsmoe_b200_calibrate_rate(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0], C.byref(base.c()),
                                         float(target), float(tol), int(iters), logits_mode, C.byref(t), C.byref(r)))
    pol = DropPolicy.two_t_from(t.value, keep_top1) if kind == "2t" else DropPolicy.one_t(t.value, keep_top1)
    pol.normalize = normalize
    return pol, r.value


def forward_rate(ctx: Context, layer: MoeLayer, x, target: float, kind: str = "2t", keep_top1=True, tol=0.005,
                 iters=40, out=None, normalize=None, logits_mode=LOGITS_TENSOR, with_stats=False, t_rate=None,
                 residual=False):
    """The forward under a per-batch rate-targeted drop mask: the threshold is
    bisected on the device and applied without a host round trip.
    t_rate (optional float64 CUDA tensor of 2) receives [t, rate]."""
    torch = _torch()
    x = _x(x, layer)
    if out is None:
        out = torch.empty_like(x)
    base = DropPolicy("2t" if kind == "2t" else "1t", 0.0, keep_top1=keep_top1, normalize=normalize)
    st = DropStatsC()
    _chk(lib().dsmoe_b200_forward_rate(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0], C.byref(base.c()),
                                       float(target), float(tol), int(iters), logits_mode, 1 if residual else 0,
                                       C.c_void_p(out.data_ptr()), _p(t_rate), C.byref(st) if with_stats else None))
    return (out, st.as_dict()) if with_stats else out


def model_forward_dropped(ctx: Context, layers, x, policy=None, logits_mode=LOGITS_TENSOR):
    """model_forward_dropped (dropping.hpp:263-274): x_{l+1} = x_l + moe_l(x_l)
    with per-layer route_and_drop; returns (output, [DropStats per layer]).
    `policy` is one DropPolicy for every layer (the reference's signature) or
    a sequence with one DropPolicy per layer — per-layer thresholds, since the
    drop rate a threshold yields varies by layer."""
    torch = _torch()
    layers = list(layers)
    if isinstance(policy, (list, tuple)):
        if len(policy) != len(layers):
            raise DsmoeError(1, f"model_forward_dropped: {len(policy)} policies for {len(layers)} layers")
        policies = list(policy)
    else:
        policies = [policy] * len(layers)
    cur = x
    stats = []
    bufs = [torch.empty_like(x), torch.empty_like(x)]
    for i, layer in enumerate(layers):
        nxt = bufs[i & 1]
        _, st = forward(ctx, layer, cur, policies[i], out=nxt, logits_mode=logits_mode, with_stats=True,
                        residual=True)
        stats.append(st)
        cur = nxt
    return cur.clone() if layers else x.clone(), stats


# ---------------------------------------------------------------- host math
def drop_stats(pre_fraction, post_fraction, replay_factor, num_shared, num_tokens, d_model, d_ffn) -> dict:
    """drop_stats (dropping.hpp:171-195) through the C ABI (host arithmetic)."""
    pre = np.ascontiguousarray(pre_fraction, np.float64).ravel()
    post = np.ascontiguousarray(post_fraction, np.float64).ravel()
    if pre.size != post.size:
        raise DsmoeError(1, "drop_stats: routing shapes differ")
    st = DropStatsC()
    _chk(lib().dsmoe_b200_drop_stats(pre.ctypes.data, post.ctypes.data, pre.size, replay_factor, num_shared,
                                     num_tokens, d_model, d_ffn, C.byref(st)))
    return st.as_dict()


def load_aware_thresholds(loads, t_max) -> np.ndarray:
    """load_aware_thresholds (ep_sim.hpp:76-89)."""
    loads = np.ascontiguousarray(loads, np.float64)
    out = np.empty_like(loads)
    _chk(lib().dsmoe_b200_load_aware_thresholds(loads.ctypes.data, loads.size, t_max, out.ctypes.data))
    return out


def simulate_step(ctx: Context, layer: MoeLayer, x, device_of, devices: int, policy: DropPolicy | None = None,
                  load_aware=True, logits_mode=LOGITS_EXACT, forward=False, routing=False):
    """simulate_step (ep_sim.hpp:110-160) on the device: the EpReport fields
    (pre / post loads, thresholds, ideal load, drop rate, speed-up, stats);
    routing=True adds the dropped RoutingDecision, forward=True the output
    moe_forward(x, post)."""
    torch = _torch()
    x = _x(x, layer)
    T = x.shape[0]
    dv = np.ascontiguousarray(device_of, np.int32)
    pre, post, th = (np.zeros(devices) for _ in range(3))
    sc = np.zeros(3)
    st = DropStatsC()
    r = None
    if routing:
        r = RoutingDecision(T, layer.K * layer.P, layer.K, layer.P,
                            torch.empty((T, layer.K * layer.P), dtype=torch.int32, device=x.device),
                            torch.empty((T, layer.K * layer.P), dtype=torch.float32, device=x.device),
                            torch.empty((T, layer.K * layer.P), dtype=torch.float64, device=x.device),
                            torch.empty((T, layer.K * layer.P), dtype=torch.uint8, device=x.device))
    ro = RoutingOut(r.indices.data_ptr(), r.raw.data_ptr(), r.normalized.data_ptr(),
                    r.fraction_code.data_ptr()) if routing else None
    y = torch.empty_like(x) if forward else None
    _chk(lib().dsmoe_b200_simulate_step(ctx.h, layer.h, C.c_void_p(x.data_ptr()), T, devices, dv.ctypes.data,
                                        C.byref((policy or DropPolicy()).c()), int(load_aware), logits_mode,
                                        pre.ctypes.data, post.ctypes.data, th.ctypes.data, sc.ctypes.data,
                                        C.byref(st), C.byref(ro) if routing else None, _p(y), 0))
    rep = {"devices": devices, "load_aware": bool(load_aware), "pre_loads": pre, "post_loads": post,
           "thresholds": th, "ideal_load": sc[0], "drop_rate": sc[1], "speedup": sc[2], "stats": st.as_dict()}
    if routing:
        r.stats = rep["stats"]
    return rep, r, y


def place_experts(num_experts: int, devices: int, strategy: str = "contiguous") -> np.ndarray:
    """place_experts (ep_sim.hpp:38-54)."""
    if not (devices >= 1 and num_experts >= devices):
        raise DsmoeError(1, "place_experts: need num_experts >= devices >= 1")
    if strategy in ("round_robin", "round-robin"):
        return (np.arange(num_experts) % devices).astype(np.int32)
    if strategy != "contiguous":
        raise DsmoeError(1, f"unknown placement strategy: {strategy}")
    if num_experts % devices:
        raise DsmoeError(1, "place_experts: contiguous placement needs num_experts divisible by devices")
    return (np.arange(num_experts) // (num_experts // devices)).astype(np.int32)


# ------------------------------------------------- offline reconstruction (K7/K8)
def profile_importance(ctx: Context, layer: MoeLayer, calib, indices, metric="abs_gate"):
    """profile_importance (reconstruct.hpp:99-149) on the device: E x d_ffn
    float64 importance, bit-equal to the reference on the same inputs.
    `indices` are the layer's own routing (route_tokens, T x K)."""
    torch = _torch()
    x = _x(calib, layer)
    idx = indices.to(device=x.device, dtype=torch.int32).contiguous()
    if idx.numel() != x.shape[0] * layer.K:
        raise DsmoeError(1, "profile_importance: routing does not match calibration batch")
    vals = torch.empty((layer.E, layer.ffn), dtype=torch.float64, device=x.device)
    _chk(lib().dsmoe_b200_profile_importance(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0],
                                             C.c_void_p(idx.data_ptr()), METRIC[metric.replace("-", "_")],
                                             C.c_void_p(vals.data_ptr())))
    return vals


def reconstruct_experts(ctx: Context, layer: MoeLayer, values):
    """build_reconstruction_map + reconstruct_experts (reconstruct.hpp:151-230)
    on the device: returns (reconstructed MoeLayer with P=2, order E x d_ffn)."""
    torch = _torch()
    values = values.to(device="cuda", dtype=torch.float64).contiguous()
    order = torch.empty((layer.E, layer.ffn), dtype=torch.int32, device=values.device)
    h = C.c_void_p()
    _chk(lib().dsmoe_b200_reconstruct(ctx.h, layer.h, C.c_void_p(values.data_ptr()), C.c_void_p(order.data_ptr()),
                                      C.byref(h)))
    return MoeLayer._wrap(h, layer), order


# ------------------------------------------------- partition API (K8b)
TRANSFORM = {"complete": 0, "partial": 1, "reverse": 2}


def transform(ctx: Context, layer: MoeLayer, mode: str, p: int = 0) -> MoeLayer:
    """complete_transform / partial_transform (transform.hpp:66-131) or
    reverse_partial (:136-170) of a device layer, re-grouped on the device;
    returns the new MoeLayer (the source is unchanged)."""
    if mode not in TRANSFORM:
        raise DsmoeError(1, "mode must be complete, partial or reverse")
    h = C.c_void_p()
    _chk(lib().dsmoe_b200_transform(ctx.h, layer.h, TRANSFORM[mode], int(p), C.byref(h)))
    return MoeLayer._wrap(h, layer)


def complete_transform(ctx: Context, layer: MoeLayer, p: int) -> MoeLayer:
    """complete_transform (transform.hpp:66-95)."""
    return transform(ctx, layer, "complete", p)


def partial_transform(ctx: Context, layer: MoeLayer, p: int) -> MoeLayer:
    """partial_transform (transform.hpp:100-131); the PartitionSpec is
    (factor p, partial, E, d_ffn, chunk d_ffn/p) and is implied by the layer."""
    return transform(ctx, layer, "partial", p)


def layer_weights(ctx: Context, layer: MoeLayer, device=True, blocks=None):
    """The layer's weights in the reference layout (moe.hpp:39-45, :75), layer
    dtype: (gate d x E, [(w1 d x w, w3 d x w, w2 w x d) per block], [shared]).
    `blocks` (optional index list) reads only those blocks (None elsewhere)."""
    torch = _torch()
    dev = "cuda" if device else "cpu"
    dt = layer.torch_dtype
    bw, sw = layer.widths()
    gate = torch.empty((layer.d, layer.E), dtype=dt, device=dev)
    _chk(lib().dsmoe_b200_layer_get_gate(ctx.h, layer.h, C.c_void_p(gate.data_ptr()), int(device)))

    def get(fn, i, w):
        w1 = torch.empty((layer.d, w), dtype=dt, device=dev)
        w3 = torch.empty_like(w1)
        w2 = torch.empty((w, layer.d), dtype=dt, device=dev)
        _chk(fn(ctx.h, layer.h, i, C.c_void_p(w1.data_ptr()), C.c_void_p(w3.data_ptr()), C.c_void_p(w2.data_ptr()),
                int(device)))
        return w1, w3, w2
    want = set(range(len(bw))) if blocks is None else set(blocks)
    out = [get(lib().dsmoe_b200_layer_get_block, b, w) if b in want else None for b, w in enumerate(bw)]
    shared = [get(lib().dsmoe_b200_layer_get_shared, i, w) for i, w in enumerate(sw)]
    return gate, out, shared


# ------------------------------------------------ expert-parallel data path
def dispatch(ctx: Context, layer: MoeLayer, x, policy: DropPolicy | None = None, t_unit=None,
             rows_out=None, scale_out=None, logits_mode=LOGITS_TENSOR, with_stats=False):
    """Route + drop + permute (+ gather into rows_out / scale_out when given).
    Returns (seg E x 3 numpy [start, full rows, total rows], R, stats)."""
    x = _x(x, layer)
    seg = np.empty((layer.E, 3), np.int32)
    R = C.c_int()
    st = DropStatsC()
    _chk(lib().dsmoe_b200_dispatch(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0],
                                   C.byref((policy or DropPolicy()).c(t_unit)), logits_mode,
                                   None if rows_out is None else C.c_void_p(rows_out.data_ptr()),
                                   None if scale_out is None else C.c_void_p(scale_out.data_ptr()),
                                   seg.ctypes.data, C.byref(R), C.byref(st) if with_stats else None))
    return seg, R.value, (st.as_dict() if with_stats else None)


def expert_ffn(ctx: Context, layer: MoeLayer, rows, row_scale, segments, y_out=None):
    """Grouped expert FFN over segments [(unit, start, n_full, n_tot), ...] of
    `rows` (CUDA tensor nrows x d); returns y (nrows x d)."""
    torch = _torch()
    if y_out is None:
        y_out = torch.empty_like(rows)
    segs = np.asarray(segments, np.int32).reshape(-1, 4)
    cols = [np.ascontiguousarray(segs[:, i]) for i in range(4)]
    _chk(lib().dsmoe_b200_expert_ffn(ctx.h, layer.h, C.c_void_p(rows.data_ptr()), C.c_void_p(row_scale.data_ptr()),
                                     rows.shape[0], segs.shape[0], *[c.ctypes.data for c in cols],
                                     C.c_void_p(y_out.data_ptr())))
    return y_out


def ep_pack(ctx: Context, layer: MoeLayer, x, nranks: int, owner, send_rows, rec_code, rec_row, rec_raw):
    """After dispatch() routed x on ctx: one row per (token, owning rank) into
    send_rows and one record per kept selection; returns (rows per rank,
    records per rank) as int64 numpy arrays."""
    own = np.ascontiguousarray(owner, np.int32)
    counts = np.zeros(2 * nranks, np.int64)
    _chk(lib().dsmoe_b200_ep_pack(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0], nranks, own.ctypes.data,
                                  C.c_void_p(send_rows.data_ptr()), C.c_void_p(rec_code.data_ptr()),
                                  C.c_void_p(rec_row.data_ptr()), C.c_void_p(rec_raw.data_ptr()), counts.ctypes.data))
    return counts[:nranks].copy(), counts[nranks:].copy()


def ep_expert(ctx: Context, layer: MoeLayer, rows, U: int, rec_code, rec_row, rec_raw, S: int, src_row_base,
              src_rec_base, out=None):
    """Routed experts over received rows: one output row per received row."""
    torch = _torch()
    if out is None:
        out = torch.empty((max(U, 1), layer.d), dtype=layer.torch_dtype, device=rows.device)
    rb = np.ascontiguousarray(src_row_base, np.int64)
    sb = np.ascontiguousarray(src_rec_base, np.int64)
    _chk(lib().dsmoe_b200_ep_expert(ctx.h, layer.h, C.c_void_p(rows.data_ptr()), U, C.c_void_p(rec_code.data_ptr()),
                                    C.c_void_p(rec_row.data_ptr()), C.c_void_p(rec_raw.data_ptr()), S, rb.ctypes.data,
                                    sb.ctypes.data, len(rb) - 1, C.c_void_p(out.data_ptr())))
    return out


def ep_combine(ctx: Context, layer: MoeLayer, ret_rows, T: int, out=None):
    """out = sum over ranks of the returned rows (send order of the last ep_pack) + shared experts."""
    torch = _torch()
    if out is None:
        out = torch.empty((T, layer.d), dtype=layer.torch_dtype, device=ret_rows.device)
    _chk(lib().dsmoe_b200_ep_combine(ctx.h, layer.h, C.c_void_p(ret_rows.data_ptr()), T, C.c_void_p(out.data_ptr())))
    return out


# ---------------------------------- EP with one host synchronisation per step
def ep_route_counts(ctx: Context, layer: MoeLayer, x, policy: DropPolicy | None = None, counts=None,
                    logits_mode=LOGITS_TENSOR):
    """Route x without drop; per-expert (full, major-only) selection counts
    (E x 2 int64 CUDA tensor), no host sync."""
    torch = _torch()
    x = _x(x, layer)
    if counts is None:
        counts = torch.empty((layer.E, 2), dtype=torch.int64, device=x.device)
    _chk(lib().dsmoe_b200_ep_route_counts(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0],
                                          C.byref((policy or DropPolicy()).c()), logits_mode, _p(counts)))
    return counts


def ep_last_counts(ctx: Context, layer: MoeLayer, T: int, counts=None):
    """(full, major-only) kept-selection counts of the last routing on ctx."""
    torch = _torch()
    if counts is None:
        counts = torch.empty((layer.E, 2), dtype=torch.int64, device="cuda")
    _chk(lib().dsmoe_b200_ep_last_counts(ctx.h, layer.h, T, _p(counts)))
    return counts


def ep_thresholds(ctx: Context, layer: MoeLayer, counts, devices: int, device_of, t_max: float, load_aware: bool,
                  t_unit=None, loads=None):
    """Device-side device_loads -> load_aware_thresholds -> owner table
    (ep_sim.hpp:59-89, :139-141) from all-reduced counts; returns (t_unit E
    float64, loads devices float64), CUDA tensors, no host sync."""
    torch = _torch()
    if t_unit is None:
        t_unit = torch.empty(layer.E, dtype=torch.float64, device=counts.device)
    if loads is None:
        loads = torch.empty(devices, dtype=torch.float64, device=counts.device)
    _chk(lib().dsmoe_b200_ep_thresholds(ctx.h, layer.h, _p(counts), devices, _p(device_of), float(t_max),
                                        int(load_aware), _p(t_unit), _p(loads)))
    return t_unit, loads


def ctx_logits(ctx: Context):
    """(device pointer, row stride, T) of the gate logits of the last routing on ctx."""
    p, ld, T = C.c_void_p(), C.c_int(), C.c_int()
    _chk(lib().dsmoe_b200_ctx_logits(ctx.h, C.byref(p), C.byref(ld), C.byref(T)))
    return p.value, ld.value, T.value


def ep_dispatch(ctx: Context, layer: MoeLayer, x, policy: DropPolicy | None, t_unit, nranks: int, dest, send_rows,
                records, counts, logits_mode=LOGITS_REUSE, logits=None):
    """Re-route under the owner thresholds, pack one row per (token,
    destination) + one 3 x int32 record per (kept selection, destination),
    counts (nranks x 2 int64: rows, records), local shared experts; no host
    sync.  dest: E x 2 int32 (bit masks) CUDA tensor — the ranks a full /
    a major-only selection of each expert goes to."""
    x = _x(x, layer)
    lp, ld = (None, 0) if logits is None else (C.c_void_p(logits[0]), int(logits[1]))
    _chk(lib().dsmoe_b200_ep_dispatch(ctx.h, layer.h, C.c_void_p(x.data_ptr()), x.shape[0],
                                      C.byref((policy or DropPolicy()).c(t_unit)), logits_mode, lp, ld, nranks,
                                      _p(dest), _p(send_rows), _p(records), _p(counts)))


def ep_expert_packed(ctx: Context, layer: MoeLayer, rows, U: int, records, S: int, src_row_base, src_rec_base,
                     out=None):
    torch = _torch()
    if out is None:
        out = torch.empty((max(U, 1), layer.d), dtype=layer.torch_dtype, device=rows.device)
    rb = np.ascontiguousarray(src_row_base, np.int64)
    sb = np.ascontiguousarray(src_rec_base, np.int64)
    _chk(lib().dsmoe_b200_ep_expert_packed(ctx.h, layer.h, C.c_void_p(rows.data_ptr()), U, _p(records), S,
                                           rb.ctypes.data, sb.ctypes.data, len(rb) - 1, C.c_void_p(out.data_ptr())))
    return out


def layer_shard_blocks(ctx: Context, layer: MoeLayer, held) -> MoeLayer:
    """An expert shard holding the physical blocks flagged in `held` (E*P)."""
    h = C.c_void_p()
    hm = np.ascontiguousarray(held, np.uint8)
    _chk(lib().dsmoe_b200_layer_shard_blocks(ctx.h, layer.h, hm.ctypes.data, C.byref(h)))
    out = MoeLayer._wrap(h, layer)
    out.shard = tuple(np.nonzero(hm)[0].tolist())
    return out


def layer_shard(ctx: Context, layer: MoeLayer, unit_lo: int, unit_hi: int) -> MoeLayer:
    """An expert shard: the same gate and shared experts, routed experts
    [unit_lo, unit_hi) only (dsmoe_b200_layer_shard)."""
    h = C.c_void_p()
    _chk(lib().dsmoe_b200_layer_shard(ctx.h, layer.h, unit_lo, unit_hi, C.byref(h)))
    out = MoeLayer._wrap(h, layer)
    out.shard = (unit_lo, unit_hi)
    return out


def combine(ctx: Context, layer: MoeLayer, y_rows, T, out=None):
    """out = sum of the returned expert rows at the last dispatch's slots + shared experts."""
    torch = _torch()
    if out is None:
        out = torch.empty((T, layer.d), dtype=layer.torch_dtype, device=y_rows.device)
    _chk(lib().dsmoe_b200_combine(ctx.h, layer.h, C.c_void_p(y_rows.data_ptr()), T, C.c_void_p(out.data_ptr())))
    return out
