"""DSMOE1 model containers and token files -> device layers,
and `infer`, the device twin of the reference's dsmoe_infer.

Format and validation follow /root/reference/proj/src/io.cpp exactly:
  8-byte magic "DSMOE1\\0\\0" (io.hpp:14), u64 LE manifest length, JSON
  manifest {format, version, scalar_width, num_layers, layers[{config, lineage,
  replay_factor, neuron_order}], tensors[{name, shape, width, offset}]},
  64-byte-aligned payloads (io.hpp:15) in the order gate, experts/e/{w1,w3,w2},
  shared/s/{w1,w3,w2} per layer (io.cpp:177-262); token files: u64 rows, u64
  cols, float32 payload (io.cpp:312-327).
Errors raise DsmoeError with the reference's status codes (io_error 4,
bad_magic 5, truncated 6, schema_error 7).  Parsing is host-side (numpy views
of the file); `to_device` packs each layer for the GPU (bf16 by default).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field

import numpy as np

from .dsmoe import DsmoeError, DropPolicy, MoeLayer, Context, model_forward_dropped, LOGITS_EXACT

MAGIC = b"DSMOE1\x00\x00"
ALIGN = 64
IO_ERROR, BAD_MAGIC, TRUNCATED, SCHEMA = 4, 5, 6, 7
LINEAGES = ("base", "complete", "partial", "reconstructed")


@dataclass
class HostLayer:
    """One MoeLayer<T> as stored (moe.hpp:73-120): numpy arrays in the
    container's scalar type."""

    config: dict
    lineage: str
    replay_factor: int
    neuron_order: list
    gate: np.ndarray
    blocks: list = field(default_factory=list)
    shared: list = field(default_factory=list)


def _read(path):
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise DsmoeError(IO_ERROR, f"cannot open for reading: {path}") from e


def _require(ok, code, msg):
    if not ok:
        raise DsmoeError(code, msg)


def parse_model(path) -> list:
    """load_model (io.cpp:268-294) + model_from_container (:177-262)."""
    raw = _read(path)
    _require(len(raw) >= 16, TRUNCATED, "container: file shorter than header")
    _require(raw[:8] == MAGIC, BAD_MAGIC, "container: bad magic")
    (mlen,) = struct.unpack_from("<Q", raw, 8)
    _require(16 + mlen <= len(raw), TRUNCATED, "container: manifest truncated")
    try:
        man = json.loads(raw[16:16 + mlen].decode("utf-8"))
    except (ValueError, UnicodeDecodeError) as e:
        raise DsmoeError(SCHEMA, f"container: manifest is not valid JSON: {e}") from e
    try:
        _require(man["format"] == "dsmoe-container", SCHEMA, "container: unknown format tag")
        _require(man["version"] == 1, SCHEMA, "container: unsupported version")
        width = man["scalar_width"]
        _require(width in (4, 8), SCHEMA, "container: scalar_width must be 4 or 8")
        dt = np.dtype("<f4") if width == 4 else np.dtype("<f8")
        nl = man["num_layers"]
        _require(nl >= 1, SCHEMA, "container: num_layers must be >= 1")
        jl = man["layers"]
        _require(isinstance(jl, list) and len(jl) == nl, SCHEMA, "container: layer list does not match num_layers")
        table = man["tensors"]
        _require(isinstance(table, list), SCHEMA, "container: tensor table missing")
        entries, prev_end = [], 0
        for e in table:
            shape = e["shape"]
            _require(isinstance(shape, list) and len(shape) == 2, SCHEMA, "container: tensor shape must be [rows, cols]")
            r, c = int(shape[0]), int(shape[1])
            _require(r >= 0 and c >= 0, SCHEMA, "container: negative tensor shape")
            _require(e["width"] == width, SCHEMA, "container: tensor width disagrees with scalar_width")
            off = int(e["offset"])
            nbytes = r * c * width
            _require(off % ALIGN == 0, SCHEMA, f"container: tensor offset not 64-byte aligned: {e['name']}")
            _require(off >= prev_end, SCHEMA, f"container: overlapping or out-of-order tensor offsets at {e['name']}")
            prev_end = off + nbytes
            _require(prev_end <= len(raw), TRUNCATED, f"container: payload truncated at {e['name']}")
            entries.append((e["name"], r, c, off))
        nxt = 0

        def take(name):
            nonlocal nxt
            _require(nxt < len(entries) and entries[nxt][0] == name, SCHEMA, f"container: expected tensor {name}")
            _, r, c, off = entries[nxt]
            nxt += 1
            return np.frombuffer(raw, dtype=dt, count=r * c, offset=off).reshape(r, c)

        layers = []
        for li in range(nl):
            j = jl[li]
            cfg = {k: j["config"][k] for k in ("d_model", "d_ffn", "num_experts", "top_k", "num_shared_experts",
                                                "gate_prenormalized")}
            lin = j["lineage"]
            _require(lin in LINEAGES, SCHEMA, f"unknown lineage tag: {lin}")
            P = int(j["replay_factor"])
            base = f"layers/{li}/"
            L = HostLayer(cfg, lin, P, j["neuron_order"], take(base + "gate"))
            for b in range(cfg["num_experts"] * P):
                eb = f"{base}experts/{b}/"
                L.blocks.append((take(eb + "w1"), take(eb + "w3"), take(eb + "w2")))
            for s in range(cfg["num_shared_experts"]):
                sb = f"{base}shared/{s}/"
                L.shared.append((take(sb + "w1"), take(sb + "w3"), take(sb + "w2")))
            _validate(L)
            layers.append(L)
        _require(nxt == len(entries), SCHEMA, "container: unused tensors in table")
        return layers
    except (KeyError, TypeError) as e:
        raise DsmoeError(SCHEMA, f"container: manifest field error: {e}") from e


def _validate(L: HostLayer):
    """MoeLayer::validate (moe.hpp:90-119) -> schema_error on a container."""
    c = L.config
    d, ffn, E = c["d_model"], c["d_ffn"], c["num_experts"]
    bad = lambda m: DsmoeError(SCHEMA, f"container: inconsistent model: {m}")
    if L.gate.shape != (d, E):
        raise bad("gate shape")
    if L.replay_factor < 1:
        raise bad("replay_factor must be >= 1")
    for e in range(E):
        tot = 0
        for p in range(L.replay_factor):
            w1, w3, w2 = L.blocks[e * L.replay_factor + p]
            if not (w1.shape[0] == d and w3.shape == w1.shape and w2.shape == (w1.shape[1], d)):
                raise bad(f"inconsistent block shapes for expert {e}")
            tot += w1.shape[1]
        if tot != ffn:
            raise bad(f"block widths of expert {e} sum to {tot}, expected {ffn}")
    for w1, w3, w2 in L.shared:
        if not (w1.shape[0] == d and w3.shape == w1.shape and w2.shape == (w1.shape[1], d)):
            raise bad("inconsistent shared expert shapes")


def load_tokens(path) -> np.ndarray:
    """load_tokens (io.cpp:312-327): float32 rows x cols."""
    raw = _read(path)
    _require(len(raw) >= 16, TRUNCATED, "token file: missing header")
    rows, cols = struct.unpack_from("<QQ", raw, 0)
    _require(rows <= (1 << 24) and cols <= (1 << 20), SCHEMA, "token file: implausible dimensions")
    _require(len(raw) >= 16 + rows * cols * 4, TRUNCATED, "token file: payload truncated")
    return np.frombuffer(raw, dtype="<f4", count=rows * cols, offset=16).reshape(rows, cols).astype(np.float32)


def to_device(host_layers, dtype="bf16", stream=None) -> list:
    """Pack parsed layers for the GPU.  fp64 containers are narrowed to the
    device type (the device path computes in fp32 / bf16)."""
    out = []
    for L in host_layers:
        c = L.config
        f = lambda a: np.ascontiguousarray(a, np.float32)
        out.append(MoeLayer(c["d_model"], c["d_ffn"], c["num_experts"], c["top_k"], f(L.gate),
                            [tuple(f(w) for w in b) for b in L.blocks], [tuple(f(w) for w in s) for s in L.shared],
                            replay_factor=L.replay_factor, dtype=dtype,
                            gate_prenormalized=bool(c["gate_prenormalized"]), stream=stream))
    return out


def load_model(path, dtype="bf16", stream=None) -> list:
    """DSMOE1 container -> device layers."""
    return to_device(parse_model(path), dtype, stream)


def policy_from(j: dict, gate_prenormalized: bool) -> DropPolicy:
    """policy_from (capi.cpp:96-112): kind none|1t|2t; 2T band defaults to
    t_drop -/+ 0.01; keep_top1 defaults to true; normalize to !prenormalized."""
    kind = j.get("kind", "none")
    if kind not in ("none", "1t", "2t"):
        raise DsmoeError(1, f"unknown drop policy kind: {kind}")
    if kind == "none":
        p = DropPolicy()
    else:
        if "t_drop" not in j:
            raise DsmoeError(1, "policy: t_drop is required")
        t = float(j["t_drop"])
        if kind == "1t":
            p = DropPolicy.one_t(t)
        else:
            p = DropPolicy.two_t(t, float(j.get("t_major", t - 0.01)), float(j.get("t_minor", t + 0.01)))
    p.keep_top1 = bool(j.get("keep_top1", True))
    p.normalize = bool(j.get("normalize", not gate_prenormalized))
    return p


def infer(layers, tokens, policy_json: dict, ctx: Context | None = None, logits_mode=LOGITS_EXACT) -> dict:
    """dsmoe_infer (capi.cpp:328-368) on the device: no-drop baseline and the
    dropped forward through the residual layer stack, aggregated drop
    accounting (units and FLOPs summed over layers), mean relative error
    (dropping.hpp:278-293, computed on the host from the two outputs)."""
    import torch
    ctx = ctx or Context()
    prenorm = bool(layers[0].prenorm)
    pol = policy_from(policy_json, prenorm)
    dt = layers[0].torch_dtype
    x = tokens if isinstance(tokens, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(tokens, np.float32))
    x = x.to(device="cuda", dtype=dt)
    base, _ = model_forward_dropped(ctx, layers, x, DropPolicy(normalize=pol.normalize), logits_mode=logits_mode)
    y, stats = model_forward_dropped(ctx, layers, x, pol, logits_mode=logits_mode)
    dropped = sum(s["dropped_units"] for s in stats)
    denom = sum(s["total_routed_units"] + s["shared_units"] for s in stats)
    a = y.double().cpu().numpy()
    b = base.double().cpu().numpy()
    diff = np.sqrt(((a - b) ** 2).sum(axis=1))
    nb = np.sqrt((b ** 2).sum(axis=1))
    rel = np.where(nb > 0, diff / np.where(nb > 0, nb, 1), diff)
    return {"policy": {"kind": pol.kind, "t_drop": pol.t_drop, "t_major": pol.t_major, "t_minor": pol.t_minor,
                       "keep_top1": pol.keep_top1, "normalize": pol.normalize},
            "drop_rate": dropped / denom if denom > 0 else 0.0, "dropped_units": dropped, "total_units": denom,
            "total_flops": sum(s["total_flops"] for s in stats), "saved_flops": sum(s["saved_flops"] for s in stats),
            "rel_error": float(rel.mean()) if len(rel) else 0.0, "per_layer": stats}
