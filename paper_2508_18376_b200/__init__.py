"""B200-native DualSparse-MoE MoE-module forward (arxiv 2508.18376).

The compute path is libdsmoe_b200.so (CUDA for sm_100a, C ABI in
include/dsmoe_b200.h); dsmoe.py mirrors the reference's C++ partition /
drop-policy / forward API on top of it; ep.py runs expert parallelism over
torch.distributed (NCCL).
"""
from .dsmoe import (  # noqa: F401
    DropPolicy, DsmoeError, MoeLayer, Context, RoutingDecision, route_and_drop, moe_forward, forward,
    drop_stats, load_aware_thresholds, place_experts, lib, last_launch_count, total_launch_count, LOGITS_TENSOR,
    LOGITS_EXACT,
    profile_importance, reconstruct_experts, model_forward_dropped, dispatch, expert_ffn, combine,
    LOGITS_REUSE, transform, complete_transform, partial_transform, layer_weights,
    calibrate_rate, forward_rate, simulate_step, ep_route_counts, ep_last_counts, ep_thresholds, ep_dispatch, ep_expert_packed, layer_shard, layer_shard_blocks,
)
