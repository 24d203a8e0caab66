"""B200-native Glinthawk two-tier decode path (arXiv 2501.11779).

Tier-1 (weights: F1/F3/classifier) and Tier-2 (KV context: F2) stages as sm_100a kernels behind
the C ABI in include/gh/gh.h (libgh.so, built in-tree); this package is the Python host mirror.
"""
from ._lib import (CudaError, FeasibilityError, GhError, NcclError, UnsupportedError, ValidationError,
                   lib)
from .spec import (CONFIGS, LLAMA2_7B, LLAMA2_13B, LLAMA2_70B, TINY, ModelSpec, attention_footprint,
                   batch_grid, engine_layout, kv_bytes_per_prompt, layer_spans, node_weight_bytes, nonattention_footprint,
                   payload, shard_plan, throughput_from, two_tier_context_slots, weights_bytes)

__all__ = [
    "CONFIGS", "LLAMA2_7B", "LLAMA2_13B", "LLAMA2_70B", "TINY", "ModelSpec", "attention_footprint",
    "batch_grid", "engine_layout", "kv_bytes_per_prompt", "layer_spans", "node_weight_bytes", "nonattention_footprint",
    "payload", "shard_plan", "throughput_from", "two_tier_context_slots", "weights_bytes", "GhError", "ValidationError",
    "FeasibilityError", "CudaError", "NcclError", "UnsupportedError", "lib",
]
