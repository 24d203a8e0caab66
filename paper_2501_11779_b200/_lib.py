"""ctypes binding of libgh.so (the C ABI declared in include/gh/gh.h).

The product path has no fallback: if the in-tree ``libgh.so`` is missing the import of any
stage object raises ``RuntimeError`` (build it with ``python -c "import __graft_entry__ as g;
g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libgh.so"

GH_OK, GH_EINTERNAL, GH_EINVAL, GH_EINFEASIBLE, GH_ECUDA, GH_ENCCL, GH_EUNSUPPORTED = range(7)
STAGE_NONATTENTION, STAGE_ATTENTION, STAGE_CLASSIFIER = 0, 1, 2


class GhError(RuntimeError):
    """Base error; ``status`` mirrors the reference exit codes (commands.hpp:14-17)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class ValidationError(GhError):
    """Reference ValidationError (proj/include/tierplan/errors.hpp:18-22), exit code 2."""


class FeasibilityError(GhError):
    """Reference FeasibilityError (errors.hpp:24-32), exit code 3; binding constraint in msg."""


class CudaError(GhError):
    pass


class NcclError(GhError):
    pass


class UnsupportedError(GhError):
    pass


STATUS_NAMES = {0: "GH_OK", 1: "GH_EINTERNAL", 2: "GH_EINVAL", 3: "GH_EINFEASIBLE", 4: "GH_ECUDA",
                5: "GH_ENCCL", 6: "GH_EUNSUPPORTED"}
_ERR = {GH_EINVAL: ValidationError, GH_EINFEASIBLE: FeasibilityError, GH_ECUDA: CudaError,
        GH_ENCCL: NcclError, GH_EUNSUPPORTED: UnsupportedError}


class GhSpec(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("n_layers", "d_model", "d_kv", "d_hidden", "n_heads",
                                           "n_kv_heads", "max_seq_len", "dtype_bytes", "vocab_size")]
    _fields_ += [("rope_theta", C.c_float), ("norm_eps", C.c_float)]


class GhEngineConfig(C.Structure):
    _fields_ = [("spec", GhSpec), ("device", C.c_int), ("weight_seed", C.c_uint64),
                ("batch", C.c_uint32), ("inflight", C.c_uint32), ("n_slots", C.c_uint32),
                ("use_graph", C.c_int),
                ("transport", C.c_int),
                ("tier1_ranks", C.c_uint32),
                ("prefill", C.c_int),
                ("kv_pages", C.c_uint32),
                ("tier1_tp", C.c_uint32)]


class GhRankLayout(C.Structure):
    _fields_ = [("role", C.c_int), ("span", C.c_int), ("tp_rank", C.c_int), ("shard", C.c_int),
                ("kp", C.c_uint32), ("layer_begin", C.c_uint32), ("layer_end", C.c_uint32),
                ("row_off", C.c_uint32), ("row_cnt", C.c_uint32)]


class GhDispatchConfig(C.Structure):
    _fields_ = [("max_new", C.c_uint32), ("on_demand", C.c_int), ("preempt_swap", C.c_int),
                ("order_shortest", C.c_int), ("prefill_chunk", C.c_uint32)]


class GhDispatchStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("steps", "admitted", "finished", "tokens", "preemptions", "swaps")]
    _fields_ += [("peak_pages", C.c_uint32), ("lane_steps", C.c_uint64), ("context_sum", C.c_uint64)]


class GhSchedConfig(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("batch", "inflight", "kp", "pages", "max_seq", "max_new")]
    _fields_ += [(n, C.c_int) for n in ("on_demand", "preempt_swap", "order_shortest")]
    _fields_ += [("prefill_chunk", C.c_uint32)]


class GhLaneInput(C.Structure):
    _fields_ = [("src", C.c_int32), ("tok", C.c_int32), ("pos", C.c_int32), ("home", C.c_uint32)]


class GhKvAction(C.Structure):
    _fields_ = [("op", C.c_int32), ("lane", C.c_uint32), ("n", C.c_uint32), ("buf", C.c_uint64)]


u64, u32, i32, i64, vp = C.c_uint64, C.c_uint32, C.c_int32, C.c_int64, C.c_void_p
P = C.POINTER
st = C.c_int  # gh_status

# name -> (restype, argtypes); the exported-symbol test checks this table against gh.h
PROTOTYPES = {
    "gh_abi_version": (C.c_int, []),
    "gh_last_error": (C.c_char_p, []),
    "gh_status_name": (C.c_char_p, [st]),
    "gh_device_count": (C.c_int, []),
    "gh_spec_validate": (st, [P(GhSpec)]),
    "gh_kv_bytes_per_prompt": (st, [P(GhSpec), u64, P(u64)]),
    "gh_nonattention_footprint": (st, [P(GhSpec), u64, P(u64), P(u64)]),
    "gh_attention_footprint": (st, [P(GhSpec), u64, u64, P(u64), P(u64)]),
    "gh_weights_bytes": (st, [P(GhSpec), P(u64)]),
    "gh_payload_bytes": (st, [P(GhSpec), P(u64)]),
    "gh_layer_spans": (st, [u64, u64, P(u64)]),
    "gh_node_weight_bytes": (st, [P(GhSpec), u64, P(u64)]),
    "gh_two_tier_context_slots": (st, [P(GhSpec), u64, u64, u64, u64, P(u64)]),
    "gh_batch_grid": (st, [u64, P(u64), u64, P(u64)]),
    "gh_throughput_from": (st, [P(i64), u64, u64, u64, P(C.c_double)]),
    "gh_shard_plan": (st, [u64, u64, P(u64), P(u64)]),
    "gh_profile_write_csv": (st, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, u64, P(u64),
                                  P(C.c_double), u64]),
    "gh_tier1_create": (st, [P(GhSpec), C.c_int, u32, u32, u64, u32, P(vp)]),
    "gh_tier1_destroy": (st, [vp]),
    "gh_tier1_embed": (st, [vp, u32, vp, vp, vp]),
    "gh_tier1_pre": (st, [vp, u32, u32, vp, vp, vp, vp]),
    "gh_tier1_post": (st, [vp, u32, u32, vp, vp, vp]),
    "gh_tier1_classify": (st, [vp, u32, vp, vp, vp, vp]),
    "gh_tier2_create": (st, [P(GhSpec), C.c_int, u32, u32, u32, P(vp)]),
    "gh_tier2_destroy": (st, [vp]),
    "gh_tier2_attend": (st, [vp, u32, u32, vp, vp, vp, vp, vp]),
    "gh_tier2_check": (st, [vp, u32, P(u32), P(i32)]),
    "gh_tier2_fill_synthetic": (st, [vp, u64, u32, u32, vp]),
    "gh_tier2_read_kv": (st, [vp, u32, u32, u32, u32, u32, vp]),
    "gh_tier2_arena_bytes": (u64, [vp]),
    "gh_tier2_create_paged": (st, [P(GhSpec), C.c_int, u32, u32, u32, u32, P(vp)]),
    "gh_tier2_map": (st, [vp, u32, u32, vp]),
    "gh_tier2_unmap": (st, [vp, u32]),
    "gh_tier2_append": (st, [vp, u32, u32, vp, vp, vp, vp]),
    "gh_tier2_pages_free": (u32, [vp]),
    "gh_comm_unique_id": (st, [P(C.c_uint8)]),
    "gh_comm_create": (st, [P(C.c_uint8), C.c_int, C.c_int, C.c_int, P(vp)]),
    "gh_comm_create_n": (st, [P(C.c_uint8), C.c_int, C.c_int, C.c_int, C.c_int, P(vp)]),
    "gh_comm_destroy": (st, [vp]),
    "gh_engine_create": (st, [P(GhEngineConfig), vp, P(vp)]),
    "gh_engine_destroy": (st, [vp]),
    "gh_engine_role": (C.c_int, [vp]),
    "gh_engine_transport": (C.c_int, [vp]),
    "gh_engine_step_device": (st, [vp, u32, vp]),
    "gh_engine_step_host": (st, [vp, u32, vp, vp, vp, vp, vp]),
    "gh_engine_step_all": (st, [vp, vp]),
    "gh_engine_step_all_host": (st, [vp, vp, vp, vp, vp]),
    "gh_engine_io": (st, [vp, u32, P(vp), P(vp), P(vp), P(vp)]),
    "gh_engine_advance": (st, [vp, u32, C.c_int, vp]),
    "gh_engine_read_next": (st, [vp, u32, vp]),
    "gh_engine_layout": (st, [u32, u32, u32, u32, u64, u32, P(GhRankLayout)]),
    "gh_dispatcher_create": (st, [vp, P(GhDispatchConfig), P(vp)]),
    "gh_dispatcher_destroy": (st, [vp]),
    "gh_dispatcher_submit": (st, [vp, vp, u32, C.c_float, u32, u32, P(u64)]),
    "gh_dispatcher_step": (st, [vp, P(C.c_int)]),
    "gh_dispatcher_run": (st, [vp, P(u64)]),
    "gh_dispatcher_result": (st, [vp, u64, vp, u32, P(u32)]),
    "gh_dispatcher_stats": (st, [vp, P(GhDispatchStats)]),
    "gh_sched_create": (st, [P(GhSchedConfig), P(vp)]),
    "gh_sched_destroy": (st, [vp]),
    "gh_sched_submit": (st, [vp, vp, u32, C.c_float, u32, u32, P(u64)]),
    "gh_sched_plan": (st, [vp, P(GhLaneInput), P(GhKvAction), u32, P(u32)]),
    "gh_sched_commit": (st, [vp]),
    "gh_sched_resolve": (st, [vp, vp]),
    "gh_sched_done": (C.c_int, [vp]),
    "gh_sched_unresolved": (u32, [vp]),
    "gh_sched_result": (st, [vp, u64, vp, u32, P(u32)]),
    "gh_sched_stats": (st, [vp, P(GhDispatchStats)]),
    "gh_engine_keep_logits": (st, [vp, C.c_int]),
    "gh_engine_read_logits": (st, [vp, u32, vp]),
    "gh_engine_tier1": (vp, [vp]),
    "gh_engine_tier2": (vp, [vp]),
    "gh_engine_kv_map": (st, [vp, u32, u32]),
    "gh_engine_kv_unmap": (st, [vp, u32]),
    "gh_engine_kv_swap": (st, [vp, u32, u32, vp, C.c_int]),
    "gh_engine_kv_swap_bytes": (C.c_uint64, [vp, u32]),
    "gh_tier2_kv_swap": (st, [vp, u32, u32, vp, C.c_int, vp]),
    "gh_tier2_kv_swap_bytes": (C.c_uint64, [vp, u32]),
    "gh_engine_set_slots": (st, [vp, u32, P(u32)]),
    "gh_engine_shard": (st, [vp, P(C.c_int), P(u32), P(u32), P(u32)]),
    "gh_engine_set_sampling": (st, [vp, u32, P(C.c_float), P(u32)]),
    "gh_tier1_classify_sample": (st, [vp, u32, vp, vp, vp, vp, vp, vp, vp]),
    "gh_kernel_launches": (u64, [C.c_int]),
    "gh_debug_gemm_bench": (st, [C.c_int] * 7 + [P(C.c_float)]),
    "gh_debug_gemm_profile": (st, [C.c_int]),
    "gh_debug_gemm_profile_dump": (st, [C.c_char_p, u64]),
    "gh_debug_gemm_trace": (st, [C.c_int] * 5 + [P(C.c_float), P(C.c_uint64), C.c_int]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree libgh.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: the CUDA extension has not been built "
                               "(run __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != GH_OK:
        msg = lib().gh_last_error().decode(errors="replace")
        raise _ERR.get(status, GhError)(status, msg)


def ptr(x) -> int | None:
    """Device/host pointer of a torch tensor, numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")
