"""Model shape contract and the reference's accounting functions.

``ModelSpec`` carries the nine TransformerSpec fields (proj/include/tierplan/model.hpp:14-28)
plus the two sidecar hyper-parameters (rope_theta, norm_eps) that the reference's strict model
JSON rejects (model.cpp:92-100).  ``to_reference_json`` writes the reference format unchanged,
``sidecar_json`` the extras.  Accounting functions call the C ABI (host-only, no GPU needed).
"""
from __future__ import annotations

import ctypes as C
import json
from collections import namedtuple
from dataclasses import asdict, dataclass, replace

from . import _lib as L


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    d_model: int
    d_kv: int
    d_hidden: int
    n_heads: int
    n_kv_heads: int
    max_seq_len: int
    dtype_bytes: int
    vocab_size: int = 0
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    def c(self) -> L.GhSpec:
        return L.GhSpec(self.n_layers, self.d_model, self.d_kv, self.d_hidden, self.n_heads,
                        self.n_kv_heads, self.max_seq_len, self.dtype_bytes, self.vocab_size,
                        self.rope_theta, self.norm_eps)

    def with_(self, **kw) -> "ModelSpec":
        return replace(self, **kw)

    # -- reference JSON (model.cpp:88-135: exactly these keys) + sidecar
    def to_reference_json(self) -> str:
        d = {k: v for k, v in asdict(self).items() if k not in ("rope_theta", "norm_eps")}
        if not d["vocab_size"]:
            d.pop("vocab_size")
        return json.dumps(d, indent=2)

    def sidecar_json(self) -> str:
        return json.dumps({"rope_theta": self.rope_theta, "norm_eps": self.norm_eps}, indent=2)

    @staticmethod
    def from_json(text: str, sidecar: str | None = None) -> "ModelSpec":
        d = json.loads(text)
        known = {"name", "n_layers", "d_model", "d_kv", "d_hidden", "n_heads", "n_kv_heads",
                 "max_seq_len", "dtype_bytes", "vocab_size"}
        unknown = set(d) - known
        if unknown:  # same strictness as the reference loader (model.cpp:92-100)
            raise L.ValidationError(L.GH_EINVAL, f"unknown model field '{sorted(unknown)[0]}'")
        extra = json.loads(sidecar) if sidecar else {}
        spec = ModelSpec(vocab_size=d.pop("vocab_size", 0), **d, **extra)
        spec.validate()
        return spec

    def validate(self) -> None:
        L.check(L.lib().gh_spec_validate(C.byref(self.c())))


# Configurations of BASELINE.json (SURVEY.md §8a shorthand C1..C5).  The 288/6 "stories15M"
# shape of C1 is the llama2.c convention (not in the reference).
TINY = ModelSpec("tiny-288x6", 6, 288, 288, 768, 6, 6, 256, 4, 32000)
LLAMA2_7B = ModelSpec("llama2-7b", 32, 4096, 4096, 11008, 32, 32, 4096, 2, 32000)
LLAMA2_13B = ModelSpec("llama2-13b", 40, 5120, 5120, 13824, 40, 40, 4096, 2, 32000)
LLAMA2_70B = ModelSpec("llama2-70b", 80, 8192, 1024, 28672, 64, 8, 8192, 2, 32000)
CONFIGS = {
    "C1": dict(spec=TINY, batch=4, ctx=None, gpus="1 (colocated)", steps=128, prompt_len=8),
    "C2": dict(spec=LLAMA2_7B.with_(max_seq_len=512), batch=64, ctx=512, gpus="1 (colocated)"),
    "C3": dict(spec=LLAMA2_7B.with_(max_seq_len=2048), batch=1024, ctx=2048, gpus="1 + 1/3/7"),
    "C4": dict(spec=LLAMA2_13B, batch=2048, ctx=4096, gpus="2/4/8 split"),
    "C5": dict(spec=LLAMA2_70B, batch=4096, ctx=8192, gpus="2 + 6"),
}


# ------------------------------------------------------------------ accounting (C ABI)
Payload = namedtuple("Payload", "tier1_to_tier2_per_token tier2_to_tier1_per_token intra_tier1_per_token")
Footprint = namedtuple("Footprint", "mem_accesses flops")


def _u64():
    return C.c_uint64(0)


def kv_bytes_per_prompt(spec: ModelSpec, seq_len: int) -> int:
    """model.cpp:40-46"""
    o = _u64()
    L.check(L.lib().gh_kv_bytes_per_prompt(C.byref(spec.c()), seq_len, C.byref(o)))
    return o.value


def nonattention_footprint(spec: ModelSpec, batch: int) -> Footprint:
    """model.cpp:48-56"""
    m, f = _u64(), _u64()
    L.check(L.lib().gh_nonattention_footprint(C.byref(spec.c()), batch, C.byref(m), C.byref(f)))
    return Footprint(m.value, f.value)


def attention_footprint(spec: ModelSpec, batch: int, seq_len: int) -> Footprint:
    """model.cpp:58-67"""
    m, f = _u64(), _u64()
    L.check(L.lib().gh_attention_footprint(C.byref(spec.c()), batch, seq_len, C.byref(m), C.byref(f)))
    return Footprint(m.value, f.value)


def weights_bytes(spec: ModelSpec) -> int:
    """model.cpp:69-77"""
    o = _u64()
    L.check(L.lib().gh_weights_bytes(C.byref(spec.c()), C.byref(o)))
    return o.value


def payload(spec: ModelSpec) -> Payload:
    """PayloadModel::for_model (netmodel.cpp:18-24)"""
    o = (C.c_uint64 * 3)()
    L.check(L.lib().gh_payload_bytes(C.byref(spec.c()), o))
    return Payload(*o)


def layer_spans(n_layers: int, nodes: int) -> list[int]:
    """optimizer.cpp:116-123"""
    o = (C.c_uint64 * max(nodes, 1))()
    L.check(L.lib().gh_layer_spans(n_layers, nodes, o))
    return list(o)


def node_weight_bytes(spec: ModelSpec, tier1_nodes: int) -> list[int]:
    """optimizer.cpp:125-136"""
    o = (C.c_uint64 * max(tier1_nodes, 1))()
    L.check(L.lib().gh_node_weight_bytes(C.byref(spec.c()), tier1_nodes, o))
    return list(o)


def two_tier_context_slots(spec: ModelSpec, tier1_nodes: int, tier2_per_tier1: int,
                           tier2_memory_per_node: int, seq_len: int) -> int:
    """optimizer.cpp:175-192"""
    o = _u64()
    L.check(L.lib().gh_two_tier_context_slots(C.byref(spec.c()), tier1_nodes, tier2_per_tier1,
                                              tier2_memory_per_node, seq_len, C.byref(o)))
    return o.value


def batch_grid(max_batch: int) -> list[int]:
    """profiles.cpp:232-245"""
    n = _u64()
    L.check(L.lib().gh_batch_grid(max_batch, None, 0, C.byref(n)))
    o = (C.c_uint64 * n.value)()
    L.check(L.lib().gh_batch_grid(max_batch, o, n.value, C.byref(n)))
    return list(o)


def throughput_from(gen_ts_ns, batch_total: int, inflight: int) -> float:
    """des.cpp:298-310: B_total * IF / mean(TBT)"""
    ts = (C.c_int64 * len(gen_ts_ns))(*gen_ts_ns)
    o = C.c_double(0)
    L.check(L.lib().gh_throughput_from(ts, len(gen_ts_ns), batch_total, inflight, C.byref(o)))
    return o.value


def shard_plan(batch: int, kp: int):
    """(offsets, counts) of the K' Tier-2 shards of a Tier-1 batch (analytic.cpp:119)."""
    off = (C.c_uint64 * max(kp, 1))()
    cnt = (C.c_uint64 * max(kp, 1))()
    L.check(L.lib().gh_shard_plan(batch, kp, off, cnt))
    return list(off), list(cnt)


def engine_layout(world: int, rank: int, batch: int, n_layers: int, tier1_ranks: int = 1, tier1_tp: int = 1) -> dict:
    """The engine's rank layout of a tier split (gh_engine_layout): role ("colocated" / "tier1" /
    "tier2"), span, tp_rank, shard, kp, layer range and the rows of each in-flight batch whose KV
    a Tier-2 rank holds."""
    out = L.GhRankLayout()
    L.check(L.lib().gh_engine_layout(world, rank, tier1_ranks, tier1_tp, n_layers, batch, C.byref(out)))
    return dict(role={0: "colocated", 1: "tier1", 2: "tier2"}[out.role], span=out.span, tp_rank=out.tp_rank,
                shard=out.shard, kp=out.kp, layers=(out.layer_begin, out.layer_end), rows=(out.row_off, out.row_cnt))
