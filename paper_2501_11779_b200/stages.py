"""Host-side mirror of the two-tier stage interface (Glinthawk compute kernels).

Stage taxonomy and names follow the reference (proj/include/tierplan/profiles.hpp:13):
``nonattention`` = Tier-1 F1 (``pre``) + F3 (``post``), ``attention`` = Tier-2 F2 (``attend``),
``classifier`` = Tier-1 ``classify``.  Every method is a thin call through the C ABI; device
buffers are torch tensors (plumbing only) passed by address, streams are torch CUDA streams.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .spec import ModelSpec


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def _torch_dtype(spec: ModelSpec):
    import torch
    return {4: torch.float32, 2: torch.bfloat16}[spec.dtype_bytes]


class Tier1:
    """Weight-holding stage for layers [layer_begin, layer_end) (a layer_spans block)."""

    def __init__(self, spec: ModelSpec, device: int = 0, layer_begin: int = 0,
                 layer_end: int | None = None, weight_seed: int = 1234, max_batch: int = 64):
        self.spec = spec
        self.layer_begin, self.layer_end = layer_begin, spec.n_layers if layer_end is None else layer_end
        h = C.c_void_p()
        L.check(L.lib().gh_tier1_create(C.byref(spec.c()), device, self.layer_begin, self.layer_end,
                                        weight_seed, max_batch, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and L is not None and L.lib is not None:
            L.lib().gh_tier1_destroy(self.h)
            self.h = None

    __del__ = close

    def embed(self, tok, x, stream=None):
        L.check(L.lib().gh_tier1_embed(self.h, tok.shape[0], L.ptr(tok), L.ptr(x), _stream(stream)))

    def pre(self, layer: int, x, pos, msg_fwd, stream=None):
        """F1 -> fwd message [x|q|k|v]"""
        L.check(L.lib().gh_tier1_pre(self.h, layer, x.shape[0], L.ptr(x), L.ptr(pos), L.ptr(msg_fwd),
                                     _stream(stream)))

    def post(self, layer: int, msg_bwd, x_next, stream=None):
        """F3 from bwd message [x|attn]"""
        L.check(L.lib().gh_tier1_post(self.h, layer, msg_bwd.shape[0], L.ptr(msg_bwd), L.ptr(x_next),
                                      _stream(stream)))

    def classify(self, x, next_tok, logits=None, stream=None):
        L.check(L.lib().gh_tier1_classify(self.h, x.shape[0], L.ptr(x), L.ptr(logits), L.ptr(next_tok),
                                          _stream(stream)))


class Tier2:
    """KV-context stage: n_slots prompt slots for layers [layer_begin, layer_end).  With
    n_pages > 0 the arena is a pool of n_pages pages of PAGE_POSITIONS positions shared by the
    slots (map() before a step attends a position, unmap() returns the pages)."""

    PAGE_POSITIONS = 64  # GH_KV_PAGE_POSITIONS

    def __init__(self, spec: ModelSpec, n_slots: int, device: int = 0, layer_begin: int = 0,
                 layer_end: int | None = None, n_pages: int = 0):
        self.spec = spec
        self.n_slots = n_slots
        self.n_pages = n_pages
        self.layer_begin, self.layer_end = layer_begin, spec.n_layers if layer_end is None else layer_end
        h = C.c_void_p()
        if n_pages:
            L.check(L.lib().gh_tier2_create_paged(C.byref(spec.c()), device, self.layer_begin, self.layer_end,
                                                  n_slots, n_pages, C.byref(h)))
        else:
            L.check(L.lib().gh_tier2_create(C.byref(spec.c()), device, self.layer_begin, self.layer_end,
                                            n_slots, C.byref(h)))
        self.h = h

    def map(self, slot: int, n_positions: int, stream=None):
        L.check(L.lib().gh_tier2_map(self.h, slot, n_positions, _stream(stream)))

    def unmap(self, slot: int):
        L.check(L.lib().gh_tier2_unmap(self.h, slot))

    @property
    def pages_free(self) -> int:
        return L.lib().gh_tier2_pages_free(self.h)

    def close(self):
        if getattr(self, "h", None) and L is not None and L.lib is not None:
            L.lib().gh_tier2_destroy(self.h)
            self.h = None

    __del__ = close

    @property
    def arena_bytes(self) -> int:
        return L.lib().gh_tier2_arena_bytes(self.h)

    def check(self, slot: np.ndarray, pos: np.ndarray):
        s = np.ascontiguousarray(slot, dtype=np.uint32)
        p = np.ascontiguousarray(pos, dtype=np.int32)
        L.check(L.lib().gh_tier2_check(self.h, len(s), s.ctypes.data_as(C.POINTER(C.c_uint32)),
                                       p.ctypes.data_as(C.POINTER(C.c_int32))))

    def attend(self, layer: int, slot, pos, msg_fwd, msg_bwd, stream=None):
        """F2: append + attention"""
        L.check(L.lib().gh_tier2_attend(self.h, layer, msg_fwd.shape[0], L.ptr(slot), L.ptr(pos),
                                        L.ptr(msg_fwd), L.ptr(msg_bwd), _stream(stream)))

    def append(self, layer: int, slot, pos, msg_fwd, stream=None):
        """KV append of every row without attention (rows of one prompt in one step)."""
        L.check(L.lib().gh_tier2_append(self.h, layer, msg_fwd.shape[0], L.ptr(slot), L.ptr(pos),
                                        L.ptr(msg_fwd), _stream(stream)))

    def fill_synthetic(self, seed: int, n_slots: int, n_positions: int, stream=None):
        L.check(L.lib().gh_tier2_fill_synthetic(self.h, seed, n_slots, n_positions, _stream(stream)))

    def read_kv(self, layer: int, slot: int, kv: int, head: int, n: int) -> np.ndarray:
        out = np.empty((n, self.spec.d_head), dtype=np.float32 if self.spec.dtype_bytes == 4 else np.uint16)
        L.check(L.lib().gh_tier2_read_kv(self.h, layer, slot, kv, head, n, out.ctypes.data))
        return out


def message_buffers(spec: ModelSpec, B: int, device: int = 0):
    """(x, msg_fwd, msg_bwd) device buffers with the PayloadModel layouts."""
    import torch
    dt = _torch_dtype(spec)
    dev = torch.device("cuda", device)
    x = torch.zeros(B, spec.d_model, dtype=dt, device=dev)
    fwd = torch.zeros(B, 2 * spec.d_model + 2 * spec.d_kv, dtype=dt, device=dev)
    bwd = torch.zeros(B, 2 * spec.d_model, dtype=dt, device=dev)
    return x, fwd, bwd


class Comm:
    """NCCL transport (one communicator per in-flight batch); ids from rank 0."""

    @staticmethod
    def unique_ids(n: int) -> bytes:
        out = b""
        for _ in range(n):
            buf = (C.c_uint8 * 128)()
            L.check(L.lib().gh_comm_unique_id(buf))
            out += bytes(buf)
        return out

    def __init__(self, ids: bytes, nranks: int, rank: int, device: int):
        n = len(ids) // 128
        buf = (C.c_uint8 * len(ids)).from_buffer_copy(ids)
        h = C.c_void_p()
        L.check(L.lib().gh_comm_create_n(buf, n, nranks, rank, device, C.byref(h)))
        self.h, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if getattr(self, "h", None):
            L.lib().gh_comm_destroy(self.h)
            self.h = None


class Engine:
    """One decode step over all layers: colocated (1 GPU) or tier split (rank 0 Tier-1,
    ranks 1.. Tier-2, PayloadModel messages every layer over peer copies or NCCL send/recv)."""

    ROLES = {0: "colocated", 1: "tier1", 2: "tier2"}
    TRANSPORTS = {"auto": 0, "nccl": 1, "peer": 2}

    def __init__(self, spec: ModelSpec, batch: int, inflight: int = 1, device: int = 0,
                 weight_seed: int = 1234, n_slots: int = 0, use_graph: bool = True,
                 comm: Comm | None = None, transport: str = "auto", tier1_ranks: int = 1,
                 kv_pages: int = 0, prefill: bool = False, tier1_tp: int = 1):
        self.spec, self.batch, self.inflight = spec, batch, inflight
        self.kv_pages = kv_pages
        self.prefill = prefill
        self.n_slots = n_slots or batch * inflight
        cfg = L.GhEngineConfig(spec.c(), device, weight_seed, batch, inflight, n_slots, int(use_graph),
                               self.TRANSPORTS[transport], tier1_ranks, int(prefill), kv_pages, tier1_tp)
        h = C.c_void_p()
        L.check(L.lib().gh_engine_create(C.byref(cfg), comm.h if comm else None, C.byref(h)))
        self.h = h
        self.comm = comm
        self.role = self.ROLES[L.lib().gh_engine_role(h)]
        self._pinned = {}
        self._swap_pool = []              # pinned host buffers recycled by kv_swap_out / kv_swap_in

    def close(self):
        if getattr(self, "h", None) and L is not None and L.lib is not None:
            L.lib().gh_engine_destroy(self.h)
            self.h = None

    __del__ = close

    @property
    def transport(self) -> str | None:
        """Inter-tier transport of the pipelined step ("nccl" / "peer"), None when colocated."""
        t = L.lib().gh_engine_transport(self.h)
        return {1: "nccl", 2: "peer"}.get(t)

    @property
    def tier2(self) -> int:
        return L.lib().gh_engine_tier2(self.h)

    def kv_map(self, slot: int, n_positions: int):
        """Paged KV: back positions [0, n_positions) of a slot with pages (no-op when contiguous)."""
        L.check(L.lib().gh_engine_kv_map(self.h, slot, n_positions))

    def kv_unmap(self, slot: int):
        L.check(L.lib().gh_engine_kv_unmap(self.h, slot))

    def kv_swap_out(self, slot: int, n_positions: int):
        """Copy positions [0, n) of a slot's context (every owned layer) to a pinned host buffer
        (page-locked, so the copies run at PCIe speed; buffers are recycled by kv_swap_in)."""
        import torch
        nbytes = L.lib().gh_engine_kv_swap_bytes(self.h, n_positions)
        pool = self._swap_pool
        fit = [i for i, b in enumerate(pool) if b.numel() >= nbytes]
        if fit:
            buf = pool.pop(min(fit, key=lambda i: pool[i].numel()))
        else:
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        L.check(L.lib().gh_engine_kv_swap(self.h, slot, n_positions, buf.data_ptr(), 1))
        return buf

    def kv_swap_in(self, slot: int, n_positions: int, buf):
        """Restore a kv_swap_out buffer into a slot mapped for n positions."""
        assert buf.numel() >= L.lib().gh_engine_kv_swap_bytes(self.h, n_positions)
        L.check(L.lib().gh_engine_kv_swap(self.h, slot, n_positions, buf.data_ptr(), 0))
        self._swap_pool.append(buf)

    def set_sampling(self, temperature, seed, ib=0):
        """Per-row temperature (0 = greedy) and seed of in-flight batch ib."""
        t = np.ascontiguousarray(temperature, dtype=np.float32)
        sd = np.ascontiguousarray(seed, dtype=np.uint32)
        L.check(L.lib().gh_engine_set_sampling(self.h, ib, t.ctypes.data_as(C.POINTER(C.c_float)),
                                               sd.ctypes.data_as(C.POINTER(C.c_uint32))))

    def shard(self):
        """(index, row offset, row count, K'): the rows whose KV this rank holds (Tier-2), or
        (-1, 0, batch, K') for Tier-1 / colocated ranks."""
        i, o, c, k = C.c_int(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        L.check(L.lib().gh_engine_shard(self.h, C.byref(i), C.byref(o), C.byref(c), C.byref(k)))
        return i.value, o.value, c.value, k.value

    def set_slots(self, slots, ib=0):
        """Context slot of every row of in-flight batch ib (colocated)."""
        s = np.ascontiguousarray(slots, dtype=np.uint32)
        L.check(L.lib().gh_engine_set_slots(self.h, ib, s.ctypes.data_as(C.POINTER(C.c_uint32))))

    def step_host(self, tok: np.ndarray | None, pos: np.ndarray | None, want_logits=False, ib=0,
                  stream=None):
        """End-to-end step through host buffers; returns (next_tokens, logits or None)."""
        if self.role == "tier2":
            L.check(L.lib().gh_engine_step_host(self.h, ib, None, None, None, None, _stream(stream)))
            return None, None
        t = np.ascontiguousarray(tok, dtype=np.int32)
        p = np.ascontiguousarray(pos, dtype=np.int32)
        nxt = np.empty(self.batch, dtype=np.int32)
        lg = np.empty((self.batch, self.spec.vocab_size), dtype=np.float32) if want_logits else None
        L.check(L.lib().gh_engine_step_host(self.h, ib, t.ctypes.data, p.ctypes.data, nxt.ctypes.data,
                                            None if lg is None else lg.ctypes.data, _stream(stream)))
        return nxt, lg

    def step_all_host(self, tok: np.ndarray | None, pos: np.ndarray | None, stream=None):
        """End-to-end pipelined step over all in-flight batches: tok/pos [inflight, batch] int32
        host arrays in, next tokens [inflight, batch] out (Tier-2 ranks pass None)."""
        if self.role == "tier2":
            L.check(L.lib().gh_engine_step_all_host(self.h, None, None, None, _stream(stream)))
            return None
        t = np.ascontiguousarray(tok, dtype=np.int32).reshape(self.inflight, self.batch)
        p = np.ascontiguousarray(pos, dtype=np.int32).reshape(self.inflight, self.batch)
        nxt = np.empty((self.inflight, self.batch), dtype=np.int32)
        L.check(L.lib().gh_engine_step_all_host(self.h, t.ctypes.data, p.ctypes.data, nxt.ctypes.data,
                                                _stream(stream)))
        return nxt

    def step_device(self, ib=0, stream=None):
        L.check(L.lib().gh_engine_step_device(self.h, ib, _stream(stream)))

    def step_all(self, stream=None):
        L.check(L.lib().gh_engine_step_all(self.h, _stream(stream)))

    def read_next(self, ib=0) -> np.ndarray:
        out = np.empty(self.batch, dtype=np.int32)
        L.check(L.lib().gh_engine_read_next(self.h, ib, out.ctypes.data))
        return out

    def keep_logits(self, keep: bool = True):
        """Every classifier run also writes its fp32 logits (read them with read_logits)."""
        L.check(L.lib().gh_engine_keep_logits(self.h, int(keep)))

    def read_logits(self, ib=0) -> np.ndarray:
        out = np.empty((self.batch, self.spec.vocab_size), dtype=np.float32)
        L.check(L.lib().gh_engine_read_logits(self.h, ib, out.ctypes.data))
        return out

    def advance(self, ib=0, pos_increment=0, stream=None):
        L.check(L.lib().gh_engine_advance(self.h, ib, pos_increment, _stream(stream)))


class Dispatcher:
    """Greedy decode driver over an Engine (Dispatcher): prompt i of the batch owns
    context slot i; prompt tokens are fed one per step (the dispatcher does not distinguish
    input and output tokens) and generation continues greedily."""

    def __init__(self, engine: Engine):
        self.engine = engine

    def generate(self, prompts: np.ndarray, max_new: int, want_logits=False):
        prompts = np.asarray(prompts, dtype=np.int32)
        B, plen = prompts.shape
        assert B == self.engine.batch
        tok = prompts[:, 0].copy()
        out, logits = [], []
        for t in range(plen - 1 + max_new):
            pos = np.full(B, t, dtype=np.int32)
            nxt, lg = self.engine.step_host(tok, pos, want_logits=want_logits)
            if t + 1 < plen:
                tok = prompts[:, t + 1].copy()
            else:
                out.append(nxt.copy())
                if want_logits:
                    logits.append(lg)
                tok = nxt
        gen = np.stack(out, axis=1) if out else np.zeros((B, 0), np.int32)
        return gen, (np.stack(logits, axis=1) if want_logits else None)


class Scheduler:
    """The dispatcher's decision logic (C++ gh_sched, host only): batch-state objects of IF
    in-flight batches x B lanes with per-shard page accounting (sched.hpp).
    plan() -> (inputs [lanes] of (src, tok, pos, home), KV actions); the caller runs the step, then
    commit(), and resolve(next tokens) for the oldest committed step (any lag).  `home` is the lane
    whose slot the row appends to and attends over: the row's own lane, or with chunked prefill
    (chunk > 1) the lane whose prompt token an otherwise idle row carries."""

    SRC_IDLE, SRC_HOST, SRC_DEVICE = 0, 1, 2
    MAP, UNMAP, SWAP_OUT, SWAP_IN = 0, 1, 2, 3

    def __init__(self, batch: int, max_new: int, inflight: int = 1, kp: int = 0, pages: int = 0, max_seq: int = 0,
                 on_demand: bool = False, preempt: str = "recompute", order: str = "fifo", chunk: int = 1):
        cfg = L.GhSchedConfig(batch, inflight, kp, pages, max_seq, max_new, int(on_demand), int(preempt == "swap"),
                              int(order == "shortest"), chunk)
        h = C.c_void_p()
        L.check(L.lib().gh_sched_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.lanes = batch * inflight
        self._in = (L.GhLaneInput * self.lanes)()
        self._acts = (L.GhKvAction * (8 * self.lanes + 16))()

    def close(self):
        if getattr(self, "h", None) and L is not None and L.lib is not None:
            L.lib().gh_sched_destroy(self.h)
            self.h = None

    __del__ = close

    def submit(self, prompt, temperature: float = 0.0, seed: int = 0, max_new: int = 0) -> int:
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        i = C.c_uint64()
        L.check(L.lib().gh_sched_submit(self.h, p.ctypes.data, len(p), temperature, seed, max_new, C.byref(i)))
        return i.value

    def plan(self):
        n = C.c_uint32()
        L.check(L.lib().gh_sched_plan(self.h, self._in, self._acts, len(self._acts), C.byref(n)))
        ins = np.array([(x.src, x.tok, x.pos, x.home) for x in self._in], np.int32).reshape(self.lanes, 4)
        return ins, [(a.op, a.lane, a.n, a.buf) for a in self._acts[:n.value]]

    def commit(self):
        L.check(L.lib().gh_sched_commit(self.h))

    def resolve(self, next_tokens=None):
        p = None if next_tokens is None else np.ascontiguousarray(next_tokens, dtype=np.int32)
        L.check(L.lib().gh_sched_resolve(self.h, None if p is None else p.ctypes.data))

    @property
    def done(self) -> bool:
        return bool(L.lib().gh_sched_done(self.h))

    @property
    def unresolved(self) -> int:
        return L.lib().gh_sched_unresolved(self.h)

    def result(self, i: int) -> np.ndarray:
        return _result(L.lib().gh_sched_result, self.h, i)

    def stats(self) -> dict:
        o = L.GhDispatchStats()
        L.check(L.lib().gh_sched_stats(self.h, C.byref(o)))
        return {f: getattr(o, f) for f, _ in o._fields_}


def _result(fn, h, i):
    n = C.c_uint32()
    L.check(fn(h, i, None, 0, C.byref(n)))
    out = np.empty(n.value, np.int32)
    L.check(fn(h, i, out.ctypes.data, n.value, C.byref(n)))
    return out


class ContinuousDispatcher:
    """Continuous batching with context-slot reuse -- a thin wrapper over
    the native batch-state dispatcher (gh_dispatcher_*, C++ sched.hpp / runtime.cu).

    The engine's IF x B rows are decode lanes, each bound to its own context slot; a request
    occupies a lane from its first prompt token until it has generated `max_new` tokens, and the
    lane (with its slot) then goes to the next queued request at position 0.  Every step decodes
    all busy lanes of every in-flight batch at their own positions through gh_engine_step_all
    (the pipelined tier split, or the colocated CUDA graphs); lane inputs, page tables and the
    sampling state are updated stream-ordered, and a step's tokens are read one step later.

    With a paged KV arena (Engine(kv_pages=...)) a request maps exactly the positions it will
    attend (prompt + max_new - 1) when it is admitted and returns its pages when it finishes; a
    request waits in the queue while its shard's pool cannot back it.  ``on_demand=True`` maps
    only the prompt and grows a page at a time; when a shard's pool is dry its most recently
    admitted request is preempted -- recomputed (``preempt="recompute"``: it re-enters the queue
    head and re-reads its prompt plus the tokens it generated) or swapped to host memory
    (``preempt="swap"``: restored into a lane of the same Tier-2 shard, resuming at its saved
    position).  ``order="shortest"`` admits the shortest prompts first.  ``chunk > 1`` (an
    Engine(prefill=True)) is chunked prefill: the idle lanes of a batch's shard carry up
    to chunk - 1 further prompt tokens of a request still reading its prompt, at consecutive
    positions of that request's slot, so a prompt of n tokens needs as few as ceil(n / chunk)
    steps when lanes are free.

    Tier split: every rank runs the same dispatcher over the same requests (SPMD); decisions depend
    only on lengths, max_new and page counts.  Tier-2 ranks apply their shard's KV actions;
    Tier-1 ranks (every tensor-parallel one) feed tokens.  Engines that are not an ``Engine`` (test
    doubles with kv_map / kv_unmap / kv_swap_out / kv_swap_in / set_sampling / step_host / shard)
    are driven by the same native decision logic (gh_sched) from Python."""

    PAGE = 64  # GH_KV_PAGE_POSITIONS

    def __init__(self, engine, on_demand: bool = False, preempt: str = "recompute", order: str = "fifo",
                 chunk: int = 1):
        if chunk > 1 and not (isinstance(engine, Engine) and engine.prefill):
            raise L.ValidationError(L.GH_EINVAL, "chunked prefill needs an Engine(prefill=True)")
        if preempt not in ("recompute", "swap"):
            raise ValueError(f"preempt must be 'recompute' or 'swap', not {preempt!r}")
        if order not in ("fifo", "shortest"):
            raise ValueError(f"order must be 'fifo' or 'shortest', not {order!r}")
        self.engine, self.on_demand, self.preempt, self.order = engine, on_demand, preempt, order
        self.chunk = max(1, int(chunk))
        self.preemptions = 0
        self.stats = {}

    def run(self, requests, max_new, sampling=None):
        """requests: sequence of 1-D int32 prompts (any lengths >= 1); max_new: tokens to generate,
        one int for all requests or one per request; sampling: optional per-request (temperature,
        seed) pairs (temperature 0 = greedy).  Returns (generated token arrays in request order --
        zeros on Tier-2 ranks -- and the step count)."""
        per = np.broadcast_to(np.asarray(max_new, dtype=np.int64), (len(requests),))
        max_new = int(per.max()) if len(requests) else 1
        eng = self.engine
        on_demand = self.on_demand and eng.kv_pages > 0
        if not isinstance(eng, Engine):
            return self._run_host(requests, max_new, sampling, on_demand, per)
        cfg = L.GhDispatchConfig(max_new, int(on_demand), int(self.preempt == "swap"), int(self.order == "shortest"),
                                 self.chunk)
        h = C.c_void_p()
        L.check(L.lib().gh_dispatcher_create(eng.h, C.byref(cfg), C.byref(h)))
        try:
            ids = []
            for i, q in enumerate(requests):
                t, sd = sampling[i] if sampling is not None else (0.0, 0)
                p = np.ascontiguousarray(q, dtype=np.int32)
                rid = C.c_uint64()
                L.check(L.lib().gh_dispatcher_submit(h, p.ctypes.data, len(p), float(t), int(sd), int(per[i]),
                                                     C.byref(rid)))
                ids.append(rid.value)
            steps = C.c_uint64()
            L.check(L.lib().gh_dispatcher_run(h, C.byref(steps)))
            out = [_result(L.lib().gh_dispatcher_result, h, i) for i in ids]
            o = L.GhDispatchStats()
            L.check(L.lib().gh_dispatcher_stats(h, C.byref(o)))
            self.stats = {f: getattr(o, f) for f, _ in o._fields_}
        finally:
            L.lib().gh_dispatcher_destroy(h)
        self.preemptions = self.stats["preemptions"]
        return out, int(steps.value)

    def _run_host(self, requests, max_new, sampling, on_demand, per):
        """The native decision logic driving a duck-typed engine from Python, one step of lag."""
        from collections import deque
        eng = self.engine
        B = eng.batch
        _, off, cnt, kp = eng.shard()
        sch = Scheduler(B, max_new, 1, kp, eng.kv_pages, getattr(getattr(eng, "spec", None), "max_seq_len", 0),
                        on_demand, self.preempt, self.order)
        ids = [sch.submit(q, *(sampling[i] if sampling is not None else (0.0, 0)), max_new=int(per[i]))
               for i, q in enumerate(requests)]
        holds = lambda lane: eng.role != "tier1" and off <= lane < off + cnt  # noqa: E731
        bufs, hist = {}, deque()
        last = np.zeros(B, np.int32)
        while not sch.done:
            ins, acts = sch.plan()
            for op, lane, n, buf in acts:
                if not holds(lane):
                    continue
                if op == Scheduler.MAP:
                    eng.kv_map(lane - off, n)
                elif op == Scheduler.UNMAP:
                    eng.kv_unmap(lane - off)
                elif op == Scheduler.SWAP_OUT:
                    bufs[buf] = eng.kv_swap_out(lane - off, n)
                else:
                    eng.kv_swap_in(lane - off, n, bufs.pop(buf))
            if not (ins[:, 0] != Scheduler.SRC_IDLE).any():
                while sch.unresolved:
                    sch.resolve(hist.popleft())
                continue
            tok = np.where(ins[:, 0] == Scheduler.SRC_DEVICE, last, ins[:, 1]).astype(np.int32)
            if eng.role == "tier2":
                eng.step_host(None, None)
                nxt = np.zeros(B, np.int32)
            else:
                nxt, _ = eng.step_host(tok, ins[:, 2].copy())
            last = np.asarray(nxt, np.int32)
            sch.commit()
            hist.append(last.copy())
            if sch.unresolved > 1:
                sch.resolve(hist.popleft())
        while sch.unresolved:
            sch.resolve(hist.popleft())
        self.stats = sch.stats()
        self.preemptions = self.stats["preemptions"]
        out = [sch.result(i) for i in ids]
        steps = self.stats["steps"]
        sch.close()
        return out, steps


class MixedDispatcher:
    """Mixed prefill + decode batches: the engine's B rows are a pool, not
    lanes.  Every step, each admitted request in its decode phase takes one row (its last token);
    a request still reading its prompt takes up to `chunk` rows, one per prompt token at
    consecutive positions of its slot (chunked prefill), so a prompt of n tokens needs
    ceil(n / chunk) steps instead of n.  The engine runs with prefill=True: every row's key and
    value are appended before attention, so the rows of one prompt see each other's keys exactly
    as they would one token per step -- each request's tokens equal decoding it alone.  The
    row of a request's last prompt token yields its first generated token.  Rows left over hold
    a dummy token in a reserved scratch slot (the last slot).  With a paged arena a request maps
    prompt + max_new - 1 positions on admission (page accounting per Tier-2 shard, kept on every
    rank) and returns them when done; a request waits while no shard can back it.

    Tier split: every rank runs the dispatcher SPMD (admission depends only on lengths).  A
    request lives on one Tier-2 shard (its slot is a local slot of that rank) and only takes rows
    of that shard's row range; each Tier-2 rank installs the slots of its own rows."""

    def __init__(self, engine: Engine, chunk: int = 16):
        if not engine.prefill:
            raise L.ValidationError(L.GH_EINVAL, "MixedDispatcher needs Engine(prefill=True)")
        if engine.n_slots < 2:
            raise L.ValidationError(L.GH_EINVAL, "MixedDispatcher needs n_slots >= 2 (one scratch slot)")
        self.engine, self.chunk = engine, chunk

    def run(self, requests, max_new: int):
        """Returns (generated token arrays in request order (zeros on Tier-2 ranks), steps)."""
        eng, B = self.engine, self.engine.batch
        role = eng.role
        _, off, cnt, kp = eng.shard()
        if kp:
            from .spec import shard_plan
            offs, cnts = shard_plan(B, kp)
        else:
            offs, cnts = [0], [B]
        nsh = len(offs)
        scratch = eng.n_slots - 1         # a local slot of every shard
        free_slots = [list(range(eng.n_slots - 1)) for _ in range(nsh)]
        queue = list(range(len(requests)))
        active = [[] for _ in range(nsh)]  # per shard: [request, local slot, fed]
        out = [[] for _ in requests]
        holds_kv = role != "tier1"
        my_shard = next((j for j in range(nsh) if offs[j] == off), 0) if role == "tier2" else 0
        # page accounting per shard (kept on every rank so that all take the same decisions)
        paged = eng.kv_pages > 0
        pages_free = [eng.kv_pages - 1] * nsh if paged else [0] * nsh  # minus the scratch page

        def pages(n):
            return -(-n // ContinuousDispatcher.PAGE)

        def mine(j):                      # this rank holds shard j's KV
            return holds_kv and (role == "colocated" or j == my_shard)

        if holds_kv:
            eng.kv_map(scratch, 1)
        last_slots = None
        steps = 0
        while queue or any(active):
            # admission (FIFO): the shard with a free slot and the fewest active requests
            while queue:
                cand = [j for j in range(nsh) if free_slots[j]]
                if not cand:
                    break
                r = queue[0]
                need = pages(len(requests[r]) + max_new - 1) if paged else 0
                cand = [k for k in cand if need <= pages_free[k]]
                if not cand:
                    if not any(active):
                        raise L.FeasibilityError(L.GH_EINFEASIBLE,
                                                 f"request {r} needs more KV pages than a Tier-2 pool holds")
                    break
                j = min(cand, key=lambda k: (len(active[k]), k))
                s = free_slots[j][0]
                if mine(j):
                    eng.kv_map(s, len(requests[r]) + max_new - 1)
                pages_free[j] -= need
                queue.pop(0)
                free_slots[j].pop(0)
                active[j].append([r, s, 0])
            tok = np.zeros(B, np.int32)
            pos = np.zeros(B, np.int32)
            slots = np.full(B, scratch, np.uint32)
            emit = []                      # (row, entry) pairs whose next token is generated
            for j in range(nsh):
                row, end = offs[j], offs[j] + cnts[j]
                for a in active[j]:
                    r, s, fed = a
                    p = requests[r]
                    if row >= end:
                        break
                    if fed < len(p):       # prefill rows
                        n = min(self.chunk, len(p) - fed, end - row)
                        tok[row:row + n] = p[fed:fed + n]
                        pos[row:row + n] = np.arange(fed, fed + n)
                        slots[row:row + n] = s
                        if fed + n == len(p):
                            emit.append((row + n - 1, j, a))
                        a[2] = fed + n
                        row += n
                    else:                  # decode row: the last generated token
                        tok[row] = out[r][-1] if out[r] else 0
                        pos[row] = len(p) + len(out[r]) - 1
                        slots[row] = s
                        emit.append((row, j, a))
                        row += 1
            if last_slots is None or not np.array_equal(slots, last_slots):
                if role == "tier2":
                    eng.set_slots(slots[off:off + cnt])
                elif role == "colocated":
                    eng.set_slots(slots)
                last_slots = slots
            if role == "tier2":
                eng.step_host(None, None)
                nxt = np.zeros(B, np.int32)
            else:
                nxt, _ = eng.step_host(tok, pos)
            steps += 1
            for rw, j, a in emit:
                r = a[0]
                out[r].append(int(nxt[rw]))
                if len(out[r]) == max_new:
                    active[j].remove(a)
                    if mine(j):
                        eng.kv_unmap(a[1])
                    if paged:
                        pages_free[j] += pages(len(requests[r]) + max_new - 1)
                    free_slots[j].append(a[1])
        return [np.array(o, np.int32) for o in out], steps
