"""NCCL tier split on real GPUs (needs >= 2 GPUs; skipped otherwise): rank 0 = Tier-1, ranks
1.. = Tier-2 holding the KV of their prompt shard.  Tokens and logits must be identical to the
colocated engine (same kernels, same batch -> same arithmetic)."""

import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from _ranks import collect, init_rank, spawn

pytestmark = pytest.mark.gpu

SPEC = gh.ModelSpec("split-gpu", 3, 512, 512, 1024, 4, 4, 64, 2, 1500)
B, STEPS = 13, 6


def n_gpus():
    try:
        return gh.lib().gh_device_count()
    except Exception:
        return 0


def prompts():
    return np.random.default_rng(9).integers(0, SPEC.vocab_size, size=(B, 3), dtype=np.int32)


def run_engine(eng, ib_count=1):
    """Greedy decode of `prompts()` on in-flight batch 0 (and a second identical batch when
    ib_count == 2, decoded through gh_engine_step_all)."""
    p = prompts()
    tok = p[:, 0].copy()
    toks, logits = [], []
    for t in range(p.shape[1] - 1 + STEPS):
        pos = np.full(B, t, np.int32)
        nxt, lg = eng.step_host(tok, pos, want_logits=True)
        if eng.role == "tier2":
            continue
        if t + 1 < p.shape[1]:
            tok = p[:, t + 1].copy()
        else:
            toks.append(nxt)
            logits.append(lg)
            tok = nxt
    return (np.stack(toks, 1), np.stack(logits, 1)) if toks else (None, None)


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200.stages import Comm, Engine
    torch.cuda.set_device(rank)
    init_rank(rank, world, port)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, rank)
    eng = Engine(SPEC, batch=B, device=rank, use_graph=False, comm=comm)
    toks, lg = run_engine(eng)
    eng.close()
    comm.close()
    if rank == 0:
        q.put((toks, lg))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 3])
def test_nccl_tier_split_matches_colocated(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2501_11779_b200.stages import Engine
    procs, q = spawn(worker, world, ())
    toks, lg = collect(procs, q, 1, 300)[0]
    ref = Engine(SPEC, batch=B, use_graph=False)
    rtoks, rlg = run_engine(ref)
    ref.close()
    assert np.array_equal(toks, rtoks)
    assert np.array_equal(lg, rlg)


def worker_all(rank, world, port, q, IF, transport="auto"):
    """step_all (pipelined, all in-flight batches) + advance for STEPS steps."""
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200.stages import Comm, Engine
    torch.cuda.set_device(rank)
    init_rank(rank, world, port)
    comm = None
    if world > 1:
        obj = [Comm.unique_ids(1) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = Comm(obj[0], world, rank, rank)
    eng = Engine(SPEC, batch=B, inflight=IF, device=rank, use_graph=False, comm=comm, transport=transport)
    used = eng.transport
    out = run_all(eng, IF)
    if rank == 0:
        q.put((out, used))
    dist.barrier()
    dist.destroy_process_group()


def run_all(eng, IF):
    p = prompts()
    for ib in range(IF):  # step 0 through the host path sets tokens/positions of every batch
        eng.step_host(np.roll(p[:, 0], ib) if eng.role != "tier2" else None,
                      np.zeros(B, np.int32) if eng.role != "tier2" else None, ib=ib)
    seq = []
    for _ in range(STEPS):
        if eng.role != "tier2":
            for ib in range(IF):
                eng.advance(ib, 1)
        eng.step_all()
        if eng.role != "tier2":
            seq.append(np.stack([eng.read_next(ib) for ib in range(IF)]))
    eng.close()
    return np.stack(seq) if seq else None


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("world,IF", [(2, 2), (3, 2), (2, 3)])
def test_pipelined_step_all_matches_colocated(world, IF, transport):
    """Pipelined step_all over NCCL send/recv and over the peer-copy transport (CUDA IPC +
    copy engines + stream-ordered flags): tokens identical to the colocated engine."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2501_11779_b200.stages import Engine
    procs, q = spawn(worker_all, world, (IF, transport))
    got, used = collect(procs, q, 1, 300)[0]
    assert used == transport
    ref = run_all(Engine(SPEC, batch=B, inflight=IF, use_graph=False), IF)
    assert np.array_equal(got, ref)


def worker_pp(rank, world, port, q, IF, n1):
    """Tier-1 pipeline stages (n1 spans, each with its own Tier-2 ranks): step_all_host for the
    first step, then advance + step_all; the last span reports the next tokens."""
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200.stages import Comm, Engine
    torch.cuda.set_device(rank)
    init_rank(rank, world, port)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, rank)
    eng = Engine(SPEC, batch=B, inflight=IF, device=rank, use_graph=False, comm=comm, transport="peer",
                 tier1_ranks=n1)
    p = prompts()
    t1 = eng.role == "tier1"
    toks = np.stack([np.roll(p[:, 0], ib) for ib in range(IF)]) if t1 else None
    eng.step_all_host(toks, np.zeros((IF, B), np.int32) if t1 else None)
    seq = []
    for _ in range(STEPS):
        if t1:
            for ib in range(IF):
                eng.advance(ib, 1)
        eng.step_all()
        if t1:
            seq.append(np.stack([eng.read_next(ib) for ib in range(IF)]))
    eng.close()
    comm.close()
    if rank == n1 - 1:
        q.put(np.stack(seq))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(n_gpus() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("IF", [2, 3, 4])
def test_tier1_pipeline_stages_match_colocated(IF):
    """SURVEY 8(e) config-5 topology at small scale: 2 Tier-1 spans (layers split by
    layer_spans), each with a dedicated Tier-2 rank; the in-flight batches run as min(IF, spans)
    groups so the spans work on different groups at once, and the first span applies
    gh_engine_advance when a batch's next step starts.  Tokens identical to the colocated engine."""
    from paper_2501_11779_b200.stages import Engine
    world, n1 = 4, 2
    procs, q = spawn(worker_pp, world, (IF, n1))
    got = collect(procs, q, 1, 300)[0]
    ref = run_all(Engine(SPEC, batch=B, inflight=IF, use_graph=False), IF)
    assert np.array_equal(got, ref)


PSPEC = gh.ModelSpec("split-paged", 2, 512, 512, 1024, 4, 4, 256, 2, 1500)
PLENS = [3, 70, 1, 33, 129, 12, 64, 65, 8, 20, 100, 2]
PNEW = 5
PB = 6


def paged_requests():
    rng = np.random.default_rng(17)
    return [rng.integers(0, PSPEC.vocab_size, size=n, dtype=np.int32) for n in PLENS]


def worker_paged(rank, world, port, q, on_demand=False, preempt="recompute", IF=1, chunk=1):
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200.stages import Comm, ContinuousDispatcher, Engine
    torch.cuda.set_device(rank)
    init_rank(rank, world, port)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, rank)
    eng = Engine(PSPEC, batch=PB, inflight=IF, device=rank, use_graph=False, comm=comm, kv_pages=8 * IF,
                 prefill=chunk > 1)
    try:
        out, steps = ContinuousDispatcher(eng, on_demand=on_demand, preempt=preempt, chunk=chunk).run(
            paged_requests(), PNEW)
    except Exception as e:  # every rank takes the same decisions: report instead of hanging
        out, steps = repr(e), -1
    eng.close()
    comm.close()
    if rank == 0:
        q.put((out, steps))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("IF", [1, 2])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("on_demand,preempt", [(False, "recompute"), (True, "recompute"), (True, "swap")])
def test_continuous_batching_paged_tier_split(world, on_demand, preempt, IF):
    """Continuous batching on paged Tier-2 ranks (SURVEY 8f-2 in the tier split) through the
    native batch-state dispatcher driving the pipelined step (IF in-flight batches, peer
    transport): every rank runs the dispatcher SPMD; each Tier-2 rank maps its own shard's lanes
    from a pool smaller than its lanes x max_seq_len, so requests wait for pages (or, on demand,
    grow page by page and preempt the latest request of the shard).  Tokens identical to the
    colocated engine with contiguous slots."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    procs, q = spawn(worker_paged, world, (on_demand, preempt, IF))
    got, steps = collect(procs, q, 1, 300)[0]
    assert steps >= 0, got
    ref = Engine(PSPEC, batch=PB, use_graph=False)
    want, ref_steps = ContinuousDispatcher(ref).run(paged_requests(), PNEW)
    ref.close()
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
    if world == 2 and not on_demand and IF == 1:
        assert steps > ref_steps  # one Tier-2 pool of 8 pages for 6 lanes: requests waited


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world,on_demand", [(2, False), (3, True)])
def test_native_chunked_prefill_tier_split(world, on_demand):
    """Chunked prefill through the native dispatcher on the pipelined split (IF 2, peer
    transport, paged Tier-2 pools): an idle row takes further prompt tokens of a request of its
    own batch and shard, each Tier-2 rank installs its rows' slot tables stream-ordered.  Tokens
    identical to the colocated engine; fewer steps than one prompt token per step."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    procs, q = spawn(worker_paged, world, (on_demand, "recompute", 2, 8))
    got, steps = collect(procs, q, 1, 300)[0]
    assert steps >= 0, got
    procs, q = spawn(worker_paged, world, (on_demand, "recompute", 2, 1))
    _, steps_lane = collect(procs, q, 1, 300)[0]
    ref = Engine(PSPEC, batch=PB, use_graph=False)
    want, _ = ContinuousDispatcher(ref).run(paged_requests(), PNEW)
    ref.close()
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
    assert steps < steps_lane, (steps, steps_lane)


def worker_mixed(rank, world, port, q, kv_pages=0):
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200.stages import Comm, Engine, MixedDispatcher
    torch.cuda.set_device(rank)
    init_rank(rank, world, port)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, rank)
    eng = Engine(PSPEC, batch=12, n_slots=5, device=rank, use_graph=False, comm=comm, prefill=True,
                 kv_pages=kv_pages)
    try:
        out, steps = MixedDispatcher(eng, chunk=8).run(paged_requests(), PNEW)
    except Exception as e:  # every rank takes the same decisions: report instead of hanging
        out, steps = repr(e), -1
    eng.close()
    comm.close()
    if rank == 0:
        q.put((out, steps))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world,kv_pages", [(2, 0), (3, 0), (2, 7), (3, 6)])
def test_mixed_prefill_tier_split(world, kv_pages):
    """Chunked prefill in the tier split: requests live on one Tier-2 shard and take
    rows of that shard only; Tier-2 ranks append every row's key / value before attention.
    Tokens identical to the colocated engine at the same row count."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    procs, q = spawn(worker_mixed, world, (kv_pages,))
    got, steps = collect(procs, q, 1, 300)[0]
    assert steps >= 0, got
    ref = Engine(PSPEC, batch=12, use_graph=False)
    want, ref_steps = ContinuousDispatcher(ref).run(paged_requests(), PNEW)
    ref.close()
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
    if not kv_pages:
        assert steps < ref_steps


SPEC7B = gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=128)  # the C2 kernels' full width, two layers


def seven_b_requests():
    rng = np.random.default_rng(23)
    return [rng.integers(0, SPEC7B.vocab_size, size=int(n), dtype=np.int32) for n in rng.integers(1, 40, 12)]


def worker_7b(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200.stages import Comm, ContinuousDispatcher, Engine
    torch.cuda.set_device(rank)
    init_rank(rank, world, port)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, rank)
    eng = Engine(SPEC7B, batch=8, inflight=2, device=rank, use_graph=False, comm=comm, transport="peer")
    out, steps = ContinuousDispatcher(eng).run(seven_b_requests(), 6)
    eng.close()
    comm.close()
    if rank == 0:
        q.put((out, steps))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 3])
def test_7b_shape_split_dispatcher_matches_colocated(world):
    """The Llama-2-7B widths (D 4096, 32 heads, FFN 11008; two layers) through the native
    dispatcher on the pipelined split (IF 2, peer transport): every request's tokens identical to
    the colocated engine's (same batch per in-flight batch, hence the same GEMM plans)."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    procs, q = spawn(worker_7b, world)
    got, steps = collect(procs, q, 1, 300)[0]
    ref = Engine(SPEC7B, batch=8, inflight=2, use_graph=False)
    want, ref_steps = ContinuousDispatcher(ref).run(seven_b_requests(), 6)
    ref.close()
    assert steps == ref_steps
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
