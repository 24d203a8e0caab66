"""SURVEY 8f-1, simulation fidelity on B200: the reference planner, fed this build's measured
stage latencies through its own plug-in boundary (the profile CSV, profiles.hpp:66-69), predicts
the throughput of a tier split (derive_two_tier_latencies optimizer.cpp:242-257 ->
simulate_two_tier des.cpp:261-281 -> throughput_from des.cpp:298-310); the same split is then run
on the GPUs and measured.  The paper's claim for its prototype is "simulation matches empirical
measurements"; here the measured / predicted ratio must lie in [0.75, 1.25].

Workload: C2 shape (Llama-2-7B, ctx 512), Tier-1 on GPU 0, one Tier-2 GPU, IF = 2 in-flight
batches of 64 prompts, peer transport.  The unmodified planner runs in-process from the prebuilt
oracle/_ref library (test infrastructure)."""
import re

import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from _ranks import collect, init_rank, spawn
from oracle import Ref, ref_available

pytestmark = pytest.mark.gpu

SPEC = gh.CONFIGS["C2"]["spec"]
CTX, B, IF, STEPS = 512, 64, 2, 20


def n_gpus():
    try:
        return gh.lib().gh_device_count()
    except Exception:
        return 0


def worker(rank, world, rdv, q):
    import torch
    import torch.distributed as dist
    from paper_2501_11779_b200 import _lib as L
    from paper_2501_11779_b200.stages import Comm, Engine
    torch.cuda.set_device(rank)
    init_rank(rank, world, rdv)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, rank)
    eng = Engine(SPEC, batch=B, inflight=IF, device=rank, use_graph=False, comm=comm, transport="peer")
    if eng.role == "tier2":
        L.check(gh.lib().gh_tier2_fill_synthetic(eng.tier2, 99, B * IF, CTX - 1, None))
    tok = np.random.default_rng(5678).integers(0, SPEC.vocab_size, size=(IF, B)).astype(np.int32)
    pos = np.full((IF, B), CTX - 1, np.int32)
    t1 = eng.role == "tier1"
    st = torch.cuda.Stream()
    eng.step_all_host(tok if t1 else None, pos if t1 else None, stream=st)
    for _ in range(3):
        eng.step_all(stream=st)
    st.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(STEPS):
        eng.step_all(stream=st)
        if t1:
            for ib in range(IF):
                eng.advance(ib, 0, stream=st)
    e1.record(st)
    st.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / STEPS], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    eng.close()
    comm.close()
    if rank == 0:
        q.put(float(ms.item()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(n_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.skipif(not ref_available(), reason="reference library not built")
def test_planner_prediction_matches_measured_split(tmp_path):
    from pathlib import Path
    from paper_2501_11779_b200.profiles import measure_stage_profile, write_profile
    root = Path(__file__).resolve().parents[1]
    rows = measure_stage_profile(SPEC, [16, 32, 64, 128], CTX, reps=10)
    t1, t2 = tmp_path / "b200_tier1.csv", tmp_path / "b200_tier2.csv"
    write_profile(t1, "b200-tier1", [r for r in rows if r[0] != "attention"])
    write_profile(t2, "b200-tier2", [r for r in rows if r[0] == "attention"])
    rc, rep = Ref.simulate(root / "configs/llama2-7b-ctx512.json", root / "configs/b200x8_cluster.json", t1, t2,
                           1, 1, B, CTX, inflight=IF)
    assert rc == 0, rep
    predicted = float(re.search(r"throughput: ([0-9.e+]+) tok/s", rep).group(1))
    procs, q = spawn(worker, 2)
    ms = collect(procs, q, 1, 300)[0]
    measured = B * IF / (ms / 1e3)
    ratio = measured / predicted
    print(f"planner {predicted:.0f} tok/s, measured {measured:.0f} tok/s ({ms:.2f} ms/step): ratio {ratio:.3f}")
    assert 0.75 <= ratio <= 1.25, (predicted, measured)
