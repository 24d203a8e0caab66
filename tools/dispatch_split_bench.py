"""Continuous batching in the tier split through the native dispatcher (SURVEY 8f-2 + the batch
state of P:471-479): every rank runs ContinuousDispatcher over the same requests (SPMD), the
engine step is the pipelined IF >= 2 split over the peer transport, Tier-2 pools are paged and
oversubscribed (on-demand growth with recompute preemption).

  torchrun --nproc-per-node 4 tools/dispatch_split_bench.py [--requests-per-lane 2] [--max-len 2048]

Workload (C3 shape: Llama-2-7B, max_seq_len 2048, K' = world - 1): lanes = IF x B with B = the
shard of bench.py --config C3 --paged (the prompts its pages hold at uniform contexts); each
Tier-2 GPU gets the pages of its two_tier_context_slots full-context slots.  Requests: prompt
length uniform in [1, 64), total length uniform in [64, max_len), so they finish at different
times and the queue refills lanes continuously.  Prints one JSON line (rank 0): steps, seconds,
lane-tokens per second (every busy lane of a step decodes one token: prompt or generated), generated
tokens per second, preemptions, and the mean context a busy lane attended.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.environ.get("GH_PKG_ROOT") or str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200.stages import Comm, ContinuousDispatcher, Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--requests-per-lane", type=float, default=2.0)
ap.add_argument("--max-len", type=int, default=2048)
ap.add_argument("--inflight", type=int, default=2)
ap.add_argument("--shard", type=int, default=163, help="lanes per Tier-2 GPU per in-flight batch")
a = ap.parse_args()

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
spec = gh.CONFIGS["C3"]["spec"]
kp = world - 1
slots = gh.two_tier_context_slots(spec, 1, kp, 179 << 30, spec.max_seq_len)
pages = slots // kp * (spec.max_seq_len // 64)
B = a.shard * kp
obj = [Comm.unique_ids(1) if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
comm = Comm(obj[0], world, rank, dev)
eng = Engine(spec, batch=B, inflight=a.inflight, device=dev, use_graph=False, comm=comm, transport="peer",
             kv_pages=pages)
rng = np.random.default_rng(4321)
n_req = int(a.requests_per_lane * B * a.inflight)
plen = rng.integers(1, 64, n_req)
total = rng.integers(64, a.max_len, n_req)
reqs = [rng.integers(0, spec.vocab_size, int(p)).astype(np.int32) for p in plen]
max_new = (total - plen).astype(np.int64)
warm = ContinuousDispatcher(eng, on_demand=True)
warm.run(reqs[: 2 * B * a.inflight], 2)  # warm-up: every lane once
torch.cuda.synchronize()
dist.barrier()
d = ContinuousDispatcher(eng, on_demand=True)
t0 = time.perf_counter()
out, steps = d.run(reqs, max_new)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
dist.barrier()
dts = torch.tensor([dt], dtype=torch.float64)
dist.all_reduce(dts, op=dist.ReduceOp.MAX)
dt = float(dts.item())
if rank == 0:
    lane_tokens = int(np.sum(plen - 1 + max_new))  # without recomputed positions
    st = d.stats
    print(json.dumps({
        "workload": f"C3 shape (7B, max_seq_len {spec.max_seq_len}), tier split 1 + {kp} GPUs, IF {a.inflight}, "
                    f"{B * a.inflight} lanes, {pages} pages of 64 positions per Tier-2 GPU ({slots // kp} full-context "
                    f"slots' worth), {n_req} requests: prompt U[1, 64), total length U[64, {a.max_len}), on-demand "
                    "paging with recompute preemption, native dispatcher (SPMD)",
        "steps": steps, "seconds": dt, "lane_tokens_per_s": st["lane_steps"] / dt,
        "request_tokens": lane_tokens, "recomputed_tokens": st["lane_steps"] - lane_tokens,
        "generated_tokens_per_s": int(np.sum(max_new)) / dt, "ms_per_step": 1e3 * dt / steps,
        "mean_context": st["context_sum"] / max(1, st["lane_steps"]),
        "mean_busy_lanes": st["lane_steps"] / max(1, steps),
        "preemptions": st["preemptions"], "admitted": st["admitted"], "peak_pages": st["peak_pages"]}))
eng.close()
comm.close()
dist.destroy_process_group()
