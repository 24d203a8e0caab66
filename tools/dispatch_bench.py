"""Continuous batching on a short paged KV pool, one B200, colocated 7B-shape engine: admission
that maps each request's whole length up front against on-demand paging with preemption
(ContinuousDispatcher(on_demand=True)), by recompute and by swap to host.

  python tools/dispatch_bench.py [--lanes 32] [--pages 96] [--requests 96] [--max-new 192]

Prints one JSON line per policy: steps, wall seconds (host loop, end to end through
Engine.step_host), generated tokens/s, preemptions.  All policies must produce identical tokens
(checked here).
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GH_PKG_ROOT") or str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lanes", type=int, default=32)
ap.add_argument("--pages", type=int, default=96)
ap.add_argument("--requests", type=int, default=96)
ap.add_argument("--max-new", type=int, default=192)
ap.add_argument("--layers", type=int, default=32)
a = ap.parse_args()
spec = gh.LLAMA2_7B.with_(n_layers=a.layers, max_seq_len=1024)
rng = np.random.default_rng(5678)
reqs = [rng.integers(0, spec.vocab_size, int(rng.integers(8, 96))).astype(np.int32) for _ in range(a.requests)]
res, toks = {}, {}
for name, od, pre in (("up_front", False, "recompute"), ("on_demand", True, "recompute"),
                      ("on_demand_swap", True, "swap")):
    eng = Engine(spec, batch=a.lanes, kv_pages=a.pages)
    d = ContinuousDispatcher(eng, on_demand=od, preempt=pre)
    d.run(reqs[:2], 4)  # warm-up (graph capture, clocks)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, steps = d.run(reqs, a.max_new)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    eng.close()
    toks[name] = out
    res[name] = {
        "steps": steps, "seconds": dt, "generated_tokens_per_s": a.requests * a.max_new / dt,
        "ms_per_step": 1e3 * dt / steps, "preemptions": d.preemptions}
same = all(np.array_equal(x, y) for n in toks for x, y in zip(toks["up_front"], toks[n]))
print(json.dumps({"workload": f"7B shape ({a.layers} layers) colocated, {a.lanes} lanes, pool {a.pages} pages of 64 "
                  f"positions, {a.requests} requests, prompts 8-95 tokens, {a.max_new} new tokens each",
                  **res, "tokens_identical": same}))
