"""Chunked prefill mixed with decode vs one token per lane per step, 7B shape, one
B200, colocated, through the public dispatchers (wall clock): one token per lane per step
(ContinuousDispatcher, native), the Python pool-model MixedDispatcher (host tokens in / out every
step), and the native dispatcher's chunked prefill into idle lanes.

  python tools/prefill_bench.py [--requests 64] [--prompt 256 512] [--new 32] [--rows 256] [--chunk 64]

Prints one JSON line with the wall time, steps and tokens/s (prompt + generated) of each.
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
from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine, MixedDispatcher  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=64)
ap.add_argument("--prompt", type=int, nargs=2, default=[256, 512])
ap.add_argument("--new", type=int, default=32)
ap.add_argument("--rows", type=int, default=256)
ap.add_argument("--chunk", type=int, default=64)
a = ap.parse_args()
spec = gh.LLAMA2_7B.with_(max_seq_len=1024)
rng = np.random.default_rng(5678)
reqs = [rng.integers(0, spec.vocab_size, size=int(n), dtype=np.int32)
        for n in rng.integers(a.prompt[0], a.prompt[1] + 1, size=a.requests)]
tokens = sum(len(r) for r in reqs) + a.requests * a.new
res = {"workload": f"7B shape, {a.requests} requests, prompts {a.prompt[0]}-{a.prompt[1]} tokens, {a.new} new each",
       "tokens": tokens}


def run(name, eng, disp):
    disp.run(reqs[:2], 2)  # warm-up (graph capture, first-touch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out, steps = disp.run(reqs, a.new)
    dt = time.perf_counter() - t0
    eng.close()
    torch.cuda.empty_cache()
    res[name] = {"seconds": dt, "steps": steps, "ms_per_step": dt / steps * 1e3, "tokens_per_s": tokens / dt}
    return out


eng = Engine(spec, batch=a.requests)
lane = run("one_token_per_lane", eng, ContinuousDispatcher(eng))
eng = Engine(spec, batch=a.rows, n_slots=a.requests + 1, prefill=True)
mixed = run(f"mixed_rows{a.rows}_chunk{a.chunk}", eng, MixedDispatcher(eng, chunk=a.chunk))
# the native dispatcher's chunked prefill: rows = lanes (a paged arena: an idle lane holds one page),
# idle lanes carry prompt tokens of requests still reading their prompts, stream-ordered inputs
pages = a.requests * -(-(a.prompt[1] + a.new - 1) // 64) + a.rows
eng = Engine(spec, batch=a.rows, prefill=True, kv_pages=pages)
native = run(f"native_lanes{a.rows}_chunk{a.chunk}", eng, ContinuousDispatcher(eng, chunk=a.chunk))
# (token parity at equal row counts is tests/test_gpu_prefill.py; here the row counts differ, so
# the bf16 GEMM plans and roundings differ and greedy continuations of random weights may too)
print(json.dumps(res))
