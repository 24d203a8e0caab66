"""Paged KV oversubscription on one B200 (the planner's oversubscription factor,
optimizer.cpp:42-45, 194-207): the same KV budget as contiguous max_seq_len slots, filled with
prompts of ragged context lengths, admits more prompts per step.

  python tools/paged_bench.py [--kv-gb 120] [--ctx 2048] [--steps 10]

Prints one JSON line: contiguous (B_full prompts at ctx-1) and paged (every prompt at its own
context, drawn uniformly from [1, ctx), admitted while pages last) tokens/s, colocated engine,
Llama-2-7B shape, device-timed (CUDA events, back-to-back steps).
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GH_PKG_ROOT") or str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402
from paper_2501_11779_b200.stages import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kv-gb", type=float, default=120.0)
ap.add_argument("--ctx", type=int, default=2048)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
spec = gh.LLAMA2_7B.with_(max_seq_len=a.ctx)
PAGE = 64
per_prompt = 2 * spec.dtype_bytes * spec.n_layers * a.ctx * spec.d_kv
b_full = int(a.kv_gb * 1e9 // per_prompt)
pages = b_full * (a.ctx // PAGE)
rng = np.random.default_rng(5678)


def timed(eng, B, pos):
    tok = rng.integers(0, spec.vocab_size, B).astype(np.int32)
    eng.step_host(tok, pos)
    s = torch.cuda.Stream()
    for _ in range(a.warmup):
        eng.step_device(stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.steps):
        eng.step_device(stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


# contiguous arena: b_full slots of ctx positions, every prompt at ctx - 1
eng = Engine(spec, batch=b_full)
L.check(gh.lib().gh_tier2_fill_synthetic(eng.tier2, 99, b_full, a.ctx - 1, None))
ms_c = timed(eng, b_full, np.full(b_full, a.ctx - 1, np.int32))
eng.close()
torch.cuda.empty_cache()

# paged arena: the same bytes as pages; prompts of ragged context admitted while pages last
ctxs, used = [], 0
while True:
    c = int(rng.integers(1, a.ctx))
    need = -(-(c + 1) // PAGE)  # positions 0..c (the new token's key lands at c)
    if used + need > pages:
        break
    ctxs.append(c)
    used += need
B = len(ctxs)
eng = Engine(spec, batch=B, kv_pages=pages)
for s, c in enumerate(ctxs):
    eng.kv_map(s, c + 1)
L.check(gh.lib().gh_tier2_fill_synthetic(eng.tier2, 99, B, a.ctx, None))
ms_p = timed(eng, B, np.array(ctxs, np.int32))
eng.close()
kv_c = b_full * (a.ctx - 1) * per_prompt / a.ctx
kv_p = sum(ctxs) * per_prompt / a.ctx
print(json.dumps({
    "workload": f"7B shape colocated, KV budget {a.kv_gb:g} GB, max_seq_len {a.ctx}",
    "contiguous": {"prompts": b_full, "ctx": a.ctx - 1, "ms_per_step": ms_c, "tokens_per_s": b_full / ms_c * 1e3,
                   "kv_read_gb_per_step": kv_c / 1e9},
    "paged": {"prompts": B, "mean_ctx": float(np.mean(ctxs)), "pages": pages, "pages_used": used,
              "ms_per_step": ms_p, "tokens_per_s": B / ms_p * 1e3, "kv_read_gb_per_step": kv_p / 1e9},
    "oversubscription": B / b_full,
}))
