"""Two colocated engines stepping concurrently on two streams of one B200 (diagnostics): does a
second independent chain of Tier-1 GEMMs fill the first one's kernel-boundary bubbles?  This is
the situation of a Tier-1 GPU with IF >= 2 in-flight batches (each batch streams the weights).

  python tools/concurrency_probe.py [--batch 64] [--ctx 2] [--steps 20]
"""
import argparse
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
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--ctx", type=int, default=2)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
spec = gh.CONFIGS["C2"]["spec"]
engs = []
for i in range(2):
    e = Engine(spec, batch=a.batch, use_graph=True)
    L.check(gh.lib().gh_tier2_fill_synthetic(e.tier2, 99 + i, a.batch, a.ctx - 1, None))
    tok = np.random.default_rng(i).integers(0, spec.vocab_size, a.batch).astype(np.int32)
    e.step_host(tok, np.full(a.batch, a.ctx - 1, np.int32))
    engs.append(e)
torch.cuda.synchronize()
ss = [torch.cuda.Stream(), torch.cuda.Stream()]


def run(which):
    for s in ss:
        s.synchronize()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ss[0])
    for s in ss[1:]:
        s.wait_event(e0)
    for _ in range(a.steps):
        for i in which:
            engs[i].step_device(stream=ss[i])
    for s in ss[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        ss[0].wait_event(ev)
    e1.record(ss[0])
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


for _ in range(2):
    run([0, 1])
one = run([0])
both = run([0, 1])
seq = run([0]) + run([1])
print(f"B={a.batch} ctx={a.ctx}: one engine {one:.3f} ms/step; two engines on two streams {both:.3f} ms "
      f"(sequential {seq:.3f} ms): concurrency gain {seq / both:.3f}x")
for e in engs:
    e.close()
