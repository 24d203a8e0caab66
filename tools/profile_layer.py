"""One decode layer (F1, F2, F3) + classifier of a config, repeated, for ncu / event timing.

  python tools/profile_layer.py [--config C2] [--reps 5] [--events]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200.stages import Tier1, Tier2, message_buffers  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--events", action="store_true")
a = ap.parse_args()
c = gh.CONFIGS[a.config]
spec, ctx = c["spec"].with_(n_layers=1), c["ctx"]
B = a.batch or c["batch"]
t1 = Tier1(spec, max_batch=B)
t2 = Tier2(spec, n_slots=B)
t2.fill_synthetic(99, B, ctx - 1)
x, fwd, bwd = message_buffers(spec, B)
x.normal_()
pos = torch.full((B,), ctx - 1, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()


def layer():
    t1.pre(0, x, pos, fwd)
    t2.attend(0, slot, pos, fwd, bwd)
    t1.post(0, bwd, x)
    t1.classify(x, nxt)


for _ in range(2):
    layer()
torch.cuda.synchronize()
if a.events:
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    res = np.zeros(4)
    for _ in range(a.reps):
        ev[0].record(); t1.pre(0, x, pos, fwd)
        ev[1].record(); t2.attend(0, slot, pos, fwd, bwd)
        ev[2].record(); t1.post(0, bwd, x)
        ev[3].record(); t1.classify(x, nxt)
        ev[4].record()
        torch.cuda.synchronize()
        res += [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(4)]
    print("us per call: pre %.1f attend %.1f post %.1f classify %.1f" % tuple(res / a.reps))
else:
    for _ in range(a.reps):
        layer()
    torch.cuda.synchronize()
print("ok")
