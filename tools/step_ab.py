"""Colocated C2 step timed four ways (diagnostics): back-to-back graph replays with / without the
advance kernel, each step synchronised, and the end-to-end host path (wall clock).

  python tools/step_ab.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402
from paper_2501_11779_b200.stages import Engine  # noqa: E402
spec = gh.CONFIGS["C2"]["spec"]; B = 64; ctx = 512
eng = Engine(spec, batch=B, use_graph=True)
L.check(gh.lib().gh_tier2_fill_synthetic(eng.tier2, 99, B, ctx - 1, None))
tok = np.random.default_rng(1).integers(0, spec.vocab_size, B).astype(np.int32)
pos = np.full(B, ctx - 1, np.int32)
eng.step_host(tok, pos)
s = torch.cuda.Stream()
def dev(n, adv, sync):
    tot = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if not sync:
        e0.record(s)
        for _ in range(n):
            eng.step_device(stream=s)
            if adv: eng.advance(pos_increment=0, stream=s)
        e1.record(s); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    for _ in range(n):
        e0.record(s); eng.step_device(stream=s)
        if adv: eng.advance(pos_increment=0, stream=s)
        e1.record(s); torch.cuda.synchronize(); tot += e0.elapsed_time(e1)
    return tot / n
for _ in range(5): eng.step_device(stream=s)
torch.cuda.synchronize()
for rep in range(2):
    print("b2b no-adv %.3f | b2b adv %.3f | sync no-adv %.3f | sync adv %.3f" % (dev(20, 0, 0), dev(20, 1, 0), dev(20, 0, 1), dev(20, 1, 1)))
    t0 = time.perf_counter(); nxt = tok
    for _ in range(20): nxt, _ = eng.step_host(nxt, pos, stream=s)
    print("e2e wall %.3f" % ((time.perf_counter() - t0) * 1e3 / 20))
