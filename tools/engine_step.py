"""Colocated engine step at an arbitrary batch (diagnostics, e.g. under ncu):

  python tools/engine_step.py --batch 192 [--ctx 512] [--steps 3] [--layers 32]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

import os  # noqa: E402
sys.path.insert(0, os.environ.get("GH_PKG_ROOT") or str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402
from paper_2501_11779_b200.stages import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=192)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--graph", type=int, default=1)
a = ap.parse_args()
spec = gh.CONFIGS["C2"]["spec"].with_(n_layers=a.layers)
B = a.batch
eng = Engine(spec, batch=B, use_graph=bool(a.graph))
L.check(gh.lib().gh_tier2_fill_synthetic(eng.tier2, 99, B, a.ctx - 1, None))
tok = np.random.default_rng(1).integers(0, spec.vocab_size, B).astype(np.int32)
pos = np.full(B, a.ctx - 1, np.int32)
eng.step_host(tok, pos)
torch.cuda.synchronize()
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(a.steps):
    eng.step_device(stream=s)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(f"B={B} ctx={a.ctx} layers={a.layers}: {ms:.3f} ms/step, {B / ms * 1e3:.0f} tok/s")
if os.environ.get("GH_PROFILE_GEMMS") == "2":  # per-launch GEMM timeline of one more step (--graph 0)
    import ctypes
    gh.lib().gh_debug_gemm_profile(2)
    eng.step_device(stream=s)
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 20)
    gh.lib().gh_debug_gemm_profile_dump(buf, 1 << 20)
    print(buf.value.decode())
eng.close()
