"""Small engine runs covering every kernel family, for compute-sanitizer (diagnostics):

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200.stages import Engine  # noqa: E402

cases = [
    (gh.ModelSpec("s-bf16", 2, 512, 512, 1024, 4, 4, 64, 2, 700), 20),      # split-K BN 32, MHA attention
    (gh.ModelSpec("s-gqa", 2, 1024, 256, 1536, 16, 4, 64, 2, 700), 9),      # GQA attention (G = 4)
    (gh.ModelSpec("s-b192", 2, 512, 512, 1024, 4, 4, 64, 2, 700), 192),     # 192-column split-K / pair
    (gh.ModelSpec("s-b300", 2, 512, 512, 1024, 4, 4, 64, 2, 700), 300),     # pair kernel, stream-K, unfused norm
    (gh.ModelSpec("s-fp32", 2, 288, 288, 768, 6, 6, 64, 4, 500), 4),        # fp32 SIMT path
]
for spec, B in cases:
    eng = Engine(spec, batch=B, use_graph=False)
    rng = np.random.default_rng(0)
    tok = rng.integers(0, spec.vocab_size, B).astype(np.int32)
    for t in range(3):
        nxt, _ = eng.step_host(tok, np.full(B, t, np.int32))
        tok = nxt
    eng.close()
    print(spec.name, B, "ok", flush=True)
