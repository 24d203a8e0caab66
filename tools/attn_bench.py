"""Time the Tier-2 attention kernel alone (CUDA events, KV >> L2) at a batch / context.

  python tools/attn_bench.py [B] [ctx] [7b|13b|70b] [paged]   (paged: shuffled 64-position pages)
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200.stages import Tier2, message_buffers  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 512
layers = 4  # rotate layers so the KV of one launch is never L2-resident from the previous
model = sys.argv[3] if len(sys.argv) > 3 else "7b"
base = {"7b": gh.LLAMA2_7B, "13b": gh.CONFIGS["C4"]["spec"], "70b": gh.CONFIGS["C5"]["spec"]}[model]
spec = base.with_(n_layers=layers, max_seq_len=ctx)
paged = len(sys.argv) > 4 and sys.argv[4] == "paged"
per = -(-ctx // 64)
t2 = Tier2(spec, n_slots=B, n_pages=B * per if paged else 0)
if paged:  # round-robin mapping: consecutive pages of a slot are B pages apart
    for r in range(per):
        for s in range(B):
            t2.map(s, min((r + 1) * 64, ctx))
t2.fill_synthetic(99, B, ctx - 1)
x, fwd, bwd = message_buffers(spec, B)
fwd.normal_()
pos = torch.full((B,), ctx - 1, dtype=torch.int32, device="cuda")
slot = torch.arange(B, dtype=torch.int32, device="cuda")
for i in range(8):
    t2.attend(i % layers, slot, pos, fwd, bwd)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(os.environ.get("GH_REPS", "40"))
e0.record()
for i in range(reps):
    t2.attend(i % layers, slot, pos, fwd, bwd)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
byts = 2 * (2 * spec.d_kv * B * ctx + 2 * B * spec.d_kv + 2 * B * spec.d_model)
print(f"{model}{' paged' if paged else ''} B={B} ctx={ctx}: {us:.1f} us  {byts / us / 1e3:.0f} GB/s")
t2.close()
