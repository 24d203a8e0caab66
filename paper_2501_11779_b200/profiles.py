"""Kernel-latency profile emission — the reference's plug-in boundary for real kernels
(proj/include/tierplan/profiles.hpp:66-69): one CSV per device with header
`device,stage,seq_len,batch_size,latency_us`, one transformer layer per row, stages
nonattention (F1+F3 at the Tier-1 batch), attention (F2 at the shard batch and context) and
classifier.  ``measure_stage_profile`` times the B200 stages with CUDA events."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import _lib as L

STAGES = {"nonattention": L.STAGE_NONATTENTION, "attention": L.STAGE_ATTENTION,
          "classifier": L.STAGE_CLASSIFIER}


def write_profile(path, device: str, rows, mode: str = "w") -> None:
    """rows: iterable of (stage, seq_len, batch_size, latency_us); written through the C ABI."""
    lib = L.lib()
    first = True
    rows = list(rows)
    if not rows:
        raise L.ValidationError(L.GH_EINVAL, "no rows")
    for stage, seq, batch, lat in rows:
        b = (C.c_uint64 * 1)(batch)
        v = (C.c_double * 1)(lat)
        m = mode if first else "a"
        L.check(lib.gh_profile_write_csv(str(path).encode(), m.encode(), device.encode(), STAGES[stage], seq, b,
                                         v, 1))
        first = False


def measure_stage_profile(spec, batches, seq_len: int, reps: int = 10, device: int = 0):
    """Per-layer latency (us) of nonattention (pre+post) and attention at each batch size on the
    GPU; KV pre-filled to seq_len-1 positions.  Returns a list of CSV rows."""
    import torch

    from .stages import Tier1, Tier2, message_buffers
    one = spec.with_(n_layers=1, max_seq_len=max(spec.max_seq_len, seq_len))
    maxb = max(batches)
    t1 = Tier1(one, device=device, max_batch=maxb)
    t2 = Tier2(one, n_slots=maxb, device=device)
    t2.fill_synthetic(99, maxb, seq_len - 1)
    rows = []
    st = torch.cuda.Stream()
    for B in batches:
        x, fwd, bwd = message_buffers(one, B, device)
        x.normal_()
        pos = torch.full((B,), seq_len - 1, dtype=torch.int32, device="cuda")
        slot = torch.arange(B, dtype=torch.int32, device="cuda")
        nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
        res = {}
        for stage in ("nonattention", "attention", "classifier"):
            def run():
                if stage == "nonattention":
                    t1.pre(0, x, pos, fwd, stream=st)
                    t1.post(0, bwd, x, stream=st)
                elif stage == "attention":
                    t2.attend(0, slot, pos, fwd, bwd, stream=st)
                else:
                    t1.classify(x, nxt, stream=st)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                run()
            e1.record(st)
            st.synchronize()
            res[stage] = e0.elapsed_time(e1) * 1e3 / reps
        rows += [("nonattention", seq_len, B, res["nonattention"]), ("attention", seq_len, B, res["attention"]),
                 ("classifier", seq_len, B, res["classifier"])]
    t1.close()
    t2.close()
    return rows
