"""Per-CTA timeline of the tcgen05 GEMM with weights streamed from HBM (diagnostics)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

import os  # noqa: E402
sys.path.insert(0, os.environ.get("GH_PKG_ROOT") or str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402

lib = gh.lib()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "w13": (22016, 4096), "w2": (4096, 11008), "lm": (32000, 4096)}
flags = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 0
for name, (N, K) in shapes.items():
    copies = max(2, int(3 * 126e6 / (N * K * 2)) + 1)
    us = C.c_float()
    tr = (C.c_uint64 * (148 * 16))()
    L.check(lib.gh_debug_gemm_trace(N, K, B, copies, 12 + 1000 * flags, C.byref(us), tr, 148 * 16))
    t = np.array(tr, dtype=np.float64).reshape(148, 16)
    if B > 128:  # CTA-pair kernel (stream-K) timeline
        t = t[t[:, 10] > 0]
        t0 = t[:, 0].min()
        rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
        q = lambda c: f"{np.nanmin(rel[:, c]):6.1f}/{np.nanmedian(rel[:, c]):6.1f}/{np.nanmax(rel[:, c]):6.1f}"
        print(f"{name:4s} {us.value:6.1f}us {2*N*K*B/us.value/1e6:5.0f}TF/s ctas {len(t)} start {q(0)} wpre {q(1)} "
              f"wait {q(2)} loads_issued {q(3)} mma_end {q(4)} contrib_acc {q(8)} contrib_pub {q(9)} "
              f"owner_acc {q(5)} partials {q(6)} epi_end {q(7)} exit {q(10)}", flush=True)
        if "-v" in sys.argv:
            idx = np.argsort(-np.nan_to_num(rel[:, 7]))[:4]
            for i in idx:
                print("   slow cta", i, " ".join(f"{c}:{rel[i, c]:.1f}" for c in range(11)),
                      "epi ns: tmem/fix/stage/store", t[i, 11:15], flush=True)
        continue
    t = t[t[:, 6] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    q = lambda c: f"{np.min(rel[:, c]):6.1f}/{np.median(rel[:, c]):6.1f}/{np.max(rel[:, c]):6.1f}"
    print(f"{name:4s} ctas {len(t):3d} {us.value:6.1f}us  {N*K*2/us.value/1e3:5.0f}GB/s  (min/med/max us) start {q(0)} wprefetch {q(1)} "
          f"wait {q(2)} first {q(3)} mma_end {q(4)} epi_end {q(5)} exit {q(6)}", flush=True)
    print("      last tile: tfull %s drained %s consumed %s published %s ready %s loaded %s reduced %s signalled %s final %s" % (
        q(7), q(8), q(9), q(10), q(11), q(15), q(12), q(13), q(14)), flush=True)
