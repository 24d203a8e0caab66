"""Sweep the tcgen05 GEMM mainloop (diagnostics): python tools/gemm_sweep.py"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402

lib = gh.lib()


def bench(N, K, B, flags=0, stages=0, cluster=0, reps=20):
    us = C.c_float()
    L.check(lib.gh_debug_gemm_bench(N, K, B, flags, stages, cluster, reps, C.byref(us)))
    return us.value


shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "w13": (22016, 4096), "w2": (4096, 11008), "lm": (32000, 4096)}
if "tp70b" in sys.argv:  # the 70B shapes of one of two tensor-parallel Tier-1 ranks
    shapes = {"qkv": (5120, 8192), "o": (8192, 4096), "w13": (28672, 8192), "w2": (8192, 14336)}
elif "70b" in sys.argv:
    shapes = {"qkv": (10240, 8192), "o": (8192, 8192), "w13": (57344, 8192), "w2": (8192, 28672)}
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for name, (N, K) in shapes.items():
    wb = N * K * 2
    base = bench(N, K, B)
    row = [f"{name:4s} N={N:6d} K={K:6d} prod {base:7.1f}us {wb / base / 1e3:6.0f}GB/s"]
    for label, kw in [("noMMA", dict(flags=1)), ("noX", dict(flags=2)), ("noHint", dict(flags=4)),
                      ("noEpi", dict(flags=8)), ("noMMA+noEpi", dict(flags=9)), ("st4", dict(stages=4)),
                      ("st6", dict(stages=6)), ("c1", dict(cluster=1)), ("c2", dict(cluster=2)),
                      ("c4", dict(cluster=4)), ("c8", dict(cluster=8))]:
        try:
            t = bench(N, K, B, **kw)
            row.append(f"{label} {t:6.1f}")
        except gh.GhError:
            row.append(f"{label}    n/a")
    print(" | ".join(row), flush=True)
