"""Large-batch Tier-1 GEMMs: planner's choice vs forced split-K vs forced CTA-pair kernel.

  python tools/gemm_large.py [B ...]        (diagnostics; weights resident, 20 repetitions)
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200 import _lib as L  # noqa: E402

lib = gh.lib()


def bench(N, K, B, flags=0, cluster=0, reps=20):
    us = C.c_float()
    L.check(lib.gh_debug_gemm_bench(N, K, B, flags, 0, cluster, reps, C.byref(us)))
    return us.value


shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "w13": (22016, 4096), "w2": (4096, 11008), "lm": (32000, 4096)}
args = [a for a in sys.argv[1:] if a.isdigit()]
if "70b" in sys.argv:
    shapes = {"qkv": (10240, 8192), "o": (8192, 8192), "w13": (57344, 8192), "w2": (8192, 28672), "lm": (32000, 8192)}
elif "13b" in sys.argv:
    shapes = {"qkv": (15360, 5120), "o": (5120, 5120), "w13": (27648, 5120), "w2": (5120, 13824), "lm": (32000, 5120)}
for B in [int(a) for a in args] or [192, 448, 1024]:
    tot = {"prod": 0.0, "split": 0.0, "pair": 0.0, "wide192": 0.0, "split128": 0.0}
    for name, (N, K) in shapes.items():
        flops = 2.0 * N * K * B
        row = [f"B={B:5d} {name:4s}"]
        for label, cl in [("prod", 0), ("split", -1), ("pair", -2), ("wide192", -3), ("split128", -4)]:
            try:
                t = bench(N, K, B, cluster=cl)
                tot[label] += t if name != "lm" else 0.0
                row.append(f"{label} {t:7.1f}us {flops / t / 1e6:6.0f}TF/s")
            except gh.GhError as e:
                row.append(f"{label} n/a ({e})")
        try:
            row.append(f"pair-noMMA {bench(N, K, B, flags=1, cluster=-2):7.1f} pair-noEpi {bench(N, K, B, flags=8, cluster=-2):7.1f}")
        except gh.GhError:
            pass
        print(" | ".join(row), flush=True)
    print(f"B={B:5d} layer (qkv+o+w13+w2): " + "  ".join(f"{k} {v:7.1f}us" for k, v in tot.items()), flush=True)
