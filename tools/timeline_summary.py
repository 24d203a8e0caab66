"""Summarise GEMM timelines (GH_PROFILE_GEMMS=2: bench.py / tools/engine_step.py print one `tl ...`
line per GEMM launch) per weight shape: mean start->exit duration, mean time from the launch's
first CTA start to its median griddepcontrol.wait return, and the mean critical-path time (this
launch's last CTA exit minus the previous launch's).

  python tools/timeline_summary.py LOG [LOG ...]     (diagnostics)
"""
import collections
import re
import sys

NAMES = {(12288, 4096): "qkv", (4096, 4096): "o", (22016, 4096): "w13", (4096, 11008): "w2", (32000, 4096): "lm"}
PAT = re.compile(r"tl (\d+) N=(\d+) K=(\d+) B=(\d+) (\w+) ctas=(\d+) start=([\d.]+) wait=([\d.]+) exit=([\d.]+)")


def launches(path, rank="0"):
    txt = open(path).read()
    i = txt.find(f"rank {rank} GEMM profile")  # bench.py (one block per rank); engine_step.py has none
    if i >= 0:
        txt = txt[i:].split("\nrank ")[0]
    return [(int(m[2]), int(m[3]), int(m[4]), m[5], float(m[7]), float(m[8]), float(m[9])) for m in PAT.finditer(txt)]


for path in sys.argv[1:]:
    L = launches(path)
    if not L:
        continue
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    prev = None
    for N, K, B, kind, s, w, e in L:
        r = agg[(NAMES.get((N, K), f"{N}x{K}"), B, kind)]
        r[0] += 1
        r[1] += e - s
        r[2] += w - s
        r[3] += e - prev if prev is not None else e - s
        prev = e
    print(f"{path}: {len(L)} launches over {L[-1][6] - L[0][4]:.0f} us")
    for (n, B, kind), r in agg.items():
        print(f"  {n:5s} B={B:4d} {kind:6s} n={r[0]:3d}  duration {r[1] / r[0]:6.1f} us  start->wait {r[2] / r[0]:5.1f} us"
              f"  critical path {r[3] / r[0]:6.1f} us")
