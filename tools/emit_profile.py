"""Measure B200 stage latencies and emit them in the reference planner's profile format
(proj/include/tierplan/profiles.hpp:66-69): one CSV per tier, one layer per row.

  python tools/emit_profile.py --config C2 --max-batch 256 --out profiles/

nonattention = F1 + F3 of one layer at the Tier-1 batch (written to <out>/b200_tier1_<cfg>.csv
together with the classifier rows); attention = F2 of one layer at the shard batch and context
(<out>/b200_tier2_<cfg>.csv).
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11779_b200 as gh  # noqa: E402
from paper_2501_11779_b200.profiles import measure_stage_profile, write_profile  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--max-batch", type=int, default=256)
ap.add_argument("--out", default="profiles")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
c = gh.CONFIGS[a.config]
spec, ctx = c["spec"], c["ctx"]
grid = gh.batch_grid(a.max_batch)
rows = measure_stage_profile(spec, grid, ctx, reps=a.reps)
out = Path(a.out)
out.mkdir(parents=True, exist_ok=True)
t1 = [r for r in rows if r[0] != "attention"]
t2 = [r for r in rows if r[0] == "attention"]
write_profile(out / f"b200_tier1_{a.config}.csv", "b200-tier1", t1)
write_profile(out / f"b200_tier2_{a.config}.csv", "b200-tier2", t2)
for r in rows:
    print(*r)
