"""The kernel-latency CSV emitted through the C ABI (gh_profile_write_csv) is consumed by the
reference's own parser (profiles.cpp:168-224) with no warnings, and latency queries through the
reference (profiles.cpp:93-129) return the emitted values."""
import ctypes as C
from pathlib import Path

import pytest

import paper_2501_11779_b200 as gh
from paper_2501_11779_b200 import _lib as L
from paper_2501_11779_b200.profiles import write_profile
from oracle import Ref, ref_available

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")


def synthetic_rows():
    grid = gh.batch_grid(1024)
    na = {b: 40.0 + 0.09 * b for b in grid}                 # monotone non-attention
    at = {b: 1.5 + 0.65 * b for b in grid}                  # linear attention
    return grid, na, at


def test_write_rejects_bad_rows(tmp_path):
    p = tmp_path / "x.csv"
    with pytest.raises(gh.ValidationError):
        write_profile(p, "b200", [("nonattention", 1, 4, 0.0)])
    with pytest.raises(gh.ValidationError):
        write_profile(p, "b,200", [("nonattention", 1, 4, 1.0)])
    with pytest.raises(gh.ValidationError):
        write_profile(p, "b200", [("nonattention", 1, 0, 1.0)])


def test_header_and_rows(tmp_path):
    p = tmp_path / "x.csv"
    write_profile(p, "b200", [("nonattention", 2048, 4, 12.5), ("attention", 2048, 4, 3.25)])
    lines = p.read_text().splitlines()
    assert lines[0] == "device,stage,seq_len,batch_size,latency_us"
    assert lines[1] == "b200,nonattention,2048,4,12.5000"


@needs_ref
def test_reference_parser_accepts_emitted_csv(tmp_path):
    grid, na, at = synthetic_rows()
    rows = [("nonattention", 2048, b, na[b]) for b in grid] + [("attention", 2048, b, at[b]) for b in grid]
    p = tmp_path / "b200.csv"
    write_profile(p, "b200-sxm", rows)
    rc, warnings = Ref.profile_check(p)
    assert rc == 0, Ref.err()
    assert warnings == 0
    for b in grid:
        rc, ns = Ref.profile_latency(p, 0, b)
        assert rc == 0 and ns == round(na[b] * 1000)
        rc, ns = Ref.profile_latency(p, 1, b, 2048)
        assert rc == 0 and ns == round(at[b] * 1000)
    # interpolation between emitted grid points (profiles.cpp:118-128)
    rc, ns = Ref.profile_latency(p, 1, 5)
    assert rc == 0 and abs(ns - round((at[4] + at[6]) / 2 * 1000)) <= 1


@needs_ref
def test_reference_parser_rejects_duplicates(tmp_path):
    p = tmp_path / "dup.csv"
    write_profile(p, "b200", [("attention", 512, 4, 1.0), ("attention", 512, 4, 2.0)])
    rc, _ = Ref.profile_check(p)
    assert rc == 2


@needs_ref
def test_reference_optimizer_on_b200_profiles(tmp_path):
    """the unmodified reference optimizer (optimizer.cpp:515-583) runs on the
    committed B200 stage profiles (the Tier-1 file also carries the attention rows, which the
    optimizer needs for single-tier candidates) and picks a two-tier configuration."""
    root = Path(__file__).resolve().parents[1]
    t1 = (root / "profiles/b200_tier1_C2.csv").read_text().splitlines()
    t2 = (root / "profiles/b200_tier2_C2.csv").read_text().splitlines()
    comb = tmp_path / "t1all.csv"
    comb.write_text("\n".join(t1 + [ln.replace("b200-tier2", "b200-tier1") for ln in t2[1:]]) + "\n")
    rc, rep = Ref.optimize(root / "configs/llama2-7b-ctx512.json", root / "configs/b200x8_cluster.json", comb,
                           root / "profiles/b200_tier2_C2.csv", 512, 4)
    assert rc == 0, rep
    assert "best config: K=1 K'=" in rep and "tok/s" in rep


@pytest.mark.skipif(not ref_available(), reason="reference library not built")
def test_reference_planner_on_cpu_profiles():
    """the host-CPU stage profiles of the C3 shape (bench.py --impl reference
    --cpu-profiles, measured on the B200 box's host) load in the unmodified planner. CPU-only
    two-tier, B200 Tier-1 + CPU Tier-2 (the paper's prototype split) and all-B200
    deployments come out in increasing order."""
    import re
    root = Path(__file__).resolve().parents[1]
    model = root / "configs/llama2-7b-ctx2048.json"
    tput = {}
    for name, cl, t1, t2 in [("cpu", "cpu_host_cluster.json", "cpu_tier1_C3.csv", "cpu_tier2_C3.csv"),
                             ("b200+cpu", "b200_cpu_cluster.json", "b200_tier1_C3.csv", "cpu_tier2_C3.csv"),
                             ("b200", "b200x8_cluster.json", "b200_tier1_C3.csv", "b200_tier2_C3.csv")]:
        rc, rep = Ref.simulate(model, root / "configs" / cl, root / "profiles" / t1, root / "profiles" / t2,
                               1, 3, 64, 2048, inflight=2)
        assert rc == 0, rep
        tput[name] = float(re.search(r"throughput: ([0-9.e+]+) tok/s", rep).group(1))
    assert 0 < tput["cpu"] < tput["b200+cpu"] < tput["b200"]


@pytest.mark.skipif(not ref_available(), reason="reference library not built")
@pytest.mark.parametrize("cfg,model,ctx,batch", [("C4", "llama2-13b-ctx4096.json", 4096, 16),
                                                 ("C5", "llama2-70b-ctx8192.json", 8192, 32)])
def test_reference_planner_on_cpu_profiles_c4_c5(cfg, model, ctx, batch):
    """The C4 / C5 host-CPU stage profiles load in the unmodified planner (CPU two-tier)."""
    import re
    root = Path(__file__).resolve().parents[1]
    rc, rep = Ref.simulate(root / "configs" / model, root / "configs/cpu_host_cluster.json",
                           root / f"profiles/cpu_tier1_{cfg}.csv", root / f"profiles/cpu_tier2_{cfg}.csv",
                           1, 3, batch, ctx, inflight=2)
    assert rc == 0, rep
    cpu = float(re.search(r"throughput: ([0-9.e+]+) tok/s", rep).group(1))
    # the B200 stage profiles of the same shape (tools/emit_profile.py) at the measured N = 4 split
    shard = {"C4": 27, "C5": 34}[cfg]
    rc, rep = Ref.simulate(root / "configs" / model, root / "configs/b200x8_cluster.json",
                           root / f"profiles/b200_tier1_{cfg}.csv", root / f"profiles/b200_tier2_{cfg}.csv",
                           1, 3, shard, ctx, inflight=2)
    assert rc == 0, rep
    b200 = float(re.search(r"throughput: ([0-9.e+]+) tok/s", rep).group(1))
    assert 0 < cpu < b200
