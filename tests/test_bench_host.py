"""Host-side logic of bench.py (CPU): the reference-style profile interpolation and the if_gh
in-flight batch choice read from the committed B200 profiles."""
import importlib.util
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    argv = sys.argv
    sys.argv = ["bench.py"]
    try:
        spec.loader.exec_module(mod)
    finally:
        sys.argv = argv
    return mod


def test_profile_latency_interpolation(bench, tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("device,stage,seq_len,batch_size,latency_us\n"
                 "d,nonattention,512,2,10.0\nd,nonattention,512,4,20.0\nd,nonattention,512,8,30.0\n")
    f = bench._profile_latency
    assert f(p, "nonattention", 1) == 10.0          # clamp below (profiles.cpp:93-129)
    assert f(p, "nonattention", 3) == 15.0          # interior interpolation
    assert f(p, "nonattention", 12) == 40.0         # top-two extrapolation


def test_if_gh_from_profiles(bench):
    import paper_2501_11779_b200 as gh
    spec = gh.CONFIGS["C2"]["spec"]
    for kp in (1, 3, 7):
        IF = bench.if_gh_from_profiles(spec, 64 * kp, 64, 512)
        assert 2 <= IF <= 8
    # Tier-1 nonattention grows with the batch while Tier-2 attention per shard is fixed, so the
    # in-flight batches needed to cover a Tier-2 round trip never grow with K'
    assert bench.if_gh_from_profiles(spec, 64 * 7, 64, 512) <= bench.if_gh_from_profiles(spec, 64, 64, 512)


def test_paged_workload_fits_every_tier2_gpu():
    """bench.py --paged: the chosen shard's pages fit each Tier-2 GPU's budget, one more prompt
    per shard would not (or the requested batch is reached), and it admits more prompts than
    the contiguous slots."""
    import numpy as np
    import bench
    import paper_2501_11779_b200 as gh
    spec = gh.CONFIGS["C3"]["spec"]
    wl = bench.paged_workload("C3", spec, 2048, 1024, 3, 2, 170, 1)
    pages, sh, kp = wl["kv_pages"], wl["shard"], wl["kp"]
    assert pages == 170 * 32 and wl["ctxs"].shape == (2, sh * kp)
    for j in range(kp):
        used = sum(int(np.sum((wl["ctxs"][ib, j * sh:(j + 1) * sh] + 64) // 64)) for ib in range(2))
        assert used <= pages
    assert sh * kp * 2 > 510            # more than the 510 contiguous C3 slots at K' = 3
    assert sh * kp * 2 <= 1024


def test_cpu_steps_runs_exact_full_steps(bench):
    """The CPU reference arm times exactly K full decode steps (all layers + classifier) after W
    untimed ones: no per-layer extrapolation."""
    import paper_2501_11779_b200 as gh
    spec = gh.TINY.with_(n_layers=2, max_seq_len=32)
    v, sample, cores, times = bench.cpu_steps(spec, 4, 16, 1, 3, threads=2)
    assert len(times) == 3 and all(t > 0 for t in times)
    assert abs(v - 4 / (sum(times) / 3)) < 1e-9 * v
    assert "3 timed full decode steps" in sample and "2 layers" in sample


def test_cpu_batch_respects_host_memory(bench, monkeypatch):
    import paper_2501_11779_b200 as gh
    spec = gh.CONFIGS["C3"]["spec"]          # 1 GiB of KV per prompt at 2048 positions
    monkeypatch.setattr(bench, "_mem_available", lambda: 64 << 30)
    B = bench.cpu_batch(spec, 64, 2048)
    assert 1 <= B < 64
    assert gh.weights_bytes(spec) + B * gh.kv_bytes_per_prompt(spec, 2048) <= 0.7 * (64 << 30)


def test_auto_tier1_spans():
    """The default C2 split uses two Tier-1 layer spans from 8 GPUs on (config-5 topology), one
    Tier-1 GPU below that and for the other configs / tensor parallelism; the span count divides
    the GPUs, and with spans the in-flight batches form one group per span."""
    import argparse
    import bench
    def a(config=None, tp=1):
        return argparse.Namespace(config=config, paged=False, tier1=0, tier1_tp=tp, shard=0, inflight=0,
                                  cpu_profiles="")
    assert [bench.auto_tier1(a(), w) for w in (1, 2, 4, 8)] == [1, 1, 1, 2]
    assert bench.auto_tier1(a("C3"), 8) == 1 and bench.auto_tier1(a(tp=2), 8) == 1
    args = a()
    args.tier1 = bench.auto_tier1(args, 8)
    wl = bench.workload(args, 8)
    assert (wl["kp"], wl["batch"], wl["shard"]) == (3, 192, 64)
    assert wl["inflight"] % 2 == 0 and wl["inflight"] >= 6
