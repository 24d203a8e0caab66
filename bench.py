#!/usr/bin/env python
"""Decode-throughput benchmark of the B200 two-tier decode path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C3]

N = 1: config C2 (Llama-2-7B shape, batch 64, context 512, both tiers colocated on one B200).
N > 1 (torchrun, one process per GPU): tier split of the same prompt shape — rank 0 = Tier-1
(weights), ranks 1..N-1 = Tier-2 (KV shards by prompt), NCCL send/recv of the PayloadModel
messages every layer, IF = 2 in-flight batches of 64 prompts per Tier-2 GPU each (weak scaling:
fixed work per Tier-2 GPU).  --config C3: context 2048 at the capacity-admitted batch
(two_tier_context_slots at 179 GiB per GPU; the requested 1024 does not fit).

A step = one decode token for every prompt of every in-flight batch, all layers + classifier +
greedy argmax, at a fixed context (each step appends at position ctx-1 and attends over ctx
positions; KV pre-filled with synthetic values).  Inputs (13.5 GB weights + KV) are far larger
than the 126 MB L2, so no L2 flush is needed between steps.

--impl reference times the reference-side CPU implementation of the path (the oracle port,
oracle/oracle.c, all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GiB = 1 << 30


def peaks():
    """(HBM GB/s, bf16 TFLOP/s sustained, kind) -- the driver-measured copy bandwidth and the
    sustained (back-to-back, under the power cap) dense bf16 rate: the Tier-1 GEMMs run inside a
    long step, so the sustained figure is their ceiling."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    """nvidia-smi clocks / throttle-reason sampler (every 20 ms) around a timed region.  The
    sampler is started and its first line awaited BEFORE the region, so that even a region of a
    few hundred milliseconds gets samples; only samples taken inside the region are kept."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.samples = []  # (time, line)
        self.t0 = self.t1 = None

    def _reader(self):
        for ln in self.proc.stdout:
            self.samples.append((time.perf_counter(), ln))

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("GH_CLOCKS_MS", "20")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._reader, daemon=True)
            self.thread.start()
            deadline = time.perf_counter() + 10
            while not self.samples and time.perf_counter() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *a):
        self.t1 = time.perf_counter()
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)
        inside = [ln for t, ln in self.samples if self.t0 <= t <= self.t1 + 0.03 and ln.strip()]
        # a region shorter than the sampling interval still reports the sample closest to it
        self.lines = inside or [ln for t, ln in self.samples[-2:] if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU baseline (oracle)
def _mem_available() -> int:
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_batch(spec, B, ctx):
    """Largest batch <= B whose oracle state (weights in the storage dtype + the KV of B prompts at
    max_seq_len) fits in 70 % of the host's available memory."""
    import paper_2501_11779_b200 as gh
    w = gh.weights_bytes(spec)
    kv = gh.kv_bytes_per_prompt(spec, spec.max_seq_len)
    avail = _mem_available()
    if not avail:
        return B
    return max(1, min(B, int((0.7 * avail - w) // kv)))


def cpu_steps(spec, B, ctx, warmup, steps, threads=0):
    """The CPU reference run of the workload: the oracle (oracle.c, fp32 compute, bf16 storage,
    OpenMP over all host threads) decodes FULL steps -- embedding, all n_layers layers (F1, F2 over
    the ctx-position context, F3) and the classifier + greedy argmax -- for B prompts at a fixed
    context (every step appends at position ctx-1, the GPU bench's steady state), with each step's
    next tokens fed back.  `warmup` untimed steps, then `steps` timed ones (>= 4
    steady-state steps; des.hpp:20-21 discards warm-up passes).  Returns (tokens/s, sample text,
    cores, per-step seconds)."""
    from oracle import Oracle, olib
    t0 = time.perf_counter()
    ora = Oracle(spec, n_slots=B, threads=threads)
    ora.fill_synthetic(99, B, ctx - 1)
    setup_s = time.perf_counter() - t0
    rng = np.random.default_rng(5678)
    tok = rng.integers(0, spec.vocab_size, size=B).astype(np.int32)
    pos = np.full(B, ctx - 1, np.int32)
    slot = np.arange(B, dtype=np.uint32)
    for _ in range(warmup):
        tok, _ = ora.step(tok, pos, slot, want_logits=False)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        tok, _ = ora.step(tok, pos, slot, want_logits=False)
        times.append(time.perf_counter() - t0)
    ora.close()
    cores = olib().or_max_threads()
    t_step = statistics.mean(times)
    sample = (f"oracle.c fp32 compute / bf16 storage on {cores} threads: {steps} timed full decode steps "
              f"(after {warmup} untimed) of batch {B}, context {ctx}: embed + {spec.n_layers} layers + "
              f"classifier/argmax, {t_step:.2f} s/step (min {min(times):.2f}, max {max(times):.2f}); "
              f"weights + KV pre-fill {setup_s:.1f} s untimed")
    return B / t_step, sample, cores, times


def cpu_stage_profiles(spec, ctx, batches, threads, out_dir, name):
    """SURVEY §8(d) CPU baseline for configurations whose KV does not fit host RAM whole (C3-C5):
    per-layer nonattention (F1+F3), attention (F2 at context ctx) and classifier latencies of
    the oracle on the host cores at each batch, written as reference-format profile CSVs
    (cpu_tier1_<name>.csv, cpu_tier2_<name>.csv, device "cpu-tier1" / "cpu-tier2").  Returns the
    rows."""
    from oracle import Oracle
    from paper_2501_11779_b200.profiles import write_profile
    one = spec.with_(n_layers=1, max_seq_len=max(spec.max_seq_len, ctx))
    maxb = max(batches)
    ora = Oracle(one, n_slots=maxb, threads=threads)
    ora.fill_synthetic(99, maxb, ctx - 1)
    rng = np.random.default_rng(5678)
    rows = []

    def best(fn, reps=2):
        t = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        return min(t) * 1e6

    for B in batches:
        x, fwd, bwd = ora.buffers(B)
        x[...] = rng.standard_normal(x.shape).astype(x.dtype)
        x2 = np.zeros_like(x)
        pos = np.full(B, ctx - 1, np.int32)
        slot = np.arange(B, dtype=np.uint32)
        ora.pre(0, x, pos, fwd)
        ora.attend(0, slot, pos, fwd, bwd)
        non = best(lambda: (ora.pre(0, x, pos, fwd), ora.post(0, bwd, x2)))
        att = best(lambda: ora.attend(0, slot, pos, fwd, bwd))
        cls = best(lambda: ora.classify(x, want_logits=False))
        rows += [("nonattention", ctx, B, non), ("attention", ctx, B, att), ("classifier", ctx, B, cls)]
        print(f"cpu B={B}: nonattention {non / 1e3:.1f} ms, attention {att / 1e3:.1f} ms, classifier "
              f"{cls / 1e3:.1f} ms per layer", file=sys.stderr, flush=True)
    ora.close()
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    write_profile(out / f"cpu_tier1_{name}.csv", "cpu-tier1", [r for r in rows if r[0] != "attention"])
    write_profile(out / f"cpu_tier2_{name}.csv", "cpu-tier2", [r for r in rows if r[0] == "attention"])
    return rows


# ------------------------------------------------------------------ configs
def _profile_latency(path: Path, stage: str, batch: int) -> float:
    """Per-layer latency (us) at `batch` from a reference-format profile CSV: linear interpolation
    between grid points, clamped below and extrapolated from the top two points above (the
    reference's KernelProfile::latency, profiles.cpp:93-129)."""
    pts = []
    for ln in path.read_text().splitlines()[1:]:
        f = ln.split(",")
        if len(f) == 5 and f[1] == stage:
            pts.append((int(f[3]), float(f[4])))
    pts.sort()
    if batch <= pts[0][0]:
        return pts[0][1]
    for (b0, l0), (b1, l1) in zip(pts, pts[1:]):
        if batch <= b1:
            return l0 + (l1 - l0) * (batch - b0) / (b1 - b0)
    (b0, l0), (b1, l1) = pts[-2], pts[-1]
    return l1 + (l1 - l0) * (batch - b1) / (b1 - b0)


def if_gh_from_profiles(spec, t1_batch: int, shard: int, ctx: int) -> int:
    """In-flight batches that keep Tier-1 busy while a batch is at Tier-2: the reference's
    if_gh = 1 + ceil((t_att + t_roundtrip) / t_noatt) (analytic.cpp:31-39), with t_noatt and
    t_att from this repo's measured B200 stage profiles (profiles/b200_tier{1,2}_C2.csv) and the
    round trip of the PayloadModel messages of one shard (netmodel.cpp:18-24) over NVLink at a
    conservative 400 GB/s plus 2 x 10 us of copy / flag latency.  At least 2."""
    import math
    root = Path(__file__).resolve().parent / "profiles"
    try:
        t_noatt = _profile_latency(root / "b200_tier1_C2.csv", "nonattention", t1_batch)
        t_att = _profile_latency(root / "b200_tier2_C2.csv", "attention", shard)
    except (OSError, IndexError, ValueError):
        return 2
    db = spec.dtype_bytes
    msg = shard * db * ((2 * spec.d_model + 2 * spec.d_kv) + 2 * spec.d_model)
    t_rt = 20.0 + msg / 400e9 * 1e6
    return max(2, 1 + math.ceil((t_att + t_rt) / t_noatt))


def auto_tier1(args, world: int) -> int:
    """Tier-1 pipeline spans of the default C2 split: one Tier-1 GPU up to 4 GPUs; from 8 GPUs on,
    two layer spans, each with (N - 2) / 2 Tier-2 GPUs (the reference's config-5 topology, P:455,
    optimizer.cpp:116-123).  One Tier-1 GPU for 7 Tier-2 GPUs would stream the weights for a batch
    of 448 prompts, where the GEMMs run at 233 us per layer (profiles/r02_gemm_timelines.txt); two
    spans at 192 prompts each share the layers (measured at 4 GPUs, r02_bench_n4_spans.json)."""
    if (args.config or "C2") != "C2" or args.tier1_tp > 1 or world < 8 or (world - 2) % 2:
        return 1
    return 2


def workload(args, world):
    import paper_2501_11779_b200 as gh
    cfg = args.config or "C2"
    c = gh.CONFIGS[cfg]
    spec, ctx = c["spec"], c["ctx"]
    if getattr(args, "cpu_profiles", ""):  # CPU stage profiles: the shape and context only
        return dict(name=cfg, spec=spec, ctx=ctx, batch=c["batch"], requested=c["batch"], inflight=1,
                    shard=c["batch"], kp=0)
    if args.paged and (world == 1 or cfg == "C2"):
        raise SystemExit("--paged is a tier-split option of C3 / C4 / C5 (tools/paged_bench.py covers one GPU)")
    if world == 1:
        if cfg in ("C4", "C5"):
            raise SystemExit(f"--config {cfg} is a tier-split configuration (run it with N >= 2 GPUs)")
        return dict(name=cfg, spec=spec, ctx=ctx, batch=c["batch"], requested=c["batch"], inflight=1,
                    shard=c["batch"], kp=0)
    n1 = max(1, args.tier1)
    tp = max(1, args.tier1_tp)
    if tp > 1:  # Tier-1 tensor parallelism: ranks 0..tp-1 share every layer, the rest are Tier-2
        if n1 > 1:
            raise SystemExit("--tier1-tp and --tier1 (pipeline spans) are exclusive")
        if world <= tp:
            raise SystemExit(f"--tier1-tp {tp}: world size {world} must be > {tp}")
        kp = world - tp
    else:
        if (world - n1) % n1 or world <= n1:
            raise SystemExit(f"--tier1 {n1}: world size {world} must be tier1 * (1 + K')")
        kp = (world - n1) // n1  # Tier-2 GPUs per Tier-1 span
    if cfg == "C2":  # weak scaling of the N=1 workload: 64 prompts per Tier-2 GPU per in-flight batch
        shard = args.shard or c["batch"]
        IF = args.inflight or if_gh_from_profiles(spec, shard * kp, shard, ctx)
        if n1 > 1 and not args.inflight:  # one group of batches per span in flight (split_step_peer)
            IF = n1 * max(3, IF)
        return dict(name="C2-split", spec=spec, ctx=ctx, batch=shard * kp, requested=shard * kp * IF,
                    inflight=IF, shard=shard, kp=kp,
                    admitted_slots=gh.two_tier_context_slots(spec, 1, kp, 179 * GiB, ctx))
    mem = 179 * GiB
    slots = gh.two_tier_context_slots(spec, n1, kp, mem, ctx)  # optimizer.cpp:175-192
    inflight = args.inflight or 2
    per_gpu = slots // kp
    shard = min(per_gpu // inflight, c["batch"] // (kp * inflight) or 1)
    if args.shard:  # e.g. the reference optimizer's choice (oracle.Ref.optimize)
        shard = args.shard
        if shard * inflight > per_gpu:
            raise SystemExit(f"--shard {shard} x IF {inflight} exceeds the {per_gpu} admitted slots per Tier-2 GPU")
    if args.paged:
        return paged_workload(cfg, spec, ctx, c["batch"], kp, inflight, per_gpu, n1)
    return dict(name=cfg, spec=spec, ctx=ctx, batch=shard * kp, requested=c["batch"], inflight=inflight,
                shard=shard, kp=kp, admitted_slots=slots)


PAGE = 64  # GH_KV_PAGE_POSITIONS


def paged_workload(cfg, spec, ctx, requested, kp, inflight, per_gpu, n1):
    """Tier split on a paged KV arena: each Tier-2 GPU gets the pages of its
    per_gpu full-context slots; every prompt has its own context drawn uniformly from [1, ctx)
    (seed 4321), and the shard is the largest that fits every Tier-2 GPU's pages (up to the
    requested batch).  Prompt g = ib * batch + j * shard + r lives on Tier-2 rank j, local slot
    ib * shard + r."""
    if n1 != 1:
        raise SystemExit("--paged: one Tier-1 rank")
    pages = per_gpu * (ctx // PAGE)
    cap = max(1, requested // (kp * inflight))
    rng = np.random.default_rng(4321)
    ctxs_all = rng.integers(1, ctx, size=cap * kp * inflight).astype(np.int32)

    def fits(shard):
        batch = shard * kp
        for j in range(kp):
            used = 0
            for ib in range(inflight):
                c = ctxs_all[:batch * inflight].reshape(inflight, batch)[ib, j * shard:(j + 1) * shard]
                used += int(np.sum((c + 1 + PAGE - 1) // PAGE))
            if used > pages:
                return False
        return True

    shard = 1
    while shard < cap and fits(shard + 1):
        shard += 1
    batch = shard * kp
    ctxs = ctxs_all[:batch * inflight].reshape(inflight, batch)
    return dict(name=cfg + "-paged", spec=spec, ctx=ctx, batch=batch, requested=requested, inflight=inflight,
                shard=shard, kp=kp, admitted_slots=per_gpu * kp, kv_pages=pages, ctxs=ctxs)


def ncu_tensor_pipe(kernel_prefix):
    """Time-weighted sm__pipe_tensor_cycles_active (% of peak) of a kernel family from the committed
    ncu --set full capture (profiles/*_ncu_full_metrics.csv, newest round first), or None."""
    import csv
    for p in sorted((ROOT / "profiles").glob("r*_ncu_full_metrics.csv"), reverse=True):
        num = den = 0.0
        with open(p) as f:
            for row in csv.DictReader(f):
                if kernel_prefix not in row.get("Kernel Name", ""):
                    continue
                t = next((v for k, v in row.items() if k.startswith("gpu__time_duration.sum")), None)
                pct = next((v for k, v in row.items() if k.startswith("sm__pipe_tensor_cycles_active")), None)
                try:
                    num += float(t) * float(pct)
                    den += float(t)
                except (TypeError, ValueError):
                    continue
        if den > 0:
            return num / den
    return None


def ncu_traffic(kernel_prefix):
    """DRAM bytes per launch (read + write) of a kernel from the committed ncu --set full capture
    (profiles/*_ncu_full_metrics.csv, newest round first), or None."""
    import csv
    for p in sorted((ROOT / "profiles").glob("r*_ncu_full_metrics.csv"), reverse=True):
        with open(p) as f:
            for row in csv.DictReader(f):
                if kernel_prefix in row.get("Kernel Name", ""):
                    rd = next((v for k, v in row.items() if k.startswith("dram__bytes_read.sum")), None)
                    wr = next((v for k, v in row.items() if k.startswith("dram__bytes_write.sum")), None)
                    try:
                        return (float(rd) + float(wr)) * 1e6  # Mbyte
                    except (TypeError, ValueError):
                        return None
    return None


def attention_bytes(spec, B, ctx):
    """SURVEY.md §8d algorithmic bytes of one attention launch (one layer):
    dtype*(2*D_kv*sum_b S_b + 2*B*D_kv + 2*B*D), S_b = ctx (cached ctx-1 + the new token)."""
    db = spec.dtype_bytes
    return db * (2 * spec.d_kv * B * ctx + 2 * B * spec.d_kv + 2 * B * spec.d_model)


def gemm_layer_bytes(spec, B):
    """weights of one layer + activations in/out of the four GEMMs (model.cpp:53 weight term)"""
    D, Dkv, Dh, db = spec.d_model, spec.d_kv, spec.d_hidden, spec.dtype_bytes
    w = D * (2 * D + 3 * Dh + 2 * Dkv)
    act = B * (D + (D + 2 * Dkv)) + B * (D + D + D) + B * (D + Dh) + B * (Dh + D + D)
    return db * (w + act)


# ------------------------------------------------------------------ our arm, 1 GPU
def run_colocated(args, wl):
    import torch
    import paper_2501_11779_b200 as gh
    from paper_2501_11779_b200 import _lib as L
    from paper_2501_11779_b200.stages import Engine, Tier1, Tier2, message_buffers

    spec, B, ctx = wl["spec"], wl["batch"], wl["ctx"]
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    eng = Engine(spec, batch=B, use_graph=True)
    lib = gh.lib()
    L.check(lib.gh_tier2_fill_synthetic(eng.tier2, 99, B, ctx - 1, None))
    rng = np.random.default_rng(5678)
    tok = rng.integers(0, spec.vocab_size, size=B).astype(np.int32)
    pos = np.full(B, ctx - 1, np.int32)
    torch.cuda.synchronize()
    n0 = lib.gh_kernel_launches(0)
    eng.step_host(tok, pos)                       # sets device tok/pos; captures the CUDA graph
    per_step_launches = lib.gh_kernel_launches(0) - n0 + 1   # captured kernels + advance
    for _ in range(args.warmup):
        eng.step_device(stream=stream)
        eng.advance(pos_increment=0, stream=stream)
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            eng.step_device(stream=stream)
            eng.advance(pos_increment=0, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    value = B / (ms / 1e3)

    # e2e through the public API (gh_engine_step_host): every step copies the host tokens and
    # positions in, replays the step and copies the next tokens out, synchronously -- the same K
    # steps as the device-timed region, timed by the host clock around them
    nxt = tok
    stream.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        nxt, _ = eng.step_host(nxt, pos, stream=stream)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps

    if os.environ.get("GH_PROFILE_GEMMS"):  # diagnostics: per-GEMM times of one eager step (serialised)
        import ctypes
        lib.gh_debug_gemm_profile(1)
        eng.step_host(tok, pos, want_logits=True, stream=stream)
        lib.gh_debug_gemm_profile(0)
        buf = ctypes.create_string_buffer(1 << 16)
        lib.gh_debug_gemm_profile_dump(buf, 1 << 16)
        print(f"GEMM profile:\n{buf.value.decode()}", file=sys.stderr)
    # dominant kernel: attention of one layer, timed alone with CUDA events on its stream
    eng.close()
    del eng
    torch.cuda.empty_cache()
    t2 = Tier2(spec.with_(n_layers=1), n_slots=B)
    t2.fill_synthetic(99, B, ctx - 1)
    x, fwd, bwd = message_buffers(spec, B)
    fwd.normal_()
    pos_d = torch.full((B,), ctx - 1, dtype=torch.int32, device="cuda")
    slot_d = torch.arange(B, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(stream):
        for _ in range(3):
            t2.attend(0, slot_d, pos_d, fwd, bwd, stream=stream)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a0.record(stream)
        for _ in range(reps):
            t2.attend(0, slot_d, pos_d, fwd, bwd, stream=stream)
        a1.record(stream)
    stream.synchronize()
    attn_ms = a0.elapsed_time(a1) / reps
    t2.close()
    # Tier-1 nonattention of one layer (pre + post), for the GEMM roofline
    t1 = Tier1(spec.with_(n_layers=1), max_batch=B)
    with torch.cuda.stream(stream):
        for _ in range(3):
            t1.pre(0, x, pos_d, fwd, stream=stream)
            t1.post(0, bwd, x, stream=stream)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(reps):
            t1.pre(0, x, pos_d, fwd, stream=stream)
            t1.post(0, bwd, x, stream=stream)
        g1.record(stream)
    stream.synchronize()
    na_ms = g0.elapsed_time(g1) / reps
    t1.close()
    return dict(ms=ms, value=value, e2e_ms=e2e_ms, launches=per_step_launches * args.steps,
                attn_ms=attn_ms, na_ms=na_ms, clocks=clk.summary())


# ------------------------------------------------------------------ our arm, tier split
def run_split(args, wl, rank, world):
    import torch
    import torch.distributed as dist
    import paper_2501_11779_b200 as gh
    from paper_2501_11779_b200 import _lib as L
    from paper_2501_11779_b200.stages import Comm, Engine

    spec, ctx, IF = wl["spec"], wl["ctx"], wl["inflight"]
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    obj = [Comm.unique_ids(1) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank, dev)
    eng = Engine(spec, batch=wl["batch"], inflight=IF, device=dev, use_graph=False, comm=comm,
                 transport=args.transport, tier1_ranks=max(1, args.tier1), kv_pages=wl.get("kv_pages", 0),
                 tier1_tp=max(1, args.tier1_tp))
    transport = eng.transport
    lib = gh.lib()
    stream = torch.cuda.Stream()
    ctxs = wl.get("ctxs")  # paged: per-prompt contexts [IF, batch]
    if eng.role == "tier2":
        if ctxs is not None:  # back each local slot with the pages of its own context
            j, sh = rank - max(1, args.tier1_tp), wl["shard"]
            for ib in range(IF):
                for r in range(sh):
                    eng.kv_map(ib * sh + r, int(ctxs[ib, j * sh + r]) + 1)
        L.check(lib.gh_tier2_fill_synthetic(eng.tier2, 99, wl["shard"] * IF, ctx - 1, None))
    rng = np.random.default_rng(5678)
    tok = rng.integers(0, spec.vocab_size, size=wl["batch"]).astype(np.int32)
    pos = np.full(wl["batch"], ctx - 1, np.int32)
    torch.cuda.synchronize()
    t1 = eng.role == "tier1"
    pos_all = ctxs if ctxs is not None else np.tile(pos, (IF, 1))
    eng.step_all_host(np.tile(tok, (IF, 1)) if t1 else None, pos_all if t1 else None, stream=stream)
    dist.barrier()
    n0 = lib.gh_kernel_launches(0)
    for _ in range(args.warmup):
        eng.step_all(stream=stream)
        if eng.role == "tier1":
            for ib in range(IF):
                eng.advance(ib, 0, stream=stream)
    stream.synchronize()
    per_step = (lib.gh_kernel_launches(0) - n0) / max(args.warmup, 1)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            eng.step_all(stream=stream)
            if eng.role == "tier1" and not os.environ.get("GH_BENCH_NO_ADVANCE"):  # (diagnostics)
                for ib in range(IF):
                    eng.advance(ib, 0, stream=stream)
            if os.environ.get("GH_BENCH_STEP_SYNC"):  # diagnostics: drain the pipeline every step
                stream.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    if os.environ.get("GH_BENCH_HOST_TIMING"):  # diagnostics: host enqueue time of one step (GPU idle)
        h0 = time.perf_counter()
        eng.step_all(stream=stream)
        h1 = time.perf_counter()
        stream.synchronize()
        print(f"rank {rank}: host enqueue {1e3 * (h1 - h0):.3f} ms/step", file=sys.stderr)
        dist.barrier()
    t = torch.tensor([ms_local], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    launches = torch.tensor([per_step * args.steps], dtype=torch.float64)
    dist.all_reduce(launches, op=dist.ReduceOp.SUM)
    # e2e: the same pipelined step through the host API: tokens/positions of every in-flight
    # batch copied in, next tokens copied out, every step
    dist.barrier()
    t0 = time.perf_counter()
    nsteps = max(2, args.steps // 2)
    toks = np.tile(tok, (IF, 1))
    poss = pos_all
    n1 = max(1, args.tier1)
    for _ in range(nsteps):
        r = eng.step_all_host(toks if eng.role == "tier1" else None, poss if eng.role == "tier1" else None,
                              stream=stream)
        if n1 > 1:  # Tier-1 stages: the last stage's next tokens go back to the first stage's host
            if rank == n1 - 1:
                dist.send(torch.from_numpy(np.ascontiguousarray(r, dtype=np.int32)), dst=0)
            elif rank == 0:
                buf = torch.zeros((IF, wl["batch"]), dtype=torch.int32)
                dist.recv(buf, src=n1 - 1)
                toks = buf.numpy()
        elif r is not None:
            toks = r
    e2e_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / nsteps], dtype=torch.float64)
    if os.environ.get("GH_PROFILE_GEMMS"):  # diagnostics: per-GEMM times of one more step (serialised)
        import ctypes
        lib.gh_debug_gemm_profile(int(os.environ["GH_PROFILE_GEMMS"]))  # 2: per-launch timeline
        eng.step_all(stream=stream)
        stream.synchronize()
        lib.gh_debug_gemm_profile(0)
        buf = ctypes.create_string_buffer(1 << 20)
        lib.gh_debug_gemm_profile_dump(buf, 1 << 20)
        print(f"rank {rank} GEMM profile:\n{buf.value.decode()}", file=sys.stderr)
    print(f"rank {rank} ({eng.role}): device {ms_local:.3f} ms/step, e2e {float(e2e_ms.item()):.3f} ms/step",
          file=sys.stderr)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    eng.close()
    comm.close()
    total = wl["batch"] * IF
    return dict(ms=ms, value=total / (ms / 1e3), e2e_ms=float(e2e_ms.item()), launches=int(launches.item()),
                clocks=clk.summary(), total=total, transport=transport)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=[None, "C2", "C3", "C4", "C5"])
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tier1", type=int, default=0,
                    help="tier split: Tier-1 pipeline stages (layer spans, each with its own Tier-2 GPUs); "
                         "0 = auto (C2: 2 spans from 8 GPUs on, else 1)")
    ap.add_argument("--tier1-tp", type=int, default=1,
                    help="tier split: Tier-1 tensor parallelism over this many GPUs (SURVEY 8f-3); the rest are Tier-2")
    ap.add_argument("--shard", type=int, default=0,
                    help="C2 tier split: prompts per Tier-2 GPU per in-flight batch (default 64, the N=1 batch)")
    ap.add_argument("--inflight", type=int, default=0,
                    help="tier split: in-flight batches (0 = if_gh from the stage profiles)")
    ap.add_argument("--cpu-profiles", default="",
                    help="with --impl reference: write the oracle's per-layer CPU stage profiles (cpu_tier{1,2}_<config>.csv) here")
    ap.add_argument("--cpu-batches", default="1,8,32,64,128")
    ap.add_argument("--paged", action="store_true",
                    help="tier split (C3/C4/C5): paged KV arena, per-prompt contexts uniform in [1, ctx)")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "peer"],
                    help="tier-split message transport (peer: copy engines + IPC flags; nccl: send/recv)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    args.tier1 = args.tier1 or auto_tier1(args, max(world, args.gpus if world == 1 else world))
    rank = int(os.environ.get("RANK", "0"))
    wl = workload(args, max(world, args.gpus if world == 1 else world))
    spec = wl["spec"]
    hbm, tf, peak_kind = peaks()
    metric = "decode tokens/s (Llama-2-7B shape, 2-tier split)"
    cfg = {"workload": f"{wl['name']}: {spec.name} shape random-init, context {wl['ctx']}, "
                       + ("both tiers colocated on 1 GPU" if wl["kp"] == 0 else
                          (f"Tier-1 tensor-parallel over {args.tier1_tp} GPUs (W_o / W_2 all-reduced in the GEMM "
                           f"epilogue over NVLink) + Tier-2 KV sharded by prompt over {wl['kp']} GPUs, IF={wl['inflight']}"
                           if args.tier1_tp > 1 else
                           f"Tier-1 on 1 GPU + Tier-2 KV sharded by prompt over {wl['kp']} GPUs, IF={wl['inflight']}"
                           if args.tier1 <= 1 else
                           f"Tier-1 pipelined over {args.tier1} GPUs (layer spans), each span with "
                           f"{wl['kp']} Tier-2 GPUs holding its layers' KV, IF={wl['inflight']}")),
           "batch": wl["batch"] * wl["inflight"], "requested_batch": wl["requested"], "ctx": wl["ctx"],
           "inflight": wl["inflight"], "dtype_storage": "bf16", "l2": "inputs larger than L2 (no flush)"}
    if "admitted_slots" in wl:
        cfg["admitted_slots"] = wl["admitted_slots"]
    if "ctxs" in wl:
        cfg["contexts"] = (f"paged KV ({wl['kv_pages']} pages of {PAGE} positions per Tier-2 GPU = its "
                           f"{wl['admitted_slots'] // wl['kp']} full-context slots); per-prompt context uniform "
                           f"in [1, {wl['ctx']}), mean {float(np.mean(wl['ctxs'])):.0f}")

    if args.impl == "reference" and args.cpu_profiles:  # CPU stage profiles
        from oracle import olib
        name = args.config or "C2"
        batches = [int(b) for b in args.cpu_batches.split(",")]
        rows = cpu_stage_profiles(spec, wl["ctx"], batches, args.cpu_threads, args.cpu_profiles, name)
        print(json.dumps({"impl": "reference", "cpu_profiles": args.cpu_profiles, "config": name, "ctx": wl["ctx"],
                          "cores": olib().or_max_threads(), "rows": rows}))
        return
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        B = cpu_batch(spec, wl["batch"] if wl["kp"] == 0 else min(wl["batch"], 64), wl["ctx"])
        # exactly W untimed + K timed full decode steps of the workload (no extrapolation)
        v, sample, cores, times = cpu_steps(spec, B, wl["ctx"], args.warmup, max(1, args.steps), args.cpu_threads)
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": v, "unit": "tokens/s", "n_gpus": 0,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": B / v * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": sample, "batch": B},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference has no decode implementation (SURVEY.md §0.2); the CPU arm is the oracle port "
                    "of the paper's CPU Tier-2 path (P:514, OpenMP)"}))
        return

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        res = run_split(args, wl, rank, world)
        cfg["transport"] = res["transport"]
        if rank != 0:
            dist.destroy_process_group()
            return
    else:
        res = run_colocated(args, wl)

    out = {"metric": metric, "value": res["value"], "unit": "tokens/s", "n_gpus": max(world, 1),
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"], "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": cfg}
    B_step = wl["batch"] * wl["inflight"]
    out["e2e"] = {"value": B_step / (res["e2e_ms"] / 1e3), "unit": "tokens/s",
                  "h2d_bytes_per_step": B_step * 8, "d2h_bytes_per_step": B_step * 4}
    out["gpu_launches"] = int(res["launches"])
    out["clocks"] = res["clocks"]
    if world == 1:
        ab = attention_bytes(spec, wl["batch"], wl["ctx"])
        ach = ab / (res["attn_ms"] / 1e3) / 1e9
        out["roofline"] = {"bound": "hbm", "kernel": "attn_gqa_tc_kernel<1> (Tier-2 F2, one layer)",
                           "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                           "peak_kind": peak_kind, "traffic": ncu_traffic("attn_gqa_tc_kernel"),
                           "traffic_source": "profiles/*_ncu_full_metrics.csv (dram read+write per launch)",
                           "algorithmic_bytes": ab,
                           "duration_us": res["attn_ms"] * 1e3, "frac_of_8TBs": ach / 8000.0}
        gb = gemm_layer_bytes(spec, wl["batch"])
        gach = gb / (res["na_ms"] / 1e3) / 1e9
        out["roofline_nonattention"] = {"bound": "hbm", "kernels": "Tier-1 F1+F3 of one layer (rmsnorm x2 + 4 "
                                        "tcgen05 GEMMs)", "achieved": gach, "peak": hbm, "unit": "GB/s",
                                        "frac": gach / hbm, "duration_us": res["na_ms"] * 1e3,
                                        "algorithmic_bytes": gb}
        # tensor roofline of the same Tier-1 GEMMs: FLOPs 2*B*D*(2D + 3D_h + 2D_kv) (model.cpp:54, MACs x 2)
        fl = 2 * wl["batch"] * spec.d_model * (2 * spec.d_model + 3 * spec.d_hidden + 2 * spec.d_kv)
        tach = fl / (res["na_ms"] / 1e3) / 1e12
        out["roofline_tensor"] = {"bound": "tensor", "kernels": "Tier-1 F1+F3 GEMMs of one layer (tcgen05)",
                                  "achieved": tach, "peak": tf, "unit": "TFLOP/s", "frac": tach / tf,
                                  "peak_kind": "measured sustained", "flops": fl,
                                  "tensor_pipe_active_pct": ncu_tensor_pipe("gemm_tc_kernel"),
                                  "note": f"B = {wl['batch']}: {fl / gb:.0f} FLOP per weight byte, far below the "
                                          "~220 FLOP/B ridge, so the HBM roofline (roofline_nonattention) binds"}
        step_bytes = spec.n_layers * (ab + gb) + spec.dtype_bytes * 2 * spec.vocab_size * spec.d_model // 2
        out["step_roofline"] = {"bytes_per_step": step_bytes, "ideal_ms": step_bytes / (hbm * 1e9) * 1e3,
                                "frac": step_bytes / (hbm * 1e9) / (res["ms"] / 1e3)}
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N = 1 figure (rank 0 only)
        B = cpu_batch(spec, wl["batch"] if wl["kp"] == 0 else min(wl["batch"], 64), wl["ctx"])
        # bounded sample (~10-30 s of CPU work): 1 untimed + 4 timed full steps, the same procedure
        # as the reference arm
        v, sample, cores, _ = cpu_steps(spec, B, wl["ctx"], 1, 4, args.cpu_threads)
        out["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample,
                               "batch": B}
    print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
