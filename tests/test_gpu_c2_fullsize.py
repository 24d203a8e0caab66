"""Parity at the benchmarked configuration: BASELINE configs[1] (C2) — Llama-2-7B shape, all 32
layers, batch 64, context 512 — through the same engine path bench.py times (CUDA graph, fused
RMSNorm from the W2/O-epilogue sums of squares, 7B split-K plans, tensor-core attention), against
the CPU fp32 oracle (oracle/oracle.c) on identical synthetic weights and KV pre-fill.

Every row's context is pre-filled with the synthetic KV (positions 0..P0-1, the bench's pre-fill)
and T = 24 decode steps run at positions P0..P0+23 (ending at the last position, 511).

* Noise floor.  The same oracle is re-run teacher-forced with every fp32 reduction in the reverse
  order (oracle.set_sum_order(1)): an equally valid fp32-compute / bf16-storage implementation
   that differs from the oracle only in summation order, exactly the freedom the GPU uses
  (split-K partials, tensor-core accumulation).  Its distance to the oracle is the bf16-storage
  noise floor after 32 residual layers; the GPU is held to that floor.
* Teacher-forced (24 steps, eager stage loop with logits, the graph's kernels): both sides are fed
  the oracle's greedy tokens.  Per step the GPU logits must satisfy
      rel-RMS  = ||g - r||_2 / ||r||_2   <= FLOOR_FACTOR * (the floor's rel-RMS) and <= REL_RMS_TOL
      max-abs  = max|g - r| / rms(r)      <= MAX_ABS_TOL
  the GPU argmax must equal the oracle's in every (step, row) pair whose oracle top-1/top-2
  margin exceeds MARGIN_TOL * rms(r), and its overall agreement may trail the floor's by at most
  AGREE_SLACK (random-init logits over 32000 tokens are nearly flat, so near-ties are common).
* Free-running (24 steps, the CUDA graph + device-side token feedback, exactly the bench step
  with pos += 1): each row's token stream must equal the oracle's free-running greedy stream up
  to its first divergence, and a divergence is only accepted where the oracle's own margin is a
  near-tie (<= MARGIN_TOL * rms(r)).

Tolerances are stated here (north star: "logits within a stated fp32/bf16 tolerance", numerics rule
P:514 "Kernel computations run at FP32, while kernel results are stored in the model's native
data type").  Both sides round every stage output to bf16; the GPU sums in a different order (split-K
partials, tensor-core accumulation), so a stored value can sit one bf16 ulp (2^-8 relative) away,
and that difference propagates through 32 residual layers.  The observed statistics are printed
(pytest -s) and summarised in profiles/r02_parity_c2_fullsize.json.
"""
import json
import os
import time

import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from oracle import Oracle, set_sum_order

pytestmark = pytest.mark.gpu

REL_RMS_TOL = 3.5e-2    # per step, logits, relative RMS (absolute cap)
FLOOR_FACTOR = 1.5      # per step, GPU rel-RMS <= FLOOR_FACTOR x the summation-order noise floor
MAX_ABS_TOL = 0.25      # per step, max |dlogit| in units of rms(ref logits)
MARGIN_TOL = 0.1        # a top-1/top-2 oracle margin below this x rms(ref) counts as a near-tie
AGREE_SLACK = 0.03      # teacher-forced argmax agreement may trail the noise floor's by this much

B, T = 64, 24


@pytest.fixture(scope="module")
def c2_run(need_gpu):
    from paper_2501_11779_b200 import _lib as L
    from paper_2501_11779_b200.stages import Engine
    c = gh.CONFIGS["C2"]
    spec, ctx = c["spec"], c["ctx"]
    assert c["batch"] == B and spec.n_layers == 32 and spec.d_model == 4096
    P0 = ctx - T                       # 488: decode positions 488..511
    rng = np.random.default_rng(5678)
    tok0 = rng.integers(0, spec.vocab_size, size=B).astype(np.int32)
    slot = np.arange(B, dtype=np.uint32)

    t0 = time.time()
    ora = Oracle(spec, n_slots=B)
    ora.fill_synthetic(99, B, P0)
    t_setup = time.time() - t0
    r_tok, r_lg = [], []
    tok = tok0
    t0 = time.time()
    for t in range(T):
        nxt, lg = ora.step(tok, np.full(B, P0 + t, np.int32), slot)
        r_tok.append(nxt.copy())
        r_lg.append(lg)
        tok = nxt
    t_oracle = time.time() - t0
    # noise floor: the same oracle, every reduction reversed, teacher-forced on the oracle's tokens
    f_tok, f_lg = [], []
    tok = tok0
    set_sum_order(1)
    try:
        for t in range(T):
            nxt, lg = ora.step(tok, np.full(B, P0 + t, np.int32), slot)
            f_tok.append(nxt.copy())
            f_lg.append(lg)
            tok = r_tok[t]
    finally:
        set_sum_order(0)
    ora.close()

    eng = Engine(spec, batch=B, use_graph=True)
    L.check(gh.lib().gh_tier2_fill_synthetic(eng.tier2, 99, B, P0, None))
    # teacher-forced: the oracle's token stream in, logits out
    g_tf_tok, g_tf_lg = [], []
    tok = tok0
    for t in range(T):
        nxt, lg = eng.step_host(tok, np.full(B, P0 + t, np.int32), want_logits=True)
        g_tf_tok.append(nxt.copy())
        g_tf_lg.append(lg)
        tok = r_tok[t]
    # free-running through the CUDA graph (the bench step), token feedback on the device
    g_fr = []
    nxt, _ = eng.step_host(tok0, np.full(B, P0, np.int32))
    g_fr.append(nxt.copy())
    for t in range(1, T):
        eng.advance(pos_increment=1)
        eng.step_device()
        g_fr.append(eng.read_next())
    eng.close()
    return dict(spec=spec, P0=P0, r_tok=np.stack(r_tok), r_lg=np.stack(r_lg), g_tf_tok=np.stack(g_tf_tok),
                g_tf_lg=np.stack(g_tf_lg), g_fr=np.stack(g_fr), f_tok=np.stack(f_tok), f_lg=np.stack(f_lg),
                t_setup=t_setup, t_oracle=t_oracle)


def _stats(r, which="g_tf"):
    out = []
    for t in range(T):
        g, ref = r[which + "_lg"][t].astype(np.float64), r["r_lg"][t].astype(np.float64)
        rms = np.sqrt(np.mean(ref ** 2))
        top2 = np.sort(ref, axis=1)[:, -2:]
        out.append(dict(step=t, rel_rms=float(np.linalg.norm(g - ref) / np.linalg.norm(ref)),
                        max_abs_over_rms=float(np.abs(g - ref).max() / rms),
                        mean_bias_over_rms=float((g - ref).mean() / rms),
                        min_margin_over_rms=float((top2[:, 1] - top2[:, 0]).min() / rms),
                        argmax_agree=int((r[which + "_tok"][t] == r["r_tok"][t]).sum())))
    return out


def _free_running(r):
    """first divergence per row and the oracle margin there (in rms units)"""
    rows = []
    for b in range(B):
        d = np.nonzero(r["g_fr"][:, b] != r["r_tok"][:, b])[0]
        if d.size == 0:
            rows.append(None)
            continue
        t = int(d[0])
        ref = r["r_lg"][t]
        rms = float(np.sqrt(np.mean(ref.astype(np.float64) ** 2)))
        top2 = np.sort(ref[b])[-2:]
        rows.append(dict(row=b, step=t, margin_over_rms=float((top2[1] - top2[0]) / rms)))
    return rows


def test_c2_fullsize_report(c2_run):
    st, fr = _stats(c2_run), _free_running(c2_run)
    rep = dict(config="C2 7B 32 layers B=64, positions %d..%d" % (c2_run["P0"], c2_run["P0"] + T - 1),
               oracle_setup_s=c2_run["t_setup"], oracle_s_per_step=c2_run["t_oracle"] / T,
               teacher_forced=st, noise_floor=_stats(c2_run, "f"), free_running_divergences=[x for x in fr if x],
               free_running_tokens_equal=int((c2_run["g_fr"] == c2_run["r_tok"]).sum()), tokens_total=T * B,
               tolerances=dict(rel_rms=REL_RMS_TOL, max_abs_over_rms=MAX_ABS_TOL, margin_over_rms=MARGIN_TOL,
                               floor_factor=FLOOR_FACTOR, agree_slack=AGREE_SLACK))
    print(json.dumps(rep, indent=1))
    out = os.environ.get("GH_PARITY_REPORT")
    if out:
        with open(out, "w") as f:
            json.dump(rep, f, indent=1)


def test_c2_teacher_forced_logits(c2_run):
    floor = max(s["rel_rms"] for s in _stats(c2_run, "f"))
    for s in _stats(c2_run):
        assert s["rel_rms"] <= min(REL_RMS_TOL, FLOOR_FACTOR * floor), (s, floor)
        assert s["max_abs_over_rms"] <= MAX_ABS_TOL, s


def test_c2_teacher_forced_argmax(c2_run):
    r = c2_run
    agree = 0
    for t in range(T):
        ref = r["r_lg"][t]
        rms = np.sqrt(np.mean(ref.astype(np.float64) ** 2))
        top2 = np.sort(ref, axis=1)[:, -2:]
        clear = (top2[:, 1] - top2[:, 0]) > MARGIN_TOL * rms
        assert np.array_equal(r["g_tf_tok"][t][clear], r["r_tok"][t][clear]), f"step {t}"
        agree += int((r["g_tf_tok"][t] == r["r_tok"][t]).sum())
    floor = sum(s["argmax_agree"] for s in _stats(r, "f")) / (T * B)
    assert agree / (T * B) >= floor - AGREE_SLACK, (agree / (T * B), floor)


def test_c2_free_running_greedy(c2_run):
    """The bench step (CUDA graph) run free: token streams equal the oracle's greedy streams; a row
    may only diverge at an oracle near-tie."""
    fr = _free_running(c2_run)
    bad = [x for x in fr if x and x["margin_over_rms"] > MARGIN_TOL]
    assert not bad, bad
    # every step before a row's first divergence is token-identical (checked by construction of
    # _free_running); after it the two streams continue from different tokens and are not compared
    assert sum(1 for x in fr if x is None or x["step"] > 0) >= B // 2
