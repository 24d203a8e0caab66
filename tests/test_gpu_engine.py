"""End-to-end decode through the engine (C ABI gh_engine_*) against the CPU oracle.

C1 (BASELINE configs[0]): tiny 288x6 model, fp32, 4 prompts (length 8) x 128 greedy tokens,
both tiers on one device.  Acceptance: generated token ids identical to the oracle's (north
star: "token ids bit-exact under greedy decode"); logits within 1e-3 absolute of the oracle's
(fp32 compute, different summation order only).  The test also reports the smallest top-1/top-2
logit margin the oracle saw, so a near-tie can be told apart from a kernel bug.
"""
import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from oracle import Oracle

pytestmark = pytest.mark.gpu


def prompts_for(spec, B, plen, seed=5678):
    return np.random.default_rng(seed).integers(0, spec.vocab_size, size=(B, plen), dtype=np.int32)


@pytest.fixture(scope="module")
def c1_run(need_gpu):
    from paper_2501_11779_b200.stages import Dispatcher, Engine
    c = gh.CONFIGS["C1"]
    spec = c["spec"]
    prompts = prompts_for(spec, c["batch"], c["prompt_len"])
    eng = Engine(spec, batch=c["batch"], use_graph=False)
    gen, lg = Dispatcher(eng).generate(prompts, c["steps"], want_logits=True)
    eng.close()
    ora = Oracle(spec, n_slots=c["batch"])
    rgen, rlg = ora.generate(prompts, c["steps"])
    ora.close()
    return dict(spec=spec, prompts=prompts, gen=gen, lg=lg, rgen=rgen, rlg=rlg)


def test_c1_greedy_tokens_bit_exact(c1_run):
    r = c1_run
    top2 = np.sort(r["rlg"], axis=-1)[..., -2:]
    margin = float((top2[..., 1] - top2[..., 0]).min())
    mism = np.argwhere(r["gen"] != r["rgen"])
    assert mism.size == 0, f"first token mismatch at {mism[0]} (min oracle margin {margin:.2e})"
    assert r["gen"].shape == (4, 128)


def test_c1_tokens_equal_transformers_llama(c1_run):
    """The same 512 tokens from Hugging Face transformers' LlamaForCausalLM holding these weights
    (tests/golden/hf_llama_c1.npz, tests/test_oracle_hf.py): an implementation independent of
    the oracle."""
    from pathlib import Path
    hf = np.load(Path(__file__).resolve().parent / "golden" / "hf_llama_c1.npz")
    assert np.array_equal(hf["prompts"], c1_run["prompts"])
    assert np.array_equal(c1_run["gen"], hf["tokens"])


def test_c1_logits_within_tolerance(c1_run):
    r = c1_run
    err = np.abs(r["lg"] - r["rlg"]).max()
    assert err < 1e-3, f"max |logit diff| {err}"


def test_c1_graph_matches_eager(need_gpu):
    """The CUDA-graph step is the same computation as the eager one (bit-identical tokens)."""
    from paper_2501_11779_b200.stages import Dispatcher, Engine
    spec = gh.TINY.with_(n_layers=3, max_seq_len=64)
    prompts = prompts_for(spec, 4, 5, seed=11)
    outs = []
    for use_graph in (False, True):
        eng = Engine(spec, batch=4, use_graph=use_graph)
        gen, _ = Dispatcher(eng).generate(prompts, 12)
        outs.append(gen)
        eng.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("spec,B,steps", [
    (gh.ModelSpec("e2e-bf16", 3, 512, 512, 1024, 4, 4, 128, 2, 2000), 20, 10),
    (gh.ModelSpec("e2e-gqa", 2, 1024, 256, 1536, 16, 4, 128, 2, 1000), 9, 6),
    # B > 256: several 128-column batch tiles and the unfused-RMSNorm fallback of the Tier-1 path
    (gh.ModelSpec("e2e-wide", 2, 512, 512, 1024, 4, 4, 64, 2, 700), 300, 3),
    # 128 < B <= 256: two batch tiles with the fused RMSNorm
    (gh.ModelSpec("e2e-b192", 2, 512, 512, 1024, 4, 4, 64, 2, 700), 192, 3),
    # Tier-1 batch of the 8-GPU split (7 x 64): CTA-pair kernel, several batch tiles, stream-K
    (gh.ModelSpec("e2e-b448", 2, 1024, 1024, 2816, 8, 8, 64, 2, 1000), 448, 2),
    # SURVEY 8(a) config shapes at full width, 2 layers: C3/C4 13B-class MHA (D 5120, 40 heads)
    # and C5 70B GQA (D 8192, 64 query / 8 KV heads, FFN 28672)
    (gh.ModelSpec("c4-13b-shape", 2, 5120, 5120, 13824, 40, 40, 64, 2, 32000), 8, 2),
    (gh.ModelSpec("c5-70b-shape", 2, 8192, 1024, 28672, 64, 8, 64, 2, 32000), 8, 2),
])
def test_bf16_engine_teacher_forced(need_gpu, spec, B, steps):
    """bf16 storage: per step, the GPU's argmax equals the oracle's wherever the oracle's top-2
    margin exceeds the logit tolerance, with both fed the oracle's token stream (teacher
    forcing), and logits agree within 2e-2 * max|logit|."""
    from paper_2501_11779_b200.stages import Engine
    prompts = prompts_for(spec, B, 4, seed=3)
    eng = Engine(spec, batch=B, use_graph=True)
    ora = Oracle(spec, n_slots=B)
    slot = np.arange(B, dtype=np.uint32)
    tok = prompts[:, 0].copy()
    agree = total = 0
    for t in range(3 + steps):
        pos = np.full(B, t, np.int32)
        g_next, g_lg = eng.step_host(tok, pos, want_logits=True)
        r_next, r_lg = ora.step(tok, pos, slot)
        tol = 2e-2 * np.abs(r_lg).max()
        assert np.abs(g_lg - r_lg).max() <= tol
        top2 = np.sort(r_lg, axis=1)[:, -2:]
        clear = (top2[:, 1] - top2[:, 0]) > 2 * tol
        assert np.array_equal(g_next[clear], r_next[clear])
        agree += int((g_next == r_next).sum())
        total += B
        tok = prompts[:, t + 1] if t + 1 < prompts.shape[1] else r_next
    eng.close()
    ora.close()
    assert agree / total > 0.9


def test_ragged_positions_engine_vs_stages(need_gpu):
    """Prompts at different positions in one batch (ragged contexts) decode like the stage API."""
    from paper_2501_11779_b200.stages import Engine
    spec = gh.ModelSpec("ragged", 2, 512, 512, 1024, 4, 4, 128, 2, 500)
    B = 6
    eng = Engine(spec, batch=B, use_graph=False)
    ora = Oracle(spec, n_slots=B)
    rng = np.random.default_rng(1)
    slot = np.arange(B, dtype=np.uint32)
    # each prompt b starts b steps late (its first token at position 0 while others are further)
    toks = rng.integers(0, spec.vocab_size, size=(B, 20), dtype=np.int32)
    for t in range(12):
        pos = np.maximum(t - np.arange(B), 0).astype(np.int32)
        tok = toks[np.arange(B), pos]
        g_next, g_lg = eng.step_host(tok, pos, want_logits=True)
        r_next, r_lg = ora.step(tok, pos, slot)
        assert np.abs(g_lg - r_lg).max() <= 2e-2 * np.abs(r_lg).max()
    eng.close()
    ora.close()


def test_continuous_batching_slot_reuse(need_gpu):
    """Continuous batching: 10 requests of different prompt lengths through 3
    lanes; a finished request's lane and context slot are reused by the next one.  Every request's
    greedy tokens equal decoding it alone with the oracle (fp32: bit-exact)."""
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    spec = gh.TINY.with_(n_layers=3, max_seq_len=64)
    rng = np.random.default_rng(21)
    reqs = [rng.integers(0, spec.vocab_size, size=int(n), dtype=np.int32) for n in rng.integers(1, 7, size=10)]
    max_new = 6
    eng = Engine(spec, batch=3, use_graph=False)
    got, steps = ContinuousDispatcher(eng).run(reqs, max_new)
    eng.close()
    ora = Oracle(spec, n_slots=1)
    for r, g in zip(reqs, got):
        ref, _ = ora.generate(r[None, :], max_new)
        assert np.array_equal(g, ref[0]), (r, g, ref[0])
    ora.close()
    assert steps < sum(len(r) - 1 + max_new for r in reqs)  # lanes were shared
