"""Temperature sampling in the classifier (batch-state temperature): per row,
T = 0 is greedy and T > 0 samples by the Gumbel-max rule with noise from (seed, position, token).
The device decision is checked bit for bit against the numpy restatement (oracle/sampling.py)
applied to the engine's own fp32 logits, on every classifier path: the fp32 SIMT path, the
split-K tcgen05 kernel (B <= 128) and the CTA-pair kernel (B > 128)."""
import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from oracle import sampling

pytestmark = pytest.mark.gpu

CASES = {
    "tiny-fp32-simt": (gh.TINY.with_(n_layers=2, max_seq_len=64), 8),
    "7b-2layer-b16": (gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=64), 16),
    "7b-2layer-b64": (gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=64), 64),
    "7b-2layer-b200-pair": (gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=64), 200),
}


@pytest.mark.parametrize("name", list(CASES))
def test_sampled_tokens_match_restatement(name, need_gpu):
    from paper_2501_11779_b200.stages import Engine
    spec, B = CASES[name]
    rng = np.random.default_rng(3)
    T = rng.choice([0.0, 0.3, 0.8, 1.0, 2.5], size=B).astype(np.float32)
    T[:2] = [0.0, 1.0]
    seed = rng.integers(0, 2**32 - 1, size=B, dtype=np.uint64).astype(np.uint32)
    eng = Engine(spec, batch=B, use_graph=True)
    greedy = Engine(spec, batch=B, use_graph=True)
    eng.set_sampling(T, seed)
    tok = rng.integers(0, spec.vocab_size, size=B).astype(np.int32)
    differs = 0
    for t in range(6):
        pos = np.full(B, t, np.int32)
        nxt, lg = eng.step_host(tok, pos, want_logits=True)
        want = sampling.sample(lg, T, seed, pos)
        assert np.array_equal(nxt, want), (t, np.nonzero(nxt != want))
        g, _ = greedy.step_host(tok, pos)
        assert np.array_equal(nxt[T == 0], g[T == 0])   # greedy rows unchanged
        differs += int(np.sum(nxt[T > 0] != g[T > 0]))
        eng.step_device()                                # the graph path samples the same way
        assert np.array_equal(eng.read_next(), want)
        tok = nxt
    assert differs > 0  # sampling actually changed some tokens
    # same seeds and positions: the same draws (reproducible)
    eng.set_sampling(T, seed)
    nxt2, _ = eng.step_host(tok, np.full(B, 6, np.int32))
    nxt3, _ = eng.step_host(tok, np.full(B, 6, np.int32))
    assert np.array_equal(nxt2, nxt3)
    eng.close()
    greedy.close()


def test_sampling_validation(need_gpu):
    from paper_2501_11779_b200 import _lib as L
    from paper_2501_11779_b200.stages import Engine
    eng = Engine(gh.TINY.with_(n_layers=1, max_seq_len=32), batch=2, use_graph=False)
    with pytest.raises(L.ValidationError):
        eng.set_sampling(np.array([1.0, -0.5], np.float32), np.zeros(2, np.uint32))
    eng.close()


def test_continuous_batching_with_sampling_matches_oracle(need_gpu):
    """Per-request temperature through the dispatcher: every request's tokens equal decoding it
    alone with the fp32 oracle's logits and the numpy sampler (same seed, same positions)."""
    from oracle import Oracle
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    spec = gh.TINY.with_(n_layers=2, max_seq_len=64)
    rng = np.random.default_rng(12)
    reqs = [rng.integers(0, spec.vocab_size, size=int(n), dtype=np.int32) for n in rng.integers(1, 6, size=7)]
    smp = [(float(t), int(sd)) for t, sd in zip([0.0, 0.7, 1.3, 0.0, 2.0, 0.4, 1.0], rng.integers(0, 2**31, 7))]
    max_new = 6
    eng = Engine(spec, batch=3, use_graph=False)
    got, _ = ContinuousDispatcher(eng).run(reqs, max_new, sampling=smp)
    eng.close()
    ora = Oracle(spec, n_slots=1)
    for r, (T, sd), g in zip(reqs, smp, got):
        tok = np.array([r[0]], np.int32)
        out = []
        for t in range(len(r) - 1 + max_new):
            _, lg = ora.step(tok, np.array([t], np.int32), np.zeros(1, np.uint32))
            nxt = sampling.sample(lg, [T], [sd], [t])
            if t + 1 < len(r):
                tok = np.array([r[t + 1]], np.int32)
            else:
                out.append(int(nxt[0]))
                tok = nxt.astype(np.int32)
        assert np.array_equal(g, np.array(out, np.int32)), (T, g, out)
    ora.close()
