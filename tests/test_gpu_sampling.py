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
