"""CPU checks of the sampling restatement (oracle/sampling.py): the Gumbel-max draws follow
softmax(logits / T), T = 0 is greedy, and the noise is a pure function of (seed, pos, token)."""
import numpy as np

from oracle import sampling


def test_gumbel_max_frequencies_follow_softmax():
    logits = np.array([[1.0, 0.2, -0.5, 2.0, 0.0]], np.float32)
    T = 0.7
    n = 20000
    counts = np.zeros(5)
    for s in range(n):
        counts[sampling.sample(logits, [T], [s], [17])[0]] += 1
    p = np.exp(logits[0] / T - (logits[0] / T).max())
    p /= p.sum()
    sd = np.sqrt(n * p * (1 - p))
    assert np.all(np.abs(counts - n * p) < 4.5 * sd + 1), (counts, n * p)


def test_greedy_and_determinism():
    rng = np.random.default_rng(0)
    lg = rng.standard_normal((6, 300)).astype(np.float32)
    T = np.array([0, 0, 0.8, 1.5, 0, 3.0], np.float32)
    seed = np.arange(6, dtype=np.uint32) * 77
    pos = np.array([0, 5, 9, 9, 1, 4096], np.int32)
    a = sampling.sample(lg, T, seed, pos)
    b = sampling.sample(lg, T, seed, pos)
    assert np.array_equal(a, b)
    for i in (0, 1, 4):
        assert a[i] == np.argmax(lg[i])
    # another position draws different noise
    assert not np.array_equal(sampling.gumbel_noise(sampling.sample_key(5, 9), 64),
                              sampling.gumbel_noise(sampling.sample_key(5, 10), 64))


def test_splitmix64_known_values():
    # splitmix64 of 0 and 1 (reference values of the published generator: state += golden,
    # then the two xor-shift-multiply rounds)
    assert int(sampling.splitmix64(0)) == 0xE220A8397B1DCDAF
    assert int(sampling.splitmix64(1)) == 0x910A2DEC89025CC1
