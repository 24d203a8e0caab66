"""Temperature sampling, restated in numpy (TEST INFRASTRUCTURE ONLY: the checker for the device
sampler in the classifier epilogue, paper_2501_11779_b200/csrc/common.cuh `sample_score`; never
imported by the product path).

The batch state of the paper's dispatcher carries a per-prompt temperature; the
reference holds no sampling code, so the rule is the standard Gumbel-max identity:
    token = argmax_r ( logit_r / T + g_r ),   g_r = -log(-log(u_r)),   u_r ~ U(0, 1)
which draws token r with probability softmax(logit / T)_r.  u_r is a counter-based uniform:
    key = splitmix64(seed << 32 | pos),  h = splitmix64(key + r),  u = ((h >> 11) + 0.5) / 2^53
T = 0 is greedy (lowest index on ties).  The score is fp32: (logit * fp32(1/T)) rounded, plus the
noise computed in float64 and rounded once, matching the device's __fmul_rn / __fadd_rn.
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + _GOLDEN
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def sample_key(seed, pos):
    seed = np.asarray(seed, dtype=np.uint64)
    pos = np.asarray(pos, dtype=np.int64).astype(np.uint32).astype(np.uint64)
    return splitmix64((seed << np.uint64(32)) | pos)


def gumbel_noise(key, V):
    """fp32 noise g[r] for r in [0, V) of one row."""
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(key) + np.arange(V, dtype=np.uint64))
    u = ((h >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53
    return (-np.log(-np.log(u))).astype(np.float32)


def sample(logits, temperature, seed, pos):
    """Tokens [B] for fp32 logits [B, V], temperature [B] (0 = greedy), seed [B], pos [B]."""
    logits = np.asarray(logits, np.float32)
    B, V = logits.shape
    out = np.empty(B, np.int32)
    for b in range(B):
        T = np.float32(temperature[b])
        if T > 0:
            inv = np.float32(1.0) / T
            sc = (logits[b] * inv).astype(np.float32) + gumbel_noise(sample_key(seed[b], pos[b]), V)
            out[b] = int(np.argmax(sc.astype(np.float32)))
        else:
            out[b] = int(np.argmax(logits[b]))
    return out
