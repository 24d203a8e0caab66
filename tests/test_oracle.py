"""The CPU oracle (test infrastructure) pinned against committed goldens and an independent
numpy restatement; the product's accounting against the reference library's recorded values."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from oracle import Oracle, randn, to_f32

GOLD = Path(__file__).resolve().parent / "golden"
SPEC_BY_NAME = {
    "tiny": gh.TINY, "llama2-7b": gh.LLAMA2_7B, "llama2-13b": gh.LLAMA2_13B, "llama2-70b": gh.LLAMA2_70B,
    "C2": gh.CONFIGS["C2"]["spec"], "C3": gh.CONFIGS["C3"]["spec"],
    "llama70b_like": gh.ModelSpec("llama2-70b-like", 80, 8192, 1024, 28672, 64, 8, 2048, 2, 32000),
    "tiny_spec": gh.ModelSpec("tiny", 1, 2, 2, 2, 1, 1, 16, 2, 0),
}


def test_rng_golden():
    for c in json.loads((GOLD / "rng.json").read_text()):
        v = randn(c["seed"], c["tid"], c["start"], 8, c["std"])
        assert [float(x).hex() for x in v] == c["f32_hex"]


def test_rng_moments():
    v = randn(1234, 99, 0, 200_000, 1.0)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1.0) < 0.01
    assert np.abs(v).max() <= 2 * np.sqrt(3) + 1e-6  # Irwin-Hall(4) support


def test_reference_accounting_golden():
    """Every recorded reference value (oracle/_ref run in the build container) equals the
    product's restatement, including the error code."""
    entries = json.loads((GOLD / "reference_accounting.json").read_text())
    fn = {
        "kv_bytes_per_prompt": lambda s, a: gh.kv_bytes_per_prompt(s, *a),
        "nonattention_footprint": lambda s, a: list(gh.nonattention_footprint(s, *a)),
        "attention_footprint": lambda s, a: list(gh.attention_footprint(s, *a)),
        "weights_bytes": lambda s, a: gh.weights_bytes(s),
        "payload": lambda s, a: list(gh.payload(s)),
        "node_weight_bytes": lambda s, a: gh.node_weight_bytes(s, *a),
        "two_tier_context_slots": lambda s, a: gh.two_tier_context_slots(s, *a),
        "layer_spans": lambda s, a: gh.layer_spans(*a),
        "batch_grid": lambda s, a: gh.batch_grid(*a),
    }
    for e in entries:
        spec = SPEC_BY_NAME.get(e["spec"])
        if e["rc"] == 0:
            assert fn[e["fn"]](spec, e["args"]) == e["value"], e
        else:
            with pytest.raises(gh.GhError) as ei:
                fn[e["fn"]](spec, e["args"])
            assert ei.value.status == e["rc"], e


def test_oracle_c1_golden():
    g = np.load(GOLD / "oracle_c1.npz")
    c = gh.CONFIGS["C1"]
    ora = Oracle(c["spec"], seed=1234, n_slots=c["batch"])
    gen, lg = ora.generate(g["prompts"], c["steps"])
    assert np.array_equal(gen, g["tokens"])
    np.testing.assert_allclose(lg.max(-1), g["logit_max"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(lg[0, 0], g["logits_p0_s0"], rtol=1e-5, atol=1e-5)


# ------------------------------------------------------------------ independent numpy restatement
def bf(x, db):
    if db == 4:
        return x.astype(np.float32)
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


def np_weight(spec, seed, tid, rows, cols, std):
    return bf(randn(seed, tid, 0, rows * cols, std).reshape(rows, cols), spec.dtype_bytes).astype(np.float64)


@pytest.mark.parametrize("spec", [
    gh.ModelSpec("np-mha", 1, 64, 64, 96, 2, 2, 32, 4, 50),
    gh.ModelSpec("np-gqa-bf16", 1, 128, 32, 64, 8, 2, 32, 2, 40),
])
def test_oracle_layer_vs_numpy(spec):
    """F1/F2/F3 + classifier of the C oracle vs a float64 numpy restatement of the same math."""
    D, Dkv, Dh, H, Hkv, db = spec.d_model, spec.d_kv, spec.d_hidden, spec.n_heads, spec.n_kv_heads, spec.dtype_bytes
    dh = D // H
    seed, B = 1234, 3
    ora = Oracle(spec, seed=seed, n_slots=B)
    ora.fill_synthetic(5, B, 7)
    tok = np.array([3, 7, 11], np.int32)
    pos = np.array([0, 4, 7], np.int32)
    slot = np.array([2, 0, 1], np.uint32)
    x, fwd, bwd = ora.buffers(B)
    ora.embed(tok, x)
    ora.pre(0, x, pos, fwd)
    ora.attend(0, slot, pos, fwd, bwd)
    xn_buf = np.zeros_like(x)
    ora.post(0, bwd, xn_buf)
    nxt, lg = ora.classify(xn_buf)

    s = 1.0 / np.sqrt(D)
    E = np_weight(spec, seed, 1, spec.vocab_size, D, 1.0)
    Wq = np_weight(spec, seed, 64 + 0, D, D, s)
    Wk = np_weight(spec, seed, 64 + 1, Dkv, D, s)
    Wv = np_weight(spec, seed, 64 + 2, Dkv, D, s)
    Wo = np_weight(spec, seed, 64 + 3, D, D, s)
    W1 = np_weight(spec, seed, 64 + 4, Dh, D, s)
    W3 = np_weight(spec, seed, 64 + 5, Dh, D, s)
    W2 = np_weight(spec, seed, 64 + 6, D, Dh, 1.0 / np.sqrt(Dh))
    Wc = np_weight(spec, seed, 2, spec.vocab_size, D, s)

    def rms(v):
        return bf(v / np.sqrt((v * v).mean(-1, keepdims=True) + spec.norm_eps), db).astype(np.float64)

    def rope(v, p):
        v = v.copy()
        i = (np.arange(v.shape[-1]) % dh) // 2
        ang = p * np.power(float(spec.rope_theta), -2.0 * i / dh)
        c, sn = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
        a, o = v[0::2].copy(), v[1::2].copy()
        v[0::2] = a * c[0::2] - o * sn[0::2]
        v[1::2] = a * sn[0::2] + o * c[0::2]
        return v

    tol = 1e-4 if db == 4 else 2e-2
    xr = E[tok]
    assert np.array_equal(to_f32(x), xr.astype(np.float32))
    for b in range(B):
        xn = rms(xr[b])
        q, k, v = rope(Wq @ xn, pos[b]), rope(Wk @ xn, pos[b]), Wv @ xn
        f = to_f32(fwd[b])
        np.testing.assert_allclose(f[D:2 * D], q, rtol=tol, atol=tol * np.abs(q).max())
        np.testing.assert_allclose(f[2 * D:2 * D + Dkv], k, rtol=tol, atol=tol * np.abs(k).max())
        # attention over the pre-filled KV + the new token, from the oracle's own arena
        qf, kf, vf = f[D:2 * D].astype(np.float64), f[2 * D:2 * D + Dkv], f[2 * D + Dkv:]
        att = np.zeros(D)
        for h in range(H):
            g = h // (H // Hkv)
            K = ora.read_kv(0, int(slot[b]), 0, g, int(pos[b]) + 1).astype(np.float64)
            V = ora.read_kv(0, int(slot[b]), 1, g, int(pos[b]) + 1).astype(np.float64)
            assert np.array_equal(K[-1], kf[g * dh:(g + 1) * dh]) and np.array_equal(V[-1], vf[g * dh:(g + 1) * dh])
            sc = K @ qf[h * dh:(h + 1) * dh] / np.sqrt(dh)
            p = np.exp(sc - sc.max())
            att[h * dh:(h + 1) * dh] = (p / p.sum()) @ V
        a = to_f32(bwd[b])[D:]
        np.testing.assert_allclose(a, att, rtol=tol, atol=tol * np.abs(att).max())
        # F3 from the oracle's attention output
        hh = bf(Wo @ a.astype(np.float64) + xr[b], db).astype(np.float64)
        hn = rms(hh)
        gg = bf((lambda z: z / (1 + np.exp(-z)))(W1 @ hn) * (W3 @ hn), db).astype(np.float64)
        x2 = W2 @ gg + hh
        np.testing.assert_allclose(to_f32(xn_buf[b]), x2, rtol=tol, atol=tol * np.abs(x2).max())
        logits = Wc @ rms(to_f32(xn_buf[b]).astype(np.float64))
        np.testing.assert_allclose(lg[b], logits, rtol=tol, atol=tol * np.abs(logits).max())
    ora.close()
