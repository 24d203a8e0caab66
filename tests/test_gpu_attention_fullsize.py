"""F2 (append + attention) at the BASELINE configs' full sizes, one layer: C3 (7B, context 2048),
C4 (13B, context 4096) and C5 (70B GQA 64/8 heads, context 8192), with ragged positions that
include the first (0) and the last (max_seq_len - 1) position, contiguous and paged arenas.

The oracle cannot hold these arenas, so a sample of (prompt, head) pairs is checked against a
plain fp32 restatement of softmax(q K^T / sqrt(d_h)) V over the kernel's own arena (read back
through gh_tier2_read_kv after the step), and size-independent properties cover every row:
x pass-through bit-exact, appended key / value bit-exact copies of the message, finite output.
Tolerance (bf16 storage, as tests/test_gpu_stages.py): |gpu - ref| <= 1.6e-2 * max|ref|."""
import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from oracle import to_f32
from paper_2501_11779_b200.stages import Tier2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = {  # spec (one layer), prompts, paged
    "C3-7b-ctx2048": (gh.LLAMA2_7B.with_(n_layers=1, max_seq_len=2048), 170, False),
    "C3-7b-ctx2048-paged": (gh.LLAMA2_7B.with_(n_layers=1, max_seq_len=2048), 96, True),
    "C4-13b-ctx4096": (gh.LLAMA2_13B.with_(n_layers=1, max_seq_len=4096), 54, False),
    "C5-70b-ctx8192": (gh.LLAMA2_70B.with_(n_layers=1, max_seq_len=8192), 64, False),
    "C5-70b-ctx8192-paged": (gh.LLAMA2_70B.with_(n_layers=1, max_seq_len=8192), 40, True),
}


def _u16(t):
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("case", list(CASES))
def test_attention_full_size(case, need_gpu):
    spec, B, paged = CASES[case]
    S, D, Dkv, dh = spec.max_seq_len, spec.d_model, spec.d_kv, spec.d_head
    H, Hkv = spec.n_heads, spec.n_kv_heads
    rng = np.random.default_rng(11)
    pos = rng.integers(0, S, B).astype(np.int32)
    pos[0], pos[1], pos[-1] = 0, S - 1, S - 2
    slot = rng.permutation(B).astype(np.uint32)
    if paged:
        pages = sum(-(-(int(p) + 1) // Tier2.PAGE_POSITIONS) for p in pos)
        t2 = Tier2(spec, n_slots=B, n_pages=pages)
        for b in range(B):
            t2.map(int(slot[b]), int(pos[b]) + 1)
    else:
        t2 = Tier2(spec, n_slots=B)
    try:
        t2.fill_synthetic(5, B, S)
        g = torch.Generator(device="cuda").manual_seed(3)
        fwd = torch.randn(B, 2 * D + 2 * Dkv, generator=g, device="cuda").to(torch.bfloat16)
        bwd = torch.zeros(B, 2 * D, dtype=torch.bfloat16, device="cuda")
        t2.attend(0, torch.from_numpy(slot.view(np.int32)).cuda(), torch.from_numpy(pos).cuda(), fwd, bwd)
        torch.cuda.synchronize()
        f, o = _u16(fwd), _u16(bwd)
        assert np.array_equal(o[:, :D], f[:, :D]), "x pass-through must be exact"
        assert np.all(np.isfinite(to_f32(o[:, D:])))
        scale = 1.0 / np.sqrt(dh)
        for b in rng.choice(B, 6, replace=False).tolist() + [0, 1]:
            L, sl = int(pos[b]) + 1, int(slot[b])
            for h in rng.choice(H, 3, replace=False).tolist() + [H - 1]:
                kvh = h // (H // Hkv)
                K = t2.read_kv(0, sl, 0, kvh, L)
                V = t2.read_kv(0, sl, 1, kvh, L)
                # the appended row is the message's key / value, bit for bit
                assert np.array_equal(K[-1], f[b, 2 * D + kvh * dh: 2 * D + (kvh + 1) * dh])
                assert np.array_equal(V[-1], f[b, 2 * D + Dkv + kvh * dh: 2 * D + Dkv + (kvh + 1) * dh])
                q = to_f32(f[b, D + h * dh: D + (h + 1) * dh]).astype(np.float64)
                s = to_f32(K).astype(np.float64) @ q * scale
                p = np.exp(s - s.max())
                ref = (p / p.sum()) @ to_f32(V).astype(np.float64)
                got = to_f32(o[b, D + h * dh: D + (h + 1) * dh])
                tol = 1.6e-2 * np.abs(ref).max()
                err = np.abs(got - ref).max()
                assert err <= tol, f"{case} prompt {b} (pos {L - 1}) head {h}: err {err:.3e} > {tol:.3e}"
    finally:
        t2.close()
