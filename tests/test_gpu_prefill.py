"""Mixed prefill + decode batches: rows of one step may hold several consecutive
prompt tokens of one request (chunked prefill) next to other requests' decode rows.

Parity: every request's greedy tokens equal decoding it alone -- against the fp32 oracle
(bit-exact) and, for bf16, against the lane-per-request ContinuousDispatcher on an engine of the
same row count (bit-identical: the GEMMs and attention are row-independent for a fixed batch).
"""
import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from paper_2501_11779_b200 import _lib as L

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _requests(spec, lens, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, spec.vocab_size, size=n, dtype=np.int32) for n in lens]


def test_mixed_prefill_fp32_matches_oracle(need_gpu):
    from oracle import Oracle
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine, MixedDispatcher
    spec = gh.TINY.with_(n_layers=3, max_seq_len=128)
    reqs = _requests(spec, [1, 37, 5, 16, 17, 40, 2, 9], 31)
    max_new = 6
    eng = Engine(spec, batch=16, n_slots=6, use_graph=False, prefill=True)
    got, steps = MixedDispatcher(eng, chunk=8).run(reqs, max_new)
    eng.close()
    ora = Oracle(spec, n_slots=1)
    for r, g in zip(reqs, got):
        ref, _ = ora.generate(r[None, :], max_new)
        assert np.array_equal(g, ref[0]), (len(r), g, ref[0])
    ora.close()
    eng = Engine(spec, batch=5, use_graph=False)
    _, steps_lane = ContinuousDispatcher(eng).run(reqs, max_new)
    eng.close()
    assert steps < 0.75 * steps_lane, (steps, steps_lane)


@pytest.mark.parametrize("paged", [False, True])
def test_mixed_prefill_bf16_matches_continuous(paged, need_gpu):
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine, MixedDispatcher
    spec = gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=256)
    reqs = _requests(spec, [3, 70, 1, 33, 129, 12, 64, 65, 8, 20], 9)
    max_new = 5
    B = 24
    ref_eng = Engine(spec, batch=B, use_graph=False)
    want, _ = ContinuousDispatcher(ref_eng).run(reqs, max_new)
    ref_eng.close()
    eng = Engine(spec, batch=B, n_slots=B + 1, use_graph=True, prefill=True,
                 kv_pages=(10 if paged else 0))   # paged: requests wait for pages
    got, steps = MixedDispatcher(eng, chunk=16).run(reqs, max_new)
    eng.close()
    for i, (w, g) in enumerate(zip(want, got)):
        assert np.array_equal(w, g), (i, len(reqs[i]), w, g)


@pytest.mark.parametrize("inflight,graph", [(1, False), (2, True)])
def test_native_chunked_prefill_fp32_matches_oracle(inflight, graph, need_gpu):
    """The native dispatcher's chunked prefill (gh_dispatch_config.prefill_chunk): idle
    lanes carry further prompt tokens of requests still reading their prompts; greedy tokens
    bit-exact against the fp32 oracle, and fewer steps than one prompt token per step."""
    from oracle import Oracle
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    spec = gh.TINY.with_(n_layers=3, max_seq_len=128)
    reqs = _requests(spec, [1, 37, 5, 16, 17, 40, 2, 9, 30, 3], 31)
    max_new = 6
    eng = Engine(spec, batch=8, inflight=inflight, use_graph=graph, prefill=True)
    got, steps = ContinuousDispatcher(eng, chunk=8).run(reqs, max_new)
    eng.close()
    ora = Oracle(spec, n_slots=1)
    for r, g in zip(reqs, got):
        ref, _ = ora.generate(r[None, :], max_new)
        assert np.array_equal(g, ref[0]), (len(r), g, ref[0])
    ora.close()
    eng = Engine(spec, batch=8, inflight=inflight, use_graph=graph)
    _, steps_lane = ContinuousDispatcher(eng).run(reqs, max_new)
    eng.close()
    assert steps < 0.75 * steps_lane, (steps, steps_lane)


@pytest.mark.parametrize("on_demand", [False, True])
def test_native_chunked_prefill_bf16_matches_lanes(on_demand, need_gpu):
    """bf16 7B widths, paged arena (on-demand growth maps each chunk's pages): tokens bit-identical
    to the lane-per-request dispatcher at the same row count (row-independent GEMMs/attention)."""
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    spec = gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=256)
    reqs = _requests(spec, [3, 70, 1, 33, 129, 12, 64, 65, 8, 20], 9)
    max_new = 5
    B = 12
    ref_eng = Engine(spec, batch=B, use_graph=False)
    want, _ = ContinuousDispatcher(ref_eng).run(reqs, max_new)
    ref_eng.close()
    eng = Engine(spec, batch=B, use_graph=True, prefill=True, kv_pages=24)
    got, _ = ContinuousDispatcher(eng, on_demand=on_demand, chunk=16).run(reqs, max_new)
    eng.close()
    for i, (w, g) in enumerate(zip(want, got)):
        assert np.array_equal(w, g), (i, len(reqs[i]), w, g)


def test_chunked_prefill_needs_prefill_engine(need_gpu):
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    eng = Engine(gh.TINY.with_(n_layers=2, max_seq_len=64), batch=4, use_graph=False)
    with pytest.raises(L.ValidationError):
        ContinuousDispatcher(eng, chunk=4)
    eng.close()


def test_tier2_append_writes_rows(need_gpu):
    from paper_2501_11779_b200.stages import Tier2, message_buffers
    spec = gh.ModelSpec("small-bf16", 2, 512, 512, 1024, 4, 4, 256, 2, 2000)
    t2 = Tier2(spec, n_slots=3)
    _, fwd, _ = message_buffers(spec, 4)
    fwd.copy_(torch.randn(fwd.shape, device="cuda").to(torch.bfloat16))
    slot = torch.tensor([2, 2, 0, 1], dtype=torch.int32, device="cuda")
    pos = torch.tensor([5, 6, 0, 200], dtype=torch.int32, device="cuda")
    t2.append(1, slot, pos, fwd)
    torch.cuda.synchronize()
    D, Dkv, dh = spec.d_model, spec.d_kv, spec.d_head
    f = fwd.cpu().view(torch.int16).numpy().view(np.uint16)
    for b in range(4):
        s, p = int(slot[b]), int(pos[b])
        for kv in (0, 1):
            for h in (0, spec.n_kv_heads - 1):
                got = t2.read_kv(1, s, kv, h, p + 1)[p]
                want = f[b, 2 * D + kv * Dkv + h * dh: 2 * D + kv * Dkv + (h + 1) * dh]
                assert np.array_equal(got, want)
    t2.close()


def test_prefill_rejected_on_split_and_validation(need_gpu):
    from paper_2501_11779_b200.stages import Engine, MixedDispatcher
    spec = gh.TINY.with_(n_layers=2, max_seq_len=64)
    eng = Engine(spec, batch=4, use_graph=False)
    with pytest.raises(L.ValidationError):
        MixedDispatcher(eng)
    with pytest.raises(L.ValidationError):
        eng.set_slots(np.array([0, 1, 2, 4], np.uint32))
    eng.close()
