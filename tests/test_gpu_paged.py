"""Paged KV arena: a pool of 64-position pages shared by the context slots.

The paged Tier-2 runs the same attention kernels as the contiguous one with the page table in the
address computation, so on the same logical KV contents and the same messages its results are
BIT-IDENTICAL to the contiguous arena's (which the stage tests hold to the oracle).  Pages are
mapped round-robin across slots so that every slot's positions are scattered over the pool.
"""
import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from paper_2501_11779_b200 import _lib as L

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PAGE = 64
SPECS = {
    "tiny-fp32": gh.TINY.with_(n_layers=2, max_seq_len=200),
    "small-bf16": gh.ModelSpec("small-bf16", 2, 512, 512, 1024, 4, 4, 256, 2, 2000),
    "dh48-bf16": gh.ModelSpec("dh48-bf16", 2, 384, 384, 768, 8, 8, 300, 2, 500),  # 128-position stages
    "dh64-bf16": gh.ModelSpec("dh64-bf16", 2, 512, 512, 768, 8, 8, 192, 2, 777),
    "gqa-bf16": gh.ModelSpec("gqa-bf16", 2, 1024, 256, 1536, 16, 4, 256, 2, 1000),
    "gqa8-dh128": gh.ModelSpec("gqa8-dh128", 2, 2048, 256, 2048, 16, 2, 320, 2, 900),  # tensor-core GQA
    "7b-2layer": gh.LLAMA2_7B.with_(n_layers=2, max_seq_len=512),
}


def _dtype(spec):
    return torch.bfloat16 if spec.dtype_bytes == 2 else torch.float32


def _bits(t):
    return t.view(torch.int16) if t.dtype == torch.bfloat16 else t.view(torch.int32)


@pytest.mark.parametrize("name", list(SPECS))
def test_paged_attention_bit_identical_to_contiguous(name, need_gpu):
    from paper_2501_11779_b200.stages import Tier2, message_buffers
    spec = SPECS[name]
    S = spec.max_seq_len
    B = 13
    n_slots = B + 2
    rng = np.random.default_rng(5)
    pos = rng.integers(0, S, size=B).astype(np.int32)
    pos[:6] = [0, 63, 64, 127, 128, S - 1]
    slot = rng.permutation(n_slots)[:B].astype(np.uint32)
    npos = int(pos.max()) + 1                     # every slot backed up to the longest context
    per_slot = -(-npos // PAGE)
    contig = Tier2(spec, n_slots=n_slots)
    paged = Tier2(spec, n_slots=n_slots, n_pages=n_slots * per_slot + 3)
    for r in range(per_slot):                     # round-robin: a slot's pages are not adjacent
        for s in range(n_slots):
            paged.map(s, min((r + 1) * PAGE, npos))
    assert paged.pages_free == 3
    contig.fill_synthetic(17, n_slots, npos)
    paged.fill_synthetic(17, n_slots, npos)
    for l in (0, 1):
        for s in (0, n_slots - 1):
            for kv in (0, 1):
                assert np.array_equal(contig.read_kv(l, s, kv, spec.n_kv_heads - 1, npos),
                                      paged.read_kv(l, s, kv, spec.n_kv_heads - 1, npos))
    paged.check(slot, pos)
    _, fwd, bwd_c = message_buffers(spec, B)
    bwd_p = torch.empty_like(bwd_c)
    g = torch.Generator(device="cuda").manual_seed(3)
    fwd.copy_(torch.randn(fwd.shape, generator=g, device="cuda", dtype=torch.float32).to(_dtype(spec)))
    d_slot = torch.from_numpy(slot.view(np.int32)).cuda()
    d_pos = torch.from_numpy(pos).cuda()
    for layer in (0, 1):
        contig.attend(layer, d_slot, d_pos, fwd, bwd_c)
        paged.attend(layer, d_slot, d_pos, fwd, bwd_p)
        torch.cuda.synchronize()
        assert torch.isfinite(bwd_c.float()).all()
        assert torch.equal(_bits(bwd_c), _bits(bwd_p)), f"layer {layer}: paged attention differs"
    for b in (0, 2, 5):                           # the appended key / value landed in the right page
        n = int(pos[b]) + 1
        for kv in (0, 1):
            assert np.array_equal(contig.read_kv(1, int(slot[b]), kv, 0, n), paged.read_kv(1, int(slot[b]), kv, 0, n))
    contig.close()
    paged.close()


def test_paged_map_errors(need_gpu):
    from paper_2501_11779_b200.stages import Tier2
    spec = SPECS["small-bf16"]
    t2 = Tier2(spec, n_slots=4, n_pages=5)
    assert t2.pages_free == 5
    t2.map(0, 130)                                # 3 pages
    assert t2.pages_free == 2
    t2.map(0, 100)                                # already backed
    assert t2.pages_free == 2
    with pytest.raises(L.FeasibilityError):       # needs 3, 2 free: nothing is allocated
        t2.map(1, 129)
    assert t2.pages_free == 2
    with pytest.raises(L.FeasibilityError):       # beyond max_seq_len
        t2.map(1, spec.max_seq_len + 1)
    with pytest.raises(L.FeasibilityError):       # slot 0 is backed up to position 191 only
        t2.check(np.array([0], np.uint32), np.array([192], np.int32))
    with pytest.raises(L.FeasibilityError):       # slot 1 has no pages
        t2.check(np.array([1], np.uint32), np.array([0], np.int32))
    t2.check(np.array([0], np.uint32), np.array([191], np.int32))
    with pytest.raises(L.ValidationError):        # fill needs every slot backed by a page
        t2.fill_synthetic(1, 2, 10)
    t2.unmap(0)
    assert t2.pages_free == 5
    t2.map(1, 129)
    assert t2.pages_free == 2
    t2.close()


def test_paged_engine_continuous_batching(need_gpu):
    """Continuous batching on a page pool smaller than lanes x max_seq_len: requests map their
    own length, wait in the queue when the pool is short, and return their pages when done.  The
    tokens equal the contiguous-arena engine's and (fp32) the oracle's."""
    from oracle import Oracle
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    spec = gh.TINY.with_(n_layers=2, max_seq_len=256)
    rng = np.random.default_rng(8)
    lens = [1, 150, 3, 70, 200, 64, 65, 9, 120, 2]
    reqs = [rng.integers(0, spec.vocab_size, size=n, dtype=np.int32) for n in lens]
    max_new = 5
    ref_eng = Engine(spec, batch=3, use_graph=False)
    want, _ = ContinuousDispatcher(ref_eng).run(reqs, max_new)
    ref_eng.close()
    eng = Engine(spec, batch=3, use_graph=False, kv_pages=6)   # 3 lanes x 4 pages would need 12
    got, steps = ContinuousDispatcher(eng).run(reqs, max_new)
    eng.close()
    for w, g in zip(want, got):
        assert np.array_equal(w, g)
    ora = Oracle(spec, n_slots=1)
    for r in (0, 3, 9):
        ref, _ = ora.generate(reqs[r][None, :], max_new)
        assert np.array_equal(got[r], ref[0])
    ora.close()
    # a request longer than the whole pool is reported, not dropped
    eng = Engine(spec, batch=2, use_graph=False, kv_pages=2)
    with pytest.raises(L.FeasibilityError):
        ContinuousDispatcher(eng).run([reqs[4]], max_new)
    eng.close()


@pytest.mark.parametrize("paged", [False, True])
def test_kv_swap_round_trip(paged, need_gpu):
    """gh_tier2_kv_swap: a slot's context saved to host and restored into another slot (other
    pages) reads back bit-identical for every layer, K / V and head."""
    from paper_2501_11779_b200.stages import Tier2
    spec = gh.LLAMA2_70B.with_(n_layers=2, max_seq_len=512)
    n = 200
    t2 = Tier2(spec, n_slots=3, n_pages=12) if paged else Tier2(spec, n_slots=3)
    try:
        if paged:
            t2.map(2, 64)     # slot 2 holds a page first, so slot 0 and slot 1 get other pages
            t2.map(0, n)
        t2.fill_synthetic(7, 1, n)
        size = L.lib().gh_tier2_kv_swap_bytes(t2.h, n)
        buf = np.zeros(size, np.uint8)
        L.check(L.lib().gh_tier2_kv_swap(t2.h, 0, n, buf.ctypes.data, 1, None))
        if paged:
            t2.map(1, n)
        L.check(L.lib().gh_tier2_kv_swap(t2.h, 1, n, buf.ctypes.data, 0, None))
        for layer in range(2):
            for kv in range(2):
                for head in range(spec.n_kv_heads):
                    assert np.array_equal(t2.read_kv(layer, 0, kv, head, n), t2.read_kv(layer, 1, kv, head, n))
        with pytest.raises(L.GhError):
            L.check(L.lib().gh_tier2_kv_swap(t2.h, 0, 513, buf.ctypes.data, 1, None))
    finally:
        t2.close()


@pytest.mark.parametrize("preempt", ["recompute", "swap"])
def test_paged_engine_on_demand_preemption(preempt, need_gpu):
    """On-demand paging: admission maps the prompt only, lanes grow a page at a time, and a dry
    pool preempts the latest request, which recomputes its context on re-admission.  The tokens
    equal the contiguous-arena engine's, with preemptions taken on a 6-page pool."""
    from paper_2501_11779_b200.stages import ContinuousDispatcher, Engine
    spec = gh.TINY.with_(n_layers=2, max_seq_len=256)
    rng = np.random.default_rng(9)
    lens = [60, 100, 3, 70, 40, 64, 65, 9]
    reqs = [rng.integers(0, spec.vocab_size, size=n, dtype=np.int32) for n in lens]
    max_new = 70
    ref_eng = Engine(spec, batch=3, use_graph=False)
    want, _ = ContinuousDispatcher(ref_eng).run(reqs, max_new)
    ref_eng.close()
    eng = Engine(spec, batch=3, use_graph=False, kv_pages=6)
    d = ContinuousDispatcher(eng, on_demand=True, preempt=preempt)
    got, steps = d.run(reqs, max_new)
    eng.close()
    assert d.preemptions > 0
    for w, g in zip(want, got):
        assert np.array_equal(w, g)


def test_paged_ragged_fill(need_gpu):
    """The synthetic fill of a paged arena stops at each slot's mapping and writes the same logical
    values as the contiguous fill."""
    from paper_2501_11779_b200.stages import Tier2
    spec = SPECS["small-bf16"]
    S = spec.max_seq_len
    lens = [1, 64, 65, 200, S]
    contig = Tier2(spec, n_slots=len(lens))
    paged = Tier2(spec, n_slots=len(lens), n_pages=sum(-(-n // PAGE) for n in lens))
    for s, n in enumerate(lens):
        paged.map(s, n)
    assert paged.pages_free == 0
    contig.fill_synthetic(4, len(lens), S)
    paged.fill_synthetic(4, len(lens), S)
    for s, n in enumerate(lens):
        for kv in (0, 1):
            assert np.array_equal(contig.read_kv(1, s, kv, 2, n), paged.read_kv(1, s, kv, 2, n))
    contig.close()
    paged.close()
