"""Edge cases of the stage ABI on the GPU: zero-row calls (an empty shard: a Tier-2
node may take no prompts in a merge) return GH_OK and leave every buffer untouched;
a batch above the Tier-1 handle's max_batch, a layer outside the handle's span and a null
message are rejected with GH_EINVAL before any launch."""
import numpy as np
import pytest

import paper_2501_11779_b200 as gh
from paper_2501_11779_b200 import _lib as L

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SPEC = gh.ModelSpec("edge-bf16", 2, 512, 256, 1024, 8, 4, 128, 2, 1000)


def _lib():
    return L.lib()


def test_zero_rows_are_no_ops(need_gpu):
    from paper_2501_11779_b200.stages import Tier1, Tier2, message_buffers
    t1 = Tier1(SPEC, max_batch=4)
    t2 = Tier2(SPEC, n_slots=4)
    x, fwd, bwd = message_buffers(SPEC, 4)
    for t in (x, fwd, bwd):
        t.fill_(1.5)
    tok = torch.zeros(4, dtype=torch.int32, device="cuda")
    pos = torch.zeros(4, dtype=torch.int32, device="cuda")
    slot = torch.arange(4, dtype=torch.int32, device="cuda")
    nxt = torch.full((4,), 7, dtype=torch.int32, device="cuda")
    logits = torch.full((4, SPEC.vocab_size), 2.0, device="cuda")
    before = [t.clone() for t in (x, fwd, bwd, nxt, logits)]
    p = L.ptr
    assert _lib().gh_tier1_embed(t1.h, 0, p(tok), p(x), None) == 0
    assert _lib().gh_tier1_pre(t1.h, 0, 0, p(x), p(pos), p(fwd), None) == 0
    assert _lib().gh_tier2_attend(t2.h, 0, 0, p(slot), p(pos), p(fwd), p(bwd), None) == 0
    assert _lib().gh_tier2_append(t2.h, 0, 0, p(slot), p(pos), p(fwd), None) == 0
    assert _lib().gh_tier1_post(t1.h, 0, 0, p(bwd), p(x), None) == 0
    assert _lib().gh_tier1_classify(t1.h, 0, p(x), p(logits), p(nxt), None) == 0
    torch.cuda.synchronize()
    for a, b in zip(before, (x, fwd, bwd, nxt, logits)):
        assert torch.equal(a, b)
    # rejected arguments: batch above max_batch, layer outside the span, null message
    assert _lib().gh_tier1_pre(t1.h, 0, 5, p(x), p(pos), p(fwd), None) == L.GH_EINVAL
    assert _lib().gh_tier2_attend(t2.h, SPEC.n_layers, 1, p(slot), p(pos), p(fwd), p(bwd), None) == L.GH_EINVAL
    assert _lib().gh_tier2_attend(t2.h, 0, 1, p(slot), p(pos), None, p(bwd), None) == L.GH_EINVAL
    assert _lib().gh_tier1_pre(t1.h, SPEC.n_layers, 1, p(x), p(pos), p(fwd), None) == L.GH_EINVAL
    torch.cuda.synchronize()
    for a, b in zip(before, (x, fwd, bwd, nxt, logits)):
        assert torch.equal(a, b)
    t1.close()
    t2.close()
