"""Host logic of ContinuousDispatcher's paged admission (CPU, no GPU): on-demand page growth with
recompute preemption against a fake engine whose next token is a hash of the lane's whole
context, so a token is right only when every position below it was written by the same request
in order (what the real KV arena requires).  Checks the page accounting never exceeds the pool,
every attended position is mapped, and each request's tokens equal decoding it alone."""
import hashlib

import numpy as np
import pytest

from paper_2501_11779_b200 import _lib as L
from paper_2501_11779_b200.stages import ContinuousDispatcher

PAGE = ContinuousDispatcher.PAGE


def _next(ctx):
    return int.from_bytes(hashlib.blake2b(np.asarray(ctx, np.int64).tobytes(), digest_size=4).digest(), "little") % 1000


class FakeEngine:
    role = "colocated"

    def __init__(self, batch, kv_pages):
        self.batch, self.kv_pages = batch, kv_pages
        self.pages = [0] * batch
        self.hist = [dict() for _ in range(batch)]
        self.peak = 0
        self.swaps = 0

    def shard(self):
        return -1, 0, self.batch, 0

    def kv_map(self, slot, n):
        self.pages[slot] = max(self.pages[slot], -(-n // PAGE))
        assert sum(self.pages) <= self.kv_pages, "pool over-committed"
        self.peak = max(self.peak, sum(self.pages))

    def kv_unmap(self, slot):
        self.pages[slot] = 0

    def set_sampling(self, t, s):
        pass

    def kv_swap_out(self, slot, n):
        assert self.pages[slot] * PAGE >= n
        self.swaps += 1
        return [self.hist[slot][i] for i in range(n)]

    def kv_swap_in(self, slot, n, buf):
        assert self.pages[slot] * PAGE >= n and len(buf) == n
        self.hist[slot] = dict(enumerate(buf))

    def step_host(self, tok, pos):
        nxt = np.zeros(self.batch, np.int32)
        for b in range(self.batch):
            p = int(pos[b])
            assert self.pages[b] * PAGE >= p + 1, "attended position not mapped"
            self.hist[b][p] = int(tok[b])
            nxt[b] = _next([self.hist[b][i] for i in range(p + 1)])
        return nxt, None


def _alone(req, max_new):
    ctx, out = list(req), []
    for _ in range(max_new):
        out.append(_next(ctx))
        ctx.append(out[-1])
    return out


def _requests(n, seed=3):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 1000, int(rng.integers(1, 150))).astype(np.int32) for _ in range(n)]


@pytest.mark.parametrize("on_demand,preempt", [(False, "recompute"), (True, "recompute"), (True, "swap")])
def test_paged_admission_matches_alone(on_demand, preempt):
    reqs, max_new, B = _requests(10), 90, 4
    eng = FakeEngine(B, kv_pages=9)
    d = ContinuousDispatcher(eng, on_demand=on_demand, preempt=preempt)
    got, steps = d.run(reqs, max_new)
    for r, g in zip(reqs, got):
        assert g.tolist() == _alone(r.tolist(), max_new)
    if on_demand:
        assert d.preemptions > 0      # this pool is too small for 4 concurrent full requests
        assert (eng.swaps > 0) == (preempt == "swap")
    else:
        assert d.preemptions == 0


def test_swap_takes_fewer_steps_than_recompute():
    reqs, max_new, B = _requests(10), 90, 4
    steps = {}
    for preempt in ("recompute", "swap"):
        d = ContinuousDispatcher(FakeEngine(B, kv_pages=9), on_demand=True, preempt=preempt)
        _, steps[preempt] = d.run(reqs, max_new)
    assert steps["swap"] < steps["recompute"]


def test_bad_preempt_policy():
    with pytest.raises(ValueError):
        ContinuousDispatcher(FakeEngine(2, 4), preempt="drop")


def test_on_demand_admits_more_than_up_front():
    """With a pool that backs every lane's prompt but not every lane's full length, on-demand
    paging runs more requests at once than mapping the full length at admission."""
    reqs, max_new, B = _requests(8, seed=5), 64, 4
    res = {}
    for od in (False, True):
        eng = FakeEngine(B, kv_pages=12)
        d = ContinuousDispatcher(eng, on_demand=od)
        got, steps = d.run(reqs, max_new)
        for r, g in zip(reqs, got):
            assert g.tolist() == _alone(r.tolist(), max_new)
        res[od] = steps
    assert res[True] <= res[False]


def test_on_demand_rejects_request_larger_than_pool():
    eng = FakeEngine(2, kv_pages=3)
    with pytest.raises(L.FeasibilityError):
        ContinuousDispatcher(eng, on_demand=True).run([np.arange(150, dtype=np.int32)], 40)


def test_shortest_first_order():
    """order="shortest": requests are admitted by prompt length (ties in request order); tokens
    are unchanged, and with one lane the admission order is exactly the sorted order."""
    reqs, max_new = _requests(7, seed=9), 20
    eng = FakeEngine(1, kv_pages=8)
    seen = []
    step = eng.step_host

    def spy(tok, pos):
        if int(pos[0]) == 0:
            seen.append(int(tok[0]))
        return step(tok, pos)
    eng.step_host = spy
    got, _ = ContinuousDispatcher(eng, order="shortest").run(reqs, max_new)
    for r, g in zip(reqs, got):
        assert g.tolist() == _alone(r.tolist(), max_new)
    want = [int(reqs[i][0]) for i in sorted(range(len(reqs)), key=lambda i: len(reqs[i]))]
    assert seen == want
    with pytest.raises(ValueError):
        ContinuousDispatcher(eng, order="random")


class FakeShardEngine(FakeEngine):
    """A rank of a tier split with K' Tier-2 shards, each with its own page pool: Tier-1 sees
    tokens and no KV; Tier-2 shard j holds lanes [off, off + cnt) and sees no tokens."""

    def __init__(self, batch, kv_pages, kp, j):
        from paper_2501_11779_b200.spec import shard_plan
        offs, cnts = shard_plan(batch, kp)
        self.kp, self.j = kp, j
        self.role = "tier1" if j < 0 else "tier2"
        self.off, self.cnt = (0, batch) if j < 0 else (offs[j], cnts[j])
        super().__init__(self.cnt, kv_pages)
        self.batch = batch
        self.maps = 0

    def shard(self):
        return self.j, self.off, self.cnt, self.kp

    def kv_map(self, slot, n):
        assert self.role == "tier2" and 0 <= slot < self.cnt
        self.maps += 1
        super().kv_map(slot, n)

    def kv_unmap(self, slot):
        assert self.role == "tier2"
        super().kv_unmap(slot)

    def kv_swap_out(self, slot, n):
        assert self.role == "tier2" and self.pages[slot] * PAGE >= n
        self.swaps += 1
        return [0] * n

    def kv_swap_in(self, slot, n, buf):
        assert self.role == "tier2" and self.pages[slot] * PAGE >= n and len(buf) == n

    def step_host(self, tok, pos):
        if self.role == "tier2":
            assert tok is None and pos is None
            return None, None
        # Tier-1: tokens only (its decisions must not depend on their values)
        return np.array([_next([int(tok[b]), int(pos[b])]) for b in range(self.batch)], np.int32), None


@pytest.mark.parametrize("preempt", ["recompute", "swap"])
def test_on_demand_spmd_decisions_agree_across_ranks(preempt):
    """Tier split SPMD: every rank runs the dispatcher over the same requests; admission and
    preemption depend only on lengths and per-shard page accounting, so the Tier-1 rank and each
    Tier-2 rank take the same number of steps and preemptions, and no shard pool over-commits."""
    reqs, max_new, B, kp, pages = _requests(12, seed=4), 70, 6, 3, 5
    runs = []
    for j in [-1] + list(range(kp)):
        eng = FakeShardEngine(B, pages, kp, j)
        d = ContinuousDispatcher(eng, on_demand=True, preempt=preempt)
        _, steps = d.run(reqs, max_new)
        runs.append((steps, d.preemptions, eng))
    assert len({(s, p) for s, p, _ in runs}) == 1, [(s, p) for s, p, _ in runs]
    assert runs[0][1] > 0
    for _, _, eng in runs[1:]:
        assert eng.peak <= pages and eng.maps > 0
    swaps = sum(eng.swaps for _, _, eng in runs[1:])  # swap preemption really happens in the split
    assert swaps > 0 if preempt == "swap" else swaps == 0


@pytest.mark.parametrize("chunk", [1, 4])
@pytest.mark.parametrize("lag", [1, 3])
@pytest.mark.parametrize("on_demand,preempt", [(False, "recompute"), (True, "recompute"), (True, "swap")])
def test_scheduler_inflight_shards_lagged_tokens(on_demand, preempt, lag, chunk):
    """The native scheduler (gh_sched) over IF = 2 in-flight batches x B = 5 lanes split into K' = 2
    Tier-2 shards with their own page pools, its tokens resolved `lag` steps late: every request's
    tokens equal decoding it alone, every attended position is mapped on the lane's own shard,
    no pool over-commits, and a swapped context comes back on the shard that saved it."""
    from paper_2501_11779_b200.stages import Scheduler
    IF, B, kp, pages, max_new = 2, 5, 2, 9, 70
    reqs = _requests(14, seed=11)
    sch = Scheduler(B, max_new, IF, kp, pages, 0, on_demand, preempt, chunk=chunk)
    ids = [sch.submit(r) for r in reqs]
    lanes = IF * B
    shard = lambda lane: 0 if lane % B < 3 else 1  # noqa: E731  (shard_plan(5, 2) = 3 + 2 rows)
    mapped = [0] * lanes
    hist = [dict() for _ in range(lanes)]
    saved = {}
    last = np.zeros(lanes, np.int32)
    pending = []
    while not sch.done:
        ins, acts = sch.plan()
        for op, lane, n, buf in acts:
            if op == Scheduler.MAP:
                mapped[lane] = max(mapped[lane], -(-n // PAGE))
            elif op == Scheduler.UNMAP:
                mapped[lane] = 0
            elif op == Scheduler.SWAP_OUT:
                assert mapped[lane] * PAGE >= n
                saved[buf] = (shard(lane), [hist[lane][i] for i in range(n)])
            else:
                sh, ctx = saved.pop(buf)
                assert sh == shard(lane) and mapped[lane] * PAGE >= n == len(ctx)
                hist[lane] = dict(enumerate(ctx))
        for j in range(kp):
            assert sum(m for lane, m in enumerate(mapped) if shard(lane) == j) <= pages
        busy = ins[:, 0] != Scheduler.SRC_IDLE
        if not busy.any():
            while sch.unresolved:
                sch.resolve(pending.pop(0))
            continue
        nxt = np.zeros(lanes, np.int32)
        rows = []
        for lane in range(lanes):
            src, tok, p, home = (int(v) for v in ins[lane])
            # a row carries only a prompt token of a lane of its own in-flight batch and shard
            assert home // B == lane // B and shard(home) == shard(lane)
            if home != lane:
                assert chunk > 1 and src == Scheduler.SRC_HOST and ins[home][0] == Scheduler.SRC_HOST
            if src == Scheduler.SRC_DEVICE:
                tok = int(last[lane])
            assert mapped[home] * PAGE >= p + 1, "attended position not mapped"
            hist[home][p] = tok
            rows.append((lane, home, p))
        for lane, home, p in rows:  # a prefill-row engine appends every row before attention
            nxt[lane] = _next([hist[home][i] for i in range(p + 1)])
        last = nxt
        sch.commit()
        pending.append(nxt.copy())
        while sch.unresolved > lag:
            sch.resolve(pending.pop(0))
    while sch.unresolved:
        sch.resolve(pending.pop(0))
    for r, i in zip(reqs, ids):
        assert sch.result(i).tolist() == _alone(r.tolist(), max_new)
    st = sch.stats()
    assert st["finished"] == len(reqs) and st["tokens"] >= len(reqs) * max_new
    if on_demand:
        assert st["preemptions"] > 0 and (st["swaps"] > 0) == (preempt == "swap")


@pytest.mark.parametrize("on_demand", [False, True])
def test_per_request_max_new(on_demand):
    """max_new per request: each request generates its own count and equals decoding it alone."""
    reqs = _requests(9, seed=21)
    per = [int(n) for n in np.random.default_rng(3).integers(1, 80, len(reqs))]
    eng = FakeEngine(3, kv_pages=9)
    got, _ = ContinuousDispatcher(eng, on_demand=on_demand).run(reqs, per)
    for r, n, g in zip(reqs, per, got):
        assert g.tolist() == _alone(r.tolist(), n)


def test_chunked_prefill_fills_idle_lanes():
    """Chunked prefill: with fewer requests than lanes, idle lanes carry further prompt
    tokens of the requests still reading their prompts, so the run takes fewer steps; tokens are
    unchanged (checked against decoding alone, as above)."""
    from paper_2501_11779_b200.stages import Scheduler
    rng = np.random.default_rng(3)
    reqs = [rng.integers(0, 1000, n).astype(np.int32) for n in (40, 33, 9, 64)]
    B, IF, kp, max_new = 8, 2, 2, 6
    steps = {}
    for chunk in (1, 8):
        sch = Scheduler(B, max_new, IF, kp, chunk=chunk)
        ids = [sch.submit(r) for r in reqs]
        hist = [dict() for _ in range(IF * B)]
        widest = 0
        while not sch.done:
            ins, _ = sch.plan()
            nxt = np.zeros(IF * B, np.int32)
            for lane in range(IF * B):
                src, tok, p, home = (int(v) for v in ins[lane])
                if src == Scheduler.SRC_DEVICE:
                    tok = int(last[lane])
                hist[home][p] = tok
            for lane in range(IF * B):
                p, home = int(ins[lane][2]), int(ins[lane][3])
                nxt[lane] = _next([hist[home][i] for i in range(p + 1)])
            widest = max(widest, max(int(np.sum(ins[:, 3] == h)) for h in range(IF * B)))
            last = nxt
            sch.commit()
            sch.resolve(nxt)
        for r, i in zip(reqs, ids):
            assert sch.result(i).tolist() == _alone(r.tolist(), max_new)
        steps[chunk] = sch.stats()["steps"]
        assert widest == (1 if chunk == 1 else 4)  # 4 lanes per (batch, shard): 1 request + 3 idle
        sch.close()
    assert steps[8] < steps[1] / 2, steps
