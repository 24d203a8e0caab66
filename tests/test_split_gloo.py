"""Tier-split protocol on CPU (gloo, world sizes 2 and 3): rank 0 plays Tier-1, ranks 1.. play
Tier-2 over their prompt shard, exchanging exactly the per-layer PayloadModel messages the GPU
engine sends over NCCL (fwd [x|q|k|v] per shard, bwd [x|attn] per shard, plus the positions at
the start of a step), with the oracle as the stage implementation.  The result must equal the
colocated oracle bit for bit (same arithmetic, same message bytes)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2501_11779_b200 as gh
from _ranks import collect, init_rank, spawn

SPEC = gh.ModelSpec("split-cpu", 2, 128, 64, 192, 4, 2, 32, 2, 97)
B, STEPS, SEED = 7, 5, 1234



def reference_tokens(B=B, spec=SPEC):
    from oracle import Oracle
    ora = Oracle(spec, seed=SEED, n_slots=B)
    prompts = np.random.default_rng(2).integers(0, spec.vocab_size, size=(B, 2), dtype=np.int32)
    gen, lg = ora.generate(prompts, STEPS)
    return prompts, gen, lg


def worker(rank, world, port, out_q, B=B):
    init_rank(rank, world, port)
    from oracle import Oracle
    kp = world - 1
    off, cnt = gh.shard_plan(B, kp)
    prompts = np.random.default_rng(2).integers(0, SPEC.vocab_size, size=(B, 2), dtype=np.int32)
    D, Dkv = SPEC.d_model, SPEC.d_kv
    if rank == 0:
        ora = Oracle(SPEC, seed=SEED, n_slots=1)        # Tier-1: weights
        x, fwd, bwd = ora.buffers(B)
        tok = prompts[:, 0].copy()
        out = []
        for t in range(1 + STEPS):
            pos = np.full(B, t, np.int32)
            for j in range(kp):                          # step header: positions of each shard
                dist.send(torch.from_numpy(pos[off[j]:off[j] + cnt[j]].copy()), dst=j + 1)
            ora.embed(tok, x)
            for layer in range(SPEC.n_layers):
                ora.pre(layer, x, pos, fwd)
                for j in range(kp):                      # fwd message shards
                    dist.send(torch.from_numpy(fwd[off[j]:off[j] + cnt[j]].view(np.int16).copy()), dst=j + 1)
                for j in range(kp):                      # bwd message shards
                    buf = torch.zeros((cnt[j], 2 * D), dtype=torch.int16)
                    dist.recv(buf, src=j + 1)
                    bwd[off[j]:off[j] + cnt[j]] = buf.numpy().view(np.uint16)
                x2 = np.zeros_like(x)
                ora.post(layer, bwd, x2)
                x = x2
            nxt, lg = ora.classify(x)
            if t >= 1:
                out.append((nxt.copy(), lg.copy()))
            tok = prompts[:, 1].copy() if t == 0 else nxt
        out_q.put((np.stack([o[0] for o in out], 1), np.stack([o[1] for o in out], 1)))
    else:
        j = rank - 1
        n = cnt[j]
        ora = Oracle(SPEC, seed=SEED, n_slots=n)         # Tier-2: KV of my shard only
        slot = np.arange(n, dtype=np.uint32)
        for t in range(1 + STEPS):
            pos_t = torch.zeros(n, dtype=torch.int32)
            dist.recv(pos_t, src=0)
            pos = pos_t.numpy()
            for layer in range(SPEC.n_layers):
                buf = torch.zeros((n, 2 * D + 2 * Dkv), dtype=torch.int16)
                dist.recv(buf, src=0)
                fwd = buf.numpy().view(np.uint16).copy()
                bwd = np.zeros((n, 2 * D), np.uint16)
                ora.attend(layer, slot, pos, fwd, bwd)
                dist.send(torch.from_numpy(bwd.view(np.int16).copy()), dst=0)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(2, B), (3, B), (8, 15)])
def test_tier_split_protocol_matches_colocated(world, B):
    """world 8 = BASELINE C3's largest layout: one Tier-1 + K' = 7 Tier-2 ranks (shards 3,2,...,2)."""
    _, gen, lg = reference_tokens(B)
    procs, q = spawn(worker, world, (B,))
    sgen, slg = collect(procs, q, 1, 240)[0]
    assert np.array_equal(sgen, gen)
    assert np.array_equal(slg, lg)


def worker_pp(rank, world, port, out_q, B=B):
    """Tier-1 pipeline stages (SURVEY 8e, config 5 at toy scale): ranks 0/1 are Tier-1 spans of
    layer_spans(N, 2), ranks 2 + s*K' + j are the K' Tier-2 ranks of span s (its layers' KV of
    prompt shard j).  Span 0 embeds, hands [x] (PayloadModel intra-Tier-1 message,
    netmodel.cpp:22) plus the positions to span 1; span 1 classifies and hands the next tokens
    back to span 0.  The layout is the engine's (gh_engine_layout)."""
    init_rank(rank, world, port)
    from oracle import Oracle
    n1 = 2
    kp = (world - n1) // n1
    off, cnt = gh.shard_plan(B, kp)
    lay = gh.engine_layout(world, rank, B, SPEC.n_layers, tier1_ranks=n1)
    spans = gh.layer_spans(SPEC.n_layers, n1)
    lo = [sum(spans[:s]) for s in range(n1)]
    prompts = np.random.default_rng(2).integers(0, SPEC.vocab_size, size=(B, 2), dtype=np.int32)
    D, Dkv = SPEC.d_model, SPEC.d_kv
    if rank < n1:
        sp = rank
        ora = Oracle(SPEC, seed=SEED, n_slots=1)
        x, fwd, bwd = ora.buffers(B)
        tok = prompts[:, 0].copy()
        out = []
        for t in range(1 + STEPS):
            if sp == 0:
                pos = np.full(B, t, np.int32)
                ora.embed(tok, x)
            else:
                pos_t = torch.zeros(B, dtype=torch.int32)
                dist.recv(pos_t, src=sp - 1)
                pos = pos_t.numpy().copy()
                xb = torch.zeros((B, D), dtype=torch.int16)
                dist.recv(xb, src=sp - 1)
                x = xb.numpy().view(np.uint16).copy()
            assert lay["role"] == "tier1" and lay["layers"] == (lo[sp], lo[sp] + spans[sp])
            for j in range(kp):                                           # positions to my Tier-2 shards
                dist.send(torch.from_numpy(pos[off[j]:off[j] + cnt[j]].copy()), dst=n1 + sp * kp + j)
            for layer in range(lo[sp], lo[sp] + spans[sp]):
                ora.pre(layer, x, pos, fwd)
                for j in range(kp):
                    dist.send(torch.from_numpy(fwd[off[j]:off[j] + cnt[j]].view(np.int16).copy()),
                              dst=n1 + sp * kp + j)
                for j in range(kp):
                    buf = torch.zeros((cnt[j], 2 * D), dtype=torch.int16)
                    dist.recv(buf, src=n1 + sp * kp + j)
                    bwd[off[j]:off[j] + cnt[j]] = buf.numpy().view(np.uint16)
                x2 = np.zeros_like(x)
                ora.post(layer, bwd, x2)
                x = x2
            if sp + 1 < n1:
                dist.send(torch.from_numpy(pos.copy()), dst=sp + 1)
                dist.send(torch.from_numpy(x.view(np.int16).copy()), dst=sp + 1)
            if sp == n1 - 1:
                nxt, lg = ora.classify(x)
                if t >= 1:
                    out.append((nxt.copy(), lg.copy()))
                dist.send(torch.from_numpy(nxt.astype(np.int32)), dst=0)
            if sp == 0:
                nt = torch.zeros(B, dtype=torch.int32)
                dist.recv(nt, src=n1 - 1)
                tok = prompts[:, 1].copy() if t == 0 else nt.numpy().copy()
        if sp == n1 - 1:
            out_q.put((np.stack([o[0] for o in out], 1), np.stack([o[1] for o in out], 1)))
    else:
        sp, j = (rank - n1) // kp, (rank - n1) % kp
        n = cnt[j]
        assert lay == dict(role="tier2", span=sp, tp_rank=0, shard=j, kp=kp, layers=(lo[sp], lo[sp] + spans[sp]),
                           rows=(off[j], n))
        ora = Oracle(SPEC, seed=SEED, n_slots=n)        # this span's layers of my shard's prompts
        slot = np.arange(n, dtype=np.uint32)
        for t in range(1 + STEPS):
            pos_t = torch.zeros(n, dtype=torch.int32)
            dist.recv(pos_t, src=sp)
            pos = pos_t.numpy()
            for layer in range(lo[sp], lo[sp] + spans[sp]):
                buf = torch.zeros((n, 2 * D + 2 * Dkv), dtype=torch.int16)
                dist.recv(buf, src=sp)
                fwd = buf.numpy().view(np.uint16).copy()
                bwd = np.zeros((n, 2 * D), np.uint16)
                ora.attend(layer, slot, pos, fwd, bwd)
                dist.send(torch.from_numpy(bwd.view(np.int16).copy()), dst=sp)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(4, B), (8, 13)])
def test_tier1_pipeline_protocol_matches_colocated(world, B):
    """world 8 = BASELINE C5 as pipeline spans: T = 2 Tier-1 spans, K' = 3 Tier-2 ranks each."""
    _, gen, lg = reference_tokens(B)
    procs, q = spawn(worker_pp, world, (B,))
    sgen, slg = collect(procs, q, 1, 240)[0]
    assert np.array_equal(sgen, gen)
    assert np.array_equal(slg, lg)


def worker_pp_groups(rank, world, port, out_q, B, IF):
    """Tier-1 pipeline spans with IF in-flight batches in the engine's order (split_step_peer):
    the batches form min(IF, spans) groups processed one after another on every rank, each
    group's batches interleaved per layer; a span hands a batch on after its last layer, the
    last span returns the batch's next tokens, and the first span takes them when that batch's
    next step starts (the deferred gh_engine_advance).  Sends are non-blocking, like the copy
    engines of the peer transport; every receive blocks, so an ordering that could deadlock
    the GPU engine's flag waits hangs here."""
    init_rank(rank, world, port)
    from oracle import Oracle
    n1 = 2
    kp = (world - n1) // n1
    ng = min(IF, n1)
    groups = [range(g * IF // ng, (g + 1) * IF // ng) for g in range(ng)]
    off, cnt = gh.shard_plan(B, kp)
    spans = gh.layer_spans(SPEC.n_layers, n1)
    lo = [sum(spans[:s]) for s in range(n1)]
    prompts = np.random.default_rng(2).integers(0, SPEC.vocab_size, size=(IF * B, 2), dtype=np.int32)
    D, Dkv = SPEC.d_model, SPEC.d_kv
    pending = []

    def isend(a, dst):
        t = torch.from_numpy(np.ascontiguousarray(a))
        pending.append((dist.isend(t, dst=dst), t))  # the tensor stays alive until the send is done

    def recv(shape, dtype, src):
        t = torch.zeros(shape, dtype=dtype)
        dist.recv(t, src=src)
        return t.numpy()

    if rank < n1:
        sp = rank
        ora = Oracle(SPEC, seed=SEED, n_slots=1)
        bufs = [ora.buffers(B) for _ in range(IF)]
        tok = [prompts[ib * B:(ib + 1) * B, 0].copy() for ib in range(IF)]
        pos = [None] * IF
        out = [[] for _ in range(IF)]
        for t in range(1 + STEPS):
            for grp in groups:
                for ib in grp:
                    x, fwd, _ = bufs[ib]
                    if sp == 0:
                        if t >= 1:  # this batch's tokens of step t - 1 from the last span
                            nt = recv(B, torch.int32, n1 - 1)
                            tok[ib] = prompts[ib * B:(ib + 1) * B, 1].copy() if t == 1 else nt.copy()
                        pos[ib] = np.full(B, t, np.int32)
                        ora.embed(tok[ib], x)
                    else:
                        pos[ib] = recv(B, torch.int32, sp - 1).copy()
                        x[:] = recv((B, D), torch.int16, sp - 1).view(np.uint16)
                    ora.pre(lo[sp], x, pos[ib], fwd)
                    for j in range(kp):  # positions + the first fwd of this batch to my shards
                        isend(pos[ib][off[j]:off[j] + cnt[j]], n1 + sp * kp + j)
                        isend(fwd[off[j]:off[j] + cnt[j]].view(np.int16), n1 + sp * kp + j)
                for layer in range(lo[sp], lo[sp] + spans[sp]):
                    for ib in grp:
                        x, fwd, bwd = bufs[ib]
                        for j in range(kp):
                            bwd[off[j]:off[j] + cnt[j]] = recv((cnt[j], 2 * D), torch.int16, n1 + sp * kp + j).view(np.uint16)
                        x2 = np.zeros_like(x)
                        ora.post(layer, bwd, x2)
                        x[:] = x2
                        if layer + 1 < lo[sp] + spans[sp]:
                            ora.pre(layer + 1, x, pos[ib], fwd)
                            for j in range(kp):
                                isend(fwd[off[j]:off[j] + cnt[j]].view(np.int16), n1 + sp * kp + j)
                        elif sp + 1 < n1:
                            isend(pos[ib], sp + 1)
                            isend(x.view(np.int16), sp + 1)
                        else:
                            nxt, lg = ora.classify(x)
                            if t >= 1:
                                out[ib].append((nxt.copy(), lg.copy()))
                            isend(nxt.astype(np.int32), 0)
        if sp == 0:  # the last step's tokens (the next step would take them)
            for grp in groups:
                for ib in grp:
                    recv(B, torch.int32, n1 - 1)
        if sp == n1 - 1:
            out_q.put([(np.stack([o[0] for o in out[ib]], 1), np.stack([o[1] for o in out[ib]], 1))
                       for ib in range(IF)])
    else:
        sp, j = (rank - n1) // kp, (rank - n1) % kp
        n = cnt[j]
        ora = Oracle(SPEC, seed=SEED, n_slots=n * IF)  # slots ib * n + i: batch ib's prompts of my shard
        pos = [None] * IF
        for t in range(1 + STEPS):
            for grp in groups:
                for layer in range(lo[sp], lo[sp] + spans[sp]):
                    for ib in grp:
                        if layer == lo[sp]:
                            pos[ib] = recv(n, torch.int32, sp).copy()
                        fwd = recv((n, 2 * D + 2 * Dkv), torch.int16, sp).view(np.uint16).copy()
                        bwd = np.zeros((n, 2 * D), np.uint16)
                        ora.attend(layer, np.arange(ib * n, (ib + 1) * n, dtype=np.uint32), pos[ib], fwd, bwd)
                        isend(bwd.view(np.int16), sp)
    for r, _ in pending:
        r.wait()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B,IF", [(4, B, 4), (8, 13, 6), (8, 13, 3)])
def test_tier1_pipeline_groups_protocol(world, B, IF):
    """The 8-GPU bench default (two Tier-1 spans, K' = 3 each, IF 6 in two groups) and uneven
    groups (IF 3): every batch's tokens and logits equal the colocated oracle's."""
    _, gen, lg = reference_tokens(IF * B)
    procs, q = spawn(worker_pp_groups, world, (B, IF))
    res = collect(procs, q, 1, 240)[0]
    for ib in range(IF):
        assert np.array_equal(res[ib][0], gen[ib * B:(ib + 1) * B])
        assert np.array_equal(res[ib][1], lg[ib * B:(ib + 1) * B])


def test_shard_plan_balanced():
    for batch, kp in ((1024, 7), (7, 3), (170, 1), (1190, 7)):
        off, cnt = gh.shard_plan(batch, kp)
        assert sum(cnt) == batch and max(cnt) - min(cnt) <= 1
        assert off == [sum(cnt[:j]) for j in range(kp)]
    with pytest.raises(gh.ValidationError):
        gh.shard_plan(2, 3)


# ------------------------------------------------------------------ Tier-1 tensor parallelism
TP_SPEC = gh.ModelSpec("tp-cpu", 2, 128, 64, 192, 4, 2, 32, 4, 97)   # fp32 storage, GQA (G = 2)


def tp_weights(spec, layer, seed=SEED):
    """The synthetic weights of one layer (oracle generator, logical [rows, cols] matrices)."""
    from oracle import randn
    D, Dkv, Dh = spec.d_model, spec.d_kv, spec.d_hidden
    sD, sH = 1.0 / np.sqrt(D), 1.0 / np.sqrt(Dh)
    tid = lambda w: 64 + layer * 16 + w  # noqa: E731  (tid_layer, oracle.c)
    return dict(q=randn(seed, tid(0), 0, D * D, sD).reshape(D, D), k=randn(seed, tid(1), 0, Dkv * D, sD).reshape(Dkv, D),
                v=randn(seed, tid(2), 0, Dkv * D, sD).reshape(Dkv, D), o=randn(seed, tid(3), 0, D * D, sD).reshape(D, D),
                w1=randn(seed, tid(4), 0, Dh * D, sD).reshape(Dh, D), w3=randn(seed, tid(5), 0, Dh * D, sD).reshape(Dh, D),
                w2=randn(seed, tid(6), 0, D * Dh, sH).reshape(D, Dh))


def _rms(x, eps):
    return x / np.sqrt((x.astype(np.float64) ** 2).mean(-1, keepdims=True) + eps).astype(np.float32)


def _rope(m, pos, spec):
    dh = spec.d_head
    i = np.arange(dh // 2)
    ang = pos[:, None].astype(np.float64) * np.power(float(spec.rope_theta), -2.0 * i / dh)[None, :]
    c, s = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
    r = m.reshape(m.shape[0], -1, dh // 2, 2)
    a, e = r[..., 0], r[..., 1]
    return np.stack([a * c[:, None] - e * s[:, None], a * s[:, None] + e * c[:, None]], -1).reshape(m.shape)


def worker_tp(rank, world, port, out_q, B):
    """Tier-1 tensor parallelism at toy scale, the engine's protocol: ranks 0..T-1
    hold head / hidden-unit slices of every layer (numpy), ranks T.. are the K' Tier-2 ranks
    (oracle F2).  Rank r sends the head block [x_r | q_r | k_r | v_r] of each shard's rows; a
    Tier-2 rank assembles the PayloadModel row from the T blocks, attends, and returns block r of
    [x | attn] to rank r.  W_o and W_2 partials are all-reduced across the T ranks (gathered and
    summed in rank order, as the GEMM epilogue does), so every TP rank holds the same x."""
    init_rank(rank, world, port)
    from oracle import Oracle
    spec, T = TP_SPEC, 2
    tp_group = dist.new_group(list(range(T)))
    lay = gh.engine_layout(world, rank, B, spec.n_layers, tier1_tp=T)
    kp = world - T
    off, cnt = gh.shard_plan(B, kp)
    D, Dkv, Dh, H = spec.d_model, spec.d_kv, spec.d_hidden, spec.n_heads
    Dt, Dkvt, Dht = D // T, Dkv // T, Dh // T
    prompts = np.random.default_rng(2).integers(0, spec.vocab_size, size=(B, 2), dtype=np.int32)
    if rank < T:
        r = rank
        assert lay["role"] == "tier1" and lay["tp_rank"] == r and lay["kp"] == kp
        ora = Oracle(spec, seed=SEED, n_slots=1)           # embedding + classifier (whole)
        W = [tp_weights(spec, l) for l in range(spec.n_layers)]
        qs, ks, hs = slice(r * Dt, (r + 1) * Dt), slice(r * Dkvt, (r + 1) * Dkvt), slice(r * Dht, (r + 1) * Dht)

        def allreduce(part):
            parts = [torch.zeros_like(torch.from_numpy(part)) for _ in range(T)]
            dist.all_gather(parts, torch.from_numpy(part), group=tp_group)
            acc = parts[0].numpy().copy()
            for p in parts[1:]:
                acc += p.numpy()
            return acc

        x = np.zeros((B, D), np.float32)
        tok = prompts[:, 0].copy()
        out = []
        for t in range(1 + STEPS):
            pos = np.full(B, t, np.int32)
            if r == 0:
                for j in range(kp):
                    dist.send(torch.from_numpy(pos[off[j]:off[j] + cnt[j]].copy()), dst=T + j)
            ora.embed(tok, x)
            for l in range(spec.n_layers):
                w = W[l]
                xn = _rms(x, spec.norm_eps)
                q = _rope(xn @ w["q"][qs].T, pos, spec)
                k = _rope(xn @ w["k"][ks].T, pos, spec)
                v = xn @ w["v"][ks].T
                blk = np.concatenate([x[:, qs], q, k, v], 1).astype(np.float32)      # [x_r|q_r|k_r|v_r]
                for j in range(kp):
                    dist.send(torch.from_numpy(np.ascontiguousarray(blk[off[j]:off[j] + cnt[j]])), dst=T + j)
                bwd = np.zeros((B, 2 * Dt), np.float32)                                 # [x_r|attn_r]
                for j in range(kp):
                    buf = torch.zeros((cnt[j], 2 * Dt), dtype=torch.float32)
                    dist.recv(buf, src=T + j)
                    bwd[off[j]:off[j] + cnt[j]] = buf.numpy()
                assert np.array_equal(bwd[:, :Dt], x[:, qs])                            # x pass-through
                h = x + allreduce(bwd[:, Dt:] @ w["o"][:, qs].T)
                hn = _rms(h, spec.norm_eps)
                g = hn @ w["w1"][hs].T
                a = g / (1.0 + np.exp(-g)) * (hn @ w["w3"][hs].T)
                x = (h + allreduce(a.astype(np.float32) @ w["w2"][:, hs].T)).astype(np.float32)
            nxt, lg = ora.classify(x)
            if t >= 1:
                out.append((nxt.copy(), lg.copy()))
            tok = prompts[:, 1].copy() if t == 0 else nxt
        out_q.put((r, np.stack([o[0] for o in out], 1), np.stack([o[1] for o in out], 1)))
    else:
        j = rank - T
        n = cnt[j]
        assert lay == dict(role="tier2", span=0, tp_rank=0, shard=j, kp=kp, layers=(0, spec.n_layers),
                           rows=(off[j], n))
        ora = Oracle(spec, seed=SEED, n_slots=n)
        slot = np.arange(n, dtype=np.uint32)
        for t in range(1 + STEPS):
            pos_t = torch.zeros(n, dtype=torch.int32)
            dist.recv(pos_t, src=0)
            pos = pos_t.numpy()
            for l in range(spec.n_layers):
                blks = []
                for r in range(T):
                    buf = torch.zeros((n, (2 * D + 2 * Dkv) // T), dtype=torch.float32)
                    dist.recv(buf, src=r)
                    blks.append(buf.numpy())
                cols = lambda i, w: [b[:, i * w:(i + 1) * w] for b in blks]  # noqa: E731
                xs = np.concatenate([b[:, :Dt] for b in blks], 1)
                qq = np.concatenate([b[:, Dt:2 * Dt] for b in blks], 1)
                kk = np.concatenate([b[:, 2 * Dt:2 * Dt + Dkvt] for b in blks], 1)
                vv = np.concatenate([b[:, 2 * Dt + Dkvt:] for b in blks], 1)
                del cols
                fwd = np.ascontiguousarray(np.concatenate([xs, qq, kk, vv], 1), dtype=np.float32)
                bwd = np.zeros((n, 2 * D), np.float32)
                ora.attend(l, slot, pos, fwd, bwd)
                for r in range(T):
                    blk = np.concatenate([bwd[:, r * Dt:(r + 1) * Dt], bwd[:, D + r * Dt:D + (r + 1) * Dt]], 1)
                    dist.send(torch.from_numpy(np.ascontiguousarray(blk)), dst=r)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(4, 9), (8, 13)])
def test_tier1_tensor_parallel_protocol(world, B):
    """world 8 = BASELINE C5: Tier-1 weights split across 2 ranks, KV across 6.  fp32 storage:
    logits within 1e-4 relative of the colocated oracle (only the summation order differs), tokens
    equal wherever the margin is clear, and both TP ranks decode identical tokens."""
    _, gen, lg = reference_tokens(B, TP_SPEC)
    procs, q = spawn(worker_tp, world, (B,))
    res = dict((r, (g, l)) for r, g, l in collect(procs, q, 2, 240))
    sgen, slg = res[0]
    assert np.array_equal(res[1][0], sgen) and np.array_equal(res[1][1], slg)
    err = np.abs(slg - lg).max()
    assert err <= 1e-4 * np.abs(lg).max(), err
    top2 = np.sort(lg, -1)[..., -2:]
    clear = (top2[..., 1] - top2[..., 0]) > 4 * err
    assert np.array_equal(sgen[clear], gen[clear])


def test_world8_layouts():
    """The engine's rank layout (gh_engine_layout) of BASELINE's 8-GPU configurations: every
    prompt row of a span lives on exactly one Tier-2 rank, shards differ by at most one prompt,
    spans cover every layer once, and the admitted batch is two_tier_context_slots'."""
    GiB = 1 << 30
    c3, c5 = gh.CONFIGS["C3"]["spec"], gh.CONFIGS["C5"]["spec"]
    cases = [  # (spec, ctx, tier1_ranks, tier1_tp, expected K', admitted slots)
        (c3, 2048, 1, 1, 7, 1190),     # C3: Tier-1 + 7 Tier-2
        (c5, 8192, 2, 1, 3, None),     # C5 as pipeline spans: 2 x (1 + 3)
        (c5, 8192, 1, 2, 6, 408),      # C5 as TP: Tier-1 over 2, KV over 6 (BASELINE configs[4])
    ]
    for spec, ctx, n1, tp, kp, slots in cases:
        adm = gh.two_tier_context_slots(spec, n1, kp, 179 * GiB, ctx)
        if slots is not None:
            assert adm == slots
        batch = adm // 2  # two in-flight batches
        lays = [gh.engine_layout(8, r, batch, spec.n_layers, tier1_ranks=n1, tier1_tp=tp) for r in range(8)]
        t1 = [L for L in lays if L["role"] == "tier1"]
        t2 = [L for L in lays if L["role"] == "tier2"]
        assert len(t1) == max(n1, tp) and len(t2) == 8 - len(t1)
        assert all(L["kp"] == kp for L in lays)
        if tp > 1:
            assert [L["tp_rank"] for L in t1] == list(range(tp))
            assert all(L["layers"] == (0, spec.n_layers) for L in lays)
        else:
            assert sorted(L["layers"] for L in t1) == [(0, 40), (40, 80)] if n1 == 2 else True
        for sp in range(n1):
            rows = sorted(L["rows"] for L in t2 if L["span"] == sp)
            assert rows[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(rows, rows[1:]))
            assert rows[-1][0] + rows[-1][1] == batch
            assert max(c for _, c in rows) - min(c for _, c in rows) <= 1
    with pytest.raises(gh.ValidationError):
        gh.engine_layout(8, 0, 100, 80, tier1_ranks=3)   # 8 - 3 not a multiple of 3 spans
    with pytest.raises(gh.UnsupportedError):
        gh.engine_layout(8, 0, 100, 80, tier1_ranks=2, tier1_tp=2)
