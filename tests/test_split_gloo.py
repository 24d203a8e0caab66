"""Tier-split protocol on CPU (gloo, world sizes 2 and 3): rank 0 plays Tier-1, ranks 1.. play
Tier-2 over their prompt shard, exchanging exactly the per-layer PayloadModel messages the GPU
engine sends over NCCL (fwd [x|q|k|v] per shard, bwd [x|attn] per shard, plus the positions at
the start of a step), with the oracle as the stage implementation.  The result must equal the
colocated oracle bit for bit (same arithmetic, same message bytes)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2501_11779_b200 as gh

SPEC = gh.ModelSpec("split-cpu", 2, 128, 64, 192, 4, 2, 32, 2, 97)
B, STEPS, SEED = 7, 5, 1234


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def reference_tokens():
    from oracle import Oracle
    ora = Oracle(SPEC, seed=SEED, n_slots=B)
    prompts = np.random.default_rng(2).integers(0, SPEC.vocab_size, size=(B, 2), dtype=np.int32)
    gen, lg = ora.generate(prompts, STEPS)
    return prompts, gen, lg


def worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
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


@pytest.mark.parametrize("world", [2, 3])
def test_tier_split_protocol_matches_colocated(world):
    _, gen, lg = reference_tokens()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    sgen, slg = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(sgen, gen)
    assert np.array_equal(slg, lg)


def worker_pp(rank, world, port, out_q):
    """Tier-1 pipeline stages (SURVEY 8e, config 5 at toy scale): ranks 0/1 are Tier-1 spans of
    layer_spans(N, 2), ranks 2/3 each the single Tier-2 rank of span 0/1 (its layers' KV). Span 0
    embeds, hands [x] (PayloadModel intra-Tier-1 message, netmodel.cpp:22) plus the positions to
    span 1; span 1 classifies and hands the next tokens back to span 0."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    n1 = 2
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
            dist.send(torch.from_numpy(pos.copy()), dst=n1 + sp)      # positions to my Tier-2
            for layer in range(lo[sp], lo[sp] + spans[sp]):
                ora.pre(layer, x, pos, fwd)
                dist.send(torch.from_numpy(fwd.view(np.int16).copy()), dst=n1 + sp)
                buf = torch.zeros((B, 2 * D), dtype=torch.int16)
                dist.recv(buf, src=n1 + sp)
                bwd[:] = buf.numpy().view(np.uint16)
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
        sp = rank - n1
        ora = Oracle(SPEC, seed=SEED, n_slots=B)        # this span's layers of every prompt
        slot = np.arange(B, dtype=np.uint32)
        for t in range(1 + STEPS):
            pos_t = torch.zeros(B, dtype=torch.int32)
            dist.recv(pos_t, src=sp)
            pos = pos_t.numpy()
            for layer in range(lo[sp], lo[sp] + spans[sp]):
                buf = torch.zeros((B, 2 * D + 2 * Dkv), dtype=torch.int16)
                dist.recv(buf, src=sp)
                fwd = buf.numpy().view(np.uint16).copy()
                bwd = np.zeros((B, 2 * D), np.uint16)
                ora.attend(layer, slot, pos, fwd, bwd)
                dist.send(torch.from_numpy(bwd.view(np.int16).copy()), dst=sp)
    dist.barrier()
    dist.destroy_process_group()


def test_tier1_pipeline_protocol_matches_colocated():
    _, gen, lg = reference_tokens()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker_pp, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    sgen, slg = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(sgen, gen)
    assert np.array_equal(slg, lg)


def test_shard_plan_balanced():
    for batch, kp in ((1024, 7), (7, 3), (170, 1), (1190, 7)):
        off, cnt = gh.shard_plan(batch, kp)
        assert sum(cnt) == batch and max(cnt) - min(cnt) <= 1
        assert off == [sum(cnt[:j]) for j in range(kp)]
    with pytest.raises(gh.ValidationError):
        gh.shard_plan(2, 3)
