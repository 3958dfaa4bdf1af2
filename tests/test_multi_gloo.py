"""World-size-2 host-side test of the doc-partitioned multi-GPU protocol on CPU (gloo).

Each rank owns a contiguous, token-balanced document range (lda.partition_docs, the
partition of P:1137-1140) with its global token base; every iteration the ranks sum their
local W counts (the per-iteration merge of P:1145, NCCL all-reduce on the GPUs, gloo here)
and sample against the merged snapshot.  The concatenated topics must equal the
single-process chain bit for bit.  The per-rank compute is the CPU oracle (test harness),
so this exercises the partition, token bases and the exchange protocol, not the kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_08725_b200.lda import partition_docs
from paper_2007_08725_b200.synth import SAMPLER_SEED, planted_corpus_np

N_DOCS, V, K, ITERS = 120, 400, 12, 4


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out, branches=3):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle

    w, d = planted_corpus_np(N_DOCS, V, 80.0, 0.5, seed=11)
    L = np.bincount(d, minlength=N_DOCS)
    bounds = partition_docs(L, world)
    cum = np.concatenate([[0], np.cumsum(L)])
    t0, t1 = int(cum[bounds[rank]]), int(cum[bounds[rank + 1]])
    shard = oracle.OracleLDA(w[t0:t1], d[t0:t1] - bounds[rank], bounds[rank + 1] - bounds[rank], V, K,
                             seed=SAMPLER_SEED, token_base=t0, branches=branches)
    for _ in range(ITERS):
        Wl = torch.from_numpy(shard.counts()[1].astype(np.int64))
        dist.all_reduce(Wl, op=dist.ReduceOp.SUM)  # the per-iteration W merge
        Wg = Wl.numpy().astype(np.int32)
        shard.iterate(1, Wg, Wg.sum(0).astype(np.int32))
    z = torch.from_numpy(shard.topics().astype(np.int64))
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(z)]))
    mx = int(max(s.item() for s in sizes))
    pad = torch.full((mx,), -1, dtype=torch.int64)
    pad[: len(z)] = z
    parts = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, pad)
    if rank == 0:
        allz = np.concatenate([p[: int(s.item())].numpy() for p, s in zip(parts, sizes)])
        np.save(out, allz)
    dist.destroy_process_group()


def test_partition_docs_balanced():
    L = np.random.default_rng(0).integers(1, 500, size=1000)
    for P in (1, 2, 3, 8):
        b = partition_docs(L, P)
        assert b[0] == 0 and b[-1] == len(L) and all(x <= y for x, y in zip(b, b[1:]))
        tok = [L[b[i]:b[i + 1]].sum() for i in range(P)]
        assert max(tok) - min(tok) <= 2 * L.max()


@pytest.mark.parametrize("branches", [3, 2])
def test_two_rank_gloo_equals_single(tmp_path, branches):
    """Doc shards + a summed W every iteration reproduce the single chain bit for bit, for the
    three-branch sampler and the two-branch (ESCA) mode alike."""
    from oracle import oracle

    oracle.build()
    out = str(tmp_path / "z.npy")
    mp.spawn(worker, args=(2, free_port(), out, branches), nprocs=2, join=True)
    w, d = planted_corpus_np(N_DOCS, V, 80.0, 0.5, seed=11)
    ref = oracle.OracleLDA(w, d, N_DOCS, V, K, seed=SAMPLER_SEED, branches=branches)
    ref.iterate(ITERS)
    assert np.array_equal(np.load(out), ref.topics().astype(np.int64))


def pack_delta(delta, b):
    """The library's k_wdelta_pack on the host: int deltas -> u32 pairs (delta + b) | (delta' + b) << 16
    (as int64 tensors: gloo has no u32 sum; every sum stays below 2^32)."""
    flat = delta.ravel().astype(np.int64)
    if len(flat) % 2:
        flat = np.concatenate([flat, [0]])
    return torch.from_numpy((flat[0::2] + b) | ((flat[1::2] + b) << 16))


def unpack_sum(psum, n, world, b):
    """k_wdelta_apply's decoding: the per-field sums minus world * b, first n entries."""
    v = psum.numpy()
    out = np.empty(2 * len(v), np.int64)
    out[0::2] = (v & 0xFFFF) - world * b
    out[1::2] = (v >> 16) - world * b
    return out[:n]


def worker_hybrid(rank, world, port, out, delta=False):
    """The library's H7 protocol on CPU: global word counts decide the dense set
    (c_v > K); per iteration the dense block [V_d x K] and n_k are all-reduced (sum), and the
    tail words' topics are all-gathered in word-major order (padded to the largest rank's
    tail-token count, static per-rank offsets exchanged once) and every rank rebuilds the
    global tail rows from them.  The per-rank chain is the CPU oracle fed the merged W."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle

    w, d = planted_corpus_np(N_DOCS, V, 80.0, 0.5, seed=11)
    L = np.bincount(d, minlength=N_DOCS)
    bounds = partition_docs(L, world)
    cum = np.concatenate([[0], np.cumsum(L)])
    t0, t1 = int(cum[bounds[rank]]), int(cum[bounds[rank + 1]])
    ws, ds = w[t0:t1], d[t0:t1] - bounds[rank]
    shard = oracle.OracleLDA(ws, ds, bounds[rank + 1] - bounds[rank], V, K, seed=SAMPLER_SEED, token_base=t0)
    # create: global counts -> dense set; static per-rank tail layout
    cnt = torch.from_numpy(np.bincount(ws, minlength=V).astype(np.int64))
    dist.all_reduce(cnt)
    dense = cnt.numpy() > K
    tail_words = np.nonzero(~dense)[0]
    local_tail_tok = np.nonzero(~dense[ws])[0]
    local_tail_tok = local_tail_tok[np.argsort(ws[local_tail_tok], kind="stable")]  # word-major
    n_loc = torch.tensor([len(local_tail_tok)])
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, n_loc)
    tail_max = int(max(s.item() for s in sizes))
    b = 32768 // world
    loc_prev = glob_prev = None
    n_delta = 0
    for _ in range(ITERS):
        z = shard.topics()
        Wl = shard.counts()[1].astype(np.int64)
        Wd = torch.from_numpy(Wl[dense].copy())
        nk = torch.from_numpy(Wl.sum(0))
        if delta and loc_prev is not None:
            # packed 16-bit deltas against the previous exchange (exchange_w): one flag
            # all-reduce decides, then the u32-pair sum rebuilds the global block
            dl = Wl[dense] - loc_prev
            over = torch.tensor([int(np.any(np.abs(dl) >= b))])
            dist.all_reduce(over)
            full = Wd.clone()
            dist.all_reduce(full)  # (check only: the int32 path's result)
            if int(over.item()) == 0:
                ps = pack_delta(dl, b)
                dist.all_reduce(ps)
                rebuilt = glob_prev + unpack_sum(ps, dl.size, world, b).reshape(dl.shape)
                assert np.array_equal(rebuilt, full.numpy())
                n_delta += 1
            Wd = full
        else:
            dist.all_reduce(Wd)
        loc_prev = Wl[dense].copy()
        glob_prev = Wd.numpy().copy()
        dist.all_reduce(nk)
        tz = torch.full((tail_max, 2), -1, dtype=torch.int64)  # (word, topic) of each tail token
        tz[: len(local_tail_tok), 0] = torch.from_numpy(ws[local_tail_tok].astype(np.int64))
        tz[: len(local_tail_tok), 1] = torch.from_numpy(z[local_tail_tok].astype(np.int64))
        parts = [torch.zeros_like(tz) for _ in range(world)]
        dist.all_gather(parts, tz)
        allt = torch.cat(parts).numpy()
        allt = allt[allt[:, 0] >= 0]
        Wg = np.zeros((V, K), np.int64)
        Wg[dense] = Wd.numpy()
        np.add.at(Wg, (allt[:, 0], allt[:, 1]), 1)  # the rebuilt global tail rows
        assert np.array_equal(Wg.sum(0), nk.numpy())
        assert np.all(Wg[tail_words].sum(1) == cnt.numpy()[tail_words])
        shard.iterate(1, Wg.astype(np.int32), nk.numpy().astype(np.int32))
    zt = torch.from_numpy(shard.topics().astype(np.int64))
    mx = int(max(s for s in [len(w)]))
    pad = torch.full((mx,), -1, dtype=torch.int64)
    pad[: len(zt)] = zt
    allp = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allp, pad)
    if delta:
        assert n_delta >= 1, "the delta path was never taken"
    if rank == 0:
        np.save(out, np.concatenate([p[p >= 0].numpy() for p in allp]))
    dist.destroy_process_group()


@pytest.mark.parametrize("delta", [False, True])
def test_two_rank_gloo_hybrid_exchange_equals_single(tmp_path, delta):
    """Dense-block all-reduce (int32 counts, or packed 16-bit deltas against the previous
    exchange whose decoded sum must equal the int32 one) + tail-topic all-gather (the H7
    protocol of the library) equals the single chain bit for bit."""
    from oracle import oracle

    oracle.build()
    out = str(tmp_path / "z.npy")
    mp.spawn(worker_hybrid, args=(2, free_port(), out, delta), nprocs=2, join=True)
    w, d = planted_corpus_np(N_DOCS, V, 80.0, 0.5, seed=11)
    ref = oracle.OracleLDA(w, d, N_DOCS, V, K, seed=SAMPLER_SEED)
    ref.iterate(ITERS)
    assert np.array_equal(np.load(out), ref.topics().astype(np.int64))
