"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic
used by bench.py at N > 1: sequence sharding, bucketed gradient all-reduce with
averaging, and the max-over-ranks timing rule."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18567_b200.dp import GradBuckets, max_over_ranks, shard_sequences


def test_shard_sequences_partition():
    for gb in (1, 7, 8, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_sequences(gb, world, r)
                assert hi - lo in (gb // world, gb // world + 1)
                seen += list(range(lo, hi))
            assert seen == list(range(gb))
    with pytest.raises(ValueError):
        shard_sequences(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gb = GradBuckets(1001, 7, dtype=torch.float32)
        # rank-dependent pattern: element e of rank r = (r + 1) * e
        gb.flat.copy_(torch.arange(1001, dtype=torch.float32) * (rank + 1))
        for i in reversed(range(7)):  # released in backward order
            gb.release(i)
        gb.finish()
        want = torch.arange(1001, dtype=torch.float32) * sum(r + 1 for r in range(world)) / world
        ok_avg = torch.allclose(gb.flat, want)
        t = max_over_ranks(10.0 + rank)
        q.put((rank, ok_avg, t, shard_sequences(64, world, rank)))
    finally:
        dist.destroy_process_group()


def test_grad_buckets_allreduce_and_max_timing_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, ok_avg, t, shard in res:
        assert ok_avg, f"rank {rank}: bucketed all-reduce average wrong"
        assert t == 11.0, "max over ranks"
    assert res[0][3] == (0, 32) and res[1][3] == (32, 64)


def _a2a_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_18567_b200.dp import head_to_seq, seq_to_head
        L, H, D = 12, 8, 5
        full = torch.arange(L * H * D, dtype=torch.float32).reshape(L, H, D)  # known to every rank
        Ls, Hs = L // world, H // world
        shard = full[rank * Ls:(rank + 1) * Ls].clone()
        heads = seq_to_head(shard, world)
        ok_fwd = torch.equal(heads, full[:, rank * Hs:(rank + 1) * Hs])
        back = head_to_seq(heads * 2.0, world)
        ok_inv = torch.equal(back, shard * 2.0)
        q.put((rank, ok_fwd, ok_inv))
    finally:
        dist.destroy_process_group()


def test_head_parallel_all_to_all_world2():
    """Ulysses-style exchange for head-parallel long context (dp.seq_to_head / head_to_seq):
    rank r ends with every row of heads [r H/N, (r+1) H/N), and the inverse restores the shard."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_fwd, ok_inv in res:
        assert ok_fwd, f"rank {rank}: seq_to_head wrong"
        assert ok_inv, f"rank {rank}: head_to_seq wrong"


def test_head_parallel_single_rank_identity():
    from paper_2603_18567_b200.dp import head_to_seq, seq_to_head
    x = torch.randn(6, 4, 3)
    assert torch.equal(seq_to_head(x, 1), x) and torch.equal(head_to_seq(x, 1), x)


def _zero2_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_18567_b200.dp import Zero2Buckets
        zb = Zero2Buckets(1000, 3, dtype=torch.float32)
        n = zb.flat.numel()
        zb.flat.copy_(torch.arange(n, dtype=torch.float32) * (rank + 1))
        for i in reversed(range(3)):
            zb.release(i)
        zb.finish()
        avg = torch.arange(n, dtype=torch.float32) * sum(r + 1 for r in range(world)) / world
        ok_rs = True
        for i, (b, s) in enumerate(zip(torch.chunk(avg, 3), zb.shards)):
            per = s.numel()
            ok_rs &= torch.allclose(s, b[rank * per:(rank + 1) * per])
        params = torch.zeros(n)
        for i, c in enumerate(torch.chunk(params, 3)):   # each rank fills only its own shard
            per = c.numel() // world
            c[rank * per:(rank + 1) * per] = 100.0 * (rank + 1) + i
        zb.gather_params(params)
        want = torch.cat([torch.cat([torch.full((c.numel() // world,), 100.0 * (r + 1) + i) for r in range(world)])
                          for i, c in enumerate(torch.chunk(torch.zeros(n), 3))])
        q.put((rank, ok_rs, bool(torch.equal(params, want))))
    finally:
        dist.destroy_process_group()


def test_zero2_reduce_scatter_and_param_all_gather_world2():
    """ZeRO-2 exchange: each rank gets the averaged shard it owns; the all-gather
    re-replicates the updated parameter shards."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_zero2_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_rs, ok_ag in res:
        assert ok_rs, f"rank {rank}: reduce-scatter shard wrong"
        assert ok_ag, f"rank {rank}: param all-gather wrong"
