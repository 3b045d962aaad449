"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic
used by bench.py at N > 1: sequence sharding, bucketed gradient all-reduce with
averaging, and the max-over-ranks timing rule."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18567_b200.dp import (GradBuckets, OptimizerStep, Zero2Buckets, exchange_grads, max_over_ranks,
                                      micro_batches, shard_sequences)


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


def test_micro_batches_cover_global_batch():
    """BASELINE configs[4]: global batch 64, micro-batches of 8 -> 64/N sequences per rank."""
    for world in (1, 2, 4, 8):
        allseq = []
        for r in range(world):
            mb = micro_batches(64, 8, world, r)
            assert len(mb) == 8 // world
            assert all(hi - lo == 8 for lo, hi in mb)
            allseq += [s for lo, hi in mb for s in range(lo, hi)]
        assert allseq == list(range(64))
    assert micro_batches(10, 4, 1, 0) == [(0, 4), (4, 8), (8, 10)]


def _opt_worker(rank, world, port, q, zero2):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, nb = 1000, 7
        Buckets = Zero2Buckets if zero2 else GradBuckets
        gb = Buckets(n, nb, dtype=torch.float64)
        calls = {"all_reduce": 0, "reduce_scatter": 0}
        orig_ar, orig_rs = dist.all_reduce, dist.reduce_scatter_tensor

        def ar(*a, **k):
            calls["all_reduce"] += 1
            return orig_ar(*a, **k)

        def rs(*a, **k):
            calls["reduce_scatter"] += 1
            return orig_rs(*a, **k)
        dist.all_reduce, dist.reduce_scatter_tensor = ar, rs
        seen = []
        e = torch.arange(gb.flat.numel(), dtype=torch.float64)

        def micro_step(m, lo, hi):
            # gradient accumulation: sequence s contributes (s + 1) * e to every parameter gradient
            assert sum(calls.values()) == 0, "no exchange before the last micro-batch's backward"
            seen.extend(range(lo, hi))
            gb.flat.add_(e * sum(s + 1 for s in range(lo, hi)))
        step = OptimizerStep(gb, 64, 8, world, rank)
        step.run(micro_step)
        dist.all_reduce, dist.reduce_scatter_tensor = orig_ar, orig_rs
        want = e * sum(s + 1 for s in range(64)) / world  # the mean over ranks of the summed gradients
        if zero2:
            per = gb.flat.numel() // nb // world
            ok = all(torch.allclose(gb.shards[i], want[i * per * world + rank * per:i * per * world + (rank + 1) * per])
                     for i in range(nb))
        else:
            ok = torch.allclose(gb.flat, want)
        q.put((rank, ok, step.exchanges, dict(calls), seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("zero2", [False, True])
def test_optimizer_step_one_exchange_after_micro_batches_world2(zero2):
    """One optimizer step at N = 2: 4 micro-batches of 8 sequences per rank, gradients accumulated
    locally, then exactly one exchange (n_buckets collectives) after the last micro-batch."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_opt_worker, args=(r, world, port, q, zero2)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    seen_all = []
    for rank, ok, nex, calls, seen in res:
        assert ok, f"rank {rank}: averaged gradients wrong"
        assert nex == 1
        assert calls["reduce_scatter" if zero2 else "all_reduce"] == 7
        seen_all += seen
    assert sorted(seen_all) == list(range(64))


def _model_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.manual_seed(0)  # identical initial parameters on every rank
        model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.SiLU(), torch.nn.Linear(32, 8)).double()
        g = torch.Generator().manual_seed(100 + rank)  # different data per rank
        x = torch.randn(64, 16, generator=g, dtype=torch.float64)
        model(x).pow(2).mean().backward()
        local = [p.grad.clone() for p in model.parameters()]
        n = sum(p.numel() for p in model.parameters())
        exchange_grads(model, GradBuckets(n, 3, dtype=torch.float64))
        # numpy copies pickle by value (a tensor would travel through a shared-memory file that can
        # vanish when this process exits before the parent reads the queue)
        q.put((rank, [t.numpy() for t in local], [p.grad.detach().clone().numpy() for p in model.parameters()]))
    finally:
        dist.destroy_process_group()


def test_exchange_real_model_grads_world2():
    """Real parameter gradients (a small MLP's backward on per-rank data) through the bucketed
    all-reduce: every rank ends with the mean of the ranks' local gradients."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_model_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    mean = [(torch.from_numpy(a) + torch.from_numpy(b)) / 2 for a, b in zip(res[0][1], res[1][1])]
    for rank, _, got in res:
        for g, m in zip(got, mean):
            assert torch.allclose(torch.from_numpy(g), m, atol=1e-12), rank
