"""Data-parallel plumbing for the TTT attention unroll.

Sequences are independent, so the attention itself needs no communication:
each rank runs its own sequences (weak scaling). The one real exchange of
draft training is the all-reduce of the draft layer's parameter gradients
(ZeRO-2 moves the same bytes as one all-reduce). This
module owns that exchange and the multi-rank timing rule; the NCCL process
group (one process per GPU, torchrun) carries it over NVLink / NVSwitch.
Host logic is backend-agnostic so tests run it on CPU with gloo.
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist


def shard_sequences(global_batch: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of sequences owned by `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def micro_batches(global_batch: int, micro: int, world: int, rank: int) -> List[Tuple[int, int]]:
    """The sequence ranges [lo, hi) of `rank`'s micro-batches for one optimizer step: its
    contiguous shard of the global batch (shard_sequences) cut into chunks of `micro` sequences
    (BASELINE configs[4]: global batch 64 at 1/2/4/8 GPUs, micro-batches of 8 -> 64/N per rank)."""
    if micro < 1:
        raise ValueError("micro-batch size must be >= 1")
    lo, hi = shard_sequences(global_batch, world, rank)
    return [(a, min(a + micro, hi)) for a in range(lo, hi, micro)]


class GradBuckets:
    """A flat draft-layer gradient buffer split into `n` buckets.

    The draft layer's parameters are shared by every TTT step and every micro-batch of an
    optimizer step, so a parameter gradient is final only after the LAST micro-batch's step-0
    backward. `release_all()` is therefore called once per optimizer step, after that backward:
    it starts the asynchronous all-reduces of the buckets in reverse parameter order (the order
    a layer-by-layer backward would finish them); `finish()` waits for all of them and applies
    the 1/world average. On NCCL the collectives run on NCCL's stream ordered after the current
    stream's work at release time. `release(i)` (one bucket) stays for finer-grained callers.
    """

    def __init__(self, numel: int, n: int, dtype=torch.bfloat16, device="cpu", group=None):
        self.flat = torch.zeros(numel, dtype=dtype, device=device)
        self.buckets: List[torch.Tensor] = list(torch.chunk(self.flat, n))
        self.group = group
        self.works = []

    def release(self, i: int) -> None:
        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return
        self.works.append(dist.all_reduce(self.buckets[i], op=dist.ReduceOp.SUM, group=self.group,
                                          async_op=True))

    def release_all(self) -> None:
        """Once per optimizer step, after the last micro-batch's full backward (see class doc)."""
        for i in reversed(range(len(self.buckets))):
            self.release(i)

    def finish(self) -> None:
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        while self.works:
            self.works.pop(0).wait()
        if world > 1:
            self.flat.mul_(1.0 / world)

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * self.flat.element_size()


class OptimizerStep:
    """One data-parallel optimizer step of draft training (BASELINE configs[4]):
    the rank runs its micro-batches (micro_batches(): 64/N sequences per rank as chunks of 8),
    each adding its draft-parameter gradients into `buckets.flat` (gradient accumulation, no
    communication), then ONE exchange — `buckets.release_all()` after the last micro-batch's
    backward, `finish()` — and, for ZeRO-2 buckets, the post-update parameter all-gather.
    `micro_step(m, lo, hi)` runs micro-batch m over sequences [lo, hi)."""

    def __init__(self, buckets: "GradBuckets", global_batch: int, micro: int, world: int, rank: int,
                 params_flat: torch.Tensor = None):
        self.buckets = buckets
        self.micro = micro_batches(global_batch, micro, world, rank)
        self.params_flat = params_flat
        self.exchanges = 0

    def run(self, micro_step) -> None:
        for m, (lo, hi) in enumerate(self.micro):
            micro_step(m, lo, hi)
        self.buckets.release_all()
        self.buckets.finish()
        if self.params_flat is not None and isinstance(self.buckets, Zero2Buckets):
            self.buckets.gather_params(self.params_flat)
        self.exchanges += 1


def exchange_grads(model: torch.nn.Module, buckets: "GradBuckets") -> None:
    """The draft's real parameter gradients through the exchange: flatten them (parameter order) into
    `buckets.flat`, reduce (release_all + finish: the bucketed all-reduce averages in place; ZeRO-2
    reduce-scatters into the owned shards), and for the all-reduce form write the averaged values
    back into the parameters' .grad. Called once per optimizer step after the last micro-batch."""
    params = [p for p in model.parameters() if p.grad is not None]
    n = sum(p.numel() for p in params)
    if n > buckets.flat.numel():
        raise ValueError("gradient buffer too small for the model")
    torch.cat([p.grad.reshape(-1).to(buckets.flat.dtype) for p in params], out=buckets.flat[:n])
    buckets.release_all()
    buckets.finish()
    if not isinstance(buckets, Zero2Buckets):
        off = 0
        for p in params:
            p.grad.copy_(buckets.flat[off:off + p.numel()].view_as(p.grad))
            off += p.numel()


def max_over_ranks(x: float, device="cpu", group=None) -> float:
    """The multi-GPU timing rule: a step takes as long as its slowest rank."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


# ---- head-parallel long context --------------------------------------
# A B = 1 sequence of L >= 16K cannot be split by sequence without an exchange inside the attention.
# Split by kv-head group instead (Ulysses-style): the projections produce sequence shards
# [L/N, H, D] per rank; one all-to-all turns them into head shards [L, H/N, D] (every query row,
# a contiguous block of H/N heads — with Hkv % N == 0 a GQA group never straddles ranks), the TTT
# attention runs locally on (Hq/N, Hkv/N) heads with no communication, and the inverse all-to-all
# returns out / dq / dk / dv to sequence shards.

def seq_to_head(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[L/N, H, D] sequence shard (rank r holds rows r L/N ..) -> [L, H/N, D] head shard (rank r
    holds heads r H/N ..). Collective over `group` (all ranks call it)."""
    Ls, H, D = x.shape
    if H % world:
        raise ValueError("heads must divide by the world size")
    send = x.reshape(Ls, world, H // world, D).permute(1, 0, 2, 3).contiguous()  # [dest rank][rows][h][d]
    if world == 1:
        return send.reshape(Ls, H, D)
    recv = torch.empty_like(send)  # [source rank = row block][rows][h][d]
    dist.all_to_all_single(recv, send, group=group)
    return recv.reshape(world * Ls, H // world, D)


def head_to_seq(y: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Inverse of seq_to_head: [L, H/N, D] head shard -> [L/N, H, D] sequence shard."""
    L, Hs, D = y.shape
    if L % world:
        raise ValueError("rows must divide by the world size")
    send = y.reshape(world, L // world, Hs, D).contiguous()  # [dest rank = row block][rows][h][d]
    if world == 1:
        return send.reshape(L, Hs, D)
    recv = torch.empty_like(send)  # [source rank = head block][rows][h][d]
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 0, 2, 3).reshape(L // world, world * Hs, D)


class Zero2Buckets(GradBuckets):
    """ZeRO-2 form of the draft gradient exchange (the draft model uses ZeRO-2,
    gradient and optimizer-state sharding): `release(i)` reduce-scatters bucket i (each rank keeps
    the averaged 1/N shard it owns — what its optimizer shard updates), and `gather_params()` is
    the post-update all-gather of those shards into the full replicated buffer. Per step this moves
    the bytes of one all-reduce, split around the optimizer step. Buckets are padded to a multiple
    of the world size."""

    def __init__(self, numel: int, n: int, dtype=torch.bfloat16, device="cpu", group=None):
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        per = -(-numel // n)                      # ceil: elements per bucket
        per = -(-per // world) * world            # padded to a multiple of the world size
        self.world = world
        self.flat = torch.zeros(per * n, dtype=dtype, device=device)
        self.buckets = list(torch.chunk(self.flat, n))
        self.shards = [torch.empty(per // world, dtype=dtype, device=device) for _ in range(n)]
        self.group = group
        self.works = []

    def release(self, i: int) -> None:
        if self.world == 1:
            self.shards[i].copy_(self.buckets[i])
            return
        self.works.append(dist.reduce_scatter_tensor(self.shards[i], self.buckets[i], op=dist.ReduceOp.SUM,
                                                     group=self.group, async_op=True))

    def finish(self) -> None:
        while self.works:
            self.works.pop(0).wait()
        if self.world > 1:
            for s in self.shards:
                s.mul_(1.0 / self.world)

    def gather_params(self, params_flat: torch.Tensor) -> None:
        """All-gather the per-rank shards of `params_flat` (same bucketing as the gradients)."""
        if self.world == 1:
            return
        n = len(self.buckets)
        chunks = list(torch.chunk(params_flat, n))
        rank = dist.get_rank(self.group)
        works = []
        for c in chunks:
            per = c.numel() // self.world
            mine = c[rank * per:(rank + 1) * per].clone()
            works.append(dist.all_gather_into_tensor(c, mine, group=self.group, async_op=True))
        for w in works:
            w.wait()
