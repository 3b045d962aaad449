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


class GradBuckets:
    """A flat draft-layer gradient buffer split into `n` buckets.

    `release(i)` starts an asynchronous all-reduce of bucket i (issued right
    after the backward call that finalises it, so it overlaps the remaining
    backward calls on the communication stream); `finish()` waits for all of
    them and applies the 1/world average. On NCCL the collective runs on its own
    stream ordered after the current stream's work at release time.
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

    def finish(self) -> None:
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        while self.works:
            self.works.pop(0).wait()
        if world > 1:
            self.flat.mul_(1.0 / world)

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * self.flat.element_size()


def max_over_ranks(x: float, device="cpu", group=None) -> float:
    """The multi-GPU timing rule: a step takes as long as its slowest rank."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
