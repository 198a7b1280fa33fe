"""Multi-GPU batch sharding for the NTT engine.

Polynomials are independent, so a batch is split into contiguous per-rank ranges with
no collective on the compute path: rank r transforms polys [start, stop) on its own GPU
(one process per GPU, torchrun).  A collective is used only when the caller asks for the
results on one rank (``gather``): NCCL all_gather on GPUs, gloo on CPU tensors.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split: the first total % world ranks get one extra item."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("shard_range: need 0 <= rank < world and total >= 0")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


@dataclass
class Sharder:
    rank: int = 0
    world: int = 1
    group: Optional[object] = None

    @classmethod
    def from_env(cls, group=None) -> "Sharder":
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(group), dist.get_world_size(group), group)
        return cls()

    def local(self, total: int) -> tuple[int, int]:
        return shard_range(total, self.rank, self.world)

    def run(self, fn: Callable, batch):
        """Apply fn to this rank's slice of a (total, N) tensor/array; returns the local result."""
        lo, hi = self.local(batch.shape[0])
        return fn(batch[lo:hi])

    def gather(self, local, total: int):
        """All ranks' local results concatenated in rank order (every rank gets the full
        tensor).  Uneven shards are padded to the largest shard for the collective."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return local
        sizes = [shard_range(total, r, self.world) for r in range(self.world)]
        rows = max(hi - lo for lo, hi in sizes)
        pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)
