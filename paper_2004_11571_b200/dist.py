"""Multi-GPU point-range sharding (PAPER.md:557-573 HM16 "N evaluations at a
time", in its contiguous-range form).

Every rank holds the full, replicated term set (its own ``Context``), evaluates a contiguous
block of the T points -- seeding a_i at its own first point by exponentiation inside k_step --
and the only collective is one gather of the G x T_r output blocks to the root over NCCL.
Term sharding (MT18's 1D decomposition) is not used: it would need a
*modular* all-reduce, which NCCL's wrapping uint64 sum cannot do exactly.

``eval_sharded`` is device-agnostic plumbing: ``eval_local(j_first, T_r, out_view)`` fills a
``[G, T_r]`` int64 tensor (the CUDA path on GPUs; the tests inject the CPU oracle under gloo).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(T: int, world: int, rank: int) -> tuple[int, int]:
    """Columns [off, off+cnt) of rank ``rank``: ceil split, trailing ranks may be short/empty."""
    per = -(-T // world) if T else 0
    off = min(rank * per, T)
    return off, max(0, min(per, T - off))


def shard_width(T: int, world: int) -> int:
    return -(-T // world) if T else 0


class ShardedEval:
    """Buffers for one (G, T, world) shape; reused across steps."""

    def __init__(self, G: int, T: int, device, group=None, root: int = 0):
        self.G, self.T, self.root, self.group = G, T, root, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.Tr = shard_width(T, self.world)
        self.off, self.cnt = shard_range(T, self.world, self.rank)
        self.is_root = self.rank == root
        self.out = torch.empty((G, T), dtype=torch.int64, device=device) if self.is_root else None
        # one rank: evaluate straight into the result
        self.local = self.out if self.world == 1 else torch.zeros((G, self.Tr), dtype=torch.int64, device=device)
        self.gathered = (torch.empty((self.world, G, self.Tr), dtype=torch.int64, device=device)
                         if self.is_root and self.world > 1 else None)

    def run(self, eval_local, j0: int, gather: bool = True):
        """One step: local evaluation of this rank's points, then the gather to the root.
        Returns the [G, T] result on the root (None elsewhere)."""
        if self.cnt:
            eval_local(j0 + self.off, self.cnt, self.local)
        if self.world == 1:
            return self.out
        if not gather:
            return None
        dist.gather(self.local, [t for t in self.gathered] if self.is_root else None, dst=self.root,
                    group=self.group)
        if not self.is_root:
            return None
        for r in range(self.world):                     # [P][G][T_r] -> [G][T]
            off, cnt = shard_range(self.T, self.world, r)
            if cnt:
                self.out[:, off: off + cnt].copy_(self.gathered[r, :, :cnt])
        return self.out
