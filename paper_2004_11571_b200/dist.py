"""Multi-GPU point-range sharding (PAPER.md:557-573 HM16 "N evaluations at a
time", in its contiguous-range form).

Every rank holds the full, replicated term set (its own ``Context``), evaluates a contiguous
block of the T points -- seeding a_i at its own first point by exponentiation inside k_step --
and the only collective is one gather of the G x T_r output blocks to the root over NCCL.
Arbitrary term sharding (MT18's 1D decomposition) would need a *modular*
all-reduce, which NCCL's wrapping uint64 sum cannot do exactly; the bucket-contiguous term
ranges of ``TermShardedEval`` (below, used by the tensor-core path) avoid it.

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


# ---------------------------------------------------------------------------------------------
# Bucket-contiguous term-range sharding (the tensor-core path's multi-GPU form).
#
# The tensor-core step (csrc/tc.cuh) evaluates 128 x 128-point chunks; with BASELINE config 5's
# T = 16384 "sharded across 1/2/4/8 GPUs", point ranges of 2048-8192 points per rank would fall
# below one chunk.  So ranks shard the TERMS instead, in the matrix method's own bucket order
# (terms sorted by (x, y) exponent): the terms, sorted by (dx, dy) descending,
# are cut into `world` contiguous ranges of ~t/world terms; every rank evaluates all T points of
# its range with its own handle (full T: whole chunks) and sends its G_r output rows to the root.
# Because the ranges are contiguous in bucket order, consecutive ranks share at most ONE bucket
# (the one cut by the boundary); the root adds those boundary rows mod p (values < p < 2^62, so
# the int64 sum cannot overflow).  No modular all-reduce is needed (MT18).
# ---------------------------------------------------------------------------------------------
def bucket_keys(exps) -> "np.ndarray":
    import numpy as np
    e = np.asarray(exps)
    return (e[:, 0].astype(np.uint64) << np.uint64(32)) | e[:, 1].astype(np.uint64)


def term_partition(exps, world: int):
    """Stable descending sort of the terms by (dx, dy) and the rank boundaries.
    Returns (order, bounds): rank r owns terms order[bounds[r]:bounds[r+1]] (~t/world each)."""
    import numpy as np
    key = bucket_keys(exps)
    order = np.argsort(~key, kind="stable")                  # descending (dx, dy)
    t = key.size
    bounds = [(r * t) // world for r in range(world + 1)]
    return order, bounds


class TermShardedEval:
    """Per-rank row bookkeeping + the root gather for term-range sharding.

    ``keys_sorted``: bucket keys of all terms in the partition order (``bucket_keys(exps)[order]``);
    ``bounds`` from ``term_partition``.  Rank r's handle produces rows for the distinct keys of
    its range, descending -- exactly the global rows row_off[r] .. row_off[r] + G_r - 1, where the
    first one is shared with rank r-1 when ``overlap[r]``.
    """

    def __init__(self, keys_sorted, bounds, T: int, p: int, device, group=None, root: int = 0):
        import numpy as np
        self.T, self.p, self.root, self.group = T, int(p), root, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        assert len(bounds) == self.world + 1
        ks = np.asarray(keys_sorted, dtype=np.uint64)
        new_row = np.ones(ks.size, dtype=bool)
        new_row[1:] = ks[1:] != ks[:-1]
        row_of = np.cumsum(new_row) - 1                          # global row of each sorted term
        self.G = int(row_of[-1]) + 1 if ks.size else 0
        self.G_r, self.row_off, self.overlap = [], [], []
        for r in range(self.world):
            a, b = bounds[r], bounds[r + 1]
            if a == b:
                self.G_r.append(0); self.row_off.append(0); self.overlap.append(False)
                continue
            self.G_r.append(int(row_of[b - 1] - row_of[a]) + 1)
            self.row_off.append(int(row_of[a]))
            self.overlap.append(bool(a > 0 and not new_row[a]))
        self.is_root = self.rank == root
        G_me = self.G_r[self.rank]
        self.out = torch.empty((self.G, T), dtype=torch.int64, device=device) if self.is_root else None
        self.local = (self.out if self.world == 1
                      else torch.zeros((G_me, T), dtype=torch.int64, device=device))
        self.shared = (torch.empty((self.world, T), dtype=torch.int64, device=device)
                       if self.is_root and self.world > 1 else None)

    def run(self, eval_local, gather: bool = True):
        """eval_local(out_view [G_r, T]) fills this rank's rows; then the root receives every
        rank's rows straight into place and adds the shared boundary rows mod p."""
        if self.G_r[self.rank]:
            eval_local(self.local)
        if self.world == 1 or not gather:
            return self.out if self.world == 1 else None
        ops = []
        if not self.is_root:
            g = self.G_r[self.rank]
            if g:
                if self.overlap[self.rank]:
                    ops.append(dist.P2POp(dist.isend, self.local[:1], self.root, self.group))
                    if g > 1:
                        ops.append(dist.P2POp(dist.isend, self.local[1:], self.root, self.group))
                else:
                    ops.append(dist.P2POp(dist.isend, self.local, self.root, self.group))
        else:
            for r in range(self.world):
                g, off = self.G_r[r], self.row_off[r]
                if not g:
                    continue
                if r == self.rank:
                    dst0 = self.shared[r:r + 1] if self.overlap[r] else self.out[off:off + 1]
                    dst0.copy_(self.local[:1])
                    if g > 1:
                        self.out[off + 1:off + g].copy_(self.local[1:])
                    continue
                if self.overlap[r]:
                    ops.append(dist.P2POp(dist.irecv, self.shared[r:r + 1], r, self.group))
                    if g > 1:
                        ops.append(dist.P2POp(dist.irecv, self.out[off + 1:off + g], r, self.group))
                else:
                    ops.append(dist.P2POp(dist.irecv, self.out[off:off + g], r, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if not self.is_root:
            return None
        for r in range(self.world):                              # boundary buckets, in rank order
            if self.G_r[r] and self.overlap[r]:
                row = self.out[self.row_off[r]]
                s = row + self.shared[r]
                row.copy_(torch.where(s >= self.p, s - self.p, s))
        return self.out
