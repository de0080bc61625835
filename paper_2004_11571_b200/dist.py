"""Multi-GPU plumbing: one process per GPU, torch.distributed for
the process group and the NCCL transfers, libpe (C ABI) for everything that touches the values.

Two decompositions, each with one gather to the root as the only collective:

* ``ShardedEval`` -- point ranges (HM16 "N evaluations at a time", in its
  contiguous-range form): every rank holds the full replicated term set (its own handle),
  evaluates a contiguous block of the T points -- seeding at its own first point -- and the
  root gathers the G x T_r blocks and puts them back into rows with ``pe_unshard_columns``.
* ``TermShardedEval`` -- bucket-contiguous term ranges (the matrix method's own sorted order,
  PAPER.md:495-503): rank r evaluates all T points of ~t/P consecutive terms; the root receives
  every rank's rows straight into place, and the <= P-1 buckets cut by a range boundary are
  summed mod p by ``pe_rows_addmod`` (PAPER.md:489-503's coefficient reduction across ranks).

This module does no modular arithmetic and no per-column copies itself: the two libpe calls
above do that on the device.  ``addmod`` / ``unshard`` may be injected (the CPU gloo tests pass
host implementations, since libpe needs a GPU); the defaults call libpe and require CUDA tensors.

``world`` / ``rank`` may be given explicitly (no process group): ``TermShardedEval.assemble`` and
``ShardedEval.assemble`` then run the root's placement on per-rank outputs held by one process,
which is how the single-GPU tests drive exactly this bookkeeping.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(T: int, world: int, rank: int) -> tuple[int, int]:
    """Columns [off, off+cnt) of rank ``rank``: ceil split, trailing ranks may be short/empty."""
    per = -(-T // world) if T else 0
    off = min(rank * per, T)
    return off, max(0, min(per, T - off))


def shard_width(T: int, world: int) -> int:
    return -(-T // world) if T else 0


def _world_rank(group, world, rank):
    if world is not None:
        return world, (0 if rank is None else rank)
    if dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _stream_of(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def libpe_addmod(p: int):
    """dst <- (dst + src) mod p on device rows (pe_rows_addmod)."""
    import paper_2004_11571_b200 as pe

    def f(dst: torch.Tensor, src: torch.Tensor):
        if not (dst.is_cuda and src.is_cuda):
            raise RuntimeError("pe_rows_addmod needs device tensors (inject addmod= for CPU tests)")
        pe.rows_addmod(p, dst.data_ptr(), dst.stride(0), src.data_ptr(), src.stride(0), dst.shape[0], dst.shape[1],
                       _stream_of(dst))
    return f


def libpe_unshard(out: torch.Tensor, blocks: torch.Tensor, T: int):
    """out[:, r*Tr + k] <- blocks[r, :, k] (pe_unshard_columns)."""
    import paper_2004_11571_b200 as pe
    if not (out.is_cuda and blocks.is_cuda):
        raise RuntimeError("pe_unshard_columns needs device tensors (inject unshard= for CPU tests)")
    P, G, Tr = blocks.shape
    pe.unshard_columns(out.data_ptr(), out.stride(0), blocks.data_ptr(), P, G, Tr, T, _stream_of(out))


class ShardedEval:
    """Point-range sharding: buffers for one (G, T, world) shape, reused across steps."""

    def __init__(self, G: int, T: int, device, group=None, root: int = 0, world=None, rank=None,
                 unshard=None):
        self.G, self.T, self.root, self.group = G, T, root, group
        self.world, self.rank = _world_rank(group, world, rank)
        self.unshard = unshard or libpe_unshard
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
        dist.gather(self.local, list(self.gathered.unbind(0)) if self.is_root else None, dst=self.root,
                    group=self.group)
        if not self.is_root:
            return None
        self.unshard(self.out, self.gathered, self.T)
        return self.out

    def assemble(self, eval_rank, j0: int):
        """Single process, no process group: rank r's block is produced by
        ``eval_rank(r, j_first, cnt, out_view)`` straight into the gather buffer, then the root's
        placement runs as in ``run``."""
        assert self.is_root and self.world > 1
        for r in range(self.world):
            off, cnt = shard_range(self.T, self.world, r)
            if cnt:
                eval_rank(r, j0 + off, cnt, self.gathered[r])
        self.unshard(self.out, self.gathered, self.T)
        return self.out


# ---------------------------------------------------------------------------------------------
# Bucket-contiguous term-range sharding (the tensor-core path's multi-GPU form).
# The terms, sorted by (dx, dy) descending, are cut into `world` contiguous ranges of ~t/world
# terms; every rank evaluates all T points of its range with its own handle (whole 8192-point
# chunks, so the tensor-core kernel keeps its full 128 x 64 tiles) and sends its G_r output rows
# to the root.  Consecutive ranks share at most ONE bucket (the one cut by the boundary); the root
# adds those rows mod p with pe_rows_addmod.  No modular all-reduce is needed (cf. PAPER.md:
# 574-576, MT18's 1D block decomposition).
# ---------------------------------------------------------------------------------------------
def bucket_keys(exps) -> np.ndarray:
    e = np.asarray(exps)
    return (e[:, 0].astype(np.uint64) << np.uint64(32)) | e[:, 1].astype(np.uint64)


# Per-bucket cost of a shard in term-equivalents beyond its terms: tile padding (~half a 256-term
# tile), its pieces' epilogues and its fix-up row (scripts/partition_probe.py: shards of many small
# buckets ran ~8 % slower than equal-term shards of one large bucket).
BUCKET_COST_TERMS = 384


def term_partition(exps, world: int, bucket_cost: int = BUCKET_COST_TERMS):
    """Stable descending sort of the terms by (dx, dy) and the rank boundaries.
    Returns (order, bounds): rank r owns terms order[bounds[r]:bounds[r+1]], the cut points chosen
    so that every rank carries about the same cost = terms + bucket_cost per bucket it touches."""
    key = bucket_keys(exps)
    order = np.argsort(~key, kind="stable")                  # descending (dx, dy)
    t = key.size
    if t == 0 or world == 1:
        return order, [(r * t) // world for r in range(world + 1)]
    ks = key[order]
    w = np.ones(t, dtype=np.float64)
    w[np.r_[True, ks[1:] != ks[:-1]]] += bucket_cost        # charge each bucket at its first term
    c = np.cumsum(w)
    targets = c[-1] * np.arange(1, world) / world
    cuts = np.searchsorted(c, targets, side="left") + 1
    bounds = [0] + [int(min(max(x, 0), t)) for x in cuts] + [t]
    for r in range(1, world + 1):                            # keep them ordered
        bounds[r] = max(bounds[r], bounds[r - 1])
    return order, bounds


class TermShardedEval:
    """Per-rank row bookkeeping + the root gather for term-range sharding.

    ``keys_sorted``: bucket keys of all terms in the partition order (``bucket_keys(exps)[order]``);
    ``bounds`` from ``term_partition``.  Rank r's handle produces rows for the distinct keys of
    its range, descending -- exactly the global rows row_off[r] .. row_off[r] + G_r - 1, where the
    first one is shared with rank r-1 when ``overlap[r]``.
    """

    def __init__(self, keys_sorted, bounds, T: int, p: int, device, group=None, root: int = 0, world=None,
                 rank=None, addmod=None):
        self.T, self.p, self.root, self.group = T, int(p), root, group
        self.world, self.rank = _world_rank(group, world, rank)
        self.addmod = addmod or libpe_addmod(self.p)
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

    def _slices(self, r):
        """Row blocks of rank r's output sent separately: the shared boundary row on its own."""
        g = self.G_r[r]
        if not g:
            return []
        if not self.overlap[r]:
            return [slice(0, g)]
        return [slice(0, 1)] + ([slice(1, g)] if g > 1 else [])

    def _targets(self, r):
        """Where the root puts rank r's rows: [(row slice of r's output, destination view)]."""
        off, t = self.row_off[r], []
        for sl in self._slices(r):
            if self.overlap[r] and sl.start == 0:
                t.append((sl, self.shared[r:r + 1]))             # boundary row: summed afterwards
            else:
                t.append((sl, self.out[off + sl.start:off + sl.stop]))
        return t

    def _combine(self):
        """Boundary buckets, in rank order: out[row_off[r]] += shared[r] (mod p, on the device)."""
        for r in range(self.world):
            if self.G_r[r] and self.overlap[r]:
                o = self.row_off[r]
                self.addmod(self.out[o:o + 1], self.shared[r:r + 1])

    def run(self, eval_local, gather: bool = True):
        """eval_local(out_view [G_r, T]) fills this rank's rows; then the root receives every
        rank's rows straight into place and adds the shared boundary rows mod p."""
        if self.G_r[self.rank]:
            eval_local(self.local)
        if self.world == 1 or not gather:
            return self.out if self.world == 1 else None
        ops = []
        if not self.is_root:
            for sl in self._slices(self.rank):
                ops.append(dist.P2POp(dist.isend, self.local[sl], self.root, self.group))
        else:
            for r in range(self.world):
                for sl, dst in self._targets(r):
                    if r == self.rank:
                        dst.copy_(self.local[sl])                # root's own rows (device copy)
                    else:
                        ops.append(dist.P2POp(dist.irecv, dst, r, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if not self.is_root:
            return None
        self._combine()
        return self.out

    # ---- overlapped form: a rank's rows in two blocks, block 0's transfer under block 1's evaluation
    def set_splits(self, splits):
        """Every rank's row split s_r (rows [0, s_r) then [s_r, G_r); 0 = one block), e.g. each
        rank's pe_row_split gathered with all_gather_object once, outside the timed loop."""
        assert len(splits) == self.world
        self.splits = [int(x) for x in splits]

    def _blocks(self, r):
        g = self.G_r[r]
        sp = getattr(self, "splits", None)
        sp = sp[r] if sp else 0
        if not g:
            return []
        return [(0, sp), (sp, g)] if 0 < sp < g else [(0, g)]

    def _slices_in(self, r, a, b):
        """The parts of rank r's transfer slices (``_slices``) inside its rows [a, b)."""
        out = []
        for sl in self._slices(r):
            lo, hi = max(sl.start, a), min(sl.stop, b)
            if lo < hi:
                out.append(slice(lo, hi))
        return out

    def _dst(self, r, sl):
        if self.overlap[r] and sl.start == 0:                    # the shared boundary row
            return self.shared[r:r + 1]
        o = self.row_off[r]
        return self.out[o + sl.start:o + sl.stop]

    def run_blocks(self, eval_rows, gather: bool = True):
        """``run`` with each rank's rows evaluated in (up to) two blocks, ``eval_rows(a, b, local)``
        filling rows [a, b) of this rank's [G_r, T] output: block 0's rows go out (NCCL P2P, on
        NCCL's stream) while block 1 is evaluated on the compute stream, so most of the gather hides
        under the second block.  Matching order per (root, rank) pair: block 0 then block 1."""
        if self.world == 1 or not gather:
            if self.G_r[self.rank]:
                eval_rows(0, self.G_r[self.rank], self.local)
            return self.out if self.world == 1 else None
        works = []
        for bi in range(2):
            mine = self._blocks(self.rank)
            if bi < len(mine):
                eval_rows(mine[bi][0], mine[bi][1], self.local)
            ops = []
            if not self.is_root:
                if bi < len(mine):
                    for sl in self._slices_in(self.rank, *mine[bi]):
                        ops.append(dist.P2POp(dist.isend, self.local[sl], self.root, self.group))
            else:
                for r in range(self.world):
                    br = self._blocks(r)
                    if bi >= len(br):
                        continue
                    for sl in self._slices_in(r, *br[bi]):
                        if r == self.rank:
                            self._dst(r, sl).copy_(self.local[sl])    # root's own rows (device copy)
                        else:
                            ops.append(dist.P2POp(dist.irecv, self._dst(r, sl), r, self.group))
            if ops:
                works += dist.batch_isend_irecv(ops)
        for w in works:
            w.wait()
        if not self.is_root:
            return None
        self._combine()
        return self.out

    def assemble(self, locals_):
        """Single process, no process group: ``locals_[r]`` is rank r's [G_r, T] output; the
        root's placement and boundary sums run exactly as in ``run``."""
        assert self.is_root and self.world > 1
        for r in range(self.world):
            for sl, dst in self._targets(r):
                dst.copy_(locals_[r][sl])
        self._combine()
        return self.out
