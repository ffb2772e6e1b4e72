"""Multi-GPU partitioning of the band operator.

* Configs 1-4: every (b, h) problem is independent -> ``head_partition`` /
  ``example_partition`` split the flat head range contiguously across ranks;
  no collective on the data path (weak scaling in ``bench.py``).
* Config 5: one very long sequence -> ``SeqShard`` splits the 128-row blocks
  contiguously across ranks.  The fused Sinkhorn step (``k_fsolve``) already
  reduces every column over fixed-order per-block partials, so a shard
  boundary is a block boundary and the only cross-rank data per full step are

    - the column partials of the <= ceil(w/128) boundary blocks on each side,
      restricted to the neighbour's columns (``partials_to_left/right``), and
    - the w-wide slice of new column duals v on each side (``v_halo``),

  plus the one-time Q/K/V halo rows.  The sharded reduction order equals the
  unsharded one, so sharded duals are bit-identical to a one-GPU run.
  ``exchange`` moves these halos with torch.distributed point-to-point
  (NCCL over NVLink for CUDA tensors, gloo for the CPU tests).

The device-side fused variant (publishing the boundary partials straight into
the neighbour's tagged-partial buffer over NVLink peer memory) is the next
step; this module is the host plan and the exchange it must reproduce.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple

import torch
import torch.distributed as dist

BLOCK = 128  # rows per block of the band kernels


def head_partition(n_heads: int, world: int, rank: int) -> range:
    """Contiguous, balanced split of the flat (b*H + h) head range."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_heads, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def example_partition(batch: int, heads: int, world: int, rank: int) -> Tuple[range, range]:
    """Weak-scaling job of ``world * batch`` examples: rank r owns examples
    [r*batch, (r+1)*batch) and their flat head range."""
    ex = range(rank * batch, (rank + 1) * batch)
    return ex, range(ex.start * heads, ex.stop * heads)


@dataclasses.dataclass(frozen=True)
class SeqShard:
    """Contiguous block-aligned sequence shard of one rank."""
    L: int
    w: int
    world: int
    rank: int
    block: int = BLOCK

    @property
    def n_blocks(self) -> int:
        return (self.L + self.block - 1) // self.block

    @property
    def blocks(self) -> range:
        """Own row blocks (balanced split of the block list)."""
        return head_partition(self.n_blocks, self.world, self.rank)

    @property
    def rows(self) -> range:
        b = self.blocks
        return range(min(b.start * self.block, self.L), min(b.stop * self.block, self.L))

    # columns = rows (square band); a rank owns the columns of its own blocks
    @property
    def cols(self) -> range:
        return self.rows

    @property
    def window(self) -> range:
        """Columns the own rows touch: own columns plus a w-wide halo each side."""
        r = self.rows
        return range(max(0, r.start - self.w), min(self.L, r.stop + self.w))

    @property
    def v_halo_left(self) -> range:
        return range(self.window.start, self.rows.start)

    @property
    def v_halo_right(self) -> range:
        return range(self.rows.stop, self.window.stop)

    def window_of_block(self, b: int) -> range:
        """Window columns of block b, clipped to [0, L)."""
        return range(max(0, b * self.block - self.w), min(self.L, (b + 1) * self.block + self.w))

    @property
    def boundary_blocks_left(self) -> range:
        """Own blocks whose windows reach columns owned by the left neighbour."""
        if self.rank == 0:
            return range(0)
        own = self.blocks
        n = 0
        for b in own:
            if self.window_of_block(b).start < self.rows.start:
                n += 1
        return range(own.start, own.start + n)

    @property
    def boundary_blocks_right(self) -> range:
        if self.rank == self.world - 1:
            return range(0)
        own = self.blocks
        n = 0
        for b in reversed(own):
            if self.window_of_block(b).stop > self.rows.stop:
                n += 1
        return range(own.stop - n, own.stop)

    def neighbour(self, side: int) -> Optional["SeqShard"]:
        r = self.rank + side
        if not 0 <= r < self.world:
            return None
        return dataclasses.replace(self, rank=r)


def exchange(plan: SeqShard, to_left: Optional[torch.Tensor], to_right: Optional[torch.Tensor],
             from_left_like: Optional[torch.Tensor], from_right_like: Optional[torch.Tensor],
             group=None) -> Tuple[Optional[torch.Tensor], Optional[torch.Tensor]]:
    """Neighbour halo exchange: send ``to_left`` to rank-1 and ``to_right`` to
    rank+1, receive into buffers shaped like ``from_*_like``.  Point-to-point
    only (no collective); the caller sizes buffers from the plan, which is
    symmetric between neighbours."""
    ops = []
    got_l = got_r = None
    if plan.rank > 0:
        got_l = torch.empty_like(from_left_like)
        ops.append(dist.P2POp(dist.isend, to_left.contiguous(), plan.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, got_l, plan.rank - 1, group))
    if plan.rank < plan.world - 1:
        got_r = torch.empty_like(from_right_like)
        ops.append(dist.P2POp(dist.isend, to_right.contiguous(), plan.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, got_r, plan.rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return got_l, got_r
