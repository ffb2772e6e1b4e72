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

  plus the one-time Q/K/V halo rows.  Every own row's and own column's
  reduction lies inside the local window, so own-row outputs equal the
  unsharded ones up to the association order of the blocked reductions: a
  local problem starts at window.start, so its 128-row blocking can differ
  from the global one (the lockstep GPU test bounds the difference at 1e-6
  rel-L2; tests/test_shard.py checks bit-identity of the f64 protocol model).
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


# --------------------------------------------------------------------------- device path
# A rank runs the band operator on its local problem = own rows plus a w-wide halo each side
# (SeqShard.window), through st_forward_halo / st_backward_halo.  The library calls back right
# after it has enqueued each kernel whose output vector the next kernel reads across the shard
# edge; the callback completes that vector's halo entries on the same stream.

def _halo_slices(plan: SeqShard):
    """(left halo width, right halo width, own [lo, hi) in local indices)."""
    hl = plan.rows.start - plan.window.start
    hr = plan.window.stop - plan.rows.stop
    return hl, hr, hl, hl + len(plan.rows)


def nccl_halo(plan: SeqShard, group=None):
    """Halo completion over torch.distributed point-to-point (NCCL over NVLink for CUDA tensors).
    The ops are stream-ordered after the producing kernel; nothing synchronises the host."""
    hl, hr, lo, hi = _halo_slices(plan)
    left, right = plan.neighbour(-1), plan.neighbour(+1)

    def ex(v: torch.Tensor) -> None:  # v: [BH, L'] view of the produced vector
        to_l = v[:, lo: lo + (left.window.stop - left.rows.stop)].contiguous() if left else None
        to_r = v[:, hi - (right.rows.start - right.window.start): hi].contiguous() if right else None
        like_l = v.new_empty((v.shape[0], hl)) if left else None
        like_r = v.new_empty((v.shape[0], hr)) if right else None
        got_l, got_r = exchange(plan, to_l, to_r, like_l, like_r, group)
        if left:
            v[:, :hl].copy_(got_l)
        if right:
            v[:, hi: hi + hr].copy_(got_r)
    return ex


class Lockstep:
    """Single-GPU emulation of the sequence-sharded run: one host thread per shard, each on its own
    CUDA stream; at every hook the shards meet at a barrier and copy each other's boundary entries
    (stream-ordered by events -- no kernel ever waits on another).  Test harness for the protocol
    nccl_halo runs across GPUs."""

    def __init__(self, plans, streams):
        import threading
        self.plans, self.streams = plans, streams
        self.barrier = threading.Barrier(len(plans))
        self.views = [None] * len(plans)
        self.ready = [torch.cuda.Event() for _ in plans]
        self.copied = [torch.cuda.Event() for _ in plans]

    def exchange_for(self, r: int):
        plan = self.plans[r]
        hl, hr, lo, hi = _halo_slices(plan)

        def ex(v: torch.Tensor) -> None:
            s = self.streams[r]
            self.views[r] = v
            self.ready[r].record(s)
            self.barrier.wait()
            nbs = [q for q in (r - 1, r + 1) if 0 <= q < len(self.plans)]
            with torch.cuda.stream(s):
                for q in nbs:
                    s.wait_event(self.ready[q])
                    o = self.plans[q]
                    vo = self.views[q]
                    _, ohr, olo, ohi = _halo_slices(o)
                    if q < r:  # its last hl own entries -> my left halo
                        v[:, :hl].copy_(vo[:, ohi - hl: ohi])
                    else:      # its first hr own entries -> my right halo
                        v[:, hi: hi + hr].copy_(vo[:, olo: olo + hr])
                self.copied[r].record(s)
            self.barrier.wait()
            for q in nbs:  # the neighbour read my vector: its copy precedes my next write of it
                s.wait_event(self.copied[q])
            self.barrier.wait()
        return ex


class _Hook:
    """ctypes st_halo_fn that maps the library's vector back to a [BH, L'] float view."""

    def __init__(self, bh: int, buffers, ex):
        self.bh, self.buffers, self.ex = bh, buffers, ex
        self.error = None
        from . import _lib
        self.cfn = _lib.HALO_FN(self)

    def __call__(self, user, kind, vec, n, stream):
        try:
            for t in self.buffers:
                base, nbytes = t.data_ptr(), t.numel() * t.element_size()
                if base <= vec < base + nbytes:
                    off = (vec - base) // 4
                    flat = t.view(-1).view(torch.uint8)[: (nbytes // 4) * 4].view(torch.float32)
                    self.ex(flat[off: off + n].view(self.bh, -1))
                    return
            raise RuntimeError("halo vector outside the registered buffers")
        except Exception as e:  # never raise through C
            self.error = e


def sharded_forward_backward(spec, Q, K, V, G, row_mask, col_mask, ex, own_rows: range, mode="one_reference"):
    """One rank's sequence-sharded fwd + bwd on its local problem (own rows + halos).
    Returns (O, dQ, dK, dV, d_eps) of the local problem; rows outside `own_rows` are unspecified
    and d_eps covers the own rows only (sum it over ranks)."""
    import ctypes
    from . import _lib
    from .band import _check, _ptr
    import dataclasses
    lib = _lib.lib
    dev = Q.device
    spec = dataclasses.replace(spec, stored_band=True)  # the halo entry points run on the stored-band kernels
    ws = torch.empty(max(spec.workspace_bytes(), 256), dtype=torch.uint8, device=dev)
    saved = torch.empty(spec.saved_bytes(), dtype=torch.uint8, device=dev)
    O = torch.empty((spec.batch, spec.heads, spec.rows, spec.head_dim), dtype=torch.float32, device=dev)
    dQ, dK, dV = (torch.empty_like(O) for _ in range(3))
    d_eps = torch.empty(spec.batch * spec.heads, dtype=torch.float32, device=dev)
    eta = torch.empty((spec.batch, spec.heads, spec.cols), dtype=torch.float32, device=dev)
    hook = _Hook(spec.batch * spec.heads, [ws, saved], ex)
    d = spec.desc()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _check(lib.st_forward_halo(ctypes.byref(d), _ptr(Q), _ptr(K), _ptr(V), _ptr(row_mask), _ptr(col_mask), _ptr(O),
                               _ptr(saved), _ptr(ws), ws.numel(), stream, hook.cfn, None))
    m = {"one_reference": _lib.ST_ONE_REFERENCE, "direct_four_plan": _lib.ST_DIRECT_FOUR_PLAN}[mode]
    _check(lib.st_backward_halo(ctypes.byref(d), _ptr(saved), _ptr(Q), _ptr(K), _ptr(V), _ptr(G), _ptr(row_mask),
                                _ptr(col_mask), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(d_eps), _ptr(eta), m, _ptr(ws),
                                ws.numel(), stream, hook.cfn, None, own_rows.start, own_rows.stop))
    if hook.error is not None:
        raise hook.error
    return O, dQ, dK, dV, d_eps
