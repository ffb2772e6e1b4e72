"""TEST INFRASTRUCTURE: an f64 numpy model of the fused block-partial Sinkhorn
step that k_fsolve runs on the GPU (row LSE with the previous dual as offset,
then fixed-order per-block column partials), driven shard by shard with
paper_2605_08123_b200.shard's plan and halo exchange.  It checks the
partitioning protocol of SURVEY §8(e) (config 5 sequence sharding) on CPU
ranks over gloo; it is not a product path and nothing in the package imports it.
"""
from __future__ import annotations

import numpy as np
import torch

from paper_2605_08123_b200 import shard


def score_band(Q, K, w, eps, mask=None):
    """S[i, k] = q_i . k_j / (sqrt(d) eps), j = i - w + k; -inf off support."""
    L, d = Q.shape
    Wf = 2 * w + 1
    S = np.full((L, Wf), -np.inf)
    for i in range(L):
        for k in range(Wf):
            j = i - w + k
            if 0 <= j < L and (mask is None or (mask[i] and mask[j])):
                S[i, k] = float(Q[i] @ K[j]) / (np.sqrt(d) * eps)
    return S


def solve(S, w, steps, plan: shard.SeqShard, group=None):
    """Run `steps` full steps on the rank's shard; returns (u, v) on own rows / columns
    (raw duals, natural log), identical on every partition."""
    L = S.shape[0]
    u = np.zeros(L)
    v = np.zeros(L)          # valid on the rank's window (own columns + halos)
    rows, win = plan.rows, plan.window
    own_blocks = plan.blocks
    col_on = np.isfinite(S).any(axis=1)  # square support: a column is active iff its row is

    for t in range(1, steps + 1):
        # ---- row pass on own rows
        unew = np.full(L, -np.inf)
        for i in rows:
            if not np.isfinite(S[i]).any():
                u[i] = 0.0
                continue
            js = np.arange(i - w, i + w + 1)
            ok = (js >= 0) & (js < L)
            x = np.where(ok, S[i] + np.where(ok, v[np.clip(js, 0, L - 1)], 0.0), -np.inf)
            o = -np.max(x) if t == 1 else u[i]
            u[i] = o - np.log(np.sum(np.exp(x + o)))
            unew[i] = u[i]
        # ---- column partials of own blocks over their windows
        part = {}
        for b in own_blocks:
            wb = plan.window_of_block(b)
            p = np.zeros(L)
            for i in range(b * plan.block, min((b + 1) * plan.block, L)):
                if not np.isfinite(unew[i]):
                    continue
                for k in range(2 * w + 1):
                    j = i - w + k
                    if wb.start <= j < wb.stop and np.isfinite(S[i, k]):
                        p[j] += np.exp(S[i, k] + unew[i] + v[j])
            part[b] = p
        # ---- exchange the boundary blocks' partials for the neighbours' columns.
        # Message to the left = my left boundary blocks over columns [win.start, rows.start)
        # (the left neighbour's right halo); to the right = my right boundary blocks over
        # [rows.stop, win.stop).  Buffers are sized from the neighbour's plan.
        if plan.world > 1:
            left, right = plan.neighbour(-1), plan.neighbour(+1)

            def pack(blocks, lo, hi):
                out = np.zeros((max(len(blocks), 1), max(hi - lo, 1)))
                for n, b in enumerate(blocks):
                    out[n, : hi - lo] = part[b][lo:hi]
                return torch.from_numpy(out)

            to_l = pack(plan.boundary_blocks_left, win.start, rows.start) if left else None
            to_r = pack(plan.boundary_blocks_right, rows.stop, win.stop) if right else None
            like_l = (torch.zeros((max(len(left.boundary_blocks_right), 1), max(left.window.stop - left.rows.stop, 1)),
                                  dtype=torch.float64) if left else None)
            like_r = (torch.zeros((max(len(right.boundary_blocks_left), 1), max(right.rows.start - right.window.start, 1)),
                                  dtype=torch.float64) if right else None)
            got_l, got_r = shard.exchange(plan, to_l, to_r, like_l, like_r, group)
            if left:  # its right boundary blocks over my columns [rows.start, left.window.stop)
                for n, b in enumerate(left.boundary_blocks_right):
                    p = np.zeros(L)
                    p[rows.start: left.window.stop] = got_l.numpy()[n, : left.window.stop - rows.start]
                    part[b] = p
            if right:  # its left boundary blocks over my columns [right.window.start, rows.stop)
                for n, b in enumerate(right.boundary_blocks_left):
                    p = np.zeros(L)
                    p[right.window.start: rows.stop] = got_r.numpy()[n, : rows.stop - right.window.start]
                    part[b] = p
        # ---- combine: own columns, blocks in ascending global order
        vnew = v.copy()
        for j in rows:
            if not col_on[j]:
                vnew[j] = 0.0
                continue
            s = 0.0
            for b in sorted(part):
                if plan.window_of_block(b).start <= j < plan.window_of_block(b).stop:
                    s += part[b][j]
            vnew[j] = v[j] - np.log(s)
        v = vnew
        # ---- v halo exchange: my first / last columns the neighbours' windows reach
        if plan.world > 1:
            left, right = plan.neighbour(-1), plan.neighbour(+1)
            to_l = torch.from_numpy(v[rows.start: left.window.stop].copy()) if left else None
            to_r = torch.from_numpy(v[right.window.start: rows.stop].copy()) if right else None
            like_l = torch.zeros(rows.start - win.start, dtype=torch.float64) if left else None
            like_r = torch.zeros(win.stop - rows.stop, dtype=torch.float64) if right else None
            got_l, got_r = shard.exchange(plan, to_l, to_r, like_l, like_r, group)
            if left:
                v[win.start: rows.start] = got_l.numpy()
            if right:
                v[rows.stop: win.stop] = got_r.numpy()
    return u[rows.start: rows.stop].copy(), v[rows.start: rows.stop].copy()


def transport(S, u, v, V, w):
    """O = P V with P = exp(S + u + v) on the band (gauge invariant)."""
    L = S.shape[0]
    O = np.zeros((L, V.shape[1]))
    for i in range(L):
        for k in range(2 * w + 1):
            j = i - w + k
            if 0 <= j < L and np.isfinite(S[i, k]):
                O[i] += np.exp(S[i, k] + u[i] + v[j]) * V[j]
    return O


# ---------------------------------------------------------------- multi-process drivers (gloo, CPU)
def _init(rank, world, port):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def seq_worker(rank, world, port, L, w, d, eps, steps, block, seed, outdir):
    """Sequence-sharded solve of one head: rank's (u, v) slice -> outdir/seq_<rank>.npz."""
    dist = _init(rank, world, port)
    rng = np.random.default_rng(seed)
    Q, K = rng.standard_normal((L, d)) * 0.7, rng.standard_normal((L, d)) * 0.7
    S = score_band(Q, K, w, eps)
    plan = shard.SeqShard(L=L, w=w, world=world, rank=rank, block=block)
    u, v = solve(S, w, steps, plan)
    np.savez(f"{outdir}/seq_{rank}.npz", u=u, v=v, rows=np.array([plan.rows.start, plan.rows.stop]))
    dist.barrier()
    dist.destroy_process_group()


def head_worker(rank, world, port, cfg_kw, outdir):
    """Batch x head sharding: each rank runs the oracle on its head slice, all-gathers O."""
    import oracle_ref
    from paper_2605_08123_b200 import configs
    dist = _init(rank, world, port)
    cfg = configs.Config(0, **cfg_kw)
    heads = shard.head_partition(cfg.B * cfg.H, world, rank)
    inp = configs.make_inputs(cfg, heads=heads)
    r = oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, heads=inp.heads)
    O = torch.from_numpy(np.ascontiguousarray(r["O"]))
    sizes = [len(shard.head_partition(cfg.B * cfg.H, world, q)) for q in range(world)]
    buf = [torch.zeros((n,) + tuple(O.shape[1:]), dtype=O.dtype) for n in sizes]
    dist.all_gather(buf, O)
    if rank == 0:
        np.save(f"{outdir}/heads_O.npy", torch.cat(buf).numpy())
    dist.barrier()
    dist.destroy_process_group()
