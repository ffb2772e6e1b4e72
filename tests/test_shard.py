"""Multi-GPU partitioning on CPU ranks: world_size-2 gloo runs of
the batch x head split (configs 1-4) and of the config-5 sequence sharding
protocol (block column partials + w-wide dual halos), against unsharded runs."""
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_ref
import shard_model
from paper_2605_08123_b200 import configs, shard


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_head_partition_covers_and_balances():
    for n in (1, 7, 32, 128):
        for world in (1, 2, 3, 8):
            parts = [shard.head_partition(n, world, r) for r in range(world)]
            assert [h for p in parts for h in p] == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    ex, hd = shard.example_partition(8, 4, 4, 2)
    assert ex == range(16, 24) and hd == range(64, 96)


@pytest.mark.parametrize("L,w,world,block", [(131072, 256, 8, 128), (1000, 40, 3, 64), (64, 5, 2, 16)])
def test_seq_shard_plan(L, w, world, block):
    plans = [shard.SeqShard(L=L, w=w, world=world, rank=r, block=block) for r in range(world)]
    assert [i for p in plans for i in p.rows] == list(range(L))       # disjoint, contiguous cover
    for p in plans:
        assert p.rows.start % block == 0
        assert p.window.start == max(0, p.rows.start - w) and p.window.stop == min(L, p.rows.stop + w)
        # exactly the blocks whose windows cross the shard edge are exchanged
        for b in p.blocks:
            crosses_l = p.rank > 0 and p.window_of_block(b).start < p.rows.start
            crosses_r = p.rank < world - 1 and p.window_of_block(b).stop > p.rows.stop
            assert (b in p.boundary_blocks_left) == crosses_l
            assert (b in p.boundary_blocks_right) == crosses_r
    if L == 131072:  # config 5 at 8 GPUs: 16384 rows per GPU, a 256-wide halo, 2 boundary blocks per side
        assert len(plans[3].rows) == 16384 and len(plans[3].v_halo_left) == 256
        assert len(plans[3].boundary_blocks_left) == 2 and len(plans[3].boundary_blocks_right) == 2


def test_seq_sharded_solve_matches_unsharded_and_oracle(tmp_path):
    """Two gloo ranks running the block-partial step with the plan's halo exchange give
    bit-identical duals to one rank, and O = P V matches the restated reference."""
    L, w, d, eps, steps, block, seed = 64, 5, 8, 0.5, 6, 16, 3
    ctx = mp.get_context("spawn")
    for world in (1, 2):
        port = _port()
        procs = [ctx.Process(target=shard_model.seq_worker,
                             args=(r, world, port, L, w, d, eps, steps, block, seed, str(tmp_path / f"w{world}")))
                 for r in range(world)]
        (tmp_path / f"w{world}").mkdir()
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
    one = np.load(tmp_path / "w1" / "seq_0.npz")
    parts = [np.load(tmp_path / "w2" / f"seq_{r}.npz") for r in range(2)]
    u2 = np.concatenate([q["u"] for q in parts])
    v2 = np.concatenate([q["v"] for q in parts])
    assert np.array_equal(one["u"], u2) and np.array_equal(one["v"], v2)
    # against the oracle (T = steps - 2 base steps + R = 2 tail steps; O is gauge invariant)
    rng = np.random.default_rng(seed)
    Q, K = rng.standard_normal((L, d)) * 0.7, rng.standard_normal((L, d)) * 0.7
    V = rng.standard_normal((L, d))
    S = shard_model.score_band(Q, K, w, eps)
    O = shard_model.transport(S, u2, v2, V, w)
    cfg = configs.Config(0, B=1, H=1, L=L, d=d, w=w, eps=eps, T=steps - 2, R=2, dtype="f32")
    r = oracle_ref.run(cfg, Q[None], K[None], V[None], np.zeros((1, L, d)), backward=False)
    assert np.max(np.abs(O - r["O"][0])) <= 1e-10 * np.max(np.abs(r["O"][0]))


def test_head_sharding_gathers_the_unsharded_result(tmp_path):
    cfg_kw = dict(B=2, H=2, L=48, d=8, w=6, eps=0.4, T=5, R=2, dtype="f32", mask="uniform_len")
    port = _port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=shard_model.head_worker, args=(r, 2, port, cfg_kw, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    cfg = configs.Config(0, **cfg_kw)
    inp = configs.make_inputs(cfg)
    full = oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask)
    assert np.array_equal(np.load(tmp_path / "heads_O.npy"), full["O"])
