"""Two processes, two GPUs, NCCL: the config-5 style sequence-sharded operator (st_forward_halo /
st_backward_halo with shard.nccl_halo) against the unsharded single-GPU run on the same inputs.
Skipped with fewer than 2 GPUs (the CPU protocol model in test_shard.py and the single-GPU lockstep
test in test_gpu_parity.py cover the exchange otherwise)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

B, H, L, d, w, eps, T, R = 1, 2, 2048, 64, 256, 0.05, 6, 2


def _inputs():
    rng = np.random.default_rng(5)
    return [(rng.standard_normal((B, H, L, d)) / np.sqrt(d)).astype(np.float32) for _ in range(4)]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2605_08123_b200 import band, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    plan = shard.SeqShard(L=L, w=w, world=world, rank=rank)
    win = plan.window
    hl = plan.rows.start - win.start
    to = lambda x: torch.from_numpy(np.ascontiguousarray(x[:, :, win.start:win.stop])).to(dev).to(torch.bfloat16)
    Q, K, V, G = (to(x) for x in _inputs())
    spec = band.BandSpec(batch=B, heads=H, seq_q=len(win), seq_k=len(win), head_dim=d, half_band=w, base_depth=T,
                         tail_depth=R, epsilon=eps, dtype="bf16")
    outs = shard.sharded_forward_backward(spec, Q, K, V, G, None, None, shard.nccl_halo(plan),
                                          range(hl, hl + len(plan.rows)))
    torch.cuda.synchronize()
    own = [o[:, :, hl:hl + len(plan.rows)].cpu().numpy() for o in outs[:4]]
    np.savez(f"{out_path}.{rank}.npz", O=own[0], dQ=own[1], dK=own[2], dV=own[3], d_eps=outs[4].cpu().numpy(),
             start=plan.rows.start, stop=plan.rows.stop)
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_sequence_sharding_matches_one_gpu(tmp_path):
    import torch.multiprocessing as mp
    from paper_2605_08123_b200 import shard
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "shard")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    # unsharded reference on GPU 0 through the same per-step kernels (a no-op halo hook)
    to = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)
    from paper_2605_08123_b200 import band
    spec = band.BandSpec(batch=B, heads=H, seq_q=L, seq_k=L, head_dim=d, half_band=w, base_depth=T, tail_depth=R,
                         epsilon=eps, dtype="bf16")
    ref = shard.sharded_forward_backward(spec, *(to(x) for x in _inputs()), None, None, lambda v: None, range(0, L))
    ref = [r.cpu().numpy() for r in ref]
    deps = 0.0
    for rank in range(2):
        z = np.load(f"{out}.{rank}.npz")
        a, b_ = int(z["start"]), int(z["stop"])
        for k, idx in (("O", 0), ("dQ", 1), ("dK", 2), ("dV", 3)):
            r = ref[idx][:, :, a:b_]
            e = np.linalg.norm(z[k] - r) / np.linalg.norm(r)
            assert e < 1e-6, (rank, k, e)
        deps = deps + z["d_eps"]
    assert np.linalg.norm(deps - ref[4]) / np.linalg.norm(ref[4]) < 1e-5
