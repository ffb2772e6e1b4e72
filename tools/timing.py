"""Quick per-config timing of the CUDA path (development helper, not the bench)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2605_08123_b200 import band, configs

def bench(cid, iters=3, L=None):
    cfg = configs.CONFIGS[cid]
    if L: cfg = cfg.replace(L=L)
    inp = configs.make_inputs(cfg)
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin)
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    b = inp.bits or {}
    dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b else torch.from_numpy(x)).cuda().reshape(shp)
    Q, K, V, G = dev(inp.Q, 'Q'), dev(inp.K, 'K'), dev(inp.V, 'V'), dev(inp.G, 'G')
    rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).cuda()
    run = band.run_surrogate(Q, K, V, spec, rm, rm)
    mode = os.environ.get("BWD_MODE", "one_reference")
    band.r2_backward(run, G, mode=mode)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf, tb = [], []
    for _ in range(iters):
        e[0].record(); run = band.run_surrogate(Q, K, V, spec, rm, rm, validate=False, saved=run.saved, out=run.output)
        e[1].record(); band.r2_backward(run, G, mode=mode); e[2].record(); torch.cuda.synchronize()
        tf.append(e[0].elapsed_time(e[1])); tb.append(e[1].elapsed_time(e[2]))
    cells = cfg.nominal_cell_steps()
    t = min(tf) + min(tb)
    print(f"config {cid} L={cfg.L} [{mode}]: fwd {min(tf):.3f} ms bwd {min(tb):.3f} ms -> {cells/(t*1e-3):.3e} band-cells/s", flush=True)

for cid in [int(x) for x in sys.argv[1:]]:
    bench(cid)
