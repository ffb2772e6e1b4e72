"""Dev check: tensor-core forward vs generic forward on the same inputs (+ timing)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2605_08123_b200 import band, configs

def run(cfg, generic, iters=3):
    inp = configs.make_inputs(cfg)
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin,
                         dustbin_cost=cfg.dustbin_cost, generic=generic)
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    b = inp.bits or {}
    dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b else torch.from_numpy(x)).cuda().reshape(shp)
    Q, K, V = dev(inp.Q, 'Q'), dev(inp.K, 'K'), dev(inp.V, 'V')
    rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).cuda()
    ws = band.Workspace()
    run = band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        e0.record(); band.run_surrogate(Q, K, V, spec, rm, rm, out=run.output, saved=run.saved, workspace=ws, validate=False); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    u, v, g = run.tail_duals(inp.row_mask, inp.col_mask)
    return run.output.cpu().numpy(), u, v, min(ts)

for cid, L in [(int(a.split(':')[0]), int(a.split(':')[1]) if ':' in a else None) for a in sys.argv[1:]]:
    cfg = configs.CONFIGS[cid] if cid in configs.CONFIGS else None
    if L: cfg = cfg.replace(L=L)
    og, ug, vg, tg = run(cfg, True)
    ot, ut, vt, tt = run(cfg, False)
    rel = np.linalg.norm(ot - og) / np.linalg.norm(og)
    du = np.abs(ut - ug).max(); dv = np.abs(vt - vg).max()
    print(f"config {cid} L={cfg.L}: O rel diff tc vs generic {rel:.2e}, max|du| {du:.2e} max|dv| {dv:.2e}; "
          f"fwd generic {tg:.3f} ms, tc {tt:.3f} ms", flush=True)
