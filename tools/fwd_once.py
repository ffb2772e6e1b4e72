"""Dev helper: run the forward of one config a few times (for ncu)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2605_08123_b200 import band, configs
cid = int(sys.argv[1]); L = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != '-' else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = configs.CONFIGS[cid]
if L: cfg = cfg.replace(L=L)
inp = configs.make_inputs(cfg)
spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                     base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin)
shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
b = inp.bits or {}
dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b else torch.from_numpy(x)).cuda().reshape(shp)
Q, K, V = dev(inp.Q, 'Q'), dev(inp.K, 'K'), dev(inp.V, 'V')
rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).cuda()
for _ in range(reps):
    run = band.run_surrogate(Q, K, V, spec, rm, rm, validate=False)
torch.cuda.synchronize()
print("done", float(run.output.abs().sum()))
