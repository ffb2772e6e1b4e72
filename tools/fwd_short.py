"""Dev helper: forward of one config with a short base solve (ncu launch timing of the step kernels)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2605_08123_b200 import band, configs
cid = int(sys.argv[1])
cfg = configs.CONFIGS[cid].replace(T=int(sys.argv[2]) if len(sys.argv) > 2 else 6)
inp = configs.make_inputs(cfg)
spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                     base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin)
shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
b = inp.bits or {}
dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b else torch.from_numpy(x)).cuda().reshape(shp)
Q, K, V = dev(inp.Q, 'Q'), dev(inp.K, 'K'), dev(inp.V, 'V')
for _ in range(2):
    band.run_surrogate(Q, K, V, spec, validate=False)
torch.cuda.synchronize()
print("done")
