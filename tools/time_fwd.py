"""Dev helper: median forward time of one config (optionally a head subset / length), no checks.
    python tools/time_fwd.py CID [L|-] [NHEADS|-] [T|-]     (env switches apply, e.g. ST_PHASE_DBG)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2605_08123_b200 import band, configs
cid = int(sys.argv[1])
cfg = configs.CONFIGS[cid]
if len(sys.argv) > 2 and sys.argv[2] != '-': cfg = cfg.replace(L=int(sys.argv[2]))
nh = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != '-' else cfg.B * cfg.H
if len(sys.argv) > 4 and sys.argv[4] != '-': cfg = cfg.replace(T=int(sys.argv[4]))
inp = configs.make_inputs(cfg, heads=range(nh))
spec = band.BandSpec(batch=nh, heads=1, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                     base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype)
shp = (nh, 1, cfg.rows, cfg.d)
b = inp.bits or {}
dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b else torch.from_numpy(x)).cuda().reshape(shp)
Q, K, V = dev(inp.Q, 'Q'), dev(inp.K, 'K'), dev(inp.V, 'V')
ws = band.Workspace()
band.run_surrogate(Q, K, V, spec, workspace=ws, validate=False)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); band.run_surrogate(Q, K, V, spec, workspace=ws, validate=False); e.record()
    torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print(f"fwd_ms {sorted(ts)[2]:.3f} env ST_PHASE_DBG={os.environ.get('ST_PHASE_DBG','0')}")
