"""Band-free sweeps (st_bfree.cu) against the stored-band kernels on the same inputs (development A/B)."""
import dataclasses, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2605_08123_b200 import band, configs


def run(cid, L, heads, mode, masked=False):
    cfg = configs.CONFIGS[cid].replace(L=L, B=1, H=heads)
    inp = configs.make_inputs(cfg)
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    b = inp.bits
    dev = lambda k: torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16).cuda().reshape(shp)
    Q, K, V, G = dev('Q'), dev('K'), dev('V'), dev('G')
    rm = None
    if masked:
        m = np.ones((cfg.B, cfg.L), np.uint8)
        m[:, cfg.L - 300:] = 0
        m[:, 1000:1100] = 0
        rm = torch.from_numpy(m).cuda()
    res = {}
    for sb in (True, False):
        spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                             base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, stored_band=sb)
        ws = band.Workspace()
        r = band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws)
        c = band.r2_backward(r, G, mode=mode, workspace=ws)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); r = band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws, validate=False)
        e[1].record(); c = band.r2_backward(r, G, mode=mode, workspace=ws); e[2].record(); torch.cuda.synchronize()
        print(f"  stored_band={sb}: ws {spec.workspace_bytes()/2**20:.0f} MiB fwd {e[0].elapsed_time(e[1]):.3f} ms bwd {e[1].elapsed_time(e[2]):.3f} ms", flush=True)
        res[sb] = dict(O=r.output, dQ=c.grad_q, dK=c.grad_k, dV=c.grad_v, eta=c.eta_v, deps=c.d_eps)
    for k in res[True]:
        a, bb = res[True][k].double(), res[False][k].double()
        err = float((a - bb).norm() / a.norm().clamp_min(1e-300))
        print(f"  {k}: rel-L2 band-free vs stored = {err:.3e}  (nan: {bool(torch.isnan(bb).any())})", flush=True)


CASES = [(4, 4096, 2, "one_reference"), (4, 4096, 2, "direct_four_plan"), (5, 8192, 2, "one_reference"),
             (4, 4000, 3, "one_reference", True), (4, 32768, 4, "one_reference"), (5, 131072, 1, "one_reference")]
if len(sys.argv) > 1:
    CASES = [(4, 16384, 4, "one_reference"), (5, 16384, 4, "direct_four_plan")]
for args in CASES:
    print("config", *args, flush=True)
    run(*args)
