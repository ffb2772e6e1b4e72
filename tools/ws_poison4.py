"""Dev helper: does the backward modify the saved state / does the forward write all of it."""
import sys, os, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', 'tests'))
from paper_2605_08123_b200 import band, configs
import test_gpu_parity as T
cfg = configs.Config(0, B=2, H=2, L=300, d=64, w=20, eps=0.2, T=8, R=2, dtype="f32", mask="uniform_len")
inp = configs.make_inputs(cfg)
b = inp.bits or {}
shp = (cfg.B, cfg.H, cfg.rows, 64)
Q, K, V, G = (T._dev(getattr(inp, k), b.get(k)).reshape(shp) for k in ("Q", "K", "V", "G"))
rm = torch.from_numpy(inp.row_mask).cuda()
spec = band.BandSpec(batch=2, heads=2, seq_q=300, seq_k=300, head_dim=64, half_band=20, base_depth=8, tail_depth=2,
                     epsilon=0.2, dtype="f32")
for fill in (0, 255):
    ws = band.Workspace()
    ws._buf = torch.full((spec.workspace_bytes() + 4096,), fill, dtype=torch.uint8, device="cuda")
    saved = torch.full_like(band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws).saved, 77)
    run = band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws, saved=saved)
    torch.cuda.synchronize()
    s0 = run.saved.clone()
    cot = band.r2_backward(run, G, workspace=ws)
    torch.cuda.synchronize()
    un = torch.nonzero(s0.view(torch.float32) == 215274704.0).flatten().tolist()
    rng = []
    for x in un:
        if rng and rng[-1][1] == x - 1: rng[-1][1] = x
        else: rng.append([x, x])
    print("untouched ranges", rng[:40], "of", s0.numel() // 4)
    print("fill", fill, "saved words untouched by fwd:", int((s0 == 77).sum()), "changed by bwd:", int((s0 != run.saved).sum()),
          "v0[:4]", s0.view(torch.float32)[3600:3604].tolist())
