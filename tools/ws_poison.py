"""Dev helper: find workspace regions read before written (poison the caller workspace with NaN bytes)."""
import sys, os, torch, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', 'tests'))
from paper_2605_08123_b200 import band, configs
import test_gpu_parity as T
cfg = configs.Config(0, B=2, H=2, L=260, d=128, w=20, eps=0.3, T=10, R=3, dtype="bf16", mask="uniform_len")
inp = configs.make_inputs(cfg)
t, rm, cm, nh = T._cert_inputs(cfg, inp)
spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=128, half_band=cfg.w,
                     base_depth=cfg.T, tail_depth=3, epsilon=cfg.eps, dtype="bf16")
def go(poison_at):
    ws = band.Workspace()
    ws._buf = torch.zeros((64 << 20,), dtype=torch.uint8, device='cuda')
    def p(stage):
        if stage == poison_at: ws._buf.fill_(255)
    p(0); run = band.run_surrogate(t["Q"], t["K"], t["V"], spec, rm, cm, workspace=ws)
    p(1); cot = band.tail_adjoint(run, t["G"], workspace=ws)
    p(2); cq, ck = band.base_solve_vjp(run, cot.eta_v, cot.eta_u, workspace=ws)
    torch.cuda.synchronize()
    out = {"O": run.output, "dQ": cot.grad_q, "dK": cot.grad_k, "dV": cot.grad_v, "eta_v": cot.eta_v, "eta_u": cot.eta_u, "cQ": cq, "cK": ck}
    return {k: float(v.double().abs().sum()) for k, v in out.items()}
ref = go(-1)
print("clean", ref)
for st in (0, 1, 2):
    r = go(st)
    print("poison before stage", st, {k: (v if not np.isclose(v, ref[k], rtol=1e-6) else "=") for k, v in r.items()})
print("env", {k: v for k, v in os.environ.items() if k.startswith("ST_")})
