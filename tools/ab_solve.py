"""Dev helper: A/B of two solve paths (env switches) on one config -- outputs compared, forward timed.

    python tools/ab_solve.py CID L NHEADS "ENV_A" "ENV_B"     (ENV: comma list of NAME=VAL, or '-')
Each arm runs in a subprocess so that the library's getenv() switches take effect.
"""
import json, os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] == "--arm":
    import numpy as np, torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
    from paper_2605_08123_b200 import band, configs
    cid, L, nh, out = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    cfg = configs.CONFIGS[cid]
    if L: cfg = cfg.replace(L=L)
    inp = configs.make_inputs(cfg, heads=range(nh))
    spec = band.BandSpec(batch=nh, heads=1, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype)
    shp = (nh, 1, cfg.rows, cfg.d)
    b = inp.bits or {}
    dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b else torch.from_numpy(x)).cuda().reshape(shp)
    Q, K, V, G = dev(inp.Q, 'Q'), dev(inp.K, 'K'), dev(inp.V, 'V'), dev(inp.G, 'G')
    ws = band.Workspace()
    run = band.run_surrogate(Q, K, V, spec, workspace=ws, validate=False)
    cot = band.r2_backward(run, G, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); band.run_surrogate(Q, K, V, spec, workspace=ws, validate=False); e.record()
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    band.launch_count(reset=True)
    band.run_surrogate(Q, K, V, spec, workspace=ws, validate=False)
    nl = band.launch_count(reset=True)
    u, v, g = run.tail_duals()
    np.savez(out, O=run.output.cpu().numpy(), dQ=cot.grad_q.cpu().numpy(), dK=cot.grad_k.cpu().numpy(),
             dV=cot.grad_v.cpu().numpy(), u=u, v=v, fwd_ms=np.array(sorted(ts)[2]), launches=np.array(nl))
    sys.exit(0)

cid, L, nh = sys.argv[1], sys.argv[2], sys.argv[3]
res = {}
for tag, envs in (("A", sys.argv[4]), ("B", sys.argv[5])):
    env = dict(os.environ)
    if envs != "-":
        for kv in envs.split(","):
            k, v = kv.split("=")
            env[k] = v
    out = f"/tmp/ab_{tag}.npz"
    subprocess.run([sys.executable, __file__, "--arm", cid, L, nh, out], env=env, check=True)
    import numpy as np
    res[tag] = dict(np.load(out))
import numpy as np
rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
print(json.dumps({"config": cid, "L": L, "heads": nh,
                  "fwd_ms": {t: float(res[t]["fwd_ms"]) for t in res},
                  "launches": {t: int(res[t]["launches"]) for t in res},
                  "rel_B_vs_A": {k: rel(res["B"][k], res["A"][k]) for k in ("O", "dQ", "dK", "dV", "u", "v")}}))
