"""One small forward + backward for compute-sanitizer (tests/test_sanitizer.py).

    python tools/sanitize_case.py NAME
NAME: c1 (config 1), c2 (config 2 geometry, L=512, 2 heads, masked), c3 (dustbin, L=256,
2 heads), bf16 (config 4 geometry, L=8192 x 3 heads = 192 row blocks > 148 CTAs),
bf16w (config 5 geometry, L=2048, 2 heads: the half-step + window-chunked stages).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2605_08123_b200 import band, configs  # noqa: E402

CASES = {
    "c1": (1, {}, None),
    "c2": (2, {"L": 512, "T": 6}, 2),
    "c3": (3, {"L": 256, "T": 5}, 2),
    "bf16": (4, {"L": 8192, "T": 4}, 3),
    "bf16w": (5, {"L": 2048, "T": 4}, 2),
}


def main(name):
    cid, kw, nh = CASES[name]
    cfg = configs.CONFIGS[cid].replace(**kw)
    heads = range(nh if nh else cfg.B * cfg.H)
    inp = configs.make_inputs(cfg, heads=heads)
    n = len(heads)
    sel = np.array([h // cfg.H for h in heads])
    rm = None if inp.row_mask is None else torch.from_numpy(np.ascontiguousarray(inp.row_mask[sel])).cuda()
    spec = band.BandSpec(batch=n, heads=1, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w, base_depth=cfg.T,
                         tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin,
                         dustbin_cost=cfg.dustbin_cost)
    shp = (n, 1, cfg.rows, cfg.d)
    b = inp.bits or {}
    dev = lambda x, k: (torch.from_numpy(b[k].astype(np.int16)).view(torch.bfloat16) if k in b
                        else torch.from_numpy(x)).cuda().reshape(shp)
    Q, K, V, G = dev(inp.Q, "Q"), dev(inp.K, "K"), dev(inp.V, "V"), dev(inp.G, "G")
    run = band.run_surrogate(Q, K, V, spec, rm, rm)
    cot = band.r2_backward(run, G)
    torch.cuda.synchronize()
    assert torch.isfinite(run.output).all() and torch.isfinite(cot.grad_q).all()
    print(f"sanitize case {name}: ok")


if __name__ == "__main__":
    main(sys.argv[1])
