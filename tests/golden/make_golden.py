"""Generates the golden fixtures in this directory (TEST INFRASTRUCTURE).

Each case is a problem container ``<name>.stp`` in the reference's container format
(src/problem.cpp:47-137; Q, K, V from the reference generator, tags "Q"/"K"/"V", plus the linear
loss cotangent "G") and a result container ``<name>.result.stp`` holding the outputs of the
restated reference path (oracle/, f64: run_surrogate + r2_backward or tail_adjoint_generic).

Run from the repo root:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_ref  # noqa: E402
from paper_2605_08123_b200 import configs, problem  # noqa: E402

MODES = {"one_reference": 0, "direct_four_plan": 1, "generic_tail": 2}

# name: (InstanceSpec kwargs, valid rows, valid cols, mode)
CASES = {
    "banded_defaults": (dict(), None, None, "one_reference"),                       # problem.hpp defaults
    "rectangular": (dict(n_rows=40, n_cols=44, head_dim=8, half_band=9, base_depth=7, tail_depth=2,
                         epsilon=0.5, seed=99), None, None, "one_reference"),
    "masked_schedule": (dict(n_rows=160, n_cols=160, head_dim=32, half_band=20, base_depth=12, epsilon=0.25,
                             stages=[(1.0, 4), (0.5, 4), (0.25, 4)], seed=5), 150, 147, "one_reference"),
    "direct_four_plan": (dict(n_rows=96, n_cols=96, head_dim=16, half_band=12, base_depth=9, epsilon=0.4,
                              seed=11), None, None, "direct_four_plan"),
    "generic_R3": (dict(n_rows=96, n_cols=96, head_dim=32, half_band=16, base_depth=10, tail_depth=3,
                        epsilon=0.5, seed=7), None, None, "generic_tail"),
    "generic_R0": (dict(n_rows=64, n_cols=64, head_dim=32, half_band=10, base_depth=6, tail_depth=0,
                        epsilon=0.7, seed=13), None, None, "generic_tail"),
}


def build(name):
    kw, vr, vc, mode = CASES[name]
    spec = problem.InstanceSpec(**kw)
    rm = None if vr is None else np.arange(spec.n_rows) < vr
    cm = None if vc is None else np.arange(spec.n_cols) < vc
    return problem.make_instance(spec, rm, cm), mode


def reference_outputs(p, mode, precision=64):
    """The restated reference path on a container's buffers."""
    s = p.spec
    rm = None if p.support.row_mask.all() else p.support.row_mask.astype(np.uint8)[None]
    cm = None if p.support.col_mask.all() else p.support.col_mask.astype(np.uint8)[None]
    m = MODES[mode]
    G = p.extra["G"]
    if s.n_rows != s.n_cols:
        r = oracle_ref.run_rect(s.n_rows, s.n_cols, s.head_dim, s.half_band, s.final_epsilon(), s.base_depth,
                                s.tail_depth, p.Q[None], p.K[None], p.V[None], G[None], rm, cm,
                                precision=precision, mode=m)
    else:
        cfg = configs.Config(0, B=1, H=1, L=s.n_rows, d=s.head_dim, w=s.half_band, eps=s.final_epsilon(),
                             T=s.base_depth, R=s.tail_depth, dtype="f32")
        r = oracle_ref.run(cfg, p.Q[None], p.K[None], p.V[None], G[None], rm, cm, precision=precision, mode=m,
                           eps_schedule=s.eps_schedule())
    out = {k: np.asarray(r[k][0], dtype=np.float64) for k in ("O", "dQ", "dK", "dV", "eta_v")}
    return out, {"d_eps": float(r["d_eps"][0])}


def main():
    for name in CASES:
        p, mode = build(name)
        problem.save_problem(os.path.join(HERE, f"{name}.stp"), p)
        outs, sc = reference_outputs(p, mode)
        problem.save_result(os.path.join(HERE, f"{name}.result.stp"), outs, sc,
                            {"mode": mode, "oracle": "oracle/ f64", "case": name})
        print(name, {k: v.shape for k, v in outs.items()}, sc)


if __name__ == "__main__":
    main()
