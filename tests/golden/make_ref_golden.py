"""Golden vectors from the REFERENCE ITSELF (oracle/_ref/libref.so: the unmodified
/root/reference headers + src/support.cpp compiled against oracle/ref_shim).

    python tests/golden/make_ref_golden.py      # needs /root/reference (this container)

For each config: a seeded head subset at a reduced length (full d, band, eps, T, R,
dtype, mask recipe), the reference's double-precision run_surrogate + r2_backward
(OneReference) outputs O, dQ, dK, dV, eta (= v-bar^(0)) and its centered tail
duals, plus the rel-L2 of the reference's own float instantiation against them
(the f32 noise floor).  Inputs are NOT stored: they regenerate bit-exactly from
the counter RNG (configs.make_inputs, seed 0).  The fixtures pin the restated
oracle on machines without /root/reference and the GPU path on the B200 box.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_ref  # noqa: E402

# (config, length override, heads)
CASES = [(1, None, 1), (2, 320, 1), (3, 160, 1), (4, 384, 1), (5, 640, 1)]
KEYS = ("O", "dQ", "dK", "dV", "eta_v")


def case_name(cid, L):
    return f"ref_config{cid}" + ("" if L is None else f"_L{L}")


def main():
    W = oracle_ref.load_configs()
    for cid, L, nh in CASES:
        cfg = W.CONFIGS[cid] if L is None else W.CONFIGS[cid].replace(L=L)
        inp = W.make_inputs(cfg, heads=range(nh))
        args = (cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask)
        r64 = oracle_ref.run_reference(*args, heads=inp.heads, precision=64)
        r32 = oracle_ref.run_reference(*args, heads=inp.heads, precision=32)
        floor = {k: np.linalg.norm(r32[k] - r64[k]) / np.linalg.norm(r64[k]) for k in KEYS}
        out = {k: r64[k] for k in KEYS}
        out.update(duals=r64["duals"], gauges=r64["gauges"], L=cfg.L, heads=np.arange(nh),
                   floor=np.array([floor[k] for k in KEYS]), keys=np.array(KEYS))
        path = os.path.join(HERE, case_name(cid, L) + ".npz")
        np.savez_compressed(path, **out)
        print(path, os.path.getsize(path), {k: f"{v:.1e}" for k, v in floor.items()})


if __name__ == "__main__":
    main()
