"""Pin the restated oracle (oracle/, the parity checker) to the REFERENCE ITSELF.

* Live (when oracle/_ref/libref.so exists, i.e. this container with /root/reference):
  the reference's unmodified run_surrogate + r2_backward (compiled against the
  Eigen-API shim, oracle/Makefile target `ref`) and the oracle run the same seeded
  inputs; double precision must agree to rounding (<= 1e-11 rel-L2; the dustbin
  embedding trick's ill-conditioned dQ to 1e-10), float to within the reference's
  own f32 noise floor.
* Fixtures (always): tests/golden/ref_*.npz hold the reference's own f64 outputs
  (tests/golden/make_ref_golden.py); the oracle must reproduce them.
"""
import glob
import os

import numpy as np
import pytest

import oracle_ref

W = oracle_ref.load_configs()
KEYS = ("O", "dQ", "dK", "dV", "eta_v")
HERE = os.path.dirname(os.path.abspath(__file__))
needs_ref = pytest.mark.skipif(not oracle_ref.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


CASES = [(1, {}, 1), (2, {"L": 512}, 2), (3, {"L": 256}, 2), (4, {"L": 1024}, 1), (5, {"L": 1024}, 1),
         (0, dict(B=1, H=1, L=1, d=4, w=0, eps=1.0, T=3, R=2, dtype="f32"), 1),
         (0, dict(B=2, H=1, L=37, d=8, w=40, eps=0.5, T=6, R=2, dtype="f32"), 2),
         (0, dict(B=2, H=2, L=130, d=16, w=9, eps=0.3, T=0, R=2, dtype="f32", mask="uniform_len"), 4),
         (0, dict(B=2, H=1, L=64, d=8, w=3, eps=0.5, T=5, R=2, dtype="f32", mask="lognormal_len", dustbin=1,
                  dustbin_cost=0.7, embed="alphabet"), 2)]


def _cfg(cid, kw):
    return W.CONFIGS[cid].replace(**kw) if cid else W.Config(0, **kw)


@needs_ref
@pytest.mark.parametrize("cid,kw,nh", CASES)
@pytest.mark.parametrize("mode", [0, 1])
def test_oracle_matches_reference_f64(cid, kw, nh, mode):
    cfg = _cfg(cid, kw)
    inp = W.make_inputs(cfg, heads=range(nh))
    args = (cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask)
    a = oracle_ref.run(*args, heads=inp.heads, precision=64, mode=mode)
    b = oracle_ref.run_reference(*args, heads=inp.heads, precision=64, mode=mode)
    for k in KEYS + ("duals", "gauges"):
        bound = 1e-10 if cfg.dustbin else 1e-11
        assert rel(a[k], b[k]) <= bound, (k, rel(a[k], b[k]))


@needs_ref
def test_oracle_matches_reference_eps_schedule():
    cfg = W.CONFIGS[2].replace(L=384)
    inp = W.make_inputs(cfg, heads=range(2))
    sched = [(0.2, 10), (0.1, 15), (0.05, 25)]
    args = (cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask)
    a = oracle_ref.run(*args, heads=inp.heads, eps_schedule=sched)
    b = oracle_ref.run_reference(*args, heads=inp.heads, eps_schedule=sched)
    for k in KEYS + ("duals", "gauges"):
        assert rel(a[k], b[k]) <= 1e-11, (k, rel(a[k], b[k]))


@needs_ref
@pytest.mark.parametrize("cid,kw,nh", CASES[:5])
def test_oracle_f32_matches_reference_f32(cid, kw, nh):
    """The float instantiations differ only in summation order (Eigen GEMM vs loops): within the
    reference's own f32-vs-f64 floor."""
    cfg = _cfg(cid, kw)
    inp = W.make_inputs(cfg, heads=range(nh))
    args = (cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask)
    a = oracle_ref.run(*args, heads=inp.heads, precision=32)
    b = oracle_ref.run_reference(*args, heads=inp.heads, precision=32)
    c = oracle_ref.run_reference(*args, heads=inp.heads, precision=64)
    for k in KEYS:
        assert rel(a[k], b[k]) <= max(1e-6, 2.5 * rel(b[k], c[k])), (k, rel(a[k], b[k]), rel(b[k], c[k]))


def _fixtures():
    return sorted(glob.glob(os.path.join(HERE, "golden", "ref_config*.npz")))


def load_fixture(path):
    z = np.load(path)
    cid = int(os.path.basename(path).split("config")[1][0])
    cfg = W.CONFIGS[cid].replace(L=int(z["L"]))
    inp = W.make_inputs(cfg, heads=range(len(z["heads"])))
    return cfg, inp, z


def test_reference_fixtures_exist():
    assert len(_fixtures()) == 5


@pytest.mark.parametrize("path", _fixtures(), ids=os.path.basename)
def test_oracle_reproduces_reference_fixtures(path):
    cfg, inp, z = load_fixture(path)
    r = oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, heads=inp.heads, precision=64)
    for k in KEYS + ("duals", "gauges"):
        bound = 1e-10 if cfg.dustbin else 1e-11
        assert rel(r[k], z[k]) <= bound, (k, rel(r[k], z[k]))
