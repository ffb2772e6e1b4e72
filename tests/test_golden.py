"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py): problem containers in the
reference's format (src/problem.cpp:47-137) with the restated reference path's f64 outputs.

CPU: the container / spec round trips of the reference's test_io.cpp, the seeded generator
reproducing the stored inputs bit-exactly, and the oracle reproducing the stored outputs.
GPU: the device path on every fixture against the stored outputs."""
import glob
import json
import os
import struct

import numpy as np
import pytest

import oracle_ref
from paper_2605_08123_b200 import problem

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.stp")) if not p.endswith(".result.stp"))


def _golden():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_fixtures_present():
    assert set(NAMES) == set(_golden().CASES), NAMES


def test_instance_spec_json_round_trip():
    """test_io.cpp:11-36."""
    s = problem.InstanceSpec(n_rows=40, n_cols=44, head_dim=6, half_band=9, base_depth=7, tail_depth=3, epsilon=0.5,
                             stages=[(2.0, 3), (0.5, 4)], seed=99, dustbin_block=5, tile_block=16)
    assert problem.InstanceSpec.from_json(json.loads(json.dumps(s.to_json()))) == s
    assert set(s.to_json()) == {"L_q", "L_k", "d", "W", "T", "R", "epsilon", "schedule", "seed", "dustbin_block",
                                "tile_block"}


def test_container_round_trip_is_bit_exact(tmp_path):
    """test_io.cpp:38-65, plus a masked support and an explicit edge list."""
    spec = problem.InstanceSpec(n_rows=24, n_cols=24, half_band=6, seed=3)
    p = problem.make_instance(spec, np.arange(24) < 20, np.arange(24) != 3)
    path = str(tmp_path / "c.stp")
    problem.save_problem(path, p)
    back = problem.load_problem(path)
    assert back.spec == spec
    for k in ("Q", "K", "V"):
        assert np.array_equal(getattr(back, k), getattr(p, k))
    assert np.array_equal(back.extra["G"], p.extra["G"])
    assert all(back.support.contains(i, j) == p.support.contains(i, j) for i in range(24) for j in range(24))
    e = problem.Support("explicit", 3, 3, 0, np.ones(3, bool), np.ones(3, bool), 0, np.array([[0, 1], [2, 2]]))
    p2 = problem.ProblemContainer(spec, e, p.Q, p.K, p.V)
    problem.save_problem(path, p2)
    b2 = problem.load_problem(path)
    assert b2.support.contains(0, 1) and b2.support.contains(2, 2) and not b2.support.contains(1, 1)
    # the layout the reference loader reads: magic, u64 header length, JSON header, f64 payload
    raw = open(path, "rb").read()
    assert raw[:8] == b"STPC0001"
    (hlen,) = struct.unpack("<Q", raw[8:16])
    hdr = json.loads(raw[16:16 + hlen])
    assert hdr["container"] == "sinktail-problem/1" and [b["name"] for b in hdr["buffers"]][:3] == ["Q", "K", "V"]
    with pytest.raises(ValueError):
        problem.load_result(path)


@pytest.mark.parametrize("name", NAMES)
def test_fixture_inputs_regenerate_bit_exactly(name):
    g = _golden()
    p, _ = g.build(name)
    stored = problem.load_problem(os.path.join(HERE, f"{name}.stp"))
    assert stored.spec == p.spec
    for k in ("Q", "K", "V"):
        assert np.array_equal(getattr(stored, k), getattr(p, k)), k
    assert np.array_equal(stored.extra["G"], p.extra["G"])
    assert np.array_equal(stored.support.row_mask, p.support.row_mask)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_fixture_outputs(name):
    g = _golden()
    p = problem.load_problem(os.path.join(HERE, f"{name}.stp"))
    outs, sc, meta = problem.load_result(os.path.join(HERE, f"{name}.result.stp"))
    got, gsc = g.reference_outputs(p, meta["mode"])
    for k, v in outs.items():
        assert rel(got[k].reshape(v.shape), v) < 1e-12, k
    assert abs(gsc["d_eps"] - sc["d_eps"]) <= 1e-10 * max(1.0, abs(sc["d_eps"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_path_matches_fixture(name):
    g = _golden()
    p = problem.load_problem(os.path.join(HERE, f"{name}.stp"))
    outs, sc, meta = problem.load_result(os.path.join(HERE, f"{name}.result.stp"))
    got = problem.run_problem(p, meta["mode"])
    ref32, sc32 = g.reference_outputs(p, meta["mode"], precision=32)
    for k, v in outs.items():
        e, fl = rel(got[k].reshape(v.shape), v), rel(ref32[k].reshape(v.shape), v)
        assert e <= max(1e-5, 1.5 * fl), (name, k, e, fl)
    de, fl = abs(got["d_eps"][0] - sc["d_eps"]), abs(sc32["d_eps"] - sc["d_eps"])
    assert de <= max(1e-4 * max(1.0, abs(sc["d_eps"])), 3.0 * fl), (de, fl)
