"""The reference's own known-answer tests, ported onto the CPU oracle (oracle/kat_tests.cpp)."""
import os
import subprocess

import numpy as np
import pytest

import oracle_ref


def test_oracle_known_answer_suite():
    oracle_ref.build()
    r = subprocess.run([oracle_ref.KAT], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert " 0 failures" in r.stdout


def test_oracle_band_count_pin():
    # test_support.cpp:56-60 / PAPER Table 5: 32,521,216 entries at L=16384, W=1024
    assert oracle_ref.lib().stoc_banded_entry_count(16384, 1024) == 32521216


def test_oracle_f32_tracks_f64_on_config1():
    """Noise floor of the reference's own f32 template vs f64 on config 1 (reported in DESIGN.md)."""
    from paper_2605_08123_b200 import configs
    cfg = configs.CONFIGS[1]
    inp = configs.make_inputs(cfg)
    r64 = oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, precision=64)
    r32 = oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, precision=32)
    for k in ("O", "dQ", "dK", "dV"):
        rel = np.linalg.norm(r32[k] - r64[k]) / np.linalg.norm(r64[k])
        assert rel < 1e-4, (k, rel)
