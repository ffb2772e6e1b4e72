"""CPU-side checks of the C-ABI library: loads, exports every declared symbol,
bit-exact RNG against the oracle, host validation and error contract (no kernels run)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle_ref
from paper_2605_08123_b200 import _lib, band, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sinkattn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


@pytest.mark.parametrize("tag,start,n,scale", [("Q", 0, 1000, 1.0), ("G", 123456789, 777, 0.5), ("dustbin_v", 5, 64, 1.0)])
def test_rng_bit_exact_with_reference_generator(tag, start, n, scale):
    a = configs.normal_fill(7, tag, start, n, scale)
    b = oracle_ref.normal_fill(7, tag, start, n, scale)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_rng_flat_index_identity():
    # test_io.cpp:68-81: entry (i, j) of a wider draw equals the same flat index
    a = configs.normal_fill(5, "Q", 0, 32).reshape(8, 4)
    wide = configs.normal_fill(5, "Q", 0, 32).reshape(4, 8)
    assert wide[0, 5] == a[1, 1]


def _spec(**kw):
    base = dict(batch=1, heads=1, seq_q=8, seq_k=8, head_dim=4, half_band=1, base_depth=3, tail_depth=2,
                epsilon=1.0)
    base.update(kw)
    return band.BandSpec(**base)


def test_validate_support_matches_reference_cases():
    # test_support.cpp:72-79
    band.validate_support(_spec(seq_q=3, seq_k=3, half_band=0), None, None)
    with pytest.raises(band.InfeasibleSupport):
        band.validate_support(_spec(seq_q=3, seq_k=3, half_band=0), None, np.array([[0, 1, 1]], np.uint8))
    with pytest.raises(band.InfeasibleSupport):
        band.validate_support(_spec(seq_q=3, seq_k=3, half_band=0), np.array([[1, 1, 0]], np.uint8), None)
    # rectangular: half band 2 leaves far columns unreachable (test_support.cpp:47-54)
    with pytest.raises(band.InfeasibleSupport):
        band.validate_support(_spec(seq_q=4, seq_k=7, half_band=2), None, None)
    band.validate_support(_spec(seq_q=4, seq_k=7, half_band=3), None, None)
    # the dustbin spoke makes every active row/col feasible
    band.validate_support(_spec(seq_q=3, seq_k=3, half_band=0, dustbin=1), None, np.array([[0, 1, 1]], np.uint8))


def _status(fn, *args):
    return fn(*args)


def test_error_contract_without_gpu():
    lib = _lib.lib
    d = _spec(epsilon=0.0).desc()
    assert lib.st_forward(ctypes.byref(d), 1, 1, 1, None, None, 1, None, None, 0, None) == _lib.ST_INVALID_TEMPERATURE
    d = _spec(tail_depth=1).desc()
    assert lib.st_backward(ctypes.byref(d), 1, 1, 1, 1, 1, None, None, 1, 1, 1, None, None, 0, None, 0,
                           None) == _lib.ST_UNSUPPORTED_DEPTH
    # the generic tail adjoint (mode 2) takes any depth up to 8, no dustbin
    for R, want in ((1, _lib.ST_MISSING_BASE_TRACE), (9, _lib.ST_UNSUPPORTED_DEPTH)):
        d = _spec(tail_depth=R).desc()
        assert lib.st_backward(ctypes.byref(d), None, 1, 1, 1, 1, None, None, 1, 1, 1, None, None,
                               _lib.ST_GENERIC_TAIL, None, 0, None) == want, R
    d = _spec(dustbin=1).desc()
    assert lib.st_backward(ctypes.byref(d), 1, 1, 1, 1, 1, None, None, 1, 1, 1, None, None,
                           _lib.ST_GENERIC_TAIL, None, 0, None) == _lib.ST_NOT_SUPPORTED
    d = _spec().desc()
    assert lib.st_backward(ctypes.byref(d), 1, 1, 1, 1, 1, None, None, 1, 1, 1, None, None, 7, None, 0,
                           None) == _lib.ST_INVALID_ARGUMENT
    assert lib.st_backward(ctypes.byref(d), None, 1, 1, 1, 1, None, None, 1, 1, 1, None, None, 0, None, 0,
                           None) == _lib.ST_MISSING_BASE_TRACE
    assert lib.st_forward(ctypes.byref(d), 1, 1, 1, None, None, 1, None, None, 0, None) == _lib.ST_WORKSPACE_TOO_SMALL
    d = _spec(head_dim=256).desc()
    assert lib.st_forward(ctypes.byref(d), 1, 1, 1, None, None, 1, None, None, 0, None) == _lib.ST_NOT_SUPPORTED
    # band-free bf16 problems: the generic tail adjoint needs the stored-band kernels (ST_FLAG_STORED_BAND)
    bf = dict(batch=1, heads=1, seq_q=512, seq_k=512, head_dim=64, half_band=128, dtype="bf16")
    d = _spec(**bf).desc()
    assert lib.st_backward(ctypes.byref(d), 1, 1, 1, 1, 1, None, None, 1, 1, 1, None, None,
                           _lib.ST_GENERIC_TAIL, None, 0, None) == _lib.ST_NOT_SUPPORTED
    assert b"ST_FLAG_STORED_BAND" in lib.st_last_error()
    d = _spec(stored_band=True, **bf).desc()
    assert lib.st_backward(ctypes.byref(d), 1, 1, 1, 1, 1, None, None, 1, 1, 1, None, None,
                           _lib.ST_GENERIC_TAIL, None, 0, None) == _lib.ST_WORKSPACE_TOO_SMALL
    d = _spec(seq_q=0).desc()
    assert lib.st_workspace_bytes(ctypes.byref(d)) == 0
    assert b"dimensions" in lib.st_last_error() or lib.st_last_error() != b""


def test_saved_state_is_O_of_L():
    s = _spec(batch=8, heads=4, seq_q=2048, seq_k=2048, head_dim=64, half_band=64)
    # 6 vectors of L per head + gauges: never the L x W plan
    assert s.saved_bytes() < 8 * 4 * (6 * 2048 * 4 + 4096)
    assert s.workspace_bytes() >= 8 * 4 * 2048 * 129 * 4  # fp32 keeps its exact f64-DMMA score band


def test_bf16_workspace_holds_no_band():
    """BASELINE configs 4 / 5 run band-free: the workspace is O(L d) packed planes + O(L) vectors, far
    below one L x W fp32 band (which ST_FLAG_STORED_BAND brings back for the stored-band kernels)."""
    for B, H, L, d, w in ((4, 8, 32768, 128, 128), (1, 16, 131072, 64, 256)):
        s = _spec(batch=B, heads=H, seq_q=L, seq_k=L, head_dim=d, half_band=w, dtype="bf16")
        band_bytes = B * H * L * (2 * w + 1) * 4
        planes = 4 * B * H * L * d * 2
        assert s.workspace_bytes() < planes + B * H * L * 4 * 48, (s.workspace_bytes(), planes)
        import dataclasses
        stored = dataclasses.replace(s, stored_band=True).workspace_bytes()
        assert stored > 4 * band_bytes  # S2, S2T, Z, ZT
        assert s.workspace_bytes() < stored / (4 if d == 128 else 12)


def test_config_table_matches_baseline():
    c = configs.CONFIGS
    assert (c[1].B, c[1].H, c[1].L, c[1].d, c[1].Wf, c[1].eps, c[1].T, c[1].R) == (1, 1, 256, 32, 33, 0.1, 20, 2)
    assert (c[2].B, c[2].H, c[2].L, c[2].d, c[2].Wf, c[2].eps, c[2].T) == (8, 4, 2048, 64, 129, 0.05, 50)
    assert (c[3].B, c[3].H, c[3].L, c[3].d, c[3].Wf, c[3].eps, c[3].T, c[3].dustbin) == (16, 8, 1024, 64, 65, 0.1, 30, 1)
    assert (c[4].B, c[4].H, c[4].L, c[4].d, c[4].Wf, c[4].eps, c[4].T, c[4].dtype) == (4, 8, 32768, 128, 257, 0.05, 100, "bf16")
    assert (c[5].B, c[5].H, c[5].L, c[5].d, c[5].Wf, c[5].eps, c[5].T, c[5].dtype) == (1, 16, 131072, 64, 513, 0.05, 50, "bf16")
    ls = configs.lengths(c[2])
    assert ls.min() >= 1024 and ls.max() <= 2048
    l3 = configs.lengths(c[3])
    assert l3.min() >= 64 and l3.max() <= 1024


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.0000001, 3.14159265], dtype=np.float64)
    bits = configs.to_bf16_bits(x)
    back = configs.bf16_bits_to_f32(bits)
    assert back[0] == 1.0 and back[1] == 1.0  # tie to even
    assert back[2] == 1.0078125
    assert abs(back[4] - 3.140625) < 1e-7


def test_eps_schedule_validation():
    """EpsSchedule::validate (trace.hpp:37-49) through the C-ABI, before any device work."""
    def desc(stages):
        return band.BandSpec(batch=1, heads=1, seq_q=8, seq_k=8, head_dim=4, half_band=1, base_depth=4,
                             epsilon=0.5, eps_schedule=stages).desc()
    def fwd(d):
        return _lib.lib.st_forward(ctypes.byref(d), None, None, None, None, None, None, None, None, 0, None)
    assert fwd(desc([(1.0, 2), (2.0, 2)])) == _lib.ST_INVALID_TEMPERATURE       # increasing temperature
    assert fwd(desc([(1.0, 2), (-0.5, 2)])) == _lib.ST_INVALID_TEMPERATURE      # non-positive
    assert fwd(desc([(1.0, 2), (0.5, 1)])) == _lib.ST_INVALID_ARGUMENT          # iterations != T
    assert fwd(desc([(1.0, 2), (0.25, 2)])) == _lib.ST_INVALID_ARGUMENT         # last stage != epsilon
    assert fwd(desc([(1.0, 2), (0.5, 2)])) == _lib.ST_INVALID_ARGUMENT          # valid schedule, null tensors
