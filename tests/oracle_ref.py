"""ctypes access to the CPU oracle (oracle/build/libstoc.so) -- the checker.

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never by the product.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "build", "libstoc.so")
KAT = os.path.join(ORACLE_DIR, "build", "kat_tests")


def build() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        D = ctypes.POINTER(ctypes.c_double)
        U8 = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.stoc_run_batch.argtypes = [I64, I64, I64, I64, I64, I64, I64, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_double, D, D, D, D, U8, U8, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, I64, I64, D, D, D, D, D, D, D, D]
        L.stoc_run_batch.restype = ctypes.c_int
        L.stoc_run_batch_sched.argtypes = L.stoc_run_batch.argtypes + [ctypes.c_int, D, ctypes.POINTER(I64)]
        L.stoc_run_batch_sched.restype = ctypes.c_int
        L.stoc_normal_fill.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64, I64, ctypes.c_double, D]
        L.stoc_normal_fill.restype = None
        L.stoc_uniform_fill.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64, I64, D]
        L.stoc_uniform_fill.restype = None
        L.stoc_last_error.restype = ctypes.c_char_p
        L.stoc_banded_entry_count.argtypes = [I64, I64]
        L.stoc_banded_entry_count.restype = I64
        _lib = L
    return _lib


def normal_fill(seed, tag, start, n, scale=1.0):
    out = np.empty(n, dtype=np.float64)
    lib().stoc_normal_fill(seed, tag.encode(), start, n, scale, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def uniform_fill(seed, tag, start, n):
    out = np.empty(n, dtype=np.float64)
    lib().stoc_uniform_fill(seed, tag.encode(), start, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def load_configs():
    """The workload table (paper_2605_08123_b200/configs.py) loaded BY PATH with the oracle's RNG
    fills installed, so a caller that must not map the product library (bench.py --impl reference)
    never imports the package."""
    import importlib.util
    path = os.path.join(ROOT, "paper_2605_08123_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("st_workloads", path)
    mod = importlib.util.module_from_spec(spec)
    import sys
    sys.modules["st_workloads"] = mod  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    mod.set_rng_backend(normal_fill, uniform_fill)
    return mod


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def run(cfg, Q, K, V, G, row_mask=None, col_mask=None, *, heads=None, precision=64, mode=0, backward=True,
        threads=None, tile_block=128, centered=True, eps_schedule=None):
    """Reference path per head: run_surrogate + r2_backward (inc/validation.hpp:102-114).

    Q, K, V, G: [nh, L', d] arrays of the heads `heads` (global b*H+h indices,
    default 0..nh-1; any float dtype, upcast exactly to double).
    row_mask/col_mask: [B, L] uint8 of the whole batch.  Returns float64 arrays.
    """
    Q, K, V, G = (np.ascontiguousarray(x, dtype=np.float64) for x in (Q, K, V, G))
    nh, Lr, d = Q.shape
    heads = range(nh) if heads is None else heads
    Lreal = cfg.L
    # one pseudo-example per head so that any head subset maps onto its own mask row
    Hh, Bb = 1, nh
    sel = np.array([h // cfg.H for h in heads], dtype=np.int64)
    if row_mask is not None:
        row_mask = np.asarray(row_mask)[sel]
    if col_mask is not None:
        col_mask = np.asarray(col_mask)[sel]
    out = {k: np.zeros_like(Q) for k in ("O", "dQ", "dK", "dV")}
    out["d_eps"] = np.zeros(nh)
    out["eta_v"] = np.zeros((nh, Lr))
    out["duals"] = np.zeros((nh, 6, Lr))
    out["gauges"] = np.zeros((nh, 3))
    P = ctypes.POINTER(ctypes.c_double)
    p = lambda a: a.ctypes.data_as(P)
    rm = None if row_mask is None else np.ascontiguousarray(row_mask, dtype=np.uint8)
    cm = None if col_mask is None else np.ascontiguousarray(col_mask, dtype=np.uint8)
    # eps_schedule: [(epsilon, iterations), ...] base-solve stages (EpsSchedule, trace.hpp:12-50)
    se = None if not eps_schedule else np.array([e for e, _ in eps_schedule], dtype=np.float64)
    si = None if not eps_schedule else np.array([n for _, n in eps_schedule], dtype=np.int64)
    code = lib().stoc_run_batch_sched(
        Bb, Hh, Lreal, d, cfg.w, cfg.T, cfg.R, cfg.eps, cfg.dustbin, cfg.dustbin_cost,
        p(Q), p(K), p(V), p(G), None if rm is None else rm.ctypes.data, None if cm is None else cm.ctypes.data,
        precision, mode, tile_block, 1 if centered else 0, threads or os.cpu_count() or 1, 0, nh,
        p(out["O"]), p(out["dQ"]) if backward else None, p(out["dK"]), p(out["dV"]), p(out["d_eps"]),
        p(out["eta_v"]), p(out["duals"]), p(out["gauges"]), 0 if se is None else len(se),
        None if se is None else p(se), None if si is None else si.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if code != 0:
        raise OracleError(code, lib().stoc_last_error().decode())
    return out


def run_rect(Lq, Lk, d, w, eps, T, R, Q, K, V, G, row_mask=None, col_mask=None, precision=64, mode=0):
    """Rectangular problems (L_q != L_k, no dustbin; build_band_support(Lq, Lk, ...), support.cpp:111):
    Q, G [nh, Lq, d]; K, V [nh, Lk, d]; masks [nh, L] (one pseudo-example per head)."""
    L_ = lib()
    if not hasattr(L_, "_rect"):
        D = ctypes.POINTER(ctypes.c_double)
        I64 = ctypes.c_int64
        L_.stoc_run_batch_rect.argtypes = [I64, I64, I64, I64, I64, I64, I64, I64, ctypes.c_double, D, D, D, D,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, D, D, D, D, D, D]
        L_.stoc_run_batch_rect.restype = ctypes.c_int
        L_._rect = True
    Q, K, V, G = (np.ascontiguousarray(x, dtype=np.float64) for x in (Q, K, V, G))
    nh = Q.shape[0]
    out = {"O": np.zeros_like(Q), "dQ": np.zeros_like(Q), "dK": np.zeros_like(K), "dV": np.zeros_like(K),
           "d_eps": np.zeros(nh), "eta_v": np.zeros((nh, Lk))}
    P = ctypes.POINTER(ctypes.c_double)
    p = lambda a: a.ctypes.data_as(P)
    rm = None if row_mask is None else np.ascontiguousarray(row_mask, dtype=np.uint8)
    cm = None if col_mask is None else np.ascontiguousarray(col_mask, dtype=np.uint8)
    code = L_.stoc_run_batch_rect(nh, 1, Lq, Lk, d, w, T, R, eps, p(Q), p(K), p(V), p(G),
                                  None if rm is None else rm.ctypes.data, None if cm is None else cm.ctypes.data,
                                  precision, mode, os.cpu_count() or 1, p(out["O"]), p(out["dQ"]), p(out["dK"]),
                                  p(out["dV"]), p(out["d_eps"]), p(out["eta_v"]))
    if code != 0:
        raise OracleError(code, lib().stoc_last_error().decode())
    return out


def run_cert(cfg, Q, K, V, G, row_mask=None, col_mask=None, *, heads=None, precision=64, eps_schedule=None):
    """Generic tail adjoint + base_solve_vjp of its base cotangent per head (the bias certificate's
    c_R = (cQ, cK), certificates.hpp:112-118).  Q, K, V, G: [nh, L, d] (no dustbin); masks [B, L]."""
    L_ = lib()
    if not hasattr(L_, "_cert"):
        D = ctypes.POINTER(ctypes.c_double)
        I64 = ctypes.c_int64
        L_.stoc_run_batch_cert.argtypes = [I64, I64, I64, I64, I64, I64, I64, ctypes.c_double, D, D, D, D,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, D, D, D, D, D, D, D, D, D]
        L_.stoc_run_batch_cert.restype = ctypes.c_int
        L_._cert = True
    Q, K, V, G = (np.ascontiguousarray(x, dtype=np.float64) for x in (Q, K, V, G))
    nh, Lr, d = Q.shape
    heads = range(nh) if heads is None else heads
    sel = np.array([h // cfg.H for h in heads], dtype=np.int64)
    rm = None if row_mask is None else np.ascontiguousarray(np.asarray(row_mask)[sel], dtype=np.uint8)
    cm = None if col_mask is None else np.ascontiguousarray(np.asarray(col_mask)[sel], dtype=np.uint8)
    out = {k: np.zeros_like(Q) for k in ("O", "dQ", "dK", "dV", "cQ", "cK")}
    out["d_eps"] = np.zeros(nh)
    out["eta_v"] = np.zeros((nh, Lr))
    out["eta_u"] = np.zeros((nh, Lr))
    se = None if not eps_schedule else np.array([e for e, _ in eps_schedule], dtype=np.float64)
    si = None if not eps_schedule else np.array([n for _, n in eps_schedule], dtype=np.int64)
    P = ctypes.POINTER(ctypes.c_double)
    p = lambda a: a.ctypes.data_as(P)
    code = L_.stoc_run_batch_cert(nh, 1, cfg.L, d, cfg.w, cfg.T, cfg.R, cfg.eps, p(Q), p(K), p(V), p(G),
                                  None if rm is None else rm.ctypes.data, None if cm is None else cm.ctypes.data,
                                  precision, os.cpu_count() or 1, 0 if se is None else len(se),
                                  None if se is None else se.ctypes.data, None if si is None else si.ctypes.data,
                                  p(out["O"]), p(out["dQ"]), p(out["dK"]), p(out["dV"]), p(out["d_eps"]),
                                  p(out["eta_u"]), p(out["eta_v"]), p(out["cQ"]), p(out["cK"]))
    if code != 0:
        raise OracleError(code, lib().stoc_last_error().decode())
    return out


# ---------------------------------------------------------------------------
# oracle/_ref/libref.so: the reference ITSELF (its unmodified headers and
# src/support.cpp compiled against oracle/ref_shim), used to pin the restatement.
# ---------------------------------------------------------------------------
REF_LIB = os.path.join(ORACLE_DIR, "_ref", "libref.so")
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib():
    global _ref
    if _ref is None:
        L = ctypes.CDLL(REF_LIB)
        D = ctypes.POINTER(ctypes.c_double)
        I64 = ctypes.c_int64
        L.refc_run.argtypes = [I64, I64, I64, I64, I64, I64, I64, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                               D, D, D, D, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, D, ctypes.POINTER(I64), D, D, D, D, D, D, D]
        L.refc_run.restype = ctypes.c_int
        L.refc_last_error.restype = ctypes.c_char_p
        _ref = L
    return _ref


def run_reference(cfg, Q, K, V, G, row_mask=None, col_mask=None, *, heads=None, precision=64, mode=0,
                  backward=True, threads=None, tile_block=128, centered=True, eps_schedule=None):
    """The reference's own run_surrogate + r2_backward per head (oracle/_ref); same arguments and
    outputs as run() except d_eps (not a reference quantity)."""
    Q, K, V, G = (np.ascontiguousarray(x, dtype=np.float64) for x in (Q, K, V, G))
    nh, Lr, d = Q.shape
    heads = range(nh) if heads is None else heads
    sel = np.array([h // cfg.H for h in heads], dtype=np.int64)
    rm = None if row_mask is None else np.ascontiguousarray(np.asarray(row_mask)[sel], dtype=np.uint8)
    cm = None if col_mask is None else np.ascontiguousarray(np.asarray(col_mask)[sel], dtype=np.uint8)
    out = {k: np.zeros_like(Q) for k in ("O", "dQ", "dK", "dV")}
    out["eta_v"] = np.zeros((nh, Lr))
    out["duals"] = np.zeros((nh, 6, Lr))
    out["gauges"] = np.zeros((nh, 3))
    se = None if not eps_schedule else np.array([e for e, _ in eps_schedule], dtype=np.float64)
    si = None if not eps_schedule else np.array([n for _, n in eps_schedule], dtype=np.int64)
    P = ctypes.POINTER(ctypes.c_double)
    p = lambda a: a.ctypes.data_as(P)
    code = ref_lib().refc_run(
        nh, cfg.L, cfg.L, d, cfg.w, cfg.T, cfg.R, cfg.eps, cfg.dustbin, cfg.dustbin_cost,
        p(Q), p(K), p(V), p(G), None if rm is None else rm.ctypes.data, None if cm is None else cm.ctypes.data,
        precision, mode, tile_block, 1 if centered else 0, threads or os.cpu_count() or 1,
        0 if se is None else len(se), None if se is None else p(se),
        None if si is None else si.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        p(out["O"]), p(out["dQ"]) if backward else None, p(out["dK"]), p(out["dV"]), p(out["eta_v"]),
        p(out["duals"]), p(out["gauges"]))
    if code != 0:
        raise OracleError(code, ref_lib().refc_last_error().decode())
    return out
