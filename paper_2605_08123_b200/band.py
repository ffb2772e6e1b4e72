"""Host-side mirror of the reference's entry points for this path.

    run_surrogate(Q, K, V, ...)      <- sinktail::run_surrogate   (include/sinktail/sinkhorn.hpp:288-302)
    r2_backward(run, G, mode=...)    <- sinktail::r2_backward     (include/sinktail/adjoint.hpp:232-373)
    build_band_support semantics     <- src/support.cpp:111-117 (masks + validate)

Same names, argument meaning and error behaviour (the reference's exception
types, include/sinktail/errors.hpp:10-39).  Tensors are torch CUDA tensors laid
out [B, H, L', d]; every call goes through the C-ABI of libsinkattn.so on the
current torch stream.  PyTorch only supplies device memory and the stream.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import lib


class SinkattnError(RuntimeError):
    pass


class InfeasibleSupport(SinkattnError):
    pass


class InvalidTemperature(SinkattnError):
    pass


class UnsupportedDepth(SinkattnError):
    pass


class MissingBaseTrace(SinkattnError):
    pass


class SizeCapExceeded(SinkattnError):
    pass


class CudaError(SinkattnError):
    pass


_STATUS = {
    _lib.ST_INVALID_ARGUMENT: ValueError,
    _lib.ST_INFEASIBLE_SUPPORT: InfeasibleSupport,
    _lib.ST_INVALID_TEMPERATURE: InvalidTemperature,
    _lib.ST_UNSUPPORTED_DEPTH: UnsupportedDepth,
    _lib.ST_MISSING_BASE_TRACE: MissingBaseTrace,
    _lib.ST_SIZE_CAP_EXCEEDED: SizeCapExceeded,
    _lib.ST_CUDA_ERROR: CudaError,
    _lib.ST_WORKSPACE_TOO_SMALL: SinkattnError,
    _lib.ST_NOT_SUPPORTED: NotImplementedError,
}


def _check(status: int) -> None:
    if status != _lib.ST_OK:
        msg = lib.st_last_error().decode(errors="replace")
        raise _STATUS.get(status, SinkattnError)(f"st status {status}: {msg}")


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


@dataclasses.dataclass(frozen=True)
class BandSpec:
    """Shape/parameter descriptor (st_desc)."""
    batch: int
    heads: int
    seq_q: int
    seq_k: int
    head_dim: int
    half_band: int
    base_depth: int
    tail_depth: int = 2
    epsilon: float = 1.0
    dtype: str = "f32"          # "f32" | "bf16"
    dustbin: int = 0
    dustbin_cost: float = 1.0
    centered: bool = True
    generic: bool = False       # force the generic (non-tensor-core) kernels (testing / ablation)
    stored_band: bool = False   # bf16 problems that would run band-free: keep the stored-band kernels
    # EpsSchedule of the base solve (trace.hpp:12-50): ((epsilon, iterations), ...), non-increasing
    # temperatures, iterations summing to base_depth, the last stage at `epsilon`.  None: one stage.
    eps_schedule: Optional[Sequence[Tuple[float, int]]] = None

    def desc(self) -> _lib.StDesc:
        d = _lib.StDesc(self.batch, self.heads, self.seq_q, self.seq_k, self.head_dim, self.half_band,
                        self.base_depth, self.tail_depth, float(self.epsilon),
                        _lib.ST_BF16 if self.dtype == "bf16" else _lib.ST_F32, int(self.dustbin),
                        float(self.dustbin_cost), int(bool(self.centered)),
                        (_lib.ST_FLAG_GENERIC if self.generic else 0) |
                        (_lib.ST_FLAG_STORED_BAND if self.stored_band else 0))
        if self.eps_schedule:
            n = len(self.eps_schedule)
            d._eps = (ctypes.c_double * n)(*[float(e) for e, _ in self.eps_schedule])  # kept alive by d
            d._its = (ctypes.c_int64 * n)(*[int(k) for _, k in self.eps_schedule])
            d.n_stages = n
            d.stage_eps = ctypes.cast(d._eps, ctypes.POINTER(ctypes.c_double))
            d.stage_iters = ctypes.cast(d._its, ctypes.POINTER(ctypes.c_int64))
        return d

    @property
    def rows(self) -> int:
        return self.seq_q + self.dustbin

    @property
    def cols(self) -> int:
        return self.seq_k + self.dustbin

    def saved_bytes(self) -> int:
        d = self.desc()
        return int(lib.st_saved_bytes(ctypes.byref(d)))

    def workspace_bytes(self) -> int:
        d = self.desc()
        return int(lib.st_workspace_bytes(ctypes.byref(d)))


class Workspace:
    """Caller-owned device scratch (the library never allocates)."""

    def __init__(self) -> None:
        self._buf: Optional[torch.Tensor] = None
        self.last_forward: Optional[object] = None  # token of the forward whose score band the buffer holds

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self._buf is None or self._buf.numel() < nbytes or self._buf.device != torch.device(device):
            self._buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            self.last_forward = None
        return self._buf


_default_ws = Workspace()


def validate_support(spec: BandSpec, row_mask: Optional[np.ndarray], col_mask: Optional[np.ndarray]) -> None:
    """SupportMask::validate (src/support.cpp:91-109) on host masks [B, L]."""
    d = spec.desc()
    rm = None if row_mask is None else np.ascontiguousarray(row_mask, dtype=np.uint8)
    cm = None if col_mask is None else np.ascontiguousarray(col_mask, dtype=np.uint8)
    _check(lib.st_validate_support(ctypes.byref(d), None if rm is None else rm.ctypes.data,
                                   None if cm is None else cm.ctypes.data))


@dataclasses.dataclass
class SurrogateRun:
    """Mirror of sinktail::SurrogateRun: output plus the O(L) saved tail state."""
    spec: BandSpec
    output: torch.Tensor
    saved: torch.Tensor
    Q: torch.Tensor
    K: torch.Tensor
    V: torch.Tensor
    row_mask: Optional[torch.Tensor]
    col_mask: Optional[torch.Tensor]
    workspace: Optional["Workspace"] = None  # holds this forward's score band until reused

    def check(self) -> None:
        """Raise the reference's exception if the forward hit an empty active reduction
        (InfeasibleSupport, sinkhorn.hpp:52-56); synchronizes the current stream."""
        d = self.spec.desc()
        _check(lib.st_check_status(ctypes.byref(d), _ptr(self.saved), torch.cuda.current_stream().cuda_stream))

    def tail_duals(self, row_mask_host=None, col_mask_host=None):
        """(u[3,BH,L'], v[3,BH,L'], gauge[3,BH]) in natural units, centered if spec.centered."""
        s = self.spec
        bh = s.batch * s.heads
        u = np.zeros((3, bh, s.rows))
        v = np.zeros((3, bh, s.cols))
        g = np.zeros((3, bh))
        d = s.desc()
        rm = None if row_mask_host is None else np.ascontiguousarray(row_mask_host, dtype=np.uint8)
        cm = None if col_mask_host is None else np.ascontiguousarray(col_mask_host, dtype=np.uint8)
        dp = ctypes.POINTER(ctypes.c_double)
        _check(lib.st_saved_duals(ctypes.byref(d), _ptr(self.saved), None if rm is None else rm.ctypes.data,
                                  None if cm is None else cm.ctypes.data, u.ctypes.data_as(dp),
                                  v.ctypes.data_as(dp), g.ctypes.data_as(dp),
                                  torch.cuda.current_stream().cuda_stream))
        return u, v, g


@dataclasses.dataclass
class CotangentSet:
    """Mirror of sinktail::CotangentSet (adjoint.hpp:19-28) plus d_eps."""
    grad_q: torch.Tensor
    grad_k: torch.Tensor
    grad_v: torch.Tensor
    d_eps: torch.Tensor   # [B*H]
    eta_v: torch.Tensor   # base cotangent v-bar^(0), [B, H, L'_k]
    eta_u: Optional[torch.Tensor] = None  # u-bar^(0), [B, H, L'_q] (tail_adjoint; nonzero only at R = 0)


def _check_tensor(name: str, t: torch.Tensor, spec: BandSpec, rows: int) -> None:
    want = torch.bfloat16 if spec.dtype == "bf16" else torch.float32
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != want:
        raise ValueError(f"{name} must be {want}, got {t.dtype}")
    if tuple(t.shape) != (spec.batch, spec.heads, rows, spec.head_dim) or not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous [{spec.batch},{spec.heads},{rows},{spec.head_dim}], "
                         f"got {tuple(t.shape)}")


def run_surrogate(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, spec: BandSpec,
                  row_mask: Optional[torch.Tensor] = None, col_mask: Optional[torch.Tensor] = None,
                  *, out: Optional[torch.Tensor] = None, saved: Optional[torch.Tensor] = None,
                  workspace: Optional[Workspace] = None, validate: bool = True) -> SurrogateRun:
    """Forward: stopped T-step base solve, R-step tail, O = P^(T+R,T+R) V (sinkhorn.hpp:288-302)."""
    _check_tensor("Q", Q, spec, spec.rows)
    _check_tensor("K", K, spec, spec.cols)
    _check_tensor("V", V, spec, spec.cols)
    for nm, m, L in (("row_mask", row_mask, spec.seq_q), ("col_mask", col_mask, spec.seq_k)):
        if m is not None and (m.dtype != torch.uint8 or tuple(m.shape) != (spec.batch, L) or not m.is_cuda):
            raise ValueError(f"{nm} must be a CUDA uint8 [{spec.batch},{L}] tensor")
    if validate:
        validate_support(spec, None if row_mask is None else row_mask.cpu().numpy(),
                         None if col_mask is None else col_mask.cpu().numpy())
    dev = Q.device
    if out is None:
        out = torch.empty((spec.batch, spec.heads, spec.rows, spec.head_dim), dtype=torch.float32, device=dev)
    if saved is None:
        saved = torch.empty(spec.saved_bytes(), dtype=torch.uint8, device=dev)
    wso = workspace or _default_ws
    ws = wso.get(spec.workspace_bytes(), dev)
    d = spec.desc()
    _check(lib.st_forward(ctypes.byref(d), _ptr(Q), _ptr(K), _ptr(V), _ptr(row_mask), _ptr(col_mask), _ptr(out),
                          _ptr(saved), _ptr(ws), ws.numel(), torch.cuda.current_stream(dev).cuda_stream))
    run = SurrogateRun(spec, out, saved, Q, K, V, row_mask, col_mask, wso)
    wso.last_forward = run
    return run


def r2_backward(run: SurrogateRun, G: torch.Tensor, mode: str = "one_reference", *,
                grads: Optional[tuple] = None, d_eps: Optional[torch.Tensor] = None,
                eta_v: Optional[torch.Tensor] = None, workspace: Optional[Workspace] = None) -> CotangentSet:
    """Exact R=2 adjoint (adjoint.hpp:232-373); mode "one_reference" or "direct_four_plan"."""
    if run.spec.tail_depth != 2:
        raise UnsupportedDepth("r2_backward requires a tail of depth 2")
    m = {"one_reference": _lib.ST_ONE_REFERENCE, "direct_four_plan": _lib.ST_DIRECT_FOUR_PLAN}[mode]
    return _backward(run, G, m, grads, d_eps, eta_v, workspace)


def tail_adjoint(run: SurrogateRun, G: torch.Tensor, *, grads: Optional[tuple] = None,
                 d_eps: Optional[torch.Tensor] = None, eta_v: Optional[torch.Tensor] = None,
                 workspace: Optional[Workspace] = None) -> CotangentSet:
    """Exact reverse pass of the tail for any depth R <= 8 (tail_adjoint_generic, adjoint.hpp:132-200):
    the score cotangent is materialised as a band, then contracted to dQ / dK / d_eps.
    eta_v = v-bar^(0) (the base-trace cotangent; dO-weighted column sums when R = 0)."""
    if not 0 <= run.spec.tail_depth <= 8:
        raise UnsupportedDepth("the generic tail adjoint supports tail depths 0..8")
    return _backward(run, G, _lib.ST_GENERIC_TAIL, grads, d_eps, eta_v, workspace, want_eta_u=True)


def base_solve_vjp(run: SurrogateRun, eta_v: torch.Tensor, eta_u: Optional[torch.Tensor] = None, *,
                   workspace: Optional[Workspace] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Pull a base-state cotangent (eta_u, eta_v) back through the T stopped base steps to (dQ, dK)
    (base_solve_vjp, certificates.hpp:25-70).  With eta = the tail adjoint's v-bar^(0) this is the
    omitted gradient c_R of the stopped surrogate (bias_certificate, certificates.hpp:112-118)."""
    spec = run.spec
    dev = run.Q.device
    for name, t, n in (("eta_v", eta_v, spec.cols), ("eta_u", eta_u, spec.rows)):
        if t is not None and (t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != spec.batch * spec.heads * n
                              or t.device != dev):
            raise ValueError(f"{name} must be a contiguous f32 [B, H, {n}] tensor on {dev}")
    gq = torch.empty((spec.batch, spec.heads, spec.rows, spec.head_dim), dtype=torch.float32, device=dev)
    gk = torch.empty((spec.batch, spec.heads, spec.cols, spec.head_dim), dtype=torch.float32, device=dev)
    d = spec.desc()
    wso = workspace or _default_ws
    ws = wso.get(int(lib.st_base_vjp_workspace_bytes(ctypes.byref(d))), dev)
    wso.last_forward = None  # the score band in the workspace is overwritten
    _check(lib.st_base_solve_vjp(ctypes.byref(d), _ptr(run.Q), _ptr(run.K), _ptr(run.row_mask), _ptr(run.col_mask),
                                 _ptr(eta_u), _ptr(eta_v), _ptr(gq), _ptr(gk), _ptr(ws), ws.numel(),
                                 torch.cuda.current_stream(dev).cuda_stream))
    return gq, gk


def _backward(run, G, m, grads, d_eps, eta_v, workspace, want_eta_u=False) -> CotangentSet:
    spec = run.spec
    _check_tensor("G", G, spec, spec.rows)
    dev = G.device
    if grads is None:
        grads = tuple(torch.empty((spec.batch, spec.heads, r, spec.head_dim), dtype=torch.float32, device=dev)
                      for r in (spec.rows, spec.cols, spec.cols))
    dQ, dK, dV = grads
    if d_eps is None:
        d_eps = torch.empty(spec.batch * spec.heads, dtype=torch.float32, device=dev)
    if eta_v is None:
        eta_v = torch.empty((spec.batch, spec.heads, spec.cols), dtype=torch.float32, device=dev)
    wso = workspace or _default_ws
    if want_eta_u:  # the generic tail adjoint runs on the stored-band kernels
        spec = dataclasses.replace(spec, stored_band=True)
    ws = wso.get(spec.workspace_bytes(), dev)
    d = spec.desc()
    if wso is run.workspace and wso.last_forward is run:
        # the workspace still holds this forward's score band (reference: r2_backward(run.scaled, ...))
        d.flags |= _lib.ST_FLAG_REUSE_BAND
    stream = torch.cuda.current_stream(dev).cuda_stream
    if want_eta_u:  # tail_adjoint_generic: the whole base cotangent
        eta_u = torch.empty((spec.batch, spec.heads, spec.rows), dtype=torch.float32, device=dev)
        _check(lib.st_tail_adjoint(ctypes.byref(d), _ptr(run.saved), _ptr(run.Q), _ptr(run.K), _ptr(run.V), _ptr(G),
                                   _ptr(run.row_mask), _ptr(run.col_mask), _ptr(dQ), _ptr(dK), _ptr(dV),
                                   _ptr(d_eps), _ptr(eta_u), _ptr(eta_v), _ptr(ws), ws.numel(), stream))
        return CotangentSet(dQ, dK, dV, d_eps, eta_v, eta_u)
    _check(lib.st_backward(ctypes.byref(d), _ptr(run.saved), _ptr(run.Q), _ptr(run.K), _ptr(run.V), _ptr(G),
                           _ptr(run.row_mask), _ptr(run.col_mask), _ptr(dQ), _ptr(dK), _ptr(dV), _ptr(d_eps),
                           _ptr(eta_v), m, _ptr(ws), ws.numel(), stream))
    return CotangentSet(dQ, dK, dV, d_eps, eta_v)


def launch_count(reset: bool = False) -> int:
    return int(lib.st_launch_count(1 if reset else 0))
