"""Omitted-gradient certificates of the tail depth (certificates.hpp:72-179), on the device path.

The stopped surrogate drops the gradient that flows through the T base steps.  For a tail depth R the
dropped part is c_R = base_solve_vjp(eta_R) where eta_R = v-bar^(0) is the base cotangent the tail
adjoint emits (tail_adjoint_generic, adjoint.hpp:132-200).  ``bias_certificate`` measures it;
``select_tail_depth`` picks the smallest R whose certified omitted gradient is below a tolerance.

Batched over the B*H heads of a BandSpec: every per-head figure is a [B*H] tensor, and the selector's
test takes the worst head (max over heads).  The reference's dense full-BPTT residual check
(certificates.hpp:127-138) is an f64 oracle computation; it lives in the test oracle
(oracle/sinktail_oracle.hpp: bias_certificate), not here.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional

import torch

from . import band


@dataclasses.dataclass
class BiasCertificate:
    tail_depth: int
    eta_norm: torch.Tensor  # [B*H]  ||(u-bar^(0), v-bar^(0))||_2
    c_inf: torch.Tensor     # [B*H]  max |c_R| over (Q, K)
    c_l2: torch.Tensor      # [B*H]  ||c_R||_2 over (Q, K)
    c_q: torch.Tensor       # [B, H, L', d]
    c_k: torch.Tensor


def bias_certificate(Q, K, V, G, spec: band.BandSpec, tail_depth: int, row_mask=None, col_mask=None, *,
                     workspace: Optional[band.Workspace] = None) -> BiasCertificate:
    """certificates.hpp:112-140 for a linear loss with output cotangent G: forward at depth R, generic
    tail adjoint, base-solve VJP of its base cotangent."""
    sp = dataclasses.replace(spec, tail_depth=int(tail_depth))
    run = band.run_surrogate(Q, K, V, sp, row_mask, col_mask, workspace=workspace)
    cot = band.tail_adjoint(run, G, workspace=workspace)
    cq, ck = band.base_solve_vjp(run, cot.eta_v, cot.eta_u, workspace=workspace)
    bh = sp.batch * sp.heads
    fq, fk = cq.reshape(bh, -1), ck.reshape(bh, -1)
    c_inf = torch.maximum(fq.abs().amax(dim=1), fk.abs().amax(dim=1))
    c_l2 = torch.sqrt((fq.double() ** 2).sum(dim=1) + (fk.double() ** 2).sum(dim=1))
    eta = torch.sqrt((cot.eta_v.reshape(bh, -1).double() ** 2).sum(dim=1) +
                     (cot.eta_u.reshape(bh, -1).double() ** 2).sum(dim=1))
    return BiasCertificate(int(tail_depth), eta, c_inf, c_l2, cq, ck)


@dataclasses.dataclass
class TailDepthSelection:
    selected: int = -1  # -1: no depth satisfies the tolerance
    used_sufficient_bound: bool = False
    trail: List[BiasCertificate] = dataclasses.field(default_factory=list)


def select_tail_depth(Q, K, V, G, spec: band.BandSpec, tau: float, r_max: int,
                      cost: Callable[[int], float] = float, operator_norm_bound: Optional[float] = None,
                      row_mask=None, col_mask=None, *, workspace: Optional[band.Workspace] = None
                      ) -> TailDepthSelection:
    """certificates.hpp:152-179: smallest R <= r_max with max-over-heads c_inf <= tau (or, given an
    operator-norm bound C_T, the sufficient test C_T * ||eta_R|| <= tau).  ``cost`` must be
    nondecreasing, so the first feasible depth is the min-cost certified choice."""
    if not tau > 0:
        raise ValueError("tolerance must be > 0")
    if r_max < 0:
        raise ValueError("R_max must be >= 0")
    if r_max > 8:
        raise band.UnsupportedDepth("tail depths above 8 are not supported")
    prev = -math.inf
    for r in range(r_max + 1):
        c = cost(r)
        if c < prev:
            raise ValueError("cost function must be nondecreasing")
        prev = c
    sel = TailDepthSelection(used_sufficient_bound=operator_norm_bound is not None)
    for r in range(r_max + 1):
        cert = bias_certificate(Q, K, V, G, spec, r, row_mask, col_mask, workspace=workspace)
        if operator_norm_bound is not None:
            ok = float(cert.eta_norm.max()) * operator_norm_bound <= tau
        else:
            ok = float(cert.c_inf.max()) <= tau
        sel.trail.append(cert)
        if ok:
            sel.selected = r
            break
    return sel
