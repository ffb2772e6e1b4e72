"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle (f64 reference path).

Error measure: rel-L2 = ||gpu - ref|| / ||ref|| per tensor, ref = the f64 oracle
(the reference algorithm in double).  Bound per tensor:
    max(TOL, 1.5 x rel-L2 of the reference's OWN f32 path vs f64)
i.e. 1e-5 for fp32 inputs unless the reference's own f32 template mode
(inc/types.hpp:18-21) cannot reach it on that problem -- then the GPU must be
at least as accurate as the reference's f32 implementation (config 3's
near-permutation plans make dQ ill-conditioned in fp32: the reference's own
f32 path shows ~4e-4 there).
bf16 configs (4, 5): both paths consume the same bf16-rounded inputs, the GPU
accumulates in fp32 (tensor-core contract); stated bound BF16_TOL = 1e-4.
A tiny absolute floor (ATOL per element) covers tensors that are exactly zero
in exact arithmetic (e.g. dQ on a diagonal support, w = 0).
"""
import numpy as np
import pytest
import torch

import oracle_ref
import parity_log
from paper_2605_08123_b200 import band, configs

FP32_TOL = 1e-5
FP32_GRAD_TOL = 1e-5
BF16_TOL = 1e-4
# d_eps = -(1/eps) sum_ij Sbar_ij S_ij is one scalar per head with heavy cancellation
# (Sbar rows nearly sum to zero); it has no reference pin, so its bound is stated separately.
DEPS_TOL = 1e-4

pytestmark = pytest.mark.gpu


def _dev(x, bits=None):
    if bits is not None:
        return torch.from_numpy(bits.astype(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def gpu_run(cfg, inp, mode="one_reference", G=None, heads_as_batch=False, eps_schedule=None, duals=True,
            stored_band=False):
    """Run the CUDA path on the generated heads; returns numpy results [nh, L', d]."""
    nh = len(inp.heads)
    if heads_as_batch or nh != cfg.B * cfg.H:
        B, H = nh, 1
        sel = np.array([h // cfg.H for h in inp.heads])
        rm = None if inp.row_mask is None else inp.row_mask[sel]
        cm = None if inp.col_mask is None else inp.col_mask[sel]
    else:
        B, H, rm, cm = cfg.B, cfg.H, inp.row_mask, inp.col_mask
    spec = band.BandSpec(batch=B, heads=H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype,
                         dustbin=cfg.dustbin, dustbin_cost=cfg.dustbin_cost, eps_schedule=eps_schedule,
                         stored_band=stored_band)
    shp = (B, H, cfg.rows, cfg.d)
    b = inp.bits or {}
    Q = _dev(inp.Q, b.get("Q")).reshape(shp)
    K = _dev(inp.K, b.get("K")).reshape(shp)
    V = _dev(inp.V, b.get("V")).reshape(shp)
    if G is None:
        Gd = _dev(inp.G, b.get("G")).reshape(shp)
    else:
        Gd = G
    rmd = None if rm is None else torch.from_numpy(rm).cuda()
    cmd = None if cm is None else torch.from_numpy(cm).cuda()
    run = band.run_surrogate(Q, K, V, spec, rmd, cmd)
    cot = band.tail_adjoint(run, Gd) if mode == "generic_tail" else band.r2_backward(run, Gd, mode=mode)
    torch.cuda.synchronize()
    u, v, g = run.tail_duals(rm, cm) if duals else (None, None, None)
    res = dict(O=run.output, dQ=cot.grad_q, dK=cot.grad_k, dV=cot.grad_v, d_eps=cot.d_eps, eta_v=cot.eta_v)
    res = {k: x.detach().cpu().numpy().astype(np.float64) for k, x in res.items()}
    for k in ("O", "dQ", "dK", "dV"):
        res[k] = res[k].reshape(nh, cfg.rows, cfg.d)
    res["eta_v"] = res["eta_v"].reshape(nh, cfg.rows)
    res["u"], res["v"], res["gauge"] = u, v, g
    return res


ATOL = 1e-7


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = max(float(np.linalg.norm(b)), ATOL * np.sqrt(b.size) / 1e-5)
    return float(np.linalg.norm(a - b) / nb)


def oracle(cfg, inp, **kw):
    return oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, heads=inp.heads, **kw)


KEYS = ("O", "dQ", "dK", "dV", "eta_v", "d_eps")


def check_against_oracle(cfg, inp, tol_o, tol_g, mode="one_reference", eps_schedule=None, case=None,
                         bounds_override=None, floor=True, stored_band=False):
    g = gpu_run(cfg, inp, mode=mode, eps_schedule=eps_schedule, stored_band=stored_band)
    m = 1 if mode == "direct_four_plan" else 0
    r = oracle(cfg, inp, precision=64, mode=m, eps_schedule=eps_schedule)
    # the reference's own f32 instantiation (the noise floor; informational for the fixed bf16 bound)
    r32 = oracle(cfg, inp, precision=32, mode=m, eps_schedule=eps_schedule) if floor else r
    errs = {k: rel(g[k], r[k]) for k in KEYS}
    floor = {k: rel(r32[k], r[k]) for k in KEYS}
    print(f"config {cfg.cid} L={cfg.L} heads={len(inp.heads)} mode={mode} rel-L2 gpu / ref-f32:",
          {k: f"{errs[k]:.2e}/{floor[k]:.2e}" for k in KEYS})
    bounds = {}
    for k in KEYS:
        tol = tol_o if k in ("O", "dV") else (max(DEPS_TOL, tol_g) if k == "d_eps" else tol_g)
        # d_eps (EXT, no reference pin) is a cancellation-heavy scalar sum of +-Sbar*S: within 3x of the
        # reference's own f32 instantiation (config 3 with scores |s2| ~ 115 sits at ~1e-3 there)
        bounds[k] = max(tol, (3.0 if k == "d_eps" else 1.5) * floor[k])
    bounds.update(bounds_override or {})
    parity_log.record(case or f"config{cfg.cid}", cfg, inp.heads, mode, errs, floor, bounds)
    assert np.all(np.isfinite(g["O"])) and np.all(np.isfinite(g["dQ"]))
    for k in KEYS:
        assert errs[k] <= bounds[k], (k, errs[k], bounds[k], errs)
    # saved tail duals (centered gauge ledger) against the oracle's centered trace
    nh = len(inp.heads)
    for rr in range(3):
        gu, ru = g["u"][rr], r["duals"][:, rr, :]
        gv, rv = g["v"][rr], r["duals"][:, 3 + rr, :]
        act_r = np.ones_like(ru, dtype=bool)
        act_c = np.ones_like(rv, dtype=bool)
        if inp.row_mask is not None:
            sel = np.array([h // cfg.H for h in inp.heads])
            act_r[:, :cfg.L] = inp.row_mask[sel] != 0
            act_c[:, :cfg.L] = inp.col_mask[sel] != 0
        scale = max(1.0, np.abs(ru[act_r]).max())
        assert np.abs(gu[act_r] - ru[act_r]).max() < 2e-4 * scale, rr
        assert np.abs(gv[act_c] - rv[act_c]).max() < 2e-4 * scale, rr
        assert np.abs(g["gauge"][rr] - r["gauges"][:, rr]).max() < 2e-4 * scale
    return g, r, errs


def test_config1_parity():
    cfg = configs.CONFIGS[1]
    check_against_oracle(cfg, configs.make_inputs(cfg), FP32_TOL, FP32_GRAD_TOL)


def test_config1_direct_four_plan_parity_and_agreement():
    cfg = configs.CONFIGS[1]
    inp = configs.make_inputs(cfg)
    g4, _, _ = check_against_oracle(cfg, inp, FP32_TOL, FP32_GRAD_TOL, mode="direct_four_plan")
    g1 = gpu_run(cfg, inp)
    for k in ("dQ", "dK", "dV"):
        assert rel(g4[k], g1[k]) < 1e-5


def test_config2_parity_full_batch():
    cfg = configs.CONFIGS[2]
    check_against_oracle(cfg, configs.make_inputs(cfg), FP32_TOL, FP32_GRAD_TOL)


def test_fp32_solve_more_blocks_than_resident_tiles():
    """Config-2 geometry with 64 heads x 16 row blocks = 1024 work items (~750 active under the masks), more
    than the 444 band tiles the persistent fp32 solve keeps resident (3 per SM): its non-resident mode
    (tiles restaged every step, window duals through `vpriv`, grid barrier per step) against the oracle."""
    cfg = configs.CONFIGS[2].replace(B=16, T=12)
    inp = configs.make_inputs(cfg)
    check_against_oracle(cfg, inp, FP32_TOL, FP32_GRAD_TOL, case="config2-B16-nonresident")


def test_config3_dustbin_parity_full_batch():
    cfg = configs.CONFIGS[3]
    g, r, _ = check_against_oracle(cfg, configs.make_inputs(cfg), FP32_TOL, FP32_GRAD_TOL)
    # constant-cost dustbin rows carry no Q/K gradient
    assert np.abs(g["dQ"][:, cfg.L]).max() == 0.0
    assert np.abs(g["dK"][:, cfg.L]).max() == 0.0


@pytest.mark.parametrize("cid,L", [(4, 4096), (5, 4096)])
def test_bf16_configs_reduced_length_parity(cid, L):
    cfg = configs.CONFIGS[cid].replace(L=L)
    inp = configs.make_inputs(cfg, heads=range(0, 2))
    check_against_oracle(cfg, inp, BF16_TOL, BF16_TOL)


@pytest.mark.parametrize("cid,L,mode", [(4, 4096, "one_reference"), (5, 4096, "direct_four_plan")])
def test_bf16_stored_band_kernels_parity(cid, L, mode):
    """ST_FLAG_STORED_BAND: the stored-band bf16 kernels (tcgen05 band write passes, k_bwdM / k_sweepW)
    that the generic tail adjoint and the sequence-sharded entry points still run on, against the oracle."""
    cfg = configs.CONFIGS[cid].replace(L=L)
    inp = configs.make_inputs(cfg, heads=range(0, 2))
    check_against_oracle(cfg, inp, BF16_TOL, BF16_TOL, mode=mode, stored_band=True,
                         case=f"config{cid}-L{L}-stored-band-{mode}")


@pytest.mark.parametrize("w,d,mask,L,mode", [(128, 128, "uniform_len", 1000, "direct_four_plan"),
                                             (256, 64, "uniform_len", 1500, "one_reference"),
                                             (256, 64, "none", 1100, "direct_four_plan"),
                                             (128, 64, "uniform_len", 650, "one_reference"),
                                             (64, 64, "uniform_len", 650, "one_reference"),
                                             (192, 128, "none", 900, "direct_four_plan"),
                                             (256, 128, "none", 300, "one_reference")])
def test_bf16_band_free_sweeps_parity(w, d, mask, L, mode):
    """The band-free tcgen05 sweeps (st_bfree.cu: transport output, C1 / R12 / C3 / R4 / R6 / C6 with the
    score and cotangent tiles recomputed per block, weights as bf16 hi/lo planes, MN-major operand chunks):
    both adjoint schedules, masked rows / columns (-inf offsets), partial last blocks, edge windows, a
    band nearly as wide as the sequence, d = 64 / 128, against the oracle."""
    cfg = configs.Config(0, B=2, H=2, L=L, d=d, w=w, eps=0.05, T=12, R=2, dtype="bf16", mask=mask,
                         in_scale=1 / np.sqrt(d))
    import dataclasses
    spec = band.BandSpec(batch=2, heads=2, seq_q=L, seq_k=L, head_dim=d, half_band=w, base_depth=12, dtype="bf16")
    # the problem is band-free: its workspace lacks the L x W band(s) of the stored-band layout
    assert dataclasses.replace(spec, stored_band=True).workspace_bytes() - spec.workspace_bytes() > 0.9 * 4 * L * (2 * w + 1) * 4
    check_against_oracle(cfg, configs.make_inputs(cfg), BF16_TOL, BF16_TOL, mode=mode,
                         case=f"bfree-w{w}-d{d}-{mask}-{mode}")


def test_small_shapes_and_edge_cases():
    """Ragged / tiny / rectangular-free edge cases the reference tests use (w=0, w>=L, L=1, odd d)."""
    cases = [
        configs.Config(0, B=1, H=1, L=1, d=4, w=0, eps=1.0, T=3, R=2, dtype="f32"),
        configs.Config(0, B=1, H=2, L=5, d=3, w=0, eps=0.7, T=4, R=2, dtype="f32"),
        configs.Config(0, B=2, H=1, L=37, d=8, w=40, eps=0.5, T=6, R=2, dtype="f32"),
        configs.Config(0, B=1, H=1, L=200, d=33, w=7, eps=0.2, T=0, R=2, dtype="f32"),
        configs.Config(0, B=2, H=2, L=130, d=16, w=9, eps=0.3, T=5, R=2, dtype="f32", mask="uniform_len"),
        configs.Config(0, B=2, H=1, L=64, d=8, w=3, eps=0.5, T=5, R=2, dtype="f32", mask="lognormal_len",
                       dustbin=1, dustbin_cost=0.7, embed="alphabet"),
    ]
    for cfg in cases:
        check_against_oracle(cfg, configs.make_inputs(cfg), 2e-5, 5e-5)


def test_infeasible_support_is_rejected():
    cfg = configs.Config(0, B=1, H=1, L=3, d=4, w=0, eps=1.0, T=2, R=2, dtype="f32")
    spec = band.BandSpec(batch=1, heads=1, seq_q=3, seq_k=3, head_dim=4, half_band=0, base_depth=2, epsilon=1.0)
    x = torch.zeros((1, 1, 3, 4), device="cuda")
    cm = torch.tensor([[0, 1, 1]], dtype=torch.uint8, device="cuda")
    with pytest.raises(band.InfeasibleSupport):
        band.run_surrogate(x, x, x, spec, None, cm)


def test_deterministic_and_linear_in_G():
    cfg = configs.CONFIGS[2].replace(B=2)
    inp = configs.make_inputs(cfg)
    a = gpu_run(cfg, inp)
    b = gpu_run(cfg, inp)
    for k in ("O", "dQ", "dK", "dV", "d_eps"):
        assert np.array_equal(a[k], b[k]), k
    # the adjoint is linear in the output cotangent
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    G1 = torch.from_numpy(inp.G).cuda().reshape(shp)
    G2 = torch.flip(G1, dims=[2]).contiguous()
    r1 = gpu_run(cfg, inp, G=G1)
    r2 = gpu_run(cfg, inp, G=G2)
    r3 = gpu_run(cfg, inp, G=(0.5 * G1 - 2.0 * G2).contiguous())
    for k in ("dQ", "dK", "dV"):
        assert rel(r3[k], 0.5 * r1[k] - 2.0 * r2[k]) < 1e-5, k


def test_bf16_workspace_is_O_of_L():
    """With a GPU driver (tensor maps available) BASELINE configs 4 / 5 need only O(L) scratch: no L x W band
    and no packed O(L d) operand plane (north_star: "O(L d) inputs plus O(L) extra HBM")."""
    for cid in (4, 5):
        cfg = configs.CONFIGS[cid]
        spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                             base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype)
        per_row = spec.workspace_bytes() / (cfg.B * cfg.H * cfg.L)
        one_plane = cfg.d * 2
        assert per_row < 48 * 4 and per_row < 1.5 * one_plane, (cid, per_row)  # ~37 fp32 words per row; < 1.5 planes


def test_bf16_band_free_deterministic_and_linear_in_G():
    """The band-free sweeps are run-to-run bit-identical (fixed-order row-part combines, no atomics on the
    data path) and the adjoint is linear in the output cotangent (config-4 geometry, several blocks per CTA)."""
    cfg = configs.CONFIGS[4].replace(L=8192, T=10)
    inp = configs.make_inputs(cfg, heads=range(6))
    a = gpu_run(cfg, inp, duals=False)
    b = gpu_run(cfg, inp, duals=False)
    for k in ("O", "dQ", "dK", "dV", "d_eps", "eta_v"):
        assert np.array_equal(a[k], b[k]), k
    shp = (6, 1, cfg.rows, cfg.d)
    G1 = _dev(inp.G, inp.bits["G"]).reshape(shp)
    G2 = torch.flip(G1, dims=[2]).contiguous()
    r1 = gpu_run(cfg, inp, G=G1, duals=False)
    r2 = gpu_run(cfg, inp, G=G2, duals=False)
    r3 = gpu_run(cfg, inp, G=(0.5 * G1 - 2.0 * G2).contiguous(), duals=False)  # exact in bf16 up to one rounding
    for k in ("dQ", "dK", "dV"):
        assert rel(r3[k], 0.5 * r1[k] - 2.0 * r2[k]) < 5e-3, k


@pytest.mark.parametrize("cid,heads", [(4, (0, 1)), (5, (0,))])
def test_bf16_full_baseline_shape_parity(cid, heads):
    """Configs 4 / 5 at their full BASELINE shapes (L = 32768 / 131072, the full band, T, eps) on a
    seeded head subset: 512 / 1024 row blocks per launch, i.e. several blocks per
    persistent CTA, so the cross-block chunk reuse and ring bookkeeping of the half-step kernel run
    exactly as in the benchmark.  Stated bf16 bound: BF16_TOL = 1e-4 rel-L2 on O, dQ, dK, dV, eta."""
    import os
    cfg = configs.CONFIGS[cid]
    inp = configs.make_inputs(cfg, heads=range(heads[0], heads[-1] + 1))
    # config 5's f32 floor run costs ~2.5 min of host time: only when the parity table is regenerated
    floor = cid == 4 or bool(os.environ.get("ST_PARITY_OUT"))
    check_against_oracle(cfg, inp, BF16_TOL, BF16_TOL, case=f"config{cid}-full-L", floor=floor)


def test_bf16_many_blocks_per_cta_parity():
    """Config-4 geometry (d = 128, W = 257) with 8 heads x 64 blocks = 512 blocks > 2 x 148 CTAs."""
    cfg = configs.CONFIGS[4].replace(L=8192)
    inp = configs.make_inputs(cfg, heads=range(8))
    check_against_oracle(cfg, inp, BF16_TOL, BF16_TOL, case="config4-L8192-8heads")


@pytest.mark.parametrize("cid", [4, 5])
def test_bf16_full_size_row_sums(cid):
    """Every head of the full configs: the row sums of the tail plan P22 (O with V = 1) are close to 1.
    The final column half-step forces the COLUMN sums to 1 for any u, so the row sums are the check
    that reaches the row solve; their deviation must stay within 2x of the oracle's on head 0 (+1e-4)."""
    cfg = configs.CONFIGS[cid]
    inp = configs.make_inputs(cfg)
    ones_bits = np.full_like(inp.bits["V"], 0x3F80)           # bf16 1.0
    inp.V = np.ones_like(inp.V)
    inp.bits = {**inp.bits, "V": ones_bits}
    g = gpu_run(cfg, inp, duals=False)
    assert np.all(np.isfinite(g["O"])) and np.all(np.isfinite(g["dQ"])) and np.all(np.isfinite(g["dK"]))
    rows = g["O"][:, :, 0]
    assert np.array_equal(g["O"][:, :, 0], g["O"][:, :, -1])
    dev = np.abs(rows - 1.0).max(axis=1)
    if cid == 4:
        # anchor: the oracle's own row-sum deviation on head 0 (forward only, ~20 s of host time)
        sub = configs.make_inputs(cfg, heads=range(1))
        r = oracle_ref.run(cfg, sub.Q, sub.K, np.ones_like(sub.V), sub.G, heads=sub.heads, precision=64,
                           backward=False)
        ref_dev = float(np.abs(r["O"][0, :, 0] - 1.0).max())
        assert abs(float(dev[0]) - ref_dev) <= 0.05 * ref_dev + 1e-4
    else:
        # config 5: head 0 is oracle-checked at full length (test_bf16_full_baseline_shape_parity); the
        # other heads must sit at its level (an oracle forward here would cost ~2.5 min of host time)
        ref_dev = float(dev[0])
    print(f"config {cid}: max |rowsum(P22) - 1| per head {dev.max():.3e} (anchor head 0: {ref_dev:.3e})")
    assert dev.max() <= 2 * ref_dev + 1e-4, dev


@pytest.mark.parametrize("cid,L", [(2, None), (4, 2048), (5, 2048)])
def test_band_reuse_matches_recompute(cid, L):
    """ST_FLAG_REUSE_BAND (backward consumes the forward's score band, as r2_backward(run.scaled, ...)
    does) gives bit-identical gradients to recomputing the band in a fresh workspace: fp32 (f64 DMMA
    band) and bf16 (tcgen05 band write passes, configs 4 / 5 geometry)."""
    cfg = configs.CONFIGS[cid].replace(B=1)
    if L:
        cfg = cfg.replace(L=L, H=2)
    inp = configs.make_inputs(cfg)
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype)
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    b_ = inp.bits or {}
    Q, K, V, G = (_dev(getattr(inp, k), b_.get(k)).reshape(shp) for k in ("Q", "K", "V", "G"))
    rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).cuda()
    ws = band.Workspace()
    run = band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws)
    a = band.r2_backward(run, G, workspace=ws)           # reuses the band
    b = band.r2_backward(run, G, workspace=band.Workspace())  # recomputes it
    for x, y in ((a.grad_q, b.grad_q), (a.grad_k, b.grad_k), (a.grad_v, b.grad_v), (a.d_eps, b.d_eps)):
        assert torch.equal(x, y)


@pytest.mark.parametrize("cid,L,nh,sched", [
    (1, None, None, [(0.4, 5), (0.2, 5), (0.1, 10)]),          # resident (TMEM) fused solve
    (2, None, 4, [(0.2, 10), (0.1, 15), (0.05, 25)]),          # masked batch, fused solve
    (3, None, 8, [(0.3, 10), (0.2, 10), (0.1, 10)]),           # dustbin: per-step kernels, band per stage
    (4, 2048, 2, [(0.2, 30), (0.1, 30), (0.05, 40)]),          # bf16: tcgen05 scores per stage
])
def test_eps_schedule_parity(cid, L, nh, sched):
    """EpsSchedule stages of the stopped base solve (trace.hpp:12-50, sinkhorn.hpp:186-195): each
    stage runs at its own temperature, the tail at the final one; against the oracle's schedule."""
    cfg = configs.CONFIGS[cid]
    if L:
        cfg = cfg.replace(L=L)
    inp = configs.make_inputs(cfg, heads=None if nh is None else range(nh))
    tol = BF16_TOL if cfg.dtype == "bf16" else FP32_TOL
    check_against_oracle(cfg, inp, tol, tol, eps_schedule=sched)


def test_eps_schedule_generic_kernels():
    cfg = configs.Config(0, B=1, H=2, L=64, d=8, w=5, eps=0.5, T=6, R=2, dtype="f32")
    check_against_oracle(cfg, configs.make_inputs(cfg), 2e-5, 5e-5, eps_schedule=[(1.0, 3), (0.5, 3)])


@pytest.mark.parametrize("Lq,Lk,d,w,masked", [(160, 150, 32, 20, False), (96, 120, 64, 33, True),
                                               (130, 126, 8, 5, False)])
def test_rectangular_parity(Lq, Lk, d, w, masked):
    """L_q != L_k supports (build_band_support(Lq, Lk, w, ...), support.cpp:111; the reference's
    rectangular adjoint test, test_adjoint.cpp:378-409) on the per-step and generic kernels."""
    rng = np.random.default_rng(7)
    nh, eps, T, R = 2, 0.3, 6, 2
    Q, G = (rng.standard_normal((nh, Lq, d)).astype(np.float32) for _ in range(2))
    K, V = (rng.standard_normal((nh, Lk, d)).astype(np.float32) for _ in range(2))
    rm = cm = None
    if masked:
        rm = (np.arange(Lq)[None, :] < np.array([[Lq - 10], [Lq]])).astype(np.uint8)
        cm = (np.arange(Lk)[None, :] < np.array([[Lk - 40], [Lk - 3]])).astype(np.uint8)
    spec = band.BandSpec(batch=nh, heads=1, seq_q=Lq, seq_k=Lk, head_dim=d, half_band=w, base_depth=T,
                         tail_depth=R, epsilon=eps)
    dev = lambda x, L: torch.from_numpy(x).cuda().reshape(nh, 1, L, d)
    run = band.run_surrogate(dev(Q, Lq), dev(K, Lk), dev(V, Lk), spec,
                             None if rm is None else torch.from_numpy(rm).cuda(),
                             None if cm is None else torch.from_numpy(cm).cuda())
    cot = band.r2_backward(run, dev(G, Lq))
    torch.cuda.synchronize()
    g = {"O": run.output, "dQ": cot.grad_q, "dK": cot.grad_k, "dV": cot.grad_v, "d_eps": cot.d_eps}
    g = {k: x.cpu().numpy().astype(np.float64).reshape(nh, -1) for k, x in g.items()}
    r = oracle_ref.run_rect(Lq, Lk, d, w, eps, T, R, Q, K, V, G, rm, cm)
    r32 = oracle_ref.run_rect(Lq, Lk, d, w, eps, T, R, Q, K, V, G, rm, cm, precision=32)
    for k in ("O", "dQ", "dK", "dV", "d_eps"):
        e, fl = rel(g[k], r[k].reshape(nh, -1)), rel(r32[k].reshape(nh, -1), r[k].reshape(nh, -1))
        tol = DEPS_TOL if k == "d_eps" else FP32_TOL
        assert e <= max(tol, (3.0 if k == "d_eps" else 1.5) * fl), (k, e, fl)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_sequence_sharded_lockstep_matches_unsharded(dtype):
    """Config-5 style sequence sharding on one GPU: two shards (own rows + w-wide halos) run the
    per-step kernels in lockstep host threads with the halo hook completing every dual / adjoint
    vector (shard.Lockstep, the protocol nccl_halo runs across GPUs); own rows / columns and the
    summed d_eps equal the unsharded run on the same kernels."""
    import threading
    from paper_2605_08123_b200 import shard
    B, H, L, d, w, eps, T, R = 1, 2, 1024, 64, 64, 0.1, 8, 2
    rng = np.random.default_rng(11)
    mk = lambda: rng.standard_normal((B, H, L, d)).astype(np.float32) / np.sqrt(d)
    Qh, Kh, Vh, Gh = mk(), mk(), mk(), mk()
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    to = lambda x: torch.from_numpy(x).cuda().to(tdt).contiguous()
    spec = lambda n: band.BandSpec(batch=B, heads=H, seq_q=n, seq_k=n, head_dim=d, half_band=w, base_depth=T,
                                   tail_depth=R, epsilon=eps, dtype=dtype)
    # unsharded, same per-step kernels (a no-op hook selects them)
    ref = shard.sharded_forward_backward(spec(L), to(Qh), to(Kh), to(Vh), to(Gh), None, None,
                                         lambda v: None, range(0, L))
    plans = [shard.SeqShard(L=L, w=w, world=2, rank=r) for r in range(2)]
    streams = [torch.cuda.Stream() for _ in plans]
    ls = shard.Lockstep(plans, streams)
    outs, errs = [None, None], []

    def run(r):
        try:
            p = plans[r]
            win = slice(p.window.start, p.window.stop)
            hl = p.rows.start - p.window.start
            with torch.cuda.stream(streams[r]):
                args = [to(x[:, :, win]) for x in (Qh, Kh, Vh, Gh)]
                outs[r] = shard.sharded_forward_backward(spec(len(p.window)), *args, None, None, ls.exchange_for(r),
                                                         range(hl, hl + len(p.rows)))
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            ls.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    torch.cuda.synchronize()
    for k in range(4):  # O, dQ (own rows), dK, dV (own columns)
        got = torch.empty_like(ref[k])
        for r, p in enumerate(plans):
            hl = p.rows.start - p.window.start
            got[:, :, p.rows.start:p.rows.stop] = outs[r][k][:, :, hl:hl + len(p.rows)]
        assert rel(got.cpu().numpy(), ref[k].cpu().numpy()) < 1e-6, k
    deps = sum(o[4] for o in outs)
    assert rel(deps.cpu().numpy(), ref[4].cpu().numpy()) < 1e-5
    # negative control: without the halo exchange the shards' edge rows are wrong
    p = plans[0]
    hl = p.rows.start - p.window.start
    alone = shard.sharded_forward_backward(spec(len(p.window)), *[to(x[:, :, p.window.start:p.window.stop])
                                                                for x in (Qh, Kh, Vh, Gh)],
                                           None, None, lambda v: None, range(hl, hl + len(p.rows)))
    edge = slice(p.rows.stop - w, p.rows.stop)
    assert rel(alone[0][:, :, edge].cpu().numpy(), ref[0][:, :, edge].cpu().numpy()) > 1e-4


@pytest.mark.parametrize("R,d,dtype,mask", [(0, 64, "f32", "none"), (1, 64, "f32", "uniform_len"),
                                            (2, 32, "f32", "uniform_len"), (3, 64, "f32", "none"),
                                            (3, 128, "bf16", "uniform_len"), (6, 64, "f32", "lognormal_len")])
def test_generic_tail_adjoint_parity(R, d, dtype, mask):
    """tail_adjoint_generic (adjoint.hpp:132-200) for tail depths 0..6 -- the reference's
    test_adjoint generic-vs-finite-difference cases run at R = 1, 2, 3 -- against the oracle's
    generic reverse pass (mode 2).  The score cotangent is materialised (k_sbar_band) and contracted
    by the RW / CW band GEMMs."""
    cfg = configs.Config(0, B=2, H=2, L=300, d=d, w=24, eps=0.3, T=8, R=R, dtype=dtype, mask=mask)
    inp = configs.make_inputs(cfg)
    g = gpu_run(cfg, inp, mode="generic_tail", duals=False)
    r = oracle(cfg, inp, precision=64, mode=2)
    r32 = oracle(cfg, inp, precision=32, mode=2)
    tol = BF16_TOL if dtype == "bf16" else FP32_TOL
    errs = {k: rel(g[k], r[k]) for k in KEYS}
    floor = {k: rel(r32[k], r[k]) for k in KEYS}
    print(f"generic tail R={R}: rel-L2 gpu / ref-f32:", {k: f"{errs[k]:.2e}/{floor[k]:.2e}" for k in KEYS})
    for k in KEYS:
        t = max(DEPS_TOL, tol) if k == "d_eps" else tol
        assert errs[k] <= max(t, (3.0 if k == "d_eps" else 1.5) * floor[k]), (k, errs)


def test_generic_tail_matches_r2_path():
    """At R = 2 the generic reverse pass and the fused one-reference path compute the same adjoint."""
    cfg = configs.CONFIGS[2].replace(L=512)
    inp = configs.make_inputs(cfg, heads=range(4))
    a = gpu_run(cfg, inp, mode="generic_tail", duals=False)
    b = gpu_run(cfg, inp, mode="one_reference", duals=False)
    for k in KEYS:
        assert rel(a[k], b[k]) <= (DEPS_TOL if k == "d_eps" else 2e-5), (k, rel(a[k], b[k]))


def _cert_inputs(cfg, inp):
    nh = len(inp.heads)
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    b = inp.bits or {}
    dev = {k: _dev(getattr(inp, k), b.get(k)).reshape(shp) for k in ("Q", "K", "V", "G")}
    rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).cuda()
    cm = None if inp.col_mask is None else torch.from_numpy(inp.col_mask).cuda()
    return dev, rm, cm, nh


@pytest.mark.parametrize("R,d,dtype,mask,sched", [(2, 64, "f32", "uniform_len", None), (0, 32, "f32", "none", None),
                                                  (1, 64, "f32", "none", [(0.6, 4), (0.3, 6)]),
                                                  (3, 128, "bf16", "uniform_len", None)])
def test_base_solve_vjp_parity(R, d, dtype, mask, sched):
    """base_solve_vjp of the tail adjoint's base cotangent (the bias certificate's c_R,
    certificates.hpp:25-70 / :112-118) against the oracle, including an epsilon schedule."""
    from paper_2605_08123_b200 import certificates
    cfg = configs.Config(0, B=2, H=2, L=260, d=d, w=20, eps=0.3, T=10, R=R, dtype=dtype, mask=mask)
    inp = configs.make_inputs(cfg)
    t, rm, cm, nh = _cert_inputs(cfg, inp)
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=R, epsilon=cfg.eps, dtype=dtype, eps_schedule=sched)
    cert = certificates.bias_certificate(t["Q"], t["K"], t["V"], t["G"], spec, R, rm, cm)
    torch.cuda.synchronize()
    r = oracle_ref.run_cert(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, eps_schedule=sched)
    r32 = oracle_ref.run_cert(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, precision=32,
                              eps_schedule=sched)
    tol = BF16_TOL if dtype == "bf16" else FP32_TOL
    for k, g in (("cQ", cert.c_q), ("cK", cert.c_k)):
        g = g.cpu().numpy().astype(np.float64).reshape(nh, cfg.rows, d)
        e, fl = rel(g, r[k]), rel(r32[k], r[k])
        print(f"base vjp R={R} {k}: rel-L2 gpu {e:.2e} ref-f32 {fl:.2e}")
        assert e <= max(tol, 1.5 * fl), (k, e, fl)
    eta = np.sqrt(np.sum(r["eta_v"] ** 2, axis=1) + np.sum(r["eta_u"] ** 2, axis=1))
    assert np.allclose(cert.eta_norm.cpu().numpy(), eta, rtol=max(tol, 1e-4) * 10)


def test_certificate_eta_decays_and_selector_is_first_feasible():
    """test_certificates.cpp:76-86 / :106-133 on the device path: ||eta_R|| strictly decreases with
    R, and the selector returns the first depth an exhaustive scan finds feasible."""
    from paper_2605_08123_b200 import certificates
    cfg = configs.Config(0, B=1, H=2, L=200, d=32, w=16, eps=0.5, T=10, R=2, dtype="f32")
    inp = configs.make_inputs(cfg)
    t, rm, cm, _ = _cert_inputs(cfg, inp)
    spec = band.BandSpec(batch=1, heads=2, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=2, epsilon=cfg.eps)
    certs = [certificates.bias_certificate(t["Q"], t["K"], t["V"], t["G"], spec, r) for r in range(5)]
    eta = np.array([c.eta_norm.cpu().numpy() for c in certs])
    assert np.all(np.diff(eta, axis=0) < 0), eta
    c_inf = [float(c.c_inf.max()) for c in certs]
    for tau in (1e3, c_inf[2] * 1.5, c_inf[4] * 0.5):
        s = certificates.select_tail_depth(t["Q"], t["K"], t["V"], t["G"], spec, tau, 4)
        want = next((r for r in range(5) if c_inf[r] <= tau), -1)
        assert s.selected == want, (tau, s.selected, want, c_inf)
    s = certificates.select_tail_depth(t["Q"], t["K"], t["V"], t["G"], spec, float(eta[1].max()) * 1.01, 4,
                                       operator_norm_bound=1.0)
    assert s.used_sufficient_bound and s.selected == 1


@pytest.mark.parametrize("dtype,w,d,mask,dustbin", [("f32", 20, 64, "uniform_len", 0), ("bf16", 20, 128, "uniform_len", 0),
                                                    ("bf16", 64, 64, "none", 0), ("f32", 64, 64, "uniform_len", 0),
                                                    ("f32", 16, 32, "none", 1), ("bf16", 128, 128, "uniform_len", 0),
                                                    ("bf16", 128, 64, "none", 0), ("bf16", 96, 128, "none", 0)])
def test_workspace_contents_do_not_matter(dtype, w, d, mask, dustbin):
    """The caller-owned workspace is scratch: a forward + backward on a workspace full of NaN bytes
    must be bit-identical to one on a zeroed workspace (guards against reads of never-written
    cells, e.g. window duals past the band or padded rows)."""
    # L = 700: several 128-row blocks per head, a partial last block; w = 128 runs the register-resident
    # full-step path (interior + edge blocks), w = 64 / 96 its generic path
    cfg = configs.Config(0, B=2, H=2, L=700 if w >= 64 else 300, d=d, w=w, eps=0.2, T=8, R=2, dtype=dtype, mask=mask,
                         dustbin=dustbin)
    inp = configs.make_inputs(cfg)
    b = inp.bits or {}
    shp = (cfg.B, cfg.H, cfg.rows, d)
    Q, K, V, G = (_dev(getattr(inp, k), b.get(k)).reshape(shp) for k in ("Q", "K", "V", "G"))
    rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).cuda()
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=d, half_band=w,
                         base_depth=cfg.T, tail_depth=2, epsilon=cfg.eps, dtype=dtype, dustbin=dustbin,
                         dustbin_cost=cfg.dustbin_cost)
    outs = []
    for fill in (0, 255):
        ws = band.Workspace()
        ws._buf = torch.full((spec.workspace_bytes() + 4096,), fill, dtype=torch.uint8, device="cuda")
        run = band.run_surrogate(Q, K, V, spec, rm, rm, workspace=ws)
        cot = band.r2_backward(run, G, workspace=ws)
        torch.cuda.synchronize()
        u, v, _ = run.tail_duals(inp.row_mask, inp.row_mask)  # the saved state's meaningful words
        outs.append([x.clone() for x in (run.output, cot.grad_q, cot.grad_k, cot.grad_v, cot.d_eps)] +
                    [torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)),
                     torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))])
    for name, a, c in zip(("O", "dQ", "dK", "dV", "d_eps", "u", "v"), *outs):
        bad = torch.nonzero(a.reshape(-1).view(torch.uint8) != c.reshape(-1).view(torch.uint8)).flatten()
        assert bad.numel() == 0, (name, bad.numel(), bad[:8].tolist())


@pytest.mark.parametrize("dtype,d,w,mask,mode", [("f32", 32, 112, "uniform_len", "one_reference"),
                                                 ("f32", 64, 96, "none", "direct_four_plan"),
                                                 ("bf16", 128, 80, "uniform_len", "one_reference")])
def test_wide_band_window_chunked_stages_parity(dtype, d, w, mask, mode):
    """Bands too wide for a 128-row SMEM tile run the window-chunked vector stages (k_bwdW: sheared
    band strips, dense chunk GEMMs): f32 and bf16 operands, masks (edge blocks, inactive rows), both
    adjoint schedules, against the oracle."""
    cfg = configs.Config(0, B=2, H=1, L=700, d=d, w=w, eps=0.1, T=12, R=2, dtype=dtype, mask=mask)
    inp = configs.make_inputs(cfg)
    tol = BF16_TOL if dtype == "bf16" else FP32_TOL
    check_against_oracle(cfg, inp, tol, tol, mode=mode)


# bf16 inputs on the dustbin config: the tensor-core solve accumulates config 3's large scores
# (|s2| ~ 115) in fp32 inside the MMA, ~1e-4 relative per score, which the score-sensitive dQ / dK
# amplify to ~1e-3 (the reference's own f32 instantiation sits at ~4e-4 there).  Stated bound:
BF16_DUSTBIN_GRAD_TOL = 2e-3


@pytest.mark.parametrize("dtype,mode", [("f32", "direct_four_plan"), ("f32", "one_reference"),
                                        ("bf16", "one_reference")])
def test_dustbin_line_kernels_parity(dtype, mode):
    """The dustbin row / column (full-length lines, split over CTAs with fixed-order partials, and the
    dustbin duals riding in the half-step launches) in both adjoint schedules and both input dtypes,
    with masked examples, against the oracle."""
    cfg = configs.CONFIGS[3].replace(B=2, H=2, L=640, dtype=dtype)
    inp = configs.make_inputs(cfg)
    if dtype == "bf16":
        check_against_oracle(cfg, inp, BF16_TOL, BF16_DUSTBIN_GRAD_TOL, mode=mode)
        return
    g, r, _ = check_against_oracle(cfg, inp, FP32_TOL, FP32_GRAD_TOL, mode=mode)
    assert np.abs(g["dQ"][:, cfg.L]).max() == 0.0
    assert np.abs(g["dK"][:, cfg.L]).max() == 0.0


def _ref_fixtures():
    import glob
    import os
    return sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_config*.npz")))


@pytest.mark.parametrize("path", _ref_fixtures(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_gpu_matches_reference_golden(path):
    """The CUDA path against the REFERENCE'S OWN outputs (tests/golden/ref_*.npz, made by the
    unmodified reference through oracle/_ref, tests/golden/make_ref_golden.py), per config."""
    import os
    z = np.load(path)
    cid = int(os.path.basename(path).split("config")[1][0])
    cfg = configs.CONFIGS[cid].replace(L=int(z["L"]))
    inp = configs.make_inputs(cfg, heads=range(len(z["heads"])))
    g = gpu_run(cfg, inp)
    keys = [str(k) for k in z["keys"]]
    floor = dict(zip(keys, z["floor"]))
    errs, bounds = {}, {}
    for k in keys:
        errs[k] = rel(g[k], z[k])
        bounds[k] = BF16_TOL if cfg.dtype == "bf16" else max(FP32_TOL, 1.5 * floor[k])
    parity_log.record(f"ref-golden-config{cid}-L{cfg.L}", cfg, inp.heads, "one_reference", errs, floor, bounds)
    print(f"reference golden config {cid} L={cfg.L}: rel-L2 gpu / ref-f32:",
          {k: f"{errs[k]:.2e}/{floor[k]:.2e}" for k in keys})
    for k in keys:
        assert errs[k] <= bounds[k], (k, errs[k], bounds[k])


@pytest.mark.parametrize("w,d,mask,L", [(128, 128, "uniform_len", 1000), (128, 64, "none", 1400), (64, 128, "uniform_len", 900),
                                        (96, 64, "none", 700)])
def test_bf16_full_step_paths_parity(w, d, mask, L):
    """The tcgen05 full-step solve (k_fstep16 + k_vmerge): its register-resident path (w = 128: interior
    and edge blocks, partial last block, masked rows / columns through -inf offsets) and its generic
    path (w = 64, 96), against the oracle."""
    cfg = configs.Config(0, B=2, H=2, L=L, d=d, w=w, eps=0.05, T=20, R=2, dtype="bf16", mask=mask,
                         in_scale=1 / np.sqrt(d))
    check_against_oracle(cfg, configs.make_inputs(cfg), BF16_TOL, BF16_TOL, case=f"fstep-w{w}-d{d}-{mask}")
