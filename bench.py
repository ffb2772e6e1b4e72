#!/usr/bin/env python
"""Benchmark: fwd+bwd band-cells/s of the banded balanced Sinkhorn attention operator.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 4]

Workload (BASELINE.json metric; the largest single-GPU config = config 4):
B=4, H=8, L=32768, d=128, half band 128 (W=257), eps=0.05, T=100, R=2, bf16
Q/K/V/dO (N(0,1)/sqrt(d), seeded), fp32 duals and accumulation.  A step =
st_forward + st_backward (one-reference schedule) over the whole batch.

    value = B*H*L*W*(T+R) / max-over-ranks(device time per step)

Multi-GPU (torchrun): the B*H independent (b, h) problems of the ONE config are
split contiguously over the ranks (shard.head_partition) -- strong scaling,
no collective in the operator.  Rank 0 prints ONE JSON line.

--impl reference: the reference algorithm on the host cores (the oracle port,
tests/oracle_ref.py -> oracle/build/libstoc.so; the product library is never
loaded on that arm), on a stated bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM, FALLBACK_BF16 = 6650.0, 1590.0
EX2_PER_CLK_SM, N_SM = 16, 148          # MUFU.EX2 issue rate (15.85 measured, tools/bench_mufu.cu)
# CPU sample per reference step: rows of each sampled head (full L for configs 1-3)
SAMPLE_ROWS = {4: 4096, 5: 4096}


def peaks():
    try:
        with open(MEASURED) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, FALLBACK_BF16, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def workload_str(cfg):
    return (f"config{cfg.cid}: B={cfg.B},H={cfg.H},L={cfg.L},d={cfg.d},W={cfg.Wf}(|i-j|<={cfg.w}),eps={cfg.eps},"
            f"T={cfg.T},R={cfg.R},{cfg.dtype}" + (",masked" if cfg.mask != "none" else "")
            + (",dustbin" if cfg.dustbin else ""))


def config_obj(cfg, world, seqshard=False):
    par = (f"sequence: L={cfg.L} split contiguously over {world} GPU(s) in 128-row blocks (all {cfg.B * cfg.H} heads "
           f"per GPU), w={cfg.w}-wide halo of every dual / adjoint vector exchanged with NCCL point-to-point after "
           "each producing kernel (shard.nccl_halo)") if seqshard else \
          (f"batch x head: the {cfg.B * cfg.H} (b,h) problems split contiguously over {world} GPU(s), "
           "no operator collective")
    return {"workload": workload_str(cfg), "seed": 0, "mode": "one_reference", "parallelism": par,
            "l2": "inputs > L2 (126 MB) and a 256 MiB flush write between timed steps"}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm (CPU restatement, f32 template mode,
# tile_block=128) on the host cores.  Imports only tests/oracle_ref.py.
# ---------------------------------------------------------------------------
def cpu_sample(cfg, threads, W):
    """One bounded sample of the workload: `threads` heads (<= B*H), each its first
    SAMPLE_ROWS[cid] rows (full L for configs 1-3) at full T, R, band and epsilon."""
    import oracle_ref
    n = min(cfg.B * cfg.H, threads)
    rows = min(cfg.L, SAMPLE_ROWS.get(cfg.cid, cfg.L))
    scfg = cfg if rows == cfg.L else cfg.replace(L=rows)
    inp = W.make_inputs(scfg, heads=range(n))

    def once():
        t0 = time.perf_counter()
        oracle_ref.run(scfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, heads=inp.heads, precision=32,
                       threads=threads, tile_block=128)
        return time.perf_counter() - t0
    cells = n * rows * cfg.Wf * (cfg.T + cfg.R)
    desc = (f"{n} of {cfg.B * cfg.H} config-{cfg.cid} heads x rows [0,{rows}) of L={cfg.L} per step, full T/R/W/eps, "
            f"run_surrogate + r2_backward(OneReference), f32 template mode (bf16 inputs upcast), tile_block 128, "
            f"{threads} threads on {cpu_model()}")
    return once, cells, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle_ref
    W = oracle_ref.load_configs()   # configs.py by path, oracle RNG: libsinkattn.so is never mapped
    cfg = W.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    once, cells, desc = cpu_sample(cfg, threads, W)
    for _ in range(args.warmup):
        once()
    ts = [once() for _ in range(args.steps)]
    t = statistics.mean(ts)
    v = cells / t
    line = {
        "impl": "reference", "metric": "fwd+bwd band-cells/s", "value": v, "unit": "band-cells/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
        "config": config_obj(cfg, args.gpus, seqshard=(args.seqshard or cfg.cid == 5) and args.gpus > 1),
        "cpu_baseline": {"value": v, "unit": "band-cells/s", "cores": threads, "kind": "port", "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "band-cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line, default=lambda o: o.item() if hasattr(o, "item") else str(o)), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML sampled from a thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_traffic(cid):
    """Measured DRAM bytes per launch of the dominant kernel (ncu --set full, profiles/)."""
    p = os.path.join(ROOT, "profiles", f"traffic_config{cid}.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--mode", default="one_reference", choices=["one_reference", "direct_four_plan"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-depth", type=int, default=2, help="pipeline depth of the e2e H2D / compute / D2H overlap")
    ap.add_argument("--seqshard", action="store_true",
                    help="shard the sequence (not the heads) over the ranks; default for --config 5 (SURVEY §8(e))")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_08123_b200 import band, configs, shard

    cfg = configs.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if (args.seqshard or cfg.cid == 5) and world > 1 or args.seqshard:
        if not dist.is_initialized():  # --seqshard on one GPU without torchrun: a one-rank group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        return run_seqshard(args, cfg, rank, world, local, dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # strong scaling: rank r owns the contiguous flat head range of the ONE config
    heads = shard.head_partition(cfg.B * cfg.H, world, rank)
    nh = len(heads)
    inp = configs.make_inputs(cfg, heads=heads)
    # each owned head is its own example (batch = nh, heads = 1), carrying its example's mask row
    sel = np.array([h // cfg.H for h in heads], dtype=np.int64)
    hrm = None if inp.row_mask is None else np.ascontiguousarray(inp.row_mask[sel])
    hcm = None if inp.col_mask is None else np.ascontiguousarray(inp.col_mask[sel])
    spec = band.BandSpec(batch=nh, heads=1, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin,
                         dustbin_cost=cfg.dustbin_cost)
    shp = (nh, 1, cfg.rows, cfg.d)
    bits = inp.bits or {}

    def host(x, k):
        if k in bits:
            return torch.from_numpy(bits[k].astype(np.int16)).view(torch.bfloat16).reshape(shp)
        return torch.from_numpy(np.ascontiguousarray(x)).reshape(shp)
    hQ, hK, hV, hG = host(inp.Q, "Q"), host(inp.K, "K"), host(inp.V, "V"), host(inp.G, "G")
    del inp
    Q, K, V, G = (x.to(dev) for x in (hQ, hK, hV, hG))
    rm = None if hrm is None else torch.from_numpy(hrm).to(dev)
    cm = None if hcm is None else torch.from_numpy(hcm).to(dev)
    band.validate_support(spec, hrm, hcm)  # once, outside the timed region

    O = torch.empty(shp, dtype=torch.float32, device=dev)
    saved = torch.empty(spec.saved_bytes(), dtype=torch.uint8, device=dev)
    grads = tuple(torch.empty_like(O) for _ in range(3))
    d_eps = torch.empty(nh, dtype=torch.float32, device=dev)
    eta_v = torch.empty((nh, 1, cfg.rows), dtype=torch.float32, device=dev)
    ws = band.Workspace()
    ws.get(spec.workspace_bytes(), dev)

    def step():
        run = band.run_surrogate(Q, K, V, spec, rm, cm, out=O, saved=saved, workspace=ws, validate=False)
        band.r2_backward(run, G, mode=args.mode, grads=grads, d_eps=d_eps, eta_v=eta_v, workspace=ws)

    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        band.launch_count(reset=True)
        graph = None
        if not args.no_graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            launches_per_step = band.launch_count(reset=True)
            graph.replay()
        else:
            step()
            launches_per_step = band.launch_count(reset=True)
        torch.cuda.synchronize(dev)

        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        with ClockSampler(local) as clk:
            for s, e in evs:
                flush.zero_()
                s.record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    step()
                e.record(stream)
            torch.cuda.synchronize(dev)
        barrier()
        ts = [s.elapsed_time(e) for s, e in evs]
    del graph
    ms = float(statistics.mean(ts))
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    cells_all = cfg.nominal_cell_steps()                      # the whole config (all ranks)
    value = cells_all / (ms_max * 1e-3)

    # --- the dominant kernel: the Sinkhorn full step, measured differentially (T vs T + dT) ---
    dT = 50
    spec2 = band.BandSpec(**{**spec.__dict__, "base_depth": cfg.T + dT})
    saved2 = torch.empty(spec2.saved_bytes(), dtype=torch.uint8, device=dev)
    ws2 = band.Workspace()

    def fwd(sp, sv, w_):
        band.run_surrogate(Q, K, V, sp, rm, cm, out=O, saved=sv, workspace=w_, validate=False)
    with torch.cuda.stream(stream):
        tf, nl, xs = {}, {}, {"a": [], "b": []}
        cases = (("a", spec, saved, ws), ("b", spec2, saved2, ws2))
        for key, sp, sv, w_ in cases:
            fwd(sp, sv, w_)
            torch.cuda.synchronize(dev)
            band.launch_count(reset=True)
            fwd(sp, sv, w_)
            nl[key] = band.launch_count(reset=True)
        for _ in range(4):  # interleaved (a, b, a, b, ...): clock drift under the power cap hits both alike
            for key, sp, sv, w_ in cases:
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                fwd(sp, sv, w_)
                e.record(stream)
                torch.cuda.synchronize(dev)
                xs[key].append(s.elapsed_time(e))
        tf = {k: statistics.median(v) for k, v in xs.items()}
        del cases
        ws2 = None
    step_ms = max(1e-6, (tf["b"] - tf["a"]) / dT)
    launches_per_full_step = max(1, (nl["b"] - nl["a"]) // dT)
    launch_us = step_ms * 1e3 / launches_per_full_step

    act_all = configs.active_cells(cfg)                     # exact active edges per Sinkhorn step (all heads)
    act = act_all * nh // (cfg.B * cfg.H) if cfg.mask == "none" else act_all  # this rank's (unmasked configs)
    P_exp = EX2_PER_CLK_SM * N_SM * (clk.max_mhz or 1965) * 1e6
    hbm, bf16, peak_src = peaks()
    # SURVEY §8(d) algorithmic counts (one-reference schedule)
    n_exp = act_all * (2 * (cfg.T + cfg.R) + 5)
    n_flop = act_all * 2 * cfg.d * (cfg.T + cfg.R + 11)
    s_in = 2 if cfg.dtype == "bf16" else 4
    n_byte = cfg.B * cfg.H * cfg.rows * cfg.d * (4 * s_in + 4 * 4)
    t_s = ms_max * 1e-3
    tp = {"exp": n_exp / P_exp, "tensor": n_flop / (bf16 * 1e12), "hbm": n_byte / (hbm * 1e9)}
    # dominant kernel (per launch): 2 ex2 per active cell per full step (§8(d)); the issued count of the
    # current schedule is stated beside it
    alg_exp_launch = 2 * act / launches_per_full_step
    traffic = load_traffic(cfg.cid)
    roofline = {
        "bound": "sfu(ex2)", "unit": "Gex2/s",
        "achieved": alg_exp_launch / (launch_us * 1e-6) / 1e9, "peak": P_exp / 1e9,
        "frac": alg_exp_launch / (launch_us * 1e-6) / P_exp,
        "traffic": None if traffic is None else traffic.get("dram_bytes_per_launch"),
        "traffic_algorithmic_bytes_per_launch": None if traffic is None else traffic.get("algorithmic_bytes_per_launch"),
        "kernel": (f"Sinkhorn full step ({launches_per_full_step} launch(es)/step), differential timing T vs T+{dT}, "
                   f"CUDA events on the launching stream"),
        "per_launch_us": launch_us, "launches_per_full_step": launches_per_full_step,
        "alg_ex2_per_launch": alg_exp_launch,
        "peak_source": f"{EX2_PER_CLK_SM} MUFU.EX2/clk/SM x {N_SM} SMs x max SM clock",
        "kernel_share_of_step": (cfg.T + cfg.R) * step_ms / ms,
        "whole_step": {
            "binding": max(tp, key=tp.get), "t_roof_ms": 1e3 * max(tp.values()),
            "frac": max(tp.values()) / t_s,
            "frac_exp": tp["exp"] / t_s, "frac_tensor": tp["tensor"] / t_s, "frac_hbm": tp["hbm"] / t_s,
            "N_exp": n_exp, "N_flop": n_flop, "N_byte": n_byte,
            "model": "SURVEY §8(d): N_exp = cells(2(T+R)+5), N_flop = cells 2d(T+R+11), N_byte = BHLd(4 s_in + 4 s_out); "
                     "P_mma = measured bf16 dense, P_hbm = measured copy"},
    }

    # --- e2e through the public API with pinned host buffers ---
    e2e = None
    if not args.no_e2e:
        hQ, hK, hV, hG = (x.pin_memory() for x in (hQ, hK, hV, hG))
        hrm_t = None if hrm is None else torch.from_numpy(hrm).pin_memory()
        hcm_t = None if hcm is None else torch.from_numpy(hcm).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in (hQ, hK, hV, hG)) + \
            sum(0 if x is None else x.numel() for x in (hrm_t, hcm_t))
        # Pipelined nb deep: step k's H2D (copy stream), fwd+bwd (compute stream) and D2H (d2h stream)
        # overlap steps k-1 / k+1; device inputs / outputs are nb-buffered and ordered by events.
        # Every step copies its own inputs in and its results (O, dQ, dK, dV, d_eps) out.
        nb = max(2, args.e2e_depth)
        din = [tuple(torch.empty_like(x) for x in (Q, K, V, G)) for _ in range(nb)]
        dms = [(None if rm is None else torch.empty_like(rm), None if cm is None else torch.empty_like(cm))
               for _ in range(nb)]
        dout = [(torch.empty_like(O), tuple(torch.empty_like(O) for _ in range(3)), torch.empty_like(d_eps),
                 torch.empty_like(eta_v), torch.empty_like(saved)) for _ in range(nb)]
        outs_hb = [[torch.empty(O.shape, dtype=torch.float32).pin_memory() for _ in range(4)] for _ in range(nb)]
        deps_hb = [torch.empty(nh, dtype=torch.float32).pin_memory() for _ in range(nb)]
        d2h = sum(x.numel() * x.element_size() for x in outs_hb[0]) + deps_hb[0].numel() * 4
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(nb)]
        ev_used = [torch.cuda.Event() for _ in range(nb)]
        ev_out = [torch.cuda.Event() for _ in range(nb)]
        for k in range(nb):
            ev_used[k].record(stream)
            ev_out[k].record(s_d2h)

        def e2e_step(k):
            b = k % nb
            (Qe, Ke, Ve, Ge), (rme, cme) = din[b], dms[b]
            Oe, gr, de, ee, sv = dout[b]
            with torch.cuda.stream(s_h2d):
                s_h2d.wait_event(ev_used[b])
                for dst, src in ((Qe, hQ), (Ke, hK), (Ve, hV), (Ge, hG), (rme, hrm_t), (cme, hcm_t)):
                    if dst is not None:
                        dst.copy_(src, non_blocking=True)
                ev_in[b].record(s_h2d)
            with torch.cuda.stream(stream):
                stream.wait_event(ev_in[b])
                stream.wait_event(ev_out[b])
                run = band.run_surrogate(Qe, Ke, Ve, spec, rme, cme, out=Oe, saved=sv, workspace=ws, validate=False)
                cot = band.r2_backward(run, Ge, mode=args.mode, grads=gr, d_eps=de, eta_v=ee, workspace=ws)
                ev_used[b].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_used[b])
                for dst, src in zip(outs_hb[b], (run.output, cot.grad_q, cot.grad_k, cot.grad_v)):
                    dst.copy_(src, non_blocking=True)
                deps_hb[b].copy_(cot.d_eps, non_blocking=True)
                ev_out[b].record(s_d2h)
        for k in range(nb):
            e2e_step(k)
        torch.cuda.synchronize(dev)
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(s_h2d)
        for k in range(args.steps):
            e2e_step(k)
        s_d2h.wait_stream(stream)
        e.record(s_d2h)
        torch.cuda.synchronize(dev)
        barrier()
        ems = s.elapsed_time(e) / args.steps
        t2 = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e = {"value": cells_all / (float(t2.item()) * 1e-3), "unit": "band-cells/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": float(t2.item()),
               "pipeline": f"{nb}-deep: H2D / fwd+bwd / D2H of consecutive steps overlap on 3 streams (pinned host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle_ref
        W = oracle_ref.load_configs()
        threads = os.cpu_count() or 1
        once, ccells, desc = cpu_sample(W.CONFIGS[cfg.cid], threads, W)
        t = once()
        cpu = {"value": ccells / t, "unit": "band-cells/s", "cores": threads, "kind": "port",
               "sample": desc + f", {t:.2f} s wall", "cpu_model": cpu_model()}

    if rank == 0:
        conf = config_obj(cfg, world)
        conf.update({"cuda_graph": not args.no_graph, "mode": args.mode, "heads_per_gpu": nh,
                     "active_cells_per_step": act_all, "nominal_cells_per_step": cfg.nominal_cells()})
        line = {
            "metric": "fwd+bwd band-cells/s", "value": value, "unit": "band-cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic", "config": conf,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps), "clocks": clk.summary(),
            "ms_per_step_all": [round(x, 4) for x in ts],
        }
        print(json.dumps(line, default=lambda o: o.item() if hasattr(o, "item") else str(o)), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_seqshard(args, cfg, rank, world, local, dev):
    """Config 5 across the ranks of one node: rank r owns a contiguous block-aligned slice of the
    sequence for every head and runs the operator on its window (own rows + w-wide halos) through
    st_forward_halo / st_backward_halo; the halo of every dual and adjoint vector is completed by NCCL
    point-to-point right after the kernel that produces it (shard.nccl_halo).  value = the whole
    config's band-cells per step / max-over-ranks device time (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_08123_b200 import band, configs, shard
    plan = shard.SeqShard(L=cfg.L, w=cfg.w, world=world, rank=rank)
    win = plan.window
    hl = plan.rows.start - win.start
    own = range(hl, hl + len(plan.rows))
    inp = configs.make_inputs(cfg)
    nh = cfg.B * cfg.H
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=len(win), seq_k=len(win), head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype)
    shp = (cfg.B, cfg.H, len(win), cfg.d)

    def dev_t(k):
        x = inp.bits[k].reshape(cfg.B, cfg.H, cfg.L, cfg.d)[:, :, win.start:win.stop]
        return torch.from_numpy(np.ascontiguousarray(x).astype(np.int16)).view(torch.bfloat16).to(dev).reshape(shp)
    Q, K, V, G = (dev_t(k) for k in ("Q", "K", "V", "G"))
    del inp
    ex = shard.nccl_halo(plan)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        return shard.sharded_forward_backward(spec, Q, K, V, G, None, None, ex, own)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        band.launch_count(reset=True)
        step()
        launches = band.launch_count(reset=True)
        torch.cuda.synchronize(dev)
        dist.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(local) as clk:
            for s_, e_ in evs:
                flush.zero_()
                s_.record(stream)
                step()
                e_.record(stream)
            torch.cuda.synchronize(dev)
        dist.barrier()
    ms = float(statistics.mean(s_.elapsed_time(e_) for s_, e_ in evs))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = cfg.nominal_cell_steps() / (ms_max * 1e-3)
    if rank == 0:
        conf = config_obj(cfg, world, seqshard=True)
        conf.update({"cuda_graph": False, "rows_per_gpu": len(plan.rows), "window_per_gpu": len(win),
                     "active_cells_per_step": configs.active_cells(cfg), "nominal_cells_per_step": cfg.nominal_cells()})
        line = {"metric": "fwd+bwd band-cells/s", "value": value, "unit": "band-cells/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic", "config": conf,
                "roofline": None, "cpu_baseline": None, "e2e": None,
                "gpu_launches": int(launches * args.steps), "clocks": clk.summary()}
        print(json.dumps(line, default=lambda o: o.item() if hasattr(o, "item") else str(o)), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
