#!/usr/bin/env python
"""Benchmark: fwd+bwd band-cells/s of the banded balanced Sinkhorn attention operator.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 2]

Workload (BASELINE.json metric on configs[1] = config 2): B=8, H=4, L=2048,
d=64, half band 64 (W=129), eps=0.05, T=50, R=2, fp32, valid lengths uniform in
[L/2, L] masked out of support and marginals; seeded synthetic inputs.
A step = st_forward + st_backward (one-reference schedule) over the batch.
value = B*H*L*W*(T+R) * n_gpus / max-over-ranks(device time per step)
(weak scaling: every rank runs its own full config-2 batch, no collective in the
operator -- batch x head partitioning).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM, FALLBACK_BF16 = 6650.0, 1590.0


def peaks():
    try:
        with open(MEASURED) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, FALLBACK_BF16, "fallback (B200_PROFILING.md)"


def workload_str(cfg):
    return (f"config{cfg.cid}: B={cfg.B},H={cfg.H},L={cfg.L},d={cfg.d},W={cfg.Wf}(|i-j|<={cfg.w}),eps={cfg.eps},"
            f"T={cfg.T},R={cfg.R},{cfg.dtype}" + (",masked" if cfg.mask != "none" else "")
            + (",dustbin" if cfg.dustbin else ""))


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm (CPU restatement, f32 template mode,
# tile_block=128) on the host cores -- the reference cannot be compiled here
# (Eigen3 / vendored headers absent), so the oracle port runs.
# ---------------------------------------------------------------------------
def cpu_sample(cfg, threads, nheads=None):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ref
    from paper_2605_08123_b200 import configs
    n = min(cfg.B * cfg.H, nheads or threads)
    inp = configs.make_inputs(cfg, heads=range(n))

    def once():
        t0 = time.perf_counter()
        oracle_ref.run(cfg, inp.Q, inp.K, inp.V, inp.G, inp.row_mask, inp.col_mask, heads=inp.heads, precision=32,
                       threads=threads, tile_block=128)
        return time.perf_counter() - t0
    cells = n * cfg.L * cfg.Wf * (cfg.T + cfg.R)
    return once, cells, n


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    once, cells, n = cpu_sample(cfg, threads)
    for _ in range(args.warmup):
        once()
    ts = [once() for _ in range(args.steps)]
    t = statistics.mean(ts)
    v = cells / t
    sample = (f"{n} of {cfg.B * cfg.H} config-{cfg.cid} heads per step (run_surrogate + r2_backward OneReference, "
              f"f32 template mode, tile_block 128), {threads} threads")
    line = {
        "impl": "reference", "metric": "fwd+bwd band-cells/s", "value": v, "unit": "band-cells/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_str(cfg), "seed": 0, "host": "cpu"},
        "cpu_baseline": {"value": v, "unit": "band-cells/s", "cores": threads, "kind": "port", "sample": sample},
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


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--mode", default="one_reference", choices=["one_reference", "direct_four_plan"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-depth", type=int, default=3, help="pipeline depth of the e2e H2D / compute / D2H overlap")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2605_08123_b200 import configs
    cfg = configs.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_08123_b200 import band

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # weak scaling: the job is world * B examples; rank r owns examples [r*B, (r+1)*B)
    # (shard.example_partition) -- independent (b, h) problems, no collective on the data path
    from paper_2605_08123_b200 import shard
    ex, heads = shard.example_partition(cfg.B, cfg.H, world, rank)
    inp = configs.make_inputs(cfg.replace(B=cfg.B * world), heads=heads)
    if inp.row_mask is not None:
        inp.row_mask, inp.col_mask = inp.row_mask[ex.start:ex.stop], inp.col_mask[ex.start:ex.stop]
    spec = band.BandSpec(batch=cfg.B, heads=cfg.H, seq_q=cfg.L, seq_k=cfg.L, head_dim=cfg.d, half_band=cfg.w,
                         base_depth=cfg.T, tail_depth=cfg.R, epsilon=cfg.eps, dtype=cfg.dtype, dustbin=cfg.dustbin,
                         dustbin_cost=cfg.dustbin_cost)
    shp = (cfg.B, cfg.H, cfg.rows, cfg.d)
    bits = inp.bits or {}

    def host(x, k):
        if k in bits:
            return torch.from_numpy(bits[k].astype(np.int16)).view(torch.bfloat16).reshape(shp)
        return torch.from_numpy(np.ascontiguousarray(x)).reshape(shp)
    hQ, hK, hV, hG = host(inp.Q, "Q"), host(inp.K, "K"), host(inp.V, "V"), host(inp.G, "G")
    Q, K, V, G = (x.to(dev) for x in (hQ, hK, hV, hG))
    rm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).to(dev)
    cm = None if inp.col_mask is None else torch.from_numpy(inp.col_mask).to(dev)
    band.validate_support(spec, inp.row_mask, inp.col_mask)  # once, outside the timed region

    O = torch.empty((cfg.B, cfg.H, cfg.rows, cfg.d), dtype=torch.float32, device=dev)
    saved = torch.empty(spec.saved_bytes(), dtype=torch.uint8, device=dev)
    grads = tuple(torch.empty_like(O) for _ in range(3))
    d_eps = torch.empty(cfg.B * cfg.H, dtype=torch.float32, device=dev)
    eta_v = torch.empty((cfg.B, cfg.H, cfg.rows), dtype=torch.float32, device=dev)
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
    ms = float(statistics.mean(ts))
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    cells = cfg.nominal_cell_steps()
    value = cells * world / (ms_max * 1e-3)

    # --- dominant kernel: one Sinkhorn full step, measured differentially ---
    # forward with T and with T + dT on the same inputs; dT full steps = dT x (row + col) launches
    dT = 20
    spec2 = band.BandSpec(**{**spec.__dict__, "base_depth": cfg.T + dT})
    ws2 = band.Workspace()
    ws2.get(spec2.workspace_bytes(), dev)
    saved2 = torch.empty(spec2.saved_bytes(), dtype=torch.uint8, device=dev)

    def fwd(sp, w_, sv):
        band.run_surrogate(Q, K, V, sp, rm, cm, out=O, saved=sv, workspace=w_, validate=False)
    with torch.cuda.stream(stream):
        tf = {}
        for key, sp, w_, sv in (("a", spec, ws, saved), ("b", spec2, ws2, saved2)):
            for _ in range(2):
                fwd(sp, w_, sv)
            xs = []
            for _ in range(5):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                fwd(sp, w_, sv)
                e.record(stream)
                torch.cuda.synchronize(dev)
                xs.append(s.elapsed_time(e))
            tf[key] = statistics.median(xs)
    step_ms = max(1e-6, (tf["b"] - tf["a"]) / dT)
    act = configs.active_cells(cfg)
    rows_cols = cfg.B * cfg.H * (cfg.rows + cfg.rows)
    alg_bytes = 4 * act + 3 * 4 * rows_cols          # one read of the active S2 band + dual read/write
    hbm, bf16, peak_src = peaks()
    achieved = alg_bytes / (step_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "step_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_full_step")
        except Exception:
            traffic = None
    exps = 2 * act
    sfu_peak = 16 * 148 * (clk.max_mhz or 1965) * 1e6
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "peak_source": peak_src,
                "kernel": "Sinkhorn full step (u and v half-steps), differential timing T vs T+20",
                "algorithmic_bytes_per_step": alg_bytes, "step_ms": step_ms,
                "step_share_of_fwd_bwd": (cfg.T + cfg.R) * step_ms / ms}
    roofline_sfu = {"bound": "sfu(ex2)", "achieved": exps / (step_ms * 1e-3) / 1e9,
                    "peak": sfu_peak / 1e9, "unit": "Gexp/s", "frac": exps / (step_ms * 1e-3) / sfu_peak,
                    "peak_source": "16 MUFU.EX2/clk/SM x 148 SMs x max SM clock (nominal)"}

    # --- e2e through the public API with pinned host buffers ---
    e2e = None
    if not args.no_e2e:
        hQ, hK, hV, hG = (x.pin_memory() for x in (hQ, hK, hV, hG))
        hrm = None if inp.row_mask is None else torch.from_numpy(inp.row_mask).pin_memory()
        hcm = None if inp.col_mask is None else torch.from_numpy(inp.col_mask).pin_memory()
        outs_h = [torch.empty(O.shape, dtype=torch.float32).pin_memory() for _ in range(4)]
        deps_h = torch.empty(cfg.B * cfg.H, dtype=torch.float32).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in (hQ, hK, hV, hG)) + \
            sum(0 if x is None else x.numel() for x in (hrm, hcm))
        d2h = sum(x.numel() * x.element_size() for x in outs_h) + deps_h.numel() * 4
        # Pipelined nb deep: step k's H2D (copy stream), fwd+bwd (compute stream) and D2H (d2h stream)
        # overlap steps k-1 / k+1; device inputs and outputs are double-buffered and ordered by events.
        # Every step still copies its own inputs in and its results out inside the timed region.
        nb = max(2, args.e2e_depth)
        din = [tuple(torch.empty_like(x) for x in (Q, K, V, G)) for _ in range(nb)]
        dms = [(None if rm is None else torch.empty_like(rm), None if cm is None else torch.empty_like(cm))
               for _ in range(nb)]
        dout = [(torch.empty_like(O), tuple(torch.empty_like(O) for _ in range(3)), torch.empty_like(d_eps),
                 torch.empty_like(eta_v), torch.empty_like(saved)) for _ in range(nb)]
        outs_hb = [[torch.empty(O.shape, dtype=torch.float32).pin_memory() for _ in range(4)] for _ in range(nb)]
        deps_hb = [torch.empty(cfg.B * cfg.H, dtype=torch.float32).pin_memory() for _ in range(nb)]
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(nb)]    # inputs of slot landed
        ev_used = [torch.cuda.Event() for _ in range(nb)]  # compute finished reading inputs / writing outputs
        ev_out = [torch.cuda.Event() for _ in range(nb)]   # outputs of slot copied to host
        for k in range(nb):
            ev_used[k].record(stream)
            ev_out[k].record(s_d2h)

        def e2e_step(k):
            b = k % nb
            (Qe, Ke, Ve, Ge), (rme, cme) = din[b], dms[b]
            Oe, gr, de, ee, sv = dout[b]
            with torch.cuda.stream(s_h2d):
                s_h2d.wait_event(ev_used[b])
                for dst, src in ((Qe, hQ), (Ke, hK), (Ve, hV), (Ge, hG), (rme, hrm), (cme, hcm)):
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
        for k in range(2 * nb):
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
        e2e = {"value": cells * world / (float(t2.item()) * 1e-3), "unit": "band-cells/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": float(t2.item()),
               "pipeline": f"{nb}-deep: H2D / fwd+bwd / D2H of consecutive steps overlap on 3 streams (pinned host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        once, ccells, n = cpu_sample(cfg, threads)
        once()
        t = once()
        cpu = {"value": ccells / t, "unit": "band-cells/s", "cores": threads, "kind": "port",
               "sample": f"{n} of {cfg.B * cfg.H} config-{cfg.cid} heads, run_surrogate + r2_backward(OneReference), "
                         f"f32 template mode, tile_block 128, {threads} threads, {t:.2f} s wall"}

    if rank == 0:
        line = {
            "metric": "fwd+bwd band-cells/s", "value": value, "unit": "band-cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": workload_str(cfg), "seed": 0, "mode": args.mode,
                       "parallelism": f"batch x head shards: {world} GPU(s) x {cfg.B} examples each, no operator collective",
                       "l2": "flushed between timed steps (256 MiB write)", "cuda_graph": graph is not None,
                       "active_cells_per_step": act, "nominal_cells_per_step": cfg.nominal_cells()},
            "roofline": roofline, "roofline_sfu": roofline_sfu, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps), "clocks": clk.summary(),
            "ms_per_step_all": [round(x, 4) for x in ts],
        }
        print(json.dumps(line, default=lambda o: o.item() if hasattr(o, "item") else str(o)), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
