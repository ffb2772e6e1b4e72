"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, pipe utilisation, stalls."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
idx = {n: i for i, n in enumerate(h)}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6,
         "Gbyte/s": 1e9, "Tbyte/s": 1e12, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3}
def val(v, n):
    """value in base units (bytes, bytes/s, microseconds, %)"""
    try:
        x = float(v[idx[n]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
    return x * SCALE.get(units[idx[n]], 1)
want = [
    ("duration_us", "gpu__time_duration.sum", 1),
    ("dram_read_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_write_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_GBps", "dram__bytes.sum.per_second", 1e-9),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("xu_pipe_pct(MUFU)", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("dmma_pipe_pct", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("tensor_pipe_pct(tcgen05)", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
]
for v in rows[2:]:
    name = v[idx["Kernel Name"]][:70]
    print(f"== {name}")
    for lab, n, sc in want:
        x = val(v, n)
        if x == x:
            print(f"   {lab:26s} {x * sc:12.3f}")
    st = [(n[33:], val(v, n)) for n in h if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    tot = sum(x for _, x in st if x == x) or 1
    print("   stalls: " + " ".join(f"{a}:{b / tot * 100:.0f}%" for a, b in sorted(st, key=lambda t: -t[1])[:6]))
