"""Per-CUDA-line stall totals from an ncu report (sass,cuda source page). Dev helper."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
fname = "?"; fn = "?"; hdr = None
acc = collections.defaultdict(float); src = {}; per_fn = collections.defaultdict(float)
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) == 2 and r[0] == "Function Name": fn = r[1][:60]; continue
    if r and r[0] == "Line No": hdr = {h: i for i, h in enumerate(r)}; si = r.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) <= si: continue
    try: v = float(r[si] or 0)
    except ValueError: continue
    key = (fn, fname, r[0]); acc[key] += v; src[key] = r[1].strip()[:90]; per_fn[fn] += v
for fnn, tot in per_fn.items():
    print("====", fnn, "samples", tot)
    items = sorted([(k, v) for k, v in acc.items() if k[0] == fnn], key=lambda x: -x[1])[:n]
    for k, v in items: print(f"{v/tot*100:5.1f}% {k[1]}:{k[2]:>5} {src[k]}")
