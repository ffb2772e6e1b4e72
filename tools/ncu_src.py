"""Summarise an ncu source page: top stall instructions per kernel (dev helper)."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur, hdr = [], None, None
for r in rows:
    if 'Warp Stall Sampling (All Samples)' in r:
        hdr = {h: i for i, h in enumerate(r)}
        cur = (hdr, []); blocks.append(cur); continue
    if cur is None or len(r) < 5:
        if len(r) and cur is not None and len(r) < 5: print("#", ",".join(r)[:120])
        continue
    cur[1].append(r)
for hdr, data in blocks:
    si = hdr['Warp Stall Sampling (All Samples)']
    def f(x):
        try: return float(x or 0)
        except ValueError: return 0.0
    tot = sum(f(r[si]) for r in data) or 1
    print("==== total samples", tot, "instructions", len(data))
    for r in sorted(data, key=lambda r: -f(r[si]))[:n]:
        print(f"{f(r[si])/tot*100:5.1f}%  {r[0][-5:]} ex={r[hdr['Instructions Executed']]:>8} {r[hdr['Source']].strip()[:90]}")
