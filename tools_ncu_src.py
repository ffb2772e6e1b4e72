"""Summarise an ncu source page: top stall instructions (dev helper)."""
import csv, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) > 5]
si = idx['Warp Stall Sampling (All Samples)']
tot = sum(float(r[si] or 0) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
    print(f"{float(r[si])/tot*100:5.1f}%  {r[0][-5:]} ex={r[idx['Instructions Executed']]:>8} {r[idx['Source']].strip()[:90]}")
