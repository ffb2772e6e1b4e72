"""Instruction mix of one kernel in an ncu report (per work item), and the top stall lines."""
import collections, csv, subprocess, sys
rep, per = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; data = []
for r in rows:
    if 'Warp Stall Sampling (All Samples)' in r:
        hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr and len(r) > 5: data.append(r)
ei, si, wi = hdr['Instructions Executed'], hdr['Source'], hdr['Warp Stall Sampling (All Samples)']
c = collections.Counter()
f = lambda x: float(x or 0) if x.replace('.', '').isdigit() else 0.0
for r in data:
    op = r[si].strip().split()
    if not op: continue
    o = op[0] if not op[0].startswith('@') else op[1]
    c[o.split('.')[0]] += f(r[ei])
tot = sum(c.values())
print(f"total warp-instr {tot:.0f}, per item {tot/per:.0f}")
for o, n in c.most_common(22): print(f"  {o:10s} {n/per:9.0f} {n/tot*100:5.1f}%")
ws = sum(f(r[wi]) for r in data) or 1
print("top stall lines:")
for r in sorted(data, key=lambda r: -f(r[wi]))[:12]:
    print(f"  {f(r[wi])/ws*100:5.1f}% ex={r[ei]:>8} {r[si].strip()[:80]}")
