"""Top SASS instructions by stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[si].isdigit()]
tot = sum(int(r[si]) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[si]))[:top]:
    st = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i]) for i in stall_cols), reverse=True)[:3]
    print(f"{int(r[si]):6d} {100*int(r[si])/tot:5.1f}%  {r[1].strip()[:60]:60s} {st}")
