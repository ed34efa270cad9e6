"""Top SASS lines by warp-stall samples from `ncu --page source --csv`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()[1:]))
hdr = rows[0]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iss] or 0), r[ia], r[isrc], r[iex]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}")
for s, a, src, ex in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  {a}  ex={ex:>8s}  {src[:90]}")
