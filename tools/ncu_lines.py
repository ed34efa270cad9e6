"""Warp-stall samples and executed instructions aggregated per CUDA source
line, from `ncu -i REP --page source --csv --print-source cuda,sass`."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, cur, tot = {}, None, 0
hdr = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        iss = r.index("Warp Stall Sampling (All Samples)")
        iex = r.index("Instructions Executed")
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[2] == "-":      # a CUDA line row
        cur = (int(r[0]), r[1].strip()[:80])
        agg.setdefault(cur, [0, 0])
        continue
    try:
        s, e = int(r[iss] or 0), int(r[iex] or 0)
    except ValueError:
        continue
    if cur:
        agg[cur][0] += s
        agg[cur][1] += e
    tot += s
print(f"total samples {tot}")
for (ln, src), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * s / max(tot, 1):5.1f}%  L{ln:<5d} ex={e:>9d}  {src}")
