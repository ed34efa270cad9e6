#!/bin/bash
# Config 5 page-size sweep on cfg2 (run on the GPU box under gpurun); one bench line per page size.
O=gpurun_out/page_sweep.jsonl
: > $O
for P in 4096 8192 16384 32768 65536; do
  timeout 900 python bench.py --page-size $P --steps 2 --warmup 3 --skip-e2e --skip-execute --skip-large \
      --cpu-sample 1 2>/dev/null | tail -1 >> $O
done
python3 - <<'PY'
import json
print("page    pages/s(M)  ms/step  pages/step   H2D GB/s  D2H GB/s  duplex %  plan-only ms  CPU port pages/s(M)")
for line in open("gpurun_out/page_sweep.jsonl"):
    d = json.loads(line)
    m = d["migration"]
    page = int(d["config"]["description"].split(", ")[-1].split()[0]) * 1024
    print(f"{page:<7d} {d['value'] / 1e6:10.2f} {d['ms_per_step']:8.1f} {d['config']['pages_per_step']:>12,d} "
          f"{m['h2d_gbs']:8.1f} {m['d2h_gbs']:9.1f} {100 * m['frac_duplex']:8.1f} {d['plan_only']['ms_per_step']:12.1f} "
          f"{d['cpu_baseline']['value'] / 1e6:14.2f}")
PY
