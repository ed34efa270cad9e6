"""Per-CTA phase stamps of k_ms_coop over one replay (needs `make phase-ts`;
GPU box).  For each launch: CTA start skew, TMA wait, classify, histogram,
barrier arrival spread, and which CTAs arrive last.

  python tools/mc_cta_replay.py cfg2"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi  # noqa: E402

_abi.LIB_PATH = os.environ.get("MSG_LIB", "tools/bin/libmsched_mcts.so")
import bench  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tasks, hw, pol, _ = bench.workload(cfg, 0)
mode = bench.workload_mode(cfg)
descs = {t.id: build_descriptors(t) for t in tasks} if mode.name == "proactive" else None
sim = engine.Simulator(tasks, hw, pol, mode, descriptors=descs)
sim.run()
sim.ctx.sync()
lib = _abi.load()
sim.reset()
sim.run()
sim.ctx.sync()
buf = (C.c_ulonglong * (256 * 160 * 8))()
lib.msg_dbg_mc_cta(buf)
grid = 148
names = ["start", "tma", "classify", "hist", "barrier_out", "bases", "end"]
rows = []
for L in range(256):
    st = [[buf[(L * 160 + c) * 8 + i] for i in range(7)] for c in range(grid)]
    if any(s[0] == 0 for s in st):
        continue
    t0 = min(s[0] for s in st)
    rel = [[(x - t0) / 1e3 for x in s] for s in st]
    arrive = [r[3] for r in rel]      # hist stamp = barrier arrival
    last = sorted(range(grid), key=lambda c: -arrive[c])[:3]
    rows.append({
        "skew": max(r[0] for r in rel),
        "tma": statistics.mean(r[1] - r[0] for r in rel), "tma_max": max(r[1] - r[0] for r in rel),
        "cls": statistics.mean(r[2] - r[1] for r in rel), "cls_max": max(r[2] - r[1] for r in rel),
        "arr_min": min(arrive), "arr_max": max(arrive), "out": max(r[4] for r in rel),
        "bases": statistics.mean(r[5] - r[4] for r in rel), "scatter": statistics.mean(r[6] - r[5] for r in rel),
        "scatter_max": max(r[6] - r[5] for r in rel), "end": max(r[6] for r in rel), "last": last,
        "last_start": [round(rel[c][0], 2) for c in last], "last_cls": [round(rel[c][2] - rel[c][1], 2) for c in last],
    })
print(f"{cfg}: {len(rows)} launches (us from the first CTA start)")
keys = ["skew", "tma", "tma_max", "cls", "cls_max", "arr_min", "arr_max", "out", "bases", "scatter", "scatter_max",
        "end"]
print(" ".join(f"{k:>8s}" for k in keys))
for r in rows[:: max(1, len(rows) // 20)]:
    print(" ".join(f"{r[k]:8.2f}" for k in keys), r["last"], r["last_start"], r["last_cls"])
print("mean " + " ".join(f"{statistics.mean(r[k] for r in rows):8.2f}" for k in keys))
