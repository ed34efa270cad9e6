"""Multisplit timing of replays through the GPU path, the way bench.py's
roofline computes it (bytes per pass over device-timed and event-timed
launch durations), plus plan-only wall time:

  python tools/ms_devtime.py cfg2 [cfg4 ...] [--migrate] [--reps N]"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi  # noqa: E402
if os.environ.get("MSG_LIB"):
    _abi.LIB_PATH = os.environ["MSG_LIB"]
import bench  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

PEAK = 6550.1
args = [a for a in sys.argv[1:] if not a.startswith("--")]
migrate = "--migrate" in sys.argv
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
for cfg in [a for a in args if not a.isdigit()] or ["cfg2"]:
    tasks, hw, pol, _ = bench.workload(cfg, 0)
    mode = bench.workload_mode(cfg)
    descs = {t.id: build_descriptors(t) for t in tasks} if mode.name == "proactive" else None
    foot = sum(a.size_bytes for t in tasks for a in t.allocations)
    pool_bytes = min(foot, int(0.6 * os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")))
    pool_pages = 0 if pool_bytes >= foot else max(1, pool_bytes // hw.page_size_bytes)
    sim = engine.Simulator(tasks, hw, pol, mode, migrate=migrate, descriptors=descs,
                           host_pool_pages=pool_pages if migrate else 0)
    sim.run()
    walls = []
    keys = ("ms_bytes", "ms_passes", "ms_dev_launches", "ms_dev_ms", "ms_ms", "ms_ev_passes")
    d = dict.fromkeys(keys, 0)
    for _ in range(reps):
        sim.reset()   # (zeroes the context's stats)
        t0 = time.perf_counter()
        m = sim.run()
        sim.ctx.sync()
        walls.append((time.perf_counter() - t0) * 1e3)
        st = sim.ctx.stats()
        for k in keys:
            d[k] += st[k]
    per = d["ms_bytes"] / max(d["ms_passes"], 1)
    out = {"cfg": cfg, "migrate": migrate, "wall_ms": [round(w, 2) for w in walls],
           "bytes_per_pass": per, "passes": d["ms_passes"] / reps}
    if d["ms_dev_launches"]:
        dms = d["ms_dev_ms"] / d["ms_dev_launches"]
        out["dev_us"] = round(dms * 1e3, 2)
        out["dev_frac"] = round(per / (dms * 1e6) / PEAK, 4)
    if d["ms_ev_passes"]:
        ems = d["ms_ms"] / d["ms_ev_passes"]
        out["ev_us"] = round(ems * 1e3, 2)
        out["ev_frac"] = round(per / (ems * 1e6) / PEAK, 4)
    print(json.dumps(out), flush=True)
    sim.close()
