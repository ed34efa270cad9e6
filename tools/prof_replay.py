"""One or more replays of a bench configuration through the GPU path (for ncu
launch lists and captures).  python tools/prof_replay.py CFG [REPS] [--migrate]"""
import os
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
migrate = "--migrate" in sys.argv
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 1
tasks, hw, pol, _ = bench.workload(cfg, 0)
mode = bench.workload_mode(cfg)
descs = {t.id: build_descriptors(t) for t in tasks} if mode.name == "proactive" else None
# migrating replays alias the pinned host pool the way bench.py does (the whole footprint may not fit host RAM)
foot = sum(a.size_bytes for t in tasks for a in t.allocations)
pool_bytes = min(foot, int(0.6 * os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")))
pool_pages = 0 if pool_bytes >= foot else max(1, pool_bytes // hw.page_size_bytes)
sim = engine.Simulator(tasks, hw, pol, mode, migrate=migrate, descriptors=descs,
                       host_pool_pages=pool_pages if migrate else 0)
for r in range(reps):
    sim.reset()
    t0 = time.perf_counter()
    m = sim.run()
    sim.ctx.sync()
    dt = time.perf_counter() - t0
    st = sim.ctx.stats()
    print(f"rep {r}: {dt * 1e3:.1f} ms wall, switches {m.context_switches}, pages {m.planned_pages}, "
          f"plan_ms {st['plan_ms']:.1f}, ms_ms {st['ms_ms']:.2f} ({st['ms_passes']} passes), kernels {st['kernels']}")
sim.close()
