"""cProfile of one plan-only replay (host-side Python overhead): python tools/py_profile.py [cfg]"""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tasks, hw, pol, _ = bench.workload(cfg, 0)
mode = bench.workload_mode(cfg)
descs = {t.id: build_descriptors(t) for t in tasks} if mode.name == "proactive" else None
sim = engine.Simulator(tasks, hw, pol, mode, descriptors=descs)
sim.run()
sim.reset()
pr = cProfile.Profile()
pr.enable()
sim.run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
