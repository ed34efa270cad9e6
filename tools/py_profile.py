"""cProfile of one plan-only replay (host-side Python overhead)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_2512_24637_b200 import engine, scenarios  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

tasks, hw, pol = scenarios.config2_llama8b()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), descriptors=descs)
sim.run()
sim.reset()
pr = cProfile.Profile()
pr.enable()
sim.run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
