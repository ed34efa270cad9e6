"""Executed replays of cfg2 with early-start and whole-batch gating, alternating
on one context; prints each replay's wall time (GPU box)."""
import dataclasses
import sys
import time

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi  # noqa: E402

if "--lib" in sys.argv:
    _abi.LIB_PATH = sys.argv[sys.argv.index("--lib") + 1]
from paper_2512_24637_b200 import engine, scenarios  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
tasks, hw, pol = scenarios.config2_llama8b()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), migrate=True, execute=True, descriptors=descs)
modes = [("early", True), ("whole", False), ("copies-only", None)]
for r in range(reps):
    for label, early in modes:
        if early is None:
            continue
        sim.mode = dataclasses.replace(sim.mode, early_start=early)
        sim.reset()
        t0 = time.perf_counter()
        sim.run()
        sim.ctx.sync()
        dt = time.perf_counter() - t0
        st = sim.ctx.stats()
        print(f"rep {r} {label:6s} {dt * 1e3:7.1f} ms  run_ms {st['run_ms']:.1f}  h2d_busy {st['h2d_busy_ms']:.0f} "
              f"d2h_busy {st['d2h_busy_ms']:.0f}", flush=True)
sim.close()
