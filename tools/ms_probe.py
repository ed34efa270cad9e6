"""Planner stats of one replay (plan-only), optionally against another build of the library.

usage: python tools/ms_probe.py cfg2|cfg4 [reps] [--lib path]
"""
import sys
import time

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi  # noqa: E402

if "--lib" in sys.argv:
    _abi.LIB_PATH = sys.argv[sys.argv.index("--lib") + 1]
from paper_2512_24637_b200 import engine, scenarios  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
tasks, hw, pol = {"cfg2": scenarios.config2_llama8b, "cfg1": scenarios.config1_gemm,
                  "cfg4": scenarios.config4_llama70b}[cfg]()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), descriptors=descs)
calls = {"n": 0, "early": 0}
orig = sim.ctx.plan_switch


def wrapped(*a, **k):
    r = orig(*a, **k)
    calls["n"] += 1
    calls["early"] += int(r[0].early_exit)
    return r


sim.ctx.plan_switch = wrapped
for r in range(reps):
    sim.reset()
    calls.update(n=0, early=0)
    s0 = sim.ctx.stats()
    t0 = time.perf_counter()
    sim.run()
    sim.ctx.sync()
    dt = time.perf_counter() - t0
    s1 = sim.ctx.stats()
    d = {k: s1[k] - s0[k] for k in ("plan_ms", "ms_ms", "ms_passes", "ms_dev_launches", "ms_dev_ms", "kernels")}
    print(f"{_abi.LIB_PATH.split('/')[-1]} rep {r}: wall {dt * 1e3:.1f} ms, plan_switch {calls['n']} "
          f"(early {calls['early']}), " + ", ".join(f"{k} {v:.2f}" if isinstance(v, float) else f"{k} {v}"
                                                     for k, v in d.items()))
sim.close()
