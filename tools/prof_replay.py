"""One replay of a configuration through the GPU path (for ncu / nsys-free profiling)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2512_24637_b200 import engine, scenarios  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
migrate = "--migrate" in sys.argv
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 1
if cfg == "cfg3":
    from paper_2512_24637_b200.workload_extra import config3_mixed

    tasks, hw, pol = config3_mixed(hbm_bytes=16 << 30, ratio=2.0, page_size=4096, task_offset=0, timeslice_s=5e-4)
else:
    tasks, hw, pol = {"cfg2": scenarios.config2_llama8b, "cfg1": scenarios.config1_gemm,
                      "cfg4": scenarios.config4_llama70b}[cfg]()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), migrate=migrate, descriptors=descs)
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
