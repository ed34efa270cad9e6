import sys, time
sys.path.insert(0, ".")
from oracle import msched_port as port
from paper_2512_24637_b200 import engine, scenarios
from paper_2512_24637_b200.analyzer import build_descriptors
for cfg in ("cfg2",):
    tasks, hw, pol = scenarios.config2_llama8b()
    t0 = time.perf_counter(); mr = port.PortSim(tasks, hw, pol, engine.Mode.um()).run(); tc = time.perf_counter() - t0
    sim = engine.Simulator(tasks, hw, pol, engine.Mode.um())
    for r in range(2):
        sim.reset(); t0 = time.perf_counter(); m = sim.run(); sim.ctx.sync(); tg = time.perf_counter() - t0
    print(cfg, "um cpu port %.1f ms gpu %.1f ms" % (tc * 1e3, tg * 1e3), m.fault_pages == mr.fault_pages, m.total_time_s == mr.total_time_s)
