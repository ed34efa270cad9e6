import sys, time
sys.path.insert(0, ".")
from paper_2512_24637_b200 import scenarios
from paper_2512_24637_b200.engine import Mode
from oracle import msched_port as port
for name, fn in (("cfg1", scenarios.config1_gemm), ("cfg2", scenarios.config2_llama8b), ("cfg4", scenarios.config4_llama70b),
                 ("cfg4x8", lambda: scenarios.config4_llama70b(n_tenants=8))):
    tasks, hw, pol = fn()
    best = 1e9
    for _ in range(2 if name != "cfg4x8" else 1):
        t0 = time.perf_counter(); m = port.PortSim(tasks, hw, pol, Mode.proactive()).run(); best = min(best, time.perf_counter() - t0)
    print(name, f"{best * 1e3:.0f} ms", m.migrated_in_pages + m.migrated_out_pages + m.fault_pages, flush=True)
