"""Host-side time per ABI call during one replay (wall clock), to separate
host/sync overhead from kernel time."""
import collections
import sys
import time

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi, engine, scenarios  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

acc = collections.defaultdict(lambda: [0, 0.0])


def wrap(name):
    f = getattr(_abi.Context, name)

    def g(self, *a, **k):
        t0 = time.perf_counter()
        try:
            return f(self, *a, **k)
        finally:
            acc[name][0] += 1
            acc[name][1] += time.perf_counter() - t0

    setattr(_abi.Context, name, g)


for nm in ("plan_switch", "touch", "release", "list_len", "um_slice", "add_commands"):
    wrap(nm)
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if cfg == "cfg3":
    from paper_2512_24637_b200.workload_extra import config3_mixed

    tasks, hw, pol = config3_mixed(hbm_bytes=16 << 30, ratio=2.0, page_size=4096, task_offset=0, timeslice_s=5e-4)
else:
    tasks, hw, pol = {"cfg2": scenarios.config2_llama8b, "cfg1": scenarios.config1_gemm,
                      "cfg4": scenarios.config4_llama70b}[cfg]()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), descriptors=descs)
for rep in range(3):
    sim.reset()
    acc.clear()
    t0 = time.perf_counter()
    sim.run()
    sim.ctx.sync()
    wall = time.perf_counter() - t0
print(f"wall {wall * 1e3:.1f} ms")
tot = 0
for k, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    tot += t
    print(f"  {k:14s} n={n:5d} total={t * 1e3:8.2f} ms avg={t / n * 1e6:8.1f} us")
print(f"  python loop + rest: {(wall - tot) * 1e3:.1f} ms")
sim.close()
