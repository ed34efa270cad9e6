"""k_ms_coop phase timings over one replay (needs `make phase-ts`; GPU box)."""
import ctypes as C, os, sys
sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi
_abi.LIB_PATH = os.environ.get("MSG_LIB", "tools/bin/libmsched_mcts.so")   # built by `make phase-ts`
from paper_2512_24637_b200 import engine, scenarios
from paper_2512_24637_b200.analyzer import build_descriptors
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tasks, hw, pol = {"cfg2": scenarios.config2_llama8b, "cfg4": scenarios.config4_llama70b}[cfg]()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), descriptors=descs)
sim.run(); sim.ctx.sync()
lib = _abi.load()
lib.msg_dbg_mc_reset()
sim.reset(); sim.run(); sim.ctx.sync()
out = (C.c_ulonglong * 49)()
lib.msg_dbg_mc_ts(out)
n = out[48]
names = ["start", "tma wait", "phase1", "hist", "barrier", "phase2", "end"]
print(f"{cfg}: {n // 148} launches; mean per-CTA elapsed since its own start (us)")
prev = 0
for i, nm in enumerate(names):
    v = out[32 + i] / n / 1e3
    print(f"{nm:9s} {v:7.2f}  (+{v - prev:5.2f})")
    prev = v
