"""k_switch_coop phase timings over one replay (needs `make phase-ts`; GPU box):
mean ns from the kernel's start (block 0) to each phase boundary; every
boundary but the last is taken after a grid barrier."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi  # noqa: E402

_abi.LIB_PATH = os.environ.get("MSG_LIB", "tools/bin/libmsched_mcts.so")
import bench  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
tasks, hw, pol, _ = bench.workload(cfg, 0)
mode = bench.workload_mode(cfg)
descs = {t.id: build_descriptors(t) for t in tasks} if mode.name == "proactive" else None
sim = engine.Simulator(tasks, hw, pol, mode, descriptors=descs)
sim.run()
lib = _abi.load()
lib.msg_dbg_mc_reset()
sim.reset()
sim.run()
sim.ctx.sync()
out = (C.c_ulonglong * 11)()
lib.msg_dbg_sw_ts(out)
n = max(out[8], 1)
names = {0: "start", 1: "units plan", 2: "multisplit", 3: "evict", 4: "install", 5: "touch scan", 7: "gather"}
print(f"{cfg}: {out[8]} launches; mean us since the kernel's start")
prev = 0.0
for i, nm in names.items():
    v = out[i] / n / 1e3
    print(f"  {nm:12s} {v:7.2f}  (+{v - prev:5.2f})")
    prev = v
print(f"  window kernel end -> switch kernel start: {out[9] / max(out[10], 1) / 1e3:.2f} us (over {out[10]} launches)")
