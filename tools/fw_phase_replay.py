"""k_windows_fused phase timings over one replay (needs `make phase-ts`; GPU box):
mean SM cycles from the kernel's first stamp to each phase boundary."""
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
out = (C.c_ulonglong * 17)()
lib.msg_dbg_fw_ts(out)
n = max(out[16], 1)
names = {0: "start", 1: "intervals", 2: "endpoints", 3: "labels", 4: "runs", 5: "run order", 6: "demand",
         7: "class start", 8: "E2 sorted", 9: "E2 compact", 10: "painted", 11: "keys folded", 12: "tuples sorted",
         13: "ranked", 15: "end"}
print(f"{cfg}: {out[16]} launches; mean SM cycles (and us at 1965 MHz) since the kernel's first stamp")
prev = 0.0
for i, nm in names.items():
    v = out[i] / n
    print(f"  {nm:14s} {v:8.0f} cyc {v / 1965:6.2f} us  (+{(v - prev) / 1965:5.2f})")
    prev = v
