"""k_window_combine_wide (on-chip radix path) and k_window_runs (window 0's
CTA) phase timings over one replay (needs `make phase-ts`; GPU box): mean SM
cycles from each kernel's first stamp to each phase boundary.

  python tools/cw_phase_replay.py frag"""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi  # noqa: E402

_abi.LIB_PATH = os.environ.get("MSG_LIB", "tools/bin/libmsched_mcts.so")
import bench  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "frag"
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
out = (C.c_ulonglong * 34)()
lib.msg_dbg_cw_ts(out)
for title, base, names in (
        ("k_window_combine_wide", 0, {0: "start", 1: "radices+endpoints", 2: "endpoints sorted", 3: "unique E",
                                      4: "painted", 5: "covered -> X", 6: "keys sorted", 7: "ranked", 15: "end"}),
        ("k_window_runs (CTA 0)", 17, {0: "start", 1: "endpoints", 2: "sorted", 3: "unique", 4: "labels",
                                       5: "runs", 6: "run order", 15: "end"})):
    n = max(out[base + 16], 1)
    print(f"{cfg} {title}: {out[base + 16]} launches; mean SM cycles (us at 1965 MHz) since the first stamp")
    prev = 0.0
    for i, nm in names.items():
        v = out[base + i] / n
        print(f"  {nm:18s} {v:8.0f} cyc {v / 1965:6.2f} us  (+{(v - prev) / 1965:5.2f})")
        prev = v
