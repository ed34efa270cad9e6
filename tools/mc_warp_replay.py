"""Per-warp phase-1 time of k_ms_coop (after the warp's first staged piece
landed) against its block count and per-entry (slow) chunks, over the last 64
launches of one replay (needs `make phase-ts`; GPU box).

  python tools/mc_warp_replay.py cfg2"""
import collections
import ctypes as C
import os
import statistics
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
sim.reset()
sim.run()
sim.ctx.sync()
lib = _abi.load()
buf = (C.c_ulonglong * (64 * 160 * 32))()
lib.msg_dbg_mc_warp(buf)
by_slow = collections.defaultdict(list)
cta_max, cta_mean = [], []
for L in range(64):
    for c in range(148):
        ts = []
        for w in range(32):
            v = buf[(L * 160 + c) * 32 + w]
            if not v:
                continue
            ns, slow, blocks = v >> 32, (v >> 16) & 0xffff, v & 0xffff
            ts.append(ns)
            by_slow[min(slow, 8)].append(ns)
        if ts:
            cta_max.append(max(ts))
            cta_mean.append(statistics.mean(ts))
print(f"{cfg}: per-warp phase-1 ns by per-entry chunks (n warps, mean, p90, max)")
for k in sorted(by_slow):
    v = sorted(by_slow[k])
    print(f"  slow={k}{'+' if k == 8 else ' '} n={len(v):6d} mean={statistics.mean(v):8.0f} p90={v[int(0.9 * len(v))]:8.0f} max={v[-1]:8.0f}")
print(f"per CTA: mean of warp means {statistics.mean(cta_mean):.0f} ns, mean of warp maxima {statistics.mean(cta_max):.0f} ns")
