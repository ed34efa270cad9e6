"""k_ms_coop phase timings on a synthetic list (needs `make phase-ts`; GPU box).

usage: python tools/mc_phase_probe.py PAGES RUN_LEN"""
import ctypes as C, random, sys
sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi
_abi.LIB_PATH = "tools/bin/libmsched_mcts.so"   # built by `make phase-ts`
from paper_2512_24637_b200._abi import Context
pages, run_len = int(sys.argv[1]), int(sys.argv[2])
rng = random.Random(1)
D = int(pages * 1.6)
ctx = Context(4096, pages)
ctx.set_domain([(0, D)])
starts = rng.sample(range(0, D // run_len), pages // run_len)
runs = sorted((s * run_len, s * run_len + run_len) for s in starts)
rng.shuffle(runs)
ctx.list_append(runs)
wins = []
for _ in range(6):
    ln = max(1, D // 120)
    wr = []
    for _ in range(40):
        s = rng.randrange(0, D - ln)
        wr.append((s, s + rng.randrange(1, ln)))
    wins.append(wr)
lib = _abi.load()
for _ in range(3):
    ctx.list_reorder(wins)
names = ["start", "tma wait", "phase1", "hist", "barrier", "phase2", "end"]
acc = [[0.0, 0.0, 0.0] for _ in names]
R = 20
out = (C.c_ulonglong * 49)()
for _ in range(R):
    lib.msg_dbg_mc_reset()
    ctx.list_reorder(wins)
    lib.msg_dbg_mc_ts(out)
    n = out[48]
    t0 = out[0]
    for i in range(7):
        acc[i][0] += (out[i] - t0) / 1e3           # earliest CTA to reach the stamp
        acc[i][1] += (out[16 + i] - t0) / 1e3      # latest CTA
        acc[i][2] += out[32 + i] / max(n, 1) / 1e3  # mean over CTAs of (stamp - own start)
print(f"launch grid {out[48]} CTAs; us from the first CTA start (earliest / latest CTA), mean per-CTA elapsed")
for i, nm in enumerate(names):
    print(f"{nm:9s} {acc[i][0] / R:7.2f} {acc[i][1] / R:7.2f}   {acc[i][2] / R:7.2f}")
