"""CPU census of k_ms_coop's work per CTA at a configuration (no GPU).

Replays the configuration on the oracle port, captures the eviction list and
the windows at every reorder, rebuilds the class boundaries the device's
class table has (the reorder's closed form), and classifies the
list exactly as k_ms_coop's phase 1 does: per 512-entry block (fast: one run
of consecutive ids inside one constant-class interval), else per 128-entry
chunk (fast likewise), else per entry.  Reports, per launch, the max/mean
over CTAs of slow chunks and the share of entries on each path.

  python tools/ms_block_census.py cfg2 [grid]
"""
import bisect
import statistics
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from oracle import msched_port as port  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
GRID = int(sys.argv[2]) if len(sys.argv) > 2 else 148
BLOCK, CHUNK = 512, 128
tasks, hw, pol, _ = bench.workload(cfg, 0)
mode = bench.workload_mode(cfg)
shots = []
orig = port.opt_reorder


def spy(rl, wins):
    wins = list(wins)
    bounds = set()
    for w in wins:
        for a, b in w.ordered:
            bounds.add(a)
            bounds.add(b)
    shots.append((list(rl.runs), sorted(bounds)))
    return orig(rl, wins)


port.opt_reorder = spy
port.PortSim(tasks, hw, pol, mode).run()

per_launch = []
for runs, bounds in shots:
    n = sum(b - a for a, b in runs)
    if n == 0:
        continue
    # list position -> (run index); run starts in list order
    starts, acc = [], 0
    for a, b in runs:
        starts.append(acc)
        acc += b - a
    E = -(-n // GRID)
    E = -(-E // BLOCK) * BLOCK

    def uniform(i0, i1):
        """entries [i0, i1) one run of consecutive ids with no class boundary inside"""
        r = bisect.bisect_right(starts, i0) - 1
        a, b = runs[r]
        if i1 - starts[r] > b - a:
            return False
        v0 = a + (i0 - starts[r])
        v1 = v0 + (i1 - i0)
        k = bisect.bisect_right(bounds, v0)
        return k >= len(bounds) or bounds[k] >= v1

    slow_per_cta, fast_blocks, fast_chunks, slow_chunks = [], 0, 0, 0
    for c in range(GRID):
        lo, hi = c * E, min(n, (c + 1) * E)
        s = 0
        i = lo
        while i < hi:
            j = min(hi, i + BLOCK)
            if j - i == BLOCK and uniform(i, j):
                fast_blocks += 1
            else:
                for k in range(i, j, CHUNK):
                    kk = min(j, k + CHUNK)
                    if kk - k == CHUNK and uniform(k, kk):
                        fast_chunks += 1
                    else:
                        slow_chunks += 1
                        s += 1
            i = j
        slow_per_cta.append(s)
    per_launch.append((n, len(runs), len(bounds), fast_blocks, fast_chunks, slow_chunks, max(slow_per_cta),
                       statistics.mean(slow_per_cta)))

print(f"{cfg}: {len(per_launch)} reorders, grid {GRID}")
print("entries  runs  bounds  fast512  fast128  slow128  max_slow/CTA  mean_slow/CTA")
for row in per_launch[:: max(1, len(per_launch) // 15)]:
    print("%8d %5d %7d %8d %8d %8d %12d %13.2f" % row)
tot = [sum(r[k] for r in per_launch) for k in (3, 4, 5)]
print("totals: fast blocks %d, fast chunks %d, slow chunks %d; mean max_slow/CTA %.1f" %
      (tot[0], tot[1], tot[2], statistics.mean(r[6] for r in per_launch)))
