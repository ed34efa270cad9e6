"""Golden fixtures for degenerate and boundary inputs, written by the REAL
reference simulator (make_golden.RecSim): empty tasks, unknown kernels with no
arguments, one-byte allocations and copies, page-straddling and overlapping
ground-truth ranges, working sets of exactly the capacity and one page more,
and more tasks than the fused window kernel takes (its fallback path).

Run in the build container (imports /root/reference):

    python tests/golden/make_golden_edge.py

Output: tests/golden/sims_edge.json.gz (read by loader.sims(), so every GPU
parity test and the oracle's golden test cover these cases).
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import make_golden as G  # noqa: E402  (imports msim and installs the recording wrappers)
from msim.core import Allocation, Arg, ByteRange, Command, CommandKind, Task  # noqa: E402
from msim.presets import get_preset  # noqa: E402
from msim.scheduler import Policy  # noqa: E402
from msim.workload import gen_vector_add  # noqa: E402

PAGE = 4096


def kern(name, args, gt, lat=2e-4):
    return Command(kind=CommandKind.KERNEL, latency_s=lat, kernel_name=name, launch_args=tuple(args),
                   ground_truth_access=tuple(ByteRange(a, n) for a, n in gt))


def h2d(dst, size, lat=1e-4):
    return Command(kind=CommandKind.MEMCPY_H2D, latency_s=lat,
                   launch_args=(Arg(0x7f0000000000), Arg(dst), Arg(size)))


def base(i):
    return (i + 1) << 40


def cases():
    out = []
    pol = Policy("rr", 1e-3)
    # 1. a task without commands next to a small streaming task
    empty = Task(id="empty", allocations=[Allocation("e0", base(0), 8 * PAGE, "empty")])
    va = gen_vector_add(24 * PAGE // 12, iterations=3, task_id="va", base_addr=base(1))
    out.append(("edge_empty_task", [empty, va], get_preset("rtx5080").with_capacity(16 * PAGE), pol))
    # 2. unknown kernels without arguments (nothing to predict: faults), mixed with known ones
    b = base(0)
    t = Task(id="noargs", allocations=[Allocation("a", b, 64 * PAGE, "noargs")])
    for r in range(4):
        t.commands.append(kern("anon", [], [(b + (8 * r) * PAGE, 8 * PAGE)]))
        t.commands.append(kern("k_ptr", [Arg(b + 32 * PAGE)], [(b + 32 * PAGE, 16 * PAGE)]))
    u = gen_vector_add(40 * PAGE // 12, iterations=3, task_id="va2", base_addr=base(1))
    out.append(("edge_unknown_kernel", [t, u], get_preset("rtx5080").with_capacity(48 * PAGE), pol))
    # 3. one-byte allocation and copies, page-straddling and overlapping/adjacent ranges
    b = base(0)
    t = Task(id="tiny", allocations=[Allocation("one", b, 1, "tiny"), Allocation("buf", b + PAGE, 20 * PAGE, "tiny")])
    t.commands += [
        h2d(b, 1),
        h2d(b + 2 * PAGE - 1, 2),                                    # straddles pages 1 and 2
        kern("k1", [Arg(b)], [(b, 1)]),
        kern("k2", [Arg(b + PAGE)], [(b + PAGE + 4095, 2), (b + PAGE, 3 * PAGE), (b + 4 * PAGE, PAGE)]),  # overlap + adjacent
        kern("k3", [Arg(b + PAGE), Arg(5)], [(b + 10 * PAGE, 1), (b + 10 * PAGE, 1), (b + 12 * PAGE - 1, 1)]),
        kern("k2", [Arg(b + PAGE)], [(b + PAGE, 6 * PAGE)]),
    ]
    v = gen_vector_add(30 * PAGE // 12, iterations=2, task_id="va3", base_addr=base(1))
    out.append(("edge_tiny_ranges", [t, v], get_preset("rtx5080").with_capacity(24 * PAGE), pol))
    # 4. two tasks whose working sets are exactly the capacity, then one page more
    for extra, name in ((0, "edge_exact_capacity"), (1, "edge_capacity_plus_one")):
        ts = []
        for i in range(2):
            bb = base(i)
            n = 16 + (extra if i == 1 else 0)
            tt = Task(id=f"x{i}", allocations=[Allocation("a", bb, n * PAGE, f"x{i}")])
            for _ in range(3):
                tt.commands.append(kern(f"sweep{i}", [Arg(bb), Arg(n * PAGE)], [(bb, n * PAGE)], lat=6e-4))
            ts.append(tt)
        out.append((name, ts, get_preset("rtx5080").with_capacity(16 * PAGE + extra * PAGE), pol))
    # 5. 20 tenants: more windows than the fused window kernel takes (16)
    ts = [gen_vector_add(6 * PAGE // 12, iterations=2, task_id=f"m{i}", base_addr=base(i)) for i in range(20)]
    out.append(("edge_many_tasks", ts, get_preset("rtx5080").with_capacity(60 * PAGE), Policy("rr", 2e-4)))
    return out


def main():
    M = G.modes_all()
    modes = ["proactive", "ideal", "um", "allocation", "late"]
    sims = []
    for name, tasks, hw, pol in cases():
        entry = {"name": name, "hw": G.enc_hw(hw), "policy": G.enc_policy(pol), "feeder": None,
                 "tasks": [G.enc_task(t) for t in tasks], "runs": {}}
        for mname in modes:
            G._CUR["case"] = name
            t0 = time.perf_counter()
            entry["runs"][mname] = {"mode": G.enc_mode(M[mname]), **G.run_case(tasks, hw, pol, M[mname])}
            r = entry["runs"][mname]
            what = r.get("error") or f"switches {r['metrics']['context_switches']}, faults {r['metrics']['fault_pages']}"
            print(f"{name:24s} {mname:11s} {time.perf_counter() - t0:6.2f}s  {what}", flush=True)
        sims.append(entry)
    with gzip.open(os.path.join(HERE, "sims_edge.json.gz"), "wt") as f:
        json.dump(sims, f)
    print("done")


if __name__ == "__main__":
    main()
