"""Generate the golden parity fixtures from the REAL reference simulator.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/sims.json.gz        full simulations: inputs, metrics, events,
                                   per-switch planner records
  tests/golden/predict.json.gz     per-command predictions + descriptors
  tests/golden/traces.json.gz      MSIM-TRACE v1 texts of generator outputs

The reference never implemented its per-switch dump, so the
records are captured here by wrapping `msim.engine` from the outside (the
reference tree is read-only and unmodified).  Long page lists are stored as
(length, sha1 of little-endian int64) to keep fixtures small.
"""

from __future__ import annotations

import dataclasses
import gzip
import hashlib
import json
import os
import random
import struct
import sys
import time

REF = os.environ.get("MSIM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import msim.engine as E  # noqa: E402
from msim.analyzer import build_descriptors, format_descriptors  # noqa: E402
from msim.core import Allocation, Arg, ByteRange, Command, CommandKind, PageSet, Task  # noqa: E402
from msim.memman import compute_window  # noqa: E402
from msim.predictor import ground_truth_prediction, predict, predict_allocation  # noqa: E402
from msim.presets import get_preset  # noqa: E402
from msim.scenarios import llm_scenario, streaming_scenario, uniform_scenario  # noqa: E402
from msim.scheduler import Policy  # noqa: E402
from msim.workload import (  # noqa: E402
    DEFAULT_MEM_BW, format_trace, gen_llm_like, gen_matmul, gen_template_corpus,
    gen_vector_add, task_base_addr,
)

OUT = os.path.dirname(os.path.abspath(__file__))
PAGE = 4096
GIB = 1 << 30
BIG = 64
ORDER_EVERY = {"cfg4": 40}   # big cases: digest the full order only every k-th switch


def digest(pages):
    pages = list(pages)
    if len(pages) <= BIG:
        return pages
    h = hashlib.sha1(struct.pack(f"<{len(pages)}q", *pages)).hexdigest()
    return {"n": len(pages), "sha1": h}


def flat(runs):
    return [p for a, b in runs for p in range(a, b)]


# ---------------------------------------------------------------------------
# task / config encoding (independent of any trace parser)


def enc_arg(a):
    if a.raw is not None:
        return {"raw": a.raw.hex()}
    return {"v": a.value, "w": a.width}


def enc_task(t):
    return {
        "id": t.id, "cursor": t.cursor, "priority": t.priority, "arrival_s": t.arrival_s,
        "allocations": [[a.id, a.base_addr, a.size_bytes] for a in t.allocations],
        "commands": [
            {"kind": c.kind.value, "lat": c.latency_s, "name": c.kernel_name,
             "args": [enc_arg(a) for a in c.launch_args], "grid": list(c.grid_dims),
             "block": list(c.block_dims),
             "gt": [[r.start_addr, r.length_bytes] for r in c.ground_truth_access]}
            for c in t.commands
        ],
    }


def enc_hw(hw):
    return dataclasses.asdict(hw)


def enc_policy(p):
    return dataclasses.asdict(p)


def enc_mode(m):
    return dataclasses.asdict(m)


# ---------------------------------------------------------------------------
# recording wrapper around the reference engine


class RecSim(E.Simulator):
    def __init__(self, *a, recorder=None, **kw):
        self._rec = recorder
        self._ctx = None
        super().__init__(*a, **kw)

    def _windows(self, timeline):
        out = []
        for e in timeline:
            if e.task_id in self.helpers:
                w = compute_window(self.helpers[e.task_id], e.resume_command_cursor, e.timeslice_s)
                out.append([e.task_id, e.resume_command_cursor, w.end_cursor])
        return out

    def _prepare_slice(self, entry, timeline):
        wins = E.timeline_windows(timeline, self.helpers)
        missing = PageSet(wins[0].demand_runs) - self.evlist.resident
        rec = {"ev": "switch", "task": entry.task_id, "windows": self._windows(timeline),
               "missing": len(missing)}
        self._rec.append(rec)
        self._ctx = rec
        try:
            return super()._prepare_slice(entry, timeline)
        finally:
            self._ctx = None

    def _gating_state(self, entry, window, plan, free):
        st = super()._gating_state(entry, window, plan, free)
        if self._ctx is not None:
            self._ctx["prefix"] = digest(
                st["prefix"][c] for c in range(entry.resume_command_cursor, window.end_cursor))
        return st

    def _touch(self, task, cmd, cur, timeline, entry, remaining_budget):
        missing = None
        if self.mode.name != "reference":
            missing = self.actual[task.id][cur] - self.evlist.resident
        box = {}
        orig = self.evlist.evict_head

        def spy(n):
            got = orig(n)
            box["evicted"] = got
            return got

        self.evlist.evict_head = spy
        try:
            stall = super()._touch(task, cmd, cur, timeline, entry, remaining_budget)
        finally:
            del self.evlist.evict_head
        if missing:
            self._rec.append({"ev": "touch", "task": task.id, "cmd": cur,
                              "missing": digest(flat(missing.runs)),
                              "evicted": digest(flat(box.get("evicted", [])))})
        return stall

    def _refresh_opt(self, task, cur, timeline, remaining_budget):
        head = compute_window(self.helpers[task.id], cur, max(remaining_budget, 1e-12))
        wins = [[task.id, cur, head.end_cursor]] + self._windows(timeline[1:])
        dt = super()._refresh_opt(task, cur, timeline, remaining_budget)
        self._rec.append({"ev": "refresh", "task": task.id, "cmd": cur, "windows": wins,
                          "order": digest(self.evlist.pages_in_order())})
        return dt


_orig_reorder = E.reorder_for_opt
_orig_plan = E.plan_migration
_CUR = {"sim": None}


def _reorder(evlist, timeline, helpers, windows=None):
    stats = _orig_reorder(evlist, timeline, helpers, windows)
    sim = _CUR["sim"]
    if sim is not None and sim._ctx is not None:
        sim._ctx["advised"] = list(stats.pages_advised.items())
        every = ORDER_EVERY.get(_CUR.get("case"), 1)
        sim._nswitch = getattr(sim, "_nswitch", 0) + 1
        if (sim._nswitch - 1) % every == 0:
            sim._ctx["order_after_reorder"] = digest(evlist.pages_in_order())
        sim._ctx["free"] = sim.capacity - len(evlist)
    return stats


def _plan(evlist, runs, cap):
    plan = _orig_plan(evlist, runs, cap)
    sim = _CUR["sim"]
    if sim is not None and sim._ctx is not None:
        sim._ctx["evict"] = digest(flat(plan.evict_runs))
        sim._ctx["populate"] = digest(flat(plan.populate_runs))
        sim._ctx["truncated"] = plan.truncated_pages
    return plan


E.reorder_for_opt = _reorder
E.plan_migration = _plan


def metrics_dict(m):
    d = dataclasses.asdict(m)
    d.pop("normalized_throughput", None)
    return d


def run_case(tasks, hw, policy, mode, feeder=None):
    rec = []
    t0 = time.perf_counter()
    try:
        sim = RecSim(tasks, hw, policy, mode, feeder=feeder, record_events=True, recorder=rec)
        _CUR["sim"] = sim
        m = sim.run()
    except (E.SimulationError, ValueError) as e:
        return {"error": type(e).__name__, "message": str(e), "records": rec}
    finally:
        _CUR["sim"] = None
    wall = time.perf_counter() - t0
    return {
        "metrics": metrics_dict(m),
        "events": [[e.t, e.kind, e.task_id, e.pages] for e in sim.events],
        "records": rec,
        "ref_wall_s": wall,
    }


# ---------------------------------------------------------------------------
# cases


def modes_all():
    return {
        "um": E.Mode.um(),
        "proactive": E.Mode.proactive(),
        "ideal": E.Mode.ideal(),
        "sequential": dataclasses.replace(E.Mode.proactive(), pipelined=False),
        "allocation": dataclasses.replace(E.Mode.proactive(), predictor="allocation"),
        "late": dataclasses.replace(E.Mode.proactive(), early_start=False),
        "oracle_pred": E.Mode("proactive", predictor="oracle"),
        "reference": E.Mode.reference(),
    }


def single_page_task(seq, base=1 << 40):
    npages = max(seq) + 1
    return Task(
        id="t", allocations=[Allocation("a", base, npages * PAGE, "t")],
        commands=[Command(kind=CommandKind.KERNEL, latency_s=1e-6, kernel_name=f"k{p}",
                          launch_args=(Arg(base + p * PAGE),),
                          ground_truth_access=(ByteRange(base + p * PAGE, PAGE),)) for p in seq])


def frag_tasks(n_tasks, npages, k, ncmds, seed0=0):
    tasks = []
    for i in range(n_tasks):
        base = task_base_addr(i)
        rng = random.Random(seed0 + i)
        cmds = []
        for _ in range(ncmds):
            pages = rng.sample(range(npages), k)
            cmds.append(Command(kind=CommandKind.KERNEL, latency_s=50e-6, kernel_name="scatter",
                                launch_args=(Arg(base, 64), Arg(k, 32)),
                                ground_truth_access=tuple(ByteRange(base + p * PAGE, PAGE) for p in pages)))
        tasks.append(Task(id=f"f{i}", allocations=[Allocation(f"f{i}.a", base, npages * PAGE, f"f{i}")],
                          commands=cmds))
    return tasks


def struct_tasks():
    """Kernels whose extents follow struct members, grid dims, strides and
    constant pointer offsets (test_analyzer.py:36-157 patterns)."""
    out = []
    for ti in range(2):
        base = task_base_addr(ti)
        buf = Allocation(f"s{ti}.buf", base, 64 * PAGE, f"s{ti}")
        strd = Allocation(f"s{ti}.str", base + 64 * PAGE, 64 * PAGE, f"s{ti}")
        off = Allocation(f"s{ti}.off", base + 128 * PAGE, 16 * PAGE, f"s{ti}")
        cmds = [Command(kind=CommandKind.MEMCPY_H2D, latency_s=5e-6,
                        launch_args=(Arg(0), Arg(off.base_addr), Arg(off.size_bytes)))]
        rng = random.Random(ti)
        for it in range(24):
            n = rng.randrange(1, 40)
            cmds.append(Command(kind=CommandKind.KERNEL, latency_s=20e-6, kernel_name="st",
                                launch_args=(Arg(base, 64), Arg(0, 64, raw=struct.pack("<II", n, 999 + it))),
                                ground_truth_access=(ByteRange(base, 1024 * n),)))
            g = rng.randrange(1, 30)
            cmds.append(Command(kind=CommandKind.KERNEL, latency_s=15e-6, kernel_name="gd",
                                launch_args=(Arg(base + 8 * PAGE, 64),), grid_dims=(g, 1, 1),
                                block_dims=(256, 1, 1),
                                ground_truth_access=(ByteRange(base + 8 * PAGE, 256 * 8 * g),)))
            cnt, ch = rng.randrange(2, 8), rng.randrange(16, 1024)
            cmds.append(Command(kind=CommandKind.KERNEL, latency_s=25e-6, kernel_name="sd",
                                launch_args=(Arg(strd.base_addr, 64), Arg(cnt, 32), Arg(ch, 32)),
                                ground_truth_access=tuple(ByteRange(strd.base_addr + j * 2 * PAGE, 4 * ch)
                                                          for j in range(cnt))))
            m = rng.randrange(1, 6)
            cmds.append(Command(kind=CommandKind.KERNEL, latency_s=10e-6, kernel_name="of",
                                launch_args=(Arg(off.base_addr - 64, 64), Arg(m, 32)),
                                ground_truth_access=(ByteRange(off.base_addr, 200 * m),)))
        out.append(Task(id=f"s{ti}", allocations=[buf, strd, off], commands=cmds))
    return out


def cfg1():
    hw = dataclasses.replace(get_preset("rtx5080"), hbm_capacity_bytes=16 * GIB, page_size_bytes=2 << 20)
    s = int((1.5 * 16 * GIB / 2 / 12) ** 0.5)
    tasks = [gen_matmul(s, s, s, count=8, task_id=f"mm{i}", base_addr=task_base_addr(i),
                        page_size=2 << 20) for i in range(2)]
    return tasks, hw, Policy("rr", 1.75e-3)


def llm_mix(n, layers, wbytes, kvbytes, steps, hw_bytes, page=PAGE, prefix="llm"):
    wpl = (int(wbytes / layers) // page) * page
    kv = (int(kvbytes / layers) // page) * page
    sched = [0.5 + 0.5 * (s + 1) / steps for s in range(steps)]
    tasks = [gen_llm_like(layers, wpl, kv, steps, sched, task_id=f"{prefix}{i}",
                          base_addr=task_base_addr(i), page_size=page, mem_bw=DEFAULT_MEM_BW)
             for i in range(n)]
    hw = dataclasses.replace(get_preset("rtx5080"), hbm_capacity_bytes=hw_bytes, page_size_bytes=page,
                             dram_capacity_bytes=max(256 * GIB, 2 * sum(
                                 a.size_bytes for t in tasks for a in t.allocations)))
    return tasks, hw, Policy("rr", 5e-3)


def cfg2():
    return llm_mix(3, 32, 7.6e9, 0.9e9, 8, 16 * GIB)


def cfg4():
    return llm_mix(4, 80, 70e9, 5e9, 3, int(180e9))


def build_cases(quick=False):
    HW = get_preset("rtx5080").with_capacity(96 << 20)
    M = modes_all()
    cases = []

    def add(name, tasks, hw, policy, modes, feeder_spec=None, gen=None):
        cases.append((name, tasks, hw, policy, modes, feeder_spec, gen))

    for r in (1.0, 1.5, 2.0, 3.0):
        tasks, pol = streaming_scenario(HW, r)
        add(f"stream_{r}", tasks, HW, pol, ["um", "proactive", "ideal", "sequential", "allocation",
                                            "late", "reference"],
            gen={"fn": "streaming_scenario", "ratio": r})
    tasks, pol = streaming_scenario(HW, 3.0, indirect_rate=0.01, seed=3)
    add("stream_ind", tasks, HW, pol, ["um", "proactive", "ideal", "allocation"],
        gen={"fn": "streaming_scenario", "ratio": 3.0, "indirect_rate": 0.01, "seed": 3})
    for r in (1.5, 2.0, 3.0):
        tasks, pol = llm_scenario(HW, r)
        add(f"llm_{r}", tasks, HW, pol, ["proactive", "allocation", "ideal", "um", "sequential"],
            gen={"fn": "llm_scenario", "ratio": r})
    hw16 = get_preset("rtx5080").with_capacity(16 << 20)
    tasks, pol = uniform_scenario(hw16, 8, 12 << 20)
    add("uniform_8", tasks, hw16, pol, ["proactive", "ideal"],
        gen={"fn": "uniform_scenario", "n_tasks": 8, "footprint": 12 << 20})
    rng = random.Random(1234)
    for k in range(25):
        npages = rng.randint(2, 64)
        length = rng.randint(10, 512)
        frames = rng.randint(1, 8)
        seq = [rng.randrange(npages) for _ in range(length)]
        hw = get_preset("rtx5080").with_capacity(frames * PAGE)
        add(f"opt_{k}", [single_page_task(seq)], hw, Policy("rr", 0.005), ["oracle_pred", "ideal"],
            gen={"fn": "opt", "seq": seq, "frames": frames})
    ftasks = frag_tasks(4, 256, 16, 40)
    fhw = get_preset("rtx5080").with_capacity(2 * 256 * PAGE)
    add("frag", ftasks, fhw, Policy("rr", 1e-3), ["ideal", "oracle_pred", "um"])
    corpus = gen_template_corpus(n_kernels=60, records_per=4, indirect_rate=0.02, seed=9)
    chw = get_preset("rtx5080").with_capacity(96 * PAGE)
    add("corpus", [corpus.task], chw, Policy("rr", 2e-4), ["proactive", "allocation", "ideal", "um"])
    stasks = struct_tasks()
    shw = get_preset("rtx5080").with_capacity(120 * PAGE)
    add("struct", stasks, shw, Policy("rr", 1e-4), ["proactive", "allocation", "ideal", "um", "late"])
    # priorities, arrivals, priority policy
    pt, ppol = llm_scenario(HW, 2.0, n_tasks=3, layers=6, decode_steps=4)
    pt[1].priority = 2
    pt[2].arrival_s = 0.004
    add("prio_rr", pt, HW, ppol, ["proactive", "ideal"])
    add("prio_pol", pt, HW, dataclasses.replace(ppol, kind="priority"), ["proactive", "um"])
    # live feeding (test_engine.py:262-289)
    ft, fpol = llm_scenario(HW, 1.5, n_tasks=2, layers=6, decode_steps=6)
    add("feed", ft, HW, fpol, ["proactive", "ideal"], feeder_spec={"task": ft[0].id, "split": len(ft[0].commands) // 2, "when_le": 2})
    # error paths
    big = Task(id="big", allocations=[Allocation("a", 1 << 40, 16 * PAGE, "big")],
               commands=[Command(kind=CommandKind.KERNEL, latency_s=1e-4, kernel_name="k",
                                 launch_args=(Arg(1 << 40),),
                                 ground_truth_access=(ByteRange(1 << 40, 16 * PAGE),))])
    add("err_cap", [big], get_preset("rtx5080").with_capacity(4 * PAGE), Policy("rr", 1.75e-3),
        ["um", "proactive", "ideal"])
    if not quick:
        t1, h1, p1 = cfg1()
        add("cfg1", t1, h1, p1, ["proactive", "ideal", "allocation", "um"], gen={"fn": "cfg1"})
        t2, h2, p2 = cfg2()
        add("cfg2", t2, h2, p2, ["proactive", "ideal"], gen={"fn": "cfg2"})
        t4, h4, p4 = cfg4()
        add("cfg4", t4, h4, p4, ["proactive"], gen={"fn": "cfg4"})
    return cases, M


def make_feeder(spec, tasks):
    if spec is None:
        return tasks, None
    src = next(t for t in tasks if t.id == spec["task"])
    head = Task(id=src.id, allocations=list(src.allocations), commands=list(src.commands[:spec["split"]]),
                priority=src.priority, arrival_s=src.arrival_s)
    tail = src.commands[spec["split"]:]
    state = {"fed": False}

    def feeder(sim):
        if not state["fed"] and sim.by_id[head.id].remaining() <= spec["when_le"]:
            sim.append_commands(head.id, tail)
            state["fed"] = True

    return [head if t.id == src.id else t for t in tasks], feeder


def main():
    quick = "--quick" in sys.argv
    cases, M = build_cases(quick)
    sims = []
    for name, tasks, hw, pol, modes, fspec, gen in cases:
        entry = {"name": name, "hw": enc_hw(hw), "policy": enc_policy(pol), "feeder": fspec,
                 "gen": gen, "tasks": [enc_task(t) for t in tasks], "runs": {}}
        for mname in modes:
            _CUR["case"] = name
            mtasks, feeder = make_feeder(fspec, tasks)
            t0 = time.perf_counter()
            entry["runs"][mname] = {"mode": enc_mode(M[mname]), **run_case(mtasks, hw, pol, M[mname], feeder)}
            print(f"{name:12s} {mname:12s} {time.perf_counter() - t0:7.2f}s", flush=True)
        sims.append(entry)
    with gzip.open(os.path.join(OUT, "sims.json.gz"), "wt") as f:
        json.dump(sims, f)

    # predictor-level goldens
    pred = []
    for label, task in [
        ("corpus5", gen_template_corpus(n_kernels=60, records_per=4, seed=5).task),
        ("corpus9", gen_template_corpus(n_kernels=30, records_per=4, indirect_rate=0.02, seed=9).task),
        ("struct0", struct_tasks()[0]),
        ("llm", gen_llm_like(3, 4 * PAGE, 4 * PAGE, 3, [0.25, 0.5, 1.0])),
        ("va", gen_vector_add(4096, iterations=3, indirect_rate=0.01, seed=5)),
        ("mm", gen_matmul(64, 64, 64, count=3)),
    ]:
        descs = build_descriptors(task)
        rows = []
        for c in task.commands:
            tp = predict(descs, c, PAGE)
            ap = predict_allocation(task.allocations, c, PAGE)
            gt = ground_truth_prediction(c, PAGE)
            rows.append({"template": [list(r) for r in tp.pages.runs], "complete": tp.complete,
                         "allocation": [list(r) for r in ap.pages.runs],
                         "truth": [list(r) for r in gt.pages.runs]})
        pred.append({"name": label, "task": enc_task(task), "descriptors": format_descriptors(descs),
                     "rows": rows})
    with gzip.open(os.path.join(OUT, "predict.json.gz"), "wt") as f:
        json.dump(pred, f)

    traces = {
        "va": format_trace(gen_vector_add(2048, iterations=2, task_id="va", indirect_rate=0.01, seed=5)),
        "mm": format_trace(gen_matmul(128, 256, 64, count=2, flops=1e12)),
        "llm": format_trace(gen_llm_like(3, 4 * PAGE, 2 * PAGE, 2, [0.5, 1.0])),
        "corpus": format_trace(gen_template_corpus(n_kernels=12, records_per=3, seed=1).task),
        "cfg2_task0": format_trace(cfg2()[0][0]),
        "cfg1_task1": format_trace(cfg1()[0][1]),
        "struct1": format_trace(struct_tasks()[1]),
    }
    with gzip.open(os.path.join(OUT, "traces.json.gz"), "wt") as f:
        json.dump(traces, f)
    print("done")


if __name__ == "__main__":
    main()
