"""Benchmark: MSched proactive memory scheduling on B200.

One step = one full replay of the configuration's trace through the GPU
path — device prediction tables resident, per switch: window build, OPT
reorder (multisplit), plan, apply, gating and touch scan on the GPU, and
the REAL migration of every planned page between pinned host DRAM and the
HBM frame arena on the copy engines.  Metric (BASELINE.json): pages
planned+migrated per second = (populate + evict + fault pages) / replay time.

The headline workload is config 4: four Llama3-70B-class
decode tenants against a 180 GB B200 HBM budget — the largest configuration
that fits one GPU.  Config 2 (3x Llama3-8B on 16 GiB) is reported as a
sub-object (`cfg2`), together with the executed-command (early start) leg.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg4|cfg2|cfg1|cfg3|cfg4x8|frag] [--page-size B] [--no-migrate]

Multi-GPU: one process per GPU (torchrun), each replaying its own
independent tenant mix under its own HBM budget (weak scaling, no
collective on the data path), bound to its GPU's NUMA
node.  Timing is on the device (CUDA events on the planner stream, all copy
streams joined), max over ranks.  `--impl reference` times the reference
itself (`msim` from baseline/_ref, its own public `Simulator.run`) on this
host's cores, one core per tenant mix (the reference is single-threaded,
SPEC.md:503); where baseline/_ref is absent, the oracle port
(oracle/msched_port.py, pinned to the reference's goldens) stands in.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pages planned+migrated/s"
UNIT = "pages/s"
CONFIGS = ["cfg4", "cfg2", "cfg1", "cfg3", "cfg4x8", "frag"]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=CONFIGS, default="cfg4")
    ap.add_argument("--page-size", type=int, default=0, help="config 5: override the page size (bytes)")
    ap.add_argument("--no-migrate", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=3, help="reference replays in the cpu_baseline sample")
    ap.add_argument("--cpu-budget-s", type=float, default=60.0,
                    help="wall budget of one CPU reference replay (fragmented configs report 'exceeded')")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-plan-only", action="store_true")
    ap.add_argument("--skip-cfg2", action="store_true", help="skip the config-2 sub-object (and its execute leg)")
    ap.add_argument("--skip-large", action="store_true", help="skip the config-4-size multisplit probe")
    ap.add_argument("--skip-execute", action="store_true", help="skip the executed-commands (early-start) leg")
    ap.add_argument("--skip-frag", action="store_true", help="skip the fragmented-configuration sub-object")
    ap.add_argument("--no-numa", action="store_true", help="do not bind the rank to its GPU's NUMA node")
    return ap.parse_args(argv)


def workload(name, rank, page=0):
    from paper_2512_24637_b200 import scenarios

    if name == "cfg1":
        tasks, hw, pol = scenarios.config1_gemm(page_size=page or (2 << 20), task_offset=2 * rank)
        desc = "2x GEMM-chain (32768^3, 8 GEMMs), 16 GiB HBM budget, RR 1.75 ms, proactive/template"
    elif name == "cfg3":
        from paper_2512_24637_b200.workload_extra import config3_mixed

        tasks, hw, pol = config3_mixed(hbm_bytes=16 << 30, ratio=2.0, page_size=page or 4096,
                                       task_offset=4 * rank, timeslice_s=5e-4)
        desc = ("stencil + SpMV (indirect x) + ResNet-style training + stencil at 2x a 16 GiB budget, "
                "RR 0.5 ms, proactive/template (faults on the SpMV gathers)")
    elif name == "cfg4":
        tasks, hw, pol = scenarios.config4_llama70b(page=page or 4096, task_offset=4 * rank)
        desc = "4x 70B-class decode (70 GB weights + 5 GB KV, 80 layers, 3 steps), 180 GB HBM budget, RR 5 ms"
    elif name == "cfg4x8":
        tasks, hw, pol = scenarios.config4_llama70b(n_tenants=8, page=page or 4096, task_offset=8 * rank)
        desc = "8x 70B-class decode (70 GB weights + 5 GB KV, 3 steps), 180 GB HBM budget (3.3x), RR 5 ms"
    elif name == "frag":
        from paper_2512_24637_b200.workload_extra import fragmented_mix

        tasks, hw, pol = fragmented_mix(page_size=page or 4096, task_offset=4 * rank)
        desc = ("fragmented: 4 tasks x 2^20-page allocations, 16 scattered single pages per command, "
                "capacity 2^21 pages, RR 1 ms, ideal predictor (SURVEY Appendix B probe, scaled up)")
    else:
        tasks, hw, pol = scenarios.config2_llama8b(page=page or 4096, task_offset=3 * rank)
        desc = ("3x Llama3-8B int8 decode (7.6 GB weights + 0.9 GB KV each, 32 layers, 8 steps), "
                "16 GiB HBM budget, RR 5 ms, proactive/template predictor")
    desc += f", {hw.page_size_bytes // 1024} KiB pages"
    return tasks, hw, pol, desc


def workload_mode(name):
    from paper_2512_24637_b200.engine import Mode

    return Mode.ideal() if name == "frag" else Mode.proactive()


# ---------------------------------------------------------------------------
# the reference itself (baseline/_ref), else the pinned port


def _ref_path():
    p = os.path.join(ROOT, "baseline", "_ref")
    return p if os.path.isdir(os.path.join(p, "msim")) else None


def reference_sim_factory(name, rank, page=0):
    """() -> object with .run() -> metrics having migrated_in/out_pages and
    fault_pages.  The reference's own Simulator from baseline/_ref when it
    is installed (tasks built by the reference's own generators with the
    same parameters as ours: the goldens pin that they are identical), else
    the oracle port on our task objects.  Returns (factory, kind, what)."""
    rp = _ref_path()
    tasks, hw, pol, _ = workload(name, rank, page)
    if rp is None:
        from oracle import msched_port as port

        mode = workload_mode(name)
        return (lambda: port.PortSim(tasks, hw, pol, mode)), "port", "oracle/msched_port.py"
    if rp not in sys.path:
        sys.path.insert(0, rp)
    import msim.engine as E
    from msim import core as mc

    from paper_2512_24637_b200.msim_plugin import to_msim_tasks

    rtasks = to_msim_tasks(mc, tasks)
    rhw = mc.HwConfig(**dataclasses.asdict(hw))
    from msim.scheduler import Policy as RPolicy

    rpol = RPolicy(kind=pol.kind, timeslice_s=pol.timeslice_s)
    rmode = E.Mode.ideal() if workload_mode(name).name == "ideal" else E.Mode.proactive()
    return (lambda: E.Simulator(rtasks, rhw, rpol, rmode)), "reference", "msim.engine.Simulator.run (baseline/_ref)"


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff,
            "python": platform.python_version()}


def time_reference(factory, reps, budget_s=None):
    """Times .run() of fresh simulators (construction — the reference's
    prediction-table build — is outside the timed region, as the GPU arm's
    `value` has its tables resident)."""
    times, m = [], None
    for _ in range(reps):
        sim = factory()
        t0 = time.perf_counter()
        if budget_s is not None:
            res = {}
            th = threading.Thread(target=lambda: res.setdefault("m", sim.run()), daemon=True)
            th.start()
            th.join(budget_s)
            if th.is_alive():
                return None, None
            m = res["m"]
        else:
            m = sim.run()
        times.append(time.perf_counter() - t0)
    return times, m


def planned(m):
    return m.migrated_in_pages + m.migrated_out_pages + m.fault_pages


def run_reference(args):
    """The reference arm: rank 0 only (other ranks exit 0), one
    single-threaded reference process per GPU-shard, each pinned to its own
    core, on the same config as our arm."""
    ws, rank, _ = dist_init()
    if rank != 0:
        return 0
    n_inst = max(1, args.gpus)
    import multiprocessing as mp

    def one(rk, q):
        try:
            os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[rk % len(os.sched_getaffinity(0))]})
        except Exception:  # noqa: BLE001
            pass
        factory, kind, what = reference_sim_factory(args.config, rk, args.page_size)
        times, m = time_reference(factory, args.warmup + args.steps)
        q.put((times[args.warmup:], planned(m), kind, what))

    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=one, args=(r, q)) for r in range(n_inst)]
    for p in procs:
        p.start()
    res = [q.get() for _ in procs]
    for p in procs:
        p.join()
    ms = max(statistics.mean(t) for t, *_ in res) * 1e3
    pages = sum(r[1] for r in res)
    value = pages / (ms / 1e3)
    kind, what = res[0][2], res[0][3]
    _, _, _, desc = workload(args.config, 0, args.page_size)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.config, "description": desc, "instances": n_inst},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_inst, "kind": kind,
                         "sample": f"{args.steps} full replays of {args.config} per core ({what}, single-threaded "
                                   "like the reference; Simulator construction outside the timed region)",
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def _cpu_child(name, page, reps, budget, q):
    """The CPU reference in a fresh interpreter pinned to one core, so the
    GPU arm's process state (pinned pools, a CUDA context, large Python heaps)
    does not slow it down."""
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[-1]})
    except Exception:  # noqa: BLE001
        pass
    factory, kind, what = reference_sim_factory(name, 0, page)
    times, m = time_reference(factory, reps, budget)
    keys = ("migrated_in_pages", "migrated_out_pages", "fault_pages", "total_time_s")
    q.put((times, None if m is None else planned(m), kind, what,
           None if m is None else {k: getattr(m, k) for k in keys}))


def cpu_baseline(args, name, page):
    """Returns (cpu_baseline object, {metric: value} of the reference's replay or None)."""
    import multiprocessing as mp

    budget = args.cpu_budget_s if name in ("cfg3", "frag") else None
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_cpu_child, args=(name, page, args.cpu_sample, budget, q), daemon=True)
    p.start()
    try:
        times, pages, kind, what, mdict = q.get(timeout=(budget or 600) * args.cpu_sample + 300)
    finally:
        p.join(timeout=5)
        if p.is_alive():
            p.kill()
    base = {"unit": UNIT, "cores": 1, "kind": kind, **host_info()}
    if times is None:
        return {**base, "value": None, "exceeded": True,
                "sample": f"one replay of {name} ({what}) exceeded the {args.cpu_budget_s:.0f} s budget"}, None
    t = statistics.median(times)
    return {**base, "value": pages / t,
            "sample": f"{args.cpu_sample} full replays of {name} ({what}; median run() {t * 1e3:.0f} ms; "
                      "fresh interpreter on one core)",
            "ms_per_replay": t * 1e3}, mdict


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md recipe)


class Clocks:
    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
                reasons = get(h)
                self.samples.append((sm, reasons))
                time.sleep(0.1)
        except Exception as e:  # noqa: BLE001
            self.error = str(e)

    def __enter__(self):
        self.max_mhz = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=2)

    def summary(self):
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
        reasons = set()
        for _, r in self.samples:
            for bit, nm in names.items():
                if r & bit:
                    reasons.add(nm)
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# host-link peaks (measured live: pinned 1 GiB copies on the copy engines)


def link_peak(torch, dev):
    """Isolated per-direction peaks, and both directions at once on two
    streams: the duplex total and each direction's own rate while the other
    runs (events on each copy stream)."""
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 0.0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = max(best, n / (a.elapsed_time(b) * 1e6))
        out[name] = best
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    best = (0.0, 0.0, 0.0)
    for _ in range(3):
        torch.cuda.synchronize(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            ev[0].record(s1)
            d.copy_(h, non_blocking=True)
            ev[1].record(s1)
        with torch.cuda.stream(s2):
            ev[2].record(s2)
            h2.copy_(d2, non_blocking=True)
            ev[3].record(s2)
        torch.cuda.synchronize(dev)
        tot = 2 * n / ((time.perf_counter() - t0) * 1e9)
        if tot > best[0]:
            best = (tot, n / (ev[0].elapsed_time(ev[1]) * 1e6), n / (ev[2].elapsed_time(ev[3]) * 1e6))
    out["duplex"], out["duplex_h2d"], out["duplex_d2h"] = best
    del h, d, h2, d2
    return out


def copy_bound_ms(h2d_bytes, d2h_bytes, pk):
    """Shortest time the host link can move these bytes: both directions
    overlap at their duplex rates until the lighter one finishes, then the
    rest runs alone at its isolated rate (engine.py:139-158's dual-CE
    pipeline, with measured rates)."""
    if not pk or not pk.get("duplex_h2d") or not pk.get("duplex_d2h"):
        return None
    th, td = h2d_bytes / (pk["duplex_h2d"] * 1e9), d2h_bytes / (pk["duplex_d2h"] * 1e9)
    if th <= td:
        rest = d2h_bytes - th * pk["duplex_d2h"] * 1e9
        t = th + rest / (pk["d2h"] * 1e9)
    else:
        rest = h2d_bytes - td * pk["duplex_h2d"] * 1e9
        t = td + rest / (pk["h2d"] * 1e9)
    return t * 1e3


# ---------------------------------------------------------------------------


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _coll_device(dist, dev):
    return "cpu" if dist.get_backend() == "gloo" else dev


def reduce_ranks(torch, xs, ws, dev, op="max"):
    if ws == 1:
        return xs
    import torch.distributed as dist

    t = torch.tensor(xs, dtype=torch.float64, device=_coll_device(dist, dev))
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


def max_over_ranks(torch, x, ws, dev):
    return reduce_ranks(torch, [x], ws, dev, "max")[0]


def sum_over_ranks(torch, x, ws, dev):
    return reduce_ranks(torch, [x], ws, dev, "sum")[0]


def multisplit_large(local, peak, reps=10):
    """The reorder multisplit at config 4's resident-list size (43.9 M pages,
    run-structured like the LLM traces: 200 K-page runs in shuffled order,
    6 windows x 40 first-access runs, two digit passes), through the C-ABI
    facade."""
    import random

    from paper_2512_24637_b200._abi import Context

    n, run = 43_900_000, 200_000
    rng = random.Random(1)
    D = int(n * 1.6)
    ctx = Context(4096, n, device=local)
    try:
        ctx.set_domain([(0, D)])
        starts = rng.sample(range(0, D // run), n // run)
        ctx.list_append([(s * run, s * run + run) for s in starts])
        wins = []
        for _ in range(6):
            ln = max(1, D // 120)
            wr = []
            for _ in range(40):
                a = rng.randrange(0, D - ln)
                wr.append((a, a + rng.randrange(1, ln)))
            wins.append(wr)
        for _ in range(3):
            ctx.list_reorder(wins)
        s0 = ctx.stats()
        for _ in range(reps):
            ctx.list_reorder(wins)
        s1 = ctx.stats()
    finally:
        ctx.close()
    passes = s1["ms_passes"] - s0["ms_passes"]
    ms = (s1["ms_ms"] - s0["ms_ms"]) / passes
    byts = (s1["ms_bytes"] - s0["ms_bytes"]) / passes
    gbs = byts / (ms * 1e6)
    return {"list_entries": n, "run_len": run, "passes": passes, "avg_launch_ms": ms,
            "algorithmic_bytes_per_launch": byts, "achieved": gbs, "peak": peak, "unit": "GB/s",
            "frac": gbs / peak}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def traffic_for(config):
    """DRAM bytes per launch of the dominant kernel from the committed
    `ncu --set full` capture for this config (newest round first)."""
    for rnd in ("r02", "r01"):
        p = os.path.join(ROOT, "profiles", rnd, f"traffic_{config}.json")
        if os.path.exists(p):
            with open(p) as f:
                return json.load(f).get("dram_bytes_per_launch"), f"profiles/{rnd}/traffic_{config}.json"
    return None, None


class Leg:
    """One Simulator replayed K times with device timing (CUDA events on the
    planner stream around run() + the join of every copy stream)."""

    def __init__(self, torch, dev, local, ws, tasks, hw, pol, mode, descs, **kw):
        from paper_2512_24637_b200 import engine

        self.torch, self.dev, self.ws = torch, dev, ws
        self.sim = engine.Simulator(tasks, hw, pol, mode, device=local, descriptors=descs, **kw)
        self.stream = torch.cuda.ExternalStream(self.sim.ctx.stream(), device=dev)

    def barrier(self):
        if self.ws > 1:
            self.torch.distributed.barrier()

    def step(self, reupload=False):
        """One replay.  reupload=True is the end-to-end step: the timed region
        also holds the public-API ingestion of the host Task objects (encode,
        H2D of the command tables, K1 prediction on the device, residency
        reset); otherwise the trace is already resident in HBM.  Inputs are
        larger than L2 and L2 is flushed before every step anyway."""
        torch, sim = self.torch, self.sim
        if not reupload:
            sim.reset()
        sim.ctx.flush_l2()
        self.barrier()
        torch.cuda.synchronize(self.dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(self.stream)
        if reupload:
            sim.reset(reupload=True)
        m = sim.run()
        sim.ctx.sync()
        b.record(self.stream)
        b.synchronize()
        torch.cuda.synchronize(self.dev)
        self.barrier()
        return a.elapsed_time(b), m

    def timed(self, steps, warmup, clocks=None):
        for _ in range(warmup):
            self.step()
        k0 = self.sim.ctx.stats()["kernels"]
        acc, times, m = None, [], None
        for _ in range(steps):
            ms, m = self.step()
            times.append(ms)
            st = self.sim.ctx.stats()   # step() resets the context: these are this step's counters
            if acc is None:
                acc = {k: 0 for k in st}
            for k, v in st.items():
                acc[k] += v if k != "kernels" else 0
        launches = self.sim.ctx.stats()["kernels"] - k0
        return times, m, {k: v / steps for k, v in acc.items()}, launches

    def close(self):
        self.sim.close()


def multisplit_roofline(st, hbm_peak, traffic=None, traffic_src=None):
    ms_bytes = st["ms_bytes"] / max(st["ms_passes"], 1)
    dev_timed = None
    if st.get("ms_dev_launches"):
        dms = st["ms_dev_ms"] / st["ms_dev_launches"]
        dev_timed = {"avg_launch_ms": dms, "achieved": ms_bytes / (dms * 1e6),
                     "frac": ms_bytes / (dms * 1e6) / hbm_peak, "launches_per_step": st["ms_dev_launches"]}
    ev_passes = st.get("ms_ev_passes", st["ms_passes"])
    if ev_passes and 2 * ev_passes >= st["ms_passes"]:
        # standalone launches (the synchronous, migrating path): CUDA events around each launch
        ms_kernel_ms = st["ms_ms"] / ev_passes
        timing = "CUDA events on the planner stream around each launch, averaged over the timed steps"
        launches = ev_passes
    elif dev_timed:
        # the async path runs the multisplit as a phase of its per-switch cooperative kernel: there is no
        # launch of its own to bracket with events, so the device clock is the timing
        ms_kernel_ms = dev_timed["avg_launch_ms"]
        timing = ("%globaltimer on the device, first CTA start to last CTA end of the multisplit phase inside "
                  "the per-switch cooperative kernel (k_switch_coop), averaged over the timed steps")
        launches = st["ms_dev_launches"]
    else:
        ms_kernel_ms, timing, launches = 0.0, "no multisplit ran", 0
    achieved = ms_bytes / (ms_kernel_ms * 1e6) if ms_kernel_ms else 0.0
    return {"bound": "hbm", "kernel": "reorder multisplit (k_ms_coop: TMA-staged, one grid barrier per pass)",
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak if hbm_peak else None, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": ms_bytes,
            "algorithmic_bytes_per_unit": "8 B per list entry (4 B id read + 4 B written) per digit pass",
            "avg_launch_ms": ms_kernel_ms, "launches_per_step": launches,
            "timing": timing, "device_timed": dev_timed}


def migration_summary(st, ms_step, pk, ws, link_all):
    h2d = st["h2d_bytes"] / (st["h2d_busy_ms"] * 1e6) if st["h2d_busy_ms"] else 0.0
    d2h = st["d2h_bytes"] / (st["d2h_busy_ms"] * 1e6) if st["d2h_busy_ms"] else 0.0
    both = (st["h2d_bytes"] + st["d2h_bytes"]) / (ms_step * 1e6)
    bound = copy_bound_ms(st["h2d_bytes"], st["d2h_bytes"], pk)
    return {"h2d_gbs": h2d, "d2h_gbs": d2h, "h2d_bytes_per_step": st["h2d_bytes"],
            "d2h_bytes_per_step": st["d2h_bytes"], "duplex_gbs_over_step": both,
            "peak_h2d_gbs": pk["h2d"], "peak_d2h_gbs": pk["d2h"], "peak_duplex_gbs": pk["duplex"],
            "peak_duplex_h2d_gbs": pk["duplex_h2d"], "peak_duplex_d2h_gbs": pk["duplex_d2h"],
            "frac_h2d": h2d / pk["h2d"] if pk["h2d"] else None,
            "frac_d2h": d2h / pk["d2h"] if pk["d2h"] else None,
            "frac_duplex": both / pk["duplex"] if pk["duplex"] else None,
            "copy_bound_ms": bound, "frac_of_copy_bound": (bound / ms_step) if bound else None,
            "copy_bound": "both directions overlapped at their measured duplex rates until the lighter one "
                          "ends, the rest at the isolated rate; frac_of_copy_bound = that time / replay time",
            "all_ranks_gbs": link_all["bytes"] / (ms_step * 1e6),
            "all_ranks_peak_duplex_gbs": link_all["peak"],
            "all_ranks_frac_duplex": (link_all["bytes"] / (ms_step * 1e6)) / link_all["peak"]
            if link_all["peak"] else None,
            "peak_kind": "measured live on every rank at once: pinned 1 GiB cudaMemcpyAsync per direction, and "
                         "both directions together on two streams (duplex), best of 3",
            "ce_batches": st["ce_batches"], "sm_batches": st["sm_batches"],
            "segments_per_step": st["h2d_segments"] + st["d2h_segments"]}


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    import torch

    ws, rank, local = dist_init()
    # test hook: ranks share the visible GPU(s) and talk over gloo, so the
    # multi-rank path can be exercised on a one-GPU box (the driver's N-GPU
    # runs use one GPU per rank and NCCL)
    shared = os.environ.get("MSG_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % max(torch.cuda.device_count(), 1)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    placement = None
    if not args.no_numa:
        from paper_2512_24637_b200.placement import bind_to_gpu

        try:
            placement = bind_to_gpu(local)
        except Exception as e:  # noqa: BLE001
            placement = {"error": str(e)}
    if ws > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2512_24637_b200.analyzer import build_descriptors

    tasks, hw, pol, desc = workload(args.config, rank, args.page_size)
    mode = workload_mode(args.config)
    descs = {t.id: build_descriptors(t) for t in tasks} if mode.name == "proactive" else None
    # every rank measures its own link at the same time (shared host memory
    # bandwidth under N concurrent migrators is part of the ceiling)
    if ws > 1:
        torch.distributed.barrier()
    pk = link_peak(torch, dev)
    peak_all = sum_over_ranks(torch, pk["duplex"], ws, dev)
    migrate = not args.no_migrate
    # pinned backing store: the whole footprint when it fits in this rank's
    # share of host RAM (60 %), else a bounded pool whose slots alias
    # (bandwidth-faithful; payload verification needs an unaliased pool)
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")

    def pool_for(tasks, hw):
        foot = sum(a.size_bytes for t in tasks for a in t.allocations)
        pool_bytes = min(foot, int(0.6 * host_ram / max(local_ws, 1)))
        return 0 if pool_bytes >= foot else max(1, pool_bytes // hw.page_size_bytes)

    pool_pages = pool_for(tasks, hw)
    leg = Leg(torch, dev, local, ws, tasks, hw, pol, mode, descs, migrate=migrate, host_pool_pages=pool_pages)
    with Clocks(local) as clk:
        times, m, st, launches_total = leg.timed(args.steps, args.warmup)
    ms_step = max_over_ranks(torch, statistics.mean(times), ws, dev)
    pages_step = sum_over_ranks(torch, m.planned_pages, ws, dev)
    link_bytes_all = sum_over_ranks(torch, st["h2d_bytes"] + st["d2h_bytes"], ws, dev)
    value = pages_step / (ms_step / 1e3)
    # e2e: the public API from host Task objects every step (encode, H2D of
    # the command tables, K1 prediction on the device, replay, metrics back)
    e2e = None
    if not args.skip_e2e:
        e_times, io = [], []
        for _ in range(max(1, min(args.steps, args.e2e_steps))):
            b0 = (leg.sim.ctx.h2d_bytes, leg.sim.ctx.d2h_bytes)
            ms_e, _ = leg.step(reupload=True)
            e_times.append(ms_e)
            io.append((leg.sim.ctx.h2d_bytes - b0[0], leg.sim.ctx.d2h_bytes - b0[1]))
        e_ms = max_over_ranks(torch, statistics.mean(e_times), ws, dev)
        e2e = {"value": pages_step / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(io[-1][0]),
               "d2h_bytes_per_step": int(io[-1][1]), "ms_per_step": e_ms, "steps": len(e_times),
               "includes": "inside the timed region: host Task objects -> encode -> H2D of the command tables "
                           "(pageable numpy buffers) -> device K1 prediction -> residency reset -> replay ("
                           + ("migration off" if args.no_migrate else "with real migration")
                           + ") -> per-switch results D2H -> metrics"}
    leg.close()
    # planning only: the same replay with the copies switched off -- the work
    # the reference itself does (it models migration time, it moves no bytes)
    plan_only = None
    if not args.skip_plan_only and migrate:
        pl = Leg(torch, dev, local, ws, tasks, hw, pol, mode, descs, migrate=False)
        p_times, _, pst, p_launch = pl.timed(args.steps, args.warmup)
        pl.close()
        p_ms = max_over_ranks(torch, statistics.mean(p_times), ws, dev)
        plan_only = {"value": pages_step / (p_ms / 1e3), "unit": UNIT, "ms_per_step": p_ms,
                     "multisplit_ms_per_step": pst["ms_ms"] if pst.get("ms_ev_passes") else pst["ms_dev_ms"],
                     "planner_stream_ms_per_step": pst["plan_ms"],
                     "gpu_launches_per_step": p_launch // max(args.steps, 1),
                     "roofline": multisplit_roofline(pst, load_peaks().get("hbm_gbs", 6550.0)),
                     "note": "replay with migration off: the reference's own work (plans + modeled timing)"}
    # config 2 as a sub-object (the round-1 headline), and the executed
    # command (early start) leg on it
    cfg2 = None
    execute = None
    # the sub-objects (config 2, executed commands, fragmented) are single-GPU
    # evidence: a scaling run (N > 1) times the headline and plan-only only
    sub_legs = ws == 1
    if sub_legs and not args.skip_cfg2 and args.config != "cfg2" and migrate:
        t2, h2, p2, d2 = workload("cfg2", rank, args.page_size)
        descs2 = {t.id: build_descriptors(t) for t in t2}
        mode2 = workload_mode("cfg2")
        l2 = Leg(torch, dev, local, ws, t2, h2, p2, mode2, descs2, migrate=True,
                 host_pool_pages=pool_for(t2, h2))
        c_times, c_m, cst, _ = l2.timed(min(args.steps, 5), min(args.warmup, 3))
        l2.close()
        c_ms = max_over_ranks(torch, statistics.mean(c_times), ws, dev)
        c_pages = sum_over_ranks(torch, c_m.planned_pages, ws, dev)
        c_link = sum_over_ranks(torch, cst["h2d_bytes"] + cst["d2h_bytes"], ws, dev)
        tr2, tr2src = traffic_for("cfg2")
        cfg2 = {"description": d2, "value": c_pages / (c_ms / 1e3), "unit": UNIT, "ms_per_step": c_ms,
                "steps": len(c_times),
                "roofline": multisplit_roofline(cst, load_peaks().get("hbm_gbs", 6550.0), tr2, tr2src),
                "migration": migration_summary(cst, c_ms, pk, ws, {"bytes": c_link, "peak": peak_all})}
        pl2 = Leg(torch, dev, local, ws, t2, h2, p2, mode2, descs2, migrate=False)
        q_times, _, qst, _ = pl2.timed(min(args.steps, 5), min(args.warmup, 3))
        pl2.close()
        q_ms = max_over_ranks(torch, statistics.mean(q_times), ws, dev)
        cfg2["plan_only"] = {"value": c_pages / (q_ms / 1e3), "ms_per_step": q_ms,
                             "roofline": multisplit_roofline(qst, load_peaks().get("hbm_gbs", 6550.0))}
        if not args.skip_execute:
            execute = execute_leg(torch, dev, local, ws, t2, h2, p2, mode2, descs2, pool_for(t2, h2), args)
    elif sub_legs and not args.skip_execute and migrate:
        execute = execute_leg(torch, dev, local, ws, tasks, hw, pol, mode, descs, pool_pages, args)
    frag = None
    if sub_legs and not args.skip_frag and args.config != "frag" and migrate:
        frag = frag_leg(torch, dev, local, ws, args, pk, peak_all, pool_for)
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6550.0)
    traffic, tsrc = traffic_for(args.config)
    roof = multisplit_roofline(st, hbm_peak, traffic, tsrc)
    roof["peak_source"] = "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6550 GB/s"
    large = None if (args.skip_large or args.config.startswith("cfg4")) else multisplit_large(local, hbm_peak)
    cpu, cpu_m = cpu_baseline(args, args.config, args.page_size)
    mig = migration_summary(st, ms_step, pk, ws, {"bytes": link_bytes_all, "peak": peak_all}) if migrate else None
    keys = ("migrated_in_pages", "migrated_out_pages", "fault_pages", "total_time_s")
    parity = {"metrics_equal_reference": None if cpu_m is None else
              {k: getattr(m, k) for k in keys} == cpu_m,
              "checked_against": cpu.get("kind")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.config, "description": desc, "migration": "real" if migrate else "off",
                   "l2": "inputs larger than L2, and L2 flushed between steps (256 MiB write)",
                   "pages_per_step": pages_step,
                   "host_pool": "whole footprint" if pool_pages == 0 else f"{pool_pages} pages (aliased)"},
        "roofline": roof,
        "roofline_large_list": large,
        "migration": mig,
        "plan_only": plan_only,
        "cfg2": cfg2,
        "frag": frag,
        "execute": execute,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches_total), "gpu_launches_per_step": int(launches_total // max(args.steps, 1)),
        "placement": placement,
        "clocks": clk.summary(),
        "parity": parity,
    }
    print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def frag_leg(torch, dev, local, ws, args, pk, peak_all, pool_for):
    """The fragmented regime the reference collapses on:
    scattered single pages, one eviction-list run per page, the migration on
    the SM gather/scatter kernel.  Parity at full size is out of the CPU's
    reach (the reference's run-list madvise is O(pages^2.3)); it is checked
    here at a reduced size against the oracle port (and in tests against the
    reference's own goldens, tests/golden/sims_frag.json.gz)."""
    from oracle import msched_port as port
    from paper_2512_24637_b200.workload_extra import fragmented_mix

    tasks, hw, pol, desc = workload("frag", int(os.environ.get("RANK", "0")))
    mode = workload_mode("frag")
    lg = Leg(torch, dev, local, ws, tasks, hw, pol, mode, None, migrate=True, host_pool_pages=pool_for(tasks, hw))
    f_times, f_m, fst, _ = lg.timed(min(args.steps, 3), 1)
    lg.close()
    f_ms = max_over_ranks(torch, statistics.mean(f_times), ws, dev)
    f_pages = sum_over_ranks(torch, f_m.planned_pages, ws, dev)
    f_link = sum_over_ranks(torch, fst["h2d_bytes"] + fst["d2h_bytes"], ws, dev)
    out = {"description": desc, "value": f_pages / (f_ms / 1e3), "unit": UNIT, "ms_per_step": f_ms,
           "steps": len(f_times), "switches": f_m.context_switches,
           "roofline": multisplit_roofline(fst, load_peaks().get("hbm_gbs", 6550.0)),
           "migration": migration_summary(fst, f_ms, pk, ws, {"bytes": f_link, "peak": peak_all}),
           "gather_gbs": {"h2d": fst["h2d_bytes"] / (fst["h2d_busy_ms"] * 1e6) if fst["h2d_busy_ms"] else None,
                          "d2h": fst["d2h_bytes"] / (fst["d2h_busy_ms"] * 1e6) if fst["d2h_busy_ms"] else None,
                          "note": "k_sm_copy (one warp per 4 KiB page, 16-byte accesses over mapped pinned memory), "
                                  "busy time by CUDA events around the gather/scatter launches"}}
    # the CPU reference at full size, bounded
    cpu, _ = cpu_baseline(argparse.Namespace(cpu_sample=1, cpu_budget_s=min(args.cpu_budget_s, 20.0)), "frag", 0)
    out["cpu_baseline"] = cpu
    # parity at the reduced size of the golden `frag_s` case
    small = dict(npages=2048, ncmds=60, capacity_pages=1024)
    st_, sh, sp = fragmented_mix(**small)
    from paper_2512_24637_b200 import engine

    sim = engine.Simulator(st_, sh, sp, mode, migrate=True, verify=True, device=local)
    try:
        mg = sim.run()
        bad = sim.ctx.verify()
    finally:
        sim.close()
    mc = port.PortSim(st_, sh, sp, mode).run()
    keys = ("migrated_in_pages", "migrated_out_pages", "fault_pages", "total_time_s", "context_switches")
    out["parity"] = {"metrics_equal_oracle": {k: getattr(mg, k) for k in keys} == {k: getattr(mc, k) for k in keys},
                     "payloads_verified": bad == 0, "size": small,
                     "note": "full size exceeds the CPU budget; the reduced size is the golden frag_s case"}
    return out


def execute_leg(torch, dev, local, ws, tasks, hw, pol, mode, descs, pool_pages, args):
    """Executed commands: every command of every slice runs on the device as
    a kernel reading its pages from HBM and occupying its modeled latency,
    gated by stream waits on the populate progress -- early start (prefix)
    vs the whole batch.  The two gatings alternate on one context (one
    untimed replay of each first), so drift of the host link between legs
    does not masquerade as a difference between them; medians resist
    outliers."""
    execute = {}
    leg = Leg(torch, dev, local, ws, tasks, hw, pol, mode, descs, migrate=True, host_pool_pages=pool_pages,
              execute=True)
    legs = (("early_start", True), ("whole_batch", False))
    for _, early in legs:
        leg.sim.mode = dataclasses.replace(leg.sim.mode, early_start=early)
        leg.step()
    e_times = {label: [] for label, _ in legs}
    e_stats = {label: {} for label, _ in legs}
    model = {}
    for _ in range(max(2, min(args.steps, 3))):
        for label, early in legs:
            leg.sim.mode = dataclasses.replace(leg.sim.mode, early_start=early)
            ms, mm = leg.step()
            e_times[label].append(ms)
            model[label] = mm.total_time_s * 1e3
            s1 = leg.sim.ctx.stats()
            e_stats[label] = {k: s1[k] for k in ("run_cmds", "run_pages", "run_ms", "run_bad_tags", "run_missing")}
    leg.close()
    for label, _ in legs:
        est = e_stats[label]
        execute[label] = {"ms_per_step": max_over_ranks(torch, statistics.median(e_times[label]), ws, dev),
                          "steps": len(e_times[label]), "ms_each": e_times[label],
                          "modeled_total_ms": model[label],
                          "commands": est["run_cmds"], "pages_read": est["run_pages"],
                          "consumer_busy_ms": est["run_ms"], "bad_payloads": est["run_bad_tags"],
                          "non_resident_reads": est["run_missing"]}
    execute["note"] = ("each executed command reads every page of its actual set from HBM and then occupies its "
                       "modeled latency, after a cuStreamWaitValue64 on the populate progress the H2D stream "
                       "publishes")
    return execute


if __name__ == "__main__":
    sys.exit(main())
