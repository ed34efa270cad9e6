"""Trace replay of one oversubscribed GPU with the memory manager on a B200.

Drop-in for the reference engine (engine.py:42-511): same `Mode`, `Metrics`,
`SimEvent`, `Simulator`, `simulate`, `simulate_normalized` surface.  The
host keeps what the north star keeps on the host — task-level scheduling,
the event loop and every FP64 timing decision, in the reference's
accumulation order, so timelines compare with `==`.  Everything that is set
algebra over pages runs on the GPU through the C ABI (`_abi.Context`):

  * per-command predicted / actual page sets   -> msg_add_commands (K1/K2)
  * window build, OPT reorder, plan, apply,
    early-start gating counts, slice touch scan -> msg_plan_switch (K3-K6, K8)
  * fault fallback with OPT refresh             -> msg_touch
  * demand paging (Mode.um)                     -> msg_um_slice
  * task release                                -> msg_release_task (K9)
  * real pinned-host <-> HBM page migration     -> the context's copy engines

There is no CPU fallback: constructing a Simulator for a memory-managed mode
without the CUDA library or a GPU raises.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _abi
from .analyzer import build_descriptors
from .model import CommandKind, HwConfig, PageSet, Task
from .tracebin import ColumnarTask, CommandColumns, encode_columns, kernel_ids_for
from .scheduler import Policy, TimelineEntry, build_timeline, project_cursor

__all__ = [
    "SimulationError", "Mode", "Metrics", "SimEvent", "evict_page_cost_s", "populate_page_cost_s",
    "sequential_time", "populate_ready", "pipeline_time", "Simulator", "simulate", "simulate_normalized",
    "um_command_duration",
]


class SimulationError(RuntimeError):
    pass


@dataclass(frozen=True)
class Mode:
    """engine.py:46-74."""

    name: str  # "um" | "proactive" | "ideal" | "reference"
    prefetch_pages: int = 16
    pipelined: bool = True
    early_start: bool = True
    predictor: str = "template"  # "template" | "allocation" | "oracle"

    @classmethod
    def um(cls, prefetch_pages: int = 16) -> "Mode":
        return cls("um", prefetch_pages=prefetch_pages)

    @classmethod
    def proactive(cls, pipelined: bool = True, early_start: bool = True, predictor: str = "template") -> "Mode":
        return cls("proactive", pipelined=pipelined, early_start=early_start, predictor=predictor)

    @classmethod
    def ideal(cls) -> "Mode":
        return cls("ideal", predictor="oracle")

    @classmethod
    def reference(cls) -> "Mode":
        return cls("reference")


@dataclass
class Metrics:
    """engine.py:77-115 (same fields, same order)."""

    total_time_s: float = 0.0
    exec_s: float = 0.0
    save_restore_s: float = 0.0
    madvise_s: float = 0.0
    migration_s: float = 0.0
    fault_s: float = 0.0
    fault_count: int = 0
    fault_pages: int = 0
    prefetched_pages: int = 0
    migrated_in_pages: int = 0
    migrated_out_pages: int = 0
    evicted_capacity_pages: int = 0
    memcpy_installed_pages: int = 0
    context_switches: int = 0
    completed_tasks: int = 0
    plan_truncations: int = 0
    page_size_bytes: int = 4096
    completion_s: dict = None
    normalized_throughput: Optional[float] = None

    def __post_init__(self):
        if self.completion_s is None:
            self.completion_s = {}

    @property
    def h2d_migration_pages(self) -> int:
        return self.migrated_in_pages + self.fault_pages

    @property
    def migrated_bytes_h2d(self) -> int:
        return self.h2d_migration_pages * self.page_size_bytes

    @property
    def migrated_bytes_d2h(self) -> int:
        return (self.migrated_out_pages + self.evicted_capacity_pages) * self.page_size_bytes

    @property
    def planned_pages(self) -> int:
        """The benchmark metric's numerator."""
        return self.migrated_in_pages + self.migrated_out_pages + self.fault_pages


@dataclass(frozen=True)
class SimEvent:
    t: float
    kind: str
    task_id: str
    pages: int = 0


# ---------------------------------------------------------------------------
# timing model (engine.py:126-166) — host FP64, unchanged


def evict_page_cost_s(hw: HwConfig) -> float:
    return hw.per_page_unmap_s + hw.page_size_bytes / hw.bw_d2h_bytes_per_s


def populate_page_cost_s(hw: HwConfig) -> float:
    return hw.page_size_bytes / hw.bw_h2d_bytes_per_s + hw.per_page_map_s


def sequential_time(hw: HwConfig, n_evict: int, n_populate: int) -> float:
    return n_evict * evict_page_cost_s(hw) + n_populate * populate_page_cost_s(hw)


def populate_ready(hw: HwConfig, j: int, free_pages: int, n_evict: int) -> float:
    """Completion of the j-th populate with eviction and population on
    separate copy engines; the makespan maximum sits at an endpoint or the
    free-frame breakpoint (engine.py:139-158)."""
    if j <= 0:
        return 0.0
    e, p = evict_page_cost_s(hw), populate_page_cost_s(hw)
    f = max(0, free_pages)
    best = 0.0
    for i in (1, min(f + 1, j), j):
        if i >= 1:
            lag = max(0, min(i, n_evict + f) - f)
            best = max(best, lag * e + (j - i + 1) * p)
    return best


def pipeline_time(hw: HwConfig, n_evict: int, n_populate: int, free_pages: int) -> float:
    return max(n_evict * evict_page_cost_s(hw), populate_ready(hw, n_populate, free_pages, n_evict))


def um_command_duration(hw: HwConfig, cmd, missing_pages: int, prefetch_pages: int = 16) -> float:
    batches = math.ceil(missing_pages / prefetch_pages) if missing_pages else 0
    return cmd.latency_s + batches * (hw.fault_control_plane_s + hw.fault_transfer_s * prefetch_pages)


def _copy_task(t: Task) -> Task:
    if isinstance(t.commands, CommandColumns):   # binary traces stay columnar (read-only columns)
        return ColumnarTask(id=t.id, allocations=t.allocations, commands=t.commands, cursor=t.cursor,
                            priority=t.priority, arrival_s=t.arrival_s)
    return Task(id=t.id, allocations=t.allocations, commands=list(t.commands), cursor=t.cursor,
                priority=t.priority, arrival_s=t.arrival_s)


def _page_span(a, page):
    return a.base_addr // page, (a.base_addr + a.size_bytes - 1) // page + 1


def domain_spans(tasks, page: int) -> list:
    """Every page the replay can name: allocations, ground-truth ranges and
    memcpy extents (the dense page map's domain)."""
    spans = []
    for t in tasks:
        for a in t.allocations:
            lo, hi = _page_span(a, page)
            if hi > lo:
                spans.append((lo, hi))
        if isinstance(t.commands, CommandColumns):
            spans.extend(_column_spans(t.commands, page))
            continue
        for c in t.commands:
            for r in c.ground_truth_access:
                spans.append((r.start_addr // page, (r.start_addr + r.length_bytes - 1) // page + 1))
            if c.kind is not CommandKind.KERNEL and c.memcpy_size > 0:
                d = c.device_range()
                spans.append((d.start_addr // page, (d.end_addr - 1) // page + 1))
    return spans


def _column_spans(cols: CommandColumns, page: int) -> list:
    """domain_spans for a columnar task: ground-truth ranges and memcpy extents."""
    out = [(a // page, (a + n - 1) // page + 1) for a, n in zip(cols.gts["start"].tolist(), cols.gts["len"].tolist())]
    mem = cols.cmds[(cols.cmds["kind"] != _abi.CMD_KERNEL) & (cols.cmds["dev_len"] > 0)]
    out.extend((a // page, (a + n - 1) // page + 1) for a, n in zip(mem["dev_addr"].tolist(), mem["dev_len"].tolist()))
    return out


class Simulator:
    """engine.py:169-473 with the memory manager on the GPU.

    Extra keyword arguments (not in the reference):
      migrate    perform the real pinned-host <-> HBM copies of every plan
      verify     stamp page ids into payloads so migration is checkable
      device     CUDA device ordinal
      recorder   list receiving per-switch planner records (parity dumps)
      host_pool_pages  bound the pinned backing store (pages alias beyond it)
      execute    run every executed command on the device as a kernel that
                 reads its pages from HBM, gated by stream waits on the
                 populate progress of the switch (early start when
                 Mode.early_start, else after the whole batch); needs migrate
    """

    def __init__(self, tasks: Sequence[Task], hw: HwConfig, policy: Policy, mode: Mode,
                 feeder: Optional[Callable[["Simulator"], None]] = None, record_events: bool = False, *,
                 migrate: bool = False, verify: bool = False, device: int = 0, recorder: list | None = None,
                 host_pool_pages: int = 0, descriptors: dict | None = None, order_every: int = 1,
                 execute: bool = False):
        self.hw, self.policy, self.mode, self.feeder = hw, policy, mode, feeder
        self.page = hw.page_size_bytes
        self.capacity = hw.hbm_capacity_pages
        # per-page copy costs of the pipelined-swap model, computed once
        # (populate_ready runs for every new gating prefix of a slice)
        self._cost_e, self._cost_p = evict_page_cost_s(hw), populate_page_cost_s(hw)
        self._source = list(tasks)
        self.record_events = record_events
        self.recorder = recorder
        self.order_every = max(1, order_every)   # dump the full list order every k-th reorder
        self._descriptors = descriptors
        if execute and not migrate:
            raise ValueError("execute=True needs migrate=True (commands read their migrated pages)")
        if execute and mode.name not in ("proactive", "ideal"):
            raise ValueError("execute=True is defined for the proactive and ideal modes")
        self.execute = execute
        self.ctx = None
        self._host_state()
        total_alloc = sum(a.size_bytes for t in self.tasks for a in t.allocations)
        if total_alloc > hw.dram_capacity_bytes:
            raise SimulationError(f"allocations ({total_alloc} B) exceed DRAM backing "
                                  f"({hw.dram_capacity_bytes} B)")
        if mode.name == "reference":
            return  # no memory management at all (engine.py:390-391, 464-465)
        if mode.name == "ideal" or mode.predictor == "oracle" or mode.name == "um":
            self._pred = _abi.PRED_TRUTH
        elif mode.predictor == "allocation":
            self._pred = _abi.PRED_ALLOCATION
        else:
            self._pred = _abi.PRED_TEMPLATE
        flags = (_abi.F_MIGRATE if migrate else 0) | (_abi.F_VERIFY_TAGS if verify else 0) | \
            (_abi.F_EXECUTE if execute else 0)
        self.ctx = _abi.Context(self.page, self.capacity, predictor=self._pred, device=device, flags=flags,
                                host_pool_pages=host_pool_pages)
        self.ctx.set_domain(domain_spans(self.tasks, self.page))
        if recorder is not None:
            self.ctx.debug(3)
        self._register_tasks()

    def _host_state(self):
        """Fresh copies of the input tasks and all host-side loop state."""
        self.tasks = [_copy_task(t) for t in self._source]
        for t in self.tasks:
            t.validate()
        self.by_id = {t.id: t for t in self.tasks}
        if len(self.by_id) != len(self.tasks):
            raise SimulationError("duplicate task ids")
        self._rr_order = [t.id for t in self.tasks]
        self.metrics = Metrics(page_size_bytes=self.page)
        self.t = 0.0
        self.events: list = []
        self._idx = {t.id: i for i, t in enumerate(self.tasks)}
        self._lat, self._selfpop = {}, {}
        self._proj_cache = {}
        for t in self.tasks:
            if isinstance(t.commands, CommandColumns):
                self._lat[t.id] = t.commands.lat.tolist()
                self._selfpop[t.id] = (t.commands.kinds() == _abi.CMD_H2D).tolist()
            else:
                self._lat[t.id] = [c.latency_s for c in t.commands]
                self._selfpop[t.id] = [c.kind is CommandKind.MEMCPY_H2D for c in t.commands]
        self._resident = 0
        self._nreorder = 0
        self._nrefresh = 0

    def _register_tasks(self):
        """Allocations, rule tables and every command's page sets (K1) to the device."""
        self._kernel_ids: dict = {}
        self._lossy: dict = {}
        self.complete: dict = {}
        for t in self.tasks:
            i = self._idx[t.id]
            self.ctx.add_task(i, [(a.base_addr, a.size_bytes) for a in t.allocations])
            kid, lossy = {}, []
            if self._pred == _abi.PRED_TEMPLATE and self.mode.name == "proactive":
                descs = (self._descriptors or {}).get(t.id) or getattr(t, "descriptors", None) or \
                    build_descriptors(t)
                names, rules, offs, lossy = _abi.lower_rules(descs)
                kid = {n: k for k, n in enumerate(names)}
                self.ctx.set_rules(i, rules, offs)
            self._kernel_ids[t.id] = kid
            self._lossy[t.id] = lossy
            self.complete[t.id] = []
            self._extend_task_tables(t, t.commands)

    def reset(self, reupload: bool = False):
        """Replay again from the start.  The device keeps its allocations; with
        reupload=False it also keeps the predicted page sets (the trace stays
        resident in HBM), with reupload=True the task tables are rebuilt from
        the host Task objects (encode, H2D, K1 prediction)."""
        # a feeder appends commands while the replay runs: the device tables
        # then hold the previous replay's appended commands, so they are
        # rebuilt from the source tasks
        reupload = reupload or self.feeder is not None
        self._host_state()
        if self.ctx is not None:
            self.ctx.reset(keep_tasks=not reupload)
            if reupload:
                self._register_tasks()

    # -- prediction tables (engine.py:222-258) ----------------------------

    def _extend_task_tables(self, task: Task, commands: Sequence):
        if not commands:
            return
        kid = self._kernel_ids[task.id]
        if isinstance(commands, CommandColumns):   # binary trace: the columns are the ABI tables
            comp = self.ctx.add_commands(self._idx[task.id], encode_columns(commands, kid))
            k = kernel_ids_for(commands, kid)
            lossy = np.asarray(list(self._lossy[task.id]) + [False], dtype=bool)
            bad = (commands.kinds() == _abi.CMD_KERNEL) & (k >= 0) & lossy[np.where(k >= 0, k, len(lossy) - 1)]
            self.complete[task.id].extend((comp.astype(bool) & ~bad).tolist())
            return
        comp = self.ctx.add_commands(self._idx[task.id], _abi.encode_commands(commands, kid))
        lossy = self._lossy[task.id]
        for c, ok in zip(commands, comp):
            k = kid.get(c.kernel_name, -1)
            self.complete[task.id].append(bool(ok) and not (c.kind is CommandKind.KERNEL and k >= 0 and lossy[k]))

    def append_commands(self, task_id: str, commands: Sequence):
        task = self.by_id[task_id]
        if task.remaining() == 0 and task.commands:
            raise SimulationError(f"cannot append to completed task {task_id!r}")
        if isinstance(task.commands, CommandColumns):
            task.commands = list(task.commands)   # a fed task becomes a plain command list
        commands = list(commands)
        task.commands.extend(commands)
        self._lat[task_id].extend(c.latency_s for c in commands)
        self._selfpop[task_id].extend(c.kind is CommandKind.MEMCPY_H2D for c in commands)
        if self.ctx is not None:
            self._extend_task_tables(task, commands)

    def predicted_pages(self, task_id: str, cmd: int) -> PageSet:
        return PageSet._raw(self.ctx.read_pages(self._idx[task_id], cmd, 0))

    def actual_pages(self, task_id: str, cmd: int) -> PageSet:
        return PageSet._raw(self.ctx.read_pages(self._idx[task_id], cmd, 1))

    # -- main loop (engine.py:262-293) ---------------------------------------

    def run(self, max_switches: int = 1_000_000) -> Metrics:
        proactive = self.mode.name in ("proactive", "ideal")
        for _ in range(max_switches):
            if self.feeder is not None:
                self.feeder(self)
            live = [t for t in self.tasks if t.remaining() > 0]
            if not live:
                break
            ready = [t for t in live if t.arrival_s <= self.t + 1e-15]
            if not ready:
                self.t = min(t.arrival_s for t in live)
                continue
            rank = {tid: i for i, tid in enumerate(self._rr_order)}
            ready.sort(key=lambda t: rank[t.id])
            timeline = build_timeline(self.policy, ready, latencies=self._lat, project=self._project)
            entry = timeline[0]
            task = self.by_id[entry.task_id]
            self._rr_order.remove(task.id)
            self._rr_order.append(task.id)
            self.metrics.context_switches += 1
            self._charge(self.hw.save_restore_s, "save_restore_s")
            slice_state = None
            if proactive:
                slice_state = self._prepare_slice(entry, timeline)
            self._emit("switch", task.id)
            self._run_slice(task, entry, timeline, slice_state)
            if task.remaining() == 0:
                self._release(task)
        else:
            raise SimulationError("context-switch budget exhausted")
        self.metrics.total_time_s = self.t
        return self.metrics

    def _charge(self, dt: float, bucket: str):
        self.t += dt
        setattr(self.metrics, bucket, getattr(self.metrics, bucket) + dt)

    def _emit(self, kind: str, task_id: str, pages: int = 0):
        if self.record_events:
            self.events.append(SimEvent(self.t, kind, task_id, pages))

    def _project(self, task_id, cursor: int, budget: float) -> int:
        """project_cursor on a task's latency column, memoised: the timeline
        and the windows walk the same (cursor, timeslice) slices switch after
        switch.  The key carries the column's length (feeders append)."""
        lat = self._lat[task_id]
        key = (task_id, cursor, budget, len(lat))
        end = self._proj_cache.get(key)
        if end is None:
            if len(self._proj_cache) > 1 << 16:
                self._proj_cache.clear()
            end = self._proj_cache[key] = project_cursor(lat, cursor, budget)
        return end

    def _windows(self, timeline) -> list:
        """(task index, cursor, end) per timeline entry: compute_window's
        FP64 walk (memman.py:186-195) on the host, integers to the GPU."""
        return [(self._idx[e.task_id], e.resume_command_cursor,
                 self._project(e.task_id, e.resume_command_cursor, e.timeslice_s)) for e in timeline]

    def _advised(self, windows, win_pages) -> dict:
        """ReorderStats.pages_advised: reversed windows, dict first-insertion
        order (memman.py:238-241)."""
        adv: dict = {}
        for (ti, _, _), n in zip(reversed(windows), reversed(win_pages.tolist())):
            tid = self.tasks[ti].id
            adv[tid] = adv.get(tid, 0) + n
        return adv

    def _madvise_cost(self, adv: dict) -> float:
        return sum(self.hw.madvise_call_s + n * self.hw.per_page_madvise_s for n in adv.values())

    # -- proactive switch (engine.py:305-361) -------------------------------

    def _prepare_slice(self, entry: TimelineEntry, timeline):
        windows = self._windows(timeline)
        dump_order = False
        if self.recorder is not None:
            dump_order = self._nreorder % self.order_every == 0
            self.ctx.debug(3 if dump_order else 1)
        out, win_pages, prefix_cnt, touch_cnt = self.ctx.plan_switch(windows)
        rec = None
        if self.recorder is not None:
            rec = {"ev": "switch", "task": entry.task_id,
                   "windows": [[self.tasks[t].id, a, b] for t, a, b in windows], "missing": int(out.missing)}
            self.recorder.append(rec)
        state = {"windows": windows, "next_missing": out.first_missing,
                 "next_missing_pages": out.first_missing_pages, "pending": None, "gate": None}
        if out.early_exit:
            self._resident = out.resident_after
            return state
        adv = self._advised(windows, win_pages)
        if self.mode.name == "proactive":
            self._charge(self._madvise_cost(adv), "madvise_s")
        free = int(out.free_before)
        n_pop, n_ev = int(out.populate), int(out.evict)
        self._nreorder += 1
        if rec is not None:
            rec.update(advised=[[k, v] for k, v in adv.items()], free=free, evict=self.ctx.debug_read(1),
                       populate=self.ctx.debug_read(2), truncated=int(out.truncated))
            if dump_order:
                rec["order_after_reorder"] = self.ctx.debug_read(0)
            self.ctx.debug(3)
        if out.truncated:
            self.metrics.plan_truncations += 1
        self.metrics.migrated_in_pages += n_pop
        self.metrics.migrated_out_pages += n_ev
        if self.execute:   # executed commands wait for their prefix, or the whole batch
            c0, c1 = windows[0][1], windows[0][2]
            if self.mode.pipelined and self.mode.early_start:
                pop, cum, gate = self._selfpop[entry.task_id], 0, {}
                for c in range(c0, c1):
                    if not pop[c]:
                        cum += int(prefix_cnt[c - c0])
                    gate[c] = min(cum, n_pop)
                state["gate"] = gate
            else:
                state["gate"] = {c: n_pop for c in range(c0, c1)}
        self._emit("migrate", entry.task_id, n_pop)
        if not self.mode.pipelined:
            self._charge(sequential_time(self.hw, n_ev, n_pop), "migration_s")
        elif self.mode.early_start:
            c0, c1 = windows[0][1], windows[0][2]
            pop = self._selfpop[entry.task_id]
            prefix, cum = {}, 0
            pc = prefix_cnt.tolist()
            for c in range(c0, c1):
                if not pop[c]:
                    cum += pc[c - c0]
                prefix[c] = min(cum, n_pop)
            if rec is not None:
                rec["prefix"] = [prefix[c] for c in range(c0, c1)]
            state["pending"] = {"prefix": prefix, "free": free, "n_evict": n_ev,
                                "evict_done": n_ev * evict_page_cost_s(self.hw)}
        else:
            self._charge(pipeline_time(self.hw, n_ev, n_pop, free), "migration_s")
        self._resident = int(out.resident_after)
        if self._resident > self.capacity:
            raise SimulationError("migration plan overflowed HBM capacity")
        return state

    # -- slice execution (engine.py:365-445) ---------------------------------

    def _run_slice(self, task: Task, entry, timeline, state):
        budget = entry.timeslice_s
        elapsed = 0.0
        offset = 0.0
        slice_start = self.t
        pending = state["pending"] if state else None
        um = None
        if self.mode.name == "um":
            end = project_cursor(self._lat[task.id], task.cursor, budget)
            try:
                um = (task.cursor,) + self.ctx.um_slice(self._idx[task.id], task.cursor, end)
            except _abi.MsgError as e:
                if e.code == _abi.MSG_E_CAPACITY:
                    raise SimulationError(str(e)) from None
                raise
            if self.recorder is not None:
                self._um_records(task.id, self.ctx.debug_read(3))
        lat, selfpop = self._lat[task.id], self._selfpop[task.id]
        # the switch-time scan names the next missing command: commands before
        # it cannot fault (the _touch call is skipped for them, same result)
        fast = self.mode.name in ("proactive", "ideal") and state is not None
        last_j, last_ready = None, 0.0   # populate_ready is pure: memo by j (the prefix repeats)
        ncmd = len(task.commands)
        if pending is not None:
            prefix, p_free, p_nev = pending["prefix"], pending["free"], pending["n_evict"]
        while task.cursor < ncmd and elapsed < budget:
            cur = task.cursor
            if pending is not None:
                j = prefix.get(cur, 0)
                if j != last_j:
                    last_j, last_ready = j, self._populate_ready(j, p_free, p_nev)
                ready = last_ready
                if ready > offset:
                    self.metrics.migration_s += ready - offset
                    offset = ready
            if not (fast and state["next_missing"] != cur):
                offset += self._touch(task, selfpop[cur], cur, timeline, state, budget - elapsed, um)
            if self.execute:
                gate = state["gate"] if state else None
                self.ctx.run_command(self._idx[task.id], cur, gate.get(cur, 0) if gate else 0, lat[cur])
            offset += lat[cur]
            elapsed += lat[cur]
            task.cursor = cur + 1
        if pending is not None and pending["evict_done"] > offset:
            self.metrics.migration_s += pending["evict_done"] - offset
            offset = pending["evict_done"]
        self.t = slice_start + offset
        self.metrics.exec_s += elapsed

    def _populate_ready(self, j: int, free_pages: int, n_evict: int) -> float:
        """populate_ready (engine.py:139-158) with the per-page costs cached:
        the same candidates and the same FP64 expressions, so the same float."""
        if j <= 0:
            return 0.0
        e, p = self._cost_e, self._cost_p
        f = free_pages if free_pages > 0 else 0
        cap = n_evict + f
        best = 0.0
        for i in (1, f + 1 if f + 1 < j else j, j):   # every candidate is >= 1 here
            lag = (i if i < cap else cap) - f
            v = (lag if lag > 0 else 0) * e + (j - i + 1) * p
            if v > best:
                best = v
        return best

    def _um_records(self, task_id, flat):
        i = 0
        flat = [int(x) for x in flat]
        while i < len(flat):
            cmd, nm = flat[i], flat[i + 1]
            miss = flat[i + 2:i + 2 + nm]
            i += 2 + nm
            ne = flat[i]
            ev = flat[i + 1:i + 1 + ne]
            i += 1 + ne
            self.recorder.append({"ev": "touch", "task": task_id, "cmd": cmd, "missing": miss, "evicted": ev})

    def _capacity_guard(self, n: int):
        if n > self.capacity:
            raise SimulationError(f"command working set ({n} pages) exceeds HBM capacity ({self.capacity} pages)")

    def _touch(self, task, is_h2d, cur, timeline, state, remaining_budget, um) -> float:
        name = self.mode.name
        if name == "reference":
            return 0.0
        if name == "um":
            c0, miss, ev = um
            n = int(miss[cur - c0])
            if not n:
                return 0.0
            self.metrics.evicted_capacity_pages += int(ev[cur - c0])
            stall = 0.0
            if is_h2d:
                self.metrics.memcpy_installed_pages += n
            else:
                stall += self._fault(n)
            self._emit("fault", task.id, n)
            return stall
        # proactive / ideal: the switch-time scan says which command misses next
        if state["next_missing"] != cur:
            return 0.0
        n = int(state["next_missing_pages"])
        self._capacity_guard(n)
        stall = 0.0
        over = self._resident + n - self.capacity
        wins = []
        head_end = None
        if over > 0:
            head_end = project_cursor(self._lat[task.id], cur, max(remaining_budget, 1e-12))
            wins = [(self._idx[task.id], cur, head_end)] + state["windows"][1:]
        scan_end = state["windows"][0][2]
        dump_order = False
        if self.recorder is not None and over > 0:
            dump_order = self._nrefresh % self.order_every == 0
            self._nrefresh += 1
            self.ctx.debug(3 if dump_order else 1)
        out, win_pages = self.ctx.touch(self._idx[task.id], cur, max(over, 0), wins, scan_end, bool(is_h2d))
        if over > 0:
            if self.recorder is not None:
                r = {"ev": "refresh", "task": task.id, "cmd": cur,
                     "windows": [[self.tasks[t].id, a, b] for t, a, b in wins]}
                if dump_order:
                    r["order"] = self.ctx.debug_read(0)
                self.recorder.append(r)
                self.ctx.debug(3)
            if self.mode.name == "proactive":
                dt = self._madvise_cost(self._advised(wins, win_pages))
                self.metrics.madvise_s += dt
                stall += dt
            self.metrics.evicted_capacity_pages += int(out.evicted)
        if is_h2d:
            self.metrics.memcpy_installed_pages += n
        else:
            stall += self._fault(n)
        self._resident = int(out.resident_after)
        if self._resident > self.capacity:
            raise SimulationError(f"residency {self._resident} pages exceeds capacity "
                                  f"{self.capacity} after command {cur} of task {task.id!r}")
        if self.recorder is not None:
            self.recorder.append({"ev": "touch", "task": task.id, "cmd": cur,
                                  "missing": self.ctx.debug_read(2),
                                  "evicted": self.ctx.debug_read(1) if over > 0 else []})
        self._emit("fault", task.id, n)
        state["next_missing"] = out.next_missing
        state["next_missing_pages"] = out.next_missing_pages
        return stall

    def _fault(self, n_pages: int) -> float:
        hw = self.hw
        self.metrics.fault_pages += n_pages
        if self.mode.name == "ideal":
            dt = n_pages * populate_page_cost_s(hw)
        else:
            batches = math.ceil(n_pages / self.mode.prefetch_pages)
            self.metrics.fault_count += batches
            self.metrics.prefetched_pages += batches * self.mode.prefetch_pages - n_pages
            dt = batches * (hw.fault_control_plane_s + hw.fault_transfer_s * self.mode.prefetch_pages)
        self.metrics.fault_s += dt
        return dt

    def _release(self, task: Task):
        self.metrics.completed_tasks += 1
        self.metrics.completion_s[task.id] = self.t
        if self.mode.name == "reference":
            return
        spans = PageSet(_page_span(a, self.page) for a in task.allocations)
        self.ctx.release(list(spans.runs))
        self._resident = self.ctx.list_len()
        self._emit("release", task.id, len(spans))

    # -- diagnostics -------------------------------------------------------

    def eviction_order(self) -> list:
        return [int(p) for p in self.ctx.list_read()] if self.ctx else []

    def stats(self) -> dict:
        return self.ctx.stats() if self.ctx else {}

    def close(self):
        if self.ctx is not None:
            self.ctx.close()
            self.ctx = None


def simulate(tasks, hw, policy, mode, feeder=None, record_events: bool = False, **kw) -> Metrics:
    sim = Simulator(tasks, hw, policy, mode, feeder, record_events, **kw)
    try:
        return sim.run()
    finally:
        sim.close()


def simulate_normalized(tasks, hw, policy, mode, feeder=None, **kw) -> Metrics:
    """engine.py:499-511."""
    m = simulate(tasks, hw, policy, mode, feeder, **kw)
    ref = simulate(tasks, hw, policy, Mode.reference(), feeder)
    m.normalized_throughput = ref.total_time_s / m.total_time_s
    return m
