"""The B200 path behind the reference's own engine loop.

`b200_simulator_class(msim.engine)` returns a subclass of the reference's
`msim.engine.Simulator` (engine.py:180-473) whose hot-path methods call
`libmsched_b200.so` instead of the pure-Python memory manager — the binding
INTEGRATION.md §2 describes, as a maintainer would add it to `msim`:

  reference method (engine.py)          here
  -----------------------------------   -----------------------------------------
  _extend_task_tables   230-258         msg_add_task / msg_set_rules /
                                        msg_add_commands (K1: predicted + actual
                                        page sets on the device; the reference's
                                        own `build_descriptors` output is lowered)
  _prepare_slice        305-340         msg_plan_switch (windows, OPT reorder,
                                        plan, apply, gating counts, touch scan)
  _gating_state         342-361         per-command counts from msg_plan_switch,
                                        min(cum, populate) on the host
  _touch / _refresh_opt 389-460         msg_touch (missing set, OPT refresh,
                                        head eviction, install); UM slices via
                                        msg_um_slice
  _release              462-473         msg_release_task

Everything else — `run`, `_run_slice`, the FP64 timing model, `Metrics`,
events, the scheduler — is the reference's own code, inherited unchanged.
The Python `EvictionList`/`HelperQueue` objects the base constructor makes
stay empty: residency lives on the GPU.

The class is built from whatever `msim.engine` module the caller passes,
so this module imports nothing from the reference.
"""

from __future__ import annotations

from . import _abi
from .model import PageSet
from .scheduler import project_cursor

__all__ = ["b200_simulator_class", "to_msim_tasks"]


def _kind(cmd) -> str:
    k = cmd.kind
    return k.value if hasattr(k, "value") else str(k)


def _domain(tasks, page: int) -> list:
    spans = []
    for t in tasks:
        for a in t.allocations:
            lo, hi = a.base_addr // page, (a.base_addr + a.size_bytes - 1) // page + 1
            if hi > lo:
                spans.append((lo, hi))
        for c in t.commands:
            for r in c.ground_truth_access:
                spans.append((r.start_addr // page, (r.start_addr + r.length_bytes - 1) // page + 1))
            if _kind(c) != "KERNEL" and c.memcpy_size > 0:
                d = c.device_range()
                spans.append((d.start_addr // page, (d.start_addr + d.length_bytes - 1) // page + 1))
    return spans


def to_msim_tasks(mc, tasks) -> list:
    """This package's Task objects -> the reference's (`mc` = msim.core),
    field for field (the types are the same dataclasses, core.py:48-281)."""
    out = []
    for t in tasks:
        allocs = [mc.Allocation(id=a.id, base_addr=a.base_addr, size_bytes=a.size_bytes, owner_task=a.owner_task)
                  for a in t.allocations]
        cmds = [mc.Command(kind=mc.CommandKind(_kind(c)), latency_s=c.latency_s, kernel_name=c.kernel_name,
                           launch_args=tuple(mc.Arg(a.value, a.width, a.raw) for a in c.launch_args),
                           grid_dims=tuple(c.grid_dims), block_dims=tuple(c.block_dims),
                           ground_truth_access=tuple(mc.ByteRange(r.start_addr, r.length_bytes)
                                                     for r in c.ground_truth_access))
                for c in t.commands]
        out.append(mc.Task(id=t.id, allocations=allocs, commands=cmds, cursor=t.cursor, priority=t.priority,
                           arrival_s=t.arrival_s))
    return out


def b200_simulator_class(E):
    """E: the reference's `msim.engine` module."""
    import importlib

    MM = importlib.import_module(E.__name__.rsplit(".", 1)[0] + ".memman")   # ReorderStats, madvise_cost_s

    class B200Simulator(E.Simulator):
        """msim.engine.Simulator with the hot path on a B200 (see module doc).

        Extra keywords: device (CUDA ordinal), migrate (real pinned-host <->
        HBM copies of every plan), host_pool_pages (bound the pinned pool)."""

        def __init__(self, tasks, hw, policy, mode, feeder=None, record_events=False, *, device=0,
                     migrate=False, host_pool_pages=0):
            self._b200 = None
            self._b200_opts = (device, migrate, host_pool_pages)
            self._lat, self._selfpop, self._idx, self._kid = {}, {}, {}, {}
            self._state = None
            self._um = None
            self._resident = 0
            super().__init__(tasks, hw, policy, mode, feeder, record_events)

        # -- context -----------------------------------------------------

        def _ctx(self):
            if self._b200 is None:
                m = self.mode
                if m.name == "ideal" or m.predictor == "oracle" or m.name == "um":
                    pred = _abi.PRED_TRUTH
                elif m.predictor == "allocation":
                    pred = _abi.PRED_ALLOCATION
                else:
                    pred = _abi.PRED_TEMPLATE
                self._pred = pred
                device, migrate, pool = self._b200_opts
                self._b200 = _abi.Context(self.page, self.capacity, predictor=pred, device=device,
                                          flags=_abi.F_MIGRATE if migrate else 0, host_pool_pages=pool)
                self._b200.set_domain(_domain(self.tasks, self.page))
                self._idx = {t.id: i for i, t in enumerate(self.tasks)}
            return self._b200

        def close(self):
            if self._b200 is not None:
                self._b200.close()
                self._b200 = None

        # -- prediction tables (engine.py:230-258) --------------------------

        def _extend_task_tables(self, task, commands):
            commands = list(commands)
            self._lat.setdefault(task.id, []).extend(c.latency_s for c in commands)
            self._selfpop.setdefault(task.id, []).extend(_kind(c) == "H2D" for c in commands)
            if self.mode.name == "reference":
                return   # no memory management (engine.py:390-391, 464-465)
            ctx = self._ctx()
            i = self._idx[task.id]
            if task.id not in self._kid:
                ctx.add_task(i, [(a.base_addr, a.size_bytes) for a in task.allocations])
                kid = {}
                if self._pred == _abi.PRED_TEMPLATE and self.mode.name == "proactive":
                    descs = self._descriptors.get(task.id, {})   # the reference's own build_descriptors
                    names, rules, offs, _ = _abi.lower_rules(descs)
                    kid = {n: k for k, n in enumerate(names)}
                    ctx.set_rules(i, rules, offs)
                self._kid[task.id] = kid
            if commands:
                ctx.add_commands(i, _abi.encode_commands(commands, self._kid[task.id]))

        # -- proactive switch (engine.py:305-361) ---------------------------

        def _windows(self, timeline):
            return [(self._idx[e.task_id], e.resume_command_cursor,
                     project_cursor(self._lat[e.task_id], e.resume_command_cursor, e.timeslice_s))
                    for e in timeline if e.task_id in self._idx]

        def _stats(self, windows, win_pages):
            adv: dict = {}
            for (ti, _, _), n in zip(reversed(windows), reversed(list(win_pages))):
                tid = self.tasks[ti].id
                adv[tid] = adv.get(tid, 0) + int(n)
            return MM.ReorderStats(pages_advised=adv)

        def _prepare_slice(self, entry, timeline):
            windows = self._windows(timeline)
            out, win_pages, prefix_cnt, _ = self._ctx().plan_switch(windows)
            self._state = {"windows": windows, "next_missing": out.first_missing,
                           "next_missing_pages": out.first_missing_pages}
            if out.early_exit:
                self._resident = int(out.resident_after)
                return None
            stats = self._stats(windows, win_pages)
            if self.mode.name == "proactive":
                self._charge(MM.madvise_cost_s(self.hw, stats), "madvise_s")
            free = int(out.free_before)
            n_pop, n_ev = int(out.populate), int(out.evict)
            if out.truncated:
                self.metrics.plan_truncations += 1
            self.metrics.migrated_in_pages += n_pop
            self.metrics.migrated_out_pages += n_ev
            self._emit("migrate", entry.task_id, n_pop)
            pending = None
            if not self.mode.pipelined:
                self._charge(E.sequential_time(self.hw, n_ev, n_pop), "migration_s")
            elif self.mode.early_start:
                # _gating_state (engine.py:342-361): cumulative new demand pages
                c0, c1 = windows[0][1], windows[0][2]
                pop, cum, prefix = self._selfpop[entry.task_id], 0, {}
                for c in range(c0, c1):
                    if not pop[c]:
                        cum += int(prefix_cnt[c - c0])
                    prefix[c] = min(cum, n_pop)
                pending = {"prefix": prefix, "free": free, "n_evict": n_ev,
                           "evict_done": n_ev * E.evict_page_cost_s(self.hw)}
            else:
                self._charge(E.pipeline_time(self.hw, n_ev, n_pop, free), "migration_s")
            self._resident = int(out.resident_after)
            if self._resident > self.capacity:
                raise E.SimulationError("migration plan overflowed HBM capacity")
            return pending

        # -- slice execution (engine.py:365-445) -----------------------------

        def _run_slice(self, task, entry, timeline, pending):
            if self.mode.name == "um":
                c0 = task.cursor
                end = project_cursor(self._lat[task.id], c0, entry.timeslice_s)
                try:
                    miss, ev = self._ctx().um_slice(self._idx[task.id], c0, end)
                except _abi.MsgError as e:
                    if e.code == _abi.MSG_E_CAPACITY:
                        raise E.SimulationError(str(e)) from None
                    raise
                self._um = (c0, miss, ev)
            elif self.mode.name != "reference" and pending is None and self._state is None:
                self._state = {"windows": [], "next_missing": -1, "next_missing_pages": 0}
            super()._run_slice(task, entry, timeline, pending)
            self._state = None
            self._um = None

        def _touch(self, task, cmd, cur, timeline, entry, remaining_budget):
            name = self.mode.name
            if name == "reference":
                return 0.0
            is_h2d = _kind(cmd) == "H2D"
            if name == "um":
                c0, miss, ev = self._um
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
            st = self._state
            if st is None or st["next_missing"] != cur:
                return 0.0
            n = int(st["next_missing_pages"])
            if n > self.capacity:
                raise E.SimulationError(f"command working set ({n} pages) exceeds HBM "
                                        f"capacity ({self.capacity} pages)")
            stall = 0.0
            over = self._resident + n - self.capacity
            wins = []
            if over > 0:
                # _refresh_opt (engine.py:447-460): head window from the cursor + the rest
                head_end = project_cursor(self._lat[task.id], cur, max(remaining_budget, 1e-12))
                wins = [(self._idx[task.id], cur, head_end)] + self._windows(timeline[1:])
            out, win_pages = self._ctx().touch(self._idx[task.id], cur, max(over, 0), wins,
                                               st["windows"][0][2] if st["windows"] else cur + 1, is_h2d)
            if over > 0:
                if name == "proactive":
                    dt = MM.madvise_cost_s(self.hw, self._stats(wins, win_pages))
                    self.metrics.madvise_s += dt
                    stall += dt
                self.metrics.evicted_capacity_pages += int(out.evicted)
            if is_h2d:
                self.metrics.memcpy_installed_pages += n
            else:
                stall += self._fault(n)
            self._resident = int(out.resident_after)
            if self._resident > self.capacity:
                raise E.SimulationError(f"residency {self._resident} pages exceeds capacity "
                                        f"{self.capacity} after command {cur} of task {task.id!r}")
            self._emit("fault", task.id, n)
            st["next_missing"] = out.next_missing
            st["next_missing_pages"] = out.next_missing_pages
            return stall

        def _refresh_opt(self, task, cur, timeline, remaining_budget):   # folded into msg_touch
            raise NotImplementedError("B200Simulator refreshes the order inside msg_touch")

        def _release(self, task):
            self.metrics.completed_tasks += 1
            self.metrics.completion_s[task.id] = self.t
            if self.mode.name == "reference":
                return
            spans = PageSet((a.base_addr // self.page, (a.base_addr + a.size_bytes - 1) // self.page + 1)
                            for a in task.allocations)
            self._ctx().release(list(spans.runs))
            self._resident = self._ctx().list_len()
            self._emit("release", task.id, len(spans))

    return B200Simulator

