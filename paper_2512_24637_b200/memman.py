"""Drop-in eviction-list / window / plan API (reference memman.py:23-341),
backed by the GPU.

`EvictionList` owns a small msg_ctx whose dense page map is [0, domain_pages);
its order lives in HBM and every mutation is a device multisplit.
`compute_window`, `reorder_for_opt` and `plan_migration` run the same kernels
the engine uses (csrc/k_plan.cu).  Only `belady_oracle` — the reference's own
brute-force verification oracle (memman.py:310-341), not part of the hot
path — is host code.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

from . import _abi
from .model import PageSet, Task
from .scheduler import project_cursor

Run = tuple

__all__ = ["EvictionList", "HelperQueue", "Window", "compute_window", "timeline_windows", "ReorderStats",
           "reorder_for_opt", "madvise_cost_s", "MigrationPlan", "plan_migration", "apply_plan",
           "belady_oracle", "DEFAULT_DOMAIN_PAGES"]

DEFAULT_DOMAIN_PAGES = 1 << 20


def _runs_of(pages) -> list:
    out: list = []
    for p in pages:
        p = int(p)
        if out and out[-1][1] == p:
            out[-1][1] = p + 1
        else:
            out.append([p, p + 1])
    return [(a, b) for a, b in out]


class EvictionList:
    """Ordered resident pages, head = next victim (memman.py:23-137)."""

    def __init__(self, domain_pages: int = DEFAULT_DOMAIN_PAGES, device: int = 0):
        self.ctx = _abi.Context(4096, domain_pages, device=device)
        self.ctx.set_domain([(0, domain_pages)])
        self.domain_pages = domain_pages
        # membership mirror, updated by every mutation from what the device
        # reports (the order itself lives only on the device): `resident` is
        # O(1) instead of a read + sort of the whole list
        self._members = PageSet()

    @property
    def resident(self) -> PageSet:
        return self._members

    def __len__(self) -> int:
        return self.ctx.list_len()

    def pages_in_order(self) -> list:
        return [int(p) for p in self.ctx.list_read()]

    @property
    def _runs(self) -> list:
        """Coalesced runs head->tail (plan_migration reads them, memman.py:296)."""
        return _runs_of(self.ctx.list_read())

    def append_tail(self, runs: Iterable[Run]):
        runs = [(a, b) for a, b in runs if b > a]
        if runs:
            self.ctx.list_append(runs)
            self._members = self._members | PageSet(runs)

    def madvise(self, pages: PageSet):
        if pages and len(self):
            self.ctx.list_madvise(list(pages.runs))

    def evict_head(self, n_pages: int) -> list:
        if n_pages <= 0:
            return []
        got = _runs_of(self.ctx.list_evict_head(n_pages))
        if got:
            self._members = self._members - PageSet(got)
        return got

    def remove(self, pages: PageSet):
        if pages and len(self):
            self.ctx.release(list(pages.runs))
            self._members = self._members - pages


@dataclass
class HelperQueue:
    """Per-task predicted page sets parallel to task.commands (memman.py:140-160)."""

    task: Task
    predicted: list = field(default_factory=list)
    self_populating: list = field(default_factory=list)

    def append(self, page_sets, self_pop=()):
        page_sets = list(page_sets)
        self_pop = list(self_pop)
        self.predicted.extend(page_sets)
        self.self_populating.extend(self_pop if self_pop else [False] * len(page_sets))


@dataclass
class Window:
    task_id: str
    ordered_runs: list
    demand_runs: list
    pages: PageSet
    end_cursor: int


_window_ctx = None


def _wctx():
    global _window_ctx
    if _window_ctx is None:
        _window_ctx = _abi.Context(4096, 1)
        _window_ctx.set_domain([(0, 1)])
    return _window_ctx


def compute_window(helper: HelperQueue, cursor: int, timeslice_s: float) -> Window:
    """memman.py:174-196: the FP64 slice walk on the host, the first-access
    run construction (k_window_runs) on the GPU."""
    cmds = helper.task.commands
    end = project_cursor([c.latency_s for c in cmds], cursor, timeslice_s)
    runs, _ = _wctx().window_runs([list(helper.predicted[c].runs) for c in range(cursor, end)])
    ordered = [(a, b) for a, b, _ in runs]
    sp = helper.self_populating
    demand = [(a, b) for a, b, k in runs if not (cursor + k < len(sp) and sp[cursor + k])]
    return Window(helper.task.id, ordered, demand, PageSet(ordered), end)


def timeline_windows(timeline, helpers: dict) -> list:
    return [compute_window(helpers[e.task_id], e.resume_command_cursor, e.timeslice_s)
            for e in timeline if e.task_id in helpers]


@dataclass
class ReorderStats:
    pages_advised: dict = field(default_factory=dict)

    @property
    def total_pages(self) -> int:
        return sum(self.pages_advised.values())


def reorder_for_opt(evlist: EvictionList, timeline, helpers: dict, windows: Sequence[Window] | None = None
                    ) -> ReorderStats:
    """memman.py:218-241 as one device multisplit."""
    if windows is None:
        windows = timeline_windows(timeline, helpers)
    windows = list(windows)
    evlist.ctx.list_reorder([w.ordered_runs for w in windows])
    stats = ReorderStats()
    for w in reversed(windows):
        stats.pages_advised[w.task_id] = stats.pages_advised.get(w.task_id, 0) + len(w.pages)
    return stats


def madvise_cost_s(hw, stats: ReorderStats) -> float:
    return sum(hw.madvise_call_s + n * hw.per_page_madvise_s for n in stats.pages_advised.values())


@dataclass
class MigrationPlan:
    evict_runs: list
    populate_runs: list
    truncated_pages: int = 0

    @property
    def evict_pages(self) -> int:
        return sum(b - a for a, b in self.evict_runs)

    @property
    def populate_pages(self) -> int:
        return sum(b - a for a, b in self.populate_runs)


def plan_migration(evlist: EvictionList, next_ws_runs: Sequence[Run], capacity_pages: int) -> MigrationPlan:
    """memman.py:269-302 on the device (k_demand_* kernels + list head)."""
    runs = [(a, b) for a, b in next_ws_runs]
    pop, ev, trunc = evlist.ctx.list_plan(runs, capacity_pages)
    return MigrationPlan(_runs_of(ev), _split_runs(pop, runs), trunc)


def _split_runs(pages, runs) -> list:
    """Populate pages (first-access order) -> the reference's populate_runs:
    the missing pieces of each requested run separately (memman.py:283-290),
    so pieces of two adjacent requested runs stay two runs."""
    out: list = []
    i, n = 0, len(pages)
    for a, b in runs:
        j = i
        while j < n and a <= int(pages[j]) < b:
            j += 1
        out.extend(_runs_of(pages[i:j]))
        i = j
    out.extend(_runs_of(pages[i:]))   # nothing is left unless runs overlap
    return out


def apply_plan(evlist: EvictionList, plan: MigrationPlan):
    evlist.evict_head(plan.evict_pages)
    evlist.append_tail(plan.populate_runs)


def belady_oracle(access_seq, frames: int):
    """Brute-force OPT, verification only (memman.py:310-341)."""
    if frames < 1:
        raise ValueError("frames must be >= 1")
    held: set = set()
    faults, trace = 0, []
    n = len(access_seq)
    for i, page in enumerate(access_seq):
        if page in held:
            continue
        faults += 1
        if len(held) >= frames:
            victim, far = -1, -1
            for q in sorted(held):
                nxt = next((j for j in range(i + 1, n) if access_seq[j] == q), n + 1)
                if nxt > far:
                    victim, far = q, nxt
            held.remove(victim)
            trace.append((i, victim))
        held.add(page)
    return faults, trace
