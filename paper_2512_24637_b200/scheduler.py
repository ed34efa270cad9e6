"""Task-level timeslice scheduling — stays on the host (north star).

Same contract as the reference scheduler (scheduler.py:16-97): a timeline of
(task, timeslice, projected resume cursor) entries that the planner turns
into per-entry page windows.  Cursor projection is FP64 in the reference's
accumulation order, because window boundaries are float decisions.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

__all__ = ["Policy", "TimelineEntry", "Timeline", "runnable_order", "build_timeline",
           "project_cursor"]


@dataclass(frozen=True)
class TimelineEntry:
    task_id: str
    timeslice_s: float
    resume_command_cursor: int


Timeline = tuple


@dataclass(frozen=True)
class Policy:
    """scheduler.py:26-36."""

    kind: str = "rr"
    timeslice_s: float = 5e-3
    horizon_rounds: int = 2

    def __post_init__(self):
        if self.timeslice_s <= 0:
            raise ValueError("timeslice must be positive")
        if self.kind not in ("rr", "priority"):
            raise ValueError(f"unknown policy kind {self.kind!r}")


def _entry(task_id: str, timeslice_s: float, cursor: int) -> TimelineEntry:
    """TimelineEntry(task_id, timeslice_s, cursor) without the frozen
    dataclass's per-field object.__setattr__ calls (the same object: equal,
    same hash and repr); build_timeline makes one per horizon entry every
    context switch."""
    e = object.__new__(TimelineEntry)
    d = e.__dict__
    d["task_id"] = task_id
    d["timeslice_s"] = timeslice_s
    d["resume_command_cursor"] = cursor
    return e


def project_cursor(latencies: Sequence[float], cursor: int, budget: float) -> int:
    """Cursor after one slice: every command that starts inside the slice
    runs to completion (scheduler.py:86-97, memman.py:186-195)."""
    spent = 0.0
    n = len(latencies)
    while cursor < n and spent < budget:
        spent += latencies[cursor]
        cursor += 1
    return cursor


def runnable_order(policy: Policy, tasks) -> list:
    """scheduler.py:39-47: live tasks, restricted to the top priority level
    under the priority policy."""
    live = [t for t in tasks if t.remaining() > 0]
    if live and policy.kind == "priority":
        top = max(t.priority for t in live)
        live = [t for t in live if t.priority == top]
    return live


def build_timeline(policy: Policy, tasks, horizon_entries: int | None = None,
                   latencies: dict | None = None, project=None) -> Timeline:
    """scheduler.py:50-83.  `latencies` (task id -> list of floats) lets the
    engine pass cached latency columns instead of walking Command objects;
    `project(task_id, cursor, budget)` (optional) stands in for
    project_cursor on them (the engine's memoised walk)."""
    live = runnable_order(policy, tasks)
    if not live:
        return ()
    if horizon_entries is None:
        horizon_entries = policy.horizon_rounds * len(live)
    lat = latencies or {t.id: [c.latency_s for c in t.commands] for t in live}
    pos = {t.id: t.cursor for t in live}
    plan = []
    rr = list(live)
    k = 0
    while len(plan) < horizon_entries and rr:
        t = rr[k % len(rr)]
        if pos[t.id] >= len(lat[t.id]):
            rr = [x for x in rr if pos[x.id] < len(lat[x.id])]
            k = 0
            continue
        plan.append(_entry(t.id, policy.timeslice_s, pos[t.id]))
        pos[t.id] = (project(t.id, pos[t.id], policy.timeslice_s) if project is not None
                     else project_cursor(lat[t.id], pos[t.id], policy.timeslice_s))
        k += 1
    return tuple(plan)
