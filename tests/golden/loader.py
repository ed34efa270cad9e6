"""Decode the golden fixtures (written by make_golden.py from the real
reference) into the product's model types.  Stdlib + product model only; no
reference import, so this runs on the GPU box too."""

from __future__ import annotations

import functools
import gzip
import hashlib
import json
import os
import struct
from types import SimpleNamespace

from paper_2512_24637_b200.model import Allocation, Arg, ByteRange, Command, CommandKind, Task

HERE = os.path.dirname(os.path.abspath(__file__))
BIG = 64


def _load(name):
    with gzip.open(os.path.join(HERE, name), "rt") as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def sims():
    """Reference-generated simulations: make_golden.py, make_golden_extra.py,
    make_golden_edge.py."""
    out = _load("sims.json.gz")
    for extra in ("sims_extra.json.gz", "sims_edge.json.gz", "sims_frag.json.gz"):
        if os.path.exists(os.path.join(HERE, extra)):
            out = out + _load(extra)
    return out


@functools.lru_cache(maxsize=None)
def predictions():
    return _load("predict.json.gz")


@functools.lru_cache(maxsize=None)
def traces():
    return _load("traces.json.gz")


def sim_case(name):
    return next(c for c in sims() if c["name"] == name)


def dec_arg(a):
    if "raw" in a:
        return Arg(0, 64, raw=bytes.fromhex(a["raw"]))
    return Arg(a["v"], a["w"])


def dec_task(d) -> Task:
    t = Task(id=d["id"], cursor=d["cursor"], priority=d["priority"], arrival_s=d["arrival_s"])
    t.allocations = [Allocation(i, b, s, d["id"]) for i, b, s in d["allocations"]]
    for c in d["commands"]:
        t.commands.append(Command(
            kind=CommandKind(c["kind"]), latency_s=c["lat"], kernel_name=c["name"],
            launch_args=tuple(dec_arg(a) for a in c["args"]), grid_dims=tuple(c["grid"]),
            block_dims=tuple(c["block"]),
            ground_truth_access=tuple(ByteRange(s, n) for s, n in c["gt"])))
    return t


def ns(d):
    return SimpleNamespace(**d)


def digest(pages):
    """Same digest make_golden.py stores for long page lists (sha1 of the
    little-endian int64 array)."""
    import numpy as np

    arr = np.asarray(pages, dtype="<i8").reshape(-1)
    if arr.size <= BIG:
        return [int(p) for p in arr]
    return {"n": int(arr.size), "sha1": hashlib.sha1(arr.tobytes()).hexdigest()}


def feeder_for(spec, tasks):
    """Rebuild the live-feeding scenario (test_engine.py:262-289)."""
    if spec is None:
        return tasks, None
    src = next(t for t in tasks if t.id == spec["task"])
    head = Task(id=src.id, allocations=list(src.allocations),
                commands=list(src.commands[:spec["split"]]), priority=src.priority,
                arrival_s=src.arrival_s)
    tail = src.commands[spec["split"]:]
    state = {"fed": False}

    def feeder(sim):
        if not state["fed"] and sim.by_id[head.id].remaining() <= spec["when_le"]:
            sim.append_commands(head.id, tail)
            state["fed"] = True

    return [head if t.id == src.id else t for t in tasks], feeder


PAGE_KEYS = ("order_after_reorder", "evict", "populate", "prefix", "order")


def canon_records(recs, case_name=None):
    """Canonical form of planner records for comparison: page lists longer
    than BIG become digests; touch lists too."""
    out = []
    for r in recs:
        r = dict(r)
        for k in PAGE_KEYS:
            if k in r and not isinstance(r[k], dict):
                r[k] = digest(r[k])
        if r.get("ev") == "touch":
            for k in ("missing", "evicted"):
                if not isinstance(r[k], dict):
                    r[k] = digest(r[k])
        if "windows" in r:
            r["windows"] = [list(w) for w in r["windows"]]
        if "advised" in r:
            r["advised"] = [list(a) for a in r["advised"]]
        out.append(r)
    return out


def align_sampled(got, want):
    """make_golden samples the full order on big cases; drop what it skipped."""
    for g, w in zip(got, want):
        if g.get("ev") == "switch" and "order_after_reorder" in g and "order_after_reorder" not in w:
            del g["order_after_reorder"]
    return got


def strip_orders(recs):
    out = []
    for r in recs:
        r = dict(r)
        r.pop("order_after_reorder", None)
        r.pop("order", None)
        out.append(r)
    return out


def sample_refresh_orders(recs, every):
    """Keep the full-order digest of every k-th refresh record only."""
    out, k = [], 0
    for r in recs:
        if r.get("ev") == "refresh":
            r = dict(r)
            if k % every:
                r.pop("order", None)
            k += 1
        out.append(r)
    return out
