"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference MSched simulator.

Every function cites the reference file:line it restates (paths are relative
to /root/reference/pkg/src/msim/).  Inputs are duck-typed: any objects with
the reference's attribute names work (the reference's own `msim` objects, or
the product package's model types), so the same task list can drive the
reference, this port and the GPU path.

Parity status: pinned.  `tests/golden/` holds fixtures produced by the real
reference (see tests/golden/make_golden.py); tests/test_oracle_golden.py
checks this module against every one of them.

Deliberate properties:
  * run-length page sets and a run-list eviction list (core.py:72-189,
    memman.py:23-137) — the same data structures and complexity as the
    reference, so timing this module is a fair CPU baseline;
  * float arithmetic in the same order as the reference (engine.py:262-473),
    so metrics and events compare with `==`;
  * an optional `recorder` that captures per-switch planner decisions
    (windows, plans, gating prefixes, touches) for parity dumps.  The
    reference never implemented its promised dump; the
    golden generator captures the same records by wrapping the reference.
"""

from __future__ import annotations

import itertools
import math
import struct
from bisect import bisect_right
from fractions import Fraction

__all__ = [
    "Runs", "norm_runs", "runs_len", "runs_or", "runs_and", "runs_sub",
    "runs_pages", "byte_pages", "ranges_pages",
    "RunList", "Win", "window_of", "windows_of", "opt_reorder", "advise_cost",
    "Plan", "make_plan", "apply_plan_runs", "belady",
    "slot_table", "struct_words", "eval_expr", "rule_regions",
    "predict_template", "predict_alloc", "predict_truth", "accuracy",
    "infer_descriptors", "descriptors_text",
    "timeline", "PortMetrics", "PortSim", "port_simulate",
    "evict_cost", "populate_cost", "seq_swap_time", "ready_time", "pipe_swap_time",
]

Runs = tuple  # tuple[tuple[int, int], ...], sorted, disjoint, non-adjacent


def _kind(cmd) -> str:
    k = cmd.kind
    return getattr(k, "value", k)


# ---------------------------------------------------------------------------
# run-length page sets (core.py:72-189)


def norm_runs(runs) -> Runs:
    """Sort and merge overlapping or touching runs (core.py:177-189)."""
    ordered = sorted((a, b) for a, b in runs if b > a)
    merged: list[list[int]] = []
    for a, b in ordered:
        if merged and a <= merged[-1][1]:
            if b > merged[-1][1]:
                merged[-1][1] = b
        else:
            merged.append([a, b])
    return tuple((a, b) for a, b in merged)


def runs_len(x: Runs) -> int:
    return sum(b - a for a, b in x)


def runs_or(x: Runs, y: Runs) -> Runs:
    """Union (core.py:126-131)."""
    if not x:
        return y
    if not y:
        return x
    return norm_runs(x + y)


def runs_and(x: Runs, y: Runs) -> Runs:
    """Intersection by a two-pointer sweep (core.py:133-149)."""
    out = []
    i = j = 0
    while i < len(x) and j < len(y):
        lo = max(x[i][0], y[j][0])
        hi = min(x[i][1], y[j][1])
        if lo < hi:
            out.append((lo, hi))
        if x[i][1] <= y[j][1]:
            i += 1
        else:
            j += 1
    return tuple(out)


def runs_sub(x: Runs, y: Runs) -> Runs:
    """Difference x - y (core.py:151-174)."""
    if not x or not y:
        return x
    out = []
    j = 0
    for a, b in x:
        pos = a
        while j < len(y) and y[j][1] <= pos:
            j += 1
        k = j
        while k < len(y) and y[k][0] < b:
            c, d = y[k]
            if c > pos:
                out.append((pos, c))
            pos = max(pos, d)
            if d >= b:
                break
            k += 1
        if pos < b:
            out.append((pos, b))
    return tuple(out)


def runs_pages(x: Runs) -> list[int]:
    return [p for a, b in x for p in range(a, b)]


def byte_pages(start: int, length: int, page: int) -> Runs:
    """Pages overlapping [start, start+length) (core.py:192-198)."""
    if length <= 0:
        raise ValueError("zero-length range")
    return ((start // page, (start + length - 1) // page + 1),)


def ranges_pages(ranges, page: int) -> Runs:
    """core.py:201-207: union of the page spans of byte ranges."""
    spans = []
    for r in ranges:
        spans.append((r.start_addr // page, (r.start_addr + r.length_bytes - 1) // page + 1))
    return norm_runs(spans)


# ---------------------------------------------------------------------------
# eviction list (memman.py:23-137)


def _append_run(dst: list, a: int, b: int):
    if dst and dst[-1][1] == a:
        dst[-1] = (dst[-1][0], b)
    else:
        dst.append((a, b))


class RunList:
    """Ordered resident runs, head = next victim (memman.py:23-137)."""

    def __init__(self):
        self.runs: list[tuple[int, int]] = []
        self.resident: Runs = ()

    def __len__(self):
        return runs_len(self.resident)

    def order(self) -> list[int]:
        return runs_pages(self.runs)

    def append(self, runs):
        """memman.py:43-56."""
        fresh = []
        for a, b in runs:
            if b <= a:
                continue
            _append_run(self.runs, a, b)
            fresh.append((a, b))
        if fresh:
            self.resident = runs_or(self.resident, norm_runs(fresh))

    def advise(self, pages: Runs):
        """Stable move of the resident members of `pages` to the tail
        (memman.py:58-91)."""
        if not pages or not self.runs:
            return
        starts = [a for a, _ in pages]
        stay: list = []
        move: list = []
        npg = len(pages)
        for a, b in self.runs:
            pos = a
            i = bisect_right(starts, pos) - 1
            if i < 0:
                i = 0
            while pos < b and i < npg:
                c, d = pages[i]
                if d <= pos:
                    i += 1
                    continue
                if c >= b:
                    break
                lo, hi = max(pos, c), min(b, d)
                if pos < lo:
                    _append_run(stay, pos, lo)
                _append_run(move, lo, hi)
                pos = hi
                if d <= b:
                    i += 1
            if pos < b:
                _append_run(stay, pos, b)
        stay.extend(move)
        merged: list = []
        for a, b in stay:
            _append_run(merged, a, b)
        self.runs = merged

    def pop_head(self, n: int) -> list:
        """memman.py:93-112."""
        if n <= 0:
            return []
        got = []
        while n > 0 and self.runs:
            a, b = self.runs[0]
            if b - a <= n:
                got.append((a, b))
                self.runs.pop(0)
                n -= b - a
            else:
                got.append((a, a + n))
                self.runs[0] = (a + n, b)
                n = 0
        if got:
            self.resident = runs_sub(self.resident, norm_runs(got))
        return got

    def drop(self, pages: Runs):
        """memman.py:114-123."""
        if not pages or not self.runs:
            return
        kept: list = []
        for a, b in self.runs:
            for c, d in runs_sub(((a, b),), pages):
                _append_run(kept, c, d)
        self.runs = kept
        self.resident = runs_sub(self.resident, pages)


# ---------------------------------------------------------------------------
# windows, OPT reordering, migration plans (memman.py:163-307)


class Win:
    """memman.py:163-171."""

    __slots__ = ("task_id", "ordered", "demand", "pages", "end", "start")

    def __init__(self, task_id, ordered, demand, pages, end, start):
        self.task_id = task_id
        self.ordered = ordered
        self.demand = demand
        self.pages = pages
        self.end = end
        self.start = start


def window_of(task_id, preds, self_pop, lat, cursor: int, budget: float) -> Win:
    """memman.py:174-196: walk from `cursor` while the profiled time is under
    budget, collecting first-access-ordered new runs."""
    ordered: list = []
    demand: list = []
    seen: Runs = ()
    spent = 0.0
    c = cursor
    n = len(lat)
    while c < n and spent < budget:
        new = runs_sub(preds[c], seen)
        if new:
            ordered.extend(new)
            if not (c < len(self_pop) and self_pop[c]):
                demand.extend(new)
            seen = runs_or(seen, new)
        spent += lat[c]
        c += 1
    return Win(task_id, ordered, demand, seen, c, cursor)


def windows_of(entries, tables) -> list:
    """memman.py:199-206."""
    out = []
    for tid, slice_s, cursor in entries:
        if tid in tables:
            t = tables[tid]
            out.append(window_of(tid, t.preds, t.self_pop, t.lat, cursor, slice_s))
    return out


def opt_reorder(rl: RunList, wins) -> dict:
    """memman.py:218-241: advise each window's runs last-to-first, windows
    last-to-first; returns {task: pages advised} in first-insertion order."""
    advised: dict = {}
    for w in reversed(list(wins)):
        for run in reversed(w.ordered):
            rl.advise((run,))
        advised[w.task_id] = advised.get(w.task_id, 0) + runs_len(w.pages)
    return advised


def advise_cost(hw, advised: dict) -> float:
    """memman.py:244-251."""
    return sum(hw.madvise_call_s + n * hw.per_page_madvise_s for n in advised.values())


class Plan:
    __slots__ = ("evict", "populate", "truncated")

    def __init__(self, evict, populate, truncated):
        self.evict = evict
        self.populate = populate
        self.truncated = truncated

    @property
    def n_evict(self):
        return sum(b - a for a, b in self.evict)

    @property
    def n_populate(self):
        return sum(b - a for a, b in self.populate)


def make_plan(rl: RunList, demand_runs, capacity: int) -> Plan:
    """memman.py:269-302."""
    populate = []
    taken = 0
    truncated = 0
    for run in demand_runs:
        for a, b in runs_sub((run,), rl.resident):
            k = min(b - a, capacity - taken)
            if k > 0:
                populate.append((a, a + k))
                taken += k
            truncated += (b - a) - k
    need = max(0, taken - (capacity - len(rl)))
    evict = []
    for a, b in rl.runs:
        if need <= 0:
            break
        k = min(b - a, need)
        evict.append((a, a + k))
        need -= k
    return Plan(evict, populate, truncated)


def apply_plan_runs(rl: RunList, plan: Plan):
    """memman.py:305-307."""
    rl.pop_head(plan.n_evict)
    rl.append(plan.populate)


def belady(seq, frames: int):
    """memman.py:310-341: brute-force OPT (farthest next use; never-used
    first; ties to the lowest page id)."""
    if frames < 1:
        raise ValueError("frames must be >= 1")
    held: set = set()
    faults = 0
    trace = []
    n = len(seq)
    for i, p in enumerate(seq):
        if p in held:
            continue
        faults += 1
        if len(held) >= frames:
            victim, far = -1, -1
            for q in sorted(held):
                nxt = next((j for j in range(i + 1, n) if seq[j] == q), n + 1)
                if nxt > far:
                    victim, far = q, nxt
            held.remove(victim)
            trace.append((i, victim))
        held.add(p)
    return faults, trace


# ---------------------------------------------------------------------------
# rule evaluation (analyzer.py:67-174)


def struct_words(raw: bytes):
    """analyzer.py:67-75: aligned 64-bit then 32-bit little-endian windows."""
    out = [(o, 64, struct.unpack_from("<Q", raw, o)[0]) for o in range(0, len(raw) - 7, 8)]
    out += [(o, 32, struct.unpack_from("<I", raw, o)[0]) for o in range(0, len(raw) - 3, 4)]
    return out


def slot_table(args, grid=(1, 1, 1), block=(1, 1, 1)) -> dict:
    """analyzer.py:78-96."""
    vals = {}
    for i, a in enumerate(args):
        if a.raw is not None:
            for o, w, v in struct_words(a.raw):
                vals[f"a{i}+{o}w{w}"] = v
        else:
            vals[f"a{i}"] = a.value
    for nm, v in zip(("gx", "gy", "gz", "bx", "by", "bz"), tuple(grid) + tuple(block)):
        vals[nm] = v
    return vals


def eval_expr(coeff: Fraction, slots, vals):
    """analyzer.py:119-128: exact coeff * prod(slots), None if a slot is
    missing or the product is not integral."""
    prod = Fraction(1)
    for s in slots:
        if s not in vals:
            return None
        prod *= vals[s]
    v = coeff * prod
    return int(v) if v.denominator == 1 else None


def rule_regions(rule, cmd):
    """analyzer.py:155-174.  `rule` is duck-typed on the reference's
    TemplateRule (kind, ptr_arg_index, offset_bytes, size/stride/chunk/count
    with .coeff/.slots).  Returns [(start, length)] or None."""
    if rule.kind == "unpredictable" or rule.ptr_arg_index >= len(cmd.launch_args):
        return None
    base = cmd.launch_args[rule.ptr_arg_index].value + rule.offset_bytes
    vals = slot_table(cmd.launch_args, cmd.grid_dims, cmd.block_dims)
    if rule.kind in ("fixed", "linear"):
        size = eval_expr(rule.size.coeff, rule.size.slots, vals)
        if size is None:
            return None
        return [(base, max(size, 1))]
    stride = eval_expr(rule.stride.coeff, rule.stride.slots, vals)
    chunk = eval_expr(rule.chunk.coeff, rule.chunk.slots, vals)
    count = eval_expr(rule.count.coeff, rule.count.slots, vals)
    if stride is None or chunk is None or count is None or count < 1:
        return None
    return [(base + j * stride, max(chunk, 1)) for j in range(count)]


def _device_extent(cmd) -> tuple:
    """core.py:254-260: the device side of a memcpy."""
    a = cmd.launch_args
    addr = a[1].value if _kind(cmd) == "H2D" else a[0].value
    return addr, a[2].value


def predict_template(descs: dict, cmd, page: int):
    """predictor.py:24-44 -> (runs, complete)."""
    if _kind(cmd) != "KERNEL":
        s, n = _device_extent(cmd)
        return byte_pages(s, n, page), True
    d = descs.get(cmd.kernel_name)
    if d is None:
        return (), False
    spans = []
    complete = True
    for rule in d.rules:
        regs = rule_regions(rule, cmd)
        if regs is None:
            complete = False
            continue
        for s, n in regs:
            spans.append((s // page, (s + n - 1) // page + 1))
    if d.unpredictable_fraction > 0.0:
        complete = False
    return norm_runs(spans), complete


def predict_alloc(allocs, cmd, page: int):
    """predictor.py:47-65."""
    if _kind(cmd) != "KERNEL":
        s, n = _device_extent(cmd)
        return byte_pages(s, n, page), True
    spans = []
    for a in cmd.launch_args:
        if a.raw is not None or a.width != 64:
            continue
        for al in allocs:
            if al.base_addr <= a.value < al.base_addr + al.size_bytes:
                spans.append(byte_pages(al.base_addr, al.size_bytes, page)[0])
                break
    return norm_runs(spans), True


def predict_truth(cmd, page: int) -> Runs:
    """predictor.py:74-77 and engine.py:246-249 (the 'actual' set)."""
    if _kind(cmd) != "KERNEL":
        s, n = _device_extent(cmd)
        return byte_pages(s, n, page)
    return ranges_pages(cmd.ground_truth_access, page)


def accuracy(predicted: Runs, actual: Runs):
    """predictor.py:80-87 (F+ is over |actual|, as the code does)."""
    n = runs_len(actual)
    if n == 0:
        return (0.0, 0.0)
    return (runs_len(runs_sub(actual, predicted)) / n, runs_len(runs_sub(predicted, actual)) / n)


# ---------------------------------------------------------------------------
# offline descriptor inference (analyzer.py:31-441)


class _Expr:
    __slots__ = ("coeff", "slots")

    def __init__(self, coeff, slots=()):
        self.coeff = coeff
        self.slots = tuple(slots)

    def text(self):
        """analyzer.py:130-133."""
        if not self.slots:
            return f"fixed:{self.coeff}"
        return "lin:" + str(self.coeff) + "*" + "*".join(self.slots)


class _Rule:
    __slots__ = ("ptr_arg_index", "kind", "offset_bytes", "size", "stride", "chunk", "count")

    def __init__(self, ptr, kind, off=0, size=None, stride=None, chunk=None, count=None):
        self.ptr_arg_index = ptr
        self.kind = kind
        self.offset_bytes = off
        self.size = size
        self.stride = stride
        self.chunk = chunk
        self.count = count


class _Desc:
    __slots__ = ("kernel_name", "rules", "profiled_latency_s", "unpredictable_fraction")

    def __init__(self, name, rules, lat):
        self.kernel_name = name
        self.rules = rules
        self.profiled_latency_s = lat
        self.unpredictable_fraction = 0.0


def _merge_overlaps(ranges):
    """analyzer.py:53-64: sort by start, merge strictly overlapping ranges."""
    out = []
    for s, n in sorted(((r.start_addr, r.length_bytes) for r in ranges), key=lambda t: t[0]):
        if out and s < out[-1][0] + out[-1][1]:
            ps, pn = out[-1]
            out[-1] = (ps, max(ps + pn, s + n) - ps)
        else:
            out.append((s, n))
    return out


class _Rec:
    __slots__ = ("args", "grid", "block", "regions", "lat", "vals")

    def __init__(self, cmd):
        self.args = cmd.launch_args
        self.grid = cmd.grid_dims
        self.block = cmd.block_dims
        self.regions = _merge_overlaps(cmd.ground_truth_access)
        self.lat = cmd.latency_s
        self.vals = slot_table(self.args, self.grid, self.block)


def _slot_rank(name: str):
    """analyzer.py:99-109."""
    if name[0] == "a":
        body = name[1:]
        if "+" in body:
            i, rest = body.split("+")
            off, w = rest.split("w")
            return (0, int(i), 1, int(off), -int(w))
        return (0, int(body), 0, 0, 0)
    return (1, ("gx", "gy", "gz", "bx", "by", "bz").index(name), 0, 0, 0)


def _is_plain64(a) -> bool:
    return a.raw is None and a.width == 64


def _pointer_args(recs):
    """analyzer.py:185-206."""
    out = []
    for i in range(len(recs[0].args)):
        if all(
            i < len(r.args) and _is_plain64(r.args[i])
            and any(s == r.args[i].value for s, _ in r.regions)
            for r in recs
        ):
            out.append(i)
    return out


def _offset_arg(recs, i):
    """analyzer.py:209-226."""
    common = None
    for r in recs:
        a = r.args[i]
        if not _is_plain64(a):
            return None
        offs = {s - a.value for s, _ in r.regions if a.value < s < 2 * a.value}
        common = offs if common is None else common & offs
        if not common:
            return None
    return min(common)


def _factor_slots(recs, ptr_idx):
    """analyzer.py:240-263."""
    names = sorted(recs[0].vals, key=_slot_rank)
    seen = set()
    out = []
    for nm in names:
        if nm[0] == "a" and "+" not in nm and int(nm[1:]) in ptr_idx:
            continue
        sig = tuple(r.vals.get(nm) for r in recs)
        if any(v is None or v <= 0 for v in sig) or sig in seen:
            continue
        seen.add(sig)
        out.append(nm)
    return out


def _fit(values, recs, slots, max_terms=3):
    """analyzer.py:266-293."""
    if all(v == values[0] for v in values):
        return _Expr(Fraction(values[0]))
    for k in range(1, max_terms + 1):
        for combo in itertools.combinations_with_replacement(slots, k):
            coeff = None
            for v, r in zip(values, recs):
                prod = 1
                for s in combo:
                    prod *= r.vals[s]
                c = Fraction(v, prod)
                if coeff is None:
                    coeff = c
                elif c != coeff:
                    coeff = False
                    break
            if coeff is not False and coeff is not None and coeff > 0:
                return _Expr(coeff, combo)
    return None


def _infer(recs, ptr, off, ptr_offsets):
    """analyzer.py:296-349."""
    fams = []
    for r in recs:
        base = r.args[ptr].value + off
        others = {r.args[i].value + o for i, o in ptr_offsets.items() if not (i == ptr and o == off)}
        ceiling = min((b for b in others if b > base), default=None)
        fam = [(s, n) for s, n in r.regions if s >= base and (ceiling is None or s < ceiling)]
        if not fam or fam[0][0] != base:
            return _Rule(ptr, "unpredictable", off)
        fams.append(fam)
    slots = _factor_slots(recs, set(ptr_offsets))
    if all(len(f) == 1 for f in fams):
        sizes = [f[0][1] for f in fams]
        if all(s == sizes[0] for s in sizes):
            return _Rule(ptr, "fixed", off, size=_Expr(Fraction(sizes[0])))
        e = _fit(sizes, recs, slots)
        if e is not None and e.slots:
            return _Rule(ptr, "linear", off, size=e)
        return _Rule(ptr, "unpredictable", off)
    strides, chunks, counts = [], [], []
    for f in fams:
        if len(f) < 2:
            return _Rule(ptr, "unpredictable", off)
        st = {f[k + 1][0] - f[k][0] for k in range(len(f) - 1)}
        ln = {n for _, n in f}
        if len(st) != 1 or len(ln) != 1:
            return _Rule(ptr, "unpredictable", off)
        strides.append(st.pop())
        chunks.append(ln.pop())
        counts.append(len(f))
    es, ec, en = _fit(strides, recs, slots), _fit(chunks, recs, slots), _fit(counts, recs, slots)
    if es is None or ec is None or en is None:
        return _Rule(ptr, "unpredictable", off)
    return _Rule(ptr, "strided", off, stride=es, chunk=ec, count=en)


def _uncovered(desc, recs, cmds):
    """analyzer.py:405-418."""
    total = misses = 0
    for r, cmd in zip(recs, cmds):
        pred = []
        for rule in desc.rules:
            regs = rule_regions(rule, cmd)
            if regs:
                pred.extend(regs)
        for s, n in r.regions:
            total += 1
            if not any(ps <= s and ps + pn >= s + n for ps, pn in pred):
                misses += 1
    return misses / total if total else 0.0


def infer_descriptors(task) -> dict:
    """analyzer.py:352-441 (build_descriptor / build_descriptors)."""
    groups: dict = {}
    for cmd in task.commands:
        if _kind(cmd) == "KERNEL":
            groups.setdefault(cmd.kernel_name, []).append(cmd)
    out = {}
    for name, cmds in groups.items():
        recs = [_Rec(c) for c in cmds]
        ptr_offsets = {i: 0 for i in _pointer_args(recs)}
        for i in range(len(recs[0].args)):
            if i not in ptr_offsets:
                c = _offset_arg(recs, i)
                if c is not None:
                    ptr_offsets[i] = c
        rules = [_infer(recs, i, o, ptr_offsets) for i, o in sorted(ptr_offsets.items())]
        d = _Desc(name, [r for r in rules if r.kind != "unpredictable"],
                  sum(r.lat for r in recs) / len(recs))
        d.unpredictable_fraction = _uncovered(d, recs, cmds)
        out[name] = d
    return out


def descriptors_text(descs: dict) -> str:
    """analyzer.py:453-474: the MSIM-DESC v1 text form."""
    lines = ["MSIM-DESC v1"]
    for name in sorted(descs):
        d = descs[name]
        lines.append(f"KERNEL {name} latency={d.profiled_latency_s!r} "
                     f"unpredictable={d.unpredictable_fraction!r}")
        for r in d.rules:
            if r.kind in ("fixed", "linear"):
                lines.append(f"RULE ptr={r.ptr_arg_index} offset={r.offset_bytes} "
                             f"kind={r.kind} size={_expr_text(r.size)}")
            else:
                lines.append(f"RULE ptr={r.ptr_arg_index} offset={r.offset_bytes} kind=strided "
                             f"stride={_expr_text(r.stride)} chunk={_expr_text(r.chunk)} "
                             f"count={_expr_text(r.count)}")
    return "\n".join(lines) + "\n"


def _expr_text(e):
    if not e.slots:
        return f"fixed:{e.coeff}"
    return "lin:" + str(e.coeff) + "*" + "*".join(e.slots)


# ---------------------------------------------------------------------------
# scheduler timeline (scheduler.py:39-97)


def _advance(lat, cursor: int, budget: float) -> int:
    """scheduler.py:86-97."""
    spent = 0.0
    c = cursor
    while c < len(lat) and spent < budget:
        spent += lat[c]
        c += 1
    return c


def timeline(policy, tasks, horizon=None):
    """scheduler.py:39-83 -> [(task_id, timeslice, cursor)].  `tasks` are
    objects with .id, .cursor, .priority and a `lat` latency list."""
    live = [t for t in tasks if len(t.lat) - t.cursor > 0]
    if not live:
        return []
    if policy.kind == "priority":
        top = max(t.priority for t in live)
        live = [t for t in live if t.priority == top]
    if horizon is None:
        horizon = policy.horizon_rounds * len(live)
    cur = {t.id: t.cursor for t in live}
    out = []
    k = 0
    alive = list(live)
    while len(out) < horizon and alive:
        t = alive[k % len(alive)]
        c = cur[t.id]
        if c >= len(t.lat):
            alive = [x for x in alive if cur[x.id] < len(x.lat)]
            if not alive:
                break
            k = 0
            continue
        out.append((t.id, policy.timeslice_s, c))
        cur[t.id] = _advance(t.lat, c, policy.timeslice_s)
        k += 1
    return out


# ---------------------------------------------------------------------------
# timing model (engine.py:126-166)


def evict_cost(hw) -> float:
    return hw.per_page_unmap_s + hw.page_size_bytes / hw.bw_d2h_bytes_per_s


def populate_cost(hw) -> float:
    return hw.page_size_bytes / hw.bw_h2d_bytes_per_s + hw.per_page_map_s


def seq_swap_time(hw, n_evict, n_pop) -> float:
    return n_evict * evict_cost(hw) + n_pop * populate_cost(hw)


def ready_time(hw, j, free, n_evict) -> float:
    """engine.py:139-158."""
    if j <= 0:
        return 0.0
    e, p = evict_cost(hw), populate_cost(hw)
    f = max(0, free)
    best = 0.0
    for i in sorted({1, min(f + 1, j), j}):
        if i < 1:
            continue
        lag = max(0, min(i, n_evict + f) - f)
        best = max(best, lag * e + (j - i + 1) * p)
    return best


def pipe_swap_time(hw, n_evict, n_pop, free) -> float:
    return max(n_evict * evict_cost(hw), ready_time(hw, n_pop, free, n_evict))


# ---------------------------------------------------------------------------
# engine (engine.py:77-473)


class SimulationError(RuntimeError):
    pass


METRIC_FIELDS = (
    "total_time_s", "exec_s", "save_restore_s", "madvise_s", "migration_s", "fault_s",
    "fault_count", "fault_pages", "prefetched_pages", "migrated_in_pages",
    "migrated_out_pages", "evicted_capacity_pages", "memcpy_installed_pages",
    "context_switches", "completed_tasks", "plan_truncations", "page_size_bytes",
    "completion_s",
)


class PortMetrics:
    """engine.py:77-115 (field names and order kept)."""

    def __init__(self, page):
        for f in METRIC_FIELDS:
            setattr(self, f, 0 if f not in ("total_time_s", "exec_s", "save_restore_s",
                                            "madvise_s", "migration_s", "fault_s") else 0.0)
        self.page_size_bytes = page
        self.completion_s = {}

    def as_dict(self):
        return {f: getattr(self, f) for f in METRIC_FIELDS}


class _TaskState:
    __slots__ = ("id", "cursor", "priority", "arrival_s", "lat", "cmds", "allocs",
                 "preds", "self_pop", "actual")

    def __init__(self, t):
        self.id = t.id
        self.cursor = t.cursor
        self.priority = t.priority
        self.arrival_s = t.arrival_s
        self.cmds = list(t.commands)
        self.lat = [c.latency_s for c in self.cmds]
        self.allocs = list(t.allocations)
        self.preds = []
        self.self_pop = []
        self.actual = []

    def remaining(self):
        return len(self.cmds) - self.cursor


class PortSim:
    """engine.py:169-473 restated over the run-list structures above.

    `recorder`, if given, is a list that receives one dict per planner
    decision: {"ev": "switch"|"touch"|"release", ...}.
    """

    def __init__(self, tasks, hw, policy, mode, feeder=None, record_events=False,
                 recorder=None, descriptors=None, order_every=1, pack=None):
        self.order_every = order_every   # record the full list order every k-th reorder (0: never)
        self.pack = pack or (lambda pages: pages)   # applied to recorded page lists (e.g. a digest)
        self._nreorder = 0
        self._nrefresh = 0
        self.hw, self.policy, self.mode, self.feeder = hw, policy, mode, feeder
        self.page = hw.page_size_bytes
        self.capacity = hw.hbm_capacity_bytes // hw.page_size_bytes
        self.tasks = [_TaskState(t) for t in tasks]
        for t, src in zip(self.tasks, tasks):
            _validate(src)
        self.by_id = {t.id: t for t in self.tasks}
        if len(self.by_id) != len(self.tasks):
            raise SimulationError("duplicate task ids")
        self.rr = [t.id for t in self.tasks]
        total = sum(a.size_bytes for t in self.tasks for a in t.allocs)
        if total > hw.dram_capacity_bytes:
            raise SimulationError(f"allocations ({total} B) exceed DRAM backing "
                                  f"({hw.dram_capacity_bytes} B)")
        self.rl = RunList()
        self.m = PortMetrics(self.page)
        self.t = 0.0
        self.events = []
        self.record_events = record_events
        self.rec = recorder
        self.descs = {}
        for t, src in zip(self.tasks, tasks):
            if mode.predictor == "template" and mode.name == "proactive":
                self.descs[t.id] = (descriptors or {}).get(t.id) or infer_descriptors(src)
            self._extend(t, t.cmds)

    # engine.py:230-249
    def _extend(self, t, cmds):
        for c in cmds:
            t.preds.append(self._predict(t, c))
            t.self_pop.append(_kind(c) == "H2D")
            t.actual.append(predict_truth(c, self.page))

    def _predict(self, t, c):
        if self.mode.name == "ideal" or self.mode.predictor == "oracle":
            return predict_truth(c, self.page)
        if self.mode.predictor == "allocation":
            return predict_alloc(t.allocs, c, self.page)[0]
        return predict_template(self.descs.get(t.id, {}), c, self.page)[0]

    def append_commands(self, task_id, commands):
        """engine.py:251-258."""
        t = self.by_id[task_id]
        if len(t.cmds) - t.cursor == 0 and t.cmds:
            raise SimulationError(f"cannot append to completed task {task_id!r}")
        commands = list(commands)
        t.cmds.extend(commands)
        t.lat.extend(c.latency_s for c in commands)
        self._extend(t, commands)

    def _charge(self, dt, bucket):
        self.t += dt
        setattr(self.m, bucket, getattr(self.m, bucket) + dt)

    def _emit(self, kind, tid, pages=0):
        if self.record_events:
            self.events.append((self.t, kind, tid, pages))

    # engine.py:262-293
    def run(self, max_switches=1_000_000):
        proactive = self.mode.name in ("proactive", "ideal")
        for _ in range(max_switches):
            if self.feeder is not None:
                self.feeder(self)
            live = [t for t in self.tasks if len(t.cmds) - t.cursor > 0]
            if not live:
                break
            ready = [t for t in live if t.arrival_s <= self.t + 1e-15]
            if not ready:
                self.t = min(t.arrival_s for t in live)
                continue
            rank = {tid: i for i, tid in enumerate(self.rr)}
            ready.sort(key=lambda t: rank[t.id])
            tl = timeline(self.policy, ready)
            tid, slice_s, cursor = tl[0]
            t = self.by_id[tid]
            self.rr.remove(tid)
            self.rr.append(tid)
            self.m.context_switches += 1
            self._charge(self.hw.save_restore_s, "save_restore_s")
            pending = self._prepare(tl) if proactive else None
            self._emit("switch", tid)
            self._slice(t, tl, pending)
            if len(t.cmds) - t.cursor == 0:
                self._release(t)
        else:
            raise SimulationError("context-switch budget exhausted")
        self.m.total_time_s = self.t
        return self.m

    # engine.py:305-340
    def _prepare(self, tl):
        wins = windows_of(tl, self.by_id)
        w0 = wins[0]
        missing = runs_sub(norm_runs(w0.demand), self.rl.resident)
        rec = None
        if self.rec is not None:
            rec = {"ev": "switch", "task": tl[0][0],
                   "windows": [(w.task_id, w.start, w.end) for w in wins],
                   "missing": runs_len(missing)}
            self.rec.append(rec)
        if not missing and len(self.rl) + runs_len(missing) - self.capacity <= 0:
            return None
        advised = opt_reorder(self.rl, wins)
        if self.mode.name == "proactive":
            self._charge(advise_cost(self.hw, advised), "madvise_s")
        free = self.capacity - len(self.rl)
        plan = make_plan(self.rl, w0.demand, self.capacity)
        if rec is not None:
            rec.update(advised=list(advised.items()), evict=self.pack(runs_pages(plan.evict)),
                       populate=self.pack(runs_pages(plan.populate)), truncated=plan.truncated, free=free)
            if self.order_every and self._nreorder % self.order_every == 0:
                rec["order_after_reorder"] = self.pack(self.rl.order())
        self._nreorder += 1
        if plan.truncated:
            self.m.plan_truncations += 1
        self.m.migrated_in_pages += plan.n_populate
        self.m.migrated_out_pages += plan.n_evict
        self._emit("migrate", tl[0][0], plan.n_populate)
        pending = None
        if not self.mode.pipelined:
            self._charge(seq_swap_time(self.hw, plan.n_evict, plan.n_populate), "migration_s")
        elif self.mode.early_start:
            pending = self._gating(tl[0], w0, plan, free)
            if rec is not None:
                rec["prefix"] = self.pack([pending["prefix"][c] for c in range(w0.start, w0.end)])
        else:
            self._charge(pipe_swap_time(self.hw, plan.n_evict, plan.n_populate, free), "migration_s")
        apply_plan_runs(self.rl, plan)
        if len(self.rl) > self.capacity:
            raise SimulationError("migration plan overflowed HBM capacity")
        return pending

    # engine.py:342-361
    def _gating(self, entry, w0, plan, free):
        t = self.by_id[entry[0]]
        seen = ()
        cum = 0
        prefix = {}
        for c in range(entry[2], w0.end):
            new = runs_sub(t.preds[c], seen)
            seen = runs_or(seen, new)
            if not t.self_pop[c]:
                cum += runs_len(runs_sub(new, self.rl.resident))
            prefix[c] = min(cum, plan.n_populate)
        return {"prefix": prefix, "free": free, "n_evict": plan.n_evict,
                "evict_done": plan.n_evict * evict_cost(self.hw)}

    # engine.py:365-387
    def _slice(self, t, tl, pending):
        budget = tl[0][1]
        spent = 0.0
        off = 0.0
        start = self.t
        while t.cursor < len(t.cmds) and spent < budget:
            c = t.cursor
            if pending is not None:
                j = pending["prefix"].get(c, 0)
                r = ready_time(self.hw, j, pending["free"], pending["n_evict"])
                if r > off:
                    self.m.migration_s += r - off
                    off = r
            off += self._touch(t, c, tl, budget - spent)
            off += t.lat[c]
            spent += t.lat[c]
            t.cursor = c + 1
        if pending is not None and pending["evict_done"] > off:
            self.m.migration_s += pending["evict_done"] - off
            off = pending["evict_done"]
        self.t = start + off
        self.m.exec_s += spent

    # engine.py:389-428
    def _touch(self, t, c, tl, remaining):
        if self.mode.name == "reference":
            return 0.0
        actual = t.actual[c]
        missing = runs_sub(actual, self.rl.resident)
        if not missing:
            if self.mode.name == "um":
                self.rl.advise(actual)
            return 0.0
        n = runs_len(missing)
        if n > self.capacity:
            raise SimulationError(f"command working set ({n} pages) exceeds HBM "
                                  f"capacity ({self.capacity} pages)")
        stall = 0.0
        over = len(self.rl) + n - self.capacity
        evicted = []
        if over > 0:
            if self.mode.name in ("proactive", "ideal"):
                stall += self._refresh(t, c, tl, remaining)
            evicted = self.rl.pop_head(over)
            self.m.evicted_capacity_pages += sum(b - a for a, b in evicted)
        if _kind(t.cmds[c]) == "H2D":
            self.m.memcpy_installed_pages += n
        else:
            stall += self._fault(n)
        self.rl.append(missing)
        if len(self.rl) > self.capacity:
            raise SimulationError(f"residency {len(self.rl)} pages exceeds capacity "
                                  f"{self.capacity} after command {c} of task {t.id!r}")
        if self.rec is not None:
            self.rec.append({"ev": "touch", "task": t.id, "cmd": c, "missing": self.pack(runs_pages(missing)),
                             "evicted": self.pack(runs_pages(evicted))})
        if self.mode.name == "um":
            self.rl.advise(actual)
        self._emit("fault", t.id, n)
        return stall

    # engine.py:430-445
    def _fault(self, n):
        hw = self.hw
        self.m.fault_pages += n
        if self.mode.name == "ideal":
            dt = n * populate_cost(hw)
        else:
            batches = math.ceil(n / self.mode.prefetch_pages)
            self.m.fault_count += batches
            self.m.prefetched_pages += batches * self.mode.prefetch_pages - n
            dt = batches * (hw.fault_control_plane_s + hw.fault_transfer_s * self.mode.prefetch_pages)
        self.m.fault_s += dt
        return dt

    # engine.py:447-460
    def _refresh(self, t, c, tl, remaining):
        head = window_of(t.id, t.preds, t.self_pop, t.lat, c, max(remaining, 1e-12))
        rest = windows_of(tl[1:], self.by_id)
        advised = opt_reorder(self.rl, [head] + rest)
        if self.rec is not None:
            r = {"ev": "refresh", "task": t.id, "cmd": c,
                 "windows": [(w.task_id, w.start, w.end) for w in [head] + rest]}
            if self.order_every and self._nrefresh % self.order_every == 0:
                r["order"] = self.pack(self.rl.order())
            self.rec.append(r)
        self._nrefresh += 1
        if self.mode.name == "proactive":
            dt = advise_cost(self.hw, advised)
            self.m.madvise_s += dt
            return dt
        return 0.0

    # engine.py:462-473
    def _release(self, t):
        self.m.completed_tasks += 1
        self.m.completion_s[t.id] = self.t
        if self.mode.name == "reference":
            return
        spans = ()
        for a in t.allocs:
            lo = a.base_addr // self.page
            hi = (a.base_addr + a.size_bytes - 1) // self.page + 1
            spans = runs_or(spans, norm_runs(((lo, hi),)))
        self.rl.drop(spans)
        self._emit("release", t.id, runs_len(spans))


def _validate(task):
    """core.py:274-281."""
    allocs = sorted(task.allocations, key=lambda a: a.base_addr)
    for a, b in zip(allocs, allocs[1:]):
        if a.base_addr + a.size_bytes > b.base_addr:
            raise ValueError(f"overlapping allocations {a.id}/{b.id}")
    if not 0 <= task.cursor <= len(task.commands):
        raise ValueError("cursor out of range")


def port_simulate(tasks, hw, policy, mode, feeder=None, record_events=False, recorder=None):
    """engine.py:488-496."""
    return PortSim(tasks, hw, policy, mode, feeder, record_events, recorder).run()
