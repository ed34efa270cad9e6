"""The drop-in memman / predictor API on the GPU, written like the
reference's own tests (test_memman.py, test_predictor.py) plus randomized
comparisons against the CPU oracle's run-list eviction list."""

import random

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import msched_port as port
from paper_2512_24637_b200 import memman, predictor
from paper_2512_24637_b200.model import ByteRange, Command, CommandKind, PageSet, Task
from paper_2512_24637_b200.scheduler import TimelineEntry
from tests.golden import loader

pytestmark = pytest.mark.gpu
PAGE = 4096


def make_list(pages, domain=4096):
    ev = memman.EvictionList(domain_pages=domain)
    for p in pages:
        ev.append_tail([(p, p + 1)])
    return ev


def test_madvise_moves_to_tail_preserving_order():          # test_memman.py:29-34
    ev = make_list([10, 20, 30, 40])
    ev.madvise(PageSet.from_pages([40, 20]))
    assert ev.pages_in_order() == [10, 30, 20, 40]


def test_madvise_nonresident_ignored():                       # :37-40
    ev = make_list([1, 2, 3])
    ev.madvise(PageSet.from_pages([99, 2]))
    assert ev.pages_in_order() == [1, 3, 2]


@settings(max_examples=60, deadline=None)
@given(st.lists(st.integers(0, 50), unique=True, max_size=30), st.sets(st.integers(0, 60), max_size=20))
def test_madvise_membership_invariance(pages, advised):       # :43-59
    ev = make_list(pages, domain=64)
    before = set(ev.resident)
    ev.madvise(PageSet.from_pages(advised))
    assert set(ev.resident) == before
    kept = [p for p in pages if p not in advised]
    order = ev.pages_in_order()
    assert [p for p in order if p not in advised] == kept
    assert order[len(kept):] == [p for p in pages if p in advised]


def test_evict_head_and_remove():                             # :62-75
    ev = make_list([5, 6, 7, 1, 2])
    assert [p for a, b in ev.evict_head(3) for p in range(a, b)] == [5, 6, 7]
    assert ev.pages_in_order() == [1, 2] and ev.evict_head(0) == []
    ev = make_list([1, 2, 3, 4, 5])
    ev.remove(PageSet.from_pages([2, 4]))
    assert ev.pages_in_order() == [1, 3, 5] and len(ev) == 3


def test_plan_migration_keeps_requested_run_boundaries():   # memman.py:283-290
    # pieces of two adjacent requested runs stay two runs, as in the reference
    plan = memman.plan_migration(memman.EvictionList(domain_pages=64), [(0, 5), (5, 10)], capacity_pages=16)
    assert plan.populate_runs == [(0, 5), (5, 10)]
    ev = make_list([2, 7])
    plan = memman.plan_migration(ev, [(0, 5), (5, 10), (20, 22)], capacity_pages=9)
    assert plan.populate_runs == [(0, 2), (3, 5), (5, 7), (8, 10), (20, 21)] and plan.truncated_pages == 1


@settings(max_examples=60, deadline=None)
@given(st.lists(st.integers(0, 60), unique=True, max_size=30),
       st.lists(st.tuples(st.integers(0, 63), st.integers(1, 8)), max_size=8), st.integers(1, 40))
def test_plan_migration_matches_oracle_runs(pages, reqs, cap):
    runs, used = [], set()
    for a, n in reqs:                     # disjoint first-access runs, as compute_window makes them
        r = [p for p in range(a, min(a + n, 64)) if p not in used]
        if r and r == list(range(r[0], r[-1] + 1)):
            runs.append((r[0], r[-1] + 1))
            used.update(r)
    pages = pages[:cap]
    ev = make_list(pages, domain=64)
    plan = memman.plan_migration(ev, runs, capacity_pages=cap)
    rl = port.RunList()
    for p in pages:
        rl.append([(p, p + 1)])
    ref = port.make_plan(rl, runs, cap)
    assert plan.populate_runs == ref.populate
    assert plan.evict_runs == ref.evict
    assert plan.truncated_pages == ref.truncated


def test_plan_migration_known_answers():                      # :118-141
    ev = make_list([0, 1, 2])
    plan = memman.plan_migration(ev, [(0, 5)], capacity_pages=8)
    assert plan.populate_runs == [(3, 5)] and plan.evict_runs == [] and plan.truncated_pages == 0
    ev = make_list([10, 11, 12, 13])
    plan = memman.plan_migration(ev, [(20, 23)], capacity_pages=4)
    assert plan.populate_pages == 3 and plan.evict_pages == 3
    assert [p for a, b in plan.evict_runs for p in range(a, b)] == [10, 11, 12]
    memman.apply_plan(ev, plan)
    assert ev.pages_in_order() == [13, 20, 21, 22]
    plan = memman.plan_migration(memman.EvictionList(domain_pages=64), [(0, 10)], capacity_pages=4)
    assert plan.populate_pages == 4 and plan.truncated_pages == 6


def _page_task(tid, seq):
    return Task(id=tid, commands=[Command(CommandKind.KERNEL, 1e-6, "touch",
                                          ground_truth_access=(ByteRange(p * PAGE, PAGE),)) for p in seq])


def _helper(task):
    h = memman.HelperQueue(task)
    h.append([PageSet([(c.ground_truth_access[0].start_addr // PAGE,) * 2]) for c in task.commands])
    h.predicted = [PageSet([(c.ground_truth_access[0].start_addr // PAGE,
                             c.ground_truth_access[0].start_addr // PAGE + 1)]) for c in task.commands]
    return h


def test_compute_window_first_access_and_slice():             # :165-176
    w = memman.compute_window(_helper(_page_task("t", [3, 1, 3, 2])), 0, 1.0)
    assert [a for a, _ in w.ordered_runs] == [3, 1, 2] and w.end_cursor == 4
    w = memman.compute_window(_helper(_page_task("t", [3, 1, 2])), 0, 1.5e-6)
    assert w.end_cursor == 2 and set(w.pages) == {3, 1}


def test_reorder_realizes_next_use_order():                   # :179-191
    ev = make_list([0, 1, 2])
    t = _page_task("t", [2, 0, 1])
    tl = (TimelineEntry("t", 1.0, 0),)
    memman.reorder_for_opt(ev, tl, {"t": _helper(t)})
    assert ev.pages_in_order() == [1, 0, 2]
    ev2 = make_list([7, 2, 9])
    memman.reorder_for_opt(ev2, tl, {"t": _helper(t)})
    assert ev2.pages_in_order()[:2] == [7, 9]


@pytest.mark.parametrize("path", [0, 8], ids=["coop", "onesweep"])
def test_multi_window_reorder_matches_oracle(path):
    """reorder_for_opt over several windows (one multisplit on the GPU) ==
    the reference's per-run madvise sequence (oracle run list)."""
    rng = random.Random(11)
    for _ in range(40):
        pages = rng.sample(range(3000), 600)
        ev = make_list([], domain=4096)
        ev.ctx.debug(path)
        rl = port.RunList()
        runs = port.norm_runs([(p, p + 1) for p in pages])
        # append in a shuffled run order to get a non-sorted list
        order = list(runs)
        rng.shuffle(order)
        ev.append_tail(order)
        rl.append(order)
        wins = []
        for w in range(rng.randint(1, 6)):
            k = rng.randint(1, 12)
            seen, wr = (), []
            for _ in range(k):
                a = rng.randrange(0, 3000)
                new = port.runs_sub(((a, a + rng.randint(1, 200)),), seen)
                wr.extend(new)
                seen = port.runs_or(seen, new)
            wins.append(memman.Window("t", wr, wr, PageSet(wr), 0))
        memman.reorder_for_opt(ev, (), {}, wins)
        port.opt_reorder(rl, [port.Win("t", w.ordered_runs, w.demand_runs, (), 0, 0) for w in wins])
        assert ev.pages_in_order() == rl.order()


def _closed_form_reorder(order, wins):
    """the reorder is a stable sort of the list by the
    tuple (class in window 0, ..., class in window W-1), class = K_w - r for
    the r-th first-access run of window w (0 if absent).  A numpy statement
    of it for list sizes the per-run madvise oracle cannot replay in time;
    the small randomized tests above pin it to the oracle."""
    import numpy as np

    order = np.asarray(order, dtype=np.int64)
    keys = []
    for runs in wins:
        k = len(runs)
        st = np.array([a for a, _ in runs], dtype=np.int64)
        en = np.array([b for _, b in runs], dtype=np.int64)
        srt = np.argsort(st, kind="stable")
        st, en, rank = st[srt], en[srt], srt
        i = np.searchsorted(st, order, side="right") - 1
        ok = (i >= 0) & (order < en[np.maximum(i, 0)])
        keys.append(np.where(ok, k - rank[np.maximum(i, 0)], 0))
    idx = np.lexsort(tuple(reversed(keys)) + ()) if keys else np.arange(len(order))
    return order[idx].tolist()


@pytest.mark.parametrize("path", [0, 8], ids=["coop", "onesweep"])
def test_large_reorder_matches_closed_form(path):
    """~1.2 M resident pages in ~68 K runs of varied length (both the
    run-chunk and the per-entry paths fire), > 2048 class segments (the class
    table is searched in global memory) and > 256 classes (two passes)."""
    rng = random.Random(5)
    D = 2_000_000
    ev = memman.EvictionList(domain_pages=D)
    ev.ctx.debug(path)
    starts = sorted(rng.sample(range(0, D, 8), 150_000))
    runs = port.norm_runs([(s, s + rng.choice((1, 3, 8, 8, 8))) for s in starts] +
                          [(a, a + rng.randrange(500, 20000)) for a in rng.sample(range(0, D - 20000), 60)])
    order = list(runs)
    rng.shuffle(order)
    ev.append_tail(order)
    cur = [p for a, b in order for p in range(a, b)]
    assert ev.pages_in_order() == cur
    for it in range(3):
        wins = []
        for w in range(4):
            seen, wr = (), []
            for _ in range(1500 if w == 0 else 40):
                a = rng.randrange(0, D - 30000)
                new = port.runs_sub(((a, a + rng.randint(1, 30000 if w else 300)),), seen)
                wr.extend(new)
                seen = port.runs_or(seen, new)
            wins.append(wr)
        memman.reorder_for_opt(ev, (), {}, [memman.Window("t", wr, wr, PageSet(wr), 0) for wr in wins])
        cur = _closed_form_reorder(cur, wins)
        assert ev.pages_in_order() == cur, it


@pytest.mark.parametrize("gap", [150, 60], ids=["one_group_of_35", "groups_of_three"])
def test_class_table_groups_match_closed_form(gap):
    """The wide class table sorts covered segments by (first window present,
    its class there) and orders each such group by the full class tuple; a
    window-1 run cut by many scattered window-0 pages makes one large group
    (> 32 segments: the full-key sort takes over) or, with later windows
    splitting it further, many small ones."""
    rng = random.Random(gap)
    D = 20000
    ev = memman.EvictionList(domain_pages=D)
    runs = port.norm_runs([(a, a + rng.randint(1, 40)) for a in range(0, 12000, 50)] + [(0, 6000)])
    order = list(runs)
    rng.shuffle(order)
    ev.append_tail(order)
    cur = [p for a, b in order for p in range(a, b)]
    for it in range(2):
        if gap > 100:   # one window-1 run cut into 35 segments of one tuple by window-0 pages
            wins = [[(p, p + 1) for p in range(100 + it, 5100, gap)], [(0, 5200)], [(7000, 7100)], [(8000, 8001)]]
        else:           # 100 window-1 runs, each cut by window 3 into three segments of two tuples
            wins = [[(p, p + 1) for p in range(5500 + it, 6000, gap)], [(a, a + 40) for a in range(0, 5000, 50)],
                    [(7000, 7100)], [(a + 10 + it, a + 17) for a in range(0, 5000, 50)]]
        memman.reorder_for_opt(ev, (), {}, [memman.Window("t", wr, wr, PageSet(wr), 0) for wr in wins])
        cur = _closed_form_reorder(cur, wins)
        assert ev.pages_in_order() == cur, it


@pytest.mark.parametrize("path", [0, 8], ids=["coop", "onesweep"])
def test_randomized_list_ops_match_oracle(path):
    rng = random.Random(7)
    for _ in range(20):
        ev = memman.EvictionList(domain_pages=20000)
        ev.ctx.debug(path)
        rl = port.RunList()
        for _ in range(25):
            op = rng.random()
            if op < 0.35:
                a = rng.randrange(0, 19000)
                runs = list(port.runs_sub(((a, a + rng.randrange(1, 600)),), rl.resident))
                ev.append_tail(runs)
                rl.append(runs)
            elif op < 0.7:
                runs = port.norm_runs([(x, x + rng.randrange(1, 400)) for x in
                                       (rng.randrange(0, 19000) for _ in range(rng.randrange(1, 6)))])
                ev.madvise(PageSet(runs))
                rl.advise(runs)
            elif op < 0.85:
                n = rng.randrange(0, 800)
                assert [p for a, b in ev.evict_head(n) for p in range(a, b)] == port.runs_pages(rl.pop_head(n))
            else:
                runs = port.norm_runs([(x, x + rng.randrange(1, 2000)) for x in
                                       (rng.randrange(0, 19000) for _ in range(rng.randrange(1, 4)))])
                ev.remove(PageSet(runs))
                rl.drop(runs)
            assert ev.pages_in_order() == rl.order()


def test_predictor_matches_reference_predictions():
    """Device rule evaluation (exact 128-bit rationals) == the reference's
    Fraction arithmetic, for template, allocation and ground-truth modes."""
    from paper_2512_24637_b200.analyzer import build_descriptors

    for case in loader.predictions():
        task = loader.dec_task(case["task"])
        descs = build_descriptors(task)
        tp = predictor.predict_task(task.commands, PAGE, "template", descs)
        ap = predictor.predict_task(task.commands, PAGE, "allocation", allocations=task.allocations)
        gp = predictor.predict_task(task.commands, PAGE, "oracle")
        for row, t, a, g in zip(case["rows"], tp, ap, gp):
            assert [list(r) for r in t.pages.runs] == row["template"], case["name"]
            assert t.complete == row["complete"], case["name"]
            assert [list(r) for r in a.pages.runs] == row["allocation"], case["name"]
            assert [list(r) for r in g.pages.runs] == row["truth"], case["name"]


def test_single_command_predictor_api():                      # test_predictor.py:56-106
    cmd = Command(CommandKind.MEMCPY_H2D, 1e-6, launch_args=tuple(
        __import__("paper_2512_24637_b200.model", fromlist=["Arg"]).Arg(v) for v in (0, 1 << 30, 3 * PAGE)))
    p = predictor.predict({}, cmd, PAGE)
    assert p.complete and list(p.pages) == [(1 << 30) // PAGE + i for i in range(3)]
    unk = Command(CommandKind.KERNEL, 1e-6, "unknown")
    p = predictor.predict({}, unk, PAGE)
    assert not p.complete and len(p.pages) == 0


def test_single_command_facades_match_reference_predictions():
    """The per-call facades (one cached task per descriptor / allocation
    table, commands appended call by call) == the reference's predictions,
    with calls of different modes and tasks interleaved."""
    from paper_2512_24637_b200.analyzer import build_descriptors

    cases = list(loader.predictions())
    tasks = [loader.dec_task(c["task"]) for c in cases]
    descs = [build_descriptors(t) for t in tasks]
    n = max(len(c["rows"]) for c in cases)
    for i in range(n):                     # command i of every task, round robin
        for case, task, d in zip(cases, tasks, descs):
            if i >= len(case["rows"]):
                continue
            cmd, row = task.commands[i], case["rows"][i]
            t = predictor.predict(d, cmd, PAGE)
            a = predictor.predict_allocation(task.allocations, cmd, PAGE)
            g = predictor.ground_truth_prediction(cmd, PAGE)
            assert [list(r) for r in t.pages.runs] == row["template"], (case["name"], i)
            assert t.complete == row["complete"], (case["name"], i)
            assert [list(r) for r in a.pages.runs] == row["allocation"], (case["name"], i)
            assert [list(r) for r in g.pages.runs] == row["truth"], (case["name"], i)


def test_read_pages_range_equals_per_command_reads():
    from paper_2512_24637_b200 import _abi
    from paper_2512_24637_b200.analyzer import build_descriptors

    case = next(iter(loader.predictions()))
    task = loader.dec_task(case["task"])
    ctx = _abi.Context(PAGE, 1, predictor=_abi.PRED_TEMPLATE, flags=_abi.F_LOOSE_DOMAIN)
    try:
        ctx.set_domain([(0, 1)])
        ctx.add_task(0, [(a.base_addr, a.size_bytes) for a in task.allocations])
        names, rules, offs, _ = _abi.lower_rules(build_descriptors(task))
        ctx.set_rules(0, rules, offs)
        ctx.add_commands(0, _abi.encode_commands(task.commands, {nm: k for k, nm in enumerate(names)}))
        n = len(task.commands)
        for which in (0, 1):
            for c0, c1 in ((0, n), (1, max(1, n - 1)), (n // 2, n // 2), (0, 1)):
                runs, off = ctx.read_pages_range(0, c0, c1, which)
                assert len(off) == c1 - c0 + 1 and off[0] == 0
                for k in range(c1 - c0):
                    got = [tuple(r) for r in runs[off[k]:off[k + 1]].tolist()]
                    assert got == ctx.read_pages(0, c0 + k, which)
        with pytest.raises(_abi.MsgError):
            ctx.read_pages_range(0, 1, 0, 0)
        with pytest.raises(_abi.MsgError):
            ctx.read_pages_range(0, 0, n + 1, 0)
    finally:
        ctx.close()
