"""Host fast paths must give the reference's exact values (no GPU): the
engine's cached populate_ready against engine.py:139-158's restatement, and
the scheduler's timeline entries against TimelineEntry's own constructor."""
import random
import types

from paper_2512_24637_b200 import engine
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scheduler import TimelineEntry, _entry, build_timeline, Policy, project_cursor


def test_cached_populate_ready_is_bit_identical():
    rng = random.Random(3)
    for name in ("rtx5080", "b200"):
        try:
            hw = get_preset(name)
        except (KeyError, ValueError):
            continue
        sim = types.SimpleNamespace(_cost_e=engine.evict_page_cost_s(hw), _cost_p=engine.populate_page_cost_s(hw))
        for _ in range(20000):
            j, free, nev = rng.randint(-2, 50000), rng.randint(-100, 50000), rng.randint(0, 50000)
            want = engine.populate_ready(hw, j, free, nev)
            got = engine.Simulator._populate_ready(sim, j, free, nev)
            assert got == want and type(got) is type(want), (name, j, free, nev)


def test_fast_timeline_entries_equal_constructed_ones():
    e = _entry("t3", 0.005, 41)
    f = TimelineEntry("t3", 0.005, 41)
    assert e == f and hash(e) == hash(f) and repr(e) == repr(f) and type(e) is TimelineEntry
    tasks = []
    for i, n in enumerate((5, 9, 3)):
        t = types.SimpleNamespace(id=f"t{i}", cursor=0, priority=0, commands=[None] * n)
        t.remaining = (lambda t=t: len(t.commands) - t.cursor)
        tasks.append(t)
    lat = {t.id: [1e-3 * (k + 1) for k in range(len(t.commands))] for t in tasks}
    tl = build_timeline(Policy("rr", 2e-3, 2), tasks, latencies=lat)
    # the same timeline built entry by entry with the public constructor
    pos, want, k = {t.id: 0 for t in tasks}, [], 0
    rr = list(tasks)
    while len(want) < 6 and rr:
        t = rr[k % len(rr)]
        if pos[t.id] >= len(lat[t.id]):
            rr = [x for x in rr if pos[x.id] < len(lat[x.id])]
            k = 0
            continue
        want.append(TimelineEntry(t.id, 2e-3, pos[t.id]))
        pos[t.id] = project_cursor(lat[t.id], pos[t.id], 2e-3)
        k += 1
    assert list(tl) == want
