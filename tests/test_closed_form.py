"""DESIGN.md section 3's claim, on the CPU: the reference's reorder
(windows last to first, each window's first-access runs last to first, one
madvise per run -- memman.py:218-241 over EvictionList.madvise, 58-91) equals
ONE stable sort of the list by the tuple (class in window 0, ..., class in
window W-1), class = K_w - r for the r-th run of window w, 0 if absent.  The
GPU multisplit implements the sort; this pins the equivalence against the
oracle's run-list madvise on random instances."""

import random

import numpy as np

from oracle import msched_port as port


def closed_form(order, wins):
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
    idx = np.lexsort(tuple(reversed(keys))) if keys else np.arange(len(order))
    return order[idx].tolist()


def test_reorder_is_one_stable_sort_by_class_tuple():
    rng = random.Random(3)
    for _ in range(150):
        pages = rng.sample(range(3000), rng.randint(1, 600))
        runs = port.norm_runs([(p, p + 1) for p in pages])
        order = list(runs)
        rng.shuffle(order)
        rl = port.RunList()
        rl.append(order)
        cur = [p for a, b in order for p in range(a, b)]
        for _ in range(2):
            wins = []
            for _ in range(rng.randint(1, 6)):
                seen, wr = (), []
                for _ in range(rng.randint(1, 12)):
                    a = rng.randrange(0, 3000)
                    new = port.runs_sub(((a, a + rng.randint(1, 200)),), seen)
                    wr.extend(new)
                    seen = port.runs_or(seen, new)
                wins.append(wr)
            port.opt_reorder(rl, [port.Win("t", w, w, (), 0, 0) for w in wins])
            cur = closed_form(cur, wins)
            assert cur == rl.order()


def test_sentinel_matters():
    """omitting the 'absent' class 0 breaks the order
    ([13, 8, 17] example): pages advised in window 1 only must sort by their
    window-1 class, after pages never advised."""
    rl = port.RunList()
    rl.append([(13, 14), (8, 9), (17, 18)])
    wins = [[(17, 18)], [(8, 9), (13, 14)]]
    port.opt_reorder(rl, [port.Win("t", w, w, (), 0, 0) for w in wins])
    assert rl.order() == closed_form([13, 8, 17], wins)
