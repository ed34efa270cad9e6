"""Pin the CPU oracle (oracle/msched_port.py) to the real reference.

Every simulation in tests/golden/sims.json.gz was produced by the reference
simulator (tests/golden/make_golden.py); the oracle must reproduce metrics,
events and every per-switch planner record exactly (floats compared with ==).
"""

import pytest

from oracle import msched_port as port
from tests.golden import loader

CASES = [(c["name"], m) for c in loader.sims() for m in c["runs"]]
SLOW = {"cfg1", "cfg2", "cfg4", "cfg5_16k", "cfg5_64k"}
# big cases: the golden generator sampled the full list order every k-th
# reorder; the port skips orders there (its run-list order dump is O(pages))
ORDER_EVERY = {"cfg4": 0, "cfg2": 0, "cfg5_16k": 0, "cfg5_64k": 0}


def run_port(case, mode_name):
    tasks = [loader.dec_task(t) for t in case["tasks"]]
    tasks, feeder = loader.feeder_for(case["feeder"], tasks)
    run = case["runs"][mode_name]
    rec = []
    sim = port.PortSim(tasks, loader.ns(case["hw"]), loader.ns(case["policy"]),
                       loader.ns(run["mode"]), feeder=feeder, record_events=True, recorder=rec,
                       order_every=ORDER_EVERY.get(case["name"], 1), pack=loader.digest)
    m = sim.run()
    return m, sim, rec


@pytest.mark.parametrize("name,mode", [
    pytest.param(n, m, marks=[pytest.mark.slow] if n in SLOW else []) for n, m in CASES])
def test_oracle_matches_reference(name, mode):
    case = loader.sim_case(name)
    want = case["runs"][mode]
    if "error" in want:
        with pytest.raises(Exception) as ei:
            run_port(case, mode)
        assert type(ei.value).__name__ == want["error"]
        assert str(ei.value) == want["message"]
        return
    m, sim, rec = run_port(case, mode)
    assert m.as_dict() == want["metrics"]
    assert [list(e) for e in sim.events] == want["events"]
    want_rec = loader.canon_records(want["records"])
    if ORDER_EVERY.get(name, 1) == 0:
        want_rec = loader.strip_orders(want_rec)
    got_rec = loader.strip_orders(loader.canon_records(rec)) if ORDER_EVERY.get(name, 1) == 0 \
        else loader.canon_records(rec)
    assert loader.align_sampled(got_rec, want_rec) == want_rec


def test_predictions_match_reference():
    for case in loader.predictions():
        task = loader.dec_task(case["task"])
        descs = port.infer_descriptors(task)
        assert port.descriptors_text(descs) == case["descriptors"], case["name"]
        for cmd, row in zip(task.commands, case["rows"]):
            runs, complete = port.predict_template(descs, cmd, 4096)
            assert [list(r) for r in runs] == row["template"]
            assert complete == row["complete"]
            assert [list(r) for r in port.predict_alloc(task.allocations, cmd, 4096)[0]] == row["allocation"]
            assert [list(r) for r in port.predict_truth(cmd, 4096)] == row["truth"]


# known answers quoted by the reference's own tests ------------------------------

def _rl(pages):
    rl = port.RunList()
    for p in pages:
        rl.append([(p, p + 1)])
    return rl


def test_known_answers_eviction_list():
    rl = _rl([10, 20, 30, 40])                       # test_memman.py:29-34
    rl.advise(port.norm_runs([(40, 41), (20, 21)]))
    assert rl.order() == [10, 30, 20, 40]
    rl = _rl([1, 2, 3])                              # test_memman.py:37-40
    rl.advise(port.norm_runs([(99, 100), (2, 3)]))
    assert rl.order() == [1, 3, 2]
    rl = _rl([5, 6, 7, 1, 2])                        # test_memman.py:62-68
    assert port.runs_pages(rl.pop_head(3)) == [5, 6, 7]
    assert rl.order() == [1, 2]
    rl = _rl([1, 2, 3, 4, 5])                        # test_memman.py:71-75
    rl.drop(port.norm_runs([(2, 3), (4, 5)]))
    assert rl.order() == [1, 3, 5] and len(rl) == 3


def test_known_answers_plans_and_belady():
    assert port.belady([1, 2, 3, 4, 1, 2, 5, 1, 2, 3, 4, 5], 3)[0] == 7   # test_memman.py:80-82
    assert port.belady([1, 2, 3, 1, 3, 1], 2) == (3, [(2, 2)])           # test_memman.py:91-95
    rl = _rl([0, 1, 2])                                                  # test_memman.py:118-123
    plan = port.make_plan(rl, [(0, 5)], 8)
    assert plan.populate == [(3, 5)] and plan.evict == [] and plan.truncated == 0
    rl = _rl([10, 11, 12, 13])                                           # test_memman.py:126-134
    plan = port.make_plan(rl, [(20, 23)], 4)
    assert port.runs_pages(plan.evict) == [10, 11, 12]
    port.apply_plan_runs(rl, plan)
    assert rl.order() == [13, 20, 21, 22]
    plan = port.make_plan(port.RunList(), [(0, 10)], 4)                  # test_memman.py:137-141
    assert plan.n_populate == 4 and plan.truncated == 6


def test_known_answers_windows_and_reorder():
    preds = [((p, p + 1),) for p in [3, 1, 3, 2]]                        # test_memman.py:165-169
    w = port.window_of("t", preds, [], [1e-6] * 4, 0, 1.0)
    assert [a for a, _ in w.ordered] == [3, 1, 2] and w.end == 4
    w = port.window_of("t", preds[:1] + preds[1:2] + [((2, 3),)], [], [1e-6] * 3, 0, 1.5e-6)
    assert w.end == 2
    rl = _rl([0, 1, 2])                                                  # test_memman.py:179-187
    w = port.window_of("t", [((2, 3),), ((0, 1),), ((1, 2),)], [], [1e-6] * 3, 0, 1.0)
    port.opt_reorder(rl, [w])
    assert rl.order() == [1, 0, 2]


def test_known_answers_pipeline_algebra():
    hw = loader.ns(dict(page_size_bytes=4096, bw_d2h_bytes_per_s=1e9, bw_h2d_bytes_per_s=1e9,
                        per_page_unmap_s=0.0, per_page_map_s=0.0))
    t = 4096 / 1e9
    for n in (1, 10, 1000):                                              # test_engine.py:112-119
        assert port.pipe_swap_time(hw, n, n, 0) == pytest.approx((n + 1) * t, rel=1e-12)
