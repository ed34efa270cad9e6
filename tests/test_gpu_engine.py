"""Simulator behaviour through the B200 engine, restating the reference's
engine tests (pkg/tests/test_engine.py): construction guards, mode
dominance, migration-timing orderings, page conservation, determinism,
arrivals, live feeding and the residency guard.  The closed-form timing
helpers (test_engine.py:76-145) are host code and run in
test_host_golden.py."""

import dataclasses

import pytest

from paper_2512_24637_b200.engine import Mode, SimulationError, Simulator, simulate, simulate_normalized
from paper_2512_24637_b200.model import Allocation, Arg, ByteRange, Command, CommandKind, Task
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scenarios import llm_scenario, streaming_scenario
from paper_2512_24637_b200.scheduler import Policy
from paper_2512_24637_b200.workload import gen_vector_add

pytestmark = pytest.mark.gpu

PAGE = 4096
HW = get_preset("rtx5080").with_capacity(96 << 20)
POLICY = Policy(kind="rr", timeslice_s=1.75e-3)


def small_task(task_id="t", pages=8, base=1 << 40, iterations=2):
    return gen_vector_add(pages * PAGE // 12, iterations=iterations, task_id=task_id, base_addr=base)


def test_zero_tasks_zero_metrics():                       # test_engine.py:47-51
    m = simulate([], HW, POLICY, Mode.um())
    assert (m.total_time_s, m.context_switches, m.completed_tasks) == (0.0, 0, 0)


def test_construction_guards():                           # :54-63
    with pytest.raises(SimulationError):
        Simulator([small_task("same"), small_task("same", base=1 << 41)], HW, POLICY, Mode.um())
    with pytest.raises(SimulationError, match="DRAM"):
        Simulator([small_task()], dataclasses.replace(HW, dram_capacity_bytes=PAGE), POLICY, Mode.um())


def test_input_tasks_not_mutated():                       # :66-70
    task = small_task()
    before = (task.cursor, len(task.commands))
    simulate([task], HW, POLICY, Mode.proactive())
    assert (task.cursor, len(task.commands)) == before


def test_underscribed_and_fitting_runs_have_no_faults():  # :147-158
    tasks, pol = streaming_scenario(HW, 1.0)
    m = simulate_normalized(tasks, HW, pol, Mode.proactive())
    assert m.normalized_throughput == pytest.approx(1.0, abs=1e-9)
    assert m.fault_pages == 0
    tasks, pol = streaming_scenario(HW, 0.8)
    for mode in (Mode.um(), Mode.proactive(), Mode.ideal()):
        assert simulate(tasks, HW, pol, mode).fault_pages == 0, mode.name


def test_mode_dominance_and_timing_orderings():           # :161-191
    tasks, pol = streaming_scenario(HW, 2.0)
    modes = {"um": Mode.um(), "alloc": dataclasses.replace(Mode.proactive(), predictor="allocation"),
             "pro": Mode.proactive(), "ideal": Mode.ideal()}
    r = {k: simulate_normalized(tasks, HW, pol, m).normalized_throughput for k, m in modes.items()}
    assert r["ideal"] >= r["pro"] - 1e-9
    assert r["pro"] > r["um"]
    assert r["ideal"] >= r["alloc"] - 1e-9
    pipe = simulate(tasks, HW, pol, Mode.proactive())
    seq = simulate(tasks, HW, pol, dataclasses.replace(Mode.proactive(), pipelined=False))
    late = simulate(tasks, HW, pol, dataclasses.replace(Mode.proactive(), early_start=False))
    assert seq.total_time_s >= pipe.total_time_s - 1e-12
    assert late.total_time_s >= pipe.total_time_s - 1e-12


def test_page_conservation_and_completions():             # :194-212
    tasks, pol = streaming_scenario(HW, 2.0)
    for mode in (Mode.um(), Mode.proactive(), Mode.ideal()):
        m = simulate(tasks, HW, pol, mode)
        assert m.h2d_migration_pages == m.migrated_in_pages + m.fault_pages
        assert m.migrated_bytes_h2d == m.h2d_migration_pages * m.page_size_bytes
        assert m.migrated_bytes_d2h == (m.migrated_out_pages + m.evicted_capacity_pages) * m.page_size_bytes
        assert set(m.completion_s) == {t.id for t in tasks}
        assert m.completed_tasks == len(tasks)
        assert all(0 < v <= m.total_time_s + 1e-12 for v in m.completion_s.values())


def test_repeat_runs_identical():                         # :215-219
    tasks, pol = streaming_scenario(HW, 2.0, seed=3)
    assert simulate(tasks, HW, pol, Mode.proactive()) == simulate(tasks, HW, pol, Mode.proactive())


def test_reset_replays_identically():
    """One context replayed twice (reset re-uploads nothing, restores the
    residency state) gives the same metrics as two fresh contexts."""
    tasks, pol = streaming_scenario(HW, 2.0, seed=3)
    sim = Simulator(tasks, HW, pol, Mode.proactive())
    try:
        a = sim.run()
        sim.reset()
        b = sim.run()
    finally:
        sim.close()
    assert a == b == simulate(tasks, HW, pol, Mode.proactive())


def test_late_arrival_gates_start():                      # :225-232
    t1, t2 = small_task("a", base=1 << 40), small_task("b", base=1 << 41)
    t2.arrival_s = 1.0
    m = simulate([t1, t2], HW, POLICY, Mode.proactive())
    assert m.completion_s["a"] < 1.0 <= m.completion_s["b"]


def _llm_pair():
    return llm_scenario(HW, 1.5, n_tasks=2, layers=6, decode_steps=6)


def test_append_after_completion_rejected():              # :243-248
    task = small_task()
    sim = Simulator([task], HW, POLICY, Mode.proactive())
    try:
        sim.run()
        with pytest.raises(SimulationError, match="completed"):
            sim.append_commands(task.id, [task.commands[-1]])
    finally:
        sim.close()


def test_append_empty_is_noop():                          # :251-260
    tasks, pol = _llm_pair()
    base = simulate(tasks, HW, pol, Mode.proactive())

    def feeder(sim):
        if sim.by_id[tasks[0].id].remaining() > 0:
            sim.append_commands(tasks[0].id, [])

    assert simulate(tasks, HW, pol, Mode.proactive(), feeder=feeder) == base


def test_incremental_feeding_matches_upfront_submission():   # :263-292
    tasks, pol = _llm_pair()
    upfront = simulate(tasks, HW, pol, Mode.proactive())
    split = len(tasks[0].commands) // 2
    head = Task(id=tasks[0].id, allocations=list(tasks[0].allocations), commands=list(tasks[0].commands[:split]),
                priority=tasks[0].priority, arrival_s=tasks[0].arrival_s)
    tail = tasks[0].commands[split:]
    state = {"fed": False}

    def feeder(sim):
        if not state["fed"] and sim.by_id[head.id].remaining() <= 2:
            sim.append_commands(head.id, tail)
            state["fed"] = True

    fed = simulate([head, tasks[1]], HW, pol, Mode.proactive(), feeder=feeder)
    assert state["fed"]
    assert fed.completed_tasks == upfront.completed_tasks
    assert fed.total_time_s == pytest.approx(upfront.total_time_s, rel=0.10)


@pytest.mark.parametrize("mode", ["um", "proactive", "ideal"])
def test_single_command_over_capacity_raises(mode):        # :295-316
    base, size = 1 << 40, 16 * PAGE
    task = Task(id="big", allocations=[Allocation("a0", base, size, "big")],
                commands=[Command(kind=CommandKind.KERNEL, latency_s=1e-4, kernel_name="touch_all",
                                  launch_args=(Arg(base),), ground_truth_access=(ByteRange(base, size),))])
    with pytest.raises(SimulationError):
        simulate([task], HW.with_capacity(4 * PAGE), POLICY, getattr(Mode, mode)())


@pytest.mark.parametrize("name", ["llm_2.0", "stream_ind", "frag", "cfg3_2.0", "edge_capacity_plus_one"])
def test_async_switch_path_equals_synchronous_path(name):
    """Plain replays run the plan's apply on the device without a host round
    trip (the multisplit decides its pass count, the apply kernels their counts);
    a recorder forces the synchronous path.  Both must leave the same metrics,
    events and final eviction order."""
    from paper_2512_24637_b200.model import HwConfig
    from tests.golden import loader

    case = loader.sim_case(name)
    for mode_name, want in case["runs"].items():
        if "error" in want:
            continue
        out = []
        for rec in (None, []):
            tasks = [loader.dec_task(t) for t in case["tasks"]]
            sim = Simulator(tasks, HwConfig(**case["hw"]), Policy(**case["policy"]), Mode(**want["mode"]),
                            record_events=True, recorder=rec)
            try:
                m = sim.run()
                out.append((dataclasses.asdict(m), [(e.t, e.kind, e.task_id, e.pages) for e in sim.events],
                            sim.eviction_order()))
            finally:
                sim.close()
        assert out[0] == out[1], (name, mode_name)
