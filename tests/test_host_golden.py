"""Host-side inputs pinned to the reference (CPU only): trace generators,
the MSIM-TRACE v1 format, the offline analyzer, the scheduler timeline, the
run-length PageSet and the FP64 timing model.  The reference's own tests are
the model (test_core.py, test_workload.py, test_analyzer.py,
test_scheduler.py, test_engine.py pipeline algebra)."""

import dataclasses
import struct
from fractions import Fraction

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2512_24637_b200 import analyzer, engine, scenarios, workload
from paper_2512_24637_b200.model import Arg, ByteRange, Command, CommandKind, PageSet, Task, pages_of
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scheduler import Policy, build_timeline, runnable_order
from tests.golden import loader

PAGE = 4096


# -- generators and trace text: byte-identical to the reference's output -------

def _struct_task(i):
    return next(c for c in loader.sims() if c["name"] == "struct")["tasks"][i]


def test_generators_match_reference_traces():
    tr = loader.traces()
    assert workload.format_trace(workload.gen_vector_add(2048, iterations=2, task_id="va", indirect_rate=0.01,
                                                         seed=5)) == tr["va"]
    assert workload.format_trace(workload.gen_matmul(128, 256, 64, count=2, flops=1e12)) == tr["mm"]
    assert workload.format_trace(workload.gen_llm_like(3, 4 * PAGE, 2 * PAGE, 2, [0.5, 1.0])) == tr["llm"]
    assert workload.format_trace(workload.gen_template_corpus(n_kernels=12, records_per=3, seed=1).task) == \
        tr["corpus"]
    assert workload.format_trace(scenarios.config2_llama8b()[0][0]) == tr["cfg2_task0"]
    assert workload.format_trace(scenarios.config1_gemm()[0][1]) == tr["cfg1_task1"]


def test_trace_round_trip_is_a_fixpoint():
    for text in loader.traces().values():
        assert workload.format_trace(workload.parse_trace(text)) == text


def test_trace_errors_carry_location():
    with pytest.raises(workload.TraceError, match="<t>:1"):
        workload.parse_trace("bogus header", source="<t>")
    with pytest.raises(workload.TraceError, match="<t>:3"):
        workload.parse_trace("MSIM-TRACE v1\nTASK id=x\nKERNEL nope\n", source="<t>")


def test_scenarios_match_golden_inputs():
    hw = get_preset("rtx5080").with_capacity(96 << 20)
    for case in loader.sims():
        g = case.get("gen")
        if not g or g["fn"] not in ("streaming_scenario", "llm_scenario", "uniform_scenario", "cfg1", "cfg2",
                                    "cfg4", "config3_mixed"):
            continue
        if g["fn"] == "streaming_scenario":
            tasks, _ = scenarios.streaming_scenario(hw, g["ratio"], indirect_rate=g.get("indirect_rate", 0.0),
                                                    seed=g.get("seed", 0))
        elif g["fn"] == "llm_scenario":
            tasks, _ = scenarios.llm_scenario(hw, g["ratio"])
        elif g["fn"] == "uniform_scenario":
            tasks, _ = scenarios.uniform_scenario(get_preset("rtx5080").with_capacity(16 << 20), g["n_tasks"],
                                                  g["footprint"])
        elif g["fn"] == "config3_mixed":
            from paper_2512_24637_b200.workload_extra import config3_mixed

            tasks = config3_mixed(ratio=g["ratio"], timeslice_s=g["timeslice_s"])[0]
        elif g["fn"] == "cfg2" and "page" in g:
            tasks = scenarios.config2_llama8b(page=g["page"])[0]
        else:
            tasks = {"cfg1": scenarios.config1_gemm, "cfg2": scenarios.config2_llama8b,
                     "cfg4": scenarios.config4_llama70b}[g["fn"]]()[0]
        want = [loader.dec_task(t) for t in case["tasks"]]
        assert [workload.format_trace(t) for t in tasks] == [workload.format_trace(t) for t in want], case["name"]


# -- offline analyzer: identical descriptor files -----------------------------

def test_analyzer_matches_reference_descriptors():
    for case in loader.predictions():
        task = loader.dec_task(case["task"])
        assert analyzer.format_descriptors(analyzer.build_descriptors(task)) == case["descriptors"], case["name"]


def test_analyzer_known_answers():
    base = 1 << 40

    def rec(args, regions, grid=(1, 1, 1)):
        return analyzer.InvocationRecord("k", tuple(args), grid, (1, 1, 1), analyzer.coalesce_regions(regions))

    r = analyzer.infer_rule([rec([Arg(base), Arg(6, 32)], [ByteRange(base, 9)]),
                             rec([Arg(base), Arg(10, 32)], [ByteRange(base, 15)])], 0)
    assert r.kind == "linear" and r.size.coeff == Fraction(3, 2) and r.size.slots == ("a1",)  # test_analyzer.py:73-81
    r = analyzer.infer_rule([rec([Arg(base)], [ByteRange(base, 2560)], (10, 1, 1)),
                             rec([Arg(base)], [ByteRange(base, 3584)], (14, 1, 1))], 0)
    assert r.size.slots == ("gx",) and r.size.coeff == 256                                   # :96-104
    raw = struct.pack("<QI", 0xAABBCCDD11223344, 77)
    sl = analyzer.slice_struct_args(raw)
    assert (0, 64, 0xAABBCCDD11223344) in sl and (8, 32, 77) in sl and (0, 32, 0x11223344) in sl
    d = analyzer.build_descriptor("k", [rec([Arg(base - 64), Arg(2, 32)], [ByteRange(base, 200)]),
                                        rec([Arg(base + PAGE - 64), Arg(3, 32)], [ByteRange(base + PAGE, 200)])])
    assert len(d.rules) == 1 and d.rules[0].offset_bytes == 64 and d.rules[0].kind == "fixed"  # :46-54
    with pytest.raises(ValueError):
        analyzer.build_descriptor("k", [])


def test_descriptor_file_round_trip(tmp_path):
    descs = analyzer.build_descriptors(workload.gen_template_corpus(n_kernels=9, seed=3).task)
    p = tmp_path / "d.msdesc"
    analyzer.save_descriptors(descs, str(p))
    assert analyzer.format_descriptors(analyzer.load_descriptors(str(p))) == analyzer.format_descriptors(descs)
    with pytest.raises(analyzer.DescriptorError):
        analyzer.load_descriptors("/dev/null")


# -- scheduler timeline (test_scheduler.py:22-60) ----------------------------------

def _task(tid, n, lat=1e-3, prio=0, cursor=0):
    return Task(id=tid, commands=[Command(CommandKind.KERNEL, lat, "k") for _ in range(n)], priority=prio,
                cursor=cursor)


def test_timeline_known_answers():
    tl = build_timeline(Policy(timeslice_s=5e-3, horizon_rounds=2), [_task("a", 100), _task("b", 100), _task("c", 100)])
    assert [e.task_id for e in tl] == ["a", "b", "c", "a", "b", "c"]
    assert [e.resume_command_cursor for e in build_timeline(Policy(timeslice_s=5e-3), [_task("a", 100)], 3)] == [0, 5, 10]
    assert build_timeline(Policy(timeslice_s=5e-3), [_task("a", 100, 2e-3)], 2)[1].resume_command_cursor == 3
    assert [e.task_id for e in build_timeline(Policy(timeslice_s=5e-3), [_task("a", 2), _task("b", 100)], 4)] == \
        ["a", "b", "b", "b"]
    assert [t.id for t in runnable_order(Policy(kind="priority"), [_task("lo", 10, prio=0),
                                                                   _task("hi", 10, prio=5)])] == ["hi"]
    assert build_timeline(Policy(), []) == ()
    with pytest.raises(ValueError):
        Policy(timeslice_s=0.0)


# -- PageSet against a plain set (test_core.py:33-51) -------------------------------

runs_st = st.lists(st.tuples(st.integers(0, 300), st.integers(0, 60)).map(lambda t: (t[0], t[0] + t[1])), max_size=8)


@settings(max_examples=200, deadline=None)
@given(runs_st, runs_st)
def test_pageset_algebra(a_runs, b_runs):
    a, b = PageSet(a_runs), PageSet(b_runs)
    sa, sb = set(a), set(b)
    assert set(a | b) == sa | sb and set(a & b) == sa & sb and set(a - b) == sa - sb and len(a) == len(sa)
    for (s0, e0), (s1, _) in zip((a - b).runs, (a - b).runs[1:]):
        assert e0 < s1


def test_pages_of_boundaries():
    assert list(pages_of(ByteRange(4095, 2), PAGE)) == [0, 1]           # test_core.py:67-69
    assert list(pages_of(ByteRange(PAGE, PAGE), PAGE)) == [1]


# -- FP64 timing model (test_engine.py:107-141) -----------------------------------

def test_pipeline_algebra():
    hw = dataclasses.replace(get_preset("rtx5080"), bw_d2h_bytes_per_s=1e9, bw_h2d_bytes_per_s=1e9)
    for n in (1, 10, 1000):
        assert engine.pipeline_time(hw, n, n, 0) == pytest.approx((n + 1) * PAGE / 1e9, rel=1e-12)
    base = get_preset("rtx5080")
    for ne, npop, free in [(5, 5, 0), (100, 40, 10), (3, 90, 0), (0, 12, 12)]:
        assert base and engine.pipeline_time(base, ne, npop, free) <= engine.sequential_time(base, ne, npop) + 1e-15
    prev = 0.0
    for j in range(1, 50):
        cur = engine.populate_ready(base, j, 4, 30)
        assert cur >= prev - 1e-15
        prev = cur


def test_um_duration_rounds_batches_up():
    hw = get_preset("rtx5080")
    cmd = Command(CommandKind.KERNEL, 1e-3, "k")
    assert engine.um_command_duration(hw, cmd, 17, 16) == pytest.approx(
        1e-3 + 2 * (hw.fault_control_plane_s + 16 * hw.fault_transfer_s))


# -- the host event loop, memory-free reference mode (no GPU needed) -------------

@pytest.mark.parametrize("name", [c["name"] for c in loader.sims() if "reference" in c["runs"]])
def test_reference_mode_loop_matches(name):
    case = loader.sim_case(name)
    want = case["runs"]["reference"]
    from paper_2512_24637_b200.model import HwConfig

    tasks = [loader.dec_task(t) for t in case["tasks"]]
    sim = engine.Simulator(tasks, HwConfig(**case["hw"]), Policy(**case["policy"]), engine.Mode.reference(),
                           record_events=True)
    got = dataclasses.asdict(sim.run())
    got.pop("normalized_throughput")
    assert got == want["metrics"]
    assert [[e.t, e.kind, e.task_id, e.pages] for e in sim.events] == want["events"]


def test_simulator_input_guards():
    hw = get_preset("rtx5080").with_capacity(96 << 20)
    t = workload.gen_vector_add(1024, task_id="same")
    with pytest.raises(engine.SimulationError):
        engine.Simulator([t, workload.gen_vector_add(1024, task_id="same", base_addr=1 << 41)], hw, Policy(),
                         engine.Mode.reference())
    with pytest.raises(engine.SimulationError, match="DRAM"):
        engine.Simulator([t], dataclasses.replace(hw, dram_capacity_bytes=PAGE), Policy(), engine.Mode.reference())


def test_acceptance_criterion_3_fault_bandwidth():
    """test_acceptance.py:222-232: a demand fault moves a page at ~0.12 GB/s,
    bulk seed copies run at the configured 41.7 GB/s link exactly."""
    from paper_2512_24637_b200.model import CommandKind
    from paper_2512_24637_b200.presets import get_preset
    from paper_2512_24637_b200.workload import DEFAULT_H2D_BW, gen_vector_add

    hw = get_preset("rtx5080").with_capacity(96 << 20)
    stall = hw.fault_control_plane_s + hw.fault_transfer_s
    assert stall == pytest.approx(33.14e-6)
    assert 4096 / stall == pytest.approx(0.12e9, rel=0.05)
    task = gen_vector_add(1 << 20, task_id="t")
    for cmd in task.commands:
        if cmd.kind is CommandKind.MEMCPY_H2D:
            assert cmd.latency_s == cmd.memcpy_size / DEFAULT_H2D_BW
    assert DEFAULT_H2D_BW == 41.7e9
