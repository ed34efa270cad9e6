"""Executed commands with early-start gating (
engine.py:139-158, 342-361, 373-378 made real): every command of every slice
runs on the device as a kernel that reads its pages from their HBM frames,
started by a stream wait on the populate progress of its switch.  The model
(Metrics, events) must not change, every page a command reads must be
resident and hold its own payload, and every executed command must run."""

import dataclasses

import pytest

from oracle import msched_port as port
from paper_2512_24637_b200 import engine
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scenarios import llm_scenario, streaming_scenario

pytestmark = pytest.mark.gpu

HW = get_preset("rtx5080").with_capacity(96 << 20)


def _actual_pages(sim, tasks):
    return sum(len(sim.actual_pages(t.id, c)) for t in tasks for c in range(len(t.commands)))


@pytest.mark.parametrize("early", [True, False], ids=["early_start", "whole_batch"])
@pytest.mark.parametrize("case", ["llm", "streaming_faults"])
def test_executed_commands_read_their_migrated_pages(case, early):
    if case == "llm":
        tasks, pol = llm_scenario(HW, 2.0, n_tasks=3, layers=6, decode_steps=4)
    else:
        tasks, pol = streaming_scenario(HW, 2.0, indirect_rate=0.01, seed=1)
    mode = engine.Mode.proactive(early_start=early)
    sim = engine.Simulator(tasks, HW, pol, mode, record_events=True, migrate=True, verify=True, execute=True)
    try:
        m = sim.run()
        st = sim.ctx.stats()
        n_cmds = sum(len(t.commands) for t in tasks)
        assert st["run_cmds"] == n_cmds
        missing = st["run_missing"]
        assert st["run_bad_tags"] == 0, "an executed command read a frame holding another page's payload"
        assert st["run_pages"] + st["run_missing"] == _actual_pages(sim, tasks)
        assert sim.ctx.verify() == 0
        events = [(e.t, e.kind, e.task_id, e.pages) for e in sim.events]
    finally:
        sim.close()
    rec = []
    ref = port.PortSim(tasks, HW, pol, mode, record_events=True, recorder=rec)
    mr = ref.run()
    got = dataclasses.asdict(m)
    got.pop("normalized_throughput")
    assert got == mr.as_dict()
    assert events == ref.events
    # The only pages an executed command may find non-resident are its own
    # pages that its own fault-path eviction removed: the reference evicts
    # from the list head without re-checking the faulting command
    # (engine.py:408-413).  Count them on the oracle.
    own = 0
    for r in rec:
        if r.get("ev") == "touch" and r.get("evicted"):
            t = ref.by_id[r["task"]]
            act = {p for a, b in t.actual[r["cmd"]] for p in range(a, b)}
            own += len(act & set(r["evicted"]))
    assert missing == own
    if case == "llm":
        assert own == 0


def test_execute_needs_migration():
    tasks, pol = llm_scenario(HW, 2.0, n_tasks=2, layers=2, decode_steps=1)
    with pytest.raises(ValueError):
        engine.Simulator(tasks, HW, pol, engine.Mode.proactive(), execute=True)
