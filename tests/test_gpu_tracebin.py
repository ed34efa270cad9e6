"""A replay from a binary trace (columns straight to msg_add_commands) equals
the CPU oracle on the original task objects."""

import dataclasses

import pytest

from oracle import msched_port as port
from paper_2512_24637_b200 import engine, tracebin
from paper_2512_24637_b200.analyzer import build_descriptors
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scenarios import llm_scenario, streaming_scenario

pytestmark = pytest.mark.gpu
HW = get_preset("rtx5080").with_capacity(96 << 20)


@pytest.mark.parametrize("case", ["llm", "streaming"])
@pytest.mark.parametrize("mode", ["proactive", "allocation", "ideal", "um"])
def test_binary_trace_replay_matches_oracle(tmp_path, case, mode):
    if case == "llm":
        tasks, pol = llm_scenario(HW, 2.0, n_tasks=3, layers=6, decode_steps=4)
    else:
        tasks, pol = streaming_scenario(HW, 2.0, indirect_rate=0.01, seed=1)
    m_ = {"proactive": engine.Mode.proactive(), "allocation": engine.Mode.proactive(predictor="allocation"),
          "ideal": engine.Mode.ideal(), "um": engine.Mode.um()}[mode]
    p = tmp_path / "trace.msimb"
    tracebin.save_trace_bin(tasks, str(p))
    cols = tracebin.load_trace_bin(str(p))
    descs = {t.id: build_descriptors(t) for t in tasks}
    sim = engine.Simulator(cols, HW, pol, m_, record_events=True, descriptors=descs)
    try:
        m = sim.run()
        events = [(e.t, e.kind, e.task_id, e.pages) for e in sim.events]
    finally:
        sim.close()
    ref = port.PortSim(tasks, HW, pol, m_, record_events=True)
    mr = ref.run()
    got = dataclasses.asdict(m)
    got.pop("normalized_throughput")
    assert got == mr.as_dict()
    assert events == ref.events
