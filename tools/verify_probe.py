import sys
sys.path.insert(0, ".")
from paper_2512_24637_b200 import engine
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scenarios import streaming_scenario, llm_scenario
HW = get_preset("rtx5080").with_capacity(96 << 20)
for name, (tasks, pol) in [("stream", streaming_scenario(HW, 2.0, indirect_rate=0.01, seed=1)), ("llm", llm_scenario(HW, 2.0, n_tasks=3, layers=6, decode_steps=4))]:
    for ex in (False, True):
        sim = engine.Simulator(tasks, HW, pol, engine.Mode.proactive(), migrate=True, verify=True, execute=ex)
        sim.run()
        print(name, "execute", ex, "bad", sim.ctx.verify(), sim.ctx.stats()["run_bad_tags"])
        sim.close()
