"""Find the first executed command that reads a wrong payload (GPU box)."""
import sys

sys.path.insert(0, ".")
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.presets import get_preset  # noqa: E402
from paper_2512_24637_b200.scenarios import streaming_scenario  # noqa: E402

HW = get_preset("rtx5080").with_capacity(96 << 20)
tasks, pol = streaming_scenario(HW, 2.0, indirect_rate=0.01, seed=1)
sync_each = "--sync" in sys.argv
sim = engine.Simulator(tasks, HW, pol, engine.Mode.proactive(), migrate=True, verify=True, execute=True)
orig = sim.ctx.run_command
log = []


def rc(idx, cmd, need):
    st0 = sim.ctx.stats() if sync_each else None
    orig(idx, cmd, need)
    if sync_each:
        st1 = sim.ctx.stats()
        if st1["run_bad_tags"] != st0["run_bad_tags"]:
            t = sim.tasks[idx]
            log.append((t.id, cmd, str(t.commands[cmd].kind), need, st1["run_bad_tags"] - st0["run_bad_tags"]))


sim.ctx.run_command = rc
sim.run()
st = sim.ctx.stats()
print("bad", st["run_bad_tags"], "missing", st["run_missing"], "cmds", st["run_cmds"], "verify", sim.ctx.verify())
for x in log[:20]:
    print(x)
