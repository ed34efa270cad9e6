"""The plugin claim, tested against the real reference: the reference's own
`msim.engine.Simulator` with its hot-path methods routed through
libmsched_b200.so (`msim_plugin.b200_simulator_class`, the binding of
INTEGRATION.md §2) must give the same `Metrics` (floats with ==), the same
events and the same errors as the unpatched reference, on the reference's
own engine loop, for every golden case and mode.

Needs the reference importable: `baseline/_ref` (installed by
`pip install --target baseline/_ref`, git-ignored, travels to the GPU box) or
`/root/reference/pkg/src` in the build container.  Skipped otherwise."""

import dataclasses
import os
import sys

import pytest

from paper_2512_24637_b200.msim_plugin import b200_simulator_class, to_msim_tasks
from tests.golden import loader

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _msim():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "msim")):
            if p not in sys.path:
                sys.path.insert(0, p)
            import msim.core as mc
            import msim.engine as E
            import msim.scheduler as S

            return mc, E, S
    return None


MSIM = _msim()
SLOW = {"cfg1", "cfg2", "cfg4", "cfg5_16k", "cfg5_64k", "cfg3_2.0", "cfg3_3.0"}
CASES = [(c["name"], m) for c in loader.sims() for m in c["runs"] if not c.get("feeder")]


def _inputs(case, mode_name):
    mc, E, S = MSIM
    tasks = to_msim_tasks(mc, [loader.dec_task(t) for t in case["tasks"]])
    hw = mc.HwConfig(**case["hw"])
    pol = S.Policy(**case["policy"])
    mode = E.Mode(**case["runs"][mode_name]["mode"])
    return tasks, hw, pol, mode


def _run(cls, case, mode_name, **kw):
    tasks, hw, pol, mode = _inputs(case, mode_name)
    try:
        sim = cls(tasks, hw, pol, mode, record_events=True, **kw)
    except Exception as e:  # noqa: BLE001
        return ("error", type(e).__name__, str(e))
    try:
        m = sim.run()
    except Exception as e:  # noqa: BLE001
        return ("error", type(e).__name__, str(e))
    finally:
        if hasattr(sim, "close"):
            sim.close()
    d = dataclasses.asdict(m)
    return ("ok", d, [(e.t, e.kind, e.task_id, e.pages) for e in sim.events])


@pytest.mark.skipif(MSIM is None, reason="the reference (msim) is not importable here")
@pytest.mark.parametrize("name,mode", [
    pytest.param(n, m, marks=[pytest.mark.slow] if n in SLOW else []) for n, m in CASES])
def test_plugin_on_reference_engine_matches_unpatched_reference(name, mode):
    _, E, _ = MSIM
    case = loader.sim_case(name)
    want = _run(E.Simulator, case, mode)
    got = _run(b200_simulator_class(E), case, mode)
    assert got == want


@pytest.mark.skipif(MSIM is None, reason="the reference (msim) is not importable here")
def test_plugin_with_real_migration_matches_unpatched_reference():
    """The same plugin moving every planned page between pinned host memory
    and the HBM frame arena (config 2-like LLM mix at reduced size)."""
    mc, E, S = MSIM
    case = loader.sim_case("llm_2.0")
    want = _run(E.Simulator, case, "proactive")
    got = _run(b200_simulator_class(E), case, "proactive", migrate=True)
    assert got == want
