"""Per-command latency of the drop-in predictor facade (predictor.predict,
one command per call, as the reference's Simulator calls it) and of the
batched form (predict_task over a task's commands), against the
reference's own predict (msim.predictor.predict) when baseline/_ref is
importable.  GPU box: python tools/predict_latency.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2512_24637_b200 import predictor  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402
from paper_2512_24637_b200.scenarios import config2_llama8b  # noqa: E402

tasks, hw, _ = config2_llama8b()
task = tasks[0]
descs = build_descriptors(task)
P = hw.page_size_bytes
cmds = list(task.commands)[:200]
for c in cmds[:20]:
    predictor.predict(descs, c, P)                    # warm the cached context
t = []
for c in cmds:
    t0 = time.perf_counter()
    predictor.predict(descs, c, P)
    t.append(time.perf_counter() - t0)
print(f"facade predict(): median {statistics.median(t) * 1e6:.1f} us/cmd, p90 "
      f"{sorted(t)[int(0.9 * len(t))] * 1e6:.1f} us over {len(t)} commands")
allc = list(task.commands)
predictor.predict_task(allc, P, "template", descs)
t0 = time.perf_counter()
predictor.predict_task(allc, P, "template", descs)
dt = time.perf_counter() - t0
print(f"batched predict_task(): {dt * 1e6 / len(allc):.2f} us/cmd over {len(allc)} commands ({dt * 1e3:.1f} ms)")
ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if os.path.isdir(os.path.join(ref, "msim")):
    sys.path.insert(0, ref)
    import msim.analyzer as RA
    import msim.core as mc
    import msim.predictor as RP
    from paper_2512_24637_b200.msim_plugin import to_msim_tasks

    rt = to_msim_tasks(mc, [task])[0]
    rd = RA.build_descriptors(rt)
    t = []
    for c in rt.commands[:200]:
        t0 = time.perf_counter()
        RP.predict(rd, c, P)
        t.append(time.perf_counter() - t0)
    print(f"reference msim predict(): median {statistics.median(t) * 1e6:.1f} us/cmd over {len(t)} commands")
