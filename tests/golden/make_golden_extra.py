"""Golden fixtures for the configurations the reference has no generator for
 and the page-size sweep (config 5).

Run in the build container (imports /root/reference):

    python tests/golden/make_golden_extra.py

Config 3 tasks come from paper_2512_24637_b200.workload_extra; they are
converted to the reference's own msim objects and replayed by the REAL
reference simulator (wrapped by make_golden.RecSim), so the fixtures are the
reference's behaviour on those traces.  Output: tests/golden/sims_extra.json.gz
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import make_golden as G  # noqa: E402  (imports msim and installs the recording wrappers)
from msim.core import Allocation, Arg, ByteRange, Command, CommandKind, Task  # noqa: E402
from msim.core import HwConfig as RefHw  # noqa: E402
from msim.scheduler import Policy as RefPolicy  # noqa: E402

from paper_2512_24637_b200.workload_extra import config3_mixed  # noqa: E402


def to_msim(t):
    d = G.enc_task(t)
    task = Task(id=d["id"], cursor=d["cursor"], priority=d["priority"], arrival_s=d["arrival_s"])
    task.allocations = [Allocation(i, b, s, d["id"]) for i, b, s in d["allocations"]]
    for c in d["commands"]:
        args = tuple(Arg(0, 64, raw=bytes.fromhex(a["raw"])) if "raw" in a else Arg(a["v"], a["w"])
                     for a in c["args"])
        task.commands.append(Command(kind=CommandKind(c["kind"]), latency_s=c["lat"], kernel_name=c["name"],
                                     launch_args=args, grid_dims=tuple(c["grid"]), block_dims=tuple(c["block"]),
                                     ground_truth_access=tuple(ByteRange(s, n) for s, n in c["gt"])))
    return task


def main():
    M = G.modes_all()
    cases = []
    for ratio, ts in ((2.0, 5e-5), (3.0, 5e-5)):
        tasks, hw, pol = config3_mixed(ratio=ratio, timeslice_s=ts)
        rhw = RefHw(**{k: getattr(hw, k) for k in G.enc_hw(G.get_preset("rtx5080"))})
        cases.append((f"cfg3_{ratio}", [to_msim(t) for t in tasks], rhw, RefPolicy(pol.kind, pol.timeslice_s),
                      ["proactive", "ideal", "um", "allocation", "sequential", "late"],
                      {"fn": "config3_mixed", "ratio": ratio, "timeslice_s": ts}))
    for page in (16384, 65536):
        tasks, hw, pol = G.llm_mix(3, 32, 7.6e9, 0.9e9, 8, 16 * G.GIB, page=page)
        cases.append((f"cfg5_{page // 1024}k", tasks, hw, pol, ["proactive", "ideal"],
                      {"fn": "cfg2", "page": page}))
    sims = []
    for name, tasks, hw, pol, modes, gen in cases:
        entry = {"name": name, "hw": G.enc_hw(hw), "policy": G.enc_policy(pol), "feeder": None, "gen": gen,
                 "tasks": [G.enc_task(t) for t in tasks], "runs": {}}
        for mname in modes:
            G._CUR["case"] = name
            t0 = time.perf_counter()
            entry["runs"][mname] = {"mode": G.enc_mode(M[mname]), **G.run_case(tasks, hw, pol, M[mname])}
            print(f"{name:12s} {mname:12s} {time.perf_counter() - t0:7.2f}s", flush=True)
        sims.append(entry)
    with gzip.open(os.path.join(HERE, "sims_extra.json.gz"), "wt") as f:
        json.dump(sims, f)
    print("done")


if __name__ == "__main__":
    main()
