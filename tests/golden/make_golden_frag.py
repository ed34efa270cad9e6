"""Golden fixtures for the fragmented configuration (bench `--config frag`,
SURVEY.md §0 fact 4 / Appendix B) at sizes the reference finishes in
seconds: the same generator (paper_2512_24637_b200.workload_extra
.fragmented_mix: scattered single pages per command, one eviction-list run per
page), converted to the reference's own msim objects and replayed by the REAL
reference simulator (wrapped by make_golden.RecSim for per-switch records).

Run in the build container (imports /root/reference):

    python tests/golden/make_golden_frag.py

Output: tests/golden/sims_frag.json.gz
"""

from __future__ import annotations

import dataclasses
import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import make_golden as G  # noqa: E402  (imports msim and installs the recording wrappers)
import msim.core as mc  # noqa: E402
from msim.scheduler import Policy as RefPolicy  # noqa: E402

from paper_2512_24637_b200.msim_plugin import to_msim_tasks  # noqa: E402
from paper_2512_24637_b200.workload_extra import fragmented_mix  # noqa: E402

CASES = [
    ("frag_s", dict(npages=2048, ncmds=60, capacity_pages=1024), ["ideal", "um", "proactive", "oracle_pred"]),
    ("frag_m", dict(npages=8192, ncmds=100, capacity_pages=2048), ["ideal", "um"]),
]


def main():
    M = G.modes_all()
    sims = []
    for name, kw, modes in CASES:
        tasks, hw, pol = fragmented_mix(**kw)
        rtasks = to_msim_tasks(mc, tasks)
        rhw = mc.HwConfig(**dataclasses.asdict(hw))
        rpol = RefPolicy(pol.kind, pol.timeslice_s)
        entry = {"name": name, "hw": G.enc_hw(rhw), "policy": G.enc_policy(rpol), "feeder": None,
                 "gen": {"fn": "fragmented_mix", **kw}, "tasks": [G.enc_task(t) for t in rtasks], "runs": {}}
        for mname in modes:
            G._CUR["case"] = name
            t0 = time.perf_counter()
            entry["runs"][mname] = {"mode": G.enc_mode(M[mname]), **G.run_case(rtasks, rhw, rpol, M[mname])}
            print(f"{name:8s} {mname:12s} {time.perf_counter() - t0:7.2f}s", flush=True)
        sims.append(entry)
    with gzip.open(os.path.join(HERE, "sims_frag.json.gz"), "wt") as f:
        json.dump(sims, f)
    print("done")


if __name__ == "__main__":
    main()
