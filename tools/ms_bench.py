"""Micro-benchmark of the eviction-list multisplit (the OPT reorder kernel)
through the C-ABI facade, on synthetic lists shaped like the configs.

  python tools/ms_bench.py [--pages N] [--run-len L] [--windows W] [--runs K] [--reps R]

The list holds N resident pages appended in runs of L consecutive ids (in a
shuffled run order, like populate batches of different tasks); each reorder
uses W windows of K first-access runs drawn over the domain.  Prints the
event-timed multisplit span per pass and the HBM fraction against
MEASURED_PEAKS.json.  Runs on the GPU box."""

import argparse
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_24637_b200._abi import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pages", type=int, default=4_150_000)
    ap.add_argument("--run-len", type=int, default=58_000)
    ap.add_argument("--windows", type=int, default=6)
    ap.add_argument("--runs", type=int, default=40)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = random.Random(a.seed)
    D = int(a.pages * 1.6)
    ctx = Context(4096, a.pages)
    ctx.set_domain([(0, D)])
    starts = rng.sample(range(0, D // a.run_len), a.pages // a.run_len) if a.run_len > 1 else \
        rng.sample(range(D), a.pages)
    runs = sorted((s * a.run_len, s * a.run_len + a.run_len) for s in starts) if a.run_len > 1 else \
        [(s, s + 1) for s in starts]
    rng.shuffle(runs)
    ctx.list_append(runs)
    wins = []
    for _ in range(a.windows):
        ln = max(1, D // (a.runs * 3))
        wr = []
        for _ in range(a.runs):
            s = rng.randrange(0, D - ln)
            wr.append((s, s + rng.randrange(1, ln)))
        wins.append(wr)
    for _ in range(3):
        ctx.list_reorder(wins)
    s0 = ctx.stats()
    for _ in range(a.reps):
        ctx.list_reorder(wins)
    s1 = ctx.stats()
    passes = s1["ms_passes"] - s0["ms_passes"]
    ms = (s1["ms_ms"] - s0["ms_ms"]) / passes
    byts = (s1["ms_bytes"] - s0["ms_bytes"]) / passes
    peak = 6546.9
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = json.load(f)["hbm_gbs"]
    except OSError:
        pass
    gbs = byts / (ms * 1e6)
    print(json.dumps({"pages": a.pages, "run_len": a.run_len, "windows": a.windows, "runs": a.runs,
                      "passes": passes, "us_per_pass": ms * 1e3, "bytes_per_pass": byts, "gbs": gbs,
                      "frac": gbs / peak}))
    ctx.close()


if __name__ == "__main__":
    main()
