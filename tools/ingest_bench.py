"""Trace ingestion: MSIM-TRACE v1 text vs MSIM-TRACE-BIN v1 (columns straight
to msg_add_commands).  Many-tenant LLM decode traces (config-4 shaped,
scaled to N commands).  Prints one JSON line.  Needs a GPU for the upload leg.

  python tools/ingest_bench.py [--tenants T] [--steps S]
"""
import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_24637_b200 import engine, tracebin, workload  # noqa: E402
from paper_2512_24637_b200.analyzer import build_descriptors  # noqa: E402
from paper_2512_24637_b200.scenarios import config4_llama70b  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tenants", type=int, default=8)
    ap.add_argument("--steps", type=int, default=40)
    a = ap.parse_args()
    tasks, hw, pol = config4_llama70b(n_tenants=a.tenants)
    # more decode steps per tenant: extend with the generator's own step commands
    tasks = [t for t in tasks]
    base = {t.id: list(t.commands) for t in tasks}
    for t in tasks:
        cmds = base[t.id]
        reps = max(1, a.steps // 3)
        t.commands = cmds * reps
    ncmd = sum(len(t.commands) for t in tasks)
    descs = {t.id: build_descriptors(type(t)(id=t.id, allocations=t.allocations, commands=base[t.id]))
             for t in tasks}
    d = tempfile.mkdtemp()
    paths = []
    t0 = time.perf_counter()
    for i, t in enumerate(tasks):
        pth = os.path.join(d, f"{i}.trace")
        workload.save_trace(t, pth)
        paths.append(pth)
    t_text_save = time.perf_counter() - t0
    t0 = time.perf_counter()
    text_tasks = [workload.load_trace(p) for p in paths]
    t_text_load = time.perf_counter() - t0
    for t, src in zip(text_tasks, tasks):
        t.id = src.id
    binp = os.path.join(d, "all.msimb")
    t0 = time.perf_counter()
    tracebin.save_trace_bin(tasks, binp)
    t_bin_save = time.perf_counter() - t0
    t0 = time.perf_counter()
    bin_tasks = tracebin.load_trace_bin(binp)
    t_bin_load = time.perf_counter() - t0
    out = {"commands": ncmd, "tenants": a.tenants, "text_bytes": sum(os.path.getsize(p) for p in paths),
           "bin_bytes": os.path.getsize(binp), "text_save_s": t_text_save, "text_load_s": t_text_load,
           "bin_save_s": t_bin_save, "bin_load_s": t_bin_load,
           "text_cmds_per_s": ncmd / t_text_load, "bin_cmds_per_s": ncmd / t_bin_load}
    # offline analysis of the whole trace: host analyzer on objects vs the
    # native analyzer (msg_analyze) on the binary columns
    t0 = time.perf_counter()
    d_obj = {t.id: build_descriptors(t, native=False) for t in text_tasks}
    out["analyze_host_objects_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    d_col = {t.id: build_descriptors(t, native=True) for t in bin_tasks}
    out["analyze_native_columns_s"] = time.perf_counter() - t0
    out["analyzer_outputs_equal"] = d_obj == d_col
    for label, ts in (("objects", text_tasks), ("columns", bin_tasks)):
        t0 = time.perf_counter()
        sim = engine.Simulator(ts, hw, pol, engine.Mode.proactive(), descriptors=descs)
        sim.ctx.sync()
        out[f"sim_init_{label}_s"] = time.perf_counter() - t0
        sim.close()
    out["load_plus_init_text_s"] = t_text_load + out["sim_init_objects_s"]
    out["load_plus_init_bin_s"] = t_bin_load + out["sim_init_columns_s"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
