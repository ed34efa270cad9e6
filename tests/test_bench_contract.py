"""bench.py's contract on the CPU: the reference arm's JSON line (the
reference itself when baseline/_ref or /root/reference is importable, else
the oracle port), the copy-bound arithmetic of the migration roofline, and
the workload table the GPU arm and the reference arm share."""

import json
import math

import pytest

import bench


def test_reference_arm_line(capsys):
    rc = bench.main(["--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1"])
    assert rc == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == bench.UNIT
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    assert line["config"]["workload"] == "cfg1" and line["value"] > 0 and line["ms_per_step"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] == 1 and cb["value"] == line["value"]
    for k in ("cpu_model", "cpu_count", "affinity", "python"):
        assert k in cb
    assert line["e2e"] == {"value": line["value"], "unit": bench.UNIT, "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly(capsys, monkeypatch):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "0"]) == 0
    assert capsys.readouterr().out.strip() == ""


def test_reference_sim_matches_port_on_config1():
    from oracle import msched_port as port

    factory, kind, _ = bench.reference_sim_factory("cfg1", 0)
    times, m = bench.time_reference(factory, 1)
    tasks, hw, pol, _ = bench.workload("cfg1", 0)
    ref = port.PortSim(tasks, hw, pol, bench.workload_mode("cfg1")).run()
    for k in ("migrated_in_pages", "migrated_out_pages", "fault_pages", "total_time_s", "madvise_s"):
        assert getattr(m, k) == getattr(ref, k), (kind, k)


PK = {"h2d": 55.0, "d2h": 57.0, "duplex": 100.0, "duplex_h2d": 50.0, "duplex_d2h": 50.0}


@pytest.mark.parametrize("h2d,d2h", [(100e9, 100e9), (80e9, 100e9), (100e9, 60e9), (0, 40e9), (10e9, 0)])
def test_copy_bound(h2d, d2h):
    got = bench.copy_bound_ms(h2d, d2h, PK)
    th, td = h2d / 50e9, d2h / 50e9
    if th <= td:
        want = th + (d2h - th * 50e9) / 57e9
    else:
        want = td + (h2d - td * 50e9) / 55e9
    assert math.isclose(got, want * 1e3, rel_tol=1e-12)
    # never below either direction alone at its isolated rate, nor below the duplex total
    assert got >= max(h2d / 55e9, d2h / 57e9, (h2d + d2h) / 100e9) * 1e3 - 1e-9


def test_copy_bound_needs_duplex_rates():
    assert bench.copy_bound_ms(1e9, 1e9, {"h2d": 1, "d2h": 1}) is None


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_workloads_are_distinct_per_rank(cfg):
    t0, _, _, d0 = bench.workload(cfg, 0)
    t1, _, _, d1 = bench.workload(cfg, 1)
    assert d0 == d1
    assert not {t.id for t in t0} & {t.id for t in t1}
    assert max(a.base_addr for t in t0 for a in t.allocations) < min(a.base_addr for t in t1 for a in t.allocations)


def _st(**kw):
    base = {"ms_ms": 0.0, "ms_passes": 0, "ms_bytes": 0, "ms_dev_launches": 0, "ms_dev_ms": 0.0, "ms_ev_passes": 0}
    base.update(kw)
    return base


def test_multisplit_roofline_timing_sources():
    # standalone launches (the migrating headline): CUDA events are the primary timing
    r = bench.multisplit_roofline(_st(ms_ms=0.9, ms_passes=10, ms_bytes=10 * 350e6, ms_dev_launches=10,
                                      ms_dev_ms=0.7, ms_ev_passes=10), 6550.0)
    assert r["timing"].startswith("CUDA events") and math.isclose(r["avg_launch_ms"], 0.09)
    assert math.isclose(r["achieved"], 350e6 / (0.09 * 1e6)) and math.isclose(r["device_timed"]["avg_launch_ms"], 0.07)
    # the async path: the multisplit is a phase of the per-switch kernel, so the device clock is primary
    # (a few standalone launches -- e.g. releases -- do not decide it)
    r = bench.multisplit_roofline(_st(ms_ms=0.05, ms_passes=100, ms_bytes=100 * 33e6, ms_dev_launches=100,
                                      ms_dev_ms=1.7, ms_ev_passes=3), 6550.0)
    assert r["timing"].startswith("%globaltimer") and math.isclose(r["avg_launch_ms"], 0.017)
    assert r["launches_per_step"] == 100 and math.isclose(r["frac"], 33e6 / (0.017 * 1e6) / 6550.0)
    # nothing ran
    r = bench.multisplit_roofline(_st(), 6550.0)
    assert r["achieved"] == 0.0 and r["device_timed"] is None
