"""Rank placement next to the GPU: the sysfs parsing and the
decision `placement.bind_to_gpu` takes, on a fake sysfs tree (CPU only)."""

import os

import pytest

from paper_2512_24637_b200 import placement


@pytest.mark.parametrize("text,want", [
    ("0-3", [0, 1, 2, 3]),
    ("0-3,8-11\n", [0, 1, 2, 3, 8, 9, 10, 11]),
    ("5", [5]),
    ("0,2,4-5,2", [0, 2, 4, 5]),
    ("", []),
])
def test_parse_cpulist(text, want):
    assert placement.parse_cpulist(text) == want


def test_parse_cpulist_rejects_inverted_ranges():
    with pytest.raises(ValueError):
        placement.parse_cpulist("7-3")


def fake_gpu(root, domain, bus, dev, node, cpus):
    p = placement.gpu_pci_path(domain, bus, dev, sysfs=str(root))
    os.makedirs(p)
    with open(os.path.join(p, "numa_node"), "w") as f:
        f.write(f"{node}\n")
    if cpus is not None:
        with open(os.path.join(p, "local_cpulist"), "w") as f:
            f.write(cpus + "\n")
    return p


def test_pci_path_format(tmp_path):
    assert placement.gpu_pci_path(0, 0x1b, 0, sysfs="/sys").endswith("/bus/pci/devices/0000:1b:00.0")


def test_decision_restricts_to_the_gpu_node(tmp_path):
    allowed = sorted(os.sched_getaffinity(0))
    node_cpus = allowed[: max(1, len(allowed) // 2)]
    spec = ",".join(str(c) for c in node_cpus)
    fake_gpu(tmp_path, 0, 0x9a, 0, 1, spec)
    d = placement.bind_to_gpu(0, sysfs=str(tmp_path), pci=(0, 0x9a, 0), apply=False)
    assert d["numa_node"] == 1 and d["cpu_list"] == node_cpus and d["pci"] == "0000:9a:00.0"
    assert d["node_cpus"] == len(node_cpus) and not d["affinity_set"]


def test_decision_ignores_cpus_outside_the_allowed_set(tmp_path):
    allowed = set(os.sched_getaffinity(0))
    fake_gpu(tmp_path, 0, 0x1b, 0, 0, "100000-100003")
    d = placement.bind_to_gpu(0, sysfs=str(tmp_path), pci=(0, 0x1b, 0), apply=False)
    assert d["cpu_list"] == [] and not (set(d["cpu_list"]) - allowed)


def test_unknown_numa_does_nothing(tmp_path):
    fake_gpu(tmp_path, 0, 0x2c, 0, -1, None)
    before = os.sched_getaffinity(0)
    d = placement.bind_to_gpu(0, sysfs=str(tmp_path), pci=(0, 0x2c, 0))
    assert d["numa_node"] == -1 and not d["affinity_set"] and not d["mempolicy_set"]
    assert os.sched_getaffinity(0) == before


def test_missing_device_does_nothing(tmp_path):
    before = os.sched_getaffinity(0)
    d = placement.bind_to_gpu(0, sysfs=str(tmp_path), pci=(0, 0x77, 0))
    assert d["numa_node"] == -1 and d["node_cpus"] == 0 and not d["affinity_set"]
    assert os.sched_getaffinity(0) == before


def test_apply_binds_affinity_in_a_child(tmp_path):
    """Applying in a forked child: affinity shrinks to the node's CPUs (the
    parent test process keeps its own)."""
    import multiprocessing as mp

    allowed = sorted(os.sched_getaffinity(0))
    if len(allowed) < 2:
        pytest.skip("needs two CPUs")
    fake_gpu(tmp_path, 0, 0x3d, 0, 0, str(allowed[0]))
    ctx = mp.get_context("fork")
    q = ctx.Queue()

    def child():
        d = placement.bind_to_gpu(0, sysfs=str(tmp_path), pci=(0, 0x3d, 0))
        q.put((d["affinity_set"], sorted(os.sched_getaffinity(0))))

    p = ctx.Process(target=child)
    p.start()
    got = q.get(timeout=30)
    p.join()
    assert got == (True, [allowed[0]])
