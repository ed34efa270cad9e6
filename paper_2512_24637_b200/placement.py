"""Host placement of one rank next to its GPU.

Each rank replays its own tenant mix and migrates pages between its GPU and
a pinned host pool.  The pool and the thread that issues the copies belong on
the NUMA node the GPU's PCIe root hangs off: a remote pool makes every copy
cross the socket interconnect, which 8 concurrent migrators share.

`bind_to_gpu(device)` reads the GPU's PCI function from sysfs
(`/sys/bus/pci/devices/<domain:bus:dev.fn>/{numa_node,local_cpulist}`),
restricts the process to that node's CPUs (`sched_setaffinity`) and makes the
node the preferred node for new memory (`set_mempolicy(MPOL_PREFERRED)`), so
the pinned pool that `msg_create` allocates afterwards (cudaHostAlloc touches
every page from this thread) lands there.  It returns what it did, for the
bench line.  Nothing here is on the device path; on hosts without NUMA
information it does nothing and says so.
"""

from __future__ import annotations

import ctypes
import os

__all__ = ["parse_cpulist", "gpu_pci_path", "numa_info", "bind_to_gpu"]

MPOL_PREFERRED = 1
_SYS_SET_MEMPOLICY = {"x86_64": 238, "aarch64": 237}


def parse_cpulist(text: str) -> list[int]:
    """Linux cpulist format ("0-3,8,10-11") -> sorted cpu ids."""
    out: set[int] = set()
    for part in text.strip().split(","):
        part = part.strip()
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-", 1)
            lo, hi = int(a), int(b)
            if hi < lo:
                raise ValueError(f"bad cpulist range {part!r}")
            out.update(range(lo, hi + 1))
        else:
            out.add(int(part))
    return sorted(out)


def gpu_pci_path(domain: int, bus: int, device: int, sysfs: str = "/sys") -> str:
    return os.path.join(sysfs, "bus", "pci", "devices", f"{domain:04x}:{bus:02x}:{device:02x}.0")


def numa_info(pci_path: str) -> dict:
    """{'node': int (-1 = unknown), 'cpus': [int]} of one PCI function."""
    node, cpus = -1, []
    try:
        with open(os.path.join(pci_path, "numa_node")) as f:
            node = int(f.read().strip())
    except (OSError, ValueError):
        pass
    try:
        with open(os.path.join(pci_path, "local_cpulist")) as f:
            cpus = parse_cpulist(f.read())
    except (OSError, ValueError):
        pass
    return {"node": node, "cpus": cpus}


def _set_preferred_node(node: int) -> bool:
    nr = _SYS_SET_MEMPOLICY.get(os.uname().machine)
    if nr is None or node < 0:
        return False
    libc = ctypes.CDLL(None, use_errno=True)
    words = node // 64 + 1
    mask = (ctypes.c_ulong * words)()
    mask[node // 64] = 1 << (node % 64)
    rc = libc.syscall(ctypes.c_long(nr), ctypes.c_int(MPOL_PREFERRED), mask, ctypes.c_ulong(words * 64 + 1))
    return rc == 0


def bind_to_gpu(device: int, sysfs: str = "/sys", pci: tuple | None = None, apply: bool = True) -> dict:
    """Pin this process's CPUs and memory preference to `device`'s NUMA node.

    `pci` = (domain, bus, device) of the GPU; by default read from
    torch.cuda.get_device_properties.  With apply=False only the decision is
    returned (tests)."""
    if pci is None:
        import torch

        p = torch.cuda.get_device_properties(device)
        pci = (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    path = gpu_pci_path(*pci, sysfs=sysfs)
    info = numa_info(path)
    try:
        allowed = sorted(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover - non-Linux
        allowed = []
    cpus = [c for c in info["cpus"] if c in set(allowed)] if allowed else info["cpus"]
    out = {"pci": "%04x:%02x:%02x.0" % tuple(pci), "numa_node": info["node"], "node_cpus": len(info["cpus"]),
           "cpus": len(cpus), "affinity_set": False, "mempolicy_set": False}
    if not apply:
        out["cpu_list"] = cpus
        return out
    if cpus and len(cpus) < len(allowed):
        os.sched_setaffinity(0, cpus)
        out["affinity_set"] = True
    if info["node"] >= 0:
        out["mempolicy_set"] = _set_preferred_node(info["node"])
    return out
