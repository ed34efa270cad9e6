"""Columnar binary traces.

The reference's `MSIM-TRACE v1` is a line-oriented text format
(workload.py:419-580) that `parse_trace` reads at ~27 K commands/s into one
Python object per command and argument; the B200 path then columnarises the
objects again for the C ABI (`_abi.encode_commands`).  Many-tenant traces of
10^5-10^6 commands make both steps the bottleneck of a replay's start-up.

`MSIM-TRACE-BIN v1` stores each task already in the C ABI's layout
(`msg_cmd`, `msg_arg`, the raw-struct blob, `msg_range` ground truth; see
include/msched_b200.h) plus a float64 latency column and the kernel-name
table, so loading is a handful of `np.frombuffer` views and the command
tables go to `msg_add_commands` without touching Python objects.  A
`ColumnarTask` keeps the `Task` interface: `commands` is a lazy sequence that
builds a `Command` only when indexed (the analyzer and the reference's own
APIs still see ordinary commands), while the engine reads the columns.

File layout (little-endian): 8-byte magic, u32 header length, JSON header
(tasks, allocations, kernel names, array offsets), then the arrays, each
64-byte aligned.  The text format stays the interchange format; both
directions convert losslessly except for the fields trace v1 does not carry
(priority, arrival: stored here, dropped there).
"""

from __future__ import annotations

import json
import struct
from collections.abc import Sequence

import numpy as np

from . import _abi
from .model import Allocation, Arg, ByteRange, Command, CommandKind, Task

MAGIC = b"MSIMTRB1"
_KINDS = {0: CommandKind.KERNEL, 1: CommandKind.MEMCPY_H2D, 2: CommandKind.MEMCPY_D2H}


class TraceBinError(ValueError):
    pass


def _align(n: int) -> int:
    return (n + 63) & ~63


class CommandColumns(Sequence):
    """A task's commands as ABI columns; indexing builds a `Command`."""

    def __init__(self, cmds, args, blob, gts, lat, names):
        self.cmds, self.args, self.blob, self.gts, self.lat, self.names = cmds, args, blob, gts, lat, names

    def __len__(self):
        return len(self.cmds)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        row = self.cmds[i]
        kind = _KINDS[int(row["kind"])]
        largs = []
        for a in self.args[int(row["arg_off"]):int(row["arg_off"]) + int(row["nargs"])]:
            value = (int(a["hi"]) << 64) | int(a["lo"])
            if int(a["raw_len"]) >= 0:
                off = int(a["raw_off"])
                largs.append(Arg(value, 64, bytes(self.blob[off:off + int(a["raw_len"])])))
            else:
                largs.append(Arg(value, int(a["width"])))
        gt = tuple(ByteRange(int(r["start"]), int(r["len"]))
                   for r in self.gts[int(row["gt_off"]):int(row["gt_off"]) + int(row["ngt"])])
        k = int(row["kernel"])
        dims = tuple(int(x) for x in row["dims"])
        return Command(kind, float(self.lat[i]), self.names[k] if k >= 0 else "", tuple(largs), dims[:3], dims[3:],
                       gt)

    def kinds(self) -> np.ndarray:
        return self.cmds["kind"]


class ColumnarTask(Task):
    """A `Task` whose commands are `CommandColumns` (loaded from a binary trace)."""

    @property
    def columns(self) -> CommandColumns | None:
        return self.commands if isinstance(self.commands, CommandColumns) else None


def _columns_of(task: Task):
    """The ABI columns of any task (a ColumnarTask's own, else encoded)."""
    if isinstance(task.commands, CommandColumns):
        c = task.commands
        return c.cmds, c.args, c.blob, c.gts, c.lat, c.names
    names = sorted({c.kernel_name for c in task.commands if c.kind is CommandKind.KERNEL and c.kernel_name})
    kid = {n: i for i, n in enumerate(names)}
    cmds, args, blob, blen, gts = _abi.encode_commands(task.commands, kid)
    lat = np.asarray([c.latency_s for c in task.commands], dtype=np.float64)
    nargs = int(cmds["nargs"].sum()) if len(cmds) else 0
    ngt = int(cmds["ngt"].sum()) if len(cmds) else 0
    return cmds, args[:nargs], blob[:blen], gts[:ngt], lat, names


def save_trace_bin(tasks: Sequence[Task], path: str):
    """Write tasks (Task or ColumnarTask) as one MSIM-TRACE-BIN v1 file."""
    header = {"version": 1, "tasks": []}
    chunks = []
    off = 0

    def put(arr):
        nonlocal off
        b = np.ascontiguousarray(arr).tobytes()
        rec = {"off": off, "nbytes": len(b), "count": int(len(arr))}
        chunks.append((off, b))
        off = _align(off + len(b))
        return rec

    for t in tasks:
        cmds, args, blob, gts, lat, names = _columns_of(t)
        header["tasks"].append({
            "id": t.id, "priority": t.priority, "arrival_s": t.arrival_s,
            "allocations": [[a.id, a.base_addr, a.size_bytes] for a in t.allocations],
            "names": list(names),
            "cmds": put(cmds), "args": put(args), "blob": put(np.asarray(blob, dtype=np.uint8)),
            "gts": put(gts), "lat": put(np.asarray(lat, dtype=np.float64)),
        })
    hj = json.dumps(header).encode()
    base = _align(len(MAGIC) + 4 + len(hj))
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<I", len(hj)) + hj)
        f.write(b"\0" * (base - (len(MAGIC) + 4 + len(hj))))
        pos = 0
        for o, b in chunks:
            f.write(b"\0" * (o - pos))
            f.write(b)
            pos = o + len(b)


def _validate_columns(cols: "CommandColumns", where: str):
    """The tables go to msg_add_commands as they are: every offset, count,
    raw-struct window, range length and kernel index must lie inside its
    array, and the per-command runs must tile the argument and ground-truth
    arrays in order (encode_columns slices them by the first and last)."""
    cm, n = cols.cmds, len(cols.cmds)
    if len(cols.lat) != n:
        raise TraceBinError(f"{where}: {len(cols.lat)} latencies for {n} commands")
    if n:
        kind = cm["kind"]
        if np.any((kind < _abi.CMD_KERNEL) | (kind > _abi.CMD_D2H)):
            raise TraceBinError(f"{where}: bad command kind")
        for off, cnt, arr, what in (("arg_off", "nargs", cols.args, "argument"),
                                    ("gt_off", "ngt", cols.gts, "ground-truth")):
            o, c = cm[off].astype(np.int64), cm[cnt].astype(np.int64)
            if np.any(o < 0) or np.any(c < 0):
                raise TraceBinError(f"{where}: negative {what} offset or count")
            if o[0] != 0 or np.any(o[1:] != o[:-1] + c[:-1]) or o[-1] + c[-1] != len(arr):
                raise TraceBinError(f"{where}: {what} runs do not tile the {what} array")
        k = cm["kernel"]
        if np.any((k < -1) | (k >= len(cols.names))):
            raise TraceBinError(f"{where}: kernel index outside the name table")
        mem = kind != _abi.CMD_KERNEL
        if np.any(cm["dev_len"][mem] <= 0) or np.any(cm["nargs"][mem] != 3):
            raise TraceBinError(f"{where}: memcpy without a positive extent and 3 arguments")
    a = cols.args
    raw = a["raw_len"] >= 0
    if np.any((a["raw_off"][raw] < 0) | (a["raw_off"][raw] + a["raw_len"][raw] > len(cols.blob))):
        raise TraceBinError(f"{where}: raw struct argument outside the blob")
    if np.any(~raw & (a["width"] != 32) & (a["width"] != 64)):
        raise TraceBinError(f"{where}: argument width must be 32 or 64")
    if len(cols.gts) and np.any(cols.gts["len"] <= 0):
        raise TraceBinError(f"{where}: zero or negative length range")


def load_trace_bin(path: str) -> list:
    """Read an MSIM-TRACE-BIN v1 file into ColumnarTasks (zero-copy views)."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != MAGIC:
        raise TraceBinError(f"{path}: not an MSIM-TRACE-BIN v1 file")
    (hl,) = struct.unpack_from("<I", data, 8)
    try:
        header = json.loads(data[12:12 + hl])
    except ValueError as e:
        raise TraceBinError(f"{path}: corrupt header: {e}") from None
    if header.get("version") != 1:
        raise TraceBinError(f"{path}: unsupported version {header.get('version')}")
    base = _align(12 + hl)
    buf = memoryview(data)

    def view(rec, dtype):
        lo = base + rec["off"]
        a = np.frombuffer(buf[lo:lo + rec["nbytes"]], dtype=dtype)
        if len(a) != rec["count"]:
            raise TraceBinError(f"{path}: array length mismatch")
        return a

    out = []
    for h in header["tasks"]:
        cols = CommandColumns(view(h["cmds"], _abi.CMD_DT), view(h["args"], _abi.ARG_DT),
                              view(h["blob"], np.uint8), view(h["gts"], _abi.RANGE_DT),
                              view(h["lat"], np.float64), list(h["names"]))
        if np.any(cols.lat <= 0):
            raise TraceBinError(f"{path}: task {h['id']!r} has non-positive latencies")
        _validate_columns(cols, f"{path}: task {h['id']!r}")
        allocs = [Allocation(a, int(b), int(s), h["id"]) for a, b, s in h["allocations"]]
        out.append(ColumnarTask(id=h["id"], allocations=allocs, commands=cols, priority=int(h["priority"]),
                                arrival_s=float(h["arrival_s"])))
    return out


def kernel_ids_for(cols: CommandColumns, kid: dict) -> np.ndarray:
    """Remap the file's kernel-name indices to a rule table's kernel ids (-1 unknown)."""
    lut = np.asarray([kid.get(n, -1) for n in cols.names] + [-1], dtype=np.int32)
    k = cols.cmds["kernel"]
    return lut[np.where(k >= 0, k, len(cols.names))]


def encode_columns(cols: CommandColumns, kid: dict, lo: int = 0, hi: int | None = None):
    """`_abi.encode_commands`' output for commands [lo, hi) of a ColumnarTask,
    built with array operations (offsets rebased to the slice)."""
    hi = len(cols) if hi is None else hi
    cm = cols.cmds[lo:hi].copy()
    cm["kernel"] = kernel_ids_for(cols, kid)[lo:hi]
    if hi > lo:
        a0, a1 = int(cm["arg_off"][0]), int(cm["arg_off"][-1] + cm["nargs"][-1])
        g0, g1 = int(cm["gt_off"][0]), int(cm["gt_off"][-1] + cm["ngt"][-1])
    else:
        a0 = a1 = g0 = g1 = 0
    cm["arg_off"] -= a0
    cm["gt_off"] -= g0
    args = cols.args[a0:a1] if a1 > a0 else np.zeros(1, _abi.ARG_DT)
    gts = cols.gts[g0:g1] if g1 > g0 else np.zeros(1, _abi.RANGE_DT)
    blob = cols.blob if len(cols.blob) else np.zeros(1, np.uint8)
    return cm, args, blob, len(cols.blob), gts


def trace_v1_to_bin(text_paths: Sequence[str], out_path: str):
    """Convert MSIM-TRACE v1 text files (one task each) to one binary trace."""
    from .workload import load_trace

    save_trace_bin([load_trace(p) for p in text_paths], out_path)
