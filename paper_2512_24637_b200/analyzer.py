"""Offline template inference: launch arguments -> access-region rules.

This is the *input producer* for the GPU predictor (the
offline analyzer is out of scope for the device; its rule table is what the
device evaluates per command).  It keeps the reference's types and matching
order (analyzer.py:31-517): per identified pointer argument one rule, tried
as fixed, then linear in a product of <= 3 integer slots, then strided; all
coefficients exact rationals.  `rule_table()` lowers descriptors to the flat
integer form the C-ABI consumes (`msg_rule` in include/msched_b200.h).
"""

from __future__ import annotations

import itertools
import struct
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional, Sequence

from .model import Arg, ByteRange, Command, CommandKind

__all__ = [
    "DESC_HEADER", "MAX_PRODUCT_TERMS", "DescriptorError", "InvocationRecord",
    "coalesce_regions", "slice_struct_args", "slot_values", "LinearExpr", "TemplateRule",
    "KernelDescriptor", "identify_pointer_args", "fit_linear_expr", "infer_rule",
    "build_descriptor", "build_descriptors", "records_from_task", "classify_regions",
    "format_descriptors", "save_descriptors", "load_descriptors",
]

DESC_HEADER = "MSIM-DESC v1"
MAX_PRODUCT_TERMS = 3
_DIMS = ("gx", "gy", "gz", "bx", "by", "bz")


class DescriptorError(ValueError):
    pass


def coalesce_regions(regions: Sequence[ByteRange]) -> tuple:
    """Sort by start; merge strictly overlapping regions only
    (analyzer.py:53-64)."""
    out: list = []
    for r in sorted(regions, key=lambda r: r.start_addr):
        if out and r.start_addr < out[-1].end_addr:
            top = out[-1]
            out[-1] = ByteRange(top.start_addr, max(top.end_addr, r.end_addr) - top.start_addr)
        else:
            out.append(r)
    return tuple(out)


@dataclass(frozen=True)
class InvocationRecord:
    kernel_name: str
    launch_args: tuple
    grid_dims: tuple = (1, 1, 1)
    block_dims: tuple = (1, 1, 1)
    observed_regions: tuple = ()
    latency_s: float = 1e-6

    @classmethod
    def from_command(cls, cmd: Command) -> "InvocationRecord":
        assert cmd.kind is CommandKind.KERNEL
        return cls(cmd.kernel_name, cmd.launch_args, cmd.grid_dims, cmd.block_dims,
                   coalesce_regions(cmd.ground_truth_access), cmd.latency_s)


def slice_struct_args(raw: bytes) -> list:
    """Aligned little-endian 64-bit windows, then 32-bit ones."""
    wide = [(o, 64, struct.unpack_from("<Q", raw, o)[0]) for o in range(0, len(raw) - 7, 8)]
    narrow = [(o, 32, struct.unpack_from("<I", raw, o)[0]) for o in range(0, len(raw) - 3, 4)]
    return wide + narrow


def slot_values(launch_args, grid_dims=(1, 1, 1), block_dims=(1, 1, 1)) -> dict:
    """analyzer.py:78-96: a{i}, a{i}+{off}w{32|64}, gx..bz."""
    vals: dict = {}
    for i, a in enumerate(launch_args):
        if a.raw is None:
            vals[f"a{i}"] = a.value
        else:
            for o, w, v in slice_struct_args(a.raw):
                vals[f"a{i}+{o}w{w}"] = v
    vals.update(zip(_DIMS, tuple(grid_dims) + tuple(block_dims)))
    return vals


def slot_rank(slot: str) -> tuple:
    """Arguments (index, then struct offset, wider first) before dims."""
    if slot[0] == "a":
        head, _, tail = slot[1:].partition("+")
        if tail:
            off, w = tail.split("w")
            return (0, int(head), 1, int(off), -int(w))
        return (0, int(head), 0, 0, 0)
    return (1, _DIMS.index(slot), 0, 0, 0)


@dataclass(frozen=True)
class LinearExpr:
    """A constant, or coeff * product(slots) (analyzer.py:112-142)."""

    coeff: Fraction
    slots: tuple = ()

    def evaluate(self, vals: dict) -> Optional[int]:
        prod = Fraction(1)
        for s in self.slots:
            if s not in vals:
                return None
            prod *= vals[s]
        v = self.coeff * prod
        return int(v) if v.denominator == 1 else None

    def serialize(self) -> str:
        if not self.slots:
            return f"fixed:{self.coeff}"
        return f"lin:{self.coeff}*" + "*".join(self.slots)

    @classmethod
    def parse(cls, s: str) -> "LinearExpr":
        if s.startswith("fixed:"):
            return cls(Fraction(s[6:]))
        if s.startswith("lin:"):
            coeff, *slots = s[4:].split("*")
            return cls(Fraction(coeff), tuple(slots))
        raise DescriptorError(f"bad linear expression {s!r}")


@dataclass(frozen=True)
class TemplateRule:
    ptr_arg_index: int
    kind: str  # fixed | linear | strided | unpredictable
    offset_bytes: int = 0
    size: Optional[LinearExpr] = None
    stride: Optional[LinearExpr] = None
    chunk: Optional[LinearExpr] = None
    count: Optional[LinearExpr] = None

    def predict_regions(self, cmd: Command) -> Optional[list]:
        """Host-side evaluation (analyzer.py:155-174).  Used only by the
        offline analyzer itself (uncovered-fraction); the GPU evaluates rules
        for the simulation (csrc/predict.cu)."""
        if self.kind == "unpredictable" or self.ptr_arg_index >= len(cmd.launch_args):
            return None
        base = cmd.launch_args[self.ptr_arg_index].value + self.offset_bytes
        vals = slot_values(cmd.launch_args, cmd.grid_dims, cmd.block_dims)
        if self.kind in ("fixed", "linear"):
            n = self.size.evaluate(vals)
            return None if n is None else [ByteRange(base, max(n, 1))]
        st, ch, ct = (e.evaluate(vals) for e in (self.stride, self.chunk, self.count))
        if st is None or ch is None or ct is None or ct < 1:
            return None
        return [ByteRange(base + j * st, max(ch, 1)) for j in range(ct)]


@dataclass
class KernelDescriptor:
    kernel_name: str
    rules: list = field(default_factory=list)
    profiled_latency_s: float = 1e-6
    unpredictable_fraction: float = 0.0


def _plain64(a: Arg) -> bool:
    return a.raw is None and a.width == 64


def identify_pointer_args(records: Sequence[InvocationRecord]) -> list:
    """64-bit args equal to a region start in every record (analyzer.py:185-206)."""
    if not records:
        raise ValueError("need at least one record")
    found = []
    for i in range(len(records[0].launch_args)):
        if all(i < len(r.launch_args) and _plain64(r.launch_args[i])
               and any(g.start_addr == r.launch_args[i].value for g in r.observed_regions)
               for r in records):
            found.append(i)
    return found


def _constant_offset(records, i) -> Optional[int]:
    """Smallest c > 0 with arg+c a region start in every record, looking only
    at starts below 2*arg (analyzer.py:209-226)."""
    common = None
    for r in records:
        a = r.launch_args[i]
        if not _plain64(a):
            return None
        here = {g.start_addr - a.value for g in r.observed_regions if a.value < g.start_addr < 2 * a.value}
        common = here if common is None else common & here
        if not common:
            return None
    return min(common)


class _Fitter:
    """Caches the per-record slot tables for one kernel's records."""

    def __init__(self, records):
        self.records = records
        self.tables = [slot_values(r.launch_args, r.grid_dims, r.block_dims) for r in records]

    def factor_slots(self, pointer_indices) -> list:
        """Positive in every record, deduplicated by value signature keeping
        the lowest-ranked name (analyzer.py:240-263)."""
        chosen, sigs = [], set()
        for name in sorted(self.tables[0], key=slot_rank):
            if name[0] == "a" and "+" not in name and int(name[1:]) in pointer_indices:
                continue
            sig = tuple(t.get(name) for t in self.tables)
            if any(v is None or v <= 0 for v in sig) or sig in sigs:
                continue
            sigs.add(sig)
            chosen.append(name)
        return chosen

    def fit(self, values, slots, max_terms=MAX_PRODUCT_TERMS) -> Optional[LinearExpr]:
        """Constant; else the first exact coeff*prod fit by (fewest factors,
        lowest slots) (analyzer.py:266-293)."""
        if len(set(values)) == 1:
            return LinearExpr(Fraction(values[0]))
        for k in range(1, max_terms + 1):
            for combo in itertools.combinations_with_replacement(slots, k):
                ratios = set()
                for v, t in zip(values, self.tables):
                    prod = 1
                    for s in combo:
                        prod *= t[s]
                    ratios.add(Fraction(v, prod))
                    if len(ratios) > 1:
                        break
                if len(ratios) == 1:
                    (c,) = ratios
                    if c > 0:
                        return LinearExpr(c, combo)
        return None


def fit_linear_expr(values, records, slots, max_terms=MAX_PRODUCT_TERMS):
    return _Fitter(records).fit(list(values), list(slots), max_terms)


def infer_rule(records, ptr_arg_index: int, offset_bytes: int = 0, all_ptr_indices=None,
               _fitter: _Fitter | None = None) -> TemplateRule:
    """analyzer.py:296-349."""
    ptrs = all_ptr_indices if all_ptr_indices is not None else {ptr_arg_index: offset_bytes}
    fitter = _fitter or _Fitter(records)
    dead = TemplateRule(ptr_arg_index, "unpredictable", offset_bytes)
    families = []
    for r in records:
        base = r.launch_args[ptr_arg_index].value + offset_bytes
        others = [r.launch_args[i].value + o for i, o in ptrs.items()
                  if not (i == ptr_arg_index and o == offset_bytes)]
        ceiling = min((b for b in others if b > base), default=None)
        fam = [g for g in r.observed_regions
               if g.start_addr >= base and (ceiling is None or g.start_addr < ceiling)]
        if not fam or fam[0].start_addr != base:
            return dead
        families.append(fam)
    slots = fitter.factor_slots(set(ptrs))
    if all(len(f) == 1 for f in families):
        sizes = [f[0].length_bytes for f in families]
        if len(set(sizes)) == 1:
            return TemplateRule(ptr_arg_index, "fixed", offset_bytes, size=LinearExpr(Fraction(sizes[0])))
        e = fitter.fit(sizes, slots)
        return TemplateRule(ptr_arg_index, "linear", offset_bytes, size=e) if e is not None and e.slots else dead
    strides, chunks, counts = [], [], []
    for fam in families:
        if len(fam) < 2:
            return dead
        st = {b.start_addr - a.start_addr for a, b in zip(fam, fam[1:])}
        ln = {g.length_bytes for g in fam}
        if len(st) != 1 or len(ln) != 1:
            return dead
        strides.append(st.pop())
        chunks.append(ln.pop())
        counts.append(len(fam))
    es, ec, en = fitter.fit(strides, slots), fitter.fit(chunks, slots), fitter.fit(counts, slots)
    if es is None or ec is None or en is None:
        return dead
    return TemplateRule(ptr_arg_index, "strided", offset_bytes, stride=es, chunk=ec, count=en)


def _as_command(r: InvocationRecord) -> Command:
    return Command(kind=CommandKind.KERNEL, kernel_name=r.kernel_name, latency_s=r.latency_s,
                   launch_args=r.launch_args, grid_dims=r.grid_dims, block_dims=r.block_dims)


def _covered(regs, g) -> bool:
    return any(p.start_addr <= g.start_addr and p.end_addr >= g.end_addr for p in regs)


def build_descriptor(kernel_name: str, records, min_records: int = 2) -> KernelDescriptor:
    """analyzer.py:352-402 (min_records is accepted and unused, as in the
    reference — SURVEY.md Appendix A)."""
    if not records:
        raise ValueError(f"no records for kernel {kernel_name!r}")
    ptrs = {i: 0 for i in identify_pointer_args(records)}
    for i in range(len(records[0].launch_args)):
        if i not in ptrs:
            c = _constant_offset(records, i)
            if c is not None:
                ptrs[i] = c
    fitter = _Fitter(records)
    rules = [infer_rule(records, i, o, ptrs, fitter) for i, o in sorted(ptrs.items())]
    desc = KernelDescriptor(kernel_name, [r for r in rules if r.kind != "unpredictable"],
                            sum(r.latency_s for r in records) / len(records))
    total = misses = 0
    for r in records:
        cmd = _as_command(r)
        regs = [g for rule in desc.rules for g in (rule.predict_regions(cmd) or [])]
        for g in r.observed_regions:
            total += 1
            misses += not _covered(regs, g)
    desc.unpredictable_fraction = misses / total if total else 0.0
    return desc


def classify_regions(desc: KernelDescriptor, records) -> dict:
    """analyzer.py:421-434."""
    counts = {"fixed": 0, "linear": 0, "strided": 0, "others": 0}
    for r in records:
        cmd = _as_command(r)
        by_rule = [(rule, rule.predict_regions(cmd) or []) for rule in desc.rules]
        for g in r.observed_regions:
            kind = next((rule.kind for rule, regs in by_rule if _covered(regs, g)), "others")
            counts[kind] += 1
    return counts


def records_from_task(task) -> dict:
    out: dict = {}
    for c in task.commands:
        if c.kind is CommandKind.KERNEL:
            out.setdefault(c.kernel_name, []).append(InvocationRecord.from_command(c))
    return out


def build_descriptors(task, native: bool = True) -> dict:
    """One descriptor per kernel name (analyzer.py:437-441).  With
    native=True the inference runs in the C-ABI library (msg_analyze, host
    C++, exact 256-bit ratio tests); kernels whose numbers fall outside its
    arithmetic, and every kernel when the library is absent, take this
    module's path.  Both give identical descriptors (tests/test_analyzer_native.py)."""
    if native:
        try:
            return _build_descriptors_native(task)
        except (ImportError, OSError, ValueError, RuntimeError):
            pass   # no library, or inputs the encoder rejects: the host path decides
    return {name: build_descriptor(name, recs) for name, recs in records_from_task(task).items()}


def _build_descriptors_native(task) -> dict:
    import numpy as np

    from . import _abi
    from .tracebin import CommandColumns

    cols = task.commands if isinstance(task.commands, CommandColumns) else None
    first = {}
    if cols is not None:   # binary trace: the columns already are the ABI tables
        kern = cols.cmds["kernel"]
        is_k = (cols.kinds() == _abi.CMD_KERNEL) & (kern >= 0)
        idx = np.flatnonzero(is_k)
        uniq, first_pos = np.unique(kern[idx], return_index=True)
        order = np.argsort(first_pos, kind="stable")
        names = [cols.names[int(uniq[o])] for o in order]
        remap = np.full(len(cols.names) + 1, -1, dtype=np.int32)
        remap[uniq[order]] = np.arange(len(order), dtype=np.int32)
        cm = cols.cmds.copy()
        cm["kernel"] = np.where(is_k, remap[np.where(kern >= 0, kern, len(cols.names))], -1)
        enc = (cm, cols.args if len(cols.args) else np.zeros(1, _abi.ARG_DT),
               cols.blob if len(cols.blob) else np.zeros(1, np.uint8), len(cols.blob),
               cols.gts if len(cols.gts) else np.zeros(1, _abi.RANGE_DT))
        lat_in = cols.lat
        for o in order:
            first[cols.names[int(uniq[o])]] = cols[int(idx[first_pos[o]])]
    else:
        names, seen = [], {}
        for c in task.commands:
            if c.kind is CommandKind.KERNEL and c.kernel_name not in seen:
                seen[c.kernel_name] = len(names)
                names.append(c.kernel_name)
                first[c.kernel_name] = c
        enc = _abi.encode_commands(task.commands, seen)
        lat_in = [c.latency_s for c in task.commands]
    if not names:
        return {}
    status, lat, unp, rules, off = _abi.analyze(enc, lat_in, len(names))
    out = {}
    recs = None
    for k, name in enumerate(names):
        if status[k]:
            recs = recs or records_from_task(task)
            out[name] = build_descriptor(name, recs[name])
            continue
        c0 = first[name]
        vals = slot_values(c0.launch_args, c0.grid_dims, c0.block_dims)
        rl = []
        for r in rules[off[k]:off[k + 1]]:
            ex = []
            for q in range(3 if int(r["kind"]) == 2 else 1):
                slots = tuple(_abi.slot_name(int(x)) for x in r["slot"][q][:int(r["nslots"][q])])
                prod = 1
                for sname in slots:
                    prod *= vals[sname]
                ex.append(LinearExpr(Fraction(int(r["v0"][q]), prod), slots))
            kind = ("fixed", "linear", "strided")[int(r["kind"])]
            if kind == "strided":
                rl.append(TemplateRule(int(r["ptr_arg"]), kind, int(r["offset"]), stride=ex[0], chunk=ex[1],
                                       count=ex[2]))
            else:
                rl.append(TemplateRule(int(r["ptr_arg"]), kind, int(r["offset"]), size=ex[0]))
        out[name] = KernelDescriptor(name, rl, float(lat[k]), float(unp[k]))
    return out


def format_descriptors(descs: dict) -> str:
    out = [DESC_HEADER]
    for name in sorted(descs):
        d = descs[name]
        out.append(f"KERNEL {name} latency={d.profiled_latency_s!r} "
                   f"unpredictable={d.unpredictable_fraction!r}")
        for r in d.rules:
            head = f"RULE ptr={r.ptr_arg_index} offset={r.offset_bytes}"
            if r.kind in ("fixed", "linear"):
                out.append(f"{head} kind={r.kind} size={r.size.serialize()}")
            else:
                out.append(f"{head} kind=strided stride={r.stride.serialize()} "
                           f"chunk={r.chunk.serialize()} count={r.count.serialize()}")
    return "\n".join(out) + "\n"


def save_descriptors(descs: dict, path: str):
    with open(path, "w", encoding="utf-8") as f:
        f.write(format_descriptors(descs))


def load_descriptors(path: str) -> dict:
    with open(path, encoding="utf-8") as f:
        lines = f.read().splitlines()
    if not lines or lines[0].strip() != DESC_HEADER:
        raise DescriptorError(f"{path}:1: missing '{DESC_HEADER}' header")
    descs: dict = {}
    cur = None
    for lineno, raw in enumerate(lines[1:], start=2):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split()
        try:
            if parts[0] == "KERNEL":
                kv = dict(p.split("=", 1) for p in parts[2:])
                cur = KernelDescriptor(parts[1], profiled_latency_s=float(kv["latency"]),
                                       unpredictable_fraction=float(kv["unpredictable"]))
                descs[parts[1]] = cur
            elif parts[0] == "RULE":
                if cur is None:
                    raise DescriptorError("RULE before KERNEL")
                kv = dict(p.split("=", 1) for p in parts[1:])
                ex = {k: LinearExpr.parse(kv[k]) for k in ("size", "stride", "chunk", "count") if k in kv}
                cur.rules.append(TemplateRule(int(kv["ptr"]), kv["kind"], int(kv.get("offset", "0")), **ex))
            else:
                raise DescriptorError(f"unknown record {parts[0]!r}")
        except (KeyError, ValueError) as e:
            raise DescriptorError(f"{path}:{lineno}: {e}") from e
    return descs
