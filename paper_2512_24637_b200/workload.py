"""Synthetic trace producers and the MSIM-TRACE v1 text format.

Input side of the hot path (SURVEY.md §8(d) configs are built from these).
Each generator reproduces the reference generator of the same name
(workload.py:23-412) command-for-command — pinned by
tests/test_host_golden.py against trace texts the reference wrote — so the
GPU path and the CPU oracle replay identical inputs.
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

from .model import Allocation, Arg, ByteRange, Command, CommandKind, Task

__all__ = [
    "TRACE_HEADER", "DEFAULT_MEM_BW", "DEFAULT_FLOPS", "DEFAULT_H2D_BW", "KV_ROW_BYTES",
    "TraceError", "task_base_addr", "gen_vector_add", "gen_matmul", "gen_llm_like",
    "decode_step_commands", "PlantedKernel", "PlantedCorpus", "gen_template_corpus",
    "format_trace", "save_trace", "parse_trace", "load_trace",
]

TRACE_HEADER = "MSIM-TRACE v1"
DEFAULT_MEM_BW = 8.5e9 / 12.7e-3      # an 8.5 GB sweep in 12.7 ms
DEFAULT_FLOPS = 50e12
DEFAULT_H2D_BW = 41.7e9
ADDRESS_SPACE_BITS = 56
KV_ROW_BYTES = 256


class TraceError(ValueError):
    pass


class _Bump:
    """Page-granular bump allocator (workload.py:38-51)."""

    def __init__(self, base: int, page: int):
        self.next = base
        self.page = page

    def take(self, size: int) -> int:
        at = self.next
        self.next += -(-size // self.page) * self.page
        if self.next >= 1 << ADDRESS_SPACE_BITS:
            raise OverflowError("simulated address space exhausted")
        return at


def task_base_addr(index: int) -> int:
    """1 TiB apart (workload.py:54-56)."""
    return (index + 1) << 40


def _seed_copies(task: Task, h2d_bw: float):
    """One H2D upload per allocation, at the link rate (workload.py:59-67)."""
    for a in task.allocations:
        task.commands.append(Command(
            kind=CommandKind.MEMCPY_H2D, latency_s=a.size_bytes / h2d_bw,
            launch_args=(Arg(0, 64), Arg(a.base_addr, 64), Arg(a.size_bytes, 64))))


def _indirect_region(rng, scratch: Allocation, n_pages: int, page: int) -> ByteRange:
    hi = scratch.size_bytes // page - n_pages
    return ByteRange(scratch.base_addr + rng.randrange(0, hi + 1) * page, n_pages * page)


def _scratch(task, bump, rate, page, tid):
    if rate <= 0:
        return None
    a = Allocation(f"{tid}.scratch", bump.take(256 * page), 256 * page, tid)
    task.allocations.append(a)
    return a


def _indirect_pages(base_bytes: int, rate: float, page: int) -> int:
    return max(1, round(-(-base_bytes // page) * rate / (1.0 - rate)))


def gen_vector_add(n_elems: int, elem_bytes: int = 4, iterations: int = 1, *,
                   task_id: str = "va", base_addr: int = 1 << 40,
                   mem_bw: float = DEFAULT_MEM_BW, h2d_bw: float = DEFAULT_H2D_BW,
                   kernel_name: str = "vector_add", indirect_rate: float = 0.0,
                   seed: int = 0, page_size: int = 4096) -> Task:
    """Streaming kernel over A, B, C; args [A, B, C, N] (workload.py:76-126)."""
    if n_elems <= 0:
        raise ValueError("n_elems must be positive")
    bump = _Bump(base_addr, page_size)
    nbytes = n_elems * elem_bytes
    task = Task(id=task_id)
    bufs = [Allocation(f"{task_id}.{nm}", bump.take(nbytes), nbytes, task_id) for nm in "ABC"]
    task.allocations.extend(bufs)
    scratch = _scratch(task, bump, indirect_rate, page_size, task_id)
    _seed_copies(task, h2d_bw)
    rng = random.Random(seed)
    for _ in range(iterations):
        touched = [ByteRange(b.base_addr, nbytes) for b in bufs]
        if scratch is not None:
            touched.append(_indirect_region(
                rng, scratch, _indirect_pages(3 * nbytes, indirect_rate, page_size), page_size))
        task.commands.append(Command(
            kind=CommandKind.KERNEL, kernel_name=kernel_name, latency_s=3 * nbytes / mem_bw,
            launch_args=tuple(Arg(b.base_addr, 64) for b in bufs) + (Arg(n_elems, 64),),
            grid_dims=(-(-n_elems // 256), 1, 1), block_dims=(256, 1, 1),
            ground_truth_access=tuple(touched)))
    task.validate()
    return task


def gen_matmul(m: int, n: int, k: int, count: int = 1, *, elem_bytes: int = 4,
               task_id: str = "mm", base_addr: int = 1 << 40, flops: float = DEFAULT_FLOPS,
               h2d_bw: float = DEFAULT_H2D_BW, kernel_name: str = "matmul",
               page_size: int = 4096) -> Task:
    """`count` GEMMs over fixed A, B, C; args [A, B, C, M, N, K]
    (workload.py:145-193)."""
    if min(m, n, k) <= 0:
        raise ValueError("dimensions must be positive")
    bump = _Bump(base_addr, page_size)
    sizes = (m * k * elem_bytes, k * n * elem_bytes, m * n * elem_bytes)
    task = Task(id=task_id)
    for nm, sz in zip("ABC", sizes):
        task.allocations.append(Allocation(f"{task_id}.{nm}", bump.take(sz), sz, task_id))
    _seed_copies(task, h2d_bw)
    ptrs = tuple(Arg(a.base_addr, 64) for a in task.allocations)
    touched = tuple(ByteRange(a.base_addr, sz) for a, sz in zip(task.allocations, sizes))
    for _ in range(count):
        task.commands.append(Command(
            kind=CommandKind.KERNEL, kernel_name=kernel_name, latency_s=2.0 * m * n * k / flops,
            launch_args=ptrs + (Arg(m, 32), Arg(n, 32), Arg(k, 32)),
            grid_dims=(-(-m // 16), -(-n // 16), 1), block_dims=(16, 16, 1),
            ground_truth_access=touched))
    task.validate()
    return task


def gen_llm_like(layers: int, weight_bytes_per_layer: int, kv_max_bytes: int,
                 decode_steps: int, kv_used_fraction_schedule: list, *,
                 task_id: str = "llm", base_addr: int = 1 << 40,
                 mem_bw: float = DEFAULT_MEM_BW, h2d_bw: float = DEFAULT_H2D_BW,
                 kernel_name: str = "decode_layer", page_size: int = 4096) -> Task:
    """Decode loop: one monolithic weight buffer sliced per layer plus per-layer
    KV buffers touched up to the live prefix (workload.py:199-241)."""
    if len(kv_used_fraction_schedule) != decode_steps:
        raise ValueError("schedule length must equal decode_steps")
    prev = 0.0
    for f in kv_used_fraction_schedule:
        if not 0.0 < f <= 1.0 or f < prev:
            raise ValueError("fractions must be in (0, 1] and non-decreasing")
        prev = f
    bump = _Bump(base_addr, page_size)
    task = Task(id=task_id)
    wbytes = layers * weight_bytes_per_layer
    task.allocations.append(Allocation(f"{task_id}.weights", bump.take(wbytes), wbytes, task_id))
    for i in range(layers):
        task.allocations.append(
            Allocation(f"{task_id}.kv{i}", bump.take(kv_max_bytes), kv_max_bytes, task_id))
    _seed_copies(task, h2d_bw)
    task.commands.extend(decode_step_commands(
        task, kv_used_fraction_schedule, weight_bytes_per_layer, kv_max_bytes,
        mem_bw=mem_bw, kernel_name=kernel_name))
    task.validate()
    return task


def decode_step_commands(task: Task, fraction_schedule: list, weight_bytes_per_layer: int,
                         kv_max_bytes: int, *, mem_bw: float = DEFAULT_MEM_BW,
                         kernel_name: str = "decode_layer") -> list:
    """workload.py:244-282: per step, one kernel per layer with a 32-bit
    seq_len argument driving the KV extent."""
    weights = task.allocations[0]
    kvs = [a for a in task.allocations[1:] if ".kv" in a.id]
    out = []
    for frac in fraction_schedule:
        seq_len = max(1, int(frac * kv_max_bytes) // KV_ROW_BYTES)
        used = seq_len * KV_ROW_BYTES
        for i, kv in enumerate(kvs):
            ptr = weights.base_addr + i * weight_bytes_per_layer
            out.append(Command(
                kind=CommandKind.KERNEL, kernel_name=kernel_name,
                latency_s=(weight_bytes_per_layer + used) / mem_bw,
                launch_args=(Arg(ptr, 64), Arg(kv.base_addr, 64), Arg(seq_len, 32)),
                ground_truth_access=(ByteRange(ptr, weight_bytes_per_layer),
                                     ByteRange(kv.base_addr, used))))
    return out


@dataclass
class PlantedKernel:
    name: str
    kind: str
    rule_page_counts: list = field(default_factory=list)
    indirect_page_counts: list = field(default_factory=list)
    coeff: int = 0
    arg_indices: tuple = ()
    fixed_size: int = 0


@dataclass
class PlantedCorpus:
    task: Task
    kernels: dict

    def expected_fneg(self, name: str) -> float:
        pk = self.kernels[name]
        rates = [ind / (ind + r) for r, ind in zip(pk.rule_page_counts, pk.indirect_page_counts)]
        return sum(rates) / len(rates)


def _corpus_cmd(name, args, access):
    return Command(kind=CommandKind.KERNEL, kernel_name=name, latency_s=10e-6,
                   launch_args=args, ground_truth_access=tuple(access))


def _plant(rng, access, scratch, rule_pages, flagged, page) -> int:
    if not flagged:
        return 0
    n = max(1, rule_pages // 32)
    access.append(_indirect_region(rng, scratch, n, page))
    return n


def gen_template_corpus(n_kernels: int = 60, records_per: int = 4,
                        indirect_rate: float = 0.0025, seed: int = 0,
                        page_size: int = 4096, task_id: str = "corpus") -> PlantedCorpus:
    """Planted fixed / linear / strided rules with an indirect fraction
    (workload.py:311-400).  The RNG call sequence is the reference's."""
    rng = random.Random(seed)
    bump = _Bump(task_base_addr(0), page_size)
    task = Task(id=task_id)
    scratch = Allocation(f"{task_id}.scratch", bump.take(4096 * page_size), 4096 * page_size, task_id)
    task.allocations.append(scratch)
    kernels = {}
    for ki in range(n_kernels):
        kind = ("fixed", "linear", "strided")[ki % 3]
        name = f"{kind}_k{ki}"
        pk = PlantedKernel(name=name, kind=kind)
        flagged = rng.random() < 12 * indirect_rate

        def record(args, access, rule_pages):
            pk.rule_page_counts.append(rule_pages)
            pk.indirect_page_counts.append(_plant(rng, access, scratch, rule_pages, flagged, page_size))
            task.commands.append(_corpus_cmd(name, args, access))

        if kind == "fixed":
            size = rng.randrange(1, 9) * page_size
            buf = Allocation(f"{task_id}.{name}", bump.take(size), size, task_id)
            task.allocations.append(buf)
            pk.fixed_size = size
            for _ in range(records_per):
                args = (Arg(buf.base_addr, 64), Arg(rng.randrange(1, 1000), 32))
                record(args, [ByteRange(buf.base_addr, size)], size // page_size)
        elif kind == "linear":
            coeff = rng.choice([2, 4, 8, 16])
            width = rng.choice([32, 64])
            max_n = 4 * page_size // coeff
            buf = Allocation(f"{task_id}.{name}", bump.take(coeff * max_n), coeff * max_n, task_id)
            task.allocations.append(buf)
            pk.coeff, pk.arg_indices = coeff, (1,)
            for _ in range(records_per):
                n = rng.randrange(page_size // coeff, max_n + 1)
                record((Arg(buf.base_addr, 64), Arg(n, width)), [ByteRange(buf.base_addr, coeff * n)],
                       -(-(coeff * n) // page_size))
        else:
            ccoeff = rng.choice([4, 8])
            stride = 4 * page_size
            max_count = 8
            span = stride * max_count
            buf = Allocation(f"{task_id}.{name}", bump.take(span), span, task_id)
            task.allocations.append(buf)
            pk.coeff, pk.arg_indices = ccoeff, (1, 2)
            for _ in range(records_per):
                count = rng.randrange(2, max_count + 1)
                elems = rng.randrange(page_size // (2 * ccoeff), page_size // ccoeff + 1)
                chunk = ccoeff * elems
                access = [ByteRange(buf.base_addr + j * stride, chunk) for j in range(count)]
                record((Arg(buf.base_addr, 64), Arg(count, 32), Arg(elems, 32)), access,
                       count * -(-chunk // page_size))
        kernels[name] = pk
    task.validate()
    return PlantedCorpus(task, kernels)


# ---------------------------------------------------------------------------
# MSIM-TRACE v1 (workload.py:419-580)


def _arg_text(a: Arg) -> str:
    return f"raw:{a.raw.hex()}" if a.raw is not None else f"{a.width}:{a.value}"


def format_trace(task: Task) -> str:
    lines = [TRACE_HEADER, f"TASK {task.id}"]
    lines += [f"ALLOC {a.id} {a.base_addr} {a.size_bytes}" for a in task.allocations]
    for c in task.commands:
        if c.kind is CommandKind.KERNEL:
            args = ",".join(_arg_text(a) for a in c.launch_args)
            acc = ",".join(f"({r.start_addr},{r.length_bytes})" for r in c.ground_truth_access)
            ln = f"KERNEL {c.kernel_name} {c.latency_s!r} args=[{args}] access=[{acc}]"
            if tuple(c.grid_dims) != (1, 1, 1) or tuple(c.block_dims) != (1, 1, 1):
                g, b = c.grid_dims, c.block_dims
                ln += f" grid=({g[0]},{g[1]},{g[2]}) block=({b[0]},{b[1]},{b[2]})"
            lines.append(ln)
        else:
            d = "H2D" if c.kind is CommandKind.MEMCPY_H2D else "D2H"
            lines.append(f"MEMCPY {d} {c.memcpy_src} {c.memcpy_dst} {c.memcpy_size} {c.latency_s!r}")
    return "\n".join(lines) + "\n"


def save_trace(task: Task, path: str):
    with open(path, "w", encoding="utf-8") as f:
        f.write(format_trace(task))


def load_trace(path: str) -> Task:
    try:
        with open(path, encoding="utf-8") as f:
            text = f.read()
    except OSError as e:
        raise TraceError(f"cannot read trace {path!r}: {e}") from e
    return parse_trace(text, source=path)


def _bracketed(s: str) -> str:
    if not (s.startswith("[") and s.endswith("]")):
        raise ValueError(f"expected bracketed list, got {s!r}")
    return s[1:-1]


def _top_level_items(s: str) -> list:
    """Split on commas outside parentheses."""
    items, depth, cur = [], 0, []
    for ch in s:
        depth += (ch == "(") - (ch == ")")
        if ch == "," and depth == 0:
            if cur:
                items.append("".join(cur))
            cur = []
        else:
            cur.append(ch)
    if cur:
        items.append("".join(cur))
    return items


def _parse_arg(tok: str) -> Arg:
    kind, val = tok.split(":", 1)
    if kind == "raw":
        return Arg(0, 64, raw=bytes.fromhex(val))
    return Arg(int(val), int(kind))


def _parens(tok: str, n: int, what: str) -> list:
    if not (tok.startswith("(") and tok.endswith(")")):
        raise ValueError(f"expected {what}, got {tok!r}")
    parts = tok[1:-1].split(",")
    if len(parts) != n:
        raise ValueError(f"expected {what}, got {tok!r}")
    return [int(p) for p in parts]


def _parse_line(task: Task, line: str):
    parts = line.split()
    tag = parts[0]
    if tag == "TASK":
        task.id = parts[1]
        task.allocations = [Allocation(a.id, a.base_addr, a.size_bytes, task.id) for a in task.allocations]
    elif tag == "ALLOC":
        task.allocations.append(Allocation(parts[1], int(parts[2]), int(parts[3]), task.id))
    elif tag == "KERNEL":
        name, lat = parts[1], float(parts[2])
        kv = dict(p.split("=", 1) for p in parts[3:])
        inner = _bracketed(kv.get("args", "[]"))
        args = tuple(_parse_arg(t) for t in inner.split(",") if t) if inner else ()
        acc = tuple(ByteRange(*_parens(t, 2, "(start,len)"))
                    for t in _top_level_items(_bracketed(kv.get("access", "[]"))))
        task.commands.append(Command(
            kind=CommandKind.KERNEL, kernel_name=name, latency_s=lat, launch_args=args,
            grid_dims=tuple(_parens(kv.get("grid", "(1,1,1)"), 3, "(x,y,z)")),
            block_dims=tuple(_parens(kv.get("block", "(1,1,1)"), 3, "(x,y,z)")),
            ground_truth_access=acc))
    elif tag == "MEMCPY":
        d, src, dst, size, lat = parts[1], int(parts[2]), int(parts[3]), int(parts[4]), float(parts[5])
        if d not in ("H2D", "D2H"):
            raise ValueError(f"bad memcpy direction {d!r}")
        task.commands.append(Command(
            kind=CommandKind.MEMCPY_H2D if d == "H2D" else CommandKind.MEMCPY_D2H, latency_s=lat,
            launch_args=(Arg(src, 64), Arg(dst, 64), Arg(size, 64))))
    else:
        raise ValueError(f"unknown record type {tag!r}")


def parse_trace(text: str, source: str = "<string>") -> Task:
    lines = text.splitlines()
    if not lines or lines[0].strip() != TRACE_HEADER:
        raise TraceError(f"{source}:1: missing '{TRACE_HEADER}' header")
    task = Task(id="trace")
    for lineno, raw in enumerate(lines[1:], start=2):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        try:
            _parse_line(task, line)
        except (ValueError, IndexError) as e:
            raise TraceError(f"{source}:{lineno}: {e}") from e
    try:
        task.validate()
    except ValueError as e:
        raise TraceError(f"{source}: {e}") from e
    return task
