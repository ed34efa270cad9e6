"""Config-3 trace generators: stencil, SpMV and ResNet-style training.

SURVEY.md §8(d) config 3 ("mixed scientific + DL kernel-launch traces at 2x")
has no generator in the reference.  These emit ordinary reference-shaped
`Task`/`Command` objects (MSIM-TRACE v1 compatible), built the way the
reference's own generators are (workload.py:23-412), so the reference
simulator, the CPU oracle and the GPU path can all replay them.  They
exercise what the LLM traces do not:

  * strided (T3) halo-band rules and pointer swapping (stencil);
  * indirect, unpredictable accesses that only the fault fallback serves
    (SpMV's gather from x, planted like workload.py:70-74);
  * one pooled allocation sliced per layer, forward then reverse-order
    backward, activations linear in a batch argument (T2) that changes
    between iterations (ResNet-style training).
"""

from __future__ import annotations

import random

from .model import Allocation, Arg, ByteRange, Command, CommandKind, Task
from .presets import GIB, get_preset
from .scheduler import Policy
from .workload import DEFAULT_FLOPS, DEFAULT_H2D_BW, DEFAULT_MEM_BW, _Bump, _seed_copies, task_base_addr

__all__ = ["gen_stencil", "gen_spmv", "gen_resnet_training", "config3_mixed"]


def _kernel(name, lat, args, access, grid=(1, 1, 1), block=(1, 1, 1)):
    return Command(kind=CommandKind.KERNEL, kernel_name=name, latency_s=lat, launch_args=tuple(args),
                   grid_dims=grid, block_dims=block, ground_truth_access=tuple(access))


def gen_stencil(rows: int, cols: int, iterations: int, *, task_id: str = "stencil", base_addr: int = 1 << 40,
                mem_bw: float = DEFAULT_MEM_BW, h2d_bw: float = DEFAULT_H2D_BW, page_size: int = 4096,
                halo_bands=(4, 8)) -> Task:
    """Hotspot-style 2-D stencil: in/out grids swapped every iteration plus a
    power grid, and a halo-exchange kernel touching `nbands` strided bands of
    two rows each (strided rule whose count follows a 32-bit argument)."""
    bump = _Bump(base_addr, page_size)
    nbytes = rows * cols * 4
    task = Task(id=task_id)
    grids = [Allocation(f"{task_id}.{nm}", bump.take(nbytes), nbytes, task_id) for nm in ("a", "b", "power")]
    task.allocations.extend(grids)
    _seed_copies(task, h2d_bw)
    src, dst, power = grids
    row_bytes = cols * 4
    for it in range(iterations):
        task.commands.append(_kernel(
            "hotspot", 3 * nbytes / mem_bw,
            [Arg(src.base_addr, 64), Arg(dst.base_addr, 64), Arg(power.base_addr, 64), Arg(rows, 32), Arg(cols, 32)],
            [ByteRange(src.base_addr, nbytes), ByteRange(dst.base_addr, nbytes), ByteRange(power.base_addr, nbytes)],
            grid=(-(-cols // 16), -(-rows // 16), 1), block=(16, 16, 1)))
        nb = halo_bands[it % len(halo_bands)]
        stride = (rows // nb) * row_bytes
        task.commands.append(_kernel(
            "halo", nb * 2 * row_bytes / mem_bw,
            [Arg(dst.base_addr, 64), Arg(nb, 32), Arg(2 * cols, 32)],
            [ByteRange(dst.base_addr + j * stride, 2 * row_bytes) for j in range(nb)]))
        src, dst = dst, src
    task.validate()
    return task


def gen_spmv(nrows: int, nnz_per_row: int, iterations: int, *, indirect_pages: int = 4, gathers: int = 6,
             task_id: str = "spmv", base_addr: int = 1 << 40, mem_bw: float = DEFAULT_MEM_BW,
             h2d_bw: float = DEFAULT_H2D_BW, page_size: int = 4096, seed: int = 0) -> Task:
    """CSR SpMV y = A x.  row_ptr, col_idx, vals and y follow fixed rules;
    x is reached only through col_idx, so its pages are scattered, not
    derivable from any argument, and served by the fault fallback."""
    bump = _Bump(base_addr, page_size)
    nnz = nrows * nnz_per_row
    task = Task(id=task_id)
    sizes = {"row_ptr": 4 * (nrows + 1), "col_idx": 4 * nnz, "vals": 4 * nnz, "x": 4 * nrows, "y": 4 * nrows}
    al = {k: Allocation(f"{task_id}.{k}", bump.take(v), v, task_id) for k, v in sizes.items()}
    task.allocations.extend(al.values())
    _seed_copies(task, h2d_bw)
    rng = random.Random(seed)
    x_pages = sizes["x"] // page_size
    lat = (sizes["row_ptr"] + sizes["col_idx"] + sizes["vals"] + sizes["y"]) / mem_bw
    for _ in range(iterations):
        access = [ByteRange(al[k].base_addr, sizes[k]) for k in ("row_ptr", "col_idx", "vals", "y")]
        for _ in range(gathers):
            off = rng.randrange(0, max(1, x_pages - indirect_pages + 1))
            access.append(ByteRange(al["x"].base_addr + off * page_size + 8,
                                    min(indirect_pages * page_size, sizes["x"]) - 16))
        task.commands.append(_kernel(
            "spmv_csr", lat,
            [Arg(al["row_ptr"].base_addr, 64), Arg(al["col_idx"].base_addr, 64), Arg(al["vals"].base_addr, 64),
             Arg(al["x"].base_addr + 4, 64), Arg(al["y"].base_addr, 64), Arg(nrows, 32), Arg(nnz, 32)],
            access, grid=(-(-nrows // 256), 1, 1), block=(256, 1, 1)))
    task.validate()
    return task


def gen_resnet_training(layer_weights, layer_acts, iterations: int, batches=(32, 64), *, task_id: str = "resnet",
                        base_addr: int = 1 << 40, flops: float = DEFAULT_FLOPS, h2d_bw: float = DEFAULT_H2D_BW,
                        page_size: int = 4096) -> Task:
    """Training loop over pooled buffers: one weight pool and one gradient
    pool sliced per layer, one activation pool whose per-layer slices scale
    with the batch argument.  Forward in layer order, backward in reverse,
    then an SGD step over the whole weight and gradient pools."""
    L = len(layer_weights)
    bmax = max(batches)
    bump = _Bump(base_addr, page_size)
    task = Task(id=task_id)
    wtot = sum(layer_weights)
    atot = sum(layer_acts) * bmax
    wpool = Allocation(f"{task_id}.weights", bump.take(wtot), wtot, task_id)
    gpool = Allocation(f"{task_id}.grads", bump.take(wtot), wtot, task_id)
    apool = Allocation(f"{task_id}.acts", bump.take(atot), atot, task_id)
    task.allocations.extend([wpool, gpool, apool])
    _seed_copies(task, h2d_bw)
    woff = [sum(layer_weights[:i]) for i in range(L)]
    aoff = [sum(layer_acts[:i]) * bmax for i in range(L)]
    for it in range(iterations):
        b = batches[it % len(batches)]
        for l in range(L):
            act = layer_acts[l] * b
            task.commands.append(_kernel(
                f"fwd{l % 4}", 2.0 * layer_weights[l] * b / flops + act / DEFAULT_MEM_BW,
                [Arg(wpool.base_addr + woff[l], 64), Arg(apool.base_addr + aoff[l], 64), Arg(b, 32),
                 Arg(layer_acts[l], 32)],
                [ByteRange(wpool.base_addr + woff[l], layer_weights[l]), ByteRange(apool.base_addr + aoff[l], act)]))
        for l in reversed(range(L)):
            act = layer_acts[l] * b
            task.commands.append(_kernel(
                f"bwd{l % 4}", 4.0 * layer_weights[l] * b / flops + act / DEFAULT_MEM_BW,
                [Arg(wpool.base_addr + woff[l], 64), Arg(gpool.base_addr + woff[l], 64),
                 Arg(apool.base_addr + aoff[l], 64), Arg(b, 32), Arg(layer_acts[l], 32)],
                [ByteRange(wpool.base_addr + woff[l], layer_weights[l]),
                 ByteRange(gpool.base_addr + woff[l], layer_weights[l]), ByteRange(apool.base_addr + aoff[l], act)]))
        task.commands.append(_kernel(
            "sgd", 2 * wtot / DEFAULT_MEM_BW, [Arg(wpool.base_addr, 64), Arg(gpool.base_addr, 64)],
            [ByteRange(wpool.base_addr, wtot), ByteRange(gpool.base_addr, wtot)]))
    task.validate()
    return task


def config3_mixed(hbm_bytes: int = 96 << 20, ratio: float = 2.0, page_size: int = 4096, task_offset: int = 0,
                  timeslice_s: float = 1e-3, seed: int = 0):
    """Config 3: stencil + SpMV + ResNet-style training (+ a second stencil)
    whose allocations total `ratio` x the HBM budget."""
    per = ratio * hbm_bytes / 4
    pg = page_size
    side = max(64, int((per / 3 / 4) ** 0.5) // 16 * 16)
    nrows = max(1024, int(per / (4 * (2 * 8 + 3))) // 1024 * 1024)
    lw = [max(pg, int(per * 0.25 / 8) // pg * pg)] * 8
    la = [max(pg, int(per * 0.25 / 8 / 64) // pg * pg)] * 8
    tasks = [
        gen_stencil(side, side, 6, task_id=f"hotspot{task_offset}", base_addr=task_base_addr(task_offset), page_size=pg),
        gen_spmv(nrows, 8, 6, task_id=f"spmv{task_offset + 1}", base_addr=task_base_addr(task_offset + 1),
                 page_size=pg, seed=seed),
        gen_resnet_training(lw, la, 2, task_id=f"resnet{task_offset + 2}", base_addr=task_base_addr(task_offset + 2),
                            page_size=pg),
        gen_stencil(side // 2 * 2, side, 8, task_id=f"stencil{task_offset + 3}",
                    base_addr=task_base_addr(task_offset + 3), page_size=pg, halo_bands=(2, 4, 8)),
    ]
    hw = get_preset("rtx5080").with_capacity(hbm_bytes)
    import dataclasses

    hw = dataclasses.replace(hw, page_size_bytes=pg, dram_capacity_bytes=max(256 * GIB, 4 * hbm_bytes))
    return tasks, hw, Policy("rr", timeslice_s)


def gen_scatter(npages: int, k: int, ncmds: int, *, task_id: str, base_addr: int, page_size: int = 4096,
                seed: int = 0, latency_s: float = 50e-6) -> Task:
    """One allocation of `npages` pages; every command touches `k` distinct
    pages drawn with `random.Random(seed)` (SURVEY.md Appendix B's fragmented
    probe: scattered single pages, one run per page in the eviction list)."""
    rng = random.Random(seed)
    pg = page_size
    cmds = []
    for _ in range(ncmds):
        pages = rng.sample(range(npages), k)
        cmds.append(Command(kind=CommandKind.KERNEL, latency_s=latency_s, kernel_name="scatter",
                            launch_args=(Arg(base_addr, 64), Arg(k, 32)),
                            ground_truth_access=tuple(ByteRange(base_addr + p * pg, pg) for p in pages)))
    return Task(id=task_id, allocations=[Allocation(f"{task_id}.a", base_addr, npages * pg, task_id)],
                commands=cmds)


def fragmented_mix(n_tasks: int = 4, npages: int = 1 << 20, k: int = 16, ncmds: int = 8192,
                   capacity_pages: int = 1 << 18, page_size: int = 4096, task_offset: int = 0,
                   timeslice_s: float = 1e-3):
    """The fragmented regime the reference collapses on (SURVEY.md §0 fact 4,
    Appendix B), scaled up: `n_tasks` tasks of `npages`-page allocations,
    `k` scattered single pages per command, against `capacity_pages` frames.
    Defaults: 4 x 2^20 pages, 16 pages/command, 8192 commands per task
    (524 K page touches, twice the 2^18-frame capacity), RR 1 ms, 4 KiB pages.
    Replayed with Mode.ideal() as in the probe."""
    import dataclasses

    tasks = [gen_scatter(npages, k, ncmds, task_id=f"f{i + task_offset}", base_addr=task_base_addr(i + task_offset),
                         page_size=page_size, seed=i + task_offset) for i in range(n_tasks)]
    hw = dataclasses.replace(get_preset("rtx5080"), hbm_capacity_bytes=capacity_pages * page_size,
                             page_size_bytes=page_size,
                             dram_capacity_bytes=max(256 * GIB, 2 * n_tasks * npages * page_size))
    return tasks, hw, Policy("rr", timeslice_s)
