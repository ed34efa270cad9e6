"""Multi-GPU plumbing on CPU (gloo, world_size 2): the path shards into
independent per-GPU tenant mixes; ranks never exchange
data, only the benchmark's max-over-ranks time and summed page counts.
Each rank replays its own shard with the CPU oracle here (no GPU), which
exercises the same sharding and reduction code bench.py uses."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import msched_port as port_mod
    from paper_2512_24637_b200.engine import Mode
    from paper_2512_24637_b200.presets import get_preset
    from paper_2512_24637_b200.scenarios import llm_mix

    tasks, hw, pol = llm_mix(2, 6, 60 * 4096 * 6, 8 * 4096 * 6, 3, 512 * 4096, task_offset=2 * rank)
    ids = [t.id for t in tasks]
    bases = [a.base_addr for t in tasks for a in t.allocations]
    from paper_2512_24637_b200.scheduler import Policy
    m = port_mod.PortSim(tasks, hw, Policy("rr", 2e-6), Mode.proactive()).run()
    pages = m.migrated_in_pages + m.migrated_out_pages + m.fault_pages
    t = float(10 + rank)
    tmax = bench.max_over_ranks(torch, t, world, "cpu")
    psum = bench.sum_over_ranks(torch, pages, world, "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, (ids, min(bases), max(bases), pages))
    if rank == 0:
        out.put((tmax, psum, gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharding_and_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, psum, gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (ids0, lo0, hi0, p0), (ids1, lo1, hi1, p1) = gathered
    assert not set(ids0) & set(ids1)                      # distinct tenants per GPU
    assert hi0 < lo1                                      # disjoint address windows
    assert tmax == 11.0                                   # max over ranks, not mean
    assert psum == p0 + p1 and p0 == p1 > 0               # identical shards, summed work
