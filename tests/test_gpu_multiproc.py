"""The multi-rank path with the GPU engine: two ranks
(gloo; both on the one visible B200, as the round's boxes have one GPU) each
replay their own tenant mix through the CUDA path with real migration, check
it against the oracle, and reduce time and pages the way bench.py does."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


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
    from paper_2512_24637_b200 import engine
    from paper_2512_24637_b200.scenarios import llm_mix
    from paper_2512_24637_b200.scheduler import Policy

    tasks, hw, _ = llm_mix(2, 6, 60 * 4096 * 6, 8 * 4096 * 6, 3, 512 * 4096, task_offset=2 * rank)
    pol = Policy("rr", 2e-6)
    sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), migrate=True, verify=True, device=0)
    try:
        m = sim.run()
        bad = sim.ctx.verify()
    finally:
        sim.close()
    ref = port_mod.PortSim(tasks, hw, pol, engine.Mode.proactive()).run()
    keys = ("migrated_in_pages", "migrated_out_pages", "fault_pages", "total_time_s")
    same = {k: getattr(m, k) for k in keys} == {k: getattr(ref, k) for k in keys}
    pages = m.planned_pages
    tmax = bench.max_over_ranks(torch, float(10 + rank), world, "cpu")
    psum = bench.sum_over_ranks(torch, pages, world, "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, (same, bad, pages))
    if rank == 0:
        out.put((tmax, psum, gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_replay_their_shards_on_the_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, psum, gathered = q.get(timeout=540)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(same for same, _, _ in gathered)           # each shard equals the oracle
    assert all(bad == 0 for _, bad, _ in gathered)        # migrated payloads intact on both ranks
    assert tmax == 11.0 and psum == sum(p for _, _, p in gathered) > 0
