"""Ad-hoc GPU diagnostics: facade known answers, randomized list ops vs the
oracle, and first-divergence search on a golden case.  Run on the GPU box."""

import random
import sys
import traceback

sys.path.insert(0, ".")

from oracle import msched_port as port  # noqa: E402
from paper_2512_24637_b200 import engine  # noqa: E402
from paper_2512_24637_b200.memman import EvictionList  # noqa: E402
from paper_2512_24637_b200.model import HwConfig, PageSet  # noqa: E402
from paper_2512_24637_b200.scheduler import Policy  # noqa: E402
from tests.golden import loader  # noqa: E402


def mk(pages):
    ev = EvictionList(domain_pages=4096)
    for p in pages:
        ev.append_tail([(p, p + 1)])
    return ev


def facade():
    ev = mk([10, 20, 30, 40])
    ev.madvise(PageSet.from_pages([40, 20]))
    print("madvise", ev.pages_in_order(), "want [10, 30, 20, 40]")
    ev = mk([5, 6, 7, 1, 2])
    print("evict", ev.evict_head(3), ev.pages_in_order(), "want [(5,8)] [1,2]")
    ev = mk([1, 2, 3, 4, 5])
    ev.remove(PageSet.from_pages([2, 4]))
    print("remove", ev.pages_in_order(), len(ev), "want [1,3,5] 3")


def randomized(n_iter=200):
    rng = random.Random(7)
    bad = 0
    for it in range(n_iter):
        ev = EvictionList(domain_pages=20000)
        rl = port.RunList()
        for step in range(20):
            op = rng.random()
            if op < 0.35:
                a = rng.randrange(0, 19000)
                b = a + rng.randrange(1, 600)
                runs = [r for r in port.runs_sub(((a, b),), rl.resident)]
                ev.append_tail(runs)
                rl.append(runs)
            elif op < 0.7:
                k = rng.randrange(1, 6)
                runs = port.norm_runs([(x, x + rng.randrange(1, 400)) for x in
                                       (rng.randrange(0, 19000) for _ in range(k))])
                ev.madvise(PageSet(runs))
                rl.advise(runs)
            elif op < 0.85:
                n = rng.randrange(0, 800)
                g = [p for a, b in ev.evict_head(n) for p in range(a, b)]
                w = port.runs_pages(rl.pop_head(n))
                if g != w:
                    print("evict mismatch", it, step)
                    bad += 1
            else:
                k = rng.randrange(1, 4)
                runs = port.norm_runs([(x, x + rng.randrange(1, 2000)) for x in
                                       (rng.randrange(0, 19000) for _ in range(k))])
                ev.remove(PageSet(runs))
                rl.drop(runs)
            if ev.pages_in_order() != rl.order():
                print("order mismatch", it, step, op, len(ev), len(rl))
                bad += 1
                break
        ev.ctx.close()
    print("randomized list ops: bad =", bad)


def first_divergence(name, mode):
    case = loader.sim_case(name)
    tasks = [loader.dec_task(t) for t in case["tasks"]]
    tasks, feeder = loader.feeder_for(case["feeder"], tasks)
    run = case["runs"][mode]
    hw = HwConfig(**case["hw"])
    pol = Policy(**case["policy"])
    rec_g, rec_o = [], []
    sim = engine.Simulator(tasks, hw, pol, engine.Mode(**run["mode"]), feeder=feeder, recorder=rec_g)
    try:
        sim.run()
    except Exception:
        traceback.print_exc()
    ptasks = [loader.dec_task(t) for t in case["tasks"]]
    ptasks, pfeeder = loader.feeder_for(case["feeder"], ptasks)
    psim = port.PortSim(ptasks, loader.ns(case["hw"]), loader.ns(case["policy"]), loader.ns(run["mode"]),
                        feeder=pfeeder, recorder=rec_o)
    try:
        psim.run()
    except Exception:
        traceback.print_exc()
    g = loader.canon_records(rec_g)
    o = loader.canon_records(rec_o)
    for i, (a, b) in enumerate(zip(g, o)):
        if a != b:
            print(f"{name}/{mode}: first divergence at record {i}")
            for k in sorted(set(a) | set(b)):
                if a.get(k) != b.get(k):
                    print("  ", k, "gpu:", str(a.get(k))[:300], "\n     oracle:", str(b.get(k))[:300])
            return
    print(f"{name}/{mode}: {len(g)} gpu records vs {len(o)} oracle records, no divergence in common prefix")


if __name__ == "__main__":
    facade()
    randomized(int(sys.argv[1]) if len(sys.argv) > 1 else 50)
    for spec in sys.argv[2:]:
        n, m = spec.split(":")
        first_divergence(n, m)
