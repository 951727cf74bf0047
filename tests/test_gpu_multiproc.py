"""Population sharding (SURVEY §8e, C4 pattern) with two real processes on one
B200: each rank owns half of the children, exchanges its top-K entries every
generation through gloo (host copies), and the result must equal the
unsharded solve bit for bit (global rows in the selection keys, global child
indices in the RNG counters).  The reference's analogue is worker-count
determinism (K/bench.py:688-705, TST/test_bench.py:257-264)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    import paper_2001_04931_b200 as P
    from paper_2001_04931_b200 import workloads as W

    spec, x0 = W.nlink_problem(6, 50, 0)
    return spec, P.KnotSchedule(50, 3), P.EmpcSettings(num_sims=1024, num_parents=64, generations=5, seed=3), x0


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2001_04931_b200.shard import PopulationShard, solve_population_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec, sched, st, x0 = _problem()
    shard = PopulationShard(spec, sched, st, rank, world)

    def all_gather(local):  # host copies: the exchange NCCL does over NVLink
        h = local.cpu()
        outs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(outs, h)
        return torch.cat(outs).cuda()

    u, best, cost = solve_population_sharded(shard, x0, all_gather)
    cands, costs = shard.local_population()
    q.put((rank, u, best, cost, cands, costs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_process_population_sharding_equals_unsharded(world):
    import paper_2001_04931_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    spec, sched, st, x0 = _problem()
    ref = P.solve_empc(spec, sched, st, x0)
    K = st.num_parents
    order = np.argsort(ref.population.costs, kind="stable")[:K]
    kids = []
    for rank, u, best, cost, cands, costs in got:
        np.testing.assert_array_equal(best, ref.best)
        np.testing.assert_array_equal(u, ref.u)
        assert cost == ref.best_cost
        # after the final exchange every rank holds the global top-K
        np.testing.assert_array_equal(cands[:K], ref.population.candidates[order])
        np.testing.assert_array_equal(costs[:K], ref.population.costs[order])
        kids.append(cands[K:])
    np.testing.assert_array_equal(np.concatenate(kids), ref.population.candidates[K:])
