"""Multi-rank host logic on CPU (gloo, world size 2): instance sharding and
the per-step result gather used by bench.py --gpus N for the batched C5
workload."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2001_04931_b200.shard import gather_instances, instance_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_instance_ranges_partition():
    for total in (1, 7, 8192):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                f, c = instance_range(total, r, world)
                seen.extend(range(f, f + c))
            assert seen == list(range(total))
    with pytest.raises(ValueError):
        instance_range(10, 2, 2)


def _worker(rank, world, port, total, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = instance_range(total, rank, world)
    # stand-in per-instance results: (u row, best cost) depend only on the instance id
    local_u = np.stack([np.full(3, float(i)) for i in range(first, first + count)]) if count else np.zeros((0, 3))
    local_c = np.arange(first, first + count, dtype=np.float64) * 0.5
    u = gather_instances(local_u, total)
    c = gather_instances(local_c, total)
    if rank == 0:
        out.put((u, c))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 16])
def test_gather_instances_gloo_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    u, c = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_array_equal(u, np.repeat(np.arange(total, dtype=float)[:, None], 3, axis=1))
    np.testing.assert_array_equal(c, np.arange(total) * 0.5)
