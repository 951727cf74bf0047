"""Multi-GPU sharding of independent MPC instances.

One process per GPU.  Instances are split into contiguous ranges, solved
with no collective inside the solve (each instance's selection is local to
its own population), and the per-instance results are gathered once per
control step.  This mirrors the reference harness's process-level parallelism
over independent tasks (K/bench.py:688-705), with results independent of the
number of ranks because every instance keeps its own RNG counters.
"""

from __future__ import annotations

import numpy as np


def instance_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of the contiguous instance block owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    per = (total + world - 1) // world
    first = min(total, rank * per)
    return first, max(0, min(per, total - first))


def gather_instances(local: np.ndarray, total: int, group=None) -> np.ndarray:
    """All-gather per-instance rows (local block of shape (count, ...)) into a
    (total, ...) array on every rank, in instance order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = instance_range(total, rank, world)
    assert local.shape[0] == count
    per = (total + world - 1) // world
    row_shape = local.shape[1:]
    buf = np.zeros((per,) + row_shape, dtype=local.dtype)
    buf[:count] = local
    t = torch.from_numpy(buf)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    full = np.concatenate([o.cpu().numpy() for o in outs])[:total]
    return full


# ---------------------------------------------------------------------------
# population sharding (C4: one very large population over W GPUs)


class PopulationShard:
    """One rank's part of a population-sharded ``solve_empc``.

    The rank holds the K elites (replicated) and the children of global child
    indices ``instance_range(N - K, rank, world)`` (and, for the cold start,
    the initial candidates ``instance_range(N, rank, world)``).  One exchange
    per generation: ``export()`` -> all-gather of W x K entries ->
    ``import_()`` ranks them identically on every rank.  Results equal the
    unsharded solve bit for bit for any ``world`` (global rows in the
    selection keys, global child indices in the RNG counters).
    """

    def __init__(self, spec, sched, settings, rank: int, world: int):
        import ctypes as C

        from . import _native as nat
        from .empc import _is_diag, _mutation_sigma, _problem_arrays  # noqa: F401
        from .param import schedule_arrays

        self.nat, self.C = nat, C
        self.spec, self.sched, self.settings = spec, sched, settings
        self.rank, self.world = rank, world
        N, K = settings.num_sims, settings.num_parents
        n, m = spec.model.Ad.shape[0], spec.model.Bd.shape[1]
        self.cb, self.cn = instance_range(N - K, rank, world)
        self.ib, self.inn = instance_range(N, rank, world)
        rows = K + max(self.cn, self.inn, 1)
        self.h = nat.Handle(n, m, spec.T, sched.p, rows, K, 1, not _is_diag(spec.Q),
                            nat.EMPC_FP64 if settings.precision == "fp64" else nat.EMPC_FP32)
        i1, i2, c = schedule_arrays(spec.T, sched.p)
        self.h.call("empc_set_schedule", nat.iptr(np.ascontiguousarray(i1)), nat.iptr(np.ascontiguousarray(i2)),
                    nat.dptr(np.ascontiguousarray(c)))
        pa = _problem_arrays(spec)
        arrs = [nat.f64(pa[k]) for k in ("Ad", "Bd", "wd", "Q", "R", "x_goal", "u_goal", "u_min", "u_max")]
        self.h.call("empc_set_problems", 0, 1, *[nat.dptr(x) for x in arrs])
        from .empc import TC_MODES, _scorer_code

        self.h.call("empc_set_scorer", _scorer_code(getattr(settings, "scorer", "rollout"), spec))
        self.h.set_tensor_cores(TC_MODES[getattr(settings, "tensor_cores", "auto")])
        self.h.call("empc_shard_setup", self.cb, self.cn, self.ib, self.inn, 1 if rank == 0 else 0)
        eb = C.c_int64()
        self.h.call("empc_shard_entry_bytes", C.byref(eb))
        self.entry_bytes = eb.value
        self.K, self.m, self.p = K, m, sched.p
        self._args = nat.empc_run_args()

    def _run_args(self, x0, generation):
        from .empc import _mutation_sigma

        nat, st = self.nat, self.settings
        a = self._args
        self._x0 = nat.f64(np.asarray(x0, float).reshape(1, -1))
        self._sg = nat.f64(_mutation_sigma(self.spec, st, np.asarray(x0, float))[None])
        a.init, a.rescore, a.evolves, a.slot_in, a.slot_out = 1, 0, 0, -1, -1
        a.generation0 = int(generation)
        a.seed = int(st.seed) & 0xFFFFFFFFFFFFFFFF
        a.mutation_prob, a.crossover_prob = float(st.mutation_prob), float(st.crossover_prob)
        a.x0, a.sigma = nat.dptr(self._x0), nat.dptr(self._sg)
        return a

    @property
    def stream_ptr(self) -> int:
        """The handle's CUDA stream: every shard call below only enqueues on it."""
        v = self.C.c_void_p()
        self.h.call("empc_get_stream", self.C.byref(v))
        return v.value or 0

    def sync(self):
        import torch

        torch.cuda.ExternalStream(self.stream_ptr).synchronize()

    def init(self, x0):
        """Stage the problem, x0, sigma and the RNG parameters; score the
        initial candidates (asynchronous)."""
        self.h.call("empc_shard_init", self.C.byref(self._run_args(x0, 1)))

    def export(self, device_ptr: int):
        """Enqueue this rank's top-K entries (K * entry_bytes) into device memory."""
        self.h.call("empc_shard_export", self.C.c_void_p(device_ptr))

    def import_(self, device_ptr: int, world: int, outputs: bool = True):
        """Rank the W x K gathered entries and install the global top-K.  With
        ``outputs`` (the last exchange of a solve) wait for it and return
        (u, best, best_cost, global row); otherwise only enqueue."""
        nat, C = self.nat, self.C
        if not outputs:
            self.h.call("empc_shard_import", C.c_void_p(device_ptr), world, None, None, None, None)
            return None
        u = np.empty(self.m)
        best = np.empty((self.p, self.m))
        cost = np.empty(1)
        row = C.c_int64()
        self.h.call("empc_shard_import", C.c_void_p(device_ptr), world, nat.dptr(u), nat.dptr(best), nat.dptr(cost),
                    C.byref(row))
        return u, best, float(cost[0]), row.value

    def evolve(self, x0, generation: int):
        """Breed and score this rank's children for ``generation`` (asynchronous;
        x0 and sigma are the ones staged by init)."""
        a = self._args
        a.generation0 = int(generation)
        self.h.call("empc_shard_evolve", self.C.byref(a))

    def local_population(self):
        """(candidates, costs) of rows [elites; this rank's children]."""
        rows = self.K + self.cn
        c = np.empty((rows, self.p, self.m))
        k = np.empty(rows)
        self.h.call("empc_shard_read", self.nat.dptr(c), self.nat.dptr(k))
        return c, k


def solve_population_sharded(shard: PopulationShard, x0, all_gather):
    """Cold solve of one population split over ranks (K/empc.py:211-236):
    init + (G-1) x [exchange, select, breed] + a final exchange for the best.

    ``all_gather(local_uint8_tensor) -> gathered_uint8_tensor`` concatenates
    every rank's export in rank order.  It runs with the handle's stream as
    torch's current stream, so ``dist.all_gather_into_tensor`` over NCCL is
    stream-ordered between the export and the import: a generation is enqueued
    back to back with no host synchronisation (a gloo exchange through host
    copies also works, synchronously).  Returns (u, best, best_cost)."""
    import torch

    K, eb = shard.K, shard.entry_bytes
    stream = torch.cuda.ExternalStream(shard.stream_ptr)
    with torch.cuda.stream(stream):
        local = torch.empty(K * eb, dtype=torch.uint8, device="cuda")
        shard.init(x0)
        for g in range(1, shard.settings.generations):
            shard.export(local.data_ptr())
            gathered = all_gather(local)
            shard.import_(gathered.data_ptr(), gathered.numel() // (K * eb), outputs=False)
            shard.evolve(x0, g)
        shard.export(local.data_ptr())
        gathered = all_gather(local)
        u, best, cost, _ = shard.import_(gathered.data_ptr(), gathered.numel() // (K * eb))
    return u, best, cost


def solve_population_emulated(spec, sched, settings, x0, world: int):
    """All ranks of a population-sharded solve in one process on one GPU,
    stepped in lock-step with an on-device gather (tests / single-GPU boxes)."""
    import torch

    shards = [PopulationShard(spec, sched, settings, r, world) for r in range(world)]
    K, eb = shards[0].K, shards[0].entry_bytes
    bufs = [torch.empty(K * eb, dtype=torch.uint8, device="cuda") for _ in range(world)]

    def exchange():
        for s, b in zip(shards, bufs):
            s.export(b.data_ptr())
            s.sync()
        allb = torch.cat(bufs)
        torch.cuda.synchronize()
        return [s.import_(allb.data_ptr(), world) for s in shards]

    for s in shards:
        s.init(x0)
    for g in range(1, settings.generations):
        exchange()
        for s in shards:
            s.evolve(x0, g)
    res = exchange()
    assert all(r[2] == res[0][2] and r[3] == res[0][3] for r in res), "ranks disagree on the best candidate"
    return res[0], shards
