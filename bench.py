"""EMPC hot-path benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl ours|reference]

A "step" is one cold ``solve_empc`` (init + G-1 generations + argmin) of the
configured workload.  Default workload: C3 (24-DoF, T=50, p=4, N=4096,
K=256, G=10), the north-star per-step latency target.  Under torchrun each
rank owns one GPU; single-problem workloads run one independent replica per
rank ("replicas only", weak scaling), the batched C5 workload shards its
instances across ranks (strong scaling: total instances fixed).

value     = candidate-rollout-steps/s, device-resident (CUDA-event time of the
            graph-captured solve, inputs already in HBM, L2 flushed between
            timed solves), summed over ranks / max-over-ranks time.
e2e       = the same metric through the public Python API (numpy in, numpy
            out: pinned H2D of the problem + x0, D2H of u / best / cost).
roofline  = rollout kernel (K2+K3+K5) FP32 FLOP/s vs the measured FFMA peak.
cpu_baseline / --impl reference = the reference algorithm (CPU oracle port
            of knotmpc.empc: numpy Philox RNG + condensed quadratic scoring)
            on this host's cores.
"""

from __future__ import annotations

import argparse
import gc
import json
import re
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EMPC solve latency per MPC step (ms) and candidate-rollout-steps/sec vs FP32 peak"
UNIT = "candidate-rollout-steps/s"
FP32_PEAK_FILE = os.path.join(ROOT, "profiles", "fp32_peak.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "rollout_traffic.json")
DESCRIPTIONS = {
    "c1": "2-DoF (4-state) linear joint system, T=20, p=2, N=100, K=6, G=10",
    "c2": "6-DoF arm, T=50, p=3, N=1024, K=64, G=10",
    "c3": "24-DoF, T=50, p=4, N=4096, K=256, G=10 (per-step solve latency target < 1 ms)",
    "c4": "48-DoF, T=200, p=5, N=16384, K=1024, G=10",
    "c5": "8192 x 12-DoF instances, T=50, p=3, N=512, K=32, G=10",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=sorted(DESCRIPTIONS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instances", type=int, default=None, help="override the instance count (C5)")
    ap.add_argument("--num-sims", type=int, default=None,
                    help="override the population size N (e.g. one rank's share of a sharded C4 population)")
    ap.add_argument("--variant", type=int, default=-1, help="force a rollout kernel variant")
    ap.add_argument("--sharded", action="store_true",
                    help="C4: run the population-sharded solve (shard.py) also at one GPU -- the N = 1 point of the "
                         "population-sharding scaling curve")
    ap.add_argument("--cpu-sample-s", type=float, default=12.0, help="CPU baseline budget (s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l2", default="flush", choices=["flush", "warm"],
                    help="warm: no L2 flush between timed solves (experiment only; the line says so)")
    ap.add_argument("--tensor-cores", default="auto", choices=["auto", "on", "off"],
                    help="FP32 rollout recursion on the tcgen05 tensor cores (TF32 split precision): auto = where it "
                         "measured faster (DESIGN.md §4.8)")
    ap.add_argument("--scorer", default="rollout", choices=["rollout", "condensed"],
                    help="rollout (the north-star kernels, default) or the reference's condensed quadratic "
                         "(SURVEY §8 f2; FP64 quadratic form, roofline against the FP64 peak)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def workload(args, rank, world):
    from paper_2001_04931_b200 import workloads as W

    w = W.WORKLOADS[args.config]
    if args.instances is not None:
        w = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, instances=args.instances)
    if args.num_sims is not None:
        w = W.Workload(w.name, w.dof, w.T, w.p, args.num_sims, w.K, w.G, instances=w.instances)
    if w.instances > 1:  # shard instances across ranks
        from paper_2001_04931_b200.shard import instance_range

        first, count = instance_range(w.instances, rank, world)
        specs, x0s = W.build(w, first, count)
        local = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, instances=count)
        return w, local, specs, x0s, "strong"
    specs, x0s = W.build(w)
    return w, w, specs, x0s, "weak"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 5]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(names, r[2:6]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_solve_time(w, specs, x0s, budget_s, max_solves=None, threads=None):
    """Time the reference algorithm (oracle port of knotmpc.empc) on the host.
    ``threads`` limits the OpenBLAS pool (threadpoolctl), None = all cores."""
    from oracle import empc_oracle as O

    try:
        from threadpoolctl import threadpool_limits, threadpool_info
    except ImportError:  # pragma: no cover
        threadpool_limits = threadpool_info = None
    import contextlib

    lim = threadpool_limits(limits=threads, user_api="blas") if (threads and threadpool_limits) else (
        contextlib.nullcontext())
    with lim:
        st = O.Settings(num_sims=w.N, num_parents=w.K, generations=w.G, seed=1)
        pr = O.Problem.from_spec(specs[0])
        x0 = x0s[0]
        O.solve_empc(pr, w.p, st, x0)  # warm-up
        times = []
        t_start = time.perf_counter()
        while not times or (time.perf_counter() - t_start < budget_s and (max_solves is None or len(times) < max_solves)):
            i = len(times) % len(specs)
            pr = O.Problem.from_spec(specs[i])
            t0 = time.perf_counter()
            O.solve_empc(pr, w.p, st, x0s[i])
            times.append(time.perf_counter() - t0)
        used = threads
        if used is None:
            try:
                used = max([d.get("num_threads", 1) for d in threadpool_info() if d.get("internal_api") == "openblas"]
                           or [1])
            except Exception:
                used = os.cpu_count()
    return times, used


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _pool_worker(task):
    """One process of the C5 CPU baseline: solve instances [first, first+count)
    of the workload with one BLAS thread (the K/bench.py:694-699 pattern)."""
    name, first, count, budget = task
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits

    from oracle import empc_oracle as O
    from paper_2001_04931_b200 import workloads as W

    with threadpool_limits(limits=1, user_api="blas"):
        w = W.WORKLOADS[name]
        specs, x0s = W.build(w, first, count)
        st = O.Settings(num_sims=w.N, num_parents=w.K, generations=w.G, seed=1)
        done, t0 = 0, time.perf_counter()
        while done < count and time.perf_counter() - t0 < budget:
            O.solve_empc(O.Problem.from_spec(specs[done]), w.p, st, x0s[done])
            done += 1
        return done, time.perf_counter() - t0


def cpu_pool_instances_per_s(name, budget_s):
    """C5 reference baseline: one worker process per host core, each with one
    BLAS thread, solving distinct instances for ``budget_s`` seconds
    (K/bench.py:694-699).  Returns (instances/s over the pool, workers, solved)."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp

    workers = os.cpu_count() or 1
    per = 512  # instances handed to each worker (more than it finishes in the budget)
    tasks = [(name, i * per, per, budget_s) for i in range(workers)]
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_pool_worker, tasks))
    solved = sum(r[0] for r in res)
    rate = sum(r[0] / r[1] for r in res if r[1] > 0)
    return rate, workers, solved, max(r[1] for r in res)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2001_04931_b200 import workloads as W

    w = W.WORKLOADS[args.config]
    if args.instances is not None:
        w = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, instances=args.instances)
    per_instance = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, 1)
    specs, x0s = W.build(per_instance) if w.instances == 1 else W.build(W.WORKLOADS[args.config], 0, 1)
    warm = max(1, min(args.warmup, 3))
    if w.instances > 1:
        # independent instances: one worker per host core, one BLAS thread each
        budget = max(5.0, min(60.0, 6.0 * args.steps))
        rate, workers, solved, took = cpu_pool_instances_per_s(args.config, budget)
        t_step = w.instances / rate
        value = per_instance.cand_steps_per_solve * w.instances / t_step
        times, threads = [t_step], workers
        sample = (f"{solved} cold solves of distinct {args.config} instances by {workers} worker processes x 1 BLAS "
                  f"thread in {took:.1f}s (oracle port of knotmpc.empc; K/bench.py:694-699 pool pattern); "
                  f"step = {w.instances} instances at the pool rate")
    else:
        times, threads = cpu_reference_solve_time(per_instance, specs[:1], x0s[:1], budget_s=0.0, max_solves=1)
        budget = 120.0
        steps = max(1, min(args.steps, int(budget / max(times[0], 1e-6))))
        cpu_reference_solve_time(per_instance, specs[:1], x0s[:1], budget_s=0.0, max_solves=warm)
        times, threads = cpu_reference_solve_time(per_instance, specs[:1], x0s[:1], budget_s=1e9, max_solves=steps)
        t_step = statistics.mean(times)
        value = per_instance.cand_steps_per_solve / t_step
        sample = f"{len(times)} cold solves of one {args.config} instance (oracle port of knotmpc.empc: numpy Philox + condensed scoring)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": len(times),
        "warmup": warm, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if w.instances > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {DESCRIPTIONS[args.config]}", "dof": w.dof, "T": w.T, "p": w.p,
                   "N": w.N, "K": w.K, "G": w.G, "instances": w.instances},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model(), "cpu_count": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "latency_ms": {"median": statistics.median(times) * 1e3},
    }
    print(json.dumps(line), flush=True)


def run_population_sharded(args, rank, world):
    """C4 over W GPUs: one population split over ranks, one NCCL all-gather of
    the ranks' top-K entries per generation.  Strong scaling:
    the total population is fixed."""
    import torch
    import torch.distributed as dist

    from paper_2001_04931_b200 import workloads as W
    from paper_2001_04931_b200.shard import PopulationShard, solve_population_sharded

    w = W.WORKLOADS[args.config]
    specs, x0s = W.build(w)
    shard = PopulationShard(specs[0], w.schedule(), w.settings(scorer=args.scorer), rank, world)
    K, eb = shard.K, shard.entry_bytes
    gathered = torch.empty(world * K * eb, dtype=torch.uint8, device="cuda")

    def all_gather(local):
        if world == 1:
            return local
        dist.all_gather_into_tensor(gathered, local)
        return gathered

    for _ in range(max(args.warmup, 3)):
        solve_population_sharded(shard, x0s[0], all_gather)
    # device time of each solve on the handle's stream (where the kernels and
    # the NCCL exchange are enqueued), max over ranks below
    stream = torch.cuda.ExternalStream(shard.stream_ptr)
    sampler = ClockSampler(0)
    times = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        u, best, cost = solve_population_sharded(shard, x0s[0], all_gather)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    t = torch.tensor([sum(times)], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    units = w.cand_steps_per_solve * args.steps
    value = units / (total_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (reference recipe: linearized N-link arms, SURVEY §8d)",
        "config": {"workload": f"{args.config}: {DESCRIPTIONS[args.config]} (population sharded over {world} GPUs, "
                               "per-generation NCCL all-gather of the ranks' top-K)", "dof": w.dof, "T": w.T,
                   "p": w.p, "N": w.N, "K": w.K, "G": w.G, "instances": 1, "l2": "not flushed (NCCL path)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(sum(v.nbytes for v in x0s) + 8 * 9 * 96 * 96),
                "d2h_bytes_per_step": int(u.nbytes + best.nbytes + 8), "api": "shard.solve_population_sharded"},
        "clocks": clocks,
        "gpu_launches": 3 * w.G * args.steps,  # init + (G-1) x (export, import, evolve) + export + import
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(args, w, specs, x0s):
    """The reference algorithm on this host's cores, next to the device run
    (BASELINE.md §4): all BLAS threads and one BLAS thread for one instance;
    C5 through a process pool of one worker per core."""
    from paper_2001_04931_b200 import workloads as W

    one = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, 1)
    budget = args.cpu_sample_s
    if w.instances > 1:
        rate, workers, solved, took = cpu_pool_instances_per_s(args.config, budget)
        value = one.cand_steps_per_solve * rate
        return {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                "sample": f"{solved} cold solves of distinct {args.config} instances in {took:.1f}s by {workers} "
                          "worker processes x 1 BLAS thread (oracle port of knotmpc.empc, K/bench.py:694-699 pool)",
                "instances_per_s": rate, "cpu_model": cpu_model(), "cpu_count": os.cpu_count()}
    times, threads = cpu_reference_solve_time(one, specs[:1], x0s[:1], budget_s=0.65 * budget)
    t1, _ = cpu_reference_solve_time(one, specs[:1], x0s[:1], budget_s=0.35 * budget, threads=1)
    return {"value": one.cand_steps_per_solve / statistics.mean(times), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(times)} cold solves of one {args.config} instance in {sum(times):.1f}s with all "
                      f"OpenBLAS threads (oracle port of knotmpc.empc: numpy Philox RNG + condensed-quadratic "
                      f"scoring); {len(t1)} more with one thread",
            "ms_per_solve": statistics.mean(times) * 1e3, "ms_per_solve_median": statistics.median(times) * 1e3,
            "single_thread": {"value": one.cand_steps_per_solve / statistics.mean(t1), "cores": 1,
                              "ms_per_solve": statistics.mean(t1) * 1e3,
                              "ms_per_solve_median": statistics.median(t1) * 1e3},
            "cpu_model": cpu_model(), "cpu_count": os.cpu_count()}


def run_ours(args):
    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("CUDA_VISIBLE_DEVICES", str(local))
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    torch.cuda.init()

    import paper_2001_04931_b200 as P
    from paper_2001_04931_b200 import _native as nat
    from paper_2001_04931_b200 import empc as E

    if args.config == "c4" and (world > 1 or args.sharded):
        return run_population_sharded(args, rank, world)
    w_total, w, specs, x0s, scaling = workload(args, rank, world)
    sched = w.schedule()
    st = w.settings(scorer=args.scorer, tensor_cores=args.tensor_cores)
    # --- device-resident path: the graph-captured cold solve
    if w.instances > 1:
        batch = P.EmpcBatch(specs, sched, st)
        ctx = batch.ctx
        sigma = batch.sigma(x0s)
    else:
        ctx = E._spec_context(specs[0], sched, st)
        sigma = E._mutation_sigma(specs[0], st, x0s[0])[None]
    if args.variant >= 0:
        ctx.h.set_variant(args.variant)
    a = nat.empc_run_args()
    x0c = nat.f64(x0s)
    sg = nat.f64(sigma)
    a.init, a.rescore, a.evolves, a.slot_in, a.slot_out = 1, 0, w.G - 1, -1, -1
    a.generation0, a.seed = 1, st.seed
    a.mutation_prob, a.crossover_prob = st.mutation_prob, st.crossover_prob
    a.x0, a.sigma = nat.dptr(x0c), nat.dptr(sg)
    import ctypes as C

    def time_device(reps, flush=1, want_rollout=False):
        ms = (C.c_float * reps)()
        rms = C.c_float(0.0)
        nr = C.c_int32(0)
        nl = C.c_int32(0)
        ctx.h.call("empc_time_device", C.byref(a), reps, flush, ms, C.byref(rms) if want_rollout else None,
                   C.byref(nr), C.byref(nl))
        return list(ms), rms.value, nr.value, nl.value

    time_device(max(args.warmup, 3))  # warm-up (graph capture on first use)
    sampler = ClockSampler(0)
    t_spin = time.perf_counter()
    while time.perf_counter() - t_spin < 0.6:  # clocks ramp under load before the timed region
        time_device(10, flush=0)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ms_each, _, nroll, nlaunch = time_device(args.steps, flush=0 if args.l2 == "warm" else 1)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    total_ms = sum(ms_each)
    # roofline pass: per-launch rollout durations (events around each launch)
    _, rollout_ms, _, _ = time_device(min(args.steps, 20), flush=0 if args.l2 == "warm" else 1, want_rollout=True)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    units_local = w.cand_steps_per_solve * args.steps
    units_total = units_local * (world if scaling == "weak" else 1) if w_total.instances == 1 else (
        w_total.cand_steps_per_solve * args.steps)
    value = units_total / (total_ms * 1e-3)

    # --- e2e through the public API (numpy in / numpy out).  Python objects
    # alive at this point are frozen out of the cyclic GC (a full collection
    # with torch loaded takes tens of ms); every call still allocates its
    # own result arrays.  At least 100 calls for the sub-ms single problems.
    n_e2e = args.steps if w.instances > 1 else max(args.steps, 100)
    e2e_times = []
    if w.instances > 1:
        batch.solve(x0s)
        gc.collect()
        gc.freeze()
        for _ in range(n_e2e):
            t0 = time.perf_counter()
            r = batch.solve(x0s)
            e2e_times.append(time.perf_counter() - t0)
        h2d = batch.probs["Ad"].nbytes + sum(v.nbytes for k, v in batch.probs.items() if k != "Ad") + x0c.nbytes + sg.nbytes
        d2h = r.u.nbytes + r.best.nbytes + r.best_cost.nbytes + 4 * w.instances
    else:
        for _ in range(10):
            P.solve_empc(specs[0], sched, st, x0s[0])
        gc.collect()
        gc.freeze()
        for _ in range(n_e2e):
            t0 = time.perf_counter()
            r = P.solve_empc(specs[0], sched, st, x0s[0])
            e2e_times.append(time.perf_counter() - t0)
        pa = E._problem_arrays(specs[0])
        h2d = sum(np.asarray(v).nbytes for v in pa.values()) + x0s[0].nbytes + sigma.nbytes + 32
        d2h = r.u.nbytes + r.best.nbytes + 8 + 4
    gc.unfreeze()
    e2e_total = sum(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_total], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = units_total * n_e2e / args.steps / e2e_total
    e2e_ms = np.asarray(e2e_times) * 1e3
    e2e_stats = {"calls": n_e2e, "latency_ms_median": float(np.median(e2e_ms)),
                 "latency_ms_q1": float(np.percentile(e2e_ms, 25)), "latency_ms_q3": float(np.percentile(e2e_ms, 75)),
                 "latency_ms_mean": float(e2e_ms.mean()), "latency_ms_max": float(e2e_ms.max()),
                 "slowest_call": int(np.argmax(e2e_ms))}
    # warm start (cold and warm): solve_empc(prev=population)
    # with the population resident on the GPU, as a closed loop calls it
    # (K/closedloop.py:109): re-score at x0 + G generations, same model
    if w.instances == 1:
        prev = P.solve_empc(specs[0], sched, st, x0s[0]).population
        for _ in range(5):
            prev = P.solve_empc(specs[0], sched, st, x0s[0], prev=prev).population
        gc.collect()
        gc.freeze()
        warm = []
        for _ in range(n_e2e):
            t0 = time.perf_counter()
            prev = P.solve_empc(specs[0], sched, st, x0s[0], prev=prev).population
            warm.append(time.perf_counter() - t0)
        gc.unfreeze()
        wm = np.asarray(warm) * 1e3
        e2e_stats["warm"] = {"calls": n_e2e, "latency_ms_median": float(np.median(wm)),
                             "latency_ms_q1": float(np.percentile(wm, 25)),
                             "latency_ms_q3": float(np.percentile(wm, 75)), "latency_ms_mean": float(wm.mean()),
                             "scored_per_solve": w.N + w.G * (w.N - w.K),
                             "note": "solve_empc(prev=population): re-score + G generations, population on the GPU"}

    # --- roofline of the dominant kernel (rollout: K2+K3 with the K5 prologue)
    condensed = args.scorer == "condensed"
    if condensed:
        # quadratic form z'Pz + 2g'z: 2 pm^2 + 4 pm FP64 flop per scored candidate
        pm = w.p * w.m
        flop_per_launch = (2 * pm * pm + 4 * pm) * w.scored_per_solve / max(nroll, 1)
    else:
        flop_per_launch = w.flop_per_candidate * w.scored_per_solve / max(nroll, 1)
    achieved = flop_per_launch / (rollout_ms * 1e-3) / 1e12
    peak, peak_src = 72.53, "tools/ffma_peak.cu on a B200 of this pool (no FP32 entry in MEASURED_PEAKS.json)"
    if os.path.exists(FP32_PEAK_FILE):
        with open(FP32_PEAK_FILE) as f:
            pk = json.load(f)
        peak, peak_src = pk["tflops"], pk.get("source", peak_src)
        if condensed:
            peak = pk.get("fp64_tflops", peak)
            peak_src = pk.get("fp64_source", peak_src)
    desc = ctx.h.describe()
    tc = re.search(r"tcgen05 tf32x3 N(\d+) K(\d+)", desc) if not condensed else None
    fp32_equiv = None
    if tc:
        # tensor-core rollout: executed TF32 tensor FLOP (3 split terms, padded
        # N / K, 128-candidate tiles) against the measured dense TF32 peak; the
        # algorithmic FP32 rate is reported beside it against the FFMA peak
        NN, NK = int(tc.group(1)), int(tc.group(2))
        def launch_tiles(nc):  # the host's TC launch plan (empc.cu plan()): 128-row MMA tiles
            if w.instances == 1:
                return -(-nc // max(1, min(128, -(-nc // 148))))
            return w.instances * -(-nc // 128)
        tiles = launch_tiles(w.N) + (w.G - 1) * launch_tiles(w.N - w.K)
        # issued K-steps: 8-column blocks of Delta = Ad - I with a nonzero entry
        # (the kernel skips all-zero blocks; every instance of a workload has
        # the same structure)
        dl = np.asarray(specs[0].model.Ad) - np.eye(w.n)
        ksteps = max(1, sum(bool(np.any(dl[:, 8 * s_:8 * s_ + 8] != 0)) for s_ in range(NK // 8)))
        tensor_flop = tiles * w.T * 3 * 2 * 128 * NN * 8 * ksteps / max(nroll, 1)
        fp32_equiv = {"achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                      "note": "algorithmic FP32 work (2Tn^2 + 2pnm per candidate) / rollout time vs the FFMA peak"}
        achieved = tensor_flop / (rollout_ms * 1e-3) / 1e12
        flop_per_launch = tensor_flop
        peak, peak_src = 821.7, "half of MEASURED_PEAKS.json bf16_tflops (TF32 MMA: same cycles, half the MACs)"
        if os.path.exists(FP32_PEAK_FILE):
            with open(FP32_PEAK_FILE) as f:
                pk = json.load(f)
            if "tf32_tflops" in pk:
                peak, peak_src = pk["tf32_tflops"], pk.get("tf32_source", peak_src)
    traffic = None
    if os.path.exists(TRAFFIC_FILE) and not condensed:
        with open(TRAFFIC_FILE) as f:
            tr = json.load(f)
        traffic = tr.get(args.config + ("_tc" if tc else ""))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32" if not condensed else "f32 population, f64 quadratic form", "scorer": args.scorer, "data": "synthetic (reference recipe: linearized N-link arms, SURVEY §8d)",
        "config": {"workload": f"{args.config}: {DESCRIPTIONS[args.config]}", "dof": w.dof, "T": w.T, "p": w.p,
                   "N": w.N, "K": w.K, "G": w.G, "instances": w_total.instances,
                   "instances_per_rank": w.instances,
                   "l2": "flushed (256 MiB write) between timed solves" if args.l2 == "flush"
                   else "NOT flushed (experiment: warm L2)",
                   "kernel_variant": ctx.h.describe()},
        "latency_ms": {"median": statistics.median(ms_each), "q1": float(np.percentile(ms_each, 25)),
                       "q3": float(np.percentile(ms_each, 75)), "min": min(ms_each)},
        "roofline": {"bound": "fp64_fma" if condensed else "tensor" if tc else "fp32_fma", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "kernel": "cond_score_kernel (breed + FP64 quadratic form)" if condensed else
                     "rollout_tc_kernel (tcgen05 kind::tf32, 3 split terms; breed + recursion + cost)" if tc else
                     "persist_kernel (whole solve in one cooperative launch: rollouts + selection)"
                     if "persistent" in desc else "rollout_kernel",
                     "fp32_equivalent": fp32_equiv,
                     "rollout_ms_per_launch": rollout_ms, "rollout_launches_per_step": nroll,
                     "flop_per_launch": flop_per_launch, "peak_source": peak_src,
                     "issued": ("half-K matvec: the all-zero left half of Delta = Ad - I is skipped, so the "
                                "recursion issues T n^2 of the 2 T n^2 algorithmic FLOP per candidate; achieved "
                                "counts the algorithmic FLOP") if "halfK" in desc else None},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                **e2e_stats, "api": "solve_empc" if w.instances == 1 else "EmpcBatch.solve"},
        "clocks": clocks,
        "gpu_launches": nlaunch * args.steps,
    }
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, w_total, specs, x0s)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def relaunch(args) -> int:
    """``bench.py --gpus N`` without a torchrun environment: start N ranks
    (one process per GPU, 127.0.0.1 rendezvous) and relay rank 0's line."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
