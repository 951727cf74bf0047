/*
 * empc_b200.h -- C ABI of the B200-native Evolutionary MPC (EMPC) hot path.
 *
 * The reference (knotmpc, pure Python) has no FFI: its boundary is the
 * Python API of knotmpc/empc.py.  These entry points are what a binding
 * (ctypes / cffi / pybind) of that API calls; each one cites the reference
 * function it replaces (paths relative to /root/reference/pkg/src/knotmpc):
 *
 *   empc_run      <- solve_empc          empc.py:211-236   (cold/warm solve)
 *                 <- init_population     empc.py:162-171   (init only)
 *                 <- evolve_generation   empc.py:174-208   (one generation)
 *   empc_score    <- _CostModel.__call__ empc.py:147-152   (batch scorer seam)
 *                 <- evaluate_cost       empc.py:155-159   (N = 1)
 *   empc_select   <- argsort(kind="stable")[:K] / argmin   empc.py:185-186, 234
 *   empc_expand   <- expand / input_at   param.py:91-116   (knots -> inputs)
 *   empc_set_schedule <- KnotSchedule.coeffs / interpolation_matrix param.py:49-111
 *   empc_set_scorer   <- _CostModel's choice of scorer     empc.py:133-152 (rollout vs
 *                        condensed quadratic from build_small_param, condense.py:268-274)
 *   empc_plant_linearize_discretize <- linearize + discretize dynamics.py:241-290
 *   empc_plant_integrate  <- integrate / rk4_step          dynamics.py:316-330
 *                        (batched, per closed-loop period: closedloop.py:103-104)
 *   empc_set_problems <- MpcSpec + DiscreteLinearModel condense.py:42-87, dynamics.py:223-238
 *
 * Conventions: row-major arrays; every pointer argument is a HOST pointer
 * borrowed for the duration of the call (device buffers are owned by the
 * handle).  Floating-point inputs/outputs are FP64 like the reference; the
 * device computes in the precision chosen at creation (FP32 default).
 * Every function returns 0 on success or a negative EMPC_E* code, with a
 * message available from empc_last_error().  One handle per host thread;
 * distinct handles may be used concurrently.
 */
#ifndef EMPC_B200_H_
#define EMPC_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  EMPC_OK = 0,
  EMPC_EINVAL = -1,   /* invalid argument (Python layer raises ValueError) */
  EMPC_ECUDA = -2,    /* CUDA runtime error (RuntimeError) */
  EMPC_ESTATE = -3,   /* call order / missing problem, schedule or population */
  EMPC_ENOMEM = -4,
};

enum { EMPC_FP32 = 0, EMPC_FP64 = 1 };

typedef struct empc_handle empc_handle;

/* Problem shape shared by all instances of a handle (EmpcSettings
 * num_sims / num_parents, empc.py:31-32; MpcSpec dims, condense.py:42-56). */
typedef struct {
  int32_t n;           /* state dimension  (model.n) */
  int32_t m;           /* input dimension  (model.m) */
  int32_t T;           /* horizon (MpcSpec.T == KnotSchedule.T) */
  int32_t p;           /* knot count (KnotSchedule.p) */
  int32_t num_sims;    /* N */
  int32_t num_parents; /* K, 1 <= K <= N */
  int32_t instances;   /* independent MPC problems batched in one handle */
  int32_t dense_q;     /* 0: Q diagonal (empc.py:114-116 fast path), 1: dense Q */
  int32_t precision;   /* EMPC_FP32 (default) or EMPC_FP64 */
  int32_t device;      /* CUDA device ordinal */
} empc_dims;

int empc_create(const empc_dims* dims, empc_handle** out);
void empc_destroy(empc_handle* h);
/* Last error message of the handle (or of the last failed empc_create when h is NULL). */
const char* empc_last_error(const empc_handle* h);

/* Knot schedule: per step k in [0,T): u_k = (1-c_k) U[idx1_k] + c_k U[idx2_k]
 * (param.py:30-46, p==1 -> idx1=idx2=0, c=0). */
int empc_set_schedule(empc_handle* h, const int32_t* idx1, const int32_t* idx2, const double* c);

/* Scorer of every subsequent run / score call:
 *   EMPC_SCORER_ROLLOUT   (0, default) FP32/FP64 horizon rollout (empc.py:85-119)
 *   EMPC_SCORER_CONDENSED (1) the reference's own condensed quadratic
 *     J(z) = z'Pz + 2q'z + c0 (empc.py:133-152), built on the device once per
 *     run in FP64 and evaluated in FP64 (costs rounded to the population
 *     precision).  Not for state-bounded specs (the reference rolls those out). */
#define EMPC_SCORER_ROLLOUT 0
#define EMPC_SCORER_CONDENSED 1
int empc_set_scorer(empc_handle* h, int32_t scorer);


/* Problems of instances [first, first+count).  Per instance, contiguous:
 * Ad[n*n] Bd[n*m] wd[n] Q[n*n] R[m*m] x_goal[n] u_goal[m] u_min[m] u_max[m]. */
int empc_set_problems(empc_handle* h, int32_t first, int32_t count, const double* Ad, const double* Bd,
                      const double* wd, const double* Q, const double* R, const double* x_goal,
                      const double* u_goal, const double* u_min, const double* u_max);

/* Population slots: device-resident (N x p x m candidates, N costs) per instance. */
int empc_pop_alloc(empc_handle* h, int32_t* slot);
int empc_pop_free(empc_handle* h, int32_t slot);
/* D2H read of a slot (FP64 out; either pointer may be NULL); generation is host-side state. */
int empc_pop_read(empc_handle* h, int32_t slot, double* cands, double* costs);
/* H2D write of a slot (e.g. a Population built on the host). costs may be NULL (zeros). */
int empc_pop_write(empc_handle* h, int32_t slot, const double* cands, const double* costs);

/* Injected random tensors (parity mode) replacing the in-kernel Philox
 * streams: the reference's draws of empc.py:168-170 / 195-199. */
typedef struct {
  const double* init;          /* instances x N x p x m, or NULL */
  const int32_t* parents;      /* evolves x instances x (N-K) x 2, or NULL */
  const uint8_t* take_second;  /* evolves x instances x (N-K) x p x m */
  const uint8_t* mutate;       /* evolves x instances x (N-K) x p x m */
  const double* noise;         /* evolves x instances x (N-K) x p x m */
} empc_injected;

typedef struct {
  int32_t init;             /* 1: cold start (uniform knots, empc.py:168-170) */
  int32_t rescore;          /* 1: re-score slot_in at x0 before evolving (empc.py:229-231) */
  int32_t evolves;          /* number of evolve_generation steps */
  int32_t slot_in;          /* population read when init == 0 (-1 otherwise) */
  int32_t slot_out;         /* slot receiving the final population (-1: keep internal only) */
  int64_t generation0;      /* Population.generation at entry (RNG key of the first evolve) */
  uint64_t seed;            /* EmpcSettings.seed */
  double mutation_prob;     /* EmpcSettings.mutation_prob */
  double crossover_prob;    /* EmpcSettings.crossover_prob */
  const double* x0;         /* instances x n */
  const double* sigma;      /* instances x m: mutation std of empc.py:73-82 (host-computed, FP64) */
  const empc_injected* inject; /* NULL: in-kernel counter-based Philox4x32-10 */
  /* outputs, each may be NULL */
  double* u_out;            /* instances x m      (EmpcResult.u) */
  double* best_out;         /* instances x p x m  (EmpcResult.best) */
  double* best_cost;        /* instances          (EmpcResult.best_cost) */
  int32_t* best_index;      /* instances          (argmin row) */
} empc_run_args;

/* Run init / rescore / evolves as one device-resident sequence (graph-captured
 * when no injection is given).  Synchronous: returns after outputs are on the host.
 * Inside the graph the inputs (x0, sigma, run parameters and the problem
 * staging, <= 1 MB) are read from the handle's mapped pinned buffers by
 * kernels, the result block is stored into mapped pinned memory, and the
 * final population goes into slot_out (ids < 4 captured, others copied after);
 * a warm start reads slot_in in place and leaves it unchanged. */
int empc_run(empc_handle* h, const empc_run_args* args);

/* Score `num` candidates per instance at x0 (instances x n) with the rollout
 * kernel: cands instances x num x p x m -> costs instances x num. */
int empc_score(empc_handle* h, const double* x0, int32_t num, const double* cands, double* costs);

/* Stable selection on given costs (instances x N): elite_idx instances x K
 * (= argsort(kind="stable")[:K]) and best_index (= argmin, first NaN wins). */
int empc_select(empc_handle* h, const double* costs, int32_t* elite_idx, int32_t* best_index);

/* Knot expansion (kernel K1): cands num x p x m -> traj num x T x m. */
int empc_expand(empc_handle* h, int32_t num, const double* cands, double* traj);

/* Device-resident timing for bench.py: `reps` replays of the run described by
 * args with inputs already in HBM (no H2D/D2H inside the timed region).
 * ms_each[reps] receives each replay's CUDA-event time; when flush_l2 != 0 a
 * buffer larger than L2 is overwritten before each replay (untimed).
 * rollout_ms (may be NULL) receives the mean duration of one rollout
 * launch and rollout_launches the number of rollout launches per replay;
 * launches_per_rep the number of kernels per replay. */
int empc_time_device(empc_handle* h, const empc_run_args* args, int32_t reps, int32_t flush_l2,
                     float* ms_each, float* rollout_ms, int32_t* rollout_launches, int32_t* launches_per_rep);

/* Selected rollout variant for diagnostics: writes a short description. */
int empc_describe(empc_handle* h, char* buf, int32_t len);

/* Rollout kernel variants compiled for this handle's padded state size
 * (register blocking / A-in-registers choices); -1 restores the heuristic. */
int empc_num_variants(empc_handle* h, int32_t* count);
int empc_set_variant(empc_handle* h, int32_t variant);
/* Rollout CTAs per SM for the launch plan (0 restores the heuristic). */
int empc_set_occupancy(empc_handle* h, int32_t ctas_per_sm);
/* Tensor-core rollout (tcgen05, TF32 split precision, FP32 populations with a
 * diagonal Q): -1 = auto (default: where it measured faster than the FFMA
 * recursion), 0 = off, 1 = on.  Same function as the FFMA rollout
 * (K/empc.py:85-119); see DESIGN.md §4.8. */
int empc_set_tensor_cores(empc_handle* h, int32_t mode);

/* Execution-path options (same results contract on every path; used by the
 * parity tests to pin each path against the others):
 *   EMPC_OPT_PERSISTENT  -1 auto (default: one cooperative launch per solve for
 *                        single FP32 problems with n >= 24, i.e. C3), 0 per-
 *                        generation launches, 1 persistent whenever the shape fits
 *   EMPC_OPT_HALF_K      1 (default) skip the all-zero left half of the columns of
 *                        Ad - I in the persistent recursion when present; 0 full matvec
 *   EMPC_OPT_INCREMENTAL_SELECT 1 (default) after the first evolve rank only the
 *                        elites + the children that beat the K-th elite; 0 rank all N
 *   EMPC_OPT_RADIX_SELECT 1: selection by radix select of the K-th key and ranking
 *                        of the K elites only (default inside the persistent solve and
 *                        for single FP32 populations with N >= 8192, e.g. C4);
 *                        0: rank by counting everywhere
 *   EMPC_OPT_SMALL_SOLVE -1 auto (default: n <= 8 with little work, e.g. C1), 0 off,
 *                        1 whenever it fits: the whole solve in ONE CTA per instance
 *                        with the population resident in shared memory
 *   EMPC_OPT_PERSIST_TILE minimum candidates per CTA of the persistent solve (0
 *                        = one wave over the SMs; larger = fewer CTAs, cheaper grid syncs)
 * empc_describe reports the path the last run took. */
#define EMPC_OPT_PERSISTENT 1
#define EMPC_OPT_HALF_K 2
#define EMPC_OPT_INCREMENTAL_SELECT 3
#define EMPC_OPT_RADIX_SELECT 4
#define EMPC_OPT_PERSIST_TILE 5
#define EMPC_OPT_SMALL_SOLVE 6
int empc_set_option(empc_handle* h, int32_t option, int32_t value);

/* Population sharding over GPUs (K/empc.py:174-208 split
 * across ranks).  A rank holds the K elites (replicated) and the children of
 * global child indices [child_base, child_base + n_children) -- and, for the
 * cold start, the initial candidates [init_base, init_base + n_init).  The
 * handle's num_sims must be >= K + max(n_children, n_init).  Per generation:
 * empc_shard_export writes this rank's top-K candidates as K self-contained
 * entries of empc_shard_entry_bytes bytes into a DEVICE buffer; the caller
 * all-gathers the W buffers (NCCL over NVLink); empc_shard_import ranks the
 * W*K entries and installs the global top-K as elites (reporting the global
 * best); empc_shard_evolve breeds and scores this rank's children.  Keys use
 * global rows and the RNG counters global child indices, so the result is
 * identical to the unsharded solve for any world size. */
/* The shard calls are ASYNCHRONOUS on the handle's stream (empc_get_stream):
 * enqueue the collective on the same stream and a generation runs without a
 * host synchronisation.  empc_shard_init stages the problem, x0, sigma and the
 * RNG parameters once; empc_shard_evolve reads only args->generation0.
 * empc_shard_import synchronises only when an output pointer is given. */
int empc_shard_setup(empc_handle* h, int64_t child_base, int32_t n_children, int64_t init_base, int32_t n_init,
                     int32_t owns_elites);
int empc_shard_entry_bytes(empc_handle* h, int64_t* bytes);
int empc_shard_init(empc_handle* h, const empc_run_args* args);
int empc_shard_export(empc_handle* h, void* dev_entries);
int empc_shard_import(empc_handle* h, const void* dev_all, int32_t world, double* u_out, double* best_out,
                      double* best_cost, int64_t* best_row);
int empc_shard_evolve(empc_handle* h, const empc_run_args* args);
int empc_shard_read(empc_handle* h, double* cands, double* costs);
/* The handle's CUDA stream (a cudaStream_t), for enqueueing collectives after
 * empc_shard_export and before empc_shard_import. */
int empc_get_stream(empc_handle* h, void** stream);

/* Batched plant linearization + discretization on the device:
 * for each of `count` operating points (x[i], u[i]) of one plant, the
 * central-difference Jacobians of the plant ODE with step eps and the affine
 * residual (dynamics.py:241-262), then the zero-order-hold discretization
 * exp([[A B w],[0 0 0]] dt) (EMPC_DISCRETIZE_EXACT) or I + A dt, B dt, w dt
 * (EMPC_DISCRETIZE_EULER) (dynamics.py:265-290).  Plants: the torque pendulum
 * (dynamics.py:33-75; n = 2, m = 1, mass/length arrays of length 1) and the
 * planar N-link chain with tip masses (dynamics.py:90-199; n = 2 links,
 * m = links, links <= 64).  Host arrays: x [count][n], u [count][m] in;
 * Ad [count][n][n], Bd [count][n][m], wd [count][n] out.  No handle; errors
 * through empc_plant_last_error(). */
#define EMPC_PLANT_PENDULUM 0
#define EMPC_PLANT_NLINK 1
#define EMPC_DISCRETIZE_EXACT 0
#define EMPC_DISCRETIZE_EULER 1
typedef struct {
  int32_t kind;          /* EMPC_PLANT_* */
  int32_t links;         /* N-link: number of links; pendulum: 1 */
  const double* mass;    /* [links] tip masses (pendulum: [1]) */
  const double* length;  /* [links] link lengths */
  double damping;        /* joint viscous damping */
  double gravity;
} empc_plant;
int empc_plant_linearize_discretize(const empc_plant* plant, int32_t count, const double* x, const double* u,
                                    double eps, double dt, int32_t method, int32_t device, double* Ad, double* Bd,
                                    double* wd);
/* RK4 integration of one zero-order-hold period of the same plants
 * (dynamics.py:316-330): x_out[i] = integrate(f, x[i], u[i], dt, substeps). */
int empc_plant_integrate(const empc_plant* plant, int32_t count, const double* x, const double* u, double dt,
                         int32_t substeps, int32_t device, double* x_out);
const char* empc_plant_last_error(void);

/* Known-answer seam for the in-kernel counter-based RNG: Philox4x32-10 of
 * `count` (ctr[4], key[2]) pairs evaluated on the device. */
int empc_philox(const uint32_t* ctr, const uint32_t* key, int32_t count, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* EMPC_B200_H_ */
