// Condensed (knot-space quadratic) scorer -- SURVEY §8 row f2.
//
// The reference scores candidates with the condensed quadratic of
// `_CostModel` (K/empc.py:122-152), built once per solve by
// `build_small_param` (K/condense.py:128-141, 197-202, 235-251, 268-274).
// Here the same function is evaluated around the reference input
// ref = u_goal stacked over the knots, which removes the cancellation of the
// reference's `z'Pz + 2q'z + c0` form (J(ref) is a cost, P ref + q a small
// gradient):
//
//   J(z) = (z-ref)' P (z-ref) + 2 g'(z-ref) + J_ref
//   P     = sum_k S_k' Q S_k + (W'W) (x) R          (K/condense.py:245-247)
//   g     = sum_k S_k' Q e_ref(k+1)                 (= q + P ref)
//   J_ref = sum_{k=0..T} e_ref(k)' Q e_ref(k)       (rollout of u = u_goal)
//
// with S_k (n x pm) the knot-to-x_{k+1} sensitivity S_k = Ad S_{k-1} +
// W[k] (x) Bd (K/condense.py:135-139) and e_ref the goal error of the u_goal
// trajectory.  Build and scoring run in FP64 whatever the population
// precision (the quadratic form has no cancellation-free FP32 evaluation).
#pragma once

#include <cuda_runtime.h>

#include "empc_kernels.cuh"

namespace empc {

// per-instance layout of the condensed model (doubles)
struct CondLayout {
  int P, g, ref, jref, stride;
};
__host__ __device__ inline CondLayout cond_layout(int pm) {
  CondLayout L;
  L.P = 0;
  L.g = pm * pm;
  L.ref = L.g + pm;
  L.jref = L.ref + pm;
  L.stride = (L.jref + 2) & ~1;
  return L;
}

struct CondBuild {
  int n, m, T, p, pm;
  StageLayout SL;
  const double* prob;   // FP64 problem staging (instances x SL.stride)
  const double* state;  // FP64 state staging (x0)
  const double* W;      // [T][p] interpolation matrix (K/param.py:91-104)
  const double* G;      // [p][p] W'W
  double* S;            // [chunk][T][n][pm] sensitivities
  double* QS;           // dense Q only: [chunk][T][n][pm] = Q S_k
  double* E;            // [chunk][T*n + 1]: Q e_ref(k+1) for k < T, then J_ref
  double* part;         // [chunk][splits][pm][pm + 1] split-K partials of [P | g]
  double* cond;         // [instances][cond_layout(pm).stride]
  int inst0;            // first instance of this chunk
  int cb;               // sensitivity columns per CTA
  int ksp;              // lanes per dot product in the sensitivity recursion
  int splits;           // split-K factor of the Gram kernel
  int dense;            // Q not diagonal
};

// launch geometry + kernels, instantiated in empc_cond.cu
template <typename S>
struct CondKernels {
  void (*prep)(CondBuild);            // grid (chunks + 1, instances): S recursion + u_goal trajectory
  void (*gram)(CondBuild);            // grid (tiles, splits, instances): [P | g] partials
  void (*finish)(CondBuild);          // grid (instances): reduce partials, + W'W (x) R, mirror
  void (*score_smem)(RolloutArgs<S>);  // breed + score, P in shared memory
  void (*score_glob)(RolloutArgs<S>);  // breed + score, P read through L1/L2
};
template <typename S>
CondKernels<S> cond_kernels();

size_t cond_prep_smem(int n, int cb, int dense);
constexpr int kCondTile = 32;    // Gram kernel output tile
constexpr int kCondRB = 4;       // rows per scoring thread chunk
constexpr int kCondCC = 2;       // candidates per scoring thread
constexpr int kCondMaxTile = 64; // candidates per scoring CTA

// shared-memory plan of the scoring kernel (host and device agree)
struct CondSmem {
  size_t us, src, bits, vec, ps, gv, zt, total;
  int pmS, tPS, nslices;
};
template <typename S>
__host__ __device__ inline CondSmem cond_smem(int pm, int m, int tileP, int nthreads, bool psm) {
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  CondSmem c;
  c.tPS = (tileP + 1) & ~1;
  c.pmS = ((pm + kCondRB - 1) / kCondRB) * kCondRB;
  const int ncg = (tileP + kCondCC - 1) / kCondCC;
  c.nslices = nthreads / ncg;
  c.us = al((size_t)c.pmS * c.tPS * sizeof(S));  // rows [pm, pmS) stay zero
  c.src = al((size_t)tileP * 2 * sizeof(int));
  c.bits = al((size_t)tileP * pm + 16);  // crossover choice, 1 byte per gene
  c.vec = al((size_t)3 * m * sizeof(S));
  c.ps = psm ? al((size_t)c.pmS * (c.pmS + 2) * sizeof(double)) : 0;
  c.gv = al((size_t)2 * c.pmS * sizeof(double));
  c.zt = al((size_t)c.pmS * c.tPS * sizeof(double));  // z - ref in FP64, [gene][cand]
  // the per-chunk partial sums ((pmS / kCondRB) x tPS doubles) overlay `us`
  c.total = c.us + c.src + c.bits + c.vec + c.ps + c.gv + c.zt;
  return c;
}

}  // namespace empc
