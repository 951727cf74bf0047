// Resident single-CTA solve for small problems (empc_small.cu): the whole
// EMPC solve of one instance in one CTA, population in shared memory.
#pragma once

#include "empc_kernels.cuh"

namespace empc {

// population and costs taken as they are (evolve_generation on a scored population)
constexpr int kSmallResident = 16;

template <typename S>
struct SmallArgs {
  Dims d;
  StageLayout SL;
  int mode;      // kInitPhilox, kInitInject, kScore (re-score pop_io, warm start) or kSmallResident
  int evolves;
  int r_diag;
  const double* prob;
  const double* state;
  const RunParams* run;
  const int* idx1;
  const int* idx2;
  const int* seg;
  const S* cw;
  const S* G;
  const S* pop_in;   // instances x N x pm: read when mode == kScore / kSmallResident
  const S* cost_in;  // instances x N: read when mode == kSmallResident
  S* pop_io;     // instances x N x pm: final population out (may be the caller's output slot)
  S* cost_io;    // instances x N
  // prob / state / run / out may point at mapped pinned host memory (the
  // public-API graph): the kernel copies the staging blocks into shared
  // memory once and writes the result block once
  double* out;   // instances x [u (m) | best (pm) | cost | index]
  const S* inj_init;
  // evolves x instances x (N-K) x {2 | pm} (NULL: in-kernel Philox)
  const int* inj_parents;
  const uint8_t* inj_take;
  const uint8_t* inj_mut;
  const double* inj_noise;
  unsigned long long* dbg;  // EMPC_PHASES: [5] cycles of thread 0 per phase (select keys, rank, draws, breed, score)
};

template <typename S>
using SmallKernel = void (*)(const SmallArgs<S>);

template <typename S>
size_t small_smem(int n, int m, int T, int p, int N, int K);
template <typename S>
SmallKernel<S> small_kernel(int n);  // NULL when n > 8

}  // namespace empc
