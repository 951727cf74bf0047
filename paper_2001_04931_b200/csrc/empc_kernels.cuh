// Kernels of the B200 EMPC hot path.  Reference: /root/reference/pkg/src/
// knotmpc/empc.py (K/empc.py) and param.py (K/param.py).
//
//   prep_kernel     per-solve problem/state conversion (FP64 host layout ->
//                   working layout, Delta = Ad - I, cost of x0)
//   rollout_kernel  K2+K3 (+K5 prologue): breed/init/load candidates, B at
//                   the knots, horizon recursion, fused quadratic cost
//   select_kernel   K4: stable top-K (argsort(kind="stable")[:K])
//   finalize_kernel argmin + best candidate extraction (K/empc.py:234-236)
//   expand_kernel   K1: knots -> per-step inputs (K/param.py:114-116)
#pragma once

#include "empc_device.cuh"

namespace empc {

enum Mode : int { kScore = 0, kInitPhilox = 1, kInitInject = 2, kBreedPhilox = 3, kBreedInject = 4 };

// Offsets (elements of S) of one instance's working block.
struct Layout {
  int dm, bm, wd, qd, qf, r, xg, ug, umin, umax, x0, sig, qxg, cost0, stride;
};

// Offsets (doubles) of the FP64 staging block of one instance (C-ABI order).
struct StageLayout {
  int ad, bd, wd, q, r, xg, ug, umin, umax, stride;  // problem
  int x0, sig, sstride;                               // state
};

// RNG / operator parameters that change per run: kept in device memory so a
// captured graph stays valid across runs (K/empc.py:27-39 settings).
struct RunParams {
  uint64_t seed;
  int64_t gen0;
  uint64_t thr_cross;  // crossover_prob * 2^32 (Bernoulli by u32 < thr)
  uint64_t thr_mut;
};

struct Dims {
  int n, m, T, p, pm, N, K, NP;
};

// ---------------------------------------------------------------------------
// prep: one CTA per instance.

template <typename S>
__global__ void prep_kernel(Dims d, Layout L, StageLayout SL, const double* __restrict__ stage_prob,
                            const double* __restrict__ stage_state, S* __restrict__ work, int dense_q) {
  const int inst = blockIdx.x;
  const double* P = stage_prob + (size_t)inst * SL.stride;
  const double* X = stage_state + (size_t)inst * SL.sstride;
  S* w = work + (size_t)inst * L.stride;
  const int n = d.n, m = d.m;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    w[L.dm + e] = (S)(P[SL.ad + e] - (i == j ? 1.0 : 0.0));  // Delta = Ad - I (FP64 subtraction)
    if (dense_q) w[L.qf + e] = (S)P[SL.q + e];
  }
  for (int e = threadIdx.x; e < n * m; e += blockDim.x) w[L.bm + e] = (S)P[SL.bd + e];
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) w[L.r + e] = (S)P[SL.r + e];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w[L.wd + i] = (S)P[SL.wd + i];
    w[L.qd + i] = (S)P[SL.q + i * n + i];
    w[L.xg + i] = (S)P[SL.xg + i];
    w[L.x0 + i] = (S)X[SL.x0 + i];
    if (dense_q) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += P[SL.q + i * n + j] * P[SL.xg + j];
      w[L.qxg + i] = (S)s;
    }
  }
  for (int l = threadIdx.x; l < m; l += blockDim.x) {
    w[L.ug + l] = (S)P[SL.ug + l];
    w[L.umin + l] = (S)P[SL.umin + l];
    w[L.umax + l] = (S)P[SL.umax + l];
    w[L.sig + l] = (S)X[SL.sig + l];
  }
  // cost of x_0 (the k = 0 state term of K/empc.py:113-118), FP64, fixed-order
  // reduction so the result is deterministic
  __shared__ double red[256];
  double part = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double ei = X[SL.x0 + i] - P[SL.xg + i];
    if (dense_q) {
      double qe = 0.0;
      for (int j = 0; j < n; ++j) qe += P[SL.q + i * n + j] * (X[SL.x0 + j] - P[SL.xg + j]);
      part += ei * qe;
    } else {
      part += P[SL.q + i * n + i] * ei * ei;
    }
  }
  red[threadIdx.x] = part;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) w[L.cost0] = (S)red[0];
}

// ---------------------------------------------------------------------------
// rollout: K2 + K3 with the K5 breed / init prologue.

template <typename S>
struct RolloutArgs {
  Dims d;
  Layout L;
  int mode;
  int nc;     // candidates scored per instance by this launch
  int row0;   // first scored row in the population arrays (K when breeding)
  int rows;   // rows per instance of the population arrays
  int tile;   // candidates per CTA
  int tileP;  // tile rounded up to CC
  int pmS;    // padded gene stride of the smem knot buffer (odd)
  int evolve; // index of this evolve within the run (RNG generation = gen0 + evolve)
  const S* work;
  const int* idx1;
  const int* idx2;
  const S* cw;
  const S* G;  // W'W (p x p)
  const S* pop_in;
  const S* cost_in;
  S* pop_out;
  S* cost_out;
  const int* elite_idx;
  const RunParams* run;
  const int* inj_parents;
  const uint8_t* inj_take;
  const uint8_t* inj_mut;
  const double* inj_noise;
  const S* inj_init;
  const double* sig64;  // FP64 sigma (staging) for reference-exact injected mutation
  int sig64_stride;
};

// Shared memory plan (host and device agree on it).
struct SmemPlan {
  size_t us, but, xt, dt, qt, sched, g, cu, src, total;
};

template <typename S>
__host__ __device__ inline SmemPlan smem_plan(int NP, int n, int m, int T, int p, int tileP, int pmS, bool areg,
                                              bool dq) {
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  SmemPlan s;
  s.us = al((size_t)tileP * pmS * sizeof(S));
  s.but = al((size_t)p * NP * tileP * sizeof(S));
  const size_t xt_elems = (size_t)2 * NP * tileP;
  const size_t ru_elems = (size_t)tileP * m;
  s.xt = al((xt_elems > ru_elems ? xt_elems : ru_elems) * sizeof(S));
  s.dt = areg ? 0 : al((size_t)NP * NP * sizeof(S));
  s.qt = dq ? al((size_t)NP * NP * sizeof(S)) : 0;
  s.sched = al((size_t)T * (2 * sizeof(int) + sizeof(S)));
  s.g = al((size_t)p * p * sizeof(S));
  s.cu = al((size_t)tileP * sizeof(S));
  s.src = al((size_t)tileP * 2 * sizeof(int));
  s.total = s.us + s.but + s.xt + s.dt + s.qt + s.sched + s.g + s.cu + s.src;
  (void)n;
  return s;
}

template <typename S, int NP, int RR, int CC, bool AREG, bool DQ, int MAXT>
__global__ void __launch_bounds__(MAXT) rollout_kernel(const RolloutArgs<S> a) {
  constexpr int NRG = NP / RR;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Dims& d = a.d;
  const int n = d.n, m = d.m, T = d.T, p = d.p, pm = d.pm;
  const int tileP = a.tileP, pmS = a.pmS;
  const int inst = blockIdx.y;
  const int tile0 = blockIdx.x * a.tile;
  const int cnt = min(a.tile, a.nc - tile0);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const S* __restrict__ W = a.work + (size_t)inst * a.L.stride;

  const SmemPlan sp = smem_plan<S>(NP, n, m, T, p, tileP, pmS, AREG, DQ);
  unsigned char* ptr = smem_raw;
  S* Us = reinterpret_cast<S*>(ptr); ptr += sp.us;
  S* BUT = reinterpret_cast<S*>(ptr); ptr += sp.but;
  S* XT = reinterpret_cast<S*>(ptr); ptr += sp.xt;
  S* Dt = reinterpret_cast<S*>(ptr); ptr += sp.dt;
  S* Qt = reinterpret_cast<S*>(ptr); ptr += sp.qt;
  int* sI1 = reinterpret_cast<int*>(ptr);
  int* sI2 = sI1 + T;
  S* sC = reinterpret_cast<S*>(sI2 + T); ptr += sp.sched;
  S* sG = reinterpret_cast<S*>(ptr); ptr += sp.g;
  S* cU = reinterpret_cast<S*>(ptr); ptr += sp.cu;
  int* src = reinterpret_cast<int*>(ptr);

  const size_t pop_base = (size_t)inst * a.rows;
  const bool breed = (a.mode == kBreedPhilox || a.mode == kBreedInject);
  const RunParams rp = *a.run;
  const uint32_t key0 = (uint32_t)rp.seed, key1 = (uint32_t)(rp.seed >> 32);
  const uint32_t gen = (uint32_t)(rp.gen0 + a.evolve);

  // ---- elite carry-over (K/empc.py:186-188, 206): rows [0, K) of the next
  // population are the sorted elites with their carried costs.  Spread over
  // the instance's CTAs.
  if (breed) {
    for (int e = blockIdx.x; e < d.K; e += gridDim.x) {
      const int s = a.elite_idx[(size_t)inst * d.K + e];
      const S* from = a.pop_in + (pop_base + s) * pm;
      S* to = a.pop_out + (pop_base + e) * pm;
      for (int g = tid; g < pm; g += nthr) to[g] = from[g];
      if (tid == 0) a.cost_out[pop_base + e] = a.cost_in[pop_base + s];
    }
  }
  if (cnt <= 0) return;

  for (int k = tid; k < T; k += nthr) {
    sI1[k] = a.idx1[k];
    sI2[k] = a.idx2[k];
    sC[k] = a.cw[k];
  }
  for (int e = tid; e < p * p; e += nthr) sG[e] = a.G[e];

  // ---- candidate knots into smem (K5 prologue)
  if (breed) {
    // parents (K/empc.py:196): two uniform elite ranks per child
    for (int c = tid; c < cnt; c += nthr) {
      const int child = tile0 + c;
      int p1, p2;
      if (a.mode == kBreedInject) {
        const int* pp = a.inj_parents + ((size_t)inst * a.nc + child) * 2;
        p1 = pp[0];
        p2 = pp[1];
      } else {
        const U4 r = philox4x32_10(U4{kParentWord, (uint32_t)child, (uint32_t)inst, gen}, key0, key1);
        p1 = (int)mulhi32(r.x, (uint32_t)d.K);  // Lemire multiply-shift, unbiased to 2^-32
        p2 = (int)mulhi32(r.y, (uint32_t)d.K);
      }
      src[2 * c] = a.elite_idx[(size_t)inst * d.K + p1];
      src[2 * c + 1] = a.elite_idx[(size_t)inst * d.K + p2];
    }
    __syncthreads();
  }
  for (int e = tid; e < tileP * pm; e += nthr) {
    const int c = e / pm, g = e - (e / pm) * pm;
    S v = S(0);
    if (c < cnt) {
      const int l = g % m;
      const int cand = tile0 + c;
      if (a.mode == kScore) {
        v = a.pop_in[(pop_base + a.row0 + cand) * pm + g];
      } else if (a.mode == kInitPhilox) {
        const U4 r = philox4x32_10(U4{(uint32_t)g, (uint32_t)cand, (uint32_t)inst, kInitTag}, key0, key1);
        const S lo = W[a.L.umin + l], hi = W[a.L.umax + l];
        v = lo + (hi - lo) * uniform01<S>(r.x, r.y);  // numpy uniform(low, high), K/empc.py:170
        v = v > hi ? hi : v;
      } else if (a.mode == kInitInject) {
        v = a.inj_init[((size_t)inst * a.nc + cand) * pm + g];
      } else {
        // crossover, mutation, clip (K/empc.py:197-204)
        const size_t gi = ((size_t)inst * a.nc + cand) * pm + g;
        bool take, mut;
        if (a.mode == kBreedInject) {
          take = a.inj_take[gi] != 0;
          mut = a.inj_mut[gi] != 0;
        } else {
          const U4 r = philox4x32_10(U4{(uint32_t)g, (uint32_t)cand, (uint32_t)inst, gen}, key0, key1);
          take = (uint64_t)r.x < rp.thr_cross;
          mut = (uint64_t)r.y < rp.thr_mut;
          if (mut) {
            const S z = normal_bm<S>(r.z, r.w);
            v = z * W[a.L.sig + l];
          }
        }
        const S par = a.pop_in[(pop_base + src[2 * c + (take ? 1 : 0)]) * pm + g];
        if (a.mode == kBreedInject) {
          // reference arithmetic in FP64: child + mutate*noise*sigma
          const double nz = mut ? a.inj_noise[gi] * a.sig64[(size_t)inst * a.sig64_stride + l] : 0.0;
          v = (S)((double)par + nz);
        } else {
          v = par + v;
        }
        const S lo = W[a.L.umin + l], hi = W[a.L.umax + l];
        v = v < lo ? lo : (v > hi ? hi : v);
      }
      if (a.mode != kScore) a.pop_out[(pop_base + a.row0 + cand) * pm + g] = v;
    }
    Us[c * pmS + g] = v;
  }
  __syncthreads();

  // ---- B at the knots (+ w), interpolated later: drive = W (x) (U Bd') + wd
  // (K/empc.py:104-105).  Layout BUT[knot][row][cand].
  {
    const S* __restrict__ Bm = W + a.L.bm;
    const S* __restrict__ wd = W + a.L.wd;
    const int tot = p * NP * tileP;
    for (int e = tid; e < tot; e += nthr) {
      const int c = e % tileP;
      const int t = e / tileP;
      const int i = t % NP, j = t / NP;
      S v = S(0);
      if (i < n) {
        v = wd[i];
        const S* u = Us + c * pmS + j * m;
        const S* b = Bm + i * m;
        for (int l = 0; l < m; ++l) v = fma(b[l], u[l], v);
      }
      BUT[(j * NP + i) * tileP + c] = v;
    }
  }
  // ---- input cost as the knot quadratic z'(W'W (x) R)z, z = U - u_goal
  // (K/empc.py:100-101); per (candidate, channel) partials in XT scratch.
  {
    S* ru = XT;
    const S* __restrict__ R = W + a.L.r;
    const S* __restrict__ ug = W + a.L.ug;
    for (int e = tid; e < tileP * m; e += nthr) {
      const int c = e / m, l = e - (e / m) * m;
      S val = S(0);
      if (c < cnt) {
        const S* u = Us + c * pmS;
        if (p <= 8) {
          S gz[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) gz[q] = S(0);
          for (int b = 0; b < p; ++b) {
            S rz = S(0);
            for (int l2 = 0; l2 < m; ++l2) rz = fma(R[l * m + l2], u[b * m + l2] - ug[l2], rz);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < p) gz[q] = fma(sG[q * p + b], rz, gz[q]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < p) val = fma(u[q * m + l] - ug[l], gz[q], val);
        } else {
          for (int q = 0; q < p; ++q) {
            S gzq = S(0);
            for (int b = 0; b < p; ++b) {
              S rz = S(0);
              for (int l2 = 0; l2 < m; ++l2) rz = fma(R[l * m + l2], u[b * m + l2] - ug[l2], rz);
              gzq = fma(sG[q * p + b], rz, gzq);
            }
            val = fma(u[q * m + l] - ug[l], gzq, val);
          }
        }
      }
      ru[e] = val;
    }
    __syncthreads();
    for (int c = tid; c < tileP; c += nthr) {
      S s = S(0);
      for (int l = 0; l < m; ++l) s += ru[c * m + l];
      cU[c] = s;
    }
  }
  // ---- model into registers / smem (A as Delta = Ad - I)
  const int rg = tid % NRG, cg = tid / NRG;
  const bool active = cg * CC < tileP;
  S areg[AREG ? RR : 1][AREG ? NP : 1];
  if constexpr (AREG) {
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const int row = rg * RR + r;
#pragma unroll
      for (int j = 0; j < NP; ++j) areg[r][j] = (row < n && j < n) ? W[a.L.dm + row * n + j] : S(0);
    }
  } else {
    for (int e = tid; e < NP * NP; e += nthr) {
      const int j = e / NP, i = e % NP;
      Dt[e] = (i < n && j < n) ? W[a.L.dm + i * n + j] : S(0);
      if constexpr (DQ) Qt[e] = (i < n && j < n) ? W[a.L.qf + i * n + j] : S(0);
    }
  }
  S qv[RR], xgv[RR], qxg[RR];
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const int row = rg * RR + r;
    qv[r] = (row < n && !DQ) ? W[a.L.qd + row] : S(0);
    xgv[r] = row < n ? W[a.L.xg + row] : S(0);
    qxg[r] = (row < n && DQ) ? W[a.L.qxg + row] : S(0);
  }
  __syncthreads();  // ru (in XT) consumed; Dt/Qt/BUT visible
  // x_0 = x0 for every candidate (K/empc.py:109)
  for (int e = tid; e < NP * tileP; e += nthr) {
    const int i = e / tileP;
    XT[e] = i < n ? W[a.L.x0 + i] : S(0);
  }
  S xo[RR][CC];
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const int row = rg * RR + r;
    const S x0r = row < n ? W[a.L.x0 + row] : S(0);
#pragma unroll
    for (int c = 0; c < CC; ++c) xo[r][c] = x0r;
  }
  S cst[CC];
#pragma unroll
  for (int c = 0; c < CC; ++c) cst[c] = S(0);
  __syncthreads();

  // ---- horizon recursion x_{k+1} = x_k + Delta x_k + drive_k
  // (K/empc.py:110-112), state cost fused per step (K/empc.py:113-118)
  const int col = cg * CC;
  for (int k = 0; k < T; ++k) {
    const S* xc = XT + (k & 1) * NP * tileP;
    S* xnb = XT + ((k & 1) ^ 1) * NP * tileP;
    S acc[RR][CC];
    S qacc[DQ ? RR : 1][DQ ? CC : 1];
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
      for (int c = 0; c < CC; ++c) acc[r][c] = S(0);
    if constexpr (DQ) {
#pragma unroll
      for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int c = 0; c < CC; ++c) qacc[r][c] = S(0);
    }
    if (active) {
#pragma unroll(AREG ? NP : 16)
      for (int j = 0; j < NP; ++j) {
        S xv[CC];
        lds_vec<S, CC>(xc + j * tileP + col, xv);
        S av[RR];
        if constexpr (AREG) {
#pragma unroll
          for (int r = 0; r < RR; ++r) av[r] = areg[r][j];
        } else {
          lds_vec<S, RR>(Dt + j * NP + rg * RR, av);
        }
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int c = 0; c < CC; ++c) acc[r][c] = fma(av[r], xv[c], acc[r][c]);
        if constexpr (DQ) {
          S qa[RR];
          lds_vec<S, RR>(Qt + j * NP + rg * RR, qa);
#pragma unroll
          for (int r = 0; r < RR; ++r)
#pragma unroll
            for (int c = 0; c < CC; ++c) qacc[r][c] = fma(qa[r], xv[c], qacc[r][c]);
        }
      }
      const int i1 = sI1[k], i2 = sI2[k];
      const S ck = sC[k], c1 = S(1) - ck;
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const int row = rg * RR + r;
        S b1[CC], b2[CC];
        lds_vec<S, CC>(BUT + (i1 * NP + row) * tileP + col, b1);
        lds_vec<S, CC>(BUT + (i2 * NP + row) * tileP + col, b2);
        S xn[CC];
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          if constexpr (DQ) {
            const S e0 = xo[r][c] - xgv[r];
            cst[c] = fma(e0, qacc[r][c] - qxg[r], cst[c]);  // cost of x_k
          }
          const S drive = fma(ck, b2[c], c1 * b1[c]);
          xn[c] = xo[r][c] + (acc[r][c] + drive);
          xo[r][c] = xn[c];
          if constexpr (!DQ) {
            const S e = xn[c] - xgv[r];
            cst[c] = fma(qv[r] * e, e, cst[c]);  // cost of x_{k+1}, diagonal Q
          }
        }
        sts_vec<S, CC>(xnb + row * tileP + col, xn);
      }
    }
    __syncthreads();
  }
  if constexpr (DQ) {
    // terminal state term e_T' Q e_T
    if (active) {
      const S* xc = XT + (T & 1) * NP * tileP;
      S qacc[RR][CC];
#pragma unroll
      for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int c = 0; c < CC; ++c) qacc[r][c] = S(0);
#pragma unroll 8
      for (int j = 0; j < NP; ++j) {
        S xv[CC], qa[RR];
        lds_vec<S, CC>(xc + j * tileP + col, xv);
        lds_vec<S, RR>(Qt + j * NP + rg * RR, qa);
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int c = 0; c < CC; ++c) qacc[r][c] = fma(qa[r], xv[c], qacc[r][c]);
      }
#pragma unroll
      for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int c = 0; c < CC; ++c) cst[c] = fma(xo[r][c] - xgv[r], qacc[r][c] - qxg[r], cst[c]);
    }
  }
  // ---- deterministic reduction over row groups (BUT is free now)
  S* red = BUT;
  if (active) {
#pragma unroll
    for (int c = 0; c < CC; ++c) red[rg * tileP + col + c] = cst[c];
  }
  __syncthreads();
  const S c0 = DQ ? S(0) : W[a.L.cost0];
  for (int c = tid; c < cnt; c += nthr) {
    S s = S(0);
    for (int g = 0; g < NRG; ++g) s += red[g * tileP + c];
    a.cost_out[pop_base + a.row0 + tile0 + c] = c0 + cU[c] + s;
  }
}

// ---------------------------------------------------------------------------
// K4 selection: bitonic sort of (cost, index) keys in shared memory, one CTA
// per instance; rows [0, K) of the sorted order are the elites.

template <typename S>
__global__ void __launch_bounds__(1024) select_kernel(const S* __restrict__ costs, int N, int K, int NP2,
                                                      int* __restrict__ elite_idx) {
  using KT = typename KeyOf<S>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KT* keys = reinterpret_cast<KT*>(smem_raw);
  const int inst = blockIdx.x;
  const S* c = costs + (size_t)inst * N;
  for (int i = threadIdx.x; i < NP2; i += blockDim.x) keys[i] = i < N ? KeyOf<S>::make(c[i], i) : KeyOf<S>::pad();
  __syncthreads();
  const int half = NP2 >> 1;
  for (int k = 2; k <= NP2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        const int lo = 2 * j * (t / j) + (t % j);
        const int hi = lo + j;
        const bool asc = (lo & k) == 0;
        const KT a = keys[lo], b = keys[hi];
        if ((b < a) == asc) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < K; e += blockDim.x) elite_idx[(size_t)inst * K + e] = keys[e].idx();
}

// ---------------------------------------------------------------------------
// finalize: argmin (first NaN, else first minimum: numpy argmin) and the
// best candidate, written as FP64 [u (m) | best (pm) | cost | index].

template <typename S>
__global__ void finalize_kernel(const S* __restrict__ cands, const S* __restrict__ costs, int N, int m, int pm,
                                double* __restrict__ out) {
  const int inst = blockIdx.x;
  const S* c = costs + (size_t)inst * N;
  uint64_t bo = ~0ull;
  int bi = 0x7FFFFFFF;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const S v = c[i];
    uint64_t o;
    if constexpr (sizeof(S) == 4) o = (v != v) ? 0ull : (uint64_t)ord32((float)v);
    else o = (v != v) ? 0ull : ord64((double)v);
    if (o < bo || (o == bo && i < bi)) { bo = o; bi = i; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t o2 = __shfl_down_sync(0xFFFFFFFFu, bo, off);
    const int i2 = __shfl_down_sync(0xFFFFFFFFu, bi, off);
    if (o2 < bo || (o2 == bo && i2 < bi)) { bo = o2; bi = i2; }
  }
  __shared__ uint64_t so[32];
  __shared__ int si[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { so[wid] = bo; si[wid] = bi; }
  __syncthreads();
  __shared__ int best;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int w = 1; w < nw; ++w)
      if (so[w] < so[0] || (so[w] == so[0] && si[w] < si[0])) { so[0] = so[w]; si[0] = si[w]; }
    best = si[0];
  }
  __syncthreads();
  const int stride = m + pm + 2;
  double* o = out + (size_t)inst * stride;
  if (cands != nullptr) {
    const S* bc = cands + ((size_t)inst * N + best) * pm;
    for (int g = threadIdx.x; g < pm; g += blockDim.x) {
      o[m + g] = (double)bc[g];
      if (g < m) o[g] = (double)bc[g];  // u = first knot (K/empc.py:236)
    }
  }
  if (threadIdx.x == 0) {
    o[m + pm] = (double)c[best];
    o[m + pm + 1] = (double)best;
  }
}

// ---------------------------------------------------------------------------
// K1: knot expansion u_k = (1 - c_k) U[idx1_k] + c_k U[idx2_k] (K/param.py:91-116)

template <typename S>
__global__ void expand_kernel(const S* __restrict__ cands, int num, int T, int p, int m, const int* __restrict__ idx1,
                              const int* __restrict__ idx2, const S* __restrict__ cw, double* __restrict__ traj) {
  const size_t tot = (size_t)num * T * m;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(e % m);
    const size_t t = e / m;
    const int k = (int)(t % T);
    const size_t c = t / T;
    const S* U = cands + c * (size_t)p * m;
    const S ck = cw[k];
    const S v = ck == S(0) ? U[idx1[k] * m + l] : fma(ck, U[idx2[k] * m + l], (S(1) - ck) * U[idx1[k] * m + l]);
    traj[e] = (double)v;
  }
}

// precision conversion helpers
template <typename S>
__global__ void cast_kernel(const double* __restrict__ in, S* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (S)in[i];
}
template <typename S>
__global__ void uncast_kernel(const S* __restrict__ in, double* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

// L2 flush for timing hygiene (writes a buffer larger than the 126 MB L2)
__global__ void flush_kernel(uint4* buf, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_uint4(v, v, v, v);
}

__global__ void philox_kernel(const uint32_t* ctr, const uint32_t* key, int count, uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const U4 r = philox4x32_10(U4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, key[2 * i], key[2 * i + 1]);
  out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
}

}  // namespace empc
