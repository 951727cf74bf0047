// Kernels of the B200 EMPC hot path.  Reference: /root/reference/pkg/src/
// knotmpc/empc.py (K/empc.py) and param.py (K/param.py).
//
//   rollout_kernel  K2+K3 (+K5 prologue): breed / init / load candidates,
//                   B at the knots, horizon recursion, fused quadratic cost.
//                   Reads the FP64 problem staging directly (no prep pass).
//   select_kernel   K4: stable top-K (argsort(kind="stable")[:K]) by a
//                   bitwise radix search for the K-th smallest (cost, index)
//                   key, compaction, and rank-by-counting of the K survivors
//   finalize_kernel argmin + best candidate extraction (K/empc.py:234-236)
//   expand_kernel   K1: knots -> per-step inputs (K/param.py:114-116)
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "empc_device.cuh"

namespace empc {

enum Mode : int { kScore = 0, kInitPhilox = 1, kInitInject = 2, kBreedPhilox = 3, kBreedInject = 4 };

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
  uint64_t thr_cross;  // round(crossover_prob * 2^32): Bernoulli by a 32-bit uniform < thr
  uint64_t thr_mut;
};

struct Dims {
  int n, m, T, p, pm, N, K, NP;
};

template <typename S>
struct RolloutArgs {
  Dims d;
  StageLayout SL;
  int mode;
  int r_diag;  // R diagonal: input cost fast path
  int nc;      // candidates scored per instance by this launch
  int row0;    // first scored row in the population arrays (K when breeding)
  int rows;    // rows per instance of the population arrays
  int tile;    // candidates per CTA
  int tileP;   // tile rounded up to CC
  int tPS;     // padded candidate stride of the knot / drive buffers
  int evolve;  // index of this evolve within the run (RNG generation = gen0 + evolve)
  int cand_base;  // global index of candidate 0 of this launch (population sharding; RNG counters)
  int copy_elites;  // 1: this launch copies the elite rows (0 when the selection kernel did)
  const double* prob;   // FP64 problem staging, instances x SL.stride
  const double* state;  // FP64 state staging (x0, sigma), instances x SL.sstride
  const int* idx1;
  const int* idx2;
  const int* seg;  // seg[k]: end (exclusive) of the run of steps with k's knot pair
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
  unsigned long long* dbg;  // optional per-CTA phase timestamps (globaltimer, ns)
  int* qcount;              // per instance: children that beat the K-th elite (incremental selection)
  void* qlist;              // per instance: [qcap] (ord key, row) pairs
  int qcap;
  const double* cond;       // condensed scorer: per instance P, g, ref, J_ref (empc_cond.h)
  int cstride;              // doubles per instance of `cond`
  int tc_multi;             // tensor-core rollout: each CTA loops over tiles (Delta staged once per CTA)
  int stagger;              // WS recursion: start delay (cycles) of warps 4-7 (sub-partition phase offset)
  // persistent solve:
  int parents_from_out;     // elites already at rows [0, K) of pop_out (read parents there)
  int draws_ready;          // phase 1a done for this tile (helper warps drew it in the previous generation)
  int draw_next;            // helper warps draw evolve `draw_evolve`'s tile during the recursion
  int draw_evolve;
  int draw_tile0, draw_cnt; // that tile (children [draw_tile0, draw_tile0 + draw_cnt))
  unsigned long long* amin; // last generation of the persistent solve: argmin key of the population
};

// doubles per instance in the problem staging block [Ad | Bd | wd | Q | R |
// x_goal | u_goal | u_min | u_max], padded even (16-byte aligned blocks);
// the layout is StageLayout (set by the engine)
__host__ __device__ inline int stage_stride(int n, int m) {
  const int s = 2 * n * n + n * m + 2 * n + m * m + 3 * m;
  return s + (s & 1);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define EMPC_MARK(I)                                                                                  \
  if (a.dbg != nullptr && threadIdx.x == 0)                                                          \
    a.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (I)] = gtimer();

template <typename S>
struct Geo {
  static constexpr int VEC = 16 / (int)sizeof(S);  // elements per 16-byte LDS
  // padded state stride: odd number of 16-byte chunks -> conflict-free rows
  __host__ __device__ static constexpr int nps(int NP) { return ((NP / VEC) % 2 == 0) ? NP + VEC : NP; }
};

// Shared memory plan (host and device agree on it).
struct SmemPlan {
  size_t us, but, xc, as, qs, sched, g, cu, src, cv, bs, off, total;
};

template <typename S>
__host__ __device__ inline SmemPlan smem_plan(int NP, int m, int T, int p, int tileP, int tPS, bool areg, bool dq,
                                              size_t persist_scratch = 0) {
  // persist_scratch > 0: persistent solve -- B gets its own region (it is
  // reused every generation) and the leading scratch (UsT, BUT, XC) is at
  // least persist_scratch bytes (the in-kernel selection's key arrays)
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const int NPS = Geo<S>::nps(NP);
  (void)areg;
  SmemPlan s;
  s.us = al((size_t)p * m * tPS * sizeof(S));
  s.but = al((size_t)p * NP * tPS * sizeof(S));
  const size_t xc = (size_t)2 * tileP * NPS, bs = (size_t)NP * (m + 1);
  s.xc = al(((persist_scratch || xc > bs) ? xc : bs) * sizeof(S));
  if (persist_scratch && s.us + s.but + s.xc < persist_scratch) s.xc += al(persist_scratch - (s.us + s.but + s.xc));
  s.bs = persist_scratch ? al(bs * sizeof(S)) : 0;
  s.as = al((size_t)NP * NPS * sizeof(S));  // A staging (copied to registers by AREG variants)
  s.qs = dq ? al((size_t)NP * NPS * sizeof(S)) : 0;
  s.sched = al((size_t)T * (3 * sizeof(int) + sizeof(S)));
  s.g = al((size_t)(p * p + 2) * sizeof(S));
  s.cu = al((size_t)tileP * sizeof(S));
  s.src = al((size_t)tileP * 2 * sizeof(int));
  s.cv = al((size_t)(4 * NP + 5 * m) * sizeof(S) + (size_t)tileP * p * m + 16);
  // persistent solve: mutation offsets of the next generation's draws (the
  // leading scratch is reused by the selection between generations)
  s.off = persist_scratch ? al((size_t)p * m * tPS * sizeof(S)) : 0;
  s.total = s.us + s.but + s.xc + s.as + s.qs + s.sched + s.g + s.cu + s.src + s.cv + s.bs + s.off;
  return s;
}

__device__ __forceinline__ uint32_t ord_key(float c) { return ord32(c); }
// numpy argmin order as one 64-bit key: NaN first, then by value, then row
__device__ __forceinline__ unsigned long long amin_key(float c, int row) {
  return ((unsigned long long)((c != c) ? 0u : ord32(c)) << 32) | (unsigned)row;
}
__device__ __forceinline__ unsigned long long amin_key(double c, int row) {
  // FP64: the top 32 bits of the orderable key, ties resolved by the full scan
  return ((unsigned long long)((c != c) ? 0u : (uint32_t)(ord64(c) >> 32)) << 32) | (unsigned)row;
}
__device__ __forceinline__ uint64_t ord_key(double c) { return ord64(c); }

// Programmatic dependent launch: wait for the producer grid (no-op when the
// kernel was launched without the attribute) / let the consumer grid start.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------
// K5 random draws of one tile of children (K/empc.py:195-199), counter-based
// Philox4x32-10 keyed by the 64-bit seed, by threads [t0, t0 + nt) of the CTA:
//   parents: counter (0xFFFFFFFF, child, instance, generation), x / y ->
//            two uniform elite ranks by Lemire's multiply-shift (K/empc.py:196);
//   genes:   per PAIR of genes (2q, 2q+1) counter (q, child, instance,
//            generation): x / y -> 32-bit crossover uniforms, z / w -> 32-bit
//            mutation uniforms, Bernoulli by u32 < round(prob * 2^32)
//            (K/empc.py:197-198); when either gene mutates, counter
//            (q | 2^31, child, instance, generation): z / w -> a Box-Muller
//            pair of standard normals scaled by sigma (K/empc.py:199, 202-203).
// Writes src[2c..2c+1] (ranks), tbits[c * pm + g] and off[g * tPS + c].
template <typename S>
__device__ __forceinline__ void draw_tile(const RunParams& rp, uint32_t gen, int K, int pm, int m, int inst,
                                          int cand0, int cnt, int tPS, int t0, int nt, int* src, uint8_t* tbits,
                                          S* off, const S* csig) {
  const uint32_t key0 = (uint32_t)rp.seed, key1 = (uint32_t)(rp.seed >> 32);
  for (int c = t0; c < cnt; c += nt) {
    const U4 r = philox4x32_10(U4{kParentWord, (uint32_t)(cand0 + c), (uint32_t)inst, gen}, key0, key1);
    src[2 * c] = (int)mulhi32(r.x, (uint32_t)K);
    src[2 * c + 1] = (int)mulhi32(r.y, (uint32_t)K);
  }
  const int hp = (pm + 1) >> 1;
  const uint64_t tc = rp.thr_cross, tm = rp.thr_mut;
#pragma unroll 2
  for (int e = t0; e < cnt * hp; e += nt) {
    const int c = e / hp, q = e - c * hp;
    const int g0 = 2 * q, g1 = g0 + 1;
    const bool two = g1 < pm;
    const int l0 = g0 % m;
    const int l1 = (l0 + 1 == m) ? 0 : l0 + 1;
    const uint32_t cand = (uint32_t)(cand0 + c);
    const U4 r = philox4x32_10(U4{(uint32_t)q, cand, (uint32_t)inst, gen}, key0, key1);
    const bool m0 = (uint64_t)r.z < tm, m1 = two && (uint64_t)r.w < tm;
    S n0 = S(0), n1 = S(0);
    if (m0 || m1) {
      const U4 b = philox4x32_10(U4{(uint32_t)q | 0x80000000u, cand, (uint32_t)inst, gen}, key0, key1);
      normal_pair<S>(b.z, b.w, n0, n1);
    }
    tbits[c * pm + g0] = (uint64_t)r.x < tc;
    off[g0 * tPS + c] = m0 ? n0 * csig[l0] : S(0);
    if (two) {
      tbits[c * pm + g1] = (uint64_t)r.y < tc;
      off[g1 * tPS + c] = m1 ? n1 * csig[l1] : S(0);
    }
  }
}

// K5 prologue shared by the rollout and the condensed scorer: random draws
// (phase 1a, independent of the producer grid; skipped when a.draws_ready --
// the persistent solve's helper warps drew them during the previous
// recursion), then -- after the PDL wait -- the elite carry-over and the
// tile's candidate knots into UsT[gene][cand] (phase 1b).  `off` holds the
// mutation offsets (UsT itself, or a dedicated buffer in the persistent
// solve).  Returns false when the CTA has no candidates.
template <typename S>
__device__ __forceinline__ bool breed_tile(const RolloutArgs<S>& a, int inst, int tile0, int cnt, int tileP, int tPS,
                                           S* UsT, int* src, uint8_t* tbits, const S* cumin, const S* cumax,
                                           const S* csig, size_t pop_base, bool elites = true, S* off = nullptr) {
  const Dims& d = a.d;
  const int m = d.m, pm = d.pm;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const double* __restrict__ X = a.state + (size_t)inst * a.SL.sstride;
  const StageLayout& SL = a.SL;
  const bool breed = (a.mode == kBreedPhilox || a.mode == kBreedInject);
  if (off == nullptr) off = UsT;
  // ---- phase 1a: random draws -- counter-based, so also independent of the
  // producer grid (the run parameters are staged by the host copy)
  const RunParams rp = *a.run;
  const uint32_t key0 = (uint32_t)rp.seed, key1 = (uint32_t)(rp.seed >> 32);
  const uint32_t gen = (uint32_t)(rp.gen0 + a.evolve);
  const bool philox_breed = a.mode == kBreedPhilox;
  if (cnt > 0) {
    if (a.mode == kBreedInject) {
      for (int c = tid; c < cnt; c += nthr) {
        const int* pp = a.inj_parents + ((size_t)inst * a.nc + tile0 + c) * 2;
        src[2 * c] = pp[0];
        src[2 * c + 1] = pp[1];
      }
    } else if (philox_breed) {
      if (!a.draws_ready)
        draw_tile<S>(rp, gen, d.K, pm, m, inst, a.cand_base + tile0, cnt, tPS, tid, nthr, src, tbits, off, csig);
    } else if (a.mode == kInitPhilox) {
      // two uniform initial knots per Philox call (K/empc.py:170): genes 2q
      // from (x, y), 2q + 1 from (z, w), counter (q, cand, instance, "INIT")
      const int hp = (pm + 1) >> 1;
#pragma unroll 2
      for (int e = tid; e < cnt * hp; e += nthr) {
        const int c = e / hp, q = e - c * hp;
        const int g0 = 2 * q, g1 = g0 + 1;
        const int l0 = g0 % m;
        const int l1 = (l0 + 1 == m) ? 0 : l0 + 1;
        const uint32_t cand = (uint32_t)(a.cand_base + tile0 + c);
        const U4 r = philox4x32_10(U4{(uint32_t)q, cand, (uint32_t)inst, kInitTag}, key0, key1);
        const S lo0 = cumin[l0], hi0 = cumax[l0];
        const S v0 = lo0 + (hi0 - lo0) * uniform01<S>(r.x, r.y);  // numpy uniform(low, high)
        UsT[g0 * tPS + c] = v0 > hi0 ? hi0 : v0;
        if (g1 < pm) {
          const S lo1 = cumin[l1], hi1 = cumax[l1];
          const S v1 = lo1 + (hi1 - lo1) * uniform01<S>(r.z, r.w);
          UsT[g1 * tPS + c] = v1 > hi1 ? hi1 : v1;
        }
      }
    }
  }

  EMPC_MARK(1)
  // ---- phase 1b: everything below reads the producer grid's outputs
  pdl_wait();
  EMPC_MARK(2)
  // elite carry-over (K/empc.py:186-188, 206): rows [0, K) of the next
  // population are the sorted elites with their carried costs.
  if (breed && a.copy_elites && elites) {  // otherwise the selection kernel already did
    for (int e = blockIdx.x; e < d.K; e += gridDim.x) {
      const int s = a.elite_idx[(size_t)inst * d.K + e];
      const S* from = a.pop_in + (pop_base + s) * pm;
      S* to = a.pop_out + (pop_base + e) * pm;
      for (int g = tid; g < pm; g += nthr) to[g] = from[g];
      if (tid == 0) a.cost_out[pop_base + e] = a.cost_in[pop_base + s];
    }
  }
  if (cnt <= 0) return false;
  EMPC_MARK(9)
  // parent rows: elite rank r is row elite_idx[r] of pop_in -- or row r of
  // pop_out when the selection already carried the elites over (persistent
  // solve: no dependent index load)
  const S* __restrict__ parents = a.parents_from_out ? a.pop_out : a.pop_in;
  if (breed && !a.parents_from_out) {
    for (int c = tid; c < cnt; c += nthr) {  // elite ranks -> population rows
      src[2 * c] = a.elite_idx[(size_t)inst * d.K + src[2 * c]];
      src[2 * c + 1] = a.elite_idx[(size_t)inst * d.K + src[2 * c + 1]];
    }
  }
  __syncthreads();  // src, phase-0/1a smem
  EMPC_MARK(10)
  // candidate knots -> UsT[gene][cand] (+ the population rows)
  if (philox_breed) {
    // crossover, mutation, clip (K/empc.py:201-204): a tight loop so the
    // parent gathers of several genes are in flight together
#pragma unroll 8
    for (int e = tid; e < cnt * pm; e += nthr) {
      const int c = e / pm, g = e - (e / pm) * pm;
      const int l = g % m;
      const bool take = tbits[e] != 0;
      const S par = parents[(pop_base + src[2 * c + (take ? 1 : 0)]) * pm + g];
      const S lo = cumin[l], hi = cumax[l];
      S v = par + off[g * tPS + c];
      v = v < lo ? lo : (v > hi ? hi : v);
      a.pop_out[(pop_base + a.row0 + tile0 + c) * pm + g] = v;
      UsT[g * tPS + c] = v;
    }
    for (int e = cnt * pm + tid; e < tileP * pm; e += nthr) {
      const int c = e / pm, g = e - (e / pm) * pm;
      UsT[g * tPS + c] = S(0);
    }
  } else
#pragma unroll 4
  for (int e = tid; e < tileP * pm; e += nthr) {
    const int c = e / pm, g = e - (e / pm) * pm;
    S v = S(0);
    if (c < cnt) {
      const int l = g % m;
      const int cand = tile0 + c;
      if (a.mode == kScore) {
        v = a.pop_in[(pop_base + a.row0 + cand) * pm + g];
      } else if (a.mode == kInitPhilox) {
        v = UsT[g * tPS + c];
      } else if (a.mode == kInitInject) {
        v = a.inj_init[((size_t)inst * a.nc + cand) * pm + g];
      } else if (philox_breed) {
        // crossover, mutation, clip (K/empc.py:201-204)
        const bool take = tbits[e] != 0;
        const S par = parents[(pop_base + src[2 * c + (take ? 1 : 0)]) * pm + g];
        const S lo = cumin[l], hi = cumax[l];
        v = par + off[g * tPS + c];
        v = v < lo ? lo : (v > hi ? hi : v);
      } else {
        // injected draws, with the reference's FP64 arithmetic child + mutate*noise*sigma
        const size_t gi = ((size_t)inst * a.nc + cand) * pm + g;
        const bool take = a.inj_take[gi] != 0, mut = a.inj_mut[gi] != 0;
        const S par = parents[(pop_base + src[2 * c + (take ? 1 : 0)]) * pm + g];
        const double nz = mut ? a.inj_noise[gi] * X[SL.sig + l] : 0.0;
        v = (S)((double)par + nz);
        const S lo = cumin[l], hi = cumax[l];
        v = v < lo ? lo : (v > hi ? hi : v);
      }
      if (a.mode != kScore || a.pop_in != a.pop_out) a.pop_out[(pop_base + a.row0 + cand) * pm + g] = v;
    }
    UsT[g * tPS + c] = v;
  }
  return true;
}

// ---------------------------------------------------------------------------
// rollout: K2 + K3 with the K5 breed / init prologue.
//
// Thread (rg, cg) owns rows {rg + r*NRG} (r < RR) of candidates
// [cg*CC, cg*CC + CC) of the tile.  States live in registers (xo) and, for
// the all-to-all of the matvec, in a double-buffered candidate-major smem
// tile XC[buf][cand][NPS]; every x load is a 16-byte broadcast with a
// compile-time offset.  A (as Delta = Ad - I) is in registers (AREG) or in
// smem rows As[row][NPS].  With KS = 2 the column range of the matvec is
// split over the lane pair (l, l ^ 16) and folded with one shuffle.
//
// Phases: (0) problem -> smem with coalesced loads, independent of the
// previous kernel (overlaps it under programmatic dependent launch);
// (1) wait for the producer, elite carry-over and breeding; (2) B at the
// knots and the knot-space input cost; (3) the horizon recursion.

// Input cost of a tile's candidates as the knot quadratic
// z'(W'W (x) R) z, z = U - u_goal (K/empc.py:100-101), for small state sizes
// (NP <= 16: few row groups, so the per-row-group channel split below leaves
// most threads idle): eight lanes per candidate take the channels
// l = lane8 (mod 8) and fold with a fixed shuffle tree; nt is a multiple of 32.
template <typename S>
__device__ __forceinline__ void input_costs(S* __restrict__ icost, const S* __restrict__ UsT, int tPS, int cnt, int m,
                                            int p, const S* sG, const S* cug, const S* crd, bool r_diag,
                                            const double* Rg, int nt) {
  const int t = threadIdx.x;
  const int g8 = (t & 31) >> 3, l8 = t & 7, w = t >> 5, nw = nt >> 5;
  for (int cb = 4 * w; cb < cnt; cb += 4 * nw) {  // warp-uniform trip count
    const int c = cb + g8;
    S val = S(0);
    if (c < cnt) {
      for (int l = l8; l < m; l += 8) {
        for (int q = 0; q < p; ++q) {
          S gz = S(0);
          for (int b = 0; b < p; ++b) {
            S rz;
            if (r_diag) {
              rz = crd[l] * (UsT[(b * m + l) * tPS + c] - cug[l]);
            } else {
              rz = S(0);
              for (int l2 = 0; l2 < m; ++l2) rz = fma((S)Rg[l * m + l2], UsT[(b * m + l2) * tPS + c] - cug[l2], rz);
            }
            gz = fma(sG[q * p + b], rz, gz);
          }
          val = fma(UsT[(q * m + l) * tPS + c] - cug[l], gz, val);
        }
      }
    }
    val += __shfl_xor_sync(0xFFFFFFFFu, val, 4);
    val += __shfl_xor_sync(0xFFFFFFFFu, val, 2);
    val += __shfl_xor_sync(0xFFFFFFFFu, val, 1);
    if (l8 == 0 && c < cnt) icost[c] = val;
  }
}

// HK: the left half of Delta's columns is exactly zero (the position columns
// of a linearized mechanism without gravity): the matvec runs over
// the right half only, split over the lane pair as usual (exact: the skipped
// products are zeros; the summation order of the rest changes)
template <typename S, int NP, int RR, int CC, bool AREG, bool DQ, int KS, bool WS, bool HK = false>
__device__ __forceinline__ void rollout_body(const RolloutArgs<S>& a, bool stage, size_t persist_scratch) {
  constexpr int NRG = NP / RR;
  constexpr int VEC = Geo<S>::VEC;
  constexpr int NPS = Geo<S>::nps(NP);
  constexpr int NSPLIT = (RR * CC >= 8) ? 1 : ((RR * CC >= 4) ? 2 : 4);
  constexpr int NPH = HK ? NP / KS / 2 : NP / KS;  // columns per reduction half
  constexpr int NJ = NPH / VEC;                    // 16-byte column groups per reduction half
  static_assert(!HK || (NP / 2) % (KS * VEC) == 0, "half-K split");
  // NJ / jbase also drive the dense-Q matvecs (e'Qe needs every column)
  static_assert(!(HK && DQ), "half-K is only valid with a diagonal Q");
  static_assert(!WS || 32 % (NRG * KS) == 0, "warp-synchronous variants need whole candidate groups per warp");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Dims& d = a.d;
  const StageLayout& SL = a.SL;
  const int n = d.n, m = d.m, T = d.T, p = d.p;
  const int tileP = a.tileP, tPS = a.tPS;
  const int inst = blockIdx.y;
  const int tile0 = blockIdx.x * a.tile;
  const int cnt = min(a.tile, a.nc - tile0);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = (nthr + 31) >> 5;
  const double* __restrict__ P = a.prob + (size_t)inst * SL.stride;
  const double* __restrict__ X = a.state + (size_t)inst * SL.sstride;

  const SmemPlan sp = smem_plan<S>(NP, m, T, p, tileP, tPS, AREG, DQ, persist_scratch);
  unsigned char* ptr = smem_raw;
  S* UsT = reinterpret_cast<S*>(ptr); ptr += sp.us;   // [gene][tPS]
  S* BUT = reinterpret_cast<S*>(ptr); ptr += sp.but;  // [knot][row][tPS]
  S* XC = reinterpret_cast<S*>(ptr); ptr += sp.xc;    // [2][tileP][NPS]; Bs [NP][m+1] in the prologue
  S* As = reinterpret_cast<S*>(ptr); ptr += sp.as;    // [NP][NPS]
  S* Qs = reinterpret_cast<S*>(ptr); ptr += sp.qs;    // [NP][NPS]
  int* sI1 = reinterpret_cast<int*>(ptr);
  int* sI2 = sI1 + T;
  int* sSeg = sI2 + T;  // end of the knot segment starting at k
  S* sC = reinterpret_cast<S*>(sSeg + T); ptr += sp.sched;
  S* sG = reinterpret_cast<S*>(ptr); ptr += sp.g;     // [p*p] + cost0
  ptr += sp.cu;  // per-candidate scratch slot of the plan (unused by this variant family)
  int* src = reinterpret_cast<int*>(ptr); ptr += sp.src;
  S* cw_ = reinterpret_cast<S*>(ptr); ptr += sp.cv;   // w, qd, xg, x0 [NP]; ug, umin, umax, sig, rdiag [m]
  S* cqd = cw_ + NP;
  S* cxg = cqd + NP;
  S* cx0 = cxg + NP;
  S* cug = cx0 + NP;
  S* cumin = cug + m;
  S* cumax = cumin + m;
  S* csig = cumax + m;
  S* crd = csig + m;
  S* Bs = persist_scratch ? reinterpret_cast<S*>(ptr) : XC;  // [NP][m+1]
  ptr += sp.bs;
  S* Off = persist_scratch ? reinterpret_cast<S*>(ptr) : nullptr;  // [gene][tPS] mutation offsets

  const size_t pop_base = (size_t)inst * a.rows;
  const bool breed = (a.mode == kBreedPhilox || a.mode == kBreedInject);

  EMPC_MARK(0)
  // ---- phase 0: problem -> smem (coalesced, all loads in flight together);
  // a persistent CTA stages even when its first tile is empty (later ones are not)
  if (stage && (cnt > 0 || persist_scratch)) {
    // [Ad | Bd | wd] (contiguous FP64 in the staging block, 16-byte aligned:
    // the host pads the per-instance stride to an even number of doubles)
    // goes to the scratch head with asynchronous 16-byte copies, all in
    // flight at once, while the small arrays below load; converted from
    // shared memory afterwards.  Falls back to direct loads when the scratch
    // head (before XC, which may alias Bs) is too small.
    const int nraw = n * n + n * m + n;
    const bool raw_ok = (size_t)nraw * 8 + 16 <= sp.us + sp.but;
    const double* raw = reinterpret_cast<const double*>(smem_raw);
    if (raw_ok) {
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
      for (int q = tid; q < (nraw + 1) / 2; q += nthr)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + 16u * (uint32_t)q),
                     "l"(P + SL.ad + 2 * q));
      asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int k = tid; k < T; k += nthr) {
      sI1[k] = a.idx1[k];
      sI2[k] = a.idx2[k];
      sSeg[k] = a.seg[k];
      sC[k] = a.cw[k];
    }
    for (int e = tid; e < p * p; e += nthr) sG[e] = a.G[e];
    if (raw_ok) {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncthreads();
    }
    const double* Ad = raw_ok ? raw : P + SL.ad;
    const double* Bd = raw_ok ? raw + n * n : P + SL.bd;
#pragma unroll 8
    for (int e = tid; e < NP * NP; e += nthr) {
      const int i = e / NP, j = e - (e / NP) * NP;
      As[i * NPS + j] = (i < n && j < n) ? (S)(Ad[i * n + j] - (i == j ? 1.0 : 0.0)) : S(0);
      if constexpr (DQ) Qs[i * NPS + j] = (i < n && j < n) ? (S)P[SL.q + i * n + j] : S(0);
    }
#pragma unroll 8
    for (int e = tid; e < NP * m; e += nthr) {
      const int i = e / m, l = e - (e / m) * m;
      Bs[i * (m + 1) + l] = i < n ? (S)Bd[i * m + l] : S(0);
    }
    // the recursion runs in error coordinates e = x - x_goal:
    //   e_{k+1} = e_k + Delta e_k + (drive_k + Delta x_goal)
    // so w picks up Delta x_goal (rows of W sum to one) and e_0 = x0 - x_goal
    for (int i = tid; i < NP; i += nthr) {
      const bool ok = i < n;
      cw_[i] = ok ? (S)P[SL.wd + i] : S(0);  // + Delta x_goal below, from As
      cqd[i] = ok ? (S)P[SL.q + i * n + i] : S(0);
      cxg[i] = ok ? (S)P[SL.xg + i] : S(0);
      cx0[i] = ok ? (S)(X[SL.x0 + i] - P[SL.xg + i]) : S(0);
    }
    for (int l = tid; l < m; l += nthr) {
      cug[l] = (S)P[SL.ug + l];
      cumin[l] = (S)P[SL.umin + l];
      cumax[l] = (S)P[SL.umax + l];
      csig[l] = (S)X[SL.sig + l];
      crd[l] = (S)P[SL.r + l * m + l];
    }
    // cost of x_0 (k = 0 state term, K/empc.py:113-118), FP64, warp 0
    if (warp == 0) {
      double part = 0.0;
      for (int i = lane; i < n; i += 32) {
        const double ei = X[SL.x0 + i] - P[SL.xg + i];
        if constexpr (DQ) {
          double qe = 0.0;
          for (int j = 0; j < n; ++j) qe = fma(P[SL.q + i * n + j], X[SL.x0 + j] - P[SL.xg + j], qe);
          part = fma(ei, qe, part);
        } else {
          part = fma(P[SL.q + i * n + i] * ei, ei, part);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, off);
      if (lane == 0) sG[p * p] = (S)part;
    }
  }

  EMPC_MARK(7)
  __syncthreads();  // phase-0 smem (bounds, sigma) is read by every thread below
  // w += Delta x_goal (error coordinates): one warp per row group, lanes over columns
  for (int i = warp; i < (stage ? n : 0); i += nwarps) {
    S acc = S(0);
    for (int j = lane; j < n; j += 32) acc = fma(As[i * NPS + j], cxg[j], acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
    if (lane == 0) cw_[i] += acc;
  }
  EMPC_MARK(8)
  uint8_t* tbits = reinterpret_cast<uint8_t*>(cw_ + 4 * NP + 5 * m);  // crossover choice, 1 byte per gene
  if (!breed_tile<S>(a, inst, tile0, cnt, tileP, tPS, UsT, src, tbits, cumin, cumax, csig, pop_base, true, Off)) {
    // a persistent CTA without candidates in this rollout (the init tile of
    // the last CTAs) still draws its next evolve tile, so that evolve finds
    // its draws ready like every other CTA
    if (WS && persist_scratch && a.draw_next && a.draw_cnt > 0)
      draw_tile<S>(*a.run, (uint32_t)(a.run->gen0 + a.draw_evolve), d.K, d.pm, m, inst, a.cand_base + a.draw_tile0,
                   a.draw_cnt, tPS, tid, nthr, src, tbits, Off, csig);
    return;
  }
  __syncthreads();
  EMPC_MARK(3)

  // ---- phase 2
  // logical thread (rg, cg); with KS = 2 the two halves of the j-reduction
  // of one logical thread are lanes l and l ^ 16 of the same warp
  const int lt = KS == 1 ? tid : (((tid >> 5) << 4) | (tid & 15));
  const int ks = KS == 1 ? 0 : ((tid >> 4) & 1);
  const int rg = lt % NRG, cg = lt / NRG;
  const bool active = cg * CC < tileP;
  // padding threads shadow candidate group 0 so that every lane of a warp
  // takes part in the shuffles; their results are never stored
  const int c0 = active ? cg * CC : 0;
  const int jbase = (HK ? NP / 2 : 0) + ks * NPH;
  // epilogue split: with KS = 2 each lane of the pair finishes half of the
  // candidates (CH of them, starting at candidate ce)
  constexpr int CH = KS == 2 ? CC / 2 : CC;
  const int ce = c0 + ks * CH;
  // B at the knots (+ w), interpolated later: drive = W (x) (U Bd') + wd
  // (K/empc.py:104-105).  BUT[knot][row][cand].  Warp-synchronous CTAs of
  // small states spread it over every thread, helpers included (items of RR
  // rows x 2 candidates x one knot; same FMA order per output): C2 166.5 ->
  // 164.8 us; at NP = 48 the extra shared loads cost more (C3 +11 us)
  constexpr int kDriveCB = (WS && CC % 2 == 0 && NP <= 16) ? 2 : 0;
  if constexpr (kDriveCB > 0) {
    const int ncb = tileP / kDriveCB;
    const int items = p * NRG * ncb;
    for (int w = tid; w < items; w += nthr) {
      const int cb = w % ncb, rest = w / ncb;
      const int rgw = rest % NRG, j = rest / NRG;
      const int cc0 = cb * kDriveCB;
      S acc[RR][kDriveCB];
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const S w0 = cw_[rgw + r * NRG];
#pragma unroll
        for (int q = 0; q < kDriveCB; ++q) acc[r][q] = w0;
      }
#pragma unroll 4
      for (int l = 0; l < m; ++l) {
        S u[kDriveCB];
        lds_vec<S, kDriveCB>(UsT + (j * m + l) * tPS + cc0, u);
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          const S b = Bs[(rgw + r * NRG) * (m + 1) + l];
#pragma unroll
          for (int q = 0; q < kDriveCB; ++q) acc[r][q] = fma(b, u[q], acc[r][q]);
        }
      }
#pragma unroll
      for (int r = 0; r < RR; ++r) sts_vec<S, kDriveCB>(BUT + (j * NP + rgw + r * NRG) * tPS + cc0, acc[r]);
    }
  } else if (active) {
    for (int j = ks; j < p; j += KS) {
      S acc[RR][CC];
#pragma unroll
      for (int r = 0; r < RR; ++r) {
        const S w = cw_[rg + r * NRG];
#pragma unroll
        for (int q = 0; q < CC; ++q) acc[r][q] = w;
      }
#pragma unroll 4
      for (int l = 0; l < m; ++l) {
        S u[CC];
        lds_vec<S, CC>(UsT + (j * m + l) * tPS + c0, u);
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          const S b = Bs[(rg + r * NRG) * (m + 1) + l];
#pragma unroll
          for (int q = 0; q < CC; ++q) acc[r][q] = fma(b, u[q], acc[r][q]);
        }
      }
#pragma unroll
      for (int r = 0; r < RR; ++r) sts_vec<S, CC>(BUT + (j * NP + rg + r * NRG) * tPS + c0, acc[r]);
    }
  }
  EMPC_MARK(11)
  // model rows: A (Delta = Ad - I) from smem into registers
  S areg[AREG ? RR : 1][AREG ? NPH : 1];
  if constexpr (AREG) {
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
      for (int jv = 0; jv < NPH / VEC; ++jv) {
        S t[VEC];
        lds_vec<S, VEC>(As + (rg + r * NRG) * NPS + jbase + jv * VEC, t);
#pragma unroll
        for (int q = 0; q < VEC; ++q) areg[r][jv * VEC + q] = t[q];
      }
  }
  EMPC_MARK(12)
  S qv[RR], xo[RR][CH];  // state rows in error coordinates
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const int row = rg + r * NRG;
    qv[r] = DQ ? S(0) : cqd[row];
#pragma unroll
    for (int q = 0; q < CH; ++q) xo[r][q] = cx0[row];
  }
  // input cost as the knot quadratic z'(W'W (x) R)z, z = U - u_goal
  // (K/empc.py:100-101): each thread seeds the state-cost accumulators of its
  // candidates with the channels l = rg (mod NRG); the row-group reduction at
  // the end then sums both terms.
  S cst[CH];
#pragma unroll
  for (int q = 0; q < CH; ++q) cst[q] = S(0);
  constexpr bool kCoopIcost = NP <= 16;
  S* icost = reinterpret_cast<S*>(reinterpret_cast<unsigned char*>(src) - sp.cu);  // the plan's per-candidate slot
  if constexpr (kCoopIcost)
    input_costs<S>(icost, UsT, tPS, cnt, m, p, sG, cug, crd, a.r_diag != 0, P + SL.r, (nthr + 31) / 32 * 32);
  if (active && !kCoopIcost) {
    for (int l = rg; l < m; l += NRG) {
      const S ugl = cug[l];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int c = ce + q;
        S val = S(0);
        if (p <= 8) {
          S gz[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) gz[t] = S(0);
          for (int b = 0; b < p; ++b) {
            S rz;
            if (a.r_diag) {
              rz = crd[l] * (UsT[(b * m + l) * tPS + c] - ugl);
            } else {
              rz = S(0);
              for (int l2 = 0; l2 < m; ++l2)
                rz = fma((S)P[SL.r + l * m + l2], UsT[(b * m + l2) * tPS + c] - cug[l2], rz);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t)
              if (t < p) gz[t] = fma(sG[t * p + b], rz, gz[t]);
          }
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < p) val = fma(UsT[(t * m + l) * tPS + c] - ugl, gz[t], val);
        } else {
          for (int t = 0; t < p; ++t) {
            S gzt = S(0);
            for (int b = 0; b < p; ++b) {
              S rz = S(0);
              for (int l2 = 0; l2 < m; ++l2)
                rz = fma((S)P[SL.r + l * m + l2], UsT[(b * m + l2) * tPS + c] - cug[l2], rz);
              gzt = fma(sG[t * p + b], rz, gzt);
            }
            val = fma(UsT[(t * m + l) * tPS + c] - ugl, gzt, val);
          }
        }
        cst[q] += val;
      }
    }
  }
  // Bs aliases XC in the per-generation kernels: consumed before the fill
  // (the persistent solve keeps Bs apart, and the barrier after the fill
  // also publishes BUT)
  if (!persist_scratch) __syncthreads();
  // x_0 = x0 for every candidate (K/empc.py:109)
  for (int e = tid; e < tileP * NPS; e += nthr) {
    const int i = e % NPS;
    XC[e] = i < NP ? cx0[i] : S(0);
  }
  __syncthreads();
  // the next kernel may start its independent prologue now
  pdl_trigger();
  EMPC_MARK(4)

  // partial products of the rows with this thread's column half, with
  // software-pipelined 16-byte loads (the next column group is in flight
  // while the current one is consumed).  With KS == 2 each lane lists its
  // own CH candidates first (base XO) and its partner's second (base XP), so
  // folding the halves is one shuffle + one add per result, no selects.
  // A macro, not a lambda, so the register arrays stay in registers.
#define EMPC_MATVEC(FROMREG, MS, XO, XP, OUT, SEEDED, SEED)                                           \
  {                                                                                                   \
    S part_[RR][CC][NSPLIT];                                                                          \
    _Pragma("unroll") for (int r = 0; r < RR; ++r)                                                    \
    _Pragma("unroll") for (int q = 0; q < CC; ++q)                                                    \
    _Pragma("unroll") for (int s = 0; s < NSPLIT; ++s) part_[r][q][s] = S(0);                         \
    if constexpr (SEEDED) {                                                                           \
      _Pragma("unroll") for (int r = 0; r < RR; ++r)                                                  \
      _Pragma("unroll") for (int q = 0; q < CH; ++q) part_[r][q][0] = (SEED)[r][q];                   \
    }                                                                                                 \
    S xv_[2][CC][VEC];                                                                                \
    _Pragma("unroll") for (int q = 0; q < CC; ++q)                                                    \
      lds_vec<S, VEC>((q < CH ? (XO) + q * NPS : (XP) + (q - CH) * NPS), xv_[0][q]);                 \
    _Pragma("unroll") for (int jj = 0; jj < NJ; ++jj) {                                               \
      if (jj + 1 < NJ) {                                                                              \
        _Pragma("unroll") for (int q = 0; q < CC; ++q)                                                \
          lds_vec<S, VEC>((q < CH ? (XO) + q * NPS : (XP) + (q - CH) * NPS) + (jj + 1) * VEC,        \
                          xv_[(jj + 1) & 1][q]);                                                      \
      }                                                                                               \
      S av_[RR][VEC];                                                                                 \
      _Pragma("unroll") for (int r = 0; r < RR; ++r) {                                                \
        if constexpr (FROMREG) {                                                                      \
          _Pragma("unroll") for (int t = 0; t < VEC; ++t) av_[r][t] = areg[r][AREG ? jj * VEC + t : 0]; \
        } else {                                                                                      \
          lds_vec<S, VEC>((MS) + (rg + r * NRG) * NPS + jbase + jj * VEC, av_[r]);                    \
        }                                                                                             \
      }                                                                                               \
      _Pragma("unroll") for (int t = 0; t < VEC; ++t)                                                 \
      _Pragma("unroll") for (int r = 0; r < RR; ++r)                                                  \
      _Pragma("unroll") for (int q = 0; q < CC; ++q)                                                  \
        part_[r][q][t % NSPLIT] = fma(av_[r][t], xv_[jj & 1][q][t], part_[r][q][t % NSPLIT]);         \
    }                                                                                                 \
    _Pragma("unroll") for (int r = 0; r < RR; ++r)                                                    \
    _Pragma("unroll") for (int q = 0; q < CH; ++q) {                                                  \
      S mine_ = part_[r][q][0];                                                                       \
      _Pragma("unroll") for (int s = 1; s < NSPLIT; ++s) mine_ += part_[r][q][s];                     \
      if constexpr (KS == 2) {                                                                        \
        S give_ = part_[r][CH + q][0];                                                                \
        _Pragma("unroll") for (int s = 1; s < NSPLIT; ++s) give_ += part_[r][CH + q][s];              \
        mine_ += __shfl_xor_sync(0xFFFFFFFFu, give_, 16);                                             \
      }                                                                                               \
      (OUT)[r][q] = mine_;                                                                            \
    }                                                                                                 \
  }

  // ---- phase 3: horizon recursion in error coordinates,
  // e_{k+1} = e_k + Delta e_k + drive'_k (K/empc.py:110-112), state cost
  // fused per step (K/empc.py:113-118).  The knot pair (i1, i2) of the drive
  // is constant over p - 1 segments of the horizon (sSeg[k] = end of the
  // segment starting at k): the endpoint b1 and slope b2 - b1 of the
  // interpolation are loaded once per segment, and the step loop carries no
  // schedule test.  The state buffers ping-pong by swapping two offsets.
  // loop-invariant addresses: own / partner candidate rows of both buffers
  const S* xo0 = XC + (size_t)ce * NPS + jbase;
  const S* xp0 = XC + (size_t)(c0 + (ks ^ 1) * CH) * NPS + jbase;
  const int bufstride = tileP * NPS;
  S* xw0 = XC + (size_t)ce * NPS + rg;
  // diagonal Q: per-row sums of e_i^2, weighted by q_i once at the end
  S srow[DQ ? 1 : RR][DQ ? 1 : CH];
#pragma unroll
  for (int r = 0; r < (DQ ? 1 : RR); ++r)
#pragma unroll
    for (int q = 0; q < (DQ ? 1 : CH); ++q) srow[r][q] = S(0);
  // WS: whole warps without candidates (CTA helpers) skip the recursion, and
  // warps 4-7 start `stagger` cycles late so that the two warps sharing an
  // SM sub-partition run their latency-bound step tails out of phase
  // (warp-uniform: a warp with any active group runs the loop; its inactive
  // lanes shadow group 0 so that __syncwarp sees the full warp)
  const bool run_loop = !WS || __any_sync(0xFFFFFFFFu, active);
  if constexpr (WS) {
    if (run_loop && a.stagger > 0 && ((warp >> 2) & 1)) {
      const long long t0 = clock64();
      while (clock64() - t0 < a.stagger) {
      }
    }
    // helper warps: the next evolve's K5 draws for this CTA's tile (counter
    // based, so they do not depend on this generation), off the critical path
    if (!run_loop && a.draw_next && a.draw_cnt > 0) {
      constexpr int kLT = KS == 1 ? 1 : 2;
      const int hstart = (kLT * NRG * (tileP / CC) + 31) / 32 * 32;
      if (tid >= hstart)
        draw_tile<S>(*a.run, (uint32_t)(a.run->gen0 + a.draw_evolve), d.K, d.pm, m, inst,
                     a.cand_base + a.draw_tile0, a.draw_cnt, tPS, tid - hstart, nthr - hstart, src, tbits, Off, csig);
    }
  }
  int rdo = 0, wro = bufstride;
  constexpr bool kSeedStep = sizeof(S) == 4;
  for (int k0 = 0; run_loop && k0 < T;) {
    const int k1 = sSeg[k0];
    const int i1 = sI1[k0], i2 = sI2[k0];
    S b1[RR][CH], db[RR][CH];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      S t2[CH];
      lds_vec<S, CH>(BUT + (i1 * NP + rg + r * NRG) * tPS + ce, b1[r]);
      lds_vec<S, CH>(BUT + (i2 * NP + rg + r * NRG) * tPS + ce, t2);
#pragma unroll
      for (int q = 0; q < CH; ++q) db[r][q] = t2[q] - b1[r][q];
    }
    for (int k = k0; k < k1; ++k) {
      const S ck = sC[k];
      // FP32: the step's e + drive seeds this lane's own accumulators, so
      // it is computed off the critical path and the folded matvec is the
      // next state (FP64 keeps the reference-order update below)
      S xd[RR][CH];
      if constexpr (kSeedStep) {
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int q = 0; q < CH; ++q) xd[r][q] = xo[r][q] + fma(ck, db[r][q], b1[r][q]);
      }
      S ax[RR][CH];
      EMPC_MATVEC(AREG, As, xo0 + rdo, xp0 + rdo, ax, kSeedStep, xd)
      S qx[DQ ? RR : 1][DQ ? CH : 1];
      if constexpr (DQ) EMPC_MATVEC(false, Qs, xo0 + rdo, xp0 + rdo, qx, false, xd)
      S* xw = xw0 + wro;
#pragma unroll
      for (int r = 0; r < RR; ++r) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          if constexpr (DQ) cst[q] = fma(xo[r][q], qx[r][q], cst[q]);  // e_k' Q e_k
          const S en = kSeedStep ? ax[r][q] : xo[r][q] + fma(ck, db[r][q], ax[r][q] + b1[r][q]);
          xo[r][q] = en;
          if constexpr (!DQ) srow[r][q] = fma(en, en, srow[r][q]);  // e_{k+1,i}^2
#ifndef EMPC_EXP_NOSTS
          if (active) xw[q * NPS + r * NRG] = en;
#endif
        }
      }
      const int t = rdo;
      rdo = wro;
      wro = t;
      // WS: all rows of a candidate group live in one warp, so the state
      // exchange of a step only needs a warp-level barrier and warps run
      // their horizons independently
#ifndef EMPC_EXP_NOBAR
      if constexpr (WS) __syncwarp(); else __syncthreads();
#endif
    }
    k0 = k1;
  }
  if constexpr (!DQ) {
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
      for (int q = 0; q < CH; ++q) cst[q] = fma(qv[r], srow[r][q], cst[q]);  // diag(Q) e'e over k = 1..T
  }
  if constexpr (WS) __syncthreads();
  if constexpr (DQ) {
    // terminal state term e_T' Q e_T
    const int rd = (T & 1) ? bufstride : 0;
    S qf[RR][CH];
    EMPC_MATVEC(false, Qs, xo0 + rd, xp0 + rd, qf, false, qf)
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
      for (int q = 0; q < CH; ++q) cst[q] = fma(xo[r][q], qf[r][q], cst[q]);
  }
  EMPC_MARK(5)
  // ---- deterministic reduction over row groups (BUT is free now)
  S* red = BUT;
  if (active) {
#pragma unroll
    for (int q = 0; q < CH; ++q) red[rg * tPS + ce + q] = cst[q];
  }
  __syncthreads();
  const S c0s = DQ ? S(0) : sG[p * p];
  // children whose key beats the K-th elite's are appended to the instance's
  // qualifier list (order is irrelevant: keys are unique and get sorted)
  using OT = typename std::conditional<sizeof(S) == 4, uint32_t, uint64_t>::type;
  OT tau = OT(0);
  const bool qual = breed && a.qcount != nullptr;
  if (qual) tau = ord_key(a.cost_in[pop_base + a.elite_idx[(size_t)inst * d.K + d.K - 1]]);
  for (int c = tid; c < cnt; c += nthr) {
    S s = S(0);
    if constexpr (kCoopIcost) s = icost[c];
    for (int g = 0; g < NRG; ++g) s += red[g * tPS + c];
    const S cost = c0s + s;
    const int row = a.row0 + tile0 + c;
    a.cost_out[pop_base + row] = cost;
    if (a.amin != nullptr) atomicMin(a.amin, amin_key(cost, row));  // last generation: distributed argmin
    if (qual) {
      const OT kc = ord_key(cost);
      if (kc < tau) {
        const int slot = atomicAdd(a.qcount + inst, 1);
        if (slot < a.qcap) {
          OT* ql = reinterpret_cast<OT*>(a.qlist) + (size_t)inst * a.qcap * 2;
          ql[2 * slot] = kc;
          ql[2 * slot + 1] = (OT)row;
        }
      }
    }
  }
  EMPC_MARK(6)
#undef EMPC_MATVEC
}

template <typename S, int NP, int RR, int CC, bool AREG, bool DQ, int KS, bool WS, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) rollout_kernel(const RolloutArgs<S> a) {
  rollout_body<S, NP, RR, CC, AREG, DQ, KS, WS>(a, true, 0);
}

// ---------------------------------------------------------------------------
// K4 selection: stable top-K (argsort(kind="stable")[:K], K/empc.py:185-186).
// Key of candidate i = (ord(cost_i), i) -- unique, so the stable order is the
// key order and the result is deterministic.  Rank by counting, spread over
// the whole GPU: every CTA loads the instance's candidate keys into shared
// memory and ranks a slice of them (one warp per candidate, lanes over the
// set); a candidate of rank r < K lands in elite slot r.
//
// Candidate set: all N rows for the first selection of a run.  After an
// evolve, rows [0, K) hold the previous elites and only children that beat
// the K-th of them (appended to a qualifier list by the rollout epilogue) can
// enter: every other key is larger than every key of this set, so ranks
// within the set are global ranks.  The qualifier lists are double-buffered
// by evolve parity; the selection resets the list the next rollout fills.

template <typename S>
struct OrdOf;
template <>
struct OrdOf<float> {
  using T = uint32_t;
  __device__ __forceinline__ static T ord(float c) { return ord32(c); }
};
template <>
struct OrdOf<double> {
  using T = uint64_t;
  __device__ __forceinline__ static T ord(double c) { return ord64(c); }
};

template <typename S>
__host__ __device__ inline size_t select_smem(int N) {
  using OT = typename std::conditional<sizeof(S) == 4, uint32_t, uint64_t>::type;
  return (size_t)N * (sizeof(OT) + sizeof(int));
}

// PF > 0 (FP32): each ranked candidate's row (pm <= 32 PF) and cost are
// loaded before its rank is known, so the elite carry-over's L2 round trip
// overlaps the counting (costs PF registers per lane)
template <typename S, int PF = 0>
__device__ __forceinline__ void select_body(const S* __restrict__ costs, int N, int K, int* __restrict__ elite_idx,
                                            int incremental, int* __restrict__ qcount_in,
                                            const void* __restrict__ qlist_in, int* __restrict__ qcount_next, int qcap,
                                            const S* __restrict__ pop_in, S* __restrict__ pop_out,
                                            S* __restrict__ cost_out, int pm) {
  using OT = typename OrdOf<S>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OT* ck = reinterpret_cast<OT*>(smem_raw);
  int* ci = reinterpret_cast<int*>(ck + N);
  const int inst = blockIdx.y;
  const S* c = costs + (size_t)inst * N;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  pdl_wait();     // costs come from the previous rollout
  int L = 0;
  bool full = !incremental || K >= N || qcount_in == nullptr;
  if (!full) {
    L = qcount_in[inst];
    full = L > qcap || K + L > N;
  }
  __syncthreads();  // all reads of the count precede its reset below
  if (blockIdx.x == 0 && tid == 0 && qcount_next != nullptr) qcount_next[inst] = 0;
  pdl_trigger();  // the next rollout may start its independent prologue
  const int M = full ? N : K + L;
  const OT* ql = full ? nullptr : reinterpret_cast<const OT*>(qlist_in) + (size_t)inst * qcap * 2;
  // FP32: one 64-bit key (ord << 32 | row) per candidate, so a comparison is
  // a single unsigned compare (same order as (ord, row) pairs)
  unsigned long long* kk = reinterpret_cast<unsigned long long*>(smem_raw);
  for (int j = tid; j < M; j += nthr) {
    if constexpr (sizeof(S) == 4) {
      if (j < K || full) kk[j] = ((unsigned long long)ord32((float)__ldcg(c + j)) << 32) | (unsigned)j;
      else kk[j] = ((unsigned long long)__ldcg(ql + 2 * (j - K)) << 32) | (unsigned)__ldcg(ql + 2 * (j - K) + 1);
    } else if (j < K || full) {
      ck[j] = OrdOf<S>::ord(c[j]);
      ci[j] = j;
    } else {
      ck[j] = ql[2 * (j - K)];
      ci[j] = (int)ql[2 * (j - K) + 1];
    }
  }
  __syncthreads();
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int e0 = blockIdx.x * per, e1 = min(M, e0 + per);
  for (int e = e0 + warp; e < e1; e += nwarps) {
    int re, cnt = 0;
    constexpr int kPF = PF > 0 ? PF : 1;
    S rowv[kPF];
    S cre = S(0);
    bool pf = false;
    if constexpr (sizeof(S) == 4) {
      const unsigned long long ke = kk[e];
      re = (int)(uint32_t)ke;
      pf = PF > 0 && pop_out != nullptr && pm <= 32 * kPF;
      if (pf) {
        const S* from = pop_in + ((size_t)inst * N + re) * pm;
#pragma unroll
        for (int i = 0; i < kPF; ++i) {
          const int g = lane + 32 * i;
          rowv[i] = g < pm ? __ldcg(from + g) : S(0);
        }
        cre = __ldcg(c + re);
      }
      for (int j = lane; j < M; j += 32) cnt += kk[j] < ke ? 1 : 0;
    } else {
      const OT ke = ck[e];
      re = ci[e];
      for (int j = lane; j < M; j += 32) {
        const OT kj = ck[j];
        cnt += (kj < ke || (kj == ke && ci[j] < re)) ? 1 : 0;
      }
    }
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (cnt < K) {
      if (lane == 0) elite_idx[(size_t)inst * K + cnt] = re;
      if (pop_out != nullptr) {
        // elite carry-over (K/empc.py:186-188, 206): rows [0, K) of the next
        // population are the sorted elites with their carried costs
        S* to = pop_out + ((size_t)inst * N + cnt) * pm;
        if (pf) {
#pragma unroll
          for (int i = 0; i < kPF; ++i) {
            const int g = lane + 32 * i;
            if (g < pm) to[g] = rowv[i];
          }
          if (lane == 0) cost_out[(size_t)inst * N + cnt] = cre;
        } else {
          const S* from = pop_in + ((size_t)inst * N + re) * pm;
          for (int g = lane; g < pm; g += 32) to[g] = from[g];
          if (lane == 0) cost_out[(size_t)inst * N + cnt] = c[re];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K4 for large candidate sets (FP32 costs, e.g. C4: N = 16384, K = 1024):
// every CTA finds the K-th smallest 64-bit key (ord(cost) << 32 | row) of the
// candidate set by an 8-bit radix select over shared memory (<= 8 histogram
// passes, usually 3), compacts the K elite keys in row order (deterministic
// block scan), and ranks only its slice of the K elites against the K elite
// keys (K^2 / CTAs comparisons instead of M^2 / CTAs).  Same result as
// select_body (unique keys: the stable argsort order); shared memory =
// radix_select_smem(N).

__host__ __device__ inline size_t radix_select_smem(int N, int K) {
  return (size_t)N * 8 + (size_t)K * 8 + 256 * 4 + 64 * 4 + 64;
}

__device__ __forceinline__ void block_exclusive_scan(int& v, int* warp_tot, int& total) {
  // exclusive prefix sum of v over the block (in thread order), total count
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  total = warp_tot[nw - 1];
  v = x - v + (warp > 0 ? warp_tot[warp - 1] : 0);
  __syncthreads();
}

// Radix-select helpers.  Bits all keys share are skipped: the block AND / OR
// of the keys gives the highest differing bit, where the first digit starts
// (a population whose costs share sign and exponent bits would otherwise
// spend a pass on one hot bin).
__device__ __forceinline__ void radix_common_bits(unsigned long long kand, unsigned long long kor, int* aux,
                                                  int& hb, unsigned long long& prefix, unsigned long long& mask) {
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned ah = __reduce_and_sync(0xFFFFFFFFu, (unsigned)(kand >> 32));
  const unsigned al = __reduce_and_sync(0xFFFFFFFFu, (unsigned)kand);
  const unsigned oh = __reduce_or_sync(0xFFFFFFFFu, (unsigned)(kor >> 32));
  const unsigned ol = __reduce_or_sync(0xFFFFFFFFu, (unsigned)kor);
  if (tid == 0) {
    aux[36] = -1; aux[37] = -1; aux[38] = 0; aux[39] = 0;
  }
  __syncthreads();
  if (lane == 0) {
    atomicAnd(&aux[36], (int)ah); atomicAnd(&aux[37], (int)al);
    atomicOr(&aux[38], (int)oh); atomicOr(&aux[39], (int)ol);
  }
  __syncthreads();
  kand = ((unsigned long long)(unsigned)aux[36] << 32) | (unsigned)aux[37];
  kor = ((unsigned long long)(unsigned)aux[38] << 32) | (unsigned)aux[39];
  const unsigned long long diff = kand ^ kor;
  hb = diff == 0ull ? 0 : 63 - __clzll(diff);
  mask = hb >= 63 ? 0ull : (~0ull << (hb + 1));
  prefix = kand & mask;
}

// After a digit histogram: the bucket holding the krem-th key (warp 0, 8 bins
// per lane); updates prefix / mask / krem, done when the bucket is taken whole.
__device__ __forceinline__ void radix_pick_bucket(const int* hist, int* aux, int shift, int& krem,
                                                  unsigned long long& prefix, unsigned long long& mask, bool& done) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __syncthreads();
  if (warp == 0) {
    int loc[8], s8 = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) { loc[q] = hist[lane * 8 + q]; s8 += loc[q]; }
    int inc = s8;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += y;
    }
    int before = inc - s8;
    if (before < krem && krem <= inc) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (before < krem && krem <= before + loc[q]) {
          aux[32] = lane * 8 + q;
          aux[33] = krem - before;
          aux[34] = loc[q];
        }
        before += loc[q];
      }
    }
  }
  __syncthreads();
  const int b = aux[32];
  krem = aux[33];
  // near the bottom the digit overlaps decided bits, which are constant over
  // the keys matching the prefix
  prefix |= (unsigned long long)b << shift;
  mask |= 255ull << shift;
  done = aux[34] == krem;
  __syncthreads();
}

// The K smallest of M unique 64-bit keys in shared memory: 8-bit radix
// select of the K-th key, then a deterministic compaction of the keys <= it
// into E in key-position order (block scan).  total = number compacted
// (min(K, M)).  All threads of the block call it.
__device__ __forceinline__ void radix_topk_compact(const unsigned long long* keys, int M, int K,
                                                   unsigned long long* E, int* hist, int* aux, int& total) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  unsigned long long kand = ~0ull, kor = 0ull;
  for (int j = tid; j < M; j += nthr) {
    const unsigned long long k = keys[j];
    kand &= k;
    kor |= k;
  }
  int hb;
  unsigned long long prefix, mask;
  radix_common_bits(kand, kor, aux, hb, prefix, mask);
  int krem = K;
  bool done = K >= M;
  for (int top = hb; top >= 0 && !done; top -= 8) {
    const int shift = top >= 7 ? top - 7 : 0;  // digit = bits [shift, shift + 8)
    for (int b = tid; b < 256; b += nthr) hist[b] = 0;
    __syncthreads();
    for (int j = tid; j < M; j += nthr) {
      const unsigned long long k = keys[j];
      if ((k & mask) == prefix) atomicAdd(&hist[(int)((k >> shift) & 255ull)], 1);
    }
    radix_pick_bucket(hist, aux, shift, krem, prefix, mask, done);
  }
  // elites: keys below the bucket, plus the bucket when it is taken whole
  // (the loop ends with exactly K keys <= thr)
  const unsigned long long thr = K >= M ? ~0ull : (prefix | ~mask);
  // ---- deterministic compaction of the K elite keys (block scan in key-position order)
  const int chunk = (M + nthr - 1) / nthr;
  const int j0 = min(M, tid * chunk), j1 = min(M, j0 + chunk);
  int cnt = 0;
  for (int j = j0; j < j1; ++j) cnt += keys[j] <= thr ? 1 : 0;
  block_exclusive_scan(cnt, aux, total);
  for (int j = j0; j < j1; ++j)
    if (keys[j] <= thr) E[cnt++] = keys[j];
  __syncthreads();
}

// Register-resident variant (M <= R * blockDim.x): thread t holds keys
// t + i * blockDim.x in kr[i], so the digit passes issue independent shared
// atomics with no shared loads in between.  E is filled in thread-major order
// (the same on every CTA: only the set matters to the ranking).
template <int R>
__device__ __forceinline__ void radix_topk_regs(const unsigned long long (&kr)[R], int M, int K,
                                                unsigned long long* E, int* hist, int* aux, int& total,
                                                unsigned long long* mk = nullptr) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  unsigned long long kand = ~0ull, kor = 0ull;
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (tid + i * nthr < M) {
      kand &= kr[i];
      kor |= kr[i];
    }
  int hb;
  unsigned long long prefix, mask;
  radix_common_bits(kand, kor, aux, hb, prefix, mask);
  if (mk != nullptr && tid == 0) mk[0] = gtimer();
  int krem = K;
  bool done = K >= M;
  for (int top = hb; top >= 0 && !done; top -= 8) {
    const int shift = top >= 7 ? top - 7 : 0;
    for (int b = tid; b < 256; b += nthr) hist[b] = 0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (tid + i * nthr < M && (kr[i] & mask) == prefix) atomicAdd(&hist[(int)((kr[i] >> shift) & 255ull)], 1);
    radix_pick_bucket(hist, aux, shift, krem, prefix, mask, done);
    if (mk != nullptr && tid == 0 && (hb - top) / 8 < 7) mk[1 + (hb - top) / 8] = gtimer();
  }
  const unsigned long long thr = K >= M ? ~0ull : (prefix | ~mask);
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) cnt += (tid + i * nthr < M && kr[i] <= thr) ? 1 : 0;
  block_exclusive_scan(cnt, aux, total);
#pragma unroll
  for (int i = 0; i < R; ++i)
    if (tid + i * nthr < M && kr[i] <= thr) E[cnt++] = kr[i];
  __syncthreads();
}

template <typename S>
__device__ __forceinline__ void select_radix_body(const S* __restrict__ costs, int N, int K, int* __restrict__ elite_idx,
                                                  int incremental, int* __restrict__ qcount_in,
                                                  const void* __restrict__ qlist_in, int* __restrict__ qcount_next,
                                                  int qcap, const S* __restrict__ pop_in, S* __restrict__ pop_out,
                                                  S* __restrict__ cost_out, int pm, int* s_elite = nullptr,
                                                  unsigned long long* fold_amin = nullptr,
                                                  unsigned long long* mk = nullptr) {
  static_assert(sizeof(S) == 4, "64-bit (ord32, row) keys: FP32 costs");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);
  const int inst = blockIdx.y;
  const S* c = costs + (size_t)inst * N;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  pdl_wait();
  int L = 0;
  bool full = !incremental || K >= N || qcount_in == nullptr;
  if (!full) {
    L = qcount_in[inst];
    full = L > qcap || K + L > N;
  }
  const int M = full ? N : K + L;
  unsigned long long* E = keys + N;                    // [K] elite keys in key-position order
  int* hist = reinterpret_cast<int*>(E + K);           // [256]
  int* aux = hist + 256;                               // [64]: warp totals, bucket / remainder broadcast
  __syncthreads();  // all reads of the count precede its reset below
  if (blockIdx.x == 0 && tid == 0 && qcount_next != nullptr) qcount_next[inst] = 0;
  pdl_trigger();
  const uint32_t* ql = full ? nullptr : reinterpret_cast<const uint32_t*>(qlist_in) + (size_t)inst * qcap * 2;
  int total;
  constexpr int kRegKeys = 16;
  if (M <= kRegKeys * nthr) {
    // keys in registers, loaded straight from the costs / qualifier list (the
    // costs were written by other CTAs before the grid barrier: L2 loads)
    unsigned long long kr[kRegKeys];
#pragma unroll
    for (int i = 0; i < kRegKeys; ++i) {
      const int j = tid + i * nthr;
      kr[i] = ~0ull;
      if (j < M) {
        if (j < K || full) kr[i] = ((unsigned long long)ord32((float)__ldcg(c + j)) << 32) | (unsigned)j;
        else kr[i] = ((unsigned long long)__ldcg(ql + 2 * (j - K)) << 32) | __ldcg(ql + 2 * (j - K) + 1);
      }
    }
    if (mk != nullptr && tid == 0) mk[0] = gtimer();
    radix_topk_regs<kRegKeys>(kr, M, K, E, hist, aux, total, mk != nullptr ? mk + 1 : nullptr);
  } else {
    for (int j = tid; j < M; j += nthr) {
      unsigned long long k;
      if (j < K || full) k = ((unsigned long long)ord32((float)c[j]) << 32) | (unsigned)j;
      else k = ((unsigned long long)ql[2 * (j - K)] << 32) | ql[2 * (j - K) + 1];
      keys[j] = k;
    }
    __syncthreads();
    radix_topk_compact(keys, M, K, E, hist, aux, total);
  }
  if (mk != nullptr && tid == 0) mk[10] = gtimer();
  const int ne = min(K, total);
  struct MarkEnd {  // mk[11]: end of the ranking / carry-over of this CTA's slice
    unsigned long long* m;
    __device__ ~MarkEnd() { if (m != nullptr && threadIdx.x == 0) m[11] = gtimer(); }
  } mark_end{mk};
  if (s_elite != nullptr) {
    // redundant mode (one grid barrier per generation): every CTA ranks ALL
    // K elites into its own shared rank -> row table (K^2 comparisons), then
    // carries over only its slice of the elite rows for the next generation
    for (int e = tid; e < ne; e += nthr) {
      const unsigned long long ke = E[e];
      int r = 0;
      for (int j = 0; j < ne; ++j) r += E[j] < ke ? 1 : 0;
      s_elite[r] = (int)(uint32_t)ke;
    }
    __syncthreads();
    const int per = (ne + gridDim.x - 1) / gridDim.x;
    const int r0 = blockIdx.x * per, r1 = min(ne, r0 + per);
    for (int r = r0 + warp; r < r1; r += nwarps) {
      const int re = s_elite[r];
      const S* from = pop_in + ((size_t)inst * N + re) * pm;
      S* to = pop_out + ((size_t)inst * N + r) * pm;
      for (int g = lane; g < pm; g += 32) to[g] = from[g];
      if (lane == 0) {
        cost_out[(size_t)inst * N + r] = c[re];
        if (fold_amin != nullptr) atomicMin(fold_amin, amin_key(c[re], r));  // the final population's elites
      }
    }
    return;
  }
  // ---- rank this CTA's slice of the elites (K keys, unique)
  const int per = (ne + gridDim.x - 1) / gridDim.x;
  const int e0 = blockIdx.x * per, e1 = min(ne, e0 + per);
  for (int e = e0 + warp; e < e1; e += nwarps) {
    const unsigned long long ke = E[e];
    int r = 0;
    for (int j = lane; j < ne; j += 32) r += E[j] < ke ? 1 : 0;
    r = __reduce_add_sync(0xFFFFFFFFu, r);
    const int re = (int)(uint32_t)ke;
    if (lane == 0) elite_idx[(size_t)inst * K + r] = re;
    if (pop_out != nullptr) {
      const S* from = pop_in + ((size_t)inst * N + re) * pm;
      S* to = pop_out + ((size_t)inst * N + r) * pm;
      for (int g = lane; g < pm; g += 32) to[g] = from[g];
      if (lane == 0) cost_out[(size_t)inst * N + r] = c[re];
    }
  }
}

template <typename S>
__global__ void __launch_bounds__(1024) select_radix_kernel(const S* __restrict__ costs, int N, int K,
                                                            int* __restrict__ elite_idx, int incremental,
                                                            int* __restrict__ qcount_in,
                                                            const void* __restrict__ qlist_in,
                                                            int* __restrict__ qcount_next, int qcap,
                                                            const S* __restrict__ pop_in, S* __restrict__ pop_out,
                                                            S* __restrict__ cost_out, int pm) {
  if constexpr (sizeof(S) == 4)
    select_radix_body<S>(costs, N, K, elite_idx, incremental, qcount_in, qlist_in, qcount_next, qcap, pop_in, pop_out,
                         cost_out, pm);
}

template <typename S>
__global__ void __launch_bounds__(256) select_kernel(const S* __restrict__ costs, int N, int K,
                                                     int* __restrict__ elite_idx, int incremental,
                                                     int* __restrict__ qcount_in, const void* __restrict__ qlist_in,
                                                     int* __restrict__ qcount_next, int qcap,
                                                     const S* __restrict__ pop_in, S* __restrict__ pop_out,
                                                     S* __restrict__ cost_out, int pm) {
  select_body<S>(costs, N, K, elite_idx, incremental, qcount_in, qlist_in, qcount_next, qcap, pop_in, pop_out,
                 cost_out, pm);
}

// ---------------------------------------------------------------------------
// Population sharding over GPUs: every rank holds the K
// elites (replicated) and its own slice of the children.  Per generation
// each rank exports its local top-K candidates as self-contained entries
// (key, global row, cost, genes); after an all-gather of W x K entries every
// rank ranks the union identically and installs the global top-K as rows
// [0, K).  Keys use GLOBAL rows and the RNG counters GLOBAL child indices, so
// the result equals the unsharded solve for any number of ranks.

template <typename S>
__host__ __device__ inline size_t shard_entry_bytes(int pm) {
  return ((size_t)24 + (size_t)pm * sizeof(S) + 15) & ~(size_t)15;
}

template <typename S>
__global__ void __launch_bounds__(256) shard_export_kernel(const S* __restrict__ pop, const S* __restrict__ costs,
                                                           int K, int pm, int incl_elites, int n_local,
                                                           long long gbase, unsigned char* __restrict__ out) {
  using OT = typename OrdOf<S>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int E0 = incl_elites ? K : 0;
  const int M = E0 + n_local;
  OT* ck = reinterpret_cast<OT*>(smem_raw);
  unsigned* cr = reinterpret_cast<unsigned*>(ck + M);  // global rows
  int* lr = reinterpret_cast<int*>(cr + M);            // local rows
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const size_t eb = shard_entry_bytes<S>(pm);
  pdl_wait();
  for (int j = tid; j < M; j += nthr) {
    const int row = j < E0 ? j : K + (j - E0);
    lr[j] = row;
    cr[j] = j < E0 ? (unsigned)j : (unsigned)(gbase + (j - E0));
    ck[j] = OrdOf<S>::ord(costs[row]);
  }
  __syncthreads();
  if (blockIdx.x == 0)  // sentinels when this rank holds fewer than K candidates
    for (int r = M + tid; r < K; r += nthr) {
      unsigned char* e = out + (size_t)r * eb;
      *reinterpret_cast<unsigned long long*>(e) = ~0ull;
      *reinterpret_cast<unsigned*>(e + 8) = 0xFFFFFFFFu - (unsigned)r;
      *reinterpret_cast<unsigned*>(e + 12) = 0u;
    }
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int e0 = blockIdx.x * per, e1 = min(M, e0 + per);
  for (int e = e0 + warp; e < e1; e += nwarps) {
    const OT ke = ck[e];
    const unsigned re = cr[e];
    int cnt = 0;
    for (int j = lane; j < M; j += 32) cnt += (ck[j] < ke || (ck[j] == ke && cr[j] < re)) ? 1 : 0;
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (cnt < K) {
      unsigned char* ent = out + (size_t)cnt * eb;
      const S* g = pop + (size_t)lr[e] * pm;
      if (lane == 0) {
        *reinterpret_cast<unsigned long long*>(ent) = (unsigned long long)ke;
        *reinterpret_cast<unsigned*>(ent + 8) = re;
        *reinterpret_cast<unsigned*>(ent + 12) = 1u;
        *reinterpret_cast<S*>(ent + 16) = costs[lr[e]];
      }
      S* dst = reinterpret_cast<S*>(ent + 24);
      for (int q = lane; q < pm; q += 32) dst[q] = g[q];
    }
  }
}

// FP32 export by radix select (the local set is K elites + ~(N-K)/W
// children: O(M^2) ranking dominated the one-rank C4 shard at 16k rows).
// Same entries, same order as shard_export_kernel.  One CTA per slice of
// the K output ranks; every CTA finds the K-th key itself.
__host__ __device__ inline size_t shard_export_radix_smem(int M, int K) {
  return (size_t)M * 8 + (size_t)M * 4 + (size_t)K * 8 + 256 * 4 + 64 * 4 + 64;
}

#ifdef EMPC_HOST_TU
__global__ void __launch_bounds__(1024) shard_export_radix_kernel(const float* __restrict__ pop,
                                                                  const float* __restrict__ costs, int K, int pm,
                                                                  int incl_elites, int n_local, long long gbase,
                                                                  unsigned char* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int E0 = incl_elites ? K : 0;
  const int M = E0 + n_local;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);  // (ord, global row)
  int* lr = reinterpret_cast<int*>(keys + M);                                     // local rows
  unsigned long long* E = reinterpret_cast<unsigned long long*>(lr + M + (M & 1));
  int* hist = reinterpret_cast<int*>(E + K);
  int* aux = hist + 256;
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const size_t eb = shard_entry_bytes<float>(pm);
  pdl_wait();
  for (int j = tid; j < M; j += nthr) {
    const int row = j < E0 ? j : K + (j - E0);
    const unsigned grow = j < E0 ? (unsigned)j : (unsigned)(gbase + (j - E0));
    lr[j] = row;
    keys[j] = ((unsigned long long)ord32(costs[row]) << 32) | grow;
  }
  if (blockIdx.x == 0)  // sentinels when this rank holds fewer than K candidates
    for (int r = M + tid; r < K; r += nthr) {
      unsigned char* e = out + (size_t)r * eb;
      *reinterpret_cast<unsigned long long*>(e) = ~0ull;
      *reinterpret_cast<unsigned*>(e + 8) = 0xFFFFFFFFu - (unsigned)r;
      *reinterpret_cast<unsigned*>(e + 12) = 0u;
    }
  int total;
  radix_topk_compact(keys, M, K, E, hist, aux, total);
  const int ne = min(K, total);
  const int per = (ne + gridDim.x - 1) / gridDim.x;
  const int e0 = blockIdx.x * per, e1 = min(ne, e0 + per);
  for (int e = e0 + warp; e < e1; e += nwarps) {
    const unsigned long long ke = E[e];
    int r = 0;
    for (int j = lane; j < ne; j += 32) r += E[j] < ke ? 1 : 0;
    r = __reduce_add_sync(0xFFFFFFFFu, r);
    // local row of this key: the global row identifies it uniquely
    const unsigned grow = (unsigned)ke;
    const int row = grow < (unsigned)E0 ? (int)grow : K + (int)((long long)grow - gbase);
    unsigned char* ent = out + (size_t)r * eb;
    const float* g = pop + (size_t)row * pm;
    if (lane == 0) {
      // the entry key is the 32-bit orderable cost, as shard_export_kernel writes it
      *reinterpret_cast<unsigned long long*>(ent) = (unsigned long long)(uint32_t)(ke >> 32);
      *reinterpret_cast<unsigned*>(ent + 8) = grow;
      *reinterpret_cast<unsigned*>(ent + 12) = 1u;
      *reinterpret_cast<float*>(ent + 16) = costs[row];
    }
    float* dst = reinterpret_cast<float*>(ent + 24);
    for (int q = lane; q < pm; q += 32) dst[q] = g[q];
  }
  (void)lr;
}
#endif  // EMPC_HOST_TU

template <typename S>
__global__ void __launch_bounds__(256) shard_import_kernel(const unsigned char* __restrict__ all, int M, int K, int pm,
                                                           int m, S* __restrict__ pop, S* __restrict__ costs,
                                                           int* __restrict__ elite_idx, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* ck = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned* cr = reinterpret_cast<unsigned*>(ck + M);
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const size_t eb = shard_entry_bytes<S>(pm);
  pdl_wait();
  for (int j = tid; j < M; j += nthr) {
    ck[j] = *reinterpret_cast<const unsigned long long*>(all + (size_t)j * eb);
    cr[j] = *reinterpret_cast<const unsigned*>(all + (size_t)j * eb + 8);
  }
  __syncthreads();
  const int per = (M + gridDim.x - 1) / gridDim.x;
  const int e0 = blockIdx.x * per, e1 = min(M, e0 + per);
  for (int e = e0 + warp; e < e1; e += nwarps) {
    const unsigned long long ke = ck[e];
    const unsigned re = cr[e];
    int cnt = 0;
    for (int j = lane; j < M; j += 32) cnt += (ck[j] < ke || (ck[j] == ke && cr[j] < re)) ? 1 : 0;
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    if (cnt < K) {
      const unsigned char* ent = all + (size_t)e * eb;
      const S* g = reinterpret_cast<const S*>(ent + 24);
      for (int q = lane; q < pm; q += 32) pop[(size_t)cnt * pm + q] = g[q];
      if (lane == 0) {
        const S c = *reinterpret_cast<const S*>(ent + 16);
        costs[cnt] = c;
        elite_idx[cnt] = cnt;
        if (cnt == 0) {
          out[m + pm] = (double)c;
          out[m + pm + 1] = (double)re;
        }
      }
      if (cnt == 0)
        for (int q = lane; q < pm; q += 32) {
          out[m + q] = (double)g[q];
          if (q < m) out[q] = (double)g[q];
        }
    }
  }
}

// ---------------------------------------------------------------------------
// finalize: argmin (first NaN, else first minimum: numpy argmin) and the
// best candidate, written as FP64 [u (m) | best (pm) | cost | index].

template <typename S>
__device__ __forceinline__ void finalize_body(const S* __restrict__ cands, const S* __restrict__ costs, int N, int m,
                                              int pm, double* __restrict__ out, int inst) {
  const S* c = costs + (size_t)inst * N;
  pdl_wait();
  uint64_t bo = ~0ull;
  int bi = 0x7FFFFFFF;
  // four independent loads in flight per thread (C4: 16k costs, one CTA)
  for (int i0 = threadIdx.x; i0 < N; i0 += 4 * blockDim.x) {
    S v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < N ? c[i] : S(0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < N) {
        uint64_t o;
        if constexpr (sizeof(S) == 4) o = (v[u] != v[u]) ? 0ull : (uint64_t)ord32((float)v[u]);
        else o = (v[u] != v[u]) ? 0ull : ord64((double)v[u]);
        if (o < bo || (o == bo && i < bi)) { bo = o; bi = i; }
      }
    }
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

template <typename S>
__global__ void finalize_kernel(const S* __restrict__ cands, const S* __restrict__ costs, int N, int m, int pm,
                                double* __restrict__ out) {
  finalize_body<S>(cands, costs, N, m, pm, out, blockIdx.x);
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

#ifdef EMPC_HOST_TU
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

#endif  // EMPC_HOST_TU

// ---------------------------------------------------------------------------
// Persistent cooperative solve (single instance, all tiles co-resident): the
// whole cold / warm solve of K/empc.py:211-236 in one launch.  The problem is
// staged into shared memory (and A into registers) once; each generation is
//   grid.sync -> distributed selection (select_body) -> grid.sync ->
//   breed + rollout of this CTA's tile (rollout_body)
// and the argmin runs on CTA 0 after the last generation.  Same kernels'
// arithmetic as the per-launch path, so results are identical to it.

template <typename S>
struct PersistArgs {
  RolloutArgs<S> ro;  // init / rescore launch of generation 0 (the rest is derived)
  int evolves;
  int tile_evolve;    // candidates per CTA for the evolves (tile for gen 0 is ro.tile)
  int incremental;
  size_t scratch;     // leading shared-memory bytes the selection needs
  S* pop[2];
  S* cost[2];
  int* qcount;        // [2] double-buffered qualifier counts
  void* qlist;        // [3][qcap] (key, row) pairs (two used unless one_sync)
  int* elite;         // elite_idx (written by the selection)
  double* out;
  int predraw;        // WS variant with helper warps: next-generation draws during the recursion
  int radix;          // selection by radix select (FP32)
  int dbg_gen;        // EMPC_PHASES: evolve whose phases are recorded (-1: every one, the last wins)
  unsigned long long* amin;  // distributed argmin key (FP32), NULL: CTA 0 scans the population
  int one_sync;       // one grid barrier per generation (redundant per-CTA selection, FP32)
  size_t elite_off;   // shared-memory offset of the per-CTA rank -> row table (one_sync)
  // injected draws of the evolves (parity mode; NULL: in-kernel Philox):
  // evolve g reads parents + g (N-K) 2, masks / noise + g (N-K) p m
  const int* inj_parents;
  const uint8_t* inj_take;
  const uint8_t* inj_mut;
  const double* inj_noise;
};

__device__ __forceinline__ unsigned char* smem_raw_persist() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return smem_raw;
}

template <typename S, int NP, int RR, int CC, bool AREG, bool DQ, int KS, bool WS, int MAXT, bool HK = false>
__global__ void __launch_bounds__(MAXT, 1) persist_kernel(const PersistArgs<S> P) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  RolloutArgs<S> a = P.ro;
  const int N = a.d.N, K = a.d.K, pm = a.d.pm;
  using OT = typename std::conditional<sizeof(S) == 4, uint32_t, uint64_t>::type;
  const size_t qstride = (size_t)a.qcap * 2 * sizeof(OT);
  const int nc = N - K;
  const int dt0 = blockIdx.x * P.tile_evolve;
  a.draw_next = P.predraw && P.evolves > 0;
  a.draw_evolve = 0;
  a.draw_tile0 = dt0;
  a.draw_cnt = min(P.tile_evolve, nc - dt0);
  // phase timers (EMPC_PHASES): CTA 0 stamps the start, the end of the init
  // rollout and the end of every generation (after `gridDim.x * 16` slots)
  unsigned long long* gt = (a.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0) ? a.dbg + gridDim.x * 16 : nullptr;
  if (gt) gt[0] = gtimer();
  // distributed argmin of the final population (FP32, at least one evolve):
  // every CTA folds its rows of the last generation into one 64-bit key;
  // reset here, first folded after two grid barriers
  const bool dist_amin = sizeof(S) == 4 && P.amin != nullptr;
  if (dist_amin && blockIdx.x == 0 && threadIdx.x == 0) *P.amin = ~0ull;
  a.amin = nullptr;
  rollout_body<S, NP, RR, CC, AREG, DQ, KS, WS, HK>(a, true, P.scratch);
  if (gt) gt[1] = gtimer();
  int cur = 0;
  // one-barrier generations (FP32): every CTA computes the whole selection
  // itself (radix select + ranking of the K elites into a shared table), so
  // breeding needs no second grid barrier.  Qualifier lists rotate over
  // three buffers: evolve g appends to B[g % 3], its selection reads
  // B[(g-1) % 3] and clears B[(g+1) % 3] (last read by evolve g-1's
  // selection, next appended after the next barrier); B[0] is cleared here.
  int* s_elite = (sizeof(S) == 4 && P.one_sync) ? reinterpret_cast<int*>(smem_raw_persist() + P.elite_off) : nullptr;
  if (s_elite != nullptr && blockIdx.x == 0 && threadIdx.x == 0) P.qcount[0] = 0;
  for (int g = 0; g < P.evolves; ++g) {
    if (gt && g > 0 && g + 1 < 30) gt[g + 1] = gtimer();
    // selection marks 13-15 of the evolve the rollout marks record
    const bool mark = a.dbg != nullptr && threadIdx.x == 0 && (P.dbg_gen < 0 || g == P.dbg_gen);
    unsigned long long* const mk = mark ? a.dbg + (size_t)blockIdx.x * 16 : nullptr;
    if (mk) mk[13] = gtimer();
    grid.sync();
    if (mk) mk[14] = gtimer();
    const int inc = (g > 0 && P.incremental) ? 1 : 0;
    if constexpr (sizeof(S) == 4) {
      if (s_elite != nullptr) {
        select_radix_body<S>(P.cost[cur], N, K, P.elite, inc, inc ? P.qcount + ((g + 2) % 3) : nullptr,
                             (const char*)P.qlist + ((g + 2) % 3) * qstride, P.qcount + ((g + 1) % 3), a.qcap,
                             P.pop[cur], P.pop[cur ^ 1], P.cost[cur ^ 1], pm, s_elite,
                             (dist_amin && g + 1 == P.evolves) ? P.amin : nullptr);
        __syncthreads();  // s_elite complete; the scratch is the rollout's again
      } else if (P.radix && !inc) {
        // the first selection ranks all N candidates (35 us by counting at
        // C3): radix select of the K-th key + ranking of the K elites only.
        // Later (incremental) sets are small enough for rank-by-counting,
        // which needs fewer passes and barriers
        select_radix_body<S>(P.cost[cur], N, K, P.elite, inc, inc ? P.qcount + ((g - 1) & 1) : nullptr,
                             (const char*)P.qlist + ((g - 1) & 1) * qstride, P.qcount + (g & 1), a.qcap,
                             P.pop[cur], P.pop[cur ^ 1], P.cost[cur ^ 1], pm, nullptr, nullptr,
                             gt != nullptr ? gt + 32 : nullptr);
      } else {
        select_body<S, (NP >= 24 ? 8 : 0)>(P.cost[cur], N, K, P.elite, inc, inc ? P.qcount + ((g - 1) & 1) : nullptr,
                       (const char*)P.qlist + ((g - 1) & 1) * qstride, P.qcount + (g & 1), a.qcap, P.pop[cur],
                       P.pop[cur ^ 1], P.cost[cur ^ 1], pm);
      }
    } else {
      select_body<S, (NP >= 24 ? 8 : 0)>(P.cost[cur], N, K, P.elite, inc, inc ? P.qcount + ((g - 1) & 1) : nullptr,
                     (const char*)P.qlist + ((g - 1) & 1) * qstride, P.qcount + (g & 1), a.qcap, P.pop[cur],
                     P.pop[cur ^ 1], P.cost[cur ^ 1], pm);
    }
    if (mk) mk[15] = gtimer();
    if (s_elite == nullptr) grid.sync();
    RolloutArgs<S> b = a;
    b.mode = P.inj_parents != nullptr ? kBreedInject : kBreedPhilox;
    if (P.dbg_gen >= 0) b.dbg = g == P.dbg_gen ? a.dbg : nullptr;  // phase marks of one chosen evolve
    if (P.inj_parents != nullptr) {
      const size_t per = (size_t)(N - K) * pm;
      b.inj_parents = P.inj_parents + (size_t)g * (N - K) * 2;
      b.inj_take = P.inj_take + (size_t)g * per;
      b.inj_mut = P.inj_mut + (size_t)g * per;
      b.inj_noise = P.inj_noise + (size_t)g * per;
    }
    b.nc = N - K;
    b.row0 = K;
    b.amin = (dist_amin && g + 1 == P.evolves) ? P.amin : nullptr;
    b.tile = P.tile_evolve;
    b.evolve = g;
    b.copy_elites = 0;
    b.parents_from_out = s_elite == nullptr ? 1 : 0;  // one-barrier mode: parents via the shared table, from pop_in
    if (s_elite != nullptr) b.elite_idx = s_elite;
    b.draws_ready = P.predraw;  // (CTAs without init candidates drew theirs at the early return)
    b.draw_next = P.predraw && g + 1 < P.evolves;
    b.draw_evolve = g + 1;
    b.pop_in = P.pop[cur];
    b.cost_in = P.cost[cur];
    b.pop_out = P.pop[cur ^ 1];
    b.cost_out = P.cost[cur ^ 1];
    const int qb = s_elite != nullptr ? g % 3 : (g & 1);
    b.qcount = P.incremental ? P.qcount + qb : nullptr;
    b.qlist = (char*)P.qlist + qb * qstride;
    rollout_body<S, NP, RR, CC, AREG, DQ, KS, WS, HK>(b, false, P.scratch);
    cur ^= 1;
  }
  if (gt && P.evolves > 0 && P.evolves + 1 < 30) gt[P.evolves + 1] = gtimer();
  if (dist_amin && P.evolves > 0 && s_elite == nullptr) {
    // the elite rows [0, K) of the final population, a slice per CTA
    const int per = (K + gridDim.x - 1) / gridDim.x;
    for (int r = blockIdx.x * per + threadIdx.x; r < min(K, (int)(blockIdx.x + 1) * per); r += blockDim.x)
      atomicMin(P.amin, amin_key(P.cost[cur][r], r));
  }
  grid.sync();
  if (blockIdx.x == 0) {
    if (dist_amin && P.evolves > 0) {
      const int best = (int)(uint32_t)*reinterpret_cast<volatile unsigned long long*>(P.amin);
      const S* bc = P.pop[cur] + (size_t)best * pm;
      for (int q = threadIdx.x; q < pm; q += blockDim.x) {
        P.out[a.d.m + q] = (double)bc[q];
        if (q < a.d.m) P.out[q] = (double)bc[q];  // u = first knot (K/empc.py:236)
      }
      if (threadIdx.x == 0) {
        P.out[a.d.m + pm] = (double)P.cost[cur][best];
        P.out[a.d.m + pm + 1] = (double)best;
      }
    } else {
      finalize_body<S>(P.pop[cur], P.cost[cur], N, a.d.m, pm, P.out, 0);
    }
  }
  if (gt) gt[31] = gtimer();
}

}  // namespace empc
