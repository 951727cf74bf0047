// Tensor-core rollout (K2 + K3 with the K5 prologue) for FP32 populations.
//
// Same function as rollout_kernel (K/empc.py:85-119 scoring of the bred
// children, K/empc.py:174-208), different machine: one CTA scores a tile of
// 128 candidates and the per-step matrix product of the recursion
//
//     e_{k+1} = e_k + Delta e_k + drive_k,    Delta = A_d - I,  e = x - x_goal
//
// runs on the 5th-generation tensor cores as D = E_k Delta' (M = 128
// candidates, N = K = n states) with the TF32 split-precision scheme
// (E = E_hi + E_lo, Delta = D_hi + D_lo, D = E_hi D_hi' + E_lo D_hi' + E_hi
// D_lo'; dropped term and TF32 truncation of the lo parts ~2^-21 relative to
// |Delta e|, itself ~dt |e|), FP32 accumulation in TMEM.  Everything else stays
// in FP32 on the CUDA cores: thread (candidate c, column group h) keeps its
// NH state coordinates, the knot-interpolated drive and the cost in
// registers, reads Delta e from its TMEM lane (c) and writes the next E_hi /
// E_lo row back to the same lane: the A operand of the next step's MMA lives
// in TMEM (tcgen05.mma with [a_tmem]), Delta hi / lo (B) in shared memory.
// The epilogue is O(n) per candidate-step against the O(n^2) of the FFMA
// recursion.
//
// Layout: TMEM columns D [0, NN), E_hi [NN, NN + NK), E_lo [NN + NK, NN + 2 NK);
// smem Dl[2][NK/4][NN][4] (empc_tc.cuh core-matrix layout), aliasing the
// breeding scratch (crossover bits, parent rows).
#pragma once

#include "empc_kernels.cuh"
#include "empc_tc.cuh"

namespace empc {

constexpr int kTcTile = 128;  // candidates per CTA = MMA M
// knot tile stride UsT[gene][kUsS]: one spare column so the breeding writes
// (consecutive genes of one child) fall in different banks
constexpr int kUsS = kTcTile + 1;

struct TcSmem {
  size_t r1, r2, r3, bs, vec, sched, g, red, bar, total;
};

// shared-memory plan of rollout_tc_kernel (host and device agree)
// multi: the CTA loops over several tiles, Delta gets its own region (r3)
// instead of aliasing the breeding scratch (r2)
__host__ __device__ inline TcSmem tc_smem(int NN, int NK, int NP, int m, int T, int p, int WG, bool multi = false) {
  auto al = [](size_t x) { return (x + 127) & ~(size_t)127; };
  const int pm = p * m;
  TcSmem s;
  s.r1 = al((size_t)pm * kUsS * 4);
  const size_t dl = (size_t)2 * NN * NK * 4, br = (size_t)kTcTile * pm + 16 + (size_t)2 * kTcTile * 4;
  s.r2 = al(multi ? br : (dl > br ? dl : br));
  s.r3 = multi ? al(dl) : 0;
  s.bs = al((size_t)NP * ((m + 3) & ~3) * 4);
  s.vec = al((size_t)(4 * NP + 5 * m) * 4);
  s.sched = al((size_t)T * 12);
  s.g = al((size_t)(p * p + 2) * 4);
  s.red = al((size_t)WG * kTcTile * 4);
  s.bar = 128;  // mbarrier + TMEM address
  s.total = s.r1 + s.r2 + s.r3 + s.bs + s.vec + s.sched + s.g + s.red + s.bar;
  return s;
}

// NN: MMA N (states, multiple of 16); NK: MMA K (states, multiple of 8);
// NH: state coordinates per thread (multiple of 4); WG: column groups,
// NH * WG >= n; threads = 128 * WG.
template <int NP, int NN, int NK, int NH, int WG, int MINB>
__global__ void __launch_bounds__(kTcTile * WG, MINB) rollout_tc_kernel(const RolloutArgs<float> a) {
  using S = float;
  static_assert(NH % 4 == 0 && NN % 16 == 0 && NK % 8 == 0 && NH * WG <= NK && NH * WG <= NN, "tc shape");
  extern __shared__ __align__(16) unsigned char smem_tc[];
  const Dims& d = a.d;
  const StageLayout& SL = a.SL;
  const int n = d.n, m = d.m, T = d.T, p = d.p;
  const int mP = (m + 3) & ~3;  // padded row stride of Bs
  const int inst = blockIdx.y;
  const bool multi = a.tc_multi != 0;
  // candidates per tile a.tile <= 128 (MMA M stays 128; rows >= cnt are
  // padding): small populations spread over all SMs
  const int tsz = a.tile;
  const int ntiles = (a.nc + tsz - 1) / tsz;
  int tile0 = blockIdx.x * tsz;
  int cnt = min(tsz, a.nc - tile0);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const int c = tid & (kTcTile - 1);  // candidate = TMEM lane
  const int h = tid >> 7;             // column group
  const double* __restrict__ P = a.prob + (size_t)inst * SL.stride;
  const double* __restrict__ X = a.state + (size_t)inst * SL.sstride;
  const size_t pop_base = (size_t)inst * a.rows;
  const bool breed = (a.mode == kBreedPhilox || a.mode == kBreedInject);

  const TcSmem sp = tc_smem(NN, NK, NP, m, T, p, WG, multi);
  unsigned char* ptr = smem_tc;
  S* R1 = reinterpret_cast<S*>(ptr); ptr += sp.r1;
  unsigned char* R2 = ptr; ptr += sp.r2;
  unsigned char* R3 = multi ? ptr : R2; ptr += sp.r3;
  S* Bs = reinterpret_cast<S*>(ptr); ptr += sp.bs;  // [NP][m]
  S* cw_ = reinterpret_cast<S*>(ptr); ptr += sp.vec;
  S* cqd = cw_ + NP;
  S* cxg = cqd + NP;
  S* cx0 = cxg + NP;
  S* cug = cx0 + NP;
  S* cumin = cug + m;
  S* cumax = cumin + m;
  S* csig = cumax + m;
  S* crd = csig + m;
  int* sI1 = reinterpret_cast<int*>(ptr);
  int* sI2 = sI1 + T;
  S* sC = reinterpret_cast<S*>(sI2 + T); ptr += sp.sched;
  S* sG = reinterpret_cast<S*>(ptr); ptr += sp.g;
  S* red = reinterpret_cast<S*>(ptr); ptr += sp.red;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(ptr);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(ptr + 8);
  uint32_t* kmask = reinterpret_cast<uint32_t*>(ptr + 12);  // K-steps (8 columns) where Delta is nonzero
  uint64_t* ebar = reinterpret_cast<uint64_t*>(ptr + 16);   // every warp's epilogue of a step is done
  S* UsT = R1;                                   // [gene][128]
  int* src = reinterpret_cast<int*>(R2);         // breeding scratch ...
  uint8_t* tbits = R2 + 2 * kTcTile * 4;
  S* Dhi = reinterpret_cast<S*>(R3);             // ... then (or beside it) Delta hi / lo [NK/4][NN][4]
  S* Dlo = Dhi + (size_t)NN * NK;
  // TMEM columns: D [0, NN), E_hi [NN, NN + NK), E_lo [NN + NK, NN + 2 NK)
  constexpr uint32_t kCols = tc::tmem_cols_for(NN + 2 * NK);

  // Column blocks of Delta that are exactly zero contribute exactly zero:
  // their K-steps are not issued (e.g. the position columns of a linearized
  // mechanism without gravity: half of K)
  auto stage_delta = [&]() {
    uint32_t lmask = 0u;
    for (int e = tid; e < NN * NK; e += nthr) {
      const int i = e / NK, j = e - (e / NK) * NK;
      const S v = (i < n && j < n) ? (S)(P[SL.ad + i * n + j] - (i == j ? 1.0 : 0.0)) : S(0);
      const S hi = tc::to_tf32(v);
      const int o = (j >> 2) * NN * 4 + i * 4 + (j & 3);
      Dhi[o] = hi;
      Dlo[o] = v - hi;
      if (v != S(0)) lmask |= 1u << (j >> 3);
    }
    if (lmask) atomicOr(kmask, lmask);
  };

  EMPC_MARK(0)
  // ---- phase 0: problem -> smem (independent of the producer grid)
  if (cnt > 0) {
    for (int k = tid; k < T; k += nthr) {
      sI1[k] = a.idx1[k];
      sI2[k] = a.idx2[k];
      sC[k] = a.cw[k];
    }
    for (int e = tid; e < p * p; e += nthr) sG[e] = a.G[e];
    for (int e = tid; e < NP * mP; e += nthr) {
      const int i = e / mP, l = e - (e / mP) * mP;
      Bs[e] = (i < n && l < m) ? (S)P[SL.bd + i * m + l] : S(0);
    }
    // error coordinates (see rollout_body): w' = w + Delta x_goal, in FP64
    for (int i = warp; i < NP; i += nwarps) {
      double acc = 0.0;
      if (i < n)
        for (int j = lane; j < n; j += 32) acc = fma(P[SL.ad + i * n + j] - (i == j ? 1.0 : 0.0), P[SL.xg + j], acc);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
      if (lane == 0) cw_[i] = i < n ? (S)(P[SL.wd + i] + acc) : S(0);
    }
    for (int i = tid; i < NP; i += nthr) {
      const bool ok = i < n;
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
    if (warp == 0) {  // k = 0 state term (diagonal Q), FP64
      double part = 0.0;
      for (int i = lane; i < n; i += 32) {
        const double ei = X[SL.x0 + i] - P[SL.xg + i];
        part = fma(P[SL.q + i * n + i] * ei, ei, part);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, off);
      if (lane == 0) sG[p * p] = (S)part;
    }
    if (warp == 0) tc::tmem_alloc(tslot, kCols);
    if (tid == 32) {
      tc::mbar_init(mbar, 1);
      tc::mbar_init(ebar, (uint32_t)nwarps);
      tc::mbar_fence_init();
      *kmask = 0u;
    }
  }
  EMPC_MARK(7)
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (multi && cnt > 0) stage_delta();  // once per CTA (own region); kmask is read after later barriers
  EMPC_MARK(8)
  const uint32_t tmem = *tslot;
  int gstep = 0;  // steps of this CTA over all its tiles (mbarrier phases)
  for (int tile = blockIdx.x, it = 0; it == 0 || tile < ntiles; tile += gridDim.x, ++it) {
  tile0 = tile * tsz;
  cnt = min(tsz, a.nc - tile0);
  // warps whose 32 TMEM lanes are all padding skip the epilogue (they still
  // follow the step barriers)
  const bool wlive = 32 * (warp & 3) < cnt;
  // ---- phase 1: K5 prologue (draws, PDL wait, elites, children -> UsT + HBM)
  if (!breed_tile<S>(a, inst, tile0, cnt, kTcTile, kUsS, UsT, src, tbits, cumin, cumax, csig, pop_base, it == 0))
    return;  // (only a CTA without any tile gets here: nothing was allocated for it)
  __syncthreads();
  EMPC_MARK(3)

  // ---- phase 2: input cost z'(W'W (x) R)z (K/empc.py:100-101) over the
  // channels l = h (mod WG), and the drive at the first knot pair
  S cst0 = S(0), cst1 = S(0);
  if (a.r_diag && p <= 8) {
    // z_b = U_b,l - u_goal,l in registers; r_l z' G z with G = W'W from smem
    for (int l = wlive ? h : m; l < m; l += WG) {
      const S ugl = cug[l];
      S z[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) z[b] = b < p ? UsT[(b * m + l) * kUsS + c] - ugl : S(0);
      S v = S(0);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (t >= p) break;
        S gz = S(0);
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (b < p) gz = fma(sG[t * p + b], z[b], gz);
        v = fma(z[t], gz, v);
      }
      cst0 = fma(crd[l], v, cst0);
    }
  } else {
    for (int l = wlive ? h : m; l < m; l += WG) {
      const S ugl = cug[l];
      for (int t = 0; t < p; ++t) {
        S gz = S(0);
        for (int b = 0; b < p; ++b) {
          S rz;
          if (a.r_diag) {
            rz = crd[l] * (UsT[(b * m + l) * kUsS + c] - ugl);
          } else {
            rz = S(0);
            for (int l2 = 0; l2 < m; ++l2)
              rz = fma((S)P[SL.r + l * m + l2], UsT[(b * m + l2) * kUsS + c] - cug[l2], rz);
          }
          gz = fma(sG[t * p + b], rz, gz);
        }
        cst0 = fma(UsT[(t * m + l) * kUsS + c] - ugl, gz, cst0);
      }
    }
  }
  EMPC_MARK(11)
  // drive at the knots (K/empc.py:104-105): b_j = w' + B U_j, held as the
  // segment start g = b_{i1} and slope hs = b_{i2} - b_{i1}.  seg_drive
  // adds B U_i1 to g (full) and B (U_i2 - U_i1) to hs, with the knots from
  // UsT[gene][cand] (smem for the whole recursion) and B rows as float4
  const int r0 = h * NH;  // first state coordinate of this thread
  S g[NH], hs[NH];
  auto seg_drive = [&](int i1, int i2, bool full) {
    if (full) {
#pragma unroll 1
      for (int l = 0; l < mP; l += 4) {
        float u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = l + q < m ? UsT[(i1 * m + l + q) * kUsS + c] : S(0);
#pragma unroll
        for (int i = 0; i < NH; ++i) {
          const float4 b = *reinterpret_cast<const float4*>(Bs + (r0 + i) * mP + l);
          g[i] = fma(b.x, u[0], fma(b.y, u[1], fma(b.z, u[2], fma(b.w, u[3], g[i]))));
        }
      }
    }
#pragma unroll 1
    for (int l = 0; l < mP; l += 4) {
      float du[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        du[q] = l + q < m ? UsT[(i2 * m + l + q) * kUsS + c] - UsT[(i1 * m + l + q) * kUsS + c] : S(0);
#pragma unroll
      for (int i = 0; i < NH; ++i) {
        const float4 b = *reinterpret_cast<const float4*>(Bs + (r0 + i) * mP + l);
        hs[i] = fma(b.x, du[0], fma(b.y, du[1], fma(b.z, du[2], fma(b.w, du[3], hs[i]))));
      }
    }
  };
  int ci1 = sI1[0], ci2 = sI2[0];
#pragma unroll
  for (int i = 0; i < NH; ++i) {
    g[i] = cw_[r0 + i];
    hs[i] = S(0);
  }
  if (wlive) seg_drive(ci1, ci2, true);
  EMPC_MARK(12)
  __syncthreads();  // the breeding scratch is consumed (UsT stays: knot changes)

  // ---- phase 3: Delta hi / lo -> smem (B operand), E_0 = e_0 (all
  // candidates) -> TMEM (A operand)
  if (!multi) stage_delta();
  S ev[NH];
#pragma unroll
  for (int i = 0; i < NH; ++i) ev[i] = cx0[r0 + i];
  const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)r0;  // my lane, my columns
  // E rows of this thread: its TMEM lane, columns NN + r0 (hi) / NN + NK + r0 (lo)
  // (the hi part is e itself: kind::tf32 reads the upper 19 bits of each
  // 32-bit element, which is exactly tf32_trunc(e); lo = e - tf32_trunc(e))
  auto store_e = [&](uint32_t qmask) {  // qmask: 8-column chunks to store (NH % 8 == 0)
    if constexpr (NH % 8 == 0) {
#pragma unroll
      for (int q = 0; q < NH / 8; ++q) {
        // per-chunk skipping pays where one thread holds every coordinate
        // (WG = 1, C5); with several column groups whole threads skip
        // (e_live below) and the unconditional store schedules better (C4)
        if (WG == 1 && !((qmask >> q) & 1u)) continue;
        float lo[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) lo[t] = ev[8 * q + t] - tc::tf32_trunc(ev[8 * q + t]);
        tc::tmem_st8(tl + NN + 8 * q, ev + 8 * q);
        tc::tmem_st8(tl + NN + NK + 8 * q, lo);
      }
    } else {
#pragma unroll
      for (int q = 0; q < NH / 4; ++q) {
        float hi[4], lo[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          hi[t] = ev[4 * q + t];
          lo[t] = ev[4 * q + t] - tc::tf32_trunc(ev[4 * q + t]);
        }
        tc::tmem_st4(tl + NN + 4 * q, hi);
        tc::tmem_st4(tl + NN + NK + 4 * q, lo);
      }
    }
    tc::tmem_wait_st();
  };
  store_e(~0u);  // (the nonzero K-steps of Delta are known after the next barrier)
  if (h == 0) {  // K padding columns stay zero
    const float z[4] = {0.f, 0.f, 0.f, 0.f};
    for (int kc = (NH * WG) / 4; kc < NK / 4; ++kc) {
      tc::tmem_st4(tl - r0 + NN + 4 * kc, z);
      tc::tmem_st4(tl - r0 + NN + NK + 4 * kc, z);
    }
    tc::tmem_wait_st();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (it == 0) pdl_trigger();
  EMPC_MARK(4)

  const uint32_t idesc = tc::idesc_tf32(kTcTile, NN);
  const uint32_t km = *kmask ? *kmask : 1u;  // Delta == 0: one K-step still clears D
  // E columns that no issued K-step reads (all-zero blocks of Delta) are not
  // stored after E_0: e.g. the position coordinates of an N-link arm
  const uint32_t emask = NH % 8 != 0 ? ~0u : (km >> (r0 / 8)) & ((1u << (NH / 8)) - 1u);
  const bool e_live = emask != 0u;
  const uint32_t tA0 = tmem + NN, tA1 = tmem + NN + NK;
  const uint64_t dB0 = tc::sdesc(tc::smem_u32(Dhi), NN * 16, 128);
  const uint64_t dB1 = tc::sdesc(tc::smem_u32(Dlo), NN * 16, 128);

  // ---- phase 4: horizon recursion, state cost fused (K/empc.py:110-118)
  // (built with -DEMPC_TC_PROF and run with EMPC_PHASES: thread 0
  // accumulates clock cycles per part of the step)
#ifdef EMPC_TC_PROF
  const bool prof = a.dbg != nullptr && tid == 0;
  long long pc[5] = {0, 0, 0, 0, 0}, t_ = prof ? clock64() : 0;
#define TC_LAP(I)                   \
  if (prof) {                       \
    const long long n_ = clock64(); \
    pc[I] += n_ - t_;               \
    t_ = n_;                        \
  }
#else
#define TC_LAP(I)
#endif
  for (int k = 0; k < T; ++k, ++gstep) {
    if (tid == 0) {
      // the previous step's epilogue is done in every warp (D read, E written)
      if (gstep > 0) {
        tc::mbar_wait(ebar, (uint32_t)((gstep - 1) & 1));
        tc::fence_after();
      }
      // D = E_lo Dhi' + E_hi Dlo' + E_hi Dhi'  (small terms first), over
      // the nonzero K-steps; the first MMA overwrites D
      uint32_t acc = 0u;
#pragma unroll
      for (int s = 0; s < NK / 8; ++s) {
        if ((km >> s) & 1u) {
          const uint64_t ob = (uint64_t)((s * 2 * NN * 16) >> 4);
          tc::mma_tf32_ts(tmem, tA1 + 8 * s, dB0 + ob, idesc, acc);
          tc::mma_tf32_ts(tmem, tA0 + 8 * s, dB1 + ob, idesc, 1);
          tc::mma_tf32_ts(tmem, tA0 + 8 * s, dB0 + ob, idesc, 1);
          acc = 1u;
        }
      }
      tc::commit(mbar);
    }
    TC_LAP(0)
    const int i1 = sI1[k], i2 = sI2[k];
    const S ck = sC[k];
    if (i1 != ci1 || i2 != ci2) {  // uniform: the knot pair of the drive moved (p - 1 times)
      // next segment (i1 = old i2): the start is the old end, g += hs, and
      // only the new slope B (U_i2 - U_i1) is a matvec; otherwise recompute
      const bool next = i1 == ci2;
#pragma unroll
      for (int i = 0; i < NH; ++i) {
        g[i] = next ? g[i] + hs[i] : cw_[r0 + i];
        hs[i] = S(0);
      }
      if (wlive) seg_drive(i1, i2, !next);
      ci1 = i1;
      ci2 = i2;
    }
    tc::mbar_wait(mbar, (uint32_t)(gstep & 1));
    tc::fence_after();
    TC_LAP(1)
    if (wlive) {
    float dv[NH];
    if constexpr (NH % 8 == 0) {
#pragma unroll
      for (int q = 0; q < NH / 8; ++q) tc::tmem_ld8(tl + 8 * q, dv + 8 * q);
    } else {
#pragma unroll
      for (int q = 0; q < NH / 4; ++q) {
        float t4[4];
        tc::tmem_ld4(tl + 4 * q, t4);
        dv[4 * q] = t4[0]; dv[4 * q + 1] = t4[1]; dv[4 * q + 2] = t4[2]; dv[4 * q + 3] = t4[3];
      }
    }
    tc::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < NH; ++i) asm volatile("" : "+f"(dv[i]));
#pragma unroll
    for (int i = 0; i < NH; i += 4) {
      const float4 q4 = *reinterpret_cast<const float4*>(cqd + r0 + i);
      const float qq[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const S en = ev[i + t] + (dv[i + t] + fma(ck, hs[i + t], g[i + t]));
        ev[i + t] = en;
        if (t & 1) cst1 = fma(qq[t] * en, en, cst1); else cst0 = fma(qq[t] * en, en, cst0);
      }
    }
    TC_LAP(2)
    if (k + 1 < T && e_live) store_e(emask);
    }
    TC_LAP(3)
    // no CTA barrier: each warp signals the MMA issuer and runs ahead to the
    // next step's MMA-completion wait
    tc::fence_before();
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(ebar)) : "memory");
    TC_LAP(4)
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
#undef TC_LAP
#ifdef EMPC_TC_PROF
  if (prof) {
    const size_t o = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16;
    a.dbg[o + 7] = (unsigned long long)pc[0];
    a.dbg[o + 8] = (unsigned long long)pc[1];
    a.dbg[o + 11] = (unsigned long long)pc[2];
    a.dbg[o + 12] = (unsigned long long)pc[3];
    a.dbg[o + 13] = (unsigned long long)pc[4];
  }
#endif
  EMPC_MARK(5)

  // ---- deterministic reduction over the column groups
  red[h * kTcTile + c] = cst0 + cst1;
  __syncthreads();
  using OT = uint32_t;
  OT tau = OT(0);
  const bool qual = breed && a.qcount != nullptr;
  if (qual) tau = ord_key(a.cost_in[pop_base + a.elite_idx[(size_t)inst * d.K + d.K - 1]]);
  const S c0s = sG[p * p];
  for (int cc = tid; cc < cnt; cc += nthr) {
    S s = S(0);
#pragma unroll
    for (int hh = 0; hh < WG; ++hh) s += red[hh * kTcTile + cc];
    const S cost = c0s + s;
    const int row = a.row0 + tile0 + cc;
    a.cost_out[pop_base + row] = cost;
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
  __syncthreads();  // red / UsT are reused by the next tile
  }  // tiles
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, kCols);
  EMPC_MARK(6)
}

}  // namespace empc
