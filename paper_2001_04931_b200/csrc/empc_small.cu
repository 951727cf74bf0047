// Resident single-CTA solve for small problems (C1: 2-DoF, N = 100, T = 20).
//
// The whole solve of K/empc.py:211-236 -- init (or re-score), G - 1 (or G)
// generations of stable selection, breeding and scoring, then argmin -- runs
// in ONE CTA per instance with the population, its costs and the problem in
// shared memory: no global round trip between generations, no grid barrier,
// one launch per solve.  A candidate is one thread: its state (n <= 8) and
// the model Delta = Ad - I live in registers and the horizon recursion needs
// no exchange.  The random streams are exactly the per-generation launches'
// (draw_tile / the init stream: same counters), so results match the other
// paths to rounding (the scoring order differs).  Reference: selection
// K/empc.py:185-188, breeding K/empc.py:195-204, scoring K/empc.py:85-119.
#include "empc_small.h"

namespace empc {

template <typename S>
struct SmallShared {
  const S *D, *W, *Q, *E0, *B, *Ug, *Rd, *R, *G, *C;
  const int *I1, *I2, *Seg;
};

template <typename S>
__host__ __device__ inline size_t small_smem_bytes(int n, int m, int T, int p, int N, int K) {
  const int pm = p * m, nc = N - K;
  const int NPV = n <= 4 ? 4 : 8;
  size_t b = 0;
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  b += al((size_t)NPV * NPV * sizeof(S));           // Delta
  b += al((size_t)NPV * m * sizeof(S));             // Bd
  b += al((size_t)3 * NPV * sizeof(S));             // w', q, e0
  b += al((size_t)(5 * m + m * m) * sizeof(S));     // ug, umin, umax, sig, rdiag, R
  b += al((size_t)T * (3 * sizeof(int) + sizeof(S)));  // schedule + segments
  b += al((size_t)(p * p + 2) * sizeof(S));         // W'W, cost of x0
  b += al((size_t)2 * N * pm * sizeof(S));          // populations
  b += al((size_t)2 * N * sizeof(S));               // costs
  b += al((size_t)(N > 64 ? N : 64) * 8);           // keys (argmin scratch at the end)
  b += al((size_t)nc * 2 * sizeof(int));            // parent ranks
  b += al((size_t)nc * pm);                         // crossover bits
  b += al((size_t)nc * pm * sizeof(S));             // mutation offsets
  b += al((size_t)stage_stride(n, m) * sizeof(double));   // problem staging block
  b += al((size_t)(n + m) * sizeof(double));              // x0, sigma
  return b + 64;
}

// full tracking cost of knots U (K/empc.py:85-119): knot-space input cost,
// drive = W (x) (U Bd') + w', recursion over the knot segments, diag-Q cost.
template <typename S, int NPV>
__device__ __forceinline__ S small_score(const S* __restrict__ U, const SmallShared<S>& sh, int m, int p, int T,
                                      int r_diag, long long* prof = nullptr) {
  long long t0 = prof ? clock64() : 0;
  // the model in registers (a reference parameter would force it to local memory)
  S Dr[NPV][NPV];
#pragma unroll
  for (int i = 0; i < NPV; ++i)
#pragma unroll
    for (int j = 0; j < NPV; ++j) Dr[i][j] = sh.D[i * NPV + j];
  S st = sh.G[p * p];
  // input cost z'(W'W (x) R) z, z = U - u_goal (K/empc.py:100-101)
  // (runtime-bounded loops stay rolled: unrolled remainders blew the kernel
  // up to ~18k instructions and the scorer ran out of the instruction cache)
#pragma unroll 1
  for (int l = 0; l < m; ++l) {
#pragma unroll 1
    for (int t = 0; t < p; ++t) {
      S gz = S(0);
#pragma unroll 1
      for (int b = 0; b < p; ++b) {
        S rz;
        if (r_diag) {
          rz = sh.Rd[l] * (U[b * m + l] - sh.Ug[l]);
        } else {
          rz = S(0);
          for (int l2 = 0; l2 < m; ++l2) rz = fma(sh.R[l * m + l2], U[b * m + l2] - sh.Ug[l2], rz);
        }
        gz = fma(sh.G[t * p + b], rz, gz);
      }
      st = fma(U[t * m + l] - sh.Ug[l], gz, st);
    }
  }
  S e[NPV], srow[NPV];
#pragma unroll
  for (int i = 0; i < NPV; ++i) {
    e[i] = sh.E0[i];
    srow[i] = S(0);
  }
  if (prof) { const long long t1 = clock64(); prof[0] += t1 - t0; t0 = t1; }
#pragma unroll 1
  for (int k0 = 0; k0 < T;) {
    const int k1 = sh.Seg[k0], i1 = sh.I1[k0], i2 = sh.I2[k0];
    S b1[NPV], db[NPV];
#pragma unroll
    for (int i = 0; i < NPV; ++i) {
      S u1 = sh.W[i], u2 = sh.W[i];
#pragma unroll 1
      for (int l = 0; l < m; ++l) {
        u1 = fma(sh.B[i * m + l], U[i1 * m + l], u1);
        u2 = fma(sh.B[i * m + l], U[i2 * m + l], u2);
      }
      b1[i] = u1;
      db[i] = u2 - u1;
    }
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      const S ck = sh.C[k];
      S en[NPV];
#pragma unroll
      for (int i = 0; i < NPV; ++i) {
        S ax = S(0);
#pragma unroll
        for (int j = 0; j < NPV; ++j) ax = fma(Dr[i][j], e[j], ax);
        en[i] = e[i] + fma(ck, db[i], ax + b1[i]);
      }
#pragma unroll
      for (int i = 0; i < NPV; ++i) {
        e[i] = en[i];
        srow[i] = fma(en[i], en[i], srow[i]);
      }
    }
    k0 = k1;
  }
#pragma unroll
  for (int i = 0; i < NPV; ++i) st = fma(sh.Q[i], srow[i], st);
  if (prof) prof[1] += clock64() - t0;
  return st;
}

template <typename S, int NPV>
__global__ void __launch_bounds__(512, 1) small_solve_kernel(const SmallArgs<S> A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using OT = typename std::conditional<sizeof(S) == 4, uint32_t, uint64_t>::type;
  const Dims& d = A.d;
  const int n = d.n, m = d.m, T = d.T, p = d.p, pm = d.pm, N = d.N, K = d.K, nc = N - K;
  const int inst = blockIdx.x;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const StageLayout& SL = A.SL;
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  unsigned char* ptr = smem_raw;
  S* sD = reinterpret_cast<S*>(ptr); ptr += al((size_t)NPV * NPV * sizeof(S));
  S* sB = reinterpret_cast<S*>(ptr); ptr += al((size_t)NPV * m * sizeof(S));
  S* sW = reinterpret_cast<S*>(ptr);
  S* sQ = sW + NPV;
  S* sE0 = sQ + NPV; ptr += al((size_t)3 * NPV * sizeof(S));
  S* sUg = reinterpret_cast<S*>(ptr);
  S* sUmin = sUg + m;
  S* sUmax = sUmin + m;
  S* sSig = sUmax + m;
  S* sRd = sSig + m;
  S* sR = sRd + m; ptr += al((size_t)(5 * m + m * m) * sizeof(S));
  int* sI1 = reinterpret_cast<int*>(ptr);
  int* sI2 = sI1 + T;
  int* sSeg = sI2 + T;
  S* sC = reinterpret_cast<S*>(sSeg + T); ptr += al((size_t)T * (3 * sizeof(int) + sizeof(S)));
  S* sG = reinterpret_cast<S*>(ptr); ptr += al((size_t)(p * p + 2) * sizeof(S));
  // two populations / cost vectors as plain pointers (an array of pointers
  // indexed by the generation parity would live in local memory and turn
  // every shared access into a generic one)
  S* const popA = reinterpret_cast<S*>(ptr);
  S* const popB = popA + (size_t)N * pm; ptr += al((size_t)2 * N * pm * sizeof(S));
  S* const costA = reinterpret_cast<S*>(ptr);
  S* const costB = costA + N; ptr += al((size_t)2 * N * sizeof(S));
  OT* keys = reinterpret_cast<OT*>(ptr); ptr += al((size_t)(N > 64 ? N : 64) * 8);
  int* src = reinterpret_cast<int*>(ptr); ptr += al((size_t)nc * 2 * sizeof(int));
  uint8_t* tbits = reinterpret_cast<uint8_t*>(ptr); ptr += al((size_t)nc * pm);
  S* off = reinterpret_cast<S*>(ptr); ptr += al((size_t)nc * pm * sizeof(S));
  double* const sP = reinterpret_cast<double*>(ptr); ptr += al((size_t)SL.stride * sizeof(double));
  double* const sX = reinterpret_cast<double*>(ptr);

  // ---- the instance's staging blocks into shared memory in one parallel
  // pass (they may live in mapped host memory), then the problem in error
  // coordinates, as the rollout kernel
  {
    const double* gp = A.prob + (size_t)inst * SL.stride;
    const double* gx = A.state + (size_t)inst * SL.sstride;
    for (int e = tid; e < SL.stride; e += nthr) sP[e] = gp[e];
    for (int e = tid; e < n + m; e += nthr) sX[e] = gx[e];
  }
  const RunParams rp = *A.run;
  __syncthreads();
  const double* __restrict__ P = sP;
  const double* __restrict__ X = sX;
  for (int e = tid; e < NPV * NPV; e += nthr) {
    const int i = e / NPV, j = e % NPV;
    sD[e] = (i < n && j < n) ? (S)(P[SL.ad + i * n + j] - (i == j ? 1.0 : 0.0)) : S(0);
  }
  for (int e = tid; e < NPV * m; e += nthr) sB[e] = e / m < n ? (S)P[SL.bd + (e / m) * m + e % m] : S(0);
  for (int i = tid; i < NPV; i += nthr) {
    double w = 0.0;
    if (i < n) {
      // w' = w + Delta x_goal (rows of W sum to one), in FP64
      w = P[SL.wd + i];
      for (int j = 0; j < n; ++j) w += (P[SL.ad + i * n + j] - (i == j ? 1.0 : 0.0)) * P[SL.xg + j];
    }
    sW[i] = (S)w;
    sQ[i] = i < n ? (S)P[SL.q + i * n + i] : S(0);
    sE0[i] = i < n ? (S)(X[SL.x0 + i] - P[SL.xg + i]) : S(0);
  }
  for (int l = tid; l < m; l += nthr) {
    sUg[l] = (S)P[SL.ug + l];
    sUmin[l] = (S)P[SL.umin + l];
    sUmax[l] = (S)P[SL.umax + l];
    sSig[l] = (S)X[SL.sig + l];
    sRd[l] = (S)P[SL.r + l * m + l];
  }
  for (int e = tid; e < m * m; e += nthr) sR[e] = (S)P[SL.r + e];
  for (int k = tid; k < T; k += nthr) {
    sI1[k] = A.idx1[k];
    sI2[k] = A.idx2[k];
    sSeg[k] = A.seg[k];
    sC[k] = A.cw[k];
  }
  for (int e = tid; e < p * p; e += nthr) sG[e] = A.G[e];
  if (tid == 0) {  // cost of x_0 (k = 0 state term), FP64
    double c0 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double ei = X[SL.x0 + i] - P[SL.xg + i];
      c0 += P[SL.q + i * n + i] * ei * ei;
    }
    sG[p * p] = (S)c0;
  }
  __syncthreads();
  const SmallShared<S> sh{sD, sW, sQ, sE0, sB, sUg, sRd, sR, sG, sC, sI1, sI2, sSeg};
  long long sprof[2] = {0, 0};
  const bool prof_on = A.dbg != nullptr && inst == 0 && tid == 0;
  auto score = [&](const S* U) -> S { return small_score<S, NPV>(U, sh, m, p, T, A.r_diag, prof_on ? sprof : nullptr); };

  const uint32_t key0 = (uint32_t)rp.seed, key1 = (uint32_t)(rp.seed >> 32);
  // ---- generation 0: init (Philox / injected) or the resident population (re-score)
  for (int e = tid; e < N * pm; e += nthr) {
    const int c = e / pm, g = e % pm;
    S v;
    if (A.mode == kInitInject) {
      v = A.inj_init[((size_t)inst * N + c) * pm + g];
    } else if (A.mode == kScore || A.mode == kSmallResident) {
      v = A.pop_in[((size_t)inst * N + c) * pm + g];
    } else {
      // the rollout kernel's init stream: counter (q, cand, instance, "INIT"),
      // genes 2q / 2q + 1 from words (x, y) / (z, w) (K/empc.py:170)
      const int q = g >> 1, l = g % m;
      const U4 r = philox4x32_10(U4{(uint32_t)q, (uint32_t)c, (uint32_t)inst, kInitTag}, key0, key1);
      const S lo = sUmin[l], hi = sUmax[l];
      const S u = (g & 1) ? uniform01<S>(r.z, r.w) : uniform01<S>(r.x, r.y);
      v = lo + (hi - lo) * u;
      v = v > hi ? hi : v;
    }
    popA[e] = v;
  }
  __syncthreads();
  for (int c = tid; c < N; c += nthr)
    costA[c] = A.mode == kSmallResident ? A.cost_in[(size_t)inst * N + c] : score(popA + (size_t)c * pm);
  __syncthreads();
  int sub = 1;
  while (sub < 32 && N * sub * 2 <= nthr) sub <<= 1;
  int cur = 0;
  // phase timers (EMPC_PHASES): cycles of thread 0 per phase, summed over generations
  const bool timed = A.dbg != nullptr && inst == 0 && tid == 0;
  long long ph[5] = {0, 0, 0, 0, 0}, tp = timed ? clock64() : 0;
  auto mark = [&](int i) {
    if (timed) {
      const long long t = clock64();
      ph[i] += t - tp;
      tp = t;
    }
  };
  for (int g = 0; g < A.evolves; ++g) {
    const int nx = cur ^ 1;
    S* const pc = cur ? popB : popA;
    S* const pn = cur ? popA : popB;
    S* const cc = cur ? costB : costA;
    S* const cn = cur ? costA : costB;
    // ---- stable selection (K/empc.py:185-188): rank of (ord(cost), row)
    // (FP32: one 64-bit key ord << 32 | row, a single unsigned compare)
    unsigned long long* const kk = reinterpret_cast<unsigned long long*>(keys);
    for (int c = tid; c < N; c += nthr) {
      if constexpr (sizeof(S) == 4) kk[c] = ((unsigned long long)ord_key(cc[c]) << 32) | (unsigned)c;
      else keys[c] = ord_key(cc[c]);
    }
    __syncthreads();
    mark(0);
    // `sub` lanes (a power of two <= 32) count the rank of one candidate
    for (int base = 0; base < N * sub; base += nthr) {
      const int t = base + tid, c = t / sub, part = t & (sub - 1);
      const bool valid = c < N;
      int r = 0;
      if (valid) {
        if constexpr (sizeof(S) == 4) {
          const unsigned long long kc = kk[c];
          for (int j = part; j < N; j += sub) r += kk[j] < kc ? 1 : 0;
        } else {
          const OT kc = keys[c];
          for (int j = part; j < N; j += sub) {
            const OT kj = keys[j];
            r += (kj < kc || (kj == kc && j < c)) ? 1 : 0;
          }
        }
      }
      for (int o = 1; o < sub; o <<= 1) r += __shfl_xor_sync(0xFFFFFFFFu, r, o);
      if (valid && r < K) {
        for (int q = part; q < pm; q += sub) pn[(size_t)r * pm + q] = pc[(size_t)c * pm + q];
        if (part == 0) cn[r] = cc[c];
      }
    }
    mark(1);
    // ---- breeding (K/empc.py:195-204): the per-generation launches' draws
    const uint32_t gen = (uint32_t)(rp.gen0 + g);
    if (nc > 0) {
      if (A.inj_parents != nullptr) {
        const int* pp = A.inj_parents + ((size_t)g * gridDim.x + inst) * nc * 2;
        for (int e = tid; e < 2 * nc; e += nthr) src[e] = pp[e];
      } else {
        draw_tile<S>(rp, gen, K, pm, m, inst, 0, nc, nc, tid, nthr, src, tbits, off, sSig);
      }
    }
    __syncthreads();
    mark(2);
    for (int e = tid; e < nc * pm; e += nthr) {
      const int c = e / pm, q = e % pm, l = q % m;
      S v;
      if (A.inj_parents != nullptr) {
        const size_t gi = (((size_t)g * gridDim.x + inst) * nc + c) * pm + q;
        const bool take = A.inj_take[gi] != 0, mut = A.inj_mut[gi] != 0;
        const S par = pn[(size_t)src[2 * c + (take ? 1 : 0)] * pm + q];
        const double nz = mut ? A.inj_noise[gi] * X[SL.sig + l] : 0.0;
        v = (S)((double)par + nz);
      } else {
        const S par = pn[(size_t)src[2 * c + (tbits[e] ? 1 : 0)] * pm + q];
        v = par + off[q * nc + c];
      }
      const S lo = sUmin[l], hi = sUmax[l];
      pn[(size_t)(K + c) * pm + q] = v < lo ? lo : (v > hi ? hi : v);
    }
    __syncthreads();
    mark(3);
    for (int c = tid; c < nc; c += nthr) cn[K + c] = score(pn + (size_t)(K + c) * pm);
    __syncthreads();
    mark(4);
    cur = nx;
  }
  if (timed) {
    for (int i = 0; i < 5; ++i) A.dbg[i] = (unsigned long long)ph[i];
    A.dbg[5] = (unsigned long long)sprof[0];
    A.dbg[6] = (unsigned long long)sprof[1];
  }
  // ---- results: population to HBM (the slot), argmin (first NaN, else first minimum)
  S* const pf = cur ? popB : popA;
  S* const cf = cur ? costB : costA;
  for (int e = tid; e < N * pm; e += nthr) A.pop_io[(size_t)inst * N * pm + e] = pf[e];
  for (int c = tid; c < N; c += nthr) A.cost_io[(size_t)inst * N + c] = cf[c];
  uint64_t bo = ~0ull;
  int bi = 0x7FFFFFFF;
  for (int c = tid; c < N; c += nthr) {
    const S v = cf[c];
    uint64_t o;
    if constexpr (sizeof(S) == 4) o = (v != v) ? 0ull : (uint64_t)ord32((float)v);
    else o = (v != v) ? 0ull : ord64((double)v);
    if (o < bo || (o == bo && c < bi)) { bo = o; bi = c; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t o2 = __shfl_down_sync(0xFFFFFFFFu, bo, o);
    const int i2 = __shfl_down_sync(0xFFFFFFFFu, bi, o);
    if (o2 < bo || (o2 == bo && i2 < bi)) { bo = o2; bi = i2; }
  }
  uint64_t* wo = reinterpret_cast<uint64_t*>(keys);  // keys are free now
  int* wi = reinterpret_cast<int*>(wo + 32);
  if ((tid & 31) == 0) { wo[tid >> 5] = bo; wi[tid >> 5] = bi; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (nthr + 31) / 32; ++w)
      if (wo[w] < wo[0] || (wo[w] == wo[0] && wi[w] < wi[0])) { wo[0] = wo[w]; wi[0] = wi[w]; }
  }
  __syncthreads();
  const int best = wi[0];
  double* o = A.out + (size_t)inst * (m + pm + 2);
  for (int q = tid; q < pm; q += nthr) {
    o[m + q] = (double)pf[(size_t)best * pm + q];
    if (q < m) o[q] = (double)pf[(size_t)best * pm + q];  // u = first knot (K/empc.py:236)
  }
  if (tid == 0) {
    o[m + pm] = (double)cf[best];
    o[m + pm + 1] = (double)best;
  }
}

template <typename S>
size_t small_smem(int n, int m, int T, int p, int N, int K) {
  return small_smem_bytes<S>(n, m, T, p, N, K);
}

template <typename S>
SmallKernel<S> small_kernel(int n) {
  if (n <= 4) return &small_solve_kernel<S, 4>;
  if (n <= 8) return &small_solve_kernel<S, 8>;
  return nullptr;
}

template size_t small_smem<float>(int, int, int, int, int, int);
template size_t small_smem<double>(int, int, int, int, int, int);
template SmallKernel<float> small_kernel<float>(int);
template SmallKernel<double> small_kernel<double>(int);

}  // namespace empc
