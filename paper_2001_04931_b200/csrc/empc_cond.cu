// Condensed scorer kernels: device build of the knot-space
// quadratic once per solve, and the breed + quadratic-form scoring kernel
// that replaces the rollout when EmpcSettings.scorer == "condensed".
// See empc_cond.h for the algebra; every kernel is FP64 arithmetic.
#include "empc_cond.h"

namespace empc {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
  return v;
}

size_t cond_prep_smem(int n, int cb, int dense) {
  const size_t A = (size_t)n * (n + 1) * (dense ? 2 : 1);
  const size_t sens = A + (size_t)3 * n * cb + cb;
  const size_t traj = A + (size_t)7 * n;
  return sizeof(double) * (sens > traj ? sens : traj);
}

// ---------------------------------------------------------------------------
// prep: CTAs [0, chunks) run the sensitivity recursion for `cb` knot columns
// each (K/condense.py:133-139: S_0 = W[0] (x) Bd, S_k = Ad S_{k-1} + W[k] (x) Bd);
// the last CTA of each instance rolls out u = u_goal for e_ref, Q e_ref and
// J_ref.  One dot product per `ksp` adjacent lanes, folded by shuffles.
__global__ void __launch_bounds__(1024) cond_prep_kernel(CondBuild b) {
  extern __shared__ __align__(16) double sm[];
  const int n = b.n, m = b.m, T = b.T, p = b.p, pm = b.pm;
  const int i = blockIdx.y, inst = b.inst0 + i;
  const double* __restrict__ P = b.prob + (size_t)inst * b.SL.stride;
  const double* __restrict__ X = b.state + (size_t)inst * b.SL.sstride;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nA = n + 1;
  double* Ad = sm;  // [n][n + 1]
  for (int e = tid; e < n * n; e += nthr) Ad[(e / n) * nA + e % n] = P[b.SL.ad + e];

  double* Qs = Ad + (size_t)n * nA;  // dense Q only
  if (b.dense)
    for (int e = tid; e < n * n; e += nthr) Qs[(e / n) * nA + e % n] = P[b.SL.q + e];
  const int ksp = b.ksp;
  const int o = tid / ksp, part = tid % ksp;
  const bool rowok = o < n;
  const int rr = rowok ? o : 0;

  if (blockIdx.x == gridDim.x - 1) {
    // ---- u_goal trajectory x_{k+1} = Ad x_k + Bd u_goal + wd: e_ref, Q e_ref
    // and J_ref.  Thread group `o` owns row o; one barrier per step.
    double* xs = (b.dense ? Qs + (size_t)n * nA : Qs);  // [2][n]
    double* bu = xs + 2 * n;
    double* xg = bu + n;
    double* qd = xg + n;
    double* t = qd + n;
    for (int r = tid; r < n; r += nthr) {
      double acc = P[b.SL.wd + r];
      for (int l = 0; l < m; ++l) acc = fma(P[b.SL.bd + r * m + l], P[b.SL.ug + l], acc);
      bu[r] = acc;
      xs[r] = X[b.SL.x0 + r];
      xg[r] = P[b.SL.xg + r];
      qd[r] = P[b.SL.q + r * n + r];
    }
    __syncthreads();
    double* E = b.E + (size_t)i * ((size_t)T * n + 1);
    double jr = 0.0;  // row o's share of J_ref, accumulated in step order
    int cur = 0;
    for (int k = 0; k <= T; ++k) {
      const double* x = xs + cur * n;
      double qe;
      if (b.dense) {
        qe = 0.0;
        for (int j = part; j < n; j += ksp) qe = fma(Qs[rr * nA + j], x[j] - xg[j], qe);
        for (int off = ksp >> 1; off > 0; off >>= 1) qe += __shfl_xor_sync(0xFFFFFFFFu, qe, off);
      } else {
        qe = qd[rr] * (x[rr] - xg[rr]);
      }
      if (rowok && part == 0) {
        jr = fma(x[rr] - xg[rr], qe, jr);
        if (k > 0) E[(size_t)(k - 1) * n + o] = qe;
      }
      if (k == T) break;
      double acc = 0.0;
      for (int j = part; j < n; j += ksp) acc = fma(Ad[rr * nA + j], x[j], acc);
      for (int off = ksp >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
      if (rowok && part == 0) xs[(cur ^ 1) * n + o] = acc + bu[o];
      cur ^= 1;
      __syncthreads();
    }
    if (rowok && part == 0) t[o] = jr;
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      for (int r = lane; r < n; r += 32) s += t[r];
      s = warp_sum(s);
      if (lane == 0) E[(size_t)T * n] = s;
    }
    return;
  }

  // ---- sensitivity columns [c0, c0 + cb)
  const int cb = b.cb;
  const int c0 = blockIdx.x * cb;
  double* Sp = b.dense ? Qs + (size_t)n * nA : Qs;  // [2][n][cb]
  double* Bc = Sp + (size_t)2 * n * cb;            // [n][cb]
  int* lcol = reinterpret_cast<int*>(Bc + (size_t)n * cb);
  for (int e = tid; e < n * cb; e += nthr) {
    const int r = e / cb, c = e % cb, col = c0 + c;
    Bc[e] = col < pm ? P[b.SL.bd + r * m + col % m] : 0.0;
  }
  for (int c = tid; c < cb; c += nthr) lcol[c] = min(c0 + c, pm - 1) / m;
  __syncthreads();
  const int r = o / cb, c = o % cb;
  const bool valid = r < n && c0 + c < pm;
  const int sr = valid ? r : 0, cc = valid ? c : 0;
  double* Sg = b.S + (size_t)i * T * n * pm;
  double* QSg = b.dense ? b.QS + (size_t)i * T * n * pm : nullptr;
  int cur = 0;
  for (int k = 0; k < T; ++k) {
    double acc = 0.0;
    if (k > 0)
      for (int j = part; j < n; j += ksp) acc = fma(Ad[sr * nA + j], Sp[(cur * n + j) * cb + cc], acc);
    for (int off = ksp >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
    const double v = fma(b.W[(size_t)k * p + lcol[cc]], Bc[sr * cb + cc], acc);
    const int nxt = cur ^ 1;
    if (valid && part == 0) {
      Sp[(nxt * n + r) * cb + c] = v;
      Sg[((size_t)k * n + r) * pm + c0 + c] = v;
    }
    __syncthreads();
    if (b.dense) {
      double q = 0.0;
      for (int j = part; j < n; j += ksp) q = fma(Qs[sr * nA + j], Sp[(nxt * n + j) * cb + cc], q);
      for (int off = ksp >> 1; off > 0; off >>= 1) q += __shfl_xor_sync(0xFFFFFFFFu, q, off);
      if (valid && part == 0) QSg[((size_t)k * n + r) * pm + c0 + c] = q;
    }
    cur = nxt;
  }
}

// ---------------------------------------------------------------------------
// Gram: partial [P | g] over a split of the T*n sensitivity rows,
//   P_ab = sum_R S[R][a] (Q S)[R][b],  g_a = sum_R S[R][a] (Q e_ref)[R]
// (K/condense.py:245-249 with the (I kron Q) product of K/condense.py:254-258).
// 32 x 32 output tiles of the upper triangle, 2 x 2 outputs per thread.
__global__ void __launch_bounds__(256) cond_gram_kernel(CondBuild b) {
  __shared__ double As[kCondTile][kCondTile + 1];
  __shared__ double Bs[kCondTile][kCondTile + 1];
  const int n = b.n, T = b.T, pm = b.pm;
  const int i = blockIdx.z, inst = b.inst0 + i;
  const double* __restrict__ P = b.prob + (size_t)inst * b.SL.stride;
  // upper-triangle tile (ta <= tb) of the pm x (pm + 1) output
  const int ntc = (pm + 1 + kCondTile - 1) / kCondTile;
  int t = blockIdx.x, ta = 0;
  while (t >= ntc - ta) { t -= ntc - ta; ++ta; }
  const int tb = ta + t;
  const int K = T * n;
  const int per = (K + b.splits - 1) / b.splits;
  const int R0 = blockIdx.y * per, R1 = min(K, R0 + per);
  const double* Sg = b.S + (size_t)i * K * pm;
  const double* QSg = b.dense ? b.QS + (size_t)i * K * pm : nullptr;
  const double* Eg = b.E + (size_t)i * ((size_t)K + 1);
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int Rc = R0; Rc < R1; Rc += kCondTile) {
    for (int e = tid; e < kCondTile * kCondTile; e += 256) {
      const int rr = e / kCondTile, cc = e % kCondTile;
      const int R = Rc + rr;
      const int a = ta * kCondTile + cc, bcol = tb * kCondTile + cc;
      double va = 0.0, vb = 0.0;
      if (R < R1) {
        if (a < pm) va = Sg[(size_t)R * pm + a];
        if (bcol < pm) {
          if (QSg) {
            vb = QSg[(size_t)R * pm + bcol];
          } else {
            const int r = R % n;
            vb = P[b.SL.q + r * n + r] * Sg[(size_t)R * pm + bcol];
          }
        } else if (bcol == pm) {
          vb = Eg[R];
        }
      }
      As[rr][cc] = va;
      Bs[rr][cc] = vb;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < kCondTile; ++rr) {
      const double a0 = As[rr][2 * ty], a1 = As[rr][2 * ty + 1];
      const double b0 = Bs[rr][2 * tx], b1 = Bs[rr][2 * tx + 1];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
  double* out = b.part + ((size_t)i * b.splits + blockIdx.y) * pm * (pm + 1);
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int a = ta * kCondTile + 2 * ty + u, bcol = tb * kCondTile + 2 * tx + v;
      if (a < pm && bcol <= pm) out[(size_t)a * (pm + 1) + bcol] = acc[u][v];
    }
}

// ---------------------------------------------------------------------------
// finish: reduce the split partials in a fixed order, mirror the upper
// triangle (exactly symmetric P, like K/condense.py:247) and add the knot
// input cost (W'W) (x) R (K/condense.py:197-202).  One thread per output.
__global__ void __launch_bounds__(256) cond_finish_kernel(CondBuild b) {
  const int m = b.m, p = b.p, pm = b.pm, T = b.T, n = b.n;
  const int i = blockIdx.y, inst = b.inst0 + i;
  const double* __restrict__ P = b.prob + (size_t)inst * b.SL.stride;
  const CondLayout L = cond_layout(pm);
  double* out = b.cond + (size_t)inst * L.stride;
  const double* part = b.part + (size_t)i * b.splits * pm * (pm + 1);
  const size_t ps = (size_t)pm * (pm + 1);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e > pm * pm + pm) return;
  if (e == pm * pm + pm) {
    out[L.jref] = b.E[(size_t)i * ((size_t)T * n + 1) + (size_t)T * n];
    return;
  }
  // element (lo, hi) of the upper triangle, or column pm (g)
  int lo, hi;
  if (e < pm * pm) {
    const int a = e / pm, c = e - (e / pm) * pm;
    lo = min(a, c);
    hi = max(a, c);
  } else {
    lo = e - pm * pm;
    hi = pm;
  }
  const double* src = part + (size_t)lo * (pm + 1) + hi;
  double s = 0.0;
  int sp = 0;
  for (; sp + 8 <= b.splits; sp += 8) {  // 8 loads in flight, summed in split order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = src[(size_t)(sp + u) * ps];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; sp < b.splits; ++sp) s += src[(size_t)sp * ps];
  if (e < pm * pm) {
    out[L.P + e] = fma(b.G[(lo / m) * p + hi / m], P[b.SL.r + (lo % m) * m + hi % m], s);
  } else {
    out[L.g + lo] = s;
    out[L.ref + lo] = P[b.SL.ug + lo % m];
  }
}

// ---------------------------------------------------------------------------
// scoring: the K5 prologue (breed_tile) followed by the quadratic form in
// place of the rollout.  Thread (cg, slice) owns candidates 2cg, 2cg+1 and
// the row chunks slice, slice + nslices, ... of P (4 rows each): per pair of
// columns one 16-byte broadcast of P per row and one load of the two
// candidates' knots feed 16 DFMAs.  Chunk partials are summed in chunk
// order, so a candidate's cost has the same bits for every tiling (batched,
// sharded or single runs agree exactly).
template <typename S, bool PSM>
__global__ void __launch_bounds__(512) cond_score_kernel(const RolloutArgs<S> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int RB = kCondRB, CC = kCondCC;
  const Dims& d = a.d;
  const int m = d.m, pm = d.pm;
  const int inst = blockIdx.y;
  const int tile0 = blockIdx.x * a.tile;
  const int cnt = min(a.tile, a.nc - tile0);
  const int tileP = a.tileP;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const CondSmem cs = cond_smem<S>(pm, m, tileP, nthr, PSM);
  const int tPS = cs.tPS, pmS = cs.pmS, PST = pmS + 2;
  unsigned char* ptr = smem_raw;
  S* UsT = reinterpret_cast<S*>(ptr); ptr += cs.us;
  int* src = reinterpret_cast<int*>(ptr); ptr += cs.src;
  uint8_t* tbits = reinterpret_cast<uint8_t*>(ptr); ptr += cs.bits;
  S* cumin = reinterpret_cast<S*>(ptr);
  S* cumax = cumin + m;
  S* csig = cumax + m; ptr += cs.vec;
  double* Ps = reinterpret_cast<double*>(ptr); ptr += cs.ps;
  double* gv = reinterpret_cast<double*>(ptr);
  double* rv = gv + pmS; ptr += cs.gv;
  double* Zt = reinterpret_cast<double*>(ptr);       // [pmS][tPS]: z - ref
  double* red = reinterpret_cast<double*>(smem_raw);  // [pmS / RB][tPS], overlays UsT after Zt is built
  const double* __restrict__ Pp = a.prob + (size_t)inst * a.SL.stride;
  const double* __restrict__ X = a.state + (size_t)inst * a.SL.sstride;
  const size_t pop_base = (size_t)inst * a.rows;
  const bool breed = (a.mode == kBreedPhilox || a.mode == kBreedInject);

  EMPC_MARK(0)
  if (cnt > 0) {
    for (int l = tid; l < m; l += nthr) {
      cumin[l] = (S)Pp[a.SL.umin + l];
      cumax[l] = (S)Pp[a.SL.umax + l];
      csig[l] = (S)X[a.SL.sig + l];
    }
    for (int e = pm * tPS + tid; e < pmS * tPS; e += nthr) UsT[e] = S(0);
  }
  __syncthreads();
  if (!breed_tile<S>(a, inst, tile0, cnt, tileP, tPS, UsT, src, tbits, cumin, cumax, csig, pop_base)) return;
  // the condensed model was written by the build kernels (visible after the
  // PDL wait inside breed_tile)
  const CondLayout L = cond_layout(pm);
  const double* __restrict__ C = a.cond + (size_t)inst * a.cstride;
  if constexpr (PSM) {
    // P rows -> shared memory with asynchronous copies (all in flight at once)
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(Ps);
    if ((pm & 1) == 0) {
      const int hp = pm >> 1;
      for (int e = tid; e < pm * hp; e += nthr) {
        const int r = e / hp, q = e - (e / hp) * hp;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + (uint32_t)((r * PST + 2 * q) * 8)),
                     "l"(C + L.P + (size_t)r * pm + 2 * q));
      }
    } else {
      for (int e = tid; e < pm * pm; e += nthr) {
        const int r = e / pm, q = e - (e / pm) * pm;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + (uint32_t)((r * PST + q) * 8)),
                     "l"(C + L.P + (size_t)r * pm + q));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    // zero padding: columns [pm, PST) of the real rows, rows [pm, pmS)
    for (int e = tid; e < pm * (PST - pm); e += nthr) {
      const int r = e / (PST - pm), q = e - (e / (PST - pm)) * (PST - pm);
      Ps[r * PST + pm + q] = 0.0;
    }
    for (int e = pm * PST + tid; e < pmS * PST; e += nthr) Ps[e] = 0.0;
  }
  for (int r = tid; r < pmS; r += nthr) {
    gv[r] = r < pm ? C[L.g + r] : 0.0;
    rv[r] = r < pm ? C[L.ref + r] : 0.0;
  }
  __syncthreads();  // UsT (breed_tile), rv
  for (int e = tid; e < pmS * tPS; e += nthr) {
    const int j = e / tPS;
    Zt[e] = (double)UsT[e] - rv[j];
  }
  if constexpr (PSM) asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();  // Zt, Ps
  pdl_trigger();
  EMPC_MARK(3)

  const int ncg = (tileP + CC - 1) / CC;
  const int cg = tid % ncg, sl = tid / ncg;
  const int c0 = cg * CC;
  const int nchunk = pmS / RB;
  auto zval = [&](int j, double (&z)[CC]) {
    const double2 t = *reinterpret_cast<const double2*>(Zt + j * tPS + c0);
    z[0] = t.x;
    z[1] = t.y;
  };
  if (sl < cs.nslices) {
    for (int ch = sl; ch < nchunk; ch += cs.nslices) {
      const int i0 = ch * RB;
      double y[RB][CC] = {};
#pragma unroll 2
      for (int j = 0; j < pmS; j += 2) {
        double z0[CC], z1[CC];
        zval(j, z0);
        zval(j + 1, z1);
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          double2 pp;
          if constexpr (PSM) {
            pp = *reinterpret_cast<const double2*>(Ps + (i0 + r) * PST + j);
          } else {
            const int row = i0 + r;
            pp.x = (row < pm && j < pm) ? __ldg(C + L.P + (size_t)row * pm + j) : 0.0;
            pp.y = (row < pm && j + 1 < pm) ? __ldg(C + L.P + (size_t)row * pm + j + 1) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < CC; ++q) {
            y[r][q] = fma(pp.x, z0[q], y[r][q]);
            y[r][q] = fma(pp.y, z1[q], y[r][q]);
          }
        }
      }
      double partc[CC] = {};
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double zi[CC];
        zval(i0 + r, zi);
        const double g2 = 2.0 * gv[i0 + r];
#pragma unroll
        for (int q = 0; q < CC; ++q) partc[q] = fma(zi[q], y[r][q] + g2, partc[q]);
      }
#pragma unroll
      for (int q = 0; q < CC; ++q) red[ch * tPS + c0 + q] = partc[q];
    }
  }
  __syncthreads();
  EMPC_MARK(5)
  using OT = typename std::conditional<sizeof(S) == 4, uint32_t, uint64_t>::type;
  OT tau = OT(0);
  const bool qual = breed && a.qcount != nullptr;
  if (qual) tau = ord_key(a.cost_in[pop_base + a.elite_idx[(size_t)inst * d.K + d.K - 1]]);
  const double jref = C[L.jref];
  for (int c = tid; c < cnt; c += nthr) {
    double s = jref;
    for (int q = 0; q < nchunk; ++q) s += red[q * tPS + c];  // fixed order: same bits for any tiling
    const S cost = (S)s;
    const int row = a.row0 + tile0 + c;
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
  EMPC_MARK(6)
}

template <typename S>
CondKernels<S> cond_kernels() {
  CondKernels<S> k;
  k.prep = cond_prep_kernel;
  k.gram = cond_gram_kernel;
  k.finish = cond_finish_kernel;
  k.score_smem = cond_score_kernel<S, true>;
  k.score_glob = cond_score_kernel<S, false>;
  return k;
}
template CondKernels<float> cond_kernels<float>();
template CondKernels<double> cond_kernels<double>();

}  // namespace empc
