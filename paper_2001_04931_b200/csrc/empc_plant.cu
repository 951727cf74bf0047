// Batched plant linearization + exact discretization on the device
// (the step before the EMPC path in every closed-loop
// period, K/closedloop.py:103-104).
//
//   linearize  (K/dynamics.py:241-262): central differences with step eps of
//              the plant ODE in x and u, w = f(x0,u0) - A x0 - B u0;
//   discretize (K/dynamics.py:265-290): exp([[A B w],[0 0 0]] dt) ("exact",
//              zero-order hold) or I + A dt, B dt, w dt ("euler").
//
// Plants: the torque pendulum (K/dynamics.py:33-75) and the planar N-link
// chain with tip masses (K/dynamics.py:90-199).  One CTA per instance.
// Every ODE evaluation is one warp: the inertia matrix in absolute link
// angles is assembled in shared memory, factored by a warp Cholesky and
// solved; the 2(n+m)+1 evaluations of the central differences are spread
// over the CTA's warps.  The matrix exponential is a Taylor series on
// X = M dt / 2^s (||X||_1 <= 1/2, 18 terms: truncation < 1e-19 relative)
// followed by s squarings, with matrix products over the whole CTA.  FP64
// throughout.  Work per 24-link instance: ~150 ODE evaluations of O(L^3)
// plus ~20 products of a 73 x 73 matrix.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/empc_b200.h"

namespace plantk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLinks = 64;

struct PlantArgs {
  int kind, links, n, m, count, method;
  double eps, dt;
  const double* mass;    // [links] (pendulum: [1])
  const double* length;  // [links]
  double damping, gravity;
  const double* x;  // [count][n]
  const double* u;  // [count][m]
  double* Ad;       // [count][n][n]
  double* Bd;       // [count][n][m]
  double* wd;       // [count][n]
  double* work;     // global matrix workspace when the exponential does not fit in smem
  int ws_smem;      // 1: exponential buffers in shared memory
};

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// f(x, u) of the plant for one warp; writes n values to out.  scratch: per
// warp L*L + 6L doubles.
__device__ void plant_ode(const PlantArgs& a, const double* x, const double* u, double* out, double* scratch,
                          const double* carried) {
  const int lane = threadIdx.x & 31;
  if (a.kind == EMPC_PLANT_PENDULUM) {
    if (lane == 0) {
      const double m = a.mass[0], l = a.length[0];
      const double q = x[0], qd = x[1];
      out[0] = qd;
      out[1] = (u[0] - a.damping * qd - m * a.gravity * l * sin(q)) / (m * l * l);
    }
    __syncwarp();
    return;
  }
  const int L = a.links;
  double* M = scratch;          // [L][L]
  double* th = M + L * L;       // absolute angles
  double* thd = th + L;         // absolute rates
  double* rhs = thd + L;        // generalized force -> solution
  double* fv = rhs + L;
  if (lane == 0) {
    double s = 0.0, sd = 0.0;
    for (int j = 0; j < L; ++j) {
      s += x[j];
      sd += x[L + j];
      th[j] = s;
      thd[j] = sd;
    }
  }
  for (int j = lane; j < L; j += 32) fv[j] = u[j] - a.damping * x[L + j];
  __syncwarp();
  // M_th[j][k] = G[j][k] l_j l_k cos(th_j - th_k), G[j][k] = carried[max(j,k)]
  for (int e = lane; e < L * L; e += 32) {
    const int j = e / L, k = e - (e / L) * L;
    const double g = carried[j > k ? j : k] * a.length[j] * a.length[k];
    M[e] = g * cos(th[j] - th[k]);
  }
  for (int j = lane; j < L; j += 32) {
    double cor = 0.0;
    for (int k = 0; k < L; ++k) {
      const double g = carried[j > k ? j : k] * a.length[j] * a.length[k];
      cor += g * sin(th[j] - th[k]) * (thd[k] * thd[k]);
    }
    const double grav = a.gravity * carried[j] * a.length[j] * cos(th[j]);
    const double y = fv[j] - (j + 1 < L ? fv[j + 1] : 0.0);
    rhs[j] = y - cor - grav;
  }
  __syncwarp();
  // Cholesky M = C C' (lower, in place), column by column
  for (int c = 0; c < L; ++c) {
    double d = 0.0;
    for (int k = lane; k < c; k += 32) d = fma(M[c * L + k], M[c * L + k], d);
    d = wsum(d);
    const double piv = sqrt(M[c * L + c] - d);
    __syncwarp();
    for (int i = c + 1 + lane; i < L; i += 32) {
      double s = M[i * L + c];
      for (int k = 0; k < c; ++k) s = fma(-M[i * L + k], M[c * L + k], s);
      M[i * L + c] = s / piv;
    }
    if (lane == 0) M[c * L + c] = piv;
    __syncwarp();
  }
  // forward then backward substitution (lane 0; L <= 64)
  if (lane == 0) {
    for (int i = 0; i < L; ++i) {
      double s = rhs[i];
      for (int k = 0; k < i; ++k) s -= M[i * L + k] * rhs[k];
      rhs[i] = s / M[i * L + i];
    }
    for (int i = L - 1; i >= 0; --i) {
      double s = rhs[i];
      for (int k = i + 1; k < L; ++k) s -= M[k * L + i] * rhs[k];
      rhs[i] = s / M[i * L + i];
    }
    // joint accelerations are differences of the absolute ones
    for (int j = 0; j < L; ++j) {
      out[j] = x[L + j];
      out[L + j] = rhs[j] - (j > 0 ? rhs[j - 1] : 0.0);
    }
  }
  __syncwarp();
}

// C = A B for N x N row-major matrices with row stride ld (whole CTA)
__device__ void matmul(const double* A, const double* B, double* C, int N, int ld) {
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
    const int i = e / N, j = e - (e / N) * N;
    double s = 0.0;
    for (int k = 0; k < N; ++k) s = fma(A[i * ld + k], B[k * ld + j], s);
    C[i * ld + j] = s;
  }
  __syncthreads();
}

// shared layout of plant_kernel (doubles): f0 [n] | X [N*N] (ws_smem) | per-warp
// work [kWarps][warp_doubles], overlaid by T1, T2, Sm [3*N*N] after the
// Jacobians (ws_smem)
__host__ __device__ inline int plant_scratch(int kind, int L) { return kind == EMPC_PLANT_NLINK ? L * L + 6 * L : 8; }
__host__ __device__ inline size_t plant_warp_doubles(int kind, int L, int n, int m) {
  return (size_t)plant_scratch(kind, L) + 2 * n + n + m;
}
__host__ __device__ inline size_t plant_smem_doubles(int kind, int L, int n, int m, bool ws_smem) {
  const size_t N = (size_t)(n + m + 1);
  const size_t work = (size_t)kWarps * plant_warp_doubles(kind, L, n, m);
  return (size_t)n + (ws_smem ? N * N + (work > 3 * N * N ? work : 3 * N * N) : work);
}

__global__ void __launch_bounds__(kThreads) plant_kernel(PlantArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double carried[kMaxLinks];
  __shared__ double red[kWarps];
  const int inst = blockIdx.x;
  const int n = a.n, m = a.m, L = a.links;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = n + m + 1;
  const int scr = plant_scratch(a.kind, L);
  double* f0 = sm;
  double* X = a.ws_smem ? f0 + n : a.work + (size_t)inst * 4 * N * N;
  double* work = a.ws_smem ? X + (size_t)N * N : f0 + n;
  double* wbuf = work + (size_t)warp * plant_warp_doubles(a.kind, L, n, m);
  double* scratch = wbuf;
  double* fp = scratch + scr;
  double* fm = fp + n;
  double* v = fm + n;  // [n + m] evaluation point
  const double* x0 = a.x + (size_t)inst * n;
  const double* u0 = a.u + (size_t)inst * m;
  if (a.kind == EMPC_PLANT_NLINK && tid == 0) {
    double c = 0.0;
    for (int j = L - 1; j >= 0; --j) {
      c += a.mass[j];
      carried[j] = c;  // mass at or beyond link j
    }
  }
  for (int e = tid; e < N * N; e += blockDim.x) X[e] = 0.0;
  __syncthreads();
  // ---- central differences (K/dynamics.py:253-261): warp per coordinate,
  // column j of [A B] = (f(v + eps e_j) - f(v - eps e_j)) / (2 eps)
  const double h2 = 2.0 * a.eps;
  for (int j = warp; j <= n + m; j += kWarps) {
    for (int i = lane; i < n + m; i += 32) v[i] = i < n ? x0[i] : u0[i - n];
    __syncwarp();
    if (j == n + m) {  // the centre f(x0, u0)
      plant_ode(a, v, v + n, f0, scratch, carried);
      continue;
    }
    if (lane == 0) v[j] += a.eps;
    __syncwarp();
    plant_ode(a, v, v + n, fp, scratch, carried);
    for (int i = lane; i < n + m; i += 32) v[i] = i < n ? x0[i] : u0[i - n];
    __syncwarp();
    if (lane == 0) v[j] -= a.eps;
    __syncwarp();
    plant_ode(a, v, v + n, fm, scratch, carried);
    for (int i = lane; i < n; i += 32) X[i * N + j] = (fp[i] - fm[i]) / h2;
    __syncwarp();
  }
  __syncthreads();
  const bool exact = a.method == EMPC_DISCRETIZE_EXACT;
  double* T1 = a.ws_smem ? work : X + (size_t)N * N;
  double* T2 = T1 + (size_t)N * N;
  double* Sm = T2 + (size_t)N * N;
  // w = f(x0,u0) - A x0 - B u0 (K/dynamics.py:261)
  for (int i = tid; i < n; i += blockDim.x) {
    double ax = 0.0, bu = 0.0;
    for (int j = 0; j < n; ++j) ax = fma(X[i * N + j], x0[j], ax);
    for (int l = 0; l < m; ++l) bu = fma(X[i * N + n + l], u0[l], bu);
    X[i * N + n + m] = f0[i] - ax - bu;
  }
  __syncthreads();
  double* Ad = a.Ad + (size_t)inst * n * n;
  double* Bd = a.Bd + (size_t)inst * n * m;
  double* wd = a.wd + (size_t)inst * n;
  if (!exact) {  // euler: I + A dt, B dt, w dt
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - (e / n) * n;
      Ad[e] = (i == j ? 1.0 : 0.0) + X[i * N + j] * a.dt;
    }
    for (int e = tid; e < n * m; e += blockDim.x) Bd[e] = X[(e / m) * N + n + e % m] * a.dt;
    for (int i = tid; i < n; i += blockDim.x) wd[i] = X[i * N + n + m] * a.dt;
    return;
  }
  // ---- exp(X dt): scale so ||X dt / 2^s||_1 <= 1/2
  double cmax = 0.0;
  for (int j = tid; j < N; j += blockDim.x) {
    double c = 0.0;
    for (int i = 0; i < N; ++i) c += fabs(X[i * N + j]);
    cmax = fmax(cmax, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xFFFFFFFFu, cmax, o));
  if (lane == 0) red[warp] = cmax;
  __syncthreads();
  double nrm = 0.0;
  for (int w = 0; w < kWarps; ++w) nrm = fmax(nrm, red[w]);
  nrm *= a.dt;
  int s = 0;
  while (nrm > 0.5 && s < 60) {
    nrm *= 0.5;
    ++s;
  }
  const double scale = ldexp(a.dt, -s);
  __syncthreads();
  for (int e = tid; e < N * N; e += blockDim.x) {
    X[e] *= scale;
    const int i = e / N, j = e - (e / N) * N;
    T1[e] = X[e];                                   // term_1 = X
    Sm[e] = (i == j ? 1.0 : 0.0) + X[e];            // I + X
  }
  __syncthreads();
  // Taylor terms: term_k = term_{k-1} X / k; added smallest-last is not
  // needed at ||X|| <= 1/2 (terms decrease geometrically)
  for (int k = 2; k <= 18; ++k) {
    matmul(T1, X, T2, N, N);
    const double inv = 1.0 / k;
    for (int e = tid; e < N * N; e += blockDim.x) {
      const double t = T2[e] * inv;
      T1[e] = t;
      Sm[e] += t;
    }
    __syncthreads();
  }
  // squarings
  double* cur = Sm;
  double* oth = T2;
  for (int q = 0; q < s; ++q) {
    matmul(cur, cur, oth, N, N);
    double* t = cur;
    cur = oth;
    oth = t;
  }
  for (int e = tid; e < n * n; e += blockDim.x) Ad[e] = cur[(e / n) * N + e % n];
  for (int e = tid; e < n * m; e += blockDim.x) Bd[e] = cur[(e / m) * N + n + e % m];
  for (int i = tid; i < n; i += blockDim.x) wd[i] = cur[i * N + n + m];
}

// RK4 ground-truth integration of one control period per instance, one warp
// per instance (K/dynamics.py:316-330, same operation order):
//   k1 = f(x), k2 = f(x + 0.5 h k1), k3 = f(x + 0.5 h k2), k4 = f(x + h k3),
//   x += (h / 6) (k1 + 2 k2 + 2 k3 + k4),  h = dt / substeps
__global__ void __launch_bounds__(kThreads) plant_integrate_kernel(PlantArgs a, int substeps, double* xout) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double carried[kMaxLinks];
  const int n = a.n, m = a.m, L = a.links;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inst = blockIdx.x * kWarps + warp;
  const int scr = (a.kind == EMPC_PLANT_NLINK) ? L * L + 6 * L : 8;
  double* base = sm + (size_t)warp * (6 * n + m + scr);
  double* x = base;
  double* k1 = x + n;
  double* k2 = k1 + n;
  double* k3 = k2 + n;
  double* k4 = k3 + n;
  double* xt = k4 + n;  // [n + m]: evaluation point and input
  double* scratch = xt + n + m;
  if (a.kind == EMPC_PLANT_NLINK && threadIdx.x == 0) {
    double c = 0.0;
    for (int j = L - 1; j >= 0; --j) {
      c += a.mass[j];
      carried[j] = c;
    }
  }
  __syncthreads();
  if (inst >= a.count) return;  // whole warp
  for (int i = lane; i < n; i += 32) x[i] = a.x[(size_t)inst * n + i];
  for (int l = lane; l < m; l += 32) xt[n + l] = a.u[(size_t)inst * m + l];
  __syncwarp();
  const double h = a.dt / substeps;
  const double hh = 0.5 * h, h6 = h / 6.0;
  for (int s = 0; s < substeps; ++s) {
    for (int i = lane; i < n; i += 32) xt[i] = x[i];
    __syncwarp();
    plant_ode(a, xt, xt + n, k1, scratch, carried);
    for (int i = lane; i < n; i += 32) xt[i] = x[i] + hh * k1[i];
    __syncwarp();
    plant_ode(a, xt, xt + n, k2, scratch, carried);
    for (int i = lane; i < n; i += 32) xt[i] = x[i] + hh * k2[i];
    __syncwarp();
    plant_ode(a, xt, xt + n, k3, scratch, carried);
    for (int i = lane; i < n; i += 32) xt[i] = x[i] + h * k3[i];
    __syncwarp();
    plant_ode(a, xt, xt + n, k4, scratch, carried);
    for (int i = lane; i < n; i += 32) x[i] = x[i] + h6 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) xout[(size_t)inst * n + i] = x[i];
}

struct Ctx {
  int dev = -1;
  cudaStream_t stream = nullptr;
  double* dbuf = nullptr;
  size_t dcap = 0;
  double* work = nullptr;
  size_t wcap = 0;
};
thread_local Ctx g_ctx;
thread_local std::string g_err;

#define PCK(x)                                                         \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e_);         \
      return EMPC_ECUDA;                                               \
    }                                                                  \
  } while (0)

}  // namespace plantk

using namespace plantk;

extern "C" const char* empc_plant_last_error(void) { return g_err.c_str(); }

extern "C" int empc_plant_linearize_discretize(const empc_plant* plant, int32_t count, const double* x, const double* u,
                                               double eps, double dt, int32_t method, int32_t device, double* Ad,
                                               double* Bd, double* wd) {
  if (!plant || !x || !u || !Ad || !Bd || !wd || count < 0) {
    g_err = "null argument";
    return EMPC_EINVAL;
  }
  if (plant->kind != EMPC_PLANT_PENDULUM && plant->kind != EMPC_PLANT_NLINK) {
    g_err = "unknown plant kind";
    return EMPC_EINVAL;
  }
  const int L = plant->kind == EMPC_PLANT_NLINK ? plant->links : 1;
  if (L < 1 || L > kMaxLinks) {
    g_err = "links must lie in [1, 64]";
    return EMPC_EINVAL;
  }
  if (!(dt > 0.0)) {
    g_err = "dt must be positive";
    return EMPC_EINVAL;
  }
  if (method != EMPC_DISCRETIZE_EXACT && method != EMPC_DISCRETIZE_EULER) {
    g_err = "unknown discretization method";
    return EMPC_EINVAL;
  }
  if (!(eps > 0.0) || !plant->mass || !plant->length) {
    g_err = "invalid plant parameters";
    return EMPC_EINVAL;
  }
  if (count == 0) return EMPC_OK;
  const int n = 2 * L, m = L, N = n + m + 1;
  Ctx& c = g_ctx;
  PCK(cudaSetDevice(device));
  if (c.dev != device || !c.stream) {
    if (!c.stream) PCK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.dev = device;
  }
  // device buffer: params | x | u | Ad | Bd | wd
  const size_t nx = (size_t)count * n, nu = (size_t)count * m;
  const size_t nA = (size_t)count * n * n, nB = (size_t)count * n * m, nw = (size_t)count * n;
  const size_t need = 2 * (size_t)L + nx + nu + nA + nB + nw;
  if (need > c.dcap) {
    if (c.dbuf) cudaFree(c.dbuf);
    PCK(cudaMalloc(&c.dbuf, need * sizeof(double)));
    c.dcap = need;
  }
  double* dmass = c.dbuf;
  double* dlen = dmass + L;
  double* dx = dlen + L;
  double* du = dx + nx;
  double* dA = du + nu;
  double* dB = dA + nA;
  double* dw = dB + nB;
  const size_t maxs = 227 * 1024 - 2048;  // static shared arrays take the rest
  const bool fits = plant_smem_doubles(plant->kind, L, n, m, true) * sizeof(double) <= maxs;
  const size_t smem = plant_smem_doubles(plant->kind, L, n, m, fits) * sizeof(double);
  if (smem > maxs) {
    g_err = "plant too large for the linearization kernel";
    return EMPC_EINVAL;
  }
  PlantArgs a{};
  a.kind = plant->kind;
  a.links = L;
  a.n = n;
  a.m = m;
  a.count = count;
  a.method = method;
  a.eps = eps;
  a.dt = dt;
  a.damping = plant->damping;
  a.gravity = plant->gravity;
  a.mass = dmass;
  a.length = dlen;
  a.x = dx;
  a.u = du;
  a.Ad = dA;
  a.Bd = dB;
  a.wd = dw;
  a.ws_smem = fits ? 1 : 0;
  if (!a.ws_smem) {
    const size_t w = (size_t)count * 4 * N * N;
    if (w > c.wcap) {
      if (c.work) cudaFree(c.work);
      PCK(cudaMalloc(&c.work, w * sizeof(double)));
      c.wcap = w;
    }
    a.work = c.work;
  }
  PCK(cudaFuncSetAttribute(plant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)maxs));
  PCK(cudaMemcpyAsync(dmass, plant->mass, L * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  PCK(cudaMemcpyAsync(dlen, plant->length, L * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  PCK(cudaMemcpyAsync(dx, x, nx * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  PCK(cudaMemcpyAsync(du, u, nu * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  plant_kernel<<<count, kThreads, smem, c.stream>>>(a);
  PCK(cudaGetLastError());
  PCK(cudaMemcpyAsync(Ad, dA, nA * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  PCK(cudaMemcpyAsync(Bd, dB, nB * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  PCK(cudaMemcpyAsync(wd, dw, nw * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  PCK(cudaStreamSynchronize(c.stream));
  return EMPC_OK;
}

extern "C" int empc_plant_integrate(const empc_plant* plant, int32_t count, const double* x, const double* u, double dt,
                                    int32_t substeps, int32_t device, double* x_out) {
  if (!plant || !x || !u || !x_out || count < 0 || substeps < 1 || !(dt > 0.0)) {
    g_err = "invalid argument";
    return EMPC_EINVAL;
  }
  if (plant->kind != EMPC_PLANT_PENDULUM && plant->kind != EMPC_PLANT_NLINK) {
    g_err = "unknown plant kind";
    return EMPC_EINVAL;
  }
  const int L = plant->kind == EMPC_PLANT_NLINK ? plant->links : 1;
  if (L < 1 || L > kMaxLinks || !plant->mass || !plant->length) {
    g_err = "invalid plant parameters";
    return EMPC_EINVAL;
  }
  if (count == 0) return EMPC_OK;
  const int n = 2 * L, m = L;
  Ctx& c = g_ctx;
  PCK(cudaSetDevice(device));
  if (c.dev != device || !c.stream) {
    if (!c.stream) PCK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.dev = device;
  }
  const size_t nx = (size_t)count * n, nu = (size_t)count * m;
  const size_t need = 2 * (size_t)L + 2 * nx + nu;
  if (need > c.dcap) {
    if (c.dbuf) cudaFree(c.dbuf);
    PCK(cudaMalloc(&c.dbuf, need * sizeof(double)));
    c.dcap = need;
  }
  double* dmass = c.dbuf;
  double* dlen = dmass + L;
  double* dx = dlen + L;
  double* du = dx + nx;
  double* dout = du + nu;
  const int scr = plant->kind == EMPC_PLANT_NLINK ? L * L + 6 * L : 8;
  const size_t smem = (size_t)kWarps * (6 * n + m + scr) * sizeof(double);
  if (smem > 227 * 1024 - 2048) {
    g_err = "plant too large for the integration kernel";
    return EMPC_EINVAL;
  }
  PlantArgs a{};
  a.kind = plant->kind;
  a.links = L;
  a.n = n;
  a.m = m;
  a.count = count;
  a.dt = dt;
  a.damping = plant->damping;
  a.gravity = plant->gravity;
  a.mass = dmass;
  a.length = dlen;
  a.x = dx;
  a.u = du;
  PCK(cudaFuncSetAttribute(plant_integrate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 2048));
  PCK(cudaMemcpyAsync(dmass, plant->mass, L * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  PCK(cudaMemcpyAsync(dlen, plant->length, L * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  PCK(cudaMemcpyAsync(dx, x, nx * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  PCK(cudaMemcpyAsync(du, u, nu * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  plant_integrate_kernel<<<(count + kWarps - 1) / kWarps, kThreads, smem, c.stream>>>(a, substeps, dout);
  PCK(cudaGetLastError());
  PCK(cudaMemcpyAsync(x_out, dout, nx * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  PCK(cudaStreamSynchronize(c.stream));
  return EMPC_OK;
}
