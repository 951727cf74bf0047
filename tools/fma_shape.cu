// Micro-benchmark of the rollout inner-product shape (tools/, not product):
// RR rows of A in registers x CC candidates, x from shared memory (LDS.128
// broadcast) or from registers; reports FFMA throughput vs the 72.5 TF peak.
#include <cstdio>
#include <cuda_runtime.h>

template <int RR, int CC, int NP, bool FROM_SMEM, int NSPLIT>
__global__ void __launch_bounds__(384, 1) shape_kernel(float* out, int iters) {
  __shared__ __align__(16) float xs[CC * 4][NP + 4];
  for (int i = threadIdx.x; i < CC * 4 * (NP + 4); i += blockDim.x) (&xs[0][0])[i] = 1e-3f * (i % 97);
  __syncthreads();
  float a[RR][NP];
#pragma unroll
  for (int r = 0; r < RR; ++r)
#pragma unroll
    for (int j = 0; j < NP; ++j) a[r][j] = 1e-4f * (threadIdx.x + r * 7 + j);
  float xr[CC][NP];
  if (!FROM_SMEM) {
#pragma unroll
    for (int q = 0; q < CC; ++q)
#pragma unroll
      for (int j = 0; j < NP; ++j) xr[q][j] = 1e-3f * (q + j);
  }
  const int grp = (threadIdx.x / 32) % 4;
  float acc[RR][CC][NSPLIT];
#pragma unroll
  for (int r = 0; r < RR; ++r)
#pragma unroll
    for (int q = 0; q < CC; ++q)
#pragma unroll
      for (int s = 0; s < NSPLIT; ++s) acc[r][q][s] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int jv = 0; jv < NP / 4; ++jv) {
      float xv[CC][4];
#pragma unroll
      for (int q = 0; q < CC; ++q) {
        if (FROM_SMEM) {
          const float4 t = *reinterpret_cast<const float4*>(&xs[grp * CC + q][jv * 4]);
          xv[q][0] = t.x; xv[q][1] = t.y; xv[q][2] = t.z; xv[q][3] = t.w;
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t) xv[q][t] = xr[q][jv * 4 + t];
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int r = 0; r < RR; ++r)
#pragma unroll
          for (int q = 0; q < CC; ++q) acc[r][q][t % NSPLIT] = fmaf(a[r][jv * 4 + t], xv[q][t], acc[r][q][t % NSPLIT]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < RR; ++r)
#pragma unroll
    for (int q = 0; q < CC; ++q)
#pragma unroll
      for (int k = 0; k < NSPLIT; ++k) s += acc[r][q][k];
  if (s == 1234.5f) out[0] = s;
}

template <int RR, int CC, int NP, bool SM, int NS>
void run(const char* name, float* out, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000, blocks = 148;
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    shape_kernel<RR, CC, NP, SM, NS><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double flop = 2.0 * RR * CC * NP * (double)iters * threads * blocks;
  printf("%-34s threads=%d  %.2f TFLOP/s  (%.1f%% of 72.5)  err=%s\n", name, threads, flop / (best * 1e-3) / 1e12,
         100.0 * flop / (best * 1e-3) / 1e12 / 72.5, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  run<2, 4, 24, true, 1>("RR2 CC4 smem-x NS1", out, 352);
  run<2, 4, 24, true, 2>("RR2 CC4 smem-x NS2", out, 352);
  run<2, 4, 24, false, 1>("RR2 CC4 reg-x NS1", out, 352);
  run<1, 4, 48, true, 2>("RR1 CC4 smem-x NS2", out, 352);
  run<2, 4, 24, true, 1>("RR2 CC4 smem-x NS1 (12 warps)", out, 384);
  run<2, 4, 24, true, 1>("RR2 CC4 smem-x NS1 (8 warps)", out, 256);
  run<3, 4, 24, true, 1>("RR3 CC4 smem-x NS1 (7 warps)", out, 224);
  run<4, 4, 24, true, 1>("RR4 CC4 smem-x NS1 (8 warps)", out, 256);
  return 0;
}
