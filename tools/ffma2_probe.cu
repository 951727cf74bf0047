// Packed FP32 FMA (FFMA2, PTX fma.rn.f32x2, sm_100a) vs scalar FFMA: FLOP
// rate with 8 independent chains per thread, at full occupancy and at the
// persistent C3 kernel's occupancy (one CTA of 256 threads per SM).  Decides
// whether the recursion's matvec gains from packing column pairs.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int MODE>
__global__ void probe(float* out, int iters, float x, float y) {
  if (MODE == 0) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], x, y);
      }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.678f) out[0] = s;
  } else {
    unsigned long long a[8];
    const unsigned long long xx = f2(x, x * 0.5f), yy = f2(y, y * 2.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = f2(threadIdx.x * 1e-3f + i, i * 0.5f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = ffma2(a[i], xx, yy);
      }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)a[i]) + __uint_as_float((unsigned)(a[i] >> 32));
    if (s == 12345.678f) out[0] = s;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  const int cfg[2][2] = {{512, 4}, {256, 1}};  // threads, CTAs per SM
  for (int c = 0; c < 2; ++c) {
    for (int mode = 0; mode < 2; ++mode) {
      const int threads = cfg[c][0], blocks = sms * cfg[c][1];
      const double flop = 2.0 * 16 * 8 * (double)iters * threads * blocks;
      float best = 1e30f;
      for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) probe<0><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        else probe<1><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 2 && ms < best) best = ms;
      }
      printf("{\"op\": \"%s\", \"threads_per_sm\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", mode ? "FFMA2" : "FFMA",
             threads * cfg[c][1], flop / (best * 1e-3) / 1e12, best);
    }
  }
  return 0;
}
