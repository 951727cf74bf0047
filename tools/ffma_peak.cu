// FP32 FFMA peak microbenchmark for the roofline denominator (SURVEY.md §8(d):
// MEASURED_PEAKS.json has no FP32 entry).  Full grid, 8 independent chains per
// thread, timed with CUDA events after warm-up.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void ffma_kernel(float* out, int iters, float x, float y) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) a[i] = fmaf(a[i], x, y);        // 3 operands, 2 shared
        else a[i] = fmaf(a[i], x, a[(i + 1) & 7]);     // 3 distinct registers
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678f) out[0] = s;
}

// FP64 DFMA peak (roofline denominator of the condensed scorer, which
// evaluates its quadratic form in FP64)
__global__ void dfma_kernel(double* out, int iters, double x, double y) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], x, y);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 4, iters = 4096;
  double flop = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  for (int mode = 0; mode < 2; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 12; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) ffma_kernel<0><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
      else ffma_kernel<1><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2 && ms < best) best = ms;
    }
    printf("{\"ffma_mode\": %d, \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d}\n",
           mode, flop / (best * 1e-3) / 1e12, best, sms, clk);
  }
  {
    double* outd;
    cudaMalloc(&outd, 8);
    const int it64 = iters / 8;
    const double flop64 = 2.0 * 8 * 16 * (double)it64 * threads * blocks;
    float best = 1e30f;
    for (int rep = 0; rep < 12; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(outd, it64, 0.999, 1e-3);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 2 && ms < best) best = ms;
    }
    printf("{\"dfma\": 1, \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d}\n", flop64 / (best * 1e-3) / 1e12, best, sms);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
