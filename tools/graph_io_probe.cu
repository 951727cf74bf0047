// Host-visible latency of a captured solve graph as a function of its copy
// nodes: launch + cudaStreamSynchronize wall time (median of 2000) for an
// empty 148-CTA kernel with the C3 public-API copies around it (H2D problem
// 47 KB + H2D state 1 KB, D2H result 1 KB, D2D population 1.6 MB + costs
// 16 KB), merged copies, and copy kernels instead of DMA nodes.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void body(float* x) {
  if (threadIdx.x == 0 && x[blockIdx.x] == 12345.f) x[blockIdx.x] = 0.f;
}
__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
// reads the host staging directly (mapped pinned memory) into device memory
__global__ void stage_kernel(const float4* __restrict__ h, float4* __restrict__ d, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) d[i] = h[i];
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const size_t prob = 47 * 1024, state = 1024, out = 1024, pop = 1600 * 1024, cost = 16 * 1024;
  char *hp, *hs, *ho;
  cudaMallocHost(&hp, prob + state);
  hs = hp + prob;
  cudaMallocHost(&ho, out);
  char *dp, *ds, *dout, *dpop, *dslot;
  cudaMalloc(&dp, prob + state);
  ds = dp + prob;
  cudaMalloc(&dout, out);
  cudaMalloc(&dpop, pop + cost);
  cudaMalloc(&dslot, pop + cost);
  float* x;
  cudaMalloc(&x, 4096);
  cudaMemset(x, 0, 4096);
  auto run = [&](const char* name, auto&& enqueue) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    enqueue();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    std::vector<double> t;
    for (int i = 0; i < 2200; ++i) {
      auto a = std::chrono::steady_clock::now();
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      auto b = std::chrono::steady_clock::now();
      if (i >= 200) t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
    }
    std::sort(t.begin(), t.end());
    printf("{\"graph\": \"%s\", \"median_us\": %.2f, \"q1_us\": %.2f, \"q3_us\": %.2f}\n", name, t[t.size() / 2],
           t[t.size() / 4], t[3 * t.size() / 4]);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  };
  run("kernel only", [&] { body<<<148, 352, 0, s>>>(x); });
  run("current: 2 H2D + kernel + D2H + 2 D2D", [&] {
    cudaMemcpyAsync(dp, hp, prob, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(ds, hs, state, cudaMemcpyHostToDevice, s);
    body<<<148, 352, 0, s>>>(x);
    cudaMemcpyAsync(ho, dout, out, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(dslot, dpop, pop, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(dslot + pop, dpop + pop, cost, cudaMemcpyDeviceToDevice, s);
  });
  run("merged: H2D + kernel + D2H + D2D", [&] {
    cudaMemcpyAsync(dp, hp, prob + state, cudaMemcpyHostToDevice, s);
    body<<<148, 352, 0, s>>>(x);
    cudaMemcpyAsync(ho, dout, out, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(dslot, dpop, pop + cost, cudaMemcpyDeviceToDevice, s);
  });
  run("merged, slot copy by kernel: H2D + kernel + copy kernel + D2H", [&] {
    cudaMemcpyAsync(dp, hp, prob + state, cudaMemcpyHostToDevice, s);
    body<<<148, 352, 0, s>>>(x);
    copy_kernel<<<148, 512, 0, s>>>((const float4*)dpop, (float4*)dslot, (pop + cost) / 16);
    cudaMemcpyAsync(ho, dout, out, cudaMemcpyDeviceToHost, s);
  });
  run("zero-copy stage kernel + kernel + copy kernel + D2H", [&] {
    stage_kernel<<<32, 256, 0, s>>>((const float4*)hp, (float4*)dp, (prob + state) / 16);
    body<<<148, 352, 0, s>>>(x);
    copy_kernel<<<148, 512, 0, s>>>((const float4*)dpop, (float4*)dslot, (pop + cost) / 16);
    cudaMemcpyAsync(ho, dout, out, cudaMemcpyDeviceToHost, s);
  });
  run("zero-copy stage kernel + kernel + copy kernel (D2H by kernel store)", [&] {
    stage_kernel<<<32, 256, 0, s>>>((const float4*)hp, (float4*)dp, (prob + state) / 16);
    body<<<148, 352, 0, s>>>(x);
    copy_kernel<<<148, 512, 0, s>>>((const float4*)dpop, (float4*)dslot, (pop + cost) / 16);
    stage_kernel<<<1, 64, 0, s>>>((const float4*)dout, (float4*)ho, out / 16);
  });
  return 0;
}
