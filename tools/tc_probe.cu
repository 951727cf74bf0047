// Probe of the tcgen05 kind::tf32 building blocks (empc_tc.cuh): one CTA
// computes D = A B^T (A: 128 x K, B: N x K, FP32) with 1 or 3 TF32 terms
// and the result is compared against an FP64 host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_2001_04931_b200/csrc tools/tc_probe.cu -o tools/tc_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "empc_tc.cuh"

using namespace empc;

__global__ void probe(const float* A, const float* B, float* D, int N, int K, int terms) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* Ahi = reinterpret_cast<float*>(sm);
  float* Alo = Ahi + 128 * K;
  float* Bhi = Alo + 128 * K;
  float* Blo = Bhi + N * K;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const float v = A[e], h = tc::to_tf32(v);
    const int o = (k / 4) * 128 * 4 + r * 4 + (k % 4);
    Ahi[o] = h;
    Alo[o] = v - h;
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const float v = B[e], h = tc::to_tf32(v);
    const int o = (k / 4) * N * 4 + r * 4 + (k % 4);
    Bhi[o] = h;
    Blo[o] = v - h;
  }
  if (tid < 32) tc::tmem_alloc(&tbase, tc::tmem_cols_for(N));
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, N);
    const uint32_t a0 = tc::smem_u32(Ahi), a1 = tc::smem_u32(Alo), b0 = tc::smem_u32(Bhi), b1 = tc::smem_u32(Blo);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t ao = s * 2 * 128 * 16, bo = s * 2 * N * 16;
      tc::mma_tf32(tm, tc::sdesc(a0 + ao, 128 * 16, 128), tc::sdesc(b0 + bo, N * 16, 128), idesc, s > 0);
      if (terms == 3) {
        tc::mma_tf32(tm, tc::sdesc(a1 + ao, 128 * 16, 128), tc::sdesc(b0 + bo, N * 16, 128), idesc, 1);
        tc::mma_tf32(tm, tc::sdesc(a0 + ao, 128 * 16, 128), tc::sdesc(b1 + bo, N * 16, 128), idesc, 1);
      }
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  const int w = tid >> 5;
  for (int c = 0; c < N; c += 4) {
    float v[4];
    tc::tmem_ld4(tm + ((uint32_t)(32 * w) << 16) + c, v);
    tc::tmem_wait_ld();
    for (int q = 0; q < 4; ++q) D[tid * N + c + q] = v[q];
  }
  tc::fence_before();
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(tm, tc::tmem_cols_for(N));
}

int main() {
  const int shapes[][2] = {{32, 24}, {16, 16}, {48, 48}, {96, 96}, {32, 32}, {112, 104}};
  int bad = 0;
  for (auto& sh : shapes) {
    const int N = sh[0], K = sh[1];
    std::vector<float> A(128 * K), B(N * K), D(128 * N);
    srand(N * 1000 + K);
    for (auto& x : A) x = (float)rand() / RAND_MAX * 2.f - 1.f;
    for (auto& x : B) x = ((float)rand() / RAND_MAX * 2.f - 1.f) * 0.01f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)(2 * 128 * K + 2 * N * K) * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int terms : {1, 3}) {
      cudaMemset(dD, 0, D.size() * 4);
      probe<<<1, 128, smem>>>(dA, dB, dD, N, K, terms);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { std::printf("N=%d K=%d: %s\n", N, K, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxrel = 0, maxabs = 0;
      for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
          double ref = 0, mag = 0;
          for (int k = 0; k < K; ++k) { ref += (double)A[i * K + k] * B[j * K + k]; mag += std::fabs((double)A[i * K + k] * B[j * K + k]); }
          const double err = std::fabs(D[i * N + j] - ref);
          maxabs = std::fmax(maxabs, err);
          maxrel = std::fmax(maxrel, err / mag);
        }
      const bool ok = terms == 3 ? maxrel < 1e-6 : maxrel < 2e-3;
      bad += !ok;
      std::printf("N=%3d K=%3d terms=%d  max |err| / sum|a b| = %.3e  max abs %.3e  %s\n", N, K, terms, maxrel, maxabs,
                  ok ? "ok" : "FAIL");
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
  }
  return bad ? 1 : 0;
}
