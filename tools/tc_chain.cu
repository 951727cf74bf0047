// Latency / throughput of chains of tcgen05.mma kind::tf32 (A in TMEM, B in
// smem) into ACC independent accumulators: cycles per MMA for M = 128 and
// several N.  Informs the tensor-core rollout's step structure.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_2001_04931_b200/csrc tools/tc_chain.cu -o tools/tc_chain
#include <cstdio>
#include "empc_tc.cuh"
using namespace empc;

__global__ void chain(int N, int nmma, int acc, int reps, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  float* B = reinterpret_cast<float*>(sm);
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) B[e] = 0.001f * (e % 7);
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) { tc::mbar_init(&mbar, 1); tc::mbar_fence_init(); }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t idesc = tc::idesc_tf32(128, N);
  const uint64_t bd = tc::sdesc(tc::smem_u32(B), N * 16, 128);
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
      for (int i = 0; i < nmma; ++i) {
        const int a = i % acc;
        // accumulators at columns a * N (<= 256), A operand at column 384
        tc::mma_tf32_ts(tm + a * N, tm + 384 + 8 * ((i / acc) & 7), bd, idesc, i >= acc);
      }
      tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, r & 1);
    const long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  if (threadIdx.x == 0) out[0] = best;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int N : {32, 48, 96, 128})
    for (int acc : {1, 2, 3, 4})
      for (int nm : {12, 36}) {
        if (acc * N > 384) continue;
        chain<<<1, 128, 64 * 1024>>>(N, nm, acc, 20, d);
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        std::printf("N=%3d acc=%d mmas=%2d: %6lld cycles, %6.1f per MMA (floor %d)\n", N, acc, nm, c, (double)c / nm,
                    128 * N / 256);
      }
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("%s\n", cudaGetErrorString(e));
  return 0;
}
