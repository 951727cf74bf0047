// Issue cost of tcgen05.mma kind::tf32 (A in TMEM) from one thread: a fully
// unrolled 36-MMA step (12 K-steps x 3 split terms) issued (a) by thread 0
// inside `if (threadIdx.x == 0)`, (b) by warp 0 through one inline-asm block
// guarded by elect.sync, (c) like (b) with 12 MMAs per asm block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -I paper_2001_04931_b200/csrc tools/tc_issue.cu -o tools/tc_issue
#include <cstdio>
#include "empc_tc.cuh"
using namespace empc;

template <int N, int MODE>
__global__ void step(int reps, long long* out, int aoff, int loff, int bmode) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  float* B = reinterpret_cast<float*>(sm);
  for (int e = threadIdx.x; e < 2 * N * 96; e += blockDim.x) {
    const float r = (float)((e * 2654435761u) % 1000u) / 1000.f - 0.5f;
    B[e] = bmode == 0 ? 0.001f * (e % 7) : bmode == 1 ? 0.f : bmode == 2 ? r * 1e-2f : (e % 5 == 0 ? r * 1e-2f : 0.f);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) { tc::mbar_init(&mbar, 1); tc::mbar_fence_init(); }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = __shfl_sync(0xffffffffu, tbase, 0);
  constexpr uint32_t idesc = tc::idesc_tf32(128, N);
  const uint64_t b0 = tc::sdesc(tc::smem_u32(B), N * 16, 128);
  const uint64_t b1 = tc::sdesc(tc::smem_u32(B + N * 96), N * 16, 128);
  const uint32_t a0 = tm + aoff, a1 = tm + aoff + loff;
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    if (MODE == 2 && threadIdx.x < 128) {  // the rollout's TMEM traffic: read D, write A hi / lo
      const uint32_t lb = tm + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16);
      float acc = 0.f;
      for (int q = 0; q < N / 4; ++q) {
        float v[4];
        tc::tmem_ld4(lb + 4 * q, v);
        tc::tmem_wait_ld();
        acc += v[0] + v[1] + v[2] + v[3];
      }
      for (int q = 0; q < 24; ++q) {
        const float w[4] = {acc * 1e-3f + 0.37f * q, 1.1f * q - 3.f, 2.f + q, 0.5f * threadIdx.x};
        tc::tmem_st4(lb + aoff + 4 * q, w);
        tc::tmem_st4(lb + aoff + loff + 4 * q, w);
      }
      tc::tmem_wait_st();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const long long t0 = clock64();
    if constexpr (MODE != 1) {
      if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < 12; ++s) {
          const uint64_t ob = (uint64_t)((s * 2 * N * 16) >> 4);
          tc::mma_tf32_ts(tm, a1 + 8 * s, b0 + ob, idesc, s > 0);
          tc::mma_tf32_ts(tm, a0 + 8 * s, b1 + ob, idesc, 1);
          tc::mma_tf32_ts(tm, a0 + 8 * s, b0 + ob, idesc, 1);
        }
        tc::commit(&mbar);
      }
    } else {
      if (threadIdx.x < 32) {
#pragma unroll
        for (int s = 0; s < 12; ++s) {
          const uint64_t ob = (uint64_t)((s * 2 * N * 16) >> 4);
          asm volatile(
              "{\n\t.reg .pred e, p;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "setp.ne.and.b32 p, %6, 0, e;\n\t"
              "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n\t"
              "@!p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %5, 1;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, 1;\n\t}\n" ::"r"(tm),
              "r"(a1 + 8 * s), "r"(a0 + 8 * s), "l"(b0 + ob), "l"(b1 + ob), "r"(idesc), "r"(s));
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                tc::smem_u32(&mbar))
            : "memory");
      }
    }
    const long long t1 = clock64();
    tc::mbar_wait(&mbar, r & 1);
    const long long t2 = clock64();
    if (t2 - t0 < best) best = t2 - t0;
    if (threadIdx.x == 0 && r == reps - 1) out[1] = t1 - t0;
  }
  if (threadIdx.x == 0) out[0] = best;
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 512);
}

template <int N, int MODE>
void run(long long* d, int aoff = 128, int loff = 128, int threads = 128, int bmode = 0) {
  cudaFuncSetAttribute(step<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  step<N, MODE><<<1, threads, 2 * N * 96 * 4>>>(20, d, aoff, loff, bmode);
  long long c[2] = {0, 0};
  cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
  std::printf("bmode=%d N=%3d mode=%d aoff=%d loff=%d thr=%d: step %6lld cycles (%5.1f per MMA, floor %d), issue %lld\n", N, MODE,
              aoff, loff, threads, c[0], c[0] / 36.0, 128 * N / 256, c[1]);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int bm = 0; bm < 4; ++bm) run<96, 2>(d, 96, 96, 512, bm);
  for (int bm = 0; bm < 4; ++bm) run<32, 2>(d, 32, 24, 256, bm);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("%s\n", cudaGetErrorString(e));
  return 0;
}
