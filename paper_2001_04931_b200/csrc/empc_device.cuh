// Device building blocks of the B200 EMPC hot path (sm_100a).
//
// Reference algorithm: /root/reference/pkg/src/knotmpc/empc.py (K/empc.py)
// and param.py.  See DESIGN.md for the data layout and the roofline of each
// kernel.  Nothing here depends on torch.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace empc {

// ---------------------------------------------------------------------------
// Counter-based RNG: Philox4x32-10 (Salmon et al., SC'11).  Replaces the
// reference's per-generation numpy Philox stream (K/empc.py:68-70) with
// per-(generation, instance, child, gene) counters so every thread draws its
// own numbers without any sequential state.

struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// counter word 0 reserved for per-child draws (parents); genes use 0..pm-1
constexpr uint32_t kParentWord = 0xFFFFFFFFu;
constexpr uint32_t kInitTag = 0x494E4954u;  // "INIT": cold-start stream

template <typename S>
__device__ __forceinline__ S uniform01(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ float uniform01<float>(uint32_t a, uint32_t) {
  return (float)(a >> 8) * 0x1.0p-24f;  // [0, 1)
}
template <>
__device__ __forceinline__ double uniform01<double>(uint32_t a, uint32_t b) {
  return (double)(((uint64_t)(a >> 5) << 26) | (b >> 6)) * 0x1.0p-53;  // numpy's 53-bit recipe
}

// standard normal by Box-Muller from two u32 words
template <typename S>
__device__ __forceinline__ S normal_bm(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ float normal_bm<float>(uint32_t a, uint32_t b) {
  // SFU intrinsics (|abs err| ~ 4e-7 on the log, ~5e-7 on the cosine over
  // [-pi, pi]): mutation noise needs distributional accuracy, not 1 ulp
  const float u1 = ((float)(a >> 8) + 1.0f) * 0x1.0p-24f;  // (0, 1]
  const float th = ((float)(b >> 8) * 0x1.0p-23f - 1.0f) * 3.14159265358979f;  // [-pi, pi)
  return -sqrtf(-2.0f * __logf(u1)) * __cosf(th);  // cos(th + pi) = -cos(th)
}
template <>
__device__ __forceinline__ double normal_bm<double>(uint32_t a, uint32_t b) {
  const double u1 = ((double)a + 1.0) * 0x1.0p-32;
  const double u2 = (double)b * 0x1.0p-32;
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return sqrt(-2.0 * log(u1)) * c;
}

// two standard normals (cos and sin branches of one Box-Muller transform)
template <typename S>
__device__ __forceinline__ void normal_pair(uint32_t a, uint32_t b, S& n0, S& n1);
template <>
__device__ __forceinline__ void normal_pair<float>(uint32_t a, uint32_t b, float& n0, float& n1) {
  const float u1 = ((float)(a >> 8) + 1.0f) * 0x1.0p-24f;  // (0, 1]
  const float th = ((float)(b >> 8) * 0x1.0p-23f - 1.0f) * 3.14159265358979f;  // [-pi, pi)
  const float r = sqrtf(-2.0f * __logf(u1));
  float sn, cs;
  __sincosf(th, &sn, &cs);
  n0 = -r * cs;  // cos(th + pi)
  n1 = -r * sn;  // sin(th + pi)
}
template <>
__device__ __forceinline__ void normal_pair<double>(uint32_t a, uint32_t b, double& n0, double& n1) {
  const double u1 = ((double)a + 1.0) * 0x1.0p-32;
  const double u2 = (double)b * 0x1.0p-32;
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  const double r = sqrt(-2.0 * log(u1));
  n0 = r * cs;
  n1 = r * sn;
}

// ---------------------------------------------------------------------------
// Orderable keys: the reference selects with a stable argsort of FP64 costs
// (K/empc.py:185) and picks argmin (K/empc.py:234).  Encoding (cost, index)
// into one unsigned key makes "stable" automatic (ties broken by index) and
// the sort deterministic.  NaN sorts last (numpy sort order); -0 == +0.

__device__ __forceinline__ uint32_t ord32(float f) {
  uint32_t b = __float_as_uint(f);
  if (f != f) b = 0x7FC00000u;         // canonical NaN, above +inf
  if (b == 0x80000000u) b = 0u;        // -0 -> +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ uint64_t ord64(double f) {
  uint64_t b = (uint64_t)__double_as_longlong(f);
  if (f != f) b = 0x7FF8000000000000ull;
  if (b == 0x8000000000000000ull) b = 0ull;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// 96-bit (cost, index) key for FP64 costs; 64-bit packed key for FP32.
struct Key64 {
  uint64_t v;
  __device__ __forceinline__ bool operator<(const Key64& o) const { return v < o.v; }
  __device__ __forceinline__ int idx() const { return (int)(uint32_t)v; }
};
struct Key96 {
  uint64_t c;
  uint32_t i, pad;
  __device__ __forceinline__ bool operator<(const Key96& o) const { return c < o.c || (c == o.c && i < o.i); }
  __device__ __forceinline__ int idx() const { return (int)i; }
};

template <typename S>
struct KeyOf;
template <>
struct KeyOf<float> {
  using type = Key64;
  __device__ __forceinline__ static Key64 make(float c, int i) { return Key64{((uint64_t)ord32(c) << 32) | (uint32_t)i}; }
  __device__ __forceinline__ static Key64 pad() { return Key64{~0ull}; }
  // argmin key: NaN first (numpy argmin returns the first NaN), then by value, then index
  __device__ __forceinline__ static uint64_t amin(float c, int i) {
    const uint64_t o = (c != c) ? 0ull : (uint64_t)ord32(c);
    return (o << 32) | (uint32_t)i;
  }
};
template <>
struct KeyOf<double> {
  using type = Key96;
  __device__ __forceinline__ static Key96 make(double c, int i) { return Key96{ord64(c), (uint32_t)i, 0u}; }
  __device__ __forceinline__ static Key96 pad() { return Key96{~0ull, 0xFFFFFFFFu, 0u}; }
};

// ---------------------------------------------------------------------------
// small vector helpers: CC consecutive S values, 16-byte aligned

template <typename S, int CC>
__device__ __forceinline__ void lds_vec(const S* __restrict__ p, S (&v)[CC]) {
  if constexpr (sizeof(S) == 4 && CC % 4 == 0) {
#pragma unroll
    for (int q = 0; q < CC / 4; ++q) {
      const float4 t = reinterpret_cast<const float4*>(p)[q];
      v[4 * q + 0] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else if constexpr (sizeof(S) == 8 && CC % 2 == 0) {
#pragma unroll
    for (int q = 0; q < CC / 2; ++q) {
      const double2 t = reinterpret_cast<const double2*>(p)[q];
      v[2 * q + 0] = t.x; v[2 * q + 1] = t.y;
    }
  } else if constexpr (sizeof(S) == 4 && CC == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
#pragma unroll
    for (int q = 0; q < CC; ++q) v[q] = p[q];
  }
}

template <typename S, int CC>
__device__ __forceinline__ void sts_vec(S* __restrict__ p, const S (&v)[CC]) {
  if constexpr (sizeof(S) == 4 && CC % 4 == 0) {
#pragma unroll
    for (int q = 0; q < CC / 4; ++q)
      reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else if constexpr (sizeof(S) == 8 && CC % 2 == 0) {
#pragma unroll
    for (int q = 0; q < CC / 2; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
  } else if constexpr (sizeof(S) == 4 && CC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int q = 0; q < CC; ++q) p[q] = v[q];
  }
}

}  // namespace empc
