// Rollout kernel variant table shared by the host engine and the
// per-precision instantiation units (empc_f32a.cu, empc_f32b.cu, empc_f64.cu).
#pragma once

#include <vector>

#include "empc_kernels.cuh"

namespace empc {

template <typename S>
struct Variant {
  int NP, RR, CC;
  bool areg, dq;
  int ks;
  bool ws;
  int maxt;
  void (*kernel)(const RolloutArgs<S>);
  const char* name;
  // tensor-core rollout (rollout_tc_kernel): RR = column groups WG, CC =
  // state coordinates per thread NH, MMA N / K extents
  int tc = 0, tc_nn = 0, tc_nk = 0;
};

// register budget per variant: registers ~ A-in-register rows + accumulators
// + operand buffers; the launch bound is the largest thread count that fits.
constexpr int maxt_for(int NP, int RR, int CC, bool areg, int elem, int KS) {
  const int words = elem / 4;
  const int regs = (areg ? RR * (NP / KS) * words : 0) + RR * CC * words * 4 + CC * 8 * words + 48;
  return regs <= 64 ? 1024 : regs <= 85 ? 768 : regs <= 128 ? 512 : regs <= 168 ? 384 : 256;
}

#define RVW(S, NP, RR, CC, AR, DQ, KS, WS)                                                                 \
  Variant<S>{NP, RR, CC, AR, DQ, KS, WS, maxt_for(NP, RR, CC, AR, sizeof(S), KS),                         \
             &rollout_kernel<S, NP, RR, CC, AR, DQ, KS, WS, maxt_for(NP, RR, CC, AR, sizeof(S), KS)>,      \
             #S " NP" #NP " RR" #RR " CC" #CC " areg=" #AR " dq=" #DQ " ks=" #KS " ws=" #WS}
#define RVK(S, NP, RR, CC, AR, DQ, KS) RVW(S, NP, RR, CC, AR, DQ, KS, false)
#define RV(S, NP, RR, CC, AR, DQ) RVK(S, NP, RR, CC, AR, DQ, 1)


template <typename S>
std::vector<Variant<S>> variants_for(int NP);

// FP32 tensor-core rollout variants (empc_f32tc.cu)
std::vector<Variant<float>> variants_f32_tc(int NP);

template <typename S>
struct PersistVariant {
  int NP, RR, CC;
  bool areg;
  int ks;
  void (*kernel)(const PersistArgs<S>);
  bool hk = false;  // half-K matvec (left half of Delta's columns zero)
  bool ws = false;  // warp-synchronous candidate groups (no CTA barrier per step)
  int maxt = 1024;  // launch bound of the instantiation
};

template <typename S>
std::vector<PersistVariant<S>> persist_variants();

}  // namespace empc
