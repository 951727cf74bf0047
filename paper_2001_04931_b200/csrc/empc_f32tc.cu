// FP32 tensor-core rollout variants (rollout_tc_kernel, empc_tc_rollout.cuh).
#include "empc_tc_rollout.cuh"
#include "empc_variants.h"

namespace empc {

// NP -> MMA N (multiple of 16), MMA K (multiple of 8), coordinates per thread
// NH, column groups WG (threads = 128 WG), CTAs per SM for the register budget
#define TCV(NP, NN, NK, NH, WG, MINB)                                                                   \
  Variant<float>{NP, WG, NH, false, false, 1, false, 128 * WG, &rollout_tc_kernel<NP, NN, NK, NH, WG, MINB>, \
                 "float NP" #NP " tcgen05 tf32x3 N" #NN " K" #NK " NH" #NH " WG" #WG, 1, NN, NK}

std::vector<Variant<float>> variants_f32_tc(int NP) {
  switch (NP) {
    case 4: return {TCV(4, 16, 8, 4, 1, 4)};
    case 8: return {TCV(8, 16, 8, 8, 1, 4)};
    case 12: return {TCV(12, 16, 16, 12, 1, 5)};
    case 16: return {TCV(16, 16, 16, 16, 1, 4)};
    case 24: return {TCV(24, 32, 24, 24, 1, 4), TCV(24, 32, 24, 12, 2, 3)};
    case 32: return {TCV(32, 32, 32, 16, 2, 2)};
    case 48: return {TCV(48, 48, 48, 24, 2, 1)};
    case 64: return {TCV(64, 64, 64, 16, 4, 1)};
    case 96: return {TCV(96, 96, 96, 24, 4, 1)};
    case 128: return {TCV(128, 128, 128, 32, 4, 1)};
  }
  return {};
}

}  // namespace empc
