// float rollout variants, NP >= 32 and the dispatcher
#include "empc_variants.h"

namespace empc {
#define FSMALL(NP) RV(float, NP, 1, 4, true, false), RV(float, NP, 2, 2, true, false), RV(float, NP, 2, 4, true, false), \
                   RV(float, NP, 4, 4, false, false), RV(float, NP, 4, 8, false, false), RV(float, NP, 4, 4, false, true)


std::vector<Variant<float>> variants_f32_small(int NP);

static std::vector<Variant<float>> variants_f32_ffma(int NP) {
  switch (NP) {
    case 32: return {FSMALL(32), RVK(float, 32, 2, 2, true, false, 2), RVK(float, 32, 1, 4, true, false, 2)};
    case 48: return {FSMALL(48), RVK(float, 48, 2, 2, true, false, 2), RVK(float, 48, 2, 4, true, false, 2),
                     RVK(float, 48, 1, 4, true, false, 2), RVK(float, 48, 4, 4, false, false, 2),
                     RVK(float, 48, 4, 2, true, false, 2), RVK(float, 48, 4, 4, true, false, 2),
                     RVW(float, 48, 3, 4, true, false, 2, true), RVW(float, 48, 3, 2, true, false, 2, true),
                     RVW(float, 48, 3, 1, true, false, 1, true), RVW(float, 48, 3, 2, true, false, 1, true)};
    case 64: return {RV(float, 64, 1, 4, true, false), RV(float, 64, 2, 2, true, false), RV(float, 64, 4, 4, false, false),
                     RV(float, 64, 4, 8, false, false), RV(float, 64, 4, 4, false, true)};
    case 96: return {RV(float, 96, 4, 4, false, false), RV(float, 96, 4, 8, false, false), RV(float, 96, 2, 4, false, false),
                     RV(float, 96, 4, 4, false, true), RVK(float, 96, 4, 4, false, false, 2), RVK(float, 96, 4, 8, false, false, 2),
                     RVW(float, 96, 6, 2, false, false, 2, true), RVW(float, 96, 6, 4, false, false, 2, true)};
    case 128: return {RV(float, 128, 4, 4, false, false), RV(float, 128, 4, 8, false, false), RV(float, 128, 4, 4, false, true)};
  }
  return variants_f32_small(NP);
}

template <>
std::vector<Variant<float>> variants_for<float>(int NP) {
  std::vector<Variant<float>> v = variants_f32_ffma(NP);
  for (auto& t : variants_f32_tc(NP)) v.push_back(t);
  return v;
}

}  // namespace empc
