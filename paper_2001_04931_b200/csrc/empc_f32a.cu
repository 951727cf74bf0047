// float rollout variants, NP <= 24 (separate TU for parallel builds)
#include "empc_variants.h"

namespace empc {
#define FSMALL(NP) RV(float, NP, 1, 4, true, false), RV(float, NP, 2, 2, true, false), RV(float, NP, 2, 4, true, false), \
                   RV(float, NP, 4, 4, false, false), RV(float, NP, 4, 8, false, false), RV(float, NP, 4, 4, false, true)


std::vector<Variant<float>> variants_f32_small(int NP) {
  switch (NP) {
    case 4: return {FSMALL(4), RVW(float, 4, 1, 4, true, false, 1, true), RVW(float, 4, 1, 2, true, false, 1, true)};
    case 8: return {FSMALL(8), RVK(float, 8, 1, 4, true, false, 2)};
    case 12: return {FSMALL(12), RVW(float, 12, 3, 4, true, false, 1, true), RVW(float, 12, 3, 2, true, false, 1, true)};
    case 16: return {FSMALL(16), RVK(float, 16, 1, 4, true, false, 2)};
    case 24: return {FSMALL(24), RVK(float, 24, 1, 4, true, false, 2), RVK(float, 24, 2, 2, true, false, 2),
                     RVK(float, 24, 4, 2, true, false, 2), RVK(float, 24, 4, 4, true, false, 2),
                     RVW(float, 24, 3, 4, true, false, 2, true), RVW(float, 24, 3, 4, true, false, 1, true)};
  }
  return {};
}

}  // namespace empc
