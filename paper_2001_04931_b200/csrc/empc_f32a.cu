// float rollout variants, NP <= 24 (separate TU for parallel builds)
#include "empc_variants.h"

namespace empc {
#define FSMALL(NP) RV(float, NP, 1, 4, true, false), RV(float, NP, 2, 2, true, false), RV(float, NP, 2, 4, true, false), \
                   RV(float, NP, 4, 4, false, false), RV(float, NP, 4, 8, false, false), RV(float, NP, 4, 4, false, true)


std::vector<Variant<float>> variants_f32_small(int NP) {
  switch (NP) {
    case 4: return {FSMALL(4)};
    case 8: return {FSMALL(8), RVK(float, 8, 1, 4, true, false, 2)};
    case 12: return {FSMALL(12)};
    case 16: return {FSMALL(16), RVK(float, 16, 1, 4, true, false, 2)};
    case 24: return {FSMALL(24), RVK(float, 24, 1, 4, true, false, 2), RVK(float, 24, 2, 2, true, false, 2),
                     RVK(float, 24, 4, 2, true, false, 2), RVK(float, 24, 4, 4, true, false, 2)};
  }
  return {};
}

}  // namespace empc
