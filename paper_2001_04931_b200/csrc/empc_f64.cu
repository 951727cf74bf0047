// double rollout variants
#include "empc_variants.h"

namespace empc {
#define DV(NP) RV(double, NP, 1, 2, true, false), RV(double, NP, 2, 4, false, false), RV(double, NP, 2, 4, false, true)
template <>
std::vector<Variant<double>> variants_for<double>(int NP) {
  switch (NP) {
    case 4: return {DV(4)};
    case 8: return {DV(8)};
    case 12: return {DV(12)};
    case 16: return {DV(16)};
    case 24: return {DV(24)};
    case 32: return {DV(32)};
    case 48: return {DV(48)};
    case 64: return {RV(double, 64, 2, 4, false, false), RV(double, 64, 2, 4, false, true)};
    case 96: return {RV(double, 96, 2, 4, false, false), RV(double, 96, 2, 4, false, true)};
    case 128: return {RV(double, 128, 2, 4, false, false), RV(double, 128, 2, 4, false, true)};
  }
  return {};
}


}  // namespace empc
