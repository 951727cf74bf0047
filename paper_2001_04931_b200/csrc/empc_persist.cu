// Persistent cooperative solve kernels for the default single-instance FP32
// variants (see persist_kernel in empc_kernels.cuh).
#include "empc_variants.h"

namespace empc {

#define PK(NP, RR, CC, AR, KS)                                                                             \
  PersistVariant<float>{NP, RR, CC, AR, KS,                                                              \
                        &persist_kernel<float, NP, RR, CC, AR, false, KS, false,                         \
                                        maxt_for(NP, RR, CC, AR, sizeof(float), KS)>,                    \
                        false, false, maxt_for(NP, RR, CC, AR, sizeof(float), KS)}

#define PKH(NP, RR, CC, AR, KS)                                                                            \
  PersistVariant<float>{NP, RR, CC, AR, KS,                                                              \
                        &persist_kernel<float, NP, RR, CC, AR, false, KS, false,                         \
                                        maxt_for(NP, RR, CC, AR, sizeof(float), KS), true>,              \
                        true, false, maxt_for(NP, RR, CC, AR, sizeof(float), KS)}

// warp-synchronous: a candidate group's rows x column halves fill one warp
// (MAXT explicit: helper warps beyond the candidate groups)
#define PKW(NP, RR, CC, AR, KS, HK, MAXT)                                                                  \
  PersistVariant<float>{NP, RR, CC, AR, KS,                                                              \
                        &persist_kernel<float, NP, RR, CC, AR, false, KS, true, MAXT, HK>, HK, true, MAXT}

template <>
std::vector<PersistVariant<float>> persist_variants<float>() {
  return {PK(4, 1, 4, true, 1),  PK(8, 1, 4, true, 1),  PK(12, 2, 2, true, 1), PK(16, 2, 2, true, 1),
          PK(24, 2, 4, true, 2), PK(32, 2, 4, true, 2), PK(48, 2, 4, true, 2), PK(48, 1, 4, true, 1),
          PKH(48, 2, 4, true, 2), PKH(48, 1, 4, true, 1), PKH(32, 2, 4, true, 2),
          PKW(48, 3, 4, true, 2, false, 256), PKW(48, 3, 4, true, 2, true, 384),
          // one warp = two candidate groups of 16 lanes x 3 rows, no split-K shuffle
          PKW(48, 3, 1, true, 1, true, 448), PKW(48, 3, 2, true, 1, true, 384),
          // small states (C1, C2): warp-synchronous groups of NRG lanes, several per warp
          PKW(4, 1, 4, true, 1, false, 512), PKW(4, 1, 2, true, 1, false, 512),
          PKW(12, 3, 4, true, 1, false, 512), PKW(12, 3, 2, true, 1, false, 512)};
}

template <>
std::vector<PersistVariant<double>> persist_variants<double>() {
  return {};
}

}  // namespace empc
