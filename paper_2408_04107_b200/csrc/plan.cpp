// plan.cpp — NEXT-3's layer-group identification: "we offline identify layers that
// have the same important and unimportant token sets (i.e., repetition ratio > 95%)", so one
// representative layer's classification (from the reused softmax denominators) serves its
// whole group (zdc_plan.group_rep).  Host-side, offline, integer arithmetic (reading c22).
#include <cstdint>

#include "api_util.h"

using namespace zdc;

extern "C" {

zdc_status zdc_layer_groups(const uint8_t* classes, int32_t n_layers, int64_t positions, int32_t threshold_bp,
                            int32_t* group_rep) {
  if (!classes || !group_rep) return fail(ZDC_ERR_INVALID_ARG, "zdc_layer_groups: null argument");
  if (n_layers <= 0 || positions <= 0 || threshold_bp < 0 || threshold_bp > 10000)
    return fail(ZDC_ERR_SHAPE, "zdc_layer_groups: n_layers %d positions %lld threshold %d bp", n_layers,
                static_cast<long long>(positions), threshold_bp);
  int cur = 0;
  group_rep[0] = 0;
  for (int l = 1; l < n_layers; ++l) {
    const uint8_t* a = classes + static_cast<int64_t>(cur) * positions;
    const uint8_t* b = classes + static_cast<int64_t>(l) * positions;
    int64_t same = 0;
    for (int64_t i = 0; i < positions; ++i) same += (a[i] != 0) == (b[i] != 0);
    // repetition ratio same / positions > threshold_bp / 10000, exactly (128-bit products)
    if (static_cast<__int128>(same) * 10000 > static_cast<__int128>(threshold_bp) * positions) {
      group_rep[l] = cur;
    } else {
      cur = l;
      group_rep[l] = l;
    }
  }
  return ZDC_OK;
}

}  // extern "C"
