// fold.cpp — placeholder for the host fp64 fold.
#include "api_util.h"
extern "C" zdc_status zdc_fold_weights(const zdc_dims*, const double*, const double*, const double*, const double*,
                                       const double*, int64_t, double*, double*, double*, double*, double*, double*,
                                       double*, double*) {
  return zdc::fail(ZDC_ERR_UNSUPPORTED, "zdc_fold_weights: not built yet");
}
