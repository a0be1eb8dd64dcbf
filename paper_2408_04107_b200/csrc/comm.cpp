// comm.cpp — placeholder for the sequence-parallel exchange.
#include "api_util.h"
#include "ctx.h"
namespace zdc {
void comm_destroy(zdc_ctx*) {}
}  // namespace zdc
extern "C" {
zdc_status zdc_comm_init(zdc_ctx*, const void*, int32_t, int32_t) {
  return zdc::fail(ZDC_ERR_UNSUPPORTED, "zdc_comm_init: not built yet");
}
zdc_status zdc_sp_prefill(zdc_ctx*, int32_t, int32_t, const uint16_t*, uint16_t*, int32_t, int32_t, int32_t,
                          zdc_sp_stats*, void*) {
  return zdc::fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_prefill: not built yet");
}
zdc_status zdc_sp_positions(int32_t, int32_t, int32_t, int32_t, int32_t*) {
  return zdc::fail(ZDC_ERR_UNSUPPORTED, "zdc_sp_positions: not built yet");
}
}
