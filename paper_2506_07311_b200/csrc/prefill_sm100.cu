// K3 placeholder: the tcgen05 prefill kernel lands in a later commit; until
// then pkv_prefill_supported() reports no support and callers use K2.
#include "pkv200.h"
#include "status.h"

extern "C" int pkv_prefill_supported(int32_t, int32_t, int32_t, int32_t, int32_t) { return 0; }
extern "C" int pkv_paged_prefill(const pkv_prefill_args*, void*) {
  return pkv::fail(PKV_CONFIG_ERROR, "tcgen05 prefill not built");
}
