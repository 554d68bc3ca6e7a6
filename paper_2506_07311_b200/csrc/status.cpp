#include "status.h"

#include "pkv200.h"

namespace pkv {
char* error_buffer() {
  static thread_local char buf[1024] = {0};
  return buf;
}
}  // namespace pkv

extern "C" const char* pkv_last_error(void) { return pkv::error_buffer(); }
extern "C" int pkv_abi_version(void) { return 1; }

// ---- debug fault injection (tests of the all-or-nothing decode step) ----
#include <atomic>

#include "pool_internal.h"

namespace {
std::atomic<int> g_fail_site{0};
}

bool pkv_debug_should_fail(int site) {
  int want = site;
  return site != 0 && g_fail_site.compare_exchange_strong(want, 0);
}

extern "C" int pkv_debug_inject_failure(int32_t site) {
  g_fail_site.store(site);
  return PKV_OK;
}
