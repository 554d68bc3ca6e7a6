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
