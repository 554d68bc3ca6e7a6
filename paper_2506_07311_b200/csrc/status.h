// Thread-local error reporting shared by the host allocator and the kernels.
#pragma once
#include <cstdarg>
#include <cstdio>

namespace pkv {

char* error_buffer();

inline int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(error_buffer(), 1024, fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace pkv
