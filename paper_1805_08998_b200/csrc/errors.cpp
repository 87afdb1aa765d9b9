// Thread-local last-error string behind hx_last_error().
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "hx_internal.h"

namespace hx {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace hx

extern "C" int hx_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return int(hx::g_last_error.size());
  std::strncpy(buf, hx::g_last_error.c_str(), len - 1);
  buf[len - 1] = '\0';
  return int(hx::g_last_error.size());
}

extern "C" int hx_version(void) { return 1; }

// Planner-only builds (no CUDA runtime linked): plain heap memory.  libhx.so overrides these
// with the page-locked cache of runtime.cu.
namespace hx {
__attribute__((weak)) void* pinned_alloc(size_t bytes) {
  void* p = std::malloc(bytes ? bytes : 1);
  if (!p) throw std::bad_alloc();
  return p;
}
__attribute__((weak)) void pinned_free(void* p, size_t) { std::free(p); }
}  // namespace hx
