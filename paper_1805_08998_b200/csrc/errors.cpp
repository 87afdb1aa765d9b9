// Thread-local last-error string behind hx_last_error().
#include <cstring>
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
