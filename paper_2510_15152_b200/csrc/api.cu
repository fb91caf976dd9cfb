// api.cu -- error reporting and version of libtlru.
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace tlru {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void clear_error() { g_err[0] = '\0'; }

static std::atomic<uint64_t> g_launches{0};
void count_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace tlru

extern "C" const char* tlru_last_error(void) { return tlru::g_err; }

extern "C" const char* tlru_version(void) { return "tlru 0.1 sm_100a"; }

extern "C" uint64_t tlru_launch_count(void) { return tlru::g_launches.load(); }
