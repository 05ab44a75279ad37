// C-ABI housekeeping: version string and the per-thread last-error message.

#include <atomic>
#include <stdarg.h>
#include <stdio.h>

#include "pba_common.cuh"

namespace pba {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace pba

extern "C" uint64_t pba_kernel_launches(void) { return pba::g_launches.load(); }

extern "C" const char* pba_version(void) { return "paper_2303_16878_b200 pba 0.1 (sm_100a)"; }

extern "C" const char* pba_last_error(void) { return pba::g_last_error; }

extern "C" int32_t pba_build_checked(void) {
#ifdef PBA_CHECKED
  return 1;
#else
  return 0;
#endif
}
