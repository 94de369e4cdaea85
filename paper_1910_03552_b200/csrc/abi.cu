// C-ABI glue: version, thread-local error message, launch checking.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace bp {

static thread_local char g_err[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);  // every kernel launch is followed by one check
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace bp

extern "C" int bp_abi_version(void) { return 1; }
extern "C" const char* bp_last_error(void) { return bp::g_err; }
extern "C" unsigned long long bp_launch_count(void) { return bp::g_launches.load(); }
