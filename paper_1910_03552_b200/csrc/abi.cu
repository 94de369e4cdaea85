// C-ABI glue: version, thread-local error message, launch checking.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace bp {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

}  // namespace bp

extern "C" int bp_abi_version(void) { return 1; }
extern "C" const char* bp_last_error(void) { return bp::g_err; }
