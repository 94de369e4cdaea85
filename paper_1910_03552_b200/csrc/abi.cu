// C-ABI glue: version, thread-local error message, launch checking.
#include <atomic>
#include <chrono>
#include <thread>
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

// Host-side wait on a completion word in pinned memory (a device kernel publishes it through the
// unified-address mapping, e.g. bp_pack_stats' seq word): spins until (*word - want) mod 2^32 is
// below 2^31, yielding the core every 1024 polls.  Called through ctypes it runs without the
// Python GIL.  Returns 0 when reached, 1 after timeout_us.
extern "C" int bp_host_wait_seq(const unsigned* word, unsigned want, long long timeout_us) {
  const volatile unsigned* w = word;
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned long long i = 0;; ++i) {
    if ((unsigned)(*w - want) < 0x80000000u) {
      std::atomic_thread_fence(std::memory_order_acquire);
      return 0;
    }
    if ((i & 1023) == 1023) {
      if (std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >
          timeout_us)
        return 1;
      std::this_thread::yield();
    }
  }
}

// Several device copies in one call (the inference graph path's input staging): dsts[i] <-
// srcs[i], bytes[i], asynchronously on `stream` (device-to-device or pinned host).
extern "C" int bp_copy_many(void* const* dsts, const void* const* srcs, const size_t* bytes, int n, void* stream) {
  for (int i = 0; i < n; ++i) {
    if (!bytes[i]) continue;
    if (cudaMemcpyAsync(dsts[i], srcs[i], bytes[i], cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess) {
      bp::set_error("bp_copy_many: copy %d failed: %s", i, cudaGetErrorString(cudaGetLastError()));
      return BP_ERR_LAUNCH;
    }
  }
  return BP_OK;
}
