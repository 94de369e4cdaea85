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

// Several copies in one call (the inference graph path's input staging): dsts[i] <- srcs[i],
// bytes[i], on `stream`, as ONE kernel launch (device or mapped pinned memory; 16-byte pieces
// when both ends allow it), instead of one driver copy per buffer.
namespace {
constexpr int kMaxCopies = 8;
struct CopyList {
  void* dst[kMaxCopies];
  const void* src[kMaxCopies];
  size_t bytes[kMaxCopies];
  int n;
};
__global__ void copy_many_kernel(const __grid_constant__ CopyList L) {
  for (int c = 0; c < L.n; ++c) {
    const size_t nb = L.bytes[c];
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(L.dst[c]) | reinterpret_cast<uintptr_t>(L.src[c]) | nb) & 15u) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(L.src[c]);
      uint4* d4 = reinterpret_cast<uint4*>(L.dst[c]);
      for (size_t i = i0; i < nb / 16; i += st) d4[i] = s4[i];
    } else {
      const uint8_t* s1 = reinterpret_cast<const uint8_t*>(L.src[c]);
      uint8_t* d1 = reinterpret_cast<uint8_t*>(L.dst[c]);
      for (size_t i = i0; i < nb; i += st) d1[i] = s1[i];
    }
  }
}
}  // namespace

extern "C" int bp_copy_many(void* const* dsts, const void* const* srcs, const size_t* bytes, int n, void* stream) {
  if (n < 0 || n > kMaxCopies) {
    bp::set_error("bp_copy_many: 0 <= n <= %d", kMaxCopies);
    return BP_ERR_ARG;
  }
  CopyList L;
  size_t total = 0;
  for (int i = 0; i < n; ++i) {
    L.dst[i] = dsts[i];
    L.src[i] = srcs[i];
    L.bytes[i] = bytes[i];
    total += bytes[i];
  }
  L.n = n;
  if (total == 0) return BP_OK;
  size_t blocks = (total / 16 + 255) / 256;
  blocks = blocks < 1 ? 1 : blocks > 296 ? 296 : blocks;
  copy_many_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(L);
  return bp::check_launch("copy_many_kernel");
}
