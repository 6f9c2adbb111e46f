// ABI housekeeping: version, thread-local error text, device properties.
#include "common.cuh"

#include <atomic>

namespace la {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// per-device SM count, cached: written once per device with the same
// value by any racing thread (relaxed atomics, no lock needed)
int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (dev < 0 || dev >= 64) return -1;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

}  // namespace la

extern "C" {

int la_abi_version(void) { return LA_ABI_VERSION; }

const char* la_last_error(void) { return la::g_err; }

int la_device_sm_count(void) { return la::sm_count(); }

}  // extern "C"
