// Thread-local error message + status plumbing for the C ABI.
#include "common.cuh"

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace skb {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SKB_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// Opt-in dynamic shared memory is a per-(kernel, device) attribute: raise it
// once per device the kernel runs on (several devices may share a process).
void ensure_smem(const void *kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  size_t &cur = done[{kernel, dev}];
  if (bytes > cur) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cur = bytes;
  }
}

}  // namespace skb

extern "C" const char *skb_version(void) { return "skiff_b200 0.1 sm_100a"; }
extern "C" const char *skb_last_error(void) { return skb::g_err; }
