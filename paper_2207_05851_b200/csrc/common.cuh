// Shared helpers for the sm_100a kernels of the translation hot path.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/skiff_b200.h"

namespace skb {

// ------------------------------------------------------------- error state
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);

#define SKB_CHECK_LAUNCH(what)                                                        \
  do {                                                                                \
    cudaError_t _e = cudaGetLastError();                                              \
    if (_e != cudaSuccess)                                                            \
      return ::skb::fail(SKB_ERR_LAUNCH, "%s: %s", what, cudaGetErrorString(_e));     \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------- programmatic dependent launch
// Every kernel of the decode step is launched with programmatic stream
// serialization: the next kernel's CTAs are scheduled while the current one
// drains, run their prologue (barrier init, TMEM alloc, descriptor and
// weight prefetch), and block in griddepcontrol.wait until the predecessor
// grid has completed and its writes are visible.  Kernels therefore touch no
// predecessor-produced memory before pdl_wait().  SKB_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define PDL_ENTRY()        \
  do {                     \
    ::skb::pdl_wait();     \
    ::skb::pdl_trigger();  \
  } while (0)

bool pdl_enabled();

// Raise a kernel's opt-in dynamic shared memory limit on the current device
// (idempotent, thread-safe, per device).
void ensure_smem(const void *kernel, size_t bytes);
template <typename F> inline void ensure_smem_fn(F *kernel, size_t bytes) {
  ensure_smem(reinterpret_cast<const void *>(kernel), bytes);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t stream, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------- element access
__device__ __forceinline__ float load_f(const void *p, int dtype, size_t i) {
  return dtype == SKB_F32 ? reinterpret_cast<const float *>(p)[i]
                          : __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i]);
}
__device__ __forceinline__ void store_f(void *p, int dtype, size_t i, float v) {
  if (dtype == SKB_F32)
    reinterpret_cast<float *>(p)[i] = v;
  else
    reinterpret_cast<__nv_bfloat16 *>(p)[i] = __float2bfloat16_rn(v);
}

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Logistic split on sign so exp never overflows (kernels.py:253-260):
// 1 / (1 + exp(-x)) for x >= 0, exp(x) / (1 + exp(x)) otherwise, written
// branch-free (exp(-|x|) is the exponential of either side, the sign picks
// the numerator) with the SFU exponential and division (relative error
// ~1e-6, far inside the 1e-4 fp32 parity bound; every kernel that needs a
// sigmoid calls this one, so all paths agree bit for bit).  The accurate
// expf + IEEE division cost ~6 us of a 7 us SSRU epilogue at M = 640
// (profiles/r2_67/68_trace_ssru.txt).
__device__ __forceinline__ float sigmoid_ref(float x) {
  const float e = __expf(-fabsf(x));
  return __fdividef(x >= 0.f ? 1.0f : e, 1.0f + e);
}

// SSRU cell (model.py:268-272): c = f * c_prev + (1 - f) * W h with
// f = sigmoid(W_f h + b_f); one definition for every epilogue path.
__device__ __forceinline__ float ssru_cell(float v, float bn, float w, float cp) {
  const float f = sigmoid_ref(v + bn);
  return f * cp + (1.0f - f) * w;
}

}  // namespace skb
