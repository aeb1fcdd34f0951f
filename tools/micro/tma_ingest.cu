// L2 -> SM ingest rate of TMA tile loads (the bound of the decode GEMMs'
// mainloop): every CTA streams 128x64 bf16 SW128 boxes (16 KB, the GEMM's
// weight k-block) of an L2-resident matrix through an S-stage smem ring; a
// consumer thread releases each stage as soon as it lands.  Reports bytes
// per SM per clock for 1 and 2 CTAs per SM and several ring depths.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_ingest tools/micro/tma_ingest.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  asm volatile(
      "{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}

__global__ void __launch_bounds__(64, 1) k_ingest(const __grid_constant__ CUtensorMap tm, int rows,
                                                   int iters, int stages, unsigned long long *clk) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(sm + stages * 16384);
  uint64_t *empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nbox_r = rows / 128;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (it >= stages) mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                   "r"(16384));
      const int box = (it * 7 + blockIdx.x * 13) % (nbox_r * 16);
      const int c = (box % 16) * 64, r = (box / 16) * 128;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              su32(sm + s * 16384)),
          "l"((uint64_t)&tm), "r"(c), "r"(r), "r"(su32(&full[s]))
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                          const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

int main() {
  const int rows = 2048, cols = 1024;  // 4 MB bf16: L2 resident
  void *buf;
  cudaMalloc(&buf, (size_t)rows * cols * 2);
  cudaMemset(buf, 0, (size_t)rows * cols * 2);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncFn enc = (EncFn)p;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *clk;
  cudaMalloc(&clk, 4096 * 8);
  cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const int iters = 2000;
  for (int active : {nsm, 40, 8})
  for (int per_sm = 1; per_sm <= 4; ++per_sm)
    for (int stages : {2, 4, 6, 8, 12}) {
      if (stages * per_sm > 13) continue;
      if (active != nsm && per_sm > 2) continue;
      const int smem = stages * 16384 + 2048;
      const int grid = active * per_sm;
      k_ingest<<<grid, 64, smem>>>(tm, rows, 50, stages, clk);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k_ingest<<<grid, 64, smem>>>(tm, rows, iters, stages, clk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)grid * iters * 16384;
      printf("SMs %3d ctas/SM %d stages %2d: %.1f GB/s total, %.1f GB/s per SM, %.1f B/clk/SM @1.965GHz  (%s)\n",
             active, per_sm, stages, bytes / ms / 1e6, bytes / ms / 1e6 / active,
             bytes / ms / 1e6 / active / 1.965, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
