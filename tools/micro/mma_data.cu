// Data dependence of tcgen05.mma issue cost (fill 0 = zero operands, 1 = random bf16).
// Issue cost of tcgen05.mma (kind::f16, cta_group::1, M=128, N=NA, K=16)
// from one thread, with and without a tcgen05.commit per 4 MMAs (one
// k-block of the GEMM ring).  One CTA, operands in (zeroed) shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_issue mma_issue.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(const void *p) {
  uint64_t a = su32(p), d = 0;
  d |= (a >> 4) & 0x3FFFull; d |= 1ull << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= 1ull << 46; d |= 2ull << 61;
  return d;
}
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(t), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(bar)), "r"(ph) : "memory");
}
template <int NA>
__global__ void k(long long *out, int mode, int nmma, int fill) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    // fill 0: zeros; 1: random bf16 pairs in (-1, 1) (sign, exponent 0x70..0x7e, random mantissa)
    const uint32_t lo = (h & 0x807fu) | ((0x70u + (h >> 7) % 15u) << 7);
    const uint32_t hi = ((h >> 16) & 0x807fu) | ((0x70u + (h >> 23) % 15u) << 7);
    reinterpret_cast<uint32_t *>(sm)[i] = fill ? (lo | (hi << 16)) : 0u;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[1])), "r"(mode >= 3 ? mode - 1 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  const int issuers = mode >= 3 ? mode - 1 : 1;  // mode 3: 2 issuing warps, 4: 3 warps
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < issuers) {
    const int w = threadIdx.x >> 5;
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NA >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc(sm), db = desc(sm + 16384);
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int i = 0; i < nmma; i += 4) {
      if (mode >= 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 4; ++k) mma(tm + w * NA, da + 2 * k, db + 2 * k, id, (i | k) ? 1u : 0u);
      if (mode == 1 || mode == 2) commit(&bar[0]);
    }
    long long t1 = clock64();
    commit(&bar[1]);
    if (w == 0) {
      wait(&bar[1], 0);
      long long t2 = clock64();
      out[0] = t1 - t0;  // issue
      out[1] = t2 - t0;  // issue + completion
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}
int main() {
  long long *o; cudaMalloc(&o, 64);
  cudaFuncSetAttribute(k<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
  cudaFuncSetAttribute(k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
  cudaFuncSetAttribute(k<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
  for (int fill = 0; fill < 2; ++fill)
  for (int na : {32, 64, 128})
    for (int mode = 0; mode < 3; mode += 2) {
      long long h[2];
      for (int rep = 0; rep < 2; ++rep) {
        if (na == 32) k<32><<<1, 128, 49152>>>(o, mode, 64, fill);
        if (na == 64) k<64><<<1, 128, 49152>>>(o, mode, 64, fill);
        if (na == 128) k<128><<<1, 128, 49152>>>(o, mode, 64, fill);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      const int iss = mode >= 3 ? mode - 1 : 1;
      printf("fill=%d N=%3d mode=%d issuers=%d: %d MMAs issue %lld cyc, done %lld cyc (%.1f cyc/MMA)\n", fill, na, mode, iss, 64 * iss, h[0], h[1], h[1] / (64.0 * iss));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
