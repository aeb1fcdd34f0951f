// Which TMA issue structure reaches the SM's L2->SM ingest limit?  The
// 1-producer ring of tma_ingest.cu saturates at ~62 B/clk per CTA however
// deep the ring, while two CTAs per SM reach ~125 B/clk.  Variants (all
// CTAs stream SW128 boxes of an L2-resident bf16 matrix, 64 columns wide):
//   P producers (one lane of warp 2p each, own ring + barriers), a consumer
//   lane per producer (warp 2p+1); B boxes of R rows per stage; 1 or 2 tensor
//   maps; or 1D cp.async.bulk copies of the same byte count.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_ingest2 tools/micro/tma_ingest2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W;}" ::"r"(su32(b)),
               "r"(ph)
               : "memory");
}

struct Args {
  int P, B, R, stages, iters, rows, two_maps, bulk1d;
  const uint8_t *raw;
};

template <int P_, int B_, int R_, int ST_, int TWO_, int BULK_>
__global__ void __launch_bounds__(256, 1) k_ingest(const __grid_constant__ CUtensorMap tm0,
                                                   const __grid_constant__ CUtensorMap tm1, Args a) {
  a.P = P_; a.B = B_; a.R = R_; a.stages = ST_; a.two_maps = TWO_; a.bulk1d = BULK_; a.rows = 2048;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  const int box_bytes = a.R * 128, stage_bytes = a.B * box_bytes;
  const int ring = a.stages * stage_bytes;
  uint64_t *bars = (uint64_t *)(sm + a.P * ring);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * a.P * a.stages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int p = warp >> 1;
  if (p < a.P && lane == 0) {
    uint64_t *full = bars + 2 * p * a.stages, *empty = full + a.stages;
    uint8_t *base = sm + p * ring;
    const int nbr = a.rows / a.R;  // boxes along rows
    if ((warp & 1) == 0) {
      for (int it = 0; it < a.iters; ++it) {
        const int s = it % a.stages;
        if (it >= a.stages) mbar_wait(&empty[s], ((it / a.stages) & 1) ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes));
        for (int b = 0; b < a.B; ++b) {
          const int box = ((it * a.B + b) * 7 + blockIdx.x * 13 + p * 5) % (nbr * 16);
          const int c = (box % 16) * 64, r = (box / 16) * a.R;
          uint8_t *dst = base + s * stage_bytes + b * box_bytes;
          if (a.bulk1d) {
            const uint8_t *src = a.raw + ((size_t)r * 1024 + c) * 2;  // contiguous bytes of the same count
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(dst)),
                "l"(src), "r"(box_bytes), "r"(su32(&full[s]))
                : "memory");
          } else {
            const CUtensorMap *m = (a.two_maps && (b & 1)) ? &tm1 : &tm0;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    su32(dst)),
                "l"((uint64_t)m), "r"(c), "r"(r), "r"(su32(&full[s]))
                : "memory");
          }
        }
      }
    } else {
      for (int it = 0; it < a.iters; ++it) {
        const int s = it % a.stages;
        mbar_wait(&full[s], (it / a.stages) & 1);
        asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      }
    }
  }
  __syncthreads();
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                          const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 2048, cols = 1024;  // 4 MB bf16 per map: L2 resident
  uint8_t *buf;
  cudaMalloc(&buf, (size_t)2 * rows * cols * 2);
  cudaMemset(buf, 0, (size_t)2 * rows * cols * 2);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  typedef void (*KF)(CUtensorMap, CUtensorMap, Args);
  struct V {
    const char *name;
    int per_sm, P, B, R, stages, two_maps, bulk1d;
    KF k;
  } vs[] = {
      {"base 1 prod, 128-row box, 6 st", 1, 1, 1, 128, 6, 0, 0, k_ingest<1,1,128,6,0,0>},
      {"2 producers x 3 st", 1, 2, 1, 128, 3, 0, 0, k_ingest<2,1,128,3,0,0>},
      {"4 producers x 2 st", 1, 4, 1, 128, 2, 0, 0, k_ingest<4,1,128,2,0,0>},
      {"4 producers x 3 st", 1, 4, 1, 128, 3, 0, 0, k_ingest<4,1,128,3,0,0>},
      {"1 prod, 2 boxes/stage, 6 st", 1, 1, 2, 128, 6, 0, 0, k_ingest<1,2,128,6,0,0>},
      {"1 prod, 2 boxes/stage 2 maps", 1, 1, 2, 128, 6, 1, 0, k_ingest<1,2,128,6,1,0>},
      {"1 prod, 4x64-row boxes/stage", 1, 1, 4, 64, 6, 0, 0, k_ingest<1,4,64,6,0,0>},
      {"1 prod, 256-row box, 3 st", 1, 1, 1, 256, 3, 0, 0, k_ingest<1,1,256,3,0,0>},
      {"1 prod, 256-row box, 6 st", 1, 1, 1, 256, 6, 0, 0, k_ingest<1,1,256,6,0,0>},
      {"1 prod, 1D bulk 16KB, 6 st", 1, 1, 1, 128, 6, 0, 1, k_ingest<1,1,128,6,0,1>},
      {"1 prod, 1D bulk 2x16KB, 6 st", 1, 1, 2, 128, 6, 0, 1, k_ingest<1,2,128,6,0,1>},
      {"2 CTA/SM base 6 st", 2, 1, 1, 128, 6, 0, 0, k_ingest<1,1,128,6,0,0>},
      {"2 CTA/SM 2 prod x 3 st", 2, 2, 1, 128, 3, 0, 0, k_ingest<2,1,128,3,0,0>},
  };
  for (int active : {nsm, 40}) {
    for (auto &v : vs) {
      const int box_bytes = v.R * 128, ring = v.stages * v.B * box_bytes;
      const int smem = v.P * ring + 2 * v.P * v.stages * 8 + 1024;
      if (smem * v.per_sm > 228 * 1024) {
        printf("%-34s: skip (smem %d)\n", v.name, smem);
        continue;
      }
      CUtensorMap tm[2];
      for (int i = 0; i < 2; ++i) {
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)v.R}, es[2] = {1, 1};
        enc(&tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf + (size_t)i * rows * cols * 2, dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      const int grid = active * v.per_sm;
      const int iters = 2000 * 16384 / (v.B * box_bytes);
      Args a{v.P, v.B, v.R, v.stages, 500, rows, v.two_maps, v.bulk1d, buf};
      cudaFuncSetAttribute(v.k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      for (int w = 0; w < 20; ++w) v.k<<<grid, 256, smem>>>(tm[0], tm[1], a);  // clocks up
      a.iters = iters;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      v.k<<<grid, 256, smem>>>(tm[0], tm[1], a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)grid * v.P * iters * v.B * box_bytes;
      printf("SMs %3d %-34s: %8.1f GB/s total, %6.1f GB/s per SM, %6.1f B/clk/SM  (%s)\n", active, v.name,
             bytes / ms / 1e6, bytes / ms / 1e6 / active, bytes / ms / 1e6 / active / 1.965,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
