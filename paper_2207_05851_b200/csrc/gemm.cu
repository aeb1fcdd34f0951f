// GEMMs of the decode path: C[M,N] = A[M,K] . W[N,K]^T with fused epilogues.
//
// Replaces skiff kernels.py:479-484 (linear) and 167-195 (matmul).  The
// reference accumulates every product in float64 (kernels.py:167-176); here
//   * bf16 operands go through a tcgen05 kernel: TMA (128B swizzle) ->
//     shared memory ring (mbarrier full/empty pipeline) -> tcgen05.mma
//     kind::f16 issued by one thread -> fp32 accumulator in TMEM ->
//     tcgen05.ld epilogue (bias / ReLU / residual add / SSRU cell);
//   * fp32 operands (the parity mode) go through a SIMT FFMA kernel with the
//     same epilogues and a fixed K order (batch-composition invariant).
// Both kernels reduce K in the same order for every M, so a row's result
// never depends on the other rows of the batch (search.py batch invariance,
// test_search.py:400-405).

#include "common.cuh"

#include <mutex>
#include <unordered_map>

namespace skb {

// ================================================================ epilogue
struct EpiArgs {
  int kind;
  const float *bias;
  void *out;
  int ldo;
  int out_dtype;
  const float *c_prev;
  float *c_next;
  const int *src_row;
  int ld_state;
  const int *step;
  long long state_stride;
  float *lse_part;
  int lse_ld;
  const unsigned *mask;
  int mask_words;
  int rows_per_group;
};

// Partial log-softmax statistics of `cnt` consecutive logits of row m
// starting at column n (a 32-column group): (max, sum exp(x - max)) over the
// row's active columns.  Empty groups give (-inf, 0).
__device__ __forceinline__ float2 group_stats(const EpiArgs &e, int m, int n, int N,
                                              const float *v, int cnt) {
  const unsigned *mrow = e.mask ? e.mask + (size_t)(m / e.rows_per_group) * e.mask_words : nullptr;
  float mx = -INFINITY;
  for (int q = 0; q < cnt; ++q) {
    const int c = n + q;
    if (c < N && (!mrow || ((mrow[c >> 5] >> (c & 31)) & 1u))) mx = fmaxf(mx, v[q]);
  }
  float s = 0.f;
  if (mx != -INFINITY)
    for (int q = 0; q < cnt; ++q) {
      const int c = n + q;
      if (c < N && (!mrow || ((mrow[c >> 5] >> (c & 31)) & 1u))) s += expf(v[q] - mx);
    }
  return make_float2(mx, s);
}

// Apply the epilogue to `cnt` consecutive accumulator columns n..n+cnt-1 of
// row m (cnt even, n even for SSRU).  v holds the raw fp32 accumulators.
__device__ __forceinline__ void epilogue_run(const EpiArgs &e, int m, int n, int N, float *v,
                                             int cnt) {
  if (e.kind == SKB_EPI_SSRU) {
    // columns (2j, 2j+1) = (W_f h, W h) for cell column j (model.py:268-272):
    // f = sigmoid(W_f h + b_f); c = f*c_prev + (1-f)*(W h); x += relu(c)
    float *x = reinterpret_cast<float *>(e.out);
    const int srow = e.src_row ? e.src_row[m] : m;
    const float *cprev = e.c_prev;
    float *cnext = e.c_next;
    if (e.step) {  // decode-loop double buffer selected by step parity
      const int t = *e.step;
      cnext = e.c_next + (t & 1) * e.state_stride;
      cprev = t == 0 ? nullptr : e.c_next + ((t + 1) & 1) * e.state_stride;
    }
    for (int q = 0; q + 1 < cnt; q += 2) {
      const int nn = n + q;
      if (nn >= N) break;
      const int j = nn >> 1;
      float fpre = v[q] + (e.bias ? e.bias[nn] : 0.f);
      float f = sigmoid_ref(fpre);
      float cp = cprev ? cprev[(size_t)srow * e.ld_state + j] : 0.f;
      float c = f * cp + (1.0f - f) * v[q + 1];
      cnext[(size_t)m * e.ld_state + j] = c;
      float *xp = x + (size_t)m * e.ldo + j;
      *xp = *xp + fmaxf(c, 0.f);
    }
    return;
  }
  if (e.kind == SKB_EPI_RESID) {
    float *x = reinterpret_cast<float *>(e.out) + (size_t)m * e.ldo;
    for (int q = 0; q < cnt; ++q) {
      const int nn = n + q;
      if (nn >= N) break;
      float t = v[q] + (e.bias ? e.bias[nn] : 0.f);
      x[nn] = x[nn] + t;
    }
    return;
  }
  const bool relu = e.kind == SKB_EPI_RELU;
  if (e.out_dtype == SKB_F32 || e.kind == SKB_EPI_LOGITS) {
    float *o = reinterpret_cast<float *>(e.out) + (size_t)m * e.ldo;
    for (int q = 0; q < cnt; ++q) {
      const int nn = n + q;
      if (nn >= N) break;
      float t = v[q] + (e.bias ? e.bias[nn] : 0.f);
      o[nn] = relu ? fmaxf(t, 0.f) : t;
    }
  } else {
    __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(e.out) + (size_t)m * e.ldo;
    for (int q = 0; q < cnt; ++q) {
      const int nn = n + q;
      if (nn >= N) break;
      float t = v[q] + (e.bias ? e.bias[nn] : 0.f);
      o[nn] = __float2bfloat16_rn(relu ? fmaxf(t, 0.f) : t);
    }
  }
}

// Vectorised fast path for a full 32-column chunk (STORE/RELU/RESID), used by
// the tcgen05 epilogue when the chunk is in-bounds and 16-byte aligned.
__device__ __forceinline__ bool epilogue_vec32(const EpiArgs &e, int m, int n, float *v) {
  if (e.kind == SKB_EPI_SSRU) return false;
  if (e.kind == SKB_EPI_LOGITS) {
    float4 *o = reinterpret_cast<float4 *>(reinterpret_cast<float *>(e.out) +
                                           (size_t)m * e.ldo + n);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return true;
  }
  if (e.bias) {
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] += __ldg(e.bias + n + q);
  }
  if (e.kind == SKB_EPI_RESID) {
    float4 *x = reinterpret_cast<float4 *>(reinterpret_cast<float *>(e.out) +
                                           (size_t)m * e.ldo + n);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 a = x[q];
      a.x += v[4 * q]; a.y += v[4 * q + 1]; a.z += v[4 * q + 2]; a.w += v[4 * q + 3];
      x[q] = a;
    }
    return true;
  }
  if (e.kind == SKB_EPI_RELU) {
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = fmaxf(v[q], 0.f);
  }
  if (e.out_dtype == SKB_F32) {
    float4 *o = reinterpret_cast<float4 *>(reinterpret_cast<float *>(e.out) +
                                           (size_t)m * e.ldo + n);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
    uint4 *o = reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(e.out) +
                                         (size_t)m * e.ldo + n);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        __nv_bfloat162 p = __floats2bfloat162_rn(v[8 * q + 2 * h], v[8 * q + 2 * h + 1]);
        w[h] = *reinterpret_cast<uint32_t *>(&p);
      }
      o[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  return true;
}

// ======================================================== tcgen05 kernel
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle atom row

template <int BN> struct Cfg {
  static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 128 ? 5 : 6);
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// SM100 UMMA shared-memory descriptor: K-major operand, 128-byte swizzle,
// 8-row core-matrix groups 1024 B apart (SBO), version 1, layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void *smem_tile) {
  const uint64_t addr = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address  [0,14)
  d |= (uint64_t)1 << 16;                // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;      // SBO            [32,46)
  d |= (uint64_t)1 << 46;                // version = 1    [46,48)
  d |= (uint64_t)2 << 61;                // SWIZZLE_128B   [61,64)
  return d;
}

// Instruction descriptor, kind::f16: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4)                      // c_format = F32
         | (1u << 7)                    // a_format = BF16
         | (1u << 10)                   // b_format = BF16
         | ((uint32_t)(N >> 3) << 17)   // n_dim
         | ((uint32_t)(M >> 4) << 24);  // m_dim
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN>
__global__ void __launch_bounds__(128, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              int M, int N, int K, EpiArgs ep) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + C::STAGES;
  uint64_t *done = empty + C::STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      const uint32_t ph = (kb / C::STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t *sa = smem + s * C::STAGE_BYTES;
      mbar_expect_tx(&full[s], C::STAGE_BYTES);
      tma_load_2d(sa, &tmA, kb * BK, m0, &full[s]);
      tma_load_2d(sa + C::A_BYTES, &tmB, kb * BK, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread)
    constexpr uint32_t idesc = idesc_bf16(BM, BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::STAGES;
      const uint32_t ph = (kb / C::STAGES) & 1;
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t *sa = smem + s * C::STAGE_BYTES;
      const uint64_t da = umma_desc_sw128(sa);
      const uint64_t db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
      for (int k = 0; k < BK / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
        umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();

  // ---- epilogue: warp w owns TMEM lanes [32w, 32w+32) = tile rows
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  const bool vec_ok = ep.kind != SKB_EPI_SSRU && (ep.ldo % 8 == 0) &&
                      ((reinterpret_cast<uintptr_t>(ep.out) & 15) == 0);
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
    const int n = n0 + c;
    if (row < M && n < N) {
      if (ep.kind == SKB_EPI_LOGITS)
        reinterpret_cast<float2 *>(ep.lse_part)[(size_t)row * ep.lse_ld + (n >> 5)] =
            group_stats(ep, row, n, N, v, 32);
      if (!(vec_ok && n + 32 <= N && epilogue_vec32(ep, row, n, v)))
        epilogue_run(ep, row, n, N, v, 32);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

// ---------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void *ptr;
  int rows, cols, ld, box_rows;
  bool operator==(const MapKey &o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey &k) const {
    size_t h = reinterpret_cast<size_t>(k.ptr);
    h = h * 1000003u ^ (size_t)k.rows;
    h = h * 1000003u ^ (size_t)k.cols;
    h = h * 1000003u ^ (size_t)k.ld;
    return h * 1000003u ^ (size_t)k.box_rows;
  }
};

// Tensor maps are host-side descriptors; cache them per (pointer, shape) so
// steady-state calls (and CUDA-graph capture) cost no re-encoding.
static int make_map(CUtensorMap *out, const void *ptr, int rows, int cols, int ld, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, rows, cols, ld, box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return SKB_OK;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SKB_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SKB_ERR_LAUNCH, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return SKB_OK;
}

template <int BN>
static int launch(int M, int N, int K, const void *A, int lda, const void *W, int ldw,
                  const EpiArgs &ep, cudaStream_t st) {
  using C = Cfg<BN>;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, BM);
  if (rc) return rc;
  rc = make_map(&mb, W, N, K, ldw, BN);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr_set = true;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  k_gemm_tc<BN><<<grid, 128, C::SMEM, st>>>(ma, mb, M, N, K, ep);
  SKB_CHECK_LAUNCH("k_gemm_tc");
  return SKB_OK;
}

}  // namespace tc

// ========================================================== SIMT kernel
// 64x64 output tile, BK=16, 256 threads, 4x4 outputs per thread.  Used for
// fp32 (parity) mode and for shapes TMA cannot describe.
template <typename T>
__global__ void __launch_bounds__(256) k_gemm_simt(int M, int N, int K, const T *__restrict__ A,
                                                   int lda, const T *__restrict__ W, int ldw,
                                                   EpiArgs ep) {
  constexpr int TM = 64, TN = 64, TK = 16;
  __shared__ float As[TK][TM + 4];
  __shared__ float Ws[TK][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    // load 64x16 of A and 64x16 of W (4 elements per thread each)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * 256;
      const int r = idx / TK, kk = idx % TK;
      const int gm = m0 + r, gn = n0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? to_f(A[(size_t)gm * lda + gk]) : 0.f;
      Ws[kk][r] = (gn < N && gk < K) ? to_f(W[(size_t)gn * ldw + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (ep.kind == SKB_EPI_LOGITS) {
      // group = 8 consecutive tx (32 columns); combine the 8 (max, sum) pairs
      float2 st = m < M ? group_stats(ep, m, n0 + tx * 4, N, acc[i], 4)
                        : make_float2(-INFINITY, 0.f);
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, st.x, o);
        const float os = __shfl_xor_sync(0xffffffffu, st.y, o);
        const float nm = fmaxf(st.x, om);
        float ns = 0.f;
        if (nm != -INFINITY) ns = st.y * expf(st.x - nm) + os * expf(om - nm);
        st = make_float2(nm, ns);
      }
      const int n = n0 + tx * 4;
      if (m < M && (tx & 7) == 0 && n < N)
        reinterpret_cast<float2 *>(ep.lse_part)[(size_t)m * ep.lse_ld + (n >> 5)] = st;
    }
    if (m < M) epilogue_run(ep, m, n0 + tx * 4, N, acc[i], 4);
  }
}

static EpiArgs to_args(const skb_epilogue *e) {
  EpiArgs a;
  a.kind = e->kind;
  a.bias = e->bias;
  a.out = e->out;
  a.ldo = e->ldo;
  a.out_dtype = e->out_dtype;
  a.c_prev = e->c_prev;
  a.c_next = e->c_next;
  a.src_row = e->src_row;
  a.ld_state = e->ld_state;
  a.step = e->step;
  a.state_stride = e->state_stride;
  a.lse_part = e->lse_part;
  a.lse_ld = e->lse_ld;
  a.mask = e->mask;
  a.mask_words = e->mask_words;
  a.rows_per_group = e->rows_per_group > 0 ? e->rows_per_group : 1;
  return a;
}

static int check_args(int in_dtype, int M, int N, int K, const void *A, const void *W,
                      const skb_epilogue *epi) {
  if (M < 0 || N <= 0 || K <= 0) return fail(SKB_ERR_SHAPE, "gemm: bad shape M=%d N=%d K=%d", M, N, K);
  if (!A || !W || !epi || !epi->out) return fail(SKB_ERR_SHAPE, "gemm: null operand");
  if (in_dtype != SKB_F32 && in_dtype != SKB_BF16) return fail(SKB_ERR_CONFIG, "gemm: dtype");
  if ((epi->kind == SKB_EPI_RESID || epi->kind == SKB_EPI_SSRU) && epi->out_dtype != SKB_F32)
    return fail(SKB_ERR_CONFIG, "gemm: residual/SSRU target must be fp32");
  if (epi->kind == SKB_EPI_SSRU && (N % 2 != 0 || !epi->c_next))
    return fail(SKB_ERR_CONFIG, "gemm: SSRU needs even N and a cell buffer");
  if (epi->kind == SKB_EPI_LOGITS && (!epi->lse_part || epi->lse_ld < (N + 31) / 32 ||
                                      epi->out_dtype != SKB_F32))
    return fail(SKB_ERR_CONFIG, "gemm: LOGITS needs fp32 out and a partials buffer");
  return SKB_OK;
}

static int gemm_simt(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
                     int ldw, const EpiArgs &ep, cudaStream_t st) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  if (in_dtype == SKB_F32)
    k_gemm_simt<float><<<grid, 256, 0, st>>>(M, N, K, (const float *)A, lda, (const float *)W, ldw, ep);
  else
    k_gemm_simt<__nv_bfloat16><<<grid, 256, 0, st>>>(M, N, K, (const __nv_bfloat16 *)A, lda,
                                                     (const __nv_bfloat16 *)W, ldw, ep);
  SKB_CHECK_LAUNCH("k_gemm_simt");
  return SKB_OK;
}

}  // namespace skb

using namespace skb;

extern "C" int skb_tc_available(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0 && tc::encode_fn() != nullptr) ? 1 : 0;
}

extern "C" int skb_gemm_simt(int in_dtype, int M, int N, int K, const void *A, int lda,
                             const void *W, int ldw, const skb_epilogue *epi, void *stream) {
  int rc = check_args(in_dtype, M, N, K, A, W, epi);
  if (rc) return rc;
  if (M == 0) return SKB_OK;
  return gemm_simt(in_dtype, M, N, K, A, lda, W, ldw, to_args(epi), as_stream(stream));
}

extern "C" int skb_gemm(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
                        int ldw, const skb_epilogue *epi, void *stream) {
  int rc = check_args(in_dtype, M, N, K, A, W, epi);
  if (rc) return rc;
  if (M == 0) return SKB_OK;
  EpiArgs ep = to_args(epi);
  cudaStream_t st = as_stream(stream);
  const bool tma_ok = in_dtype == SKB_BF16 && K % 8 == 0 && lda % 8 == 0 && ldw % 8 == 0 &&
                      (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  if (!tma_ok) return gemm_simt(in_dtype, M, N, K, A, lda, W, ldw, ep, st);
  // Tile width: the widest N tile that still fills the 148 SMs.
  const long mt = (M + tc::BM - 1) / tc::BM;
  if (N >= 4096 && mt * ((N + 255) / 256) >= 148) return tc::launch<256>(M, N, K, A, lda, W, ldw, ep, st);
  if (mt * ((N + 127) / 128) >= 148) return tc::launch<128>(M, N, K, A, lda, W, ldw, ep, st);
  return tc::launch<64>(M, N, K, A, lda, W, ldw, ep, st);
}
