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

#include <cstdlib>
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
  // split-K (set by the launcher)
  int splits;
  float *ws;
  unsigned *counters;
  // fused LayerNorm of the residual rows (RESID, swap-AB kernel)
  const float *ln_gain;
  const float *ln_bias;
  float ln_eps;
  __nv_bfloat16 *ln_out;
  int ln_ldo;
  unsigned *ln_counter;
  // LayerNorm of the input rows computed in the swap-AB kernel's prologue
  const float *lnx;
  int lnx_ld;
  const float *lnx_g;
  const float *lnx_b;
  float lnx_eps;
  int late_trigger;  // swap-AB kernel: release dependents once the accumulator is ready
  // int8 GEMM (skb_gemm_i8): per-row scales of the int8 activations [M] and
  // weights [N]; out = (f32(acc) * a_scale[m]) * w_scale[n] (+bias ...)
  const float *a_scale;
  const float *w_scale;
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
      float cp = cprev ? cprev[(size_t)srow * e.ld_state + j] : 0.f;
      float c = ssru_cell(v[q], e.bias ? e.bias[nn] : 0.f, v[q + 1], cp);
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
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;  // per accumulator (2 allocated)
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

// Instruction descriptor, kind::i8: s8 x s8 -> s32, both K-major.
__host__ __device__ constexpr uint32_t idesc_s8(int M, int N) {
  return (2u << 4)                      // c_format = S32
         | (1u << 7)                    // a_format = signed 8-bit
         | (1u << 10)                   // b_format = signed 8-bit
         | ((uint32_t)(N >> 3) << 17)   // n_dim
         | ((uint32_t)(M >> 4) << 24);  // m_dim
}

// K = 32 int8 per instruction: the same 32-byte step through the SW128 atom
// as K = 16 bf16, so the smem pipeline is byte-for-byte the bf16 one.
__device__ __forceinline__ void umma_s8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
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

__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, int c0, int c1,
                                               uint64_t *bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Fast partial log-softmax statistics for the tcgen05 epilogue (bf16 mode):
// same as group_stats but with the SFU exponential (ex2.approx); the
// resulting log-sum-exp differs from expf's by < 1e-6 relative.
__device__ __forceinline__ float2 group_stats_fast(const EpiArgs &e, int m, int n, int N,
                                                   const float *v) {
  const unsigned *mrow = e.mask ? e.mask + (size_t)(m / e.rows_per_group) * e.mask_words : nullptr;
  unsigned bits = 0xffffffffu;
  if (mrow) bits = mrow[n >> 5];
  if (n + 32 > N) bits &= (N - n) >= 32 ? 0xffffffffu : ((1u << (N - n)) - 1u);
  float mx = -INFINITY;
#pragma unroll
  for (int q = 0; q < 32; ++q)
    if ((bits >> q) & 1u) mx = fmaxf(mx, v[q]);
  float s = 0.f;
  if (mx != -INFINITY) {
    const float ml = mx * 1.4426950408889634f;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if ((bits >> q) & 1u) s += exp2f(fmaf(v[q], 1.4426950408889634f, -ml));
  }
  return make_float2(mx, s);
}

// Persistent, warp-specialised tcgen05 GEMM.
// With CS > 1 the CTAs run as clusters of CS along N: the CS CTAs of a
// cluster work on the same M tile (CS adjacent N tiles) and each loads only
// BM/CS rows of every A (activation) k-block, multicast by TMA into all CS
// CTAs' shared memory — A's L2->SM traffic drops CS-fold.  A stage is
// refilled only after every CTA of the cluster has released it (the MMA
// commit arrives on all CS empty barriers).
//   warp 0      : TMA producer (one elected lane) over all tiles of this CTA
//   warp 1      : MMA issuer (one lane): K loop into one of two TMEM
//                 accumulators, tcgen05.commit -> smem slot free / tile done
//   warps 2..5  : epilogue (TMEM lane quarter = warp % 4), overlapping the
//                 next tile's MMA thanks to the second accumulator
// Tiles are visited M-fastest so the CTAs working at the same time share the
// weight (B) tile: each weight byte comes from HBM once, the small
// activation matrix stays L2-resident.
template <int BN, int CS>
__global__ void __launch_bounds__(192, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              int M, int N, int K, EpiArgs ep) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + C::STAGES;
  uint64_t *tfull = empty + C::STAGES;   // [2] accumulator ready
  uint64_t *tempty = tfull + 2;          // [2] accumulator drained
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (M + BM - 1) / BM;
  const int num_tiles = mt * ((N + BN - 1) / BN);
  const int nk = (K + BK - 1) / BK;
  const int S = CS > 1 ? 1 : ep.splits;
  const int kps = (nk + S - 1) / S;  // k-blocks per split
  const int nt = (N + BN - 1) / BN;
  const int num_units = CS > 1 ? ((nt + CS - 1) / CS) * mt : num_tiles * S;
  const int rank = CS > 1 ? (int)cluster_rank() : 0;
  const int u_first = CS > 1 ? (int)blockIdx.x / CS : (int)blockIdx.x;
  const int u_step = CS > 1 ? (int)gridDim.x / CS : (int)gridDim.x;
  constexpr uint16_t CMASK = (uint16_t)((1u << CS) - 1u);
  constexpr int A_SLICE = BM / CS;  // rows of each A k-block this CTA loads
  __shared__ int last_flag[2];
  (void)num_tiles;
  // unit u -> (tile, split): M fastest, then split, then N, so concurrently
  // running CTAs share both the weight tile and its K slice.  In cluster
  // mode a unit is (M tile, group of CS N tiles); this CTA takes N tile
  // group*CS + rank.
  auto decode = [&](int u, int &m0, int &n0, int &tile, int &split, int &kb0, int &kb1) {
    const int mb = u % mt;
    const int rest = u / mt;
    int nb;
    if (CS > 1) {
      split = 0;
      nb = rest * CS + rank;
    } else {
      split = rest % S;
      nb = rest / S;
    }
    m0 = mb * BM;
    n0 = nb * BN;
    tile = nb * mt + mb;
    kb0 = split * kps;
    kb1 = min(nk, kb0 + kps);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);  // every CTA of the cluster releases the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (CS > 1) cluster_sync_all();  // peers' barriers exist before any multicast

  if (warp == 0) {
    if (lane == 0) {
      // PDL prologue: the weight (B) tiles of the first pipeline stages do
      // not depend on the previous kernel, so they are fetched while it
      // drains; activations (A) only after griddepcontrol.wait.
      int pre = 0;
      int pm0 = 0, pn0 = 0;
      if (u_first < num_units) {
        int tile, split, kb0, kb1;
        decode(u_first, pm0, pn0, tile, split, kb0, kb1);
        pre = min(C::STAGES, kb1 - kb0);
        for (int q = 0; q < pre; ++q) {
          uint8_t *sa = smem + q * C::STAGE_BYTES;
          mbar_expect_tx(&full[q], C::STAGE_BYTES);
          tma_load_2d(sa + C::A_BYTES, &tmB, (kb0 + q) * BK, pn0, &full[q]);
        }
      }
      pdl_wait();
      pdl_trigger();
      int it = 0;
      auto load_a = [&](uint8_t *sa, int kb, int m0, uint64_t *bar) {
        if (CS > 1)  // my slice of the A tile, into every CTA of the cluster
          tma_load_2d_mc(sa + rank * A_SLICE * 128, &tmA, kb * BK, m0 + rank * A_SLICE, bar, CMASK);
        else
          tma_load_2d(sa, &tmA, kb * BK, m0, bar);
      };
      for (int u = u_first; u < num_units; u += u_step) {
        int m0, n0, tile, split, kb0, kb1;
        decode(u, m0, n0, tile, split, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          uint8_t *sa = smem + s * C::STAGE_BYTES;
          if (it < pre) {  // B already in flight for this stage
            if (CS > 1) mbar_wait(&empty[s], ph ^ 1);  // (passes: fresh barriers)
            load_a(sa, kb, m0, &full[s]);
            continue;
          }
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          load_a(sa, kb, m0, &full[s]);
          tma_load_2d(sa + C::A_BYTES, &tmB, kb * BK, n0, &full[s]);
        }
      }
    } else {
      pdl_wait();
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      int it = 0, local = 0;
      for (int u = u_first; u < num_units; u += u_step, ++local) {
        int m0, n0, tile, split, kb0, kb1;
        decode(u, m0, n0, tile, split, kb0, kb1);
        const int acc = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * C::TMEM_COLS;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t *sa = smem + s * C::STAGE_BYTES;
          const uint64_t da = umma_desc_sw128(sa);
          const uint64_t db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
            umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          if (CS > 1)
            umma_commit_mc(&empty[s], CMASK);  // release the stage in every CTA
          else
            umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ---- epilogue warps 2..5
    pdl_wait();
    const int quarter = warp & 3;
    const bool vec_ok = ep.kind != SKB_EPI_SSRU && (ep.ldo % 8 == 0) &&
                        ((reinterpret_cast<uintptr_t>(ep.out) & 15) == 0);
    int local = 0;
    const int erow = quarter * 32 + lane;  // row within the tile
    for (int u = u_first; u < num_units; u += u_step, ++local) {
      int m0, n0, tile, split, kb0, kb1;
      decode(u, m0, n0, tile, split, kb0, kb1);
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m0 + erow;
      const uint32_t tbase = tmem + acc * C::TMEM_COLS + ((uint32_t)(quarter * 32) << 16);
      if (S == 1) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tmem_ld32(tbase + (uint32_t)c, v);
          const int n = n0 + c;
          if (row < M && n < N) {
            if (ep.kind == SKB_EPI_LOGITS)
              reinterpret_cast<float2 *>(ep.lse_part)[(size_t)row * ep.lse_ld + (n >> 5)] =
                  group_stats_fast(ep, row, n, N, v);
            if (!(vec_ok && n + 32 <= N && epilogue_vec32(ep, row, n, v)))
              epilogue_run(ep, row, n, N, v, 32);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        continue;
      }
      // ---- split-K: park this split's fp32 tile in the workspace
      float *wsp = ep.ws + ((size_t)(tile * S + split) * BM + erow) * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(tbase + (uint32_t)c, v);
        float4 *o = reinterpret_cast<float4 *>(wsp + c);
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) {
        const unsigned prev = atomicAdd(ep.counters + tile, 1u);
        last_flag[acc] = prev == (unsigned)(S - 1);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (!last_flag[acc]) continue;
      __threadfence();
      // last split to arrive: sum partials in split order, run the epilogue
      if (row < M) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          const int n = n0 + c;
          if (n >= N) break;
          float v[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = 0.f;
          for (int sp = 0; sp < S; ++sp) {
            const float4 *src = reinterpret_cast<const float4 *>(
                ep.ws + ((size_t)(tile * S + sp) * BM + erow) * BN + c);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 a = __ldcg(src + q);
              v[4 * q] += a.x; v[4 * q + 1] += a.y; v[4 * q + 2] += a.z; v[4 * q + 3] += a.w;
            }
          }
          if (ep.kind == SKB_EPI_LOGITS)
            reinterpret_cast<float2 *>(ep.lse_part)[(size_t)row * ep.lse_ld + (n >> 5)] =
                group_stats_fast(ep, row, n, N, v);
          if (!(vec_ok && n + 32 <= N && epilogue_vec32(ep, row, n, v)))
            epilogue_run(ep, row, n, N, v, 32);
        }
      }
      if (threadIdx.x == 64) ep.counters[tile] = 0u;  // ready for the next launch
    }
  }
  __syncthreads();
  // no peer may still multicast into / arrive on this CTA's shared memory
  if (CS > 1) cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * C::TMEM_COLS));
  }
}

// ---------------------------------------------------------- host side
static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

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
static int make_map(CUtensorMap *out, const void *ptr, int rows, int cols, int ld, int box_rows,
                    bool i8 = false) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, rows, cols, i8 ? -ld : ld, box_rows};
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
  // one box row = one 128-byte swizzle atom: 64 bf16 or 128 int8 elements
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * (i8 ? 1 : 2)};
  cuuint32_t box[2] = {(cuuint32_t)(i8 ? 2 * BK : BK), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void *>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SKB_ERR_LAUNCH, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return SKB_OK;
}

template <int BN, int CS>
static int launch(int M, int N, int K, const void *A, int lda, const void *W, int ldw,
                  EpiArgs ep, cudaStream_t st, int splits = 1) {
  using C = Cfg<BN>;
  ep.splits = CS > 1 ? 1 : splits;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, lda, BM / CS);
  if (rc) return rc;
  rc = make_map(&mb, W, N, K, ldw, BN);
  if (rc) return rc;
  ensure_smem_fn(k_gemm_tc<BN, CS>, C::SMEM);
  const int mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
  const int nsm = num_sms();
  int grid;
  if (CS > 1) {
    const int clusters = ((nt + CS - 1) / CS) * mt;
    const int maxc = nsm / CS;
    grid = (clusters < maxc ? clusters : maxc) * CS;
  } else {
    const int tiles = mt * nt * ep.splits;
    grid = tiles < nsm ? tiles : nsm;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CS > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CS;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k_gemm_tc<BN, CS>, ma, mb, M, N, K, ep);
  SKB_CHECK_LAUNCH("k_gemm_tc");
  return SKB_OK;
}

// tile-config overrides (tests / tuning): env SKB_GEMM_BN|CS|SPLITS at load,
// or skb_gemm_force() at run time; 0 = automatic
thread_local int g_force_bn = -1, g_force_cs = 0, g_force_s = 0;  // test/tuning overrides
void init_forces() {
  if (g_force_bn >= 0) return;
  const char *e = getenv("SKB_GEMM_BN");
  g_force_bn = e ? atoi(e) : 0;
  e = getenv("SKB_GEMM_CS");
  g_force_cs = e ? atoi(e) : 0;
  e = getenv("SKB_GEMM_SPLITS");
  g_force_s = e ? atoi(e) : 0;
}

}  // namespace tc

// ================================================ swap-AB decode GEMM (sw)
// The decode step's GEMMs have few activation rows (M = batch x beam, 640 at
// the benchmark) against wide weight matrices.  Laid out the usual way
// (activations on the MMA M side) they give only ceil(M/128) x N/BN tiles,
// far fewer than 148 SMs, each streaming a long K.  This kernel swaps the
// operands: the weight tile (128 output columns n) is the MMA A operand and
// an Na-row activation tile is the MMA B operand (Na = 16..256, a multiple
// of 16), so D^T[n, m] accumulates in TMEM with lane = n, column = m.  Na is
// chosen so that (N/128) x (M/Na) x CS fills the SMs, and every CTA runs a
// single tile with the WHOLE shared memory as a TMA ring: most of the K
// range is in flight at once, and the weight k-blocks (which do not depend
// on the previous kernel) are all requested before griddepcontrol.wait.
// Long-K shapes split K across a cluster of CS CTAs; the fp32 partial tiles
// are reduced through distributed shared memory in rank order
// (deterministic, no L2 round trip, no atomics), each CTA finishing 1/CS of
// the tile.  CS is chosen from (N, K) alone, so a row's result does not
// depend on the batch size (test_search.py:400-405).
namespace sw {

#ifdef SKB_GEMM_TRACE
__device__ unsigned long long g_trace[1024 * 16];
__device__ int g_dbg;
#define SW_STAMP(slot)                                                                    \
  do {                                                                                    \
    unsigned long long _t;                                                                \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                \
    const int _c = blockIdx.x + blockIdx.y * gridDim.x;                                   \
    if (_c < 1024) g_trace[_c * 16 + (slot)] = _t;                                         \
  } while (0)
#else
#define SW_STAMP(slot) \
  do {                 \
  } while (0)
#endif

constexpr int W_BYTES = 128 * tc::BK * 2;  // 16 KB weight k-block
constexpr int PUSH_ROWS = 8;               // split-K slices up to this many rows: st.async push


constexpr int SMEM_MAX = 232448;          // 227 KB opt-in

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// the small-slice reduction (st.async from registers) for Na/CS rows per CTA
__host__ __device__ constexpr bool push_small(int Na, int CS) {
  return CS > 1 && Na / CS <= PUSH_ROWS && ((Na / CS) & (Na / CS - 1)) == 0;
}

// Rows c..c+15 of output column `row` (v) belong to owners c/CPR ..; send
// each owner its CPR rows (one vector st.async, tx bytes on the owner's
// rbar) or keep them (plain st.shared) — slot [rank][row][0..CPR).
template <int CPR>
__device__ __forceinline__ void push_slices(const float *v, int c, int rank, uint32_t rbase,
                                            uint32_t rbar, int row) {
#pragma unroll
  for (int q = 0; q < 16 / CPR; ++q) {
    const int p = c / CPR + q;
    const uint32_t a = rbase + (uint32_t)((rank * 128 + row) * CPR) * 4u;
    const float *w = v + q * CPR;
#pragma unroll
    for (int h = 0; h < (CPR + 3) / 4; ++h) {
      const uint32_t ah = a + 16u * h;
      if (p == rank) {
        if (CPR == 1)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(ah), "f"(w[0]) : "memory");
        else if (CPR == 2)
          asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(ah), "f"(w[0]), "f"(w[1]) : "memory");
        else
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(ah), "f"(w[4 * h]), "f"(w[4 * h + 1]),
                       "f"(w[4 * h + 2]), "f"(w[4 * h + 3])
                       : "memory");
      } else {
        const uint32_t ra = mapa(ah, (uint32_t)p), rm = mapa(rbar, (uint32_t)p);
        if (CPR == 1)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
                       "r"(__float_as_uint(w[0])), "r"(rm)
                       : "memory");
        else if (CPR == 2)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1,%2}, [%3];" ::"r"(ra),
                       "r"(__float_as_uint(w[0])), "r"(__float_as_uint(w[1])), "r"(rm)
                       : "memory");
        else
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(ra),
                       "r"(__float_as_uint(w[4 * h])), "r"(__float_as_uint(w[4 * h + 1])),
                       "r"(__float_as_uint(w[4 * h + 2])), "r"(__float_as_uint(w[4 * h + 3])), "r"(rm)
                       : "memory");
      }
    }
  }
}

// Epilogue of one element (m, n).  Lanes of a warp hold consecutive n for
// the same m, so every store is coalesced.  The kernel is instantiated per
// epilogue kind and cluster size: each variant carries only its own code (a
// decode step runs ~40 different kernels back to back, so every launch
// starts with a cold instruction cache and code size is latency).
template <int KIND>
__device__ __forceinline__ void epi_one(const EpiArgs &e, int m, int n, float v, float bn) {
  const size_t o = (size_t)m * e.ldo + n;
  if (KIND == SKB_EPI_RESID) {
    float *x = reinterpret_cast<float *>(e.out) + o;
    *x = *x + (v + bn);
    return;
  }
  float t = v + bn;
  if (KIND == SKB_EPI_RELU) t = fmaxf(t, 0.f);
  if (e.out_dtype == SKB_F32)
    reinterpret_cast<float *>(e.out)[o] = t;
  else
    reinterpret_cast<__nv_bfloat16 *>(e.out)[o] = __float2bfloat16_rn(t);
}

// SSRU cell on the lane pair (2j, 2j+1) = (W_f h, W h); called by all 32
// lanes (the partner value comes by shuffle).
__device__ __forceinline__ void epi_ssru(const EpiArgs &e, const float *cprev, float *cnext,
                                         int m, int n, float v, float bn, bool ok) {
  const float w = __shfl_xor_sync(0xffffffffu, v, 1);
  if (!ok || (n & 1)) return;
  const int j = n >> 1;
  const int srow = e.src_row ? e.src_row[m] : m;
  const float cp = cprev ? cprev[(size_t)srow * e.ld_state + j] : 0.f;
  const float c = ssru_cell(v, bn, w, cp);
  cnext[(size_t)m * e.ld_state + j] = c;
  float *xp = reinterpret_cast<float *>(e.out) + (size_t)m * e.ldo + j;
  *xp = *xp + fmaxf(c, 0.f);
}

// 16 consecutive activation rows m0..m0+15 of output column n.  SSRU: all
// loads of the 16 rows (parent-row indices, then the parents' cells and the
// residual rows) are issued before any store — one row at a time, every
// row's loads waited behind the previous row's stores (they may alias as far
// as the compiler knows), which made the SSRU GEMM ~10x its mainloop at
// M = 640 (profiles/r2_60_graph_ssru128.txt).
// SSRU epilogue in two halves so loads can run ahead of the stores (and of
// the accumulator): the parents' cells and the residual rows of rows
// m0..m0+15 (they never alias this call's stores: c_next is the other half
// of the step double buffer, x rows are the call's own)...
__device__ __forceinline__ void ssru_load16(const EpiArgs &e, const float *cprev, int M, int m0, int n,
                                            bool nok, float (&cp)[16], float (&xo)[16], bool want_x = true) {
  const int j = n >> 1;
  const bool even = (n & 1) == 0;
  const float *x = reinterpret_cast<const float *>(e.out);
  int srow[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int m = m0 + i;
    srow[i] = (nok && even && m < M && e.src_row) ? __ldg(e.src_row + m) : m;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int m = m0 + i;
    const bool ok = nok && even && m < M;
    cp[i] = (ok && cprev) ? __ldcg(cprev + (size_t)srow[i] * e.ld_state + j) : 0.f;
    xo[i] = (ok && want_x) ? __ldcg(x + (size_t)m * e.ldo + j) : 0.f;
  }
}

// ...then the cells and the residual update (all 32 lanes: the W h partner
// value comes by shuffle).
__device__ __forceinline__ void ssru_store16(const EpiArgs &e, float *cnext, int M, int m0, int n, bool nok,
                                             float bn, const float *v, const float (&cp)[16],
                                             const float (&xo)[16]) {
  const int j = n >> 1;
  const bool even = (n & 1) == 0;
  float *x = reinterpret_cast<float *>(e.out);
  float w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = __shfl_xor_sync(0xffffffffu, v[i], 1);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int m = m0 + i;
    if (nok && even && m < M) {
      const float c = ssru_cell(v[i], bn, w[i], cp[i]);
      cnext[(size_t)m * e.ld_state + j] = c;
      x[(size_t)m * e.ldo + j] = xo[i] + fmaxf(c, 0.f);
    }
  }
}

// Staged variant (TMA-store epilogue): the cells and relu(cells) of rows
// mloc..mloc+15 into two [Na][64] fp32 shared tiles (local column row / 2);
// one TMA store writes c_next and one TMA reduce-add applies x += relu(c).
__device__ __forceinline__ void ssru_stage16(uint32_t stgc, uint32_t stgx, int mloc, int row, bool nok,
                                             int n, float bn, const float *v, const float (&cp)[16]) {
  float w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = __shfl_xor_sync(0xffffffffu, v[i], 1);
  if (!nok || (n & 1)) return;
  const uint32_t col = (uint32_t)(row >> 1) * 4u;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float c = ssru_cell(v[i], bn, w[i], cp[i]);
    const uint32_t o = (uint32_t)(mloc + i) * 256u + col;
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(stgc + o), "f"(c) : "memory");
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(stgx + o), "f"(fmaxf(c, 0.f)) : "memory");
  }
}

template <int KIND>
__device__ __forceinline__ void epi16(const EpiArgs &e, const float *cprev, float *cnext, int M,
                                      int m0, int n, bool nok, float bn, const float *v) {
  if constexpr (KIND == SKB_EPI_SSRU) {
    float cp[16], xo[16];
    ssru_load16(e, cprev, M, m0, n, nok, cp, xo);
    ssru_store16(e, cnext, M, m0, n, nok, bn, v, cp, xo);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int m = m0 + i;
      if (nok && m < M) epi_one<KIND>(e, m, n, v[i], bn);
    }
  }
}

__device__ __forceinline__ void sts4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// Stage 16 outputs (activation rows mloc..mloc+15, output column `row` of
// the tile) into the shared-memory tile [rows][128] that one TMA store (or
// TMA reduce-add, for the residual) writes out.  Lanes hold consecutive
// columns, so every st.shared is conflict-free.
template <int KIND>
__device__ __forceinline__ void stage16(uint32_t base, bool bf16, int mloc, int row, float bn,
                                        const float *v) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float t = v[i] + bn;
    if (KIND == SKB_EPI_RELU) t = fmaxf(t, 0.f);
    if (bf16) {
      const __nv_bfloat16 b = __float2bfloat16_rn(t);
      asm volatile("st.shared.b16 [%0], %1;" ::"r"(base + (uint32_t)((mloc + i) * 128 + row) * 2u),
                   "h"(*reinterpret_cast<const unsigned short *>(&b))
                   : "memory");
    } else {
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(base + (uint32_t)((mloc + i) * 128 + row) * 4u),
                   "f"(t)
                   : "memory");
    }
  }
}

// Epilogue warps: make the staged tile visible to the TMA unit, then one
// thread writes it with a bulk tensor store (x += tile for the residual).
// `before_store` runs on all 128 epilogue threads once the tile is complete
// in shared memory and before the store is issued.
template <int KIND, typename F>
__device__ __forceinline__ void flush_tile(const CUtensorMap *tmO, uint32_t base, int c0, int c1,
                                           bool leader, F before_store, bool full_wait = false,
                                           bool defer_wait = false) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("bar.sync 1, 128;" ::: "memory");
  before_store();
  if (leader) {
    if (KIND == SKB_EPI_RESID)
      asm volatile(
          "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
              reinterpret_cast<uint64_t>(tmO)),
          "r"(c0), "r"(c1), "r"(base)
          : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                       reinterpret_cast<uint64_t>(tmO)),
                   "r"(c0), "r"(c1), "r"(base)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (full_wait)  // the writes themselves are complete (another CTA reads them)
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    else if (!defer_wait)  // (deferred: the caller waits before the CTA exits)
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// One LayerNorm row (kernels.py:298-324), warp per row: the same arithmetic
// and order as k_layernorm_reg<NV> (elementwise.cu), NV = d / 128 <= 8.
// x is read from L2 (written by other CTAs' bulk reduce of this kernel).
__device__ __forceinline__ void ln_row(const EpiArgs &e, int m, int d, int lane) {
  const int nv = d >> 7;
  const float4 *xr = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(e.out) +
                                                      (size_t)m * e.ldo);
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = i < nv ? __ldcg(xr + lane + 32 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  const float mu = warp_sum(s) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) {
      const float a = v[i].x - mu, b = v[i].y - mu, c = v[i].z - mu, f = v[i].w - mu;
      q += (a * a + b * b) + (c * c + f * f);
    }
  const float inv = 1.0f / sqrtf(warp_sum(q) / (float)d + e.ln_eps);
  const float4 *g4 = reinterpret_cast<const float4 *>(e.ln_gain);
  const float4 *b4 = reinterpret_cast<const float4 *>(e.ln_bias);
  uint2 *o = reinterpret_cast<uint2 *>(e.ln_out + (size_t)m * e.ln_ldo);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) {
      const int c4 = lane + 32 * i;
      const float4 g = __ldg(g4 + c4), bb = __ldg(b4 + c4);
      const float o0 = ((v[i].x - mu) * inv) * g.x + bb.x, o1 = ((v[i].y - mu) * inv) * g.y + bb.y;
      const float o2 = ((v[i].z - mu) * inv) * g.z + bb.z, o3 = ((v[i].w - mu) * inv) * g.w + bb.w;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t *>(&p0);
      w.y = *reinterpret_cast<uint32_t *>(&p1);
      o[c4] = w;
    }
}

// Prologue LayerNorm (kernels.py:298-324) of input row m into row rl of the
// kernel's resident activation panel: K-major bf16, one [Na][64] SW128 tile
// per 64-column k-block, i.e. exactly the bytes a TMA load of LN(x) would
// have placed there.  Same arithmetic as ln_row / k_layernorm_reg (bitwise).
__device__ __forceinline__ void ln_row_panel(const EpiArgs &e, int m, int rl, int d, int Na,
                                             uint8_t *panel, int lane, const float4 (&g)[8],
                                             const float4 (&bb)[8], int kb0, int kb1) {
  const int nv = d >> 7;
  const float4 *xr = reinterpret_cast<const float4 *>(e.lnx + (size_t)m * e.lnx_ld);
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = i < nv ? __ldcg(xr + lane + 32 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  const float mu = warp_sum(s) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) {
      const float a = v[i].x - mu, b = v[i].y - mu, c = v[i].z - mu, f = v[i].w - mu;
      q += (a * a + b * b) + (c * c + f * f);
    }
  const float inv = 1.0f / sqrtf(warp_sum(q) / (float)d + e.lnx_eps);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < nv) {
      const int c4 = lane + 32 * i;
      const float o0 = ((v[i].x - mu) * inv) * g[i].x + bb[i].x, o1 = ((v[i].y - mu) * inv) * g[i].y + bb[i].y;
      const float o2 = ((v[i].z - mu) * inv) * g[i].z + bb[i].z, o3 = ((v[i].w - mu) * inv) * g[i].w + bb[i].w;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t *>(&p0);
      w.y = *reinterpret_cast<uint32_t *>(&p1);
      // statistics over the whole row; only this CTA's k-blocks are stored
      const int c = 4 * c4, cc = c & 63, kb = c >> 6;
      if (kb >= kb0 && kb < kb1)
        *reinterpret_cast<uint2 *>(panel + (size_t)(kb - kb0) * Na * 128 + rl * 128 +
                                   ((((cc >> 3) ^ (rl & 7))) << 4) + (cc & 7) * 2) = w;
    }
}

// LOGITS epilogue (model.py:577-581, kernels.py:287-295): partial
// log-softmax statistics (max, sum exp(x - max)) of every 32-column group of
// the staged fp32 logit tile, over the row's active columns.  Two lanes share
// a group (16 values each: four 16-byte shared loads, their order rotated by
// lane so a warp's 32 loads hit distinct bank quads), a warp covers 4 rows x
// 4 groups per step, and each reduction is ONE xor-shuffle with the partner
// half — the earlier 8-lanes-per-group layout spent 6 dependent shuffle
// levels per row (5.7 us of a 67 us output projection at M = 640,
// profiles/r2_91_stats.txt).  Fixed per-lane order: deterministic and
// independent of M.
__device__ __forceinline__ void logits_stats(const EpiArgs &e, uint32_t stg, int M, int N, int m0,
                                             int n0, int rows, int warp_e, int lane,
                                             uint32_t smask = 0) {
  constexpr float L2E = 1.4426950408889634f;
  const int rr = lane >> 3, g = (lane >> 1) & 3, h = lane & 1;  // row in the step, group, half
  const int n = n0 + g * 32;
  unsigned tail = 0xffffffffu;
  if (n >= N) tail = 0u;
  else if (N - n < 32) tail = (1u << (N - n)) - 1u;
#pragma unroll 1
  for (int mb = 4 * warp_e; mb < rows && m0 + mb < M; mb += 16) {
    const int ml = mb + rr, m = m0 + ml;
    const bool ok = ml < rows && m < M;
    float v[16];
    unsigned bits = 0u;
    if (ok) {
      unsigned w = tail;
      if (e.mask && tail) {
        if (smask) {  // staged ahead of the accumulator (logits_mask_stage)
          unsigned mw;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(mw) : "r"(smask + (uint32_t)(ml * 4 + g) * 4u));
          w &= mw;
        } else {
          w &= e.mask[(size_t)(m / e.rows_per_group) * e.mask_words + (n >> 5)];
        }
      }
      bits = (w >> (16 * h)) & 0xffffu;
      const uint32_t base = stg + (uint32_t)(ml * 128 + g * 32 + h * 16) * 4u;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int kk = (k + lane) & 3;  // chunk kk of the half in slot k
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[4 * k]), "=f"(v[4 * k + 1]), "=f"(v[4 * k + 2]), "=f"(v[4 * k + 3])
                     : "r"(base + (uint32_t)kk * 16u));
        const unsigned b = (bits >> (4 * kk)) & 0xfu;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (!((b >> q) & 1u)) v[4 * k + q] = -INFINITY;  // masked / past N
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = -INFINITY;
    }
    float mx = v[0];
#pragma unroll
    for (int q = 1; q < 16; ++q) mx = fmaxf(mx, v[q]);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    // ex2.approx (SFU) on x - max, whose log-sum-exp differs from expf's by
    // < 1e-6 relative; ex2(-inf) = +0 for masked columns
    const float ml2 = mx == -INFINITY ? 0.f : mx * L2E;
    float acc = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      float e2;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(fmaf(v[q], L2E, -ml2)));
      acc += e2;
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (h == 0 && ok && n < N)
      reinterpret_cast<float2 *>(e.lse_part)[(size_t)m * e.lse_ld + (n >> 5)] = make_float2(mx, acc);
  }
}

// Restricted vocabulary: the tile's column-mask words [rows][4 groups] into
// shared memory while the MMAs run (they were written before the decode
// loop), so the statistics pass reads them from shared memory instead of
// one dependent L2 load per row batch.
__device__ __forceinline__ void logits_mask_stage(const EpiArgs &e, uint32_t smask, int M, int N, int m0,
                                                  int n0, int rows, int tid) {
#pragma unroll 1
  for (int i = tid; i < rows * 4; i += 128) {
    const int ml = i >> 2, g = i & 3, m = m0 + ml, n = n0 + 32 * g;
    const unsigned w = (m < M && n < N)
                           ? __ldg(e.mask + (size_t)(m / e.rows_per_group) * e.mask_words + (n >> 5))
                           : 0u;
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(smask + (uint32_t)i * 4u), "r"(w) : "memory");
  }
}

//   warp 0 : TMA producer (one lane)   warp 1 : MMA issuer (one lane)
//   warps 2..5 : epilogue, TMEM lane quarter = warp % 4
// grid (weight tiles x activation tiles, CS), cluster (1, CS): the CS CTAs
// of a cluster share the output tile and split K.
template <int KIND, int CS, bool LNX = false, bool I8 = false>
__global__ void __launch_bounds__(192, 1)
    k_gemm_sw(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
              const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2, int M,
              int N, int K, int Na, int stages, int stg_off, int tma_out, EpiArgs ep) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  // prologue-LayerNorm mode: the ring holds weight tiles only and the
  // normalised activation rows sit in a resident panel [nk][Na][64] (SW128)
  // (a separate instantiation: its registers would lower co-residency of
  // the plain kernel)
  constexpr bool lnx = LNX && KIND != SKB_EPI_RESID && KIND != SKB_EPI_SSRU;
  constexpr bool lnout = LNX && KIND == SKB_EPI_RESID;  // fused LayerNorm of the updated rows
  const int SB = lnx ? W_BYTES : W_BYTES + Na * 128;
  uint8_t *panel = smem + stages * SB;
  // (with a K split the panel holds this CTA's k-blocks only)
  const int panel_bytes = lnx ? (((K + BK - 1) / BK + CS - 1) / CS) * Na * 128 : 0;
  // small-slice K split (<= PUSH_ROWS rows per CTA): peers push their partial
  // slices straight from registers into this CTA's receive area (st.async),
  // which therefore lives outside the ring (a peer may finish first)
  const bool apush = push_small(Na, CS);
  float *arecv = reinterpret_cast<float *>(smem + stages * SB + panel_bytes);  // [CS][128][cpr]
  const int arecv_bytes = apush ? Na * 512 : 0;
  // LOGITS over a restricted vocabulary: the tile's mask words [Na][4]
  const int smask_bytes = (KIND == SKB_EPI_LOGITS && ep.mask) ? Na * 16 : 0;
  const uint32_t smask = smask_bytes ? smem_u32(smem + stages * SB + panel_bytes + arecv_bytes) : 0u;
  uint64_t *full =
      reinterpret_cast<uint64_t *>(smem + stages * SB + panel_bytes + arecv_bytes + smask_bytes);
  uint64_t *empty = full + stages;
  uint64_t *tfull = empty + stages;
  uint64_t *rbar = tfull + 1;  // split-K: peers' partial slices landed
  uint64_t *xready = rbar + 1;  // prologue LayerNorm: panel written
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xready + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = CS > 1 ? (int)blockIdx.y : 0;
  const int n_at = (M + Na - 1) / Na;
  const int at = (int)blockIdx.x % n_at, wt = (int)blockIdx.x / n_at;
  const int m0 = at * Na, n0 = wt * 128;
  constexpr int KBE = I8 ? 2 * BK : BK;  // elements per 128-byte k-block
  const int nk = (K + KBE - 1) / KBE;
  const int kb0 = rank * nk / CS, kb1 = (rank + 1) * nk / CS;
  const int nkc = kb1 - kb0;
  int tcols = 32;
  while (tcols < Na) tcols <<= 1;

  if (threadIdx.x == 0) {
    SW_STAMP(0);
#pragma unroll 1
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(rbar, 1);
    mbar_init(xready, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    if (tma_out)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmO)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();  // reconverge the warp (lane-divergent roles) before bar.sync
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (apush) {
    // the (CS-1) peer slices this CTA will receive; then announce to the
    // cluster that this CTA's barriers exist (waited for only right before
    // the first st.async, long after — off the critical path)
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(rbar)),
                   "r"((uint32_t)((CS - 1) * Na * 512 / CS))
                   : "memory");
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }

  if (warp == 0) {
    if (lane == 0) {
      // weights first: independent of the previous kernel (PDL prologue)
      const int pre = nkc < stages ? nkc : stages;
#ifdef SKB_GEMM_TRACE
      // timing experiments: 4 = skip the activation loads, 5 = skip weights, 6 = both
      const int ldbg = g_dbg;
#else
      constexpr int ldbg = 0;
#endif
      const int sbx = ldbg == 6 ? 0 : (lnx ? W_BYTES : (ldbg == 4 ? W_BYTES : (ldbg == 5 ? SB - W_BYTES : SB)));
#pragma unroll 1
      for (int q = 0; q < pre; ++q) {
        mbar_expect_tx(&full[q], sbx);
        if (ldbg != 5 && ldbg != 6) tma_load_2d(smem + q * SB, &tmW, (kb0 + q) * KBE, n0, &full[q]);
      }
      pdl_wait();
      if (!ep.late_trigger) pdl_trigger();
      SW_STAMP(2);
#pragma unroll 1
      for (int q = 0; q < pre; ++q)
        if (ldbg != 4 && ldbg != 6 && !lnx) tma_load_2d(smem + q * SB + W_BYTES, &tmX, (kb0 + q) * KBE, m0, &full[q]);
#pragma unroll 1
      for (int it = pre; it < nkc; ++it) {
        const int s = it % stages;
        const uint32_t ph = (it / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t *st = smem + s * SB;
        mbar_expect_tx(&full[s], sbx);
        if (ldbg != 5 && ldbg != 6) tma_load_2d(st, &tmW, (kb0 + it) * KBE, n0, &full[s]);
        if (ldbg != 4 && ldbg != 6 && !lnx) tma_load_2d(st + W_BYTES, &tmX, (kb0 + it) * KBE, m0, &full[s]);
      }
    } else {
      pdl_wait();
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      const uint32_t idesc = I8 ? idesc_s8(128, Na) : idesc_bf16(128, Na);
      if (lnx) {
        mbar_wait(xready, 0);
        SW_STAMP(14);
      }
#pragma unroll 1
      for (int it = 0; it < nkc; ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        if (it == 0) SW_STAMP(3);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t *st = smem + s * SB;
        const uint64_t da = umma_desc_sw128(st);
        const uint64_t db = umma_desc_sw128(lnx ? panel + (size_t)it * Na * 128 : st + W_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          if constexpr (I8)
            umma_s8(tmem, da + 2 * k, db + 2 * k, idesc, (it > 0 || k > 0) ? 1u : 0u);
          else
            umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (it > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
  }
  // epilogue state (warps 2..5)
  const int row = (warp & 3) * 32 + lane;  // weight row within the tile = output column
  const int n = n0 + row;
  const bool nok = n < N;
  const float *cprev = nullptr;
  float *cnext = nullptr;
  if (warp >= 2) {
    if constexpr (lnx) {
      // before the grid dependency: gain / bias (parameters) into registers,
      // zero rows past M (they feed only output columns never stored)
      float4 lg[8], lb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < (K >> 7)) {
          lg[i] = __ldg(reinterpret_cast<const float4 *>(ep.lnx_g) + lane + 32 * i);
          lb[i] = __ldg(reinterpret_cast<const float4 *>(ep.lnx_b) + lane + 32 * i);
        }
#pragma unroll 1
      for (int rl = warp - 2; rl < Na; rl += 4)
        if (m0 + rl >= M)
#pragma unroll 1
          for (int c = kb0 * 8 + lane; c < kb1 * 8; c += 32)
            *reinterpret_cast<uint4 *>(panel + (size_t)((c >> 3) - kb0) * Na * 128 + rl * 128 + (c & 7) * 16) =
                make_uint4(0u, 0u, 0u, 0u);
      pdl_wait();
      // normalise this tile's activation rows into the panel
#pragma unroll 1
      for (int rl = warp - 2; rl < Na && m0 + rl < M; rl += 4)
        ln_row_panel(ep, m0 + rl, rl, K, Na, panel, lane, lg, lb, kb0, kb1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(xready);
      if (warp == 2 && lane == 0) SW_STAMP(13);
    } else {
      pdl_wait();
    }
    if (KIND == SKB_EPI_SSRU) {
      cprev = ep.c_prev;
      cnext = ep.c_next;
      if (ep.step) {  // decode-loop double buffer selected by step parity
        const int t = *ep.step;
        cnext = ep.c_next + (t & 1) * ep.state_stride;
        cprev = t == 0 ? nullptr : ep.c_next + ((t + 1) & 1) * ep.state_stride;
      }
    }
    // SSRU, whole-K tiles: the first 16 rows' parent cells and residual rows
    // are read while the MMAs run (software-pipelined below)
    float scp[16], sxo[16];
    if constexpr (KIND == SKB_EPI_SSRU && CS == 1) ssru_load16(ep, cprev, M, m0, n, nok, scp, sxo, tma_out != 2);
    if constexpr (KIND == SKB_EPI_LOGITS)
      if (smask) logits_mask_stage(ep, smask, M, N, m0, n0, Na, threadIdx.x - 64);
    mbar_wait(tfull, 0);
    if (ep.late_trigger == 1 && warp == 2 && lane == 0) pdl_trigger();  // (2: only at exit)
    if (warp == 2 && lane == 0) SW_STAMP(5);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    if (CS == 1) {
      const float bn = (ep.bias && nok) ? __ldg(ep.bias + n) : 0.f;
#ifdef SKB_GEMM_TRACE
      const int dbg = g_dbg;
#else
      constexpr int dbg = 0;
#endif
      const uint32_t stg = smem_u32(smem) + (uint32_t)stg_off;
      const bool bf16 = ep.out_dtype == SKB_BF16 && KIND != SKB_EPI_RESID;
#pragma unroll 1
      const float wsc = (I8 && nok) ? __ldg(ep.w_scale + n) : 0.f;
      for (int c = 0; c < Na && m0 + c < M; c += 16) {
        float v[16];
        if (dbg != 2)
          tmem_ld16(tb + (uint32_t)c, v);
        else
          for (int i = 0; i < 16; ++i) v[i] = (float)i;
        if (dbg == 1) continue;
        if constexpr (KIND == SKB_EPI_SSRU) {
          // next chunk's loads before this chunk's stores
          const bool more = c + 16 < Na && m0 + c + 16 < M;
          float ncp[16], nxo[16];
          if (more) {
            if (dbg == 7) {
#pragma unroll
              for (int i = 0; i < 16; ++i) ncp[i] = nxo[i] = 0.f;
            } else {
              ssru_load16(ep, cprev, M, m0 + c + 16, n, nok, ncp, nxo, tma_out != 2);
            }
          }
          if (dbg == 6) {  // trace experiments: cells computed, nothing stored
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) acc += ssru_cell(v[i], bn, __shfl_xor_sync(0xffffffffu, v[i], 1), scp[i]) + sxo[i];
            if (acc == 12345.f) cnext[0] = acc;
          } else if (tma_out == 2) {  // staged: TMA store / reduce-add after the last chunk
            const uint32_t stgc = smem_u32(smem) + (uint32_t)stg_off;
            ssru_stage16(stgc, stgc + (uint32_t)Na * 256u, c, row, nok, n, bn, v, scp);
          } else {
            ssru_store16(ep, cnext, M, m0 + c, n, nok, bn, v, scp, sxo);
          }
          if (more) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              scp[i] = ncp[i];
              sxo[i] = nxo[i];
            }
          }
          continue;
        }
        if constexpr (I8) {
          // quant.py:124-128: (float32(acc) * a_scale) * w_scale, each
          // product rounded on its own (no FMA), the bias added after
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int m = m0 + c + i;
            const float as = m < M ? __ldg(ep.a_scale + m) : 0.f;
            v[i] = __fmul_rn(__fmul_rn(__int2float_rn(__float_as_int(v[i])), as), wsc);
          }
        }
        if (KIND != SKB_EPI_SSRU && tma_out)
          stage16<KIND>(stg, bf16, c, row, bn, v);
        else
          epi16<KIND>(ep, cprev, cnext, M, m0 + c, n, nok, bn, v);
      }
      if constexpr (KIND == SKB_EPI_SSRU) {
        if (tma_out == 2 && dbg != 1) {
          // c_next [halves][M][d] (3D map: the step's half) and x += relu(c)
          const uint32_t stgc = smem_u32(smem) + (uint32_t)stg_off;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (warp == 2 && lane == 0) {
            const int half = ep.step ? (*ep.step & 1) : 0;
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmO2)),
                "r"(n0 >> 1), "r"(m0), "r"(half), "r"(stgc)
                : "memory");
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmO)),
                "r"(n0 >> 1), "r"(m0), "r"(0), "r"(stgc + (uint32_t)Na * 256u)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
        }
      }
      if (KIND != SKB_EPI_SSRU && tma_out && dbg != 1) {
        // LOGITS: the store engine and the group statistics both only read
        // the staged tile, so the store is issued first and the statistics
        // run while it streams out; the leader waits for the store's reads
        // before the CTA exits.  (Statistics taken from the accumulator
        // registers instead — warp reductions over the 32 lanes of a group —
        // measured 1.7x slower than this shared-memory pass.)
        flush_tile<KIND>(&tmO, stg, n0, m0, warp == 2 && lane == 0, [] {}, lnout,
                         KIND == SKB_EPI_LOGITS);
        if constexpr (KIND == SKB_EPI_LOGITS) {
          if (warp == 3 && lane == 0) SW_STAMP(11);
          if (dbg != 3) logits_stats(ep, stg, M, N, m0, n0, Na, warp - 2, lane, smask);
          if (warp == 3 && lane == 0) SW_STAMP(12);
          if (warp == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
      }
    } else if (apush) {
      // small slices: every CTA owns rows [rank*cpr, (rank+1)*cpr) of the
      // tile.  Each thread (output column `row`) sends every other owner its
      // rows of the partial straight from registers with vector st.async into
      // the owner's receive area arecv[src][row][cpr] (the tx bytes complete
      // on the owner's rbar; nothing of the sender's shared memory is read,
      // so the sender may exit at once) and keeps its own rows there too.  No
      // cluster barrier on the critical path: the only one (barriers
      // initialised) was entered at kernel start.  The owner sums in rank
      // order (the fp32 order of the push path below) and stores from
      // registers.
      const int cpr = Na / CS;
      const uint32_t rbase = smem_u32(arecv), rb = smem_u32(rbar);
      __syncwarp();
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' rbar initialised
#pragma unroll 1
      for (int c = 0; c < Na; c += 16) {
        float v[16];
        tmem_ld16(tb + (uint32_t)c, v);
        if (cpr == 1)
          push_slices<1>(v, c, rank, rbase, rb, row);
        else if (cpr == 2)
          push_slices<2>(v, c, rank, rbase, rb, row);
        else if (cpr == 4)
          push_slices<4>(v, c, rank, rbase, rb, row);
        else
          push_slices<8>(v, c, rank, rbase, rb, row);
      }
      mbar_wait(rbar, 0);
      if (warp == 2 && lane == 0) SW_STAMP(9);
      const float bn = (ep.bias && nok) ? __ldg(ep.bias + n) : 0.f;
      const int c0 = rank * cpr;
#pragma unroll 1
      for (int j = 0; j < cpr; ++j) {
        const int m = m0 + c0 + j;
        float acc = 0.f;
#pragma unroll
        for (int src = 0; src < CS; ++src) {
          float x;
          asm volatile("ld.shared.f32 %0, [%1];"
                       : "=f"(x)
                       : "r"(rbase + (uint32_t)((src * 128 + row) * cpr + j) * 4u)
                       : "memory");
          acc = src == 0 ? x : acc + x;
        }
        if (KIND == SKB_EPI_SSRU)
          epi_ssru(ep, cprev, cnext, m, n, acc, bn, nok && m < M);
        else if (nok && m < M)
          epi_one<KIND>(ep, m, n, acc, bn);
      }
      if (warp == 2 && lane == 0) SW_STAMP(4);
    } else {
      // park the fp32 partial in my shared memory: part[m][128] (row-major
      // in m, so the slice each peer finishes is one contiguous block)
      const uint32_t pbase = smem_u32(smem) + (uint32_t)row * 4u;
#pragma unroll 1
      for (int c = 0; c < Na; c += 16) {
        float v[16];
        tmem_ld16(tb + (uint32_t)c, v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(pbase + (uint32_t)(c + i) * 512u), "f"(v[i])
                       : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (warp == 2 && lane == 0)  // expect the CS-1 slices the peers push to me
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(rbar)),
                     "r"((uint32_t)((CS - 1) * (Na / CS) * 512))
                     : "memory");
    }
  }
  __syncwarp();
  if (warp == 2 && lane == 0) SW_STAMP(1);
  if (CS > 1 && apush && warp < 2)
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // pairs the early arrive
  if (CS > 1 && !apush) {
    // split-K reduction, push model: every CTA bulk-copies slice p of its
    // partial into CTA p's receive slot [my rank] (async copy engine over
    // the cluster network), then CTA p sums its slice in rank order.
    const int cpr = Na / CS;  // activation rows finished by this CTA
    const int c0 = rank * cpr;
    const uint32_t part = smem_u32(smem);
    const uint32_t recv = part + (uint32_t)Na * 512u;  // [CS][cpr][128] fp32
    cluster_sync_all();  // all partials written, every ring drained
    if (warp == 2 && lane == 0) SW_STAMP(8);
    if (warp == 2 && lane == 0) {
#pragma unroll 1
      for (int p = 0; p < CS; ++p) {
        if (p == rank) continue;
        const uint32_t dst = mapa(recv + (uint32_t)(rank * cpr) * 512u, (uint32_t)p);
        const uint32_t bar = mapa(smem_u32(rbar), (uint32_t)p);
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "r"(part + (uint32_t)(p * cpr) * 512u), "r"((uint32_t)(cpr * 512)), "r"(bar)
            : "memory");
      }
    }
    if (warp >= 2) {
      const float bn = (ep.bias && nok) ? __ldg(ep.bias + n) : 0.f;
      const uint32_t stg = smem_u32(smem) + (uint32_t)stg_off;
      const bool bf16 = ep.out_dtype == SKB_BF16 && KIND != SKB_EPI_RESID;
      mbar_wait(rbar, 0);
      if (warp == 2 && lane == 0) SW_STAMP(9);
#pragma unroll 1
      for (int j0 = 0; j0 < cpr && m0 + c0 + j0 < M; j0 += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int jj = j0 + i < cpr ? j0 + i : cpr - 1;
          float acc = 0.f;
#pragma unroll
          for (int src = 0; src < CS; ++src) {  // fixed rank order: deterministic
            const uint32_t a = src == rank ? part + (uint32_t)(c0 + jj) * 512u
                                           : recv + (uint32_t)(src * cpr + jj) * 512u;
            float x;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a + (uint32_t)row * 4u) : "memory");
            acc = src == 0 ? x : acc + x;
          }
          v[i] = acc;
        }
        if (KIND != SKB_EPI_SSRU && tma_out) {
          stage16<KIND>(stg, bf16, j0, row, bn, v);
        } else {
          const int lim = min(M, m0 + c0 + cpr);  // rows beyond my slice are a peer's
          epi16<KIND>(ep, cprev, cnext, lim, m0 + c0 + j0, n, nok, bn, v);
        }
      }
      if (warp == 2 && lane == 0) SW_STAMP(10);
      if (KIND != SKB_EPI_SSRU && tma_out)
        flush_tile<KIND>(&tmO, stg, n0, m0 + c0, warp == 2 && lane == 0, [] {},
                         lnout);
    }
    if (warp == 2 && lane == 0) SW_STAMP(4);
    cluster_sync_all();  // peers are done reading my shared memory
  }
  // ---- fused LayerNorm of this activation-row tile (RESID): every CTA that
  // writes columns of the tile (n_wt x CS of them) takes an arrival ticket
  // once its writes are complete; the CTA drawing the tile's last ticket
  // normalises all of the tile's rows (no CTA ever waits for another, so
  // the kernel cannot deadlock however few of its CTAs are resident).
  // Same arithmetic as the LN kernel.
  if (lnout && warp >= 2) {
    volatile uint32_t &ln_last = tmem_slot[1];  // flag beside the TMEM address (dynamic smem)
    if (warp == 2 && lane == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      const unsigned G = (unsigned)(((N + 127) / 128) * CS);
      const unsigned tk = atomicAdd(ep.ln_counter + at, 1u);
      ln_last = (tk % G) == G - 1;
      if (ln_last) __threadfence();
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (ln_last)
      for (int rl = warp - 2; rl < Na && m0 + rl < M; rl += 4) ln_row(ep, m0 + rl, N, lane);
  }
  __syncwarp();  // reconverge the warp (lane-divergent roles) before bar.sync
  __syncthreads();
#ifdef SKB_GEMM_TRACE
  if (threadIdx.x == 0) {
    SW_STAMP(6);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int c = blockIdx.x + blockIdx.y * gridDim.x;
    if (c < 1024) g_trace[c * 16 + 7] = smid;
  }
#endif
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

// Output tensor map for the TMA-store epilogue: [rows M][cols N] of fp32 or
// bf16 at pitch ld, box = 128 columns x box_rows rows, no swizzle.
// Output tensor maps of a swap-AB launch: a = the output (or x), b = the
// SSRU cell buffer (unused by the other epilogues).
struct OutMaps {
  CUtensorMap a, b;
};

// fp32 [halves][rows][cols] (row pitch ld, half pitch half_stride elements),
// box 64 columns x box_rows rows x 1: the SSRU epilogue's TMA store of the
// cells into the step's half of the double buffer and its TMA reduce-add of
// relu(c) into x (halves = 1), rows past `rows` clipped within each half.
static int make_map_ssru(CUtensorMap *out, const void *ptr, int rows, int cols, int ld, int halves,
                         long long half_stride, int box_rows) {
  tc::EncodeTiledFn fn = tc::encode_fn();
  if (!fn) return fail(SKB_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)halves};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(halves > 1 ? half_stride : (long long)ld * rows) * 4};
  cuuint32_t box[3] = {64u, (cuuint32_t)box_rows, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SKB_ERR_LAUNCH, "cuTensorMapEncodeTiled(ssru) failed (%d)", (int)r);
  return SKB_OK;
}

static int make_map_out(CUtensorMap *out, const void *ptr, int rows, int cols, int ld, bool f32,
                        int box_rows) {
  static std::mutex mu;
  static std::unordered_map<tc::MapKey, CUtensorMap, tc::MapKeyHash> cache;
  tc::MapKey key{ptr, rows, cols, ld * (f32 ? -1 : 1), box_rows};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return SKB_OK;
    }
  }
  tc::EncodeTiledFn fn = tc::encode_fn();
  if (!fn) return fail(SKB_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  const int es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {128u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void *>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SKB_ERR_LAUNCH, "cuTensorMapEncodeTiled(out) failed (%d)", (int)r);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *out;
  return SKB_OK;
}

template <int KIND, int CS, bool LNX = false, bool I8 = false>
static int launch_t(int M, int N, int K, const CUtensorMap &mw, const CUtensorMap &mx,
                    const OutMaps &mo, int Na, int stages, int stg_off, int tma_out,
                    size_t smem, EpiArgs ep, cudaStream_t st) {
  ensure_smem_fn(k_gemm_sw<KIND, CS, LNX, I8>, SMEM_MAX);
  if (CS > 8)  // 16-CTA clusters are opt-in (non-portable) on B200
    cudaFuncSetAttribute(k_gemm_sw<KIND, CS, LNX, I8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int n_wt = (N + 127) / 128, n_at = (M + Na - 1) / Na;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_wt * n_at, CS);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CS > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = CS;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k_gemm_sw<KIND, CS, LNX, I8>, mw, mx, mo.a, mo.b, M, N, K, Na, stages,
                     stg_off, tma_out, ep);
  SKB_CHECK_LAUNCH("k_gemm_sw");
  return SKB_OK;
}

template <int KIND>
static int launch_k2(int M, int N, int K, const CUtensorMap &mw, const CUtensorMap &mx,
                     const OutMaps &mo, int Na, int CS, int stages, int stg_off, int tma_out,
                     size_t smem, EpiArgs ep, cudaStream_t st) {
  if constexpr (KIND == SKB_EPI_STORE || KIND == SKB_EPI_RELU)
    if (ep.lnx) {
      if (CS == 8)
        return launch_t<KIND, 8, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
      if (CS == 4)
        return launch_t<KIND, 4, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
      return launch_t<KIND, 1, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
    }
  if constexpr (KIND == SKB_EPI_RESID)
    if (ep.ln_out) {
      if (CS == 8)
        return launch_t<KIND, 8, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
      if (CS == 4)
        return launch_t<KIND, 4, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
      if (CS == 2)
        return launch_t<KIND, 2, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
      return launch_t<KIND, 1, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
    }
  if constexpr (KIND != SKB_EPI_LOGITS)
    if (CS == 16)
      return launch_t<KIND, 16>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
  if (CS == 8)
    return launch_t<KIND, 8>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
  if (CS == 4)
    return launch_t<KIND, 4>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
  if (CS == 2)
    return launch_t<KIND, 2>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
  return launch_t<KIND, 1>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
}


static int launch(int M, int N, int K, const void *X, int ldx, const void *W, int ldw, EpiArgs ep,
                  cudaStream_t st, int Na, int CS, int conc, bool i8 = false) {
  ep.splits = 1;
  // When the dependent grid launches (PDL trigger): right after this grid's
  // own dependency wait with one decode stream (the next kernel's CTAs become
  // resident and prefetch their weights under this one), but only once the
  // accumulator is complete when several streams share the device — early
  // dependents would sit in SM slots the other streams' kernels can use.
  // Measured on B200: 3 streams 4898 -> 5094 sentences/s, 1 stream 3197 ->
  // 3079 if late.  SKB_PDL_LATE=0|1 forces either.
  static int late_env = -2;
  if (late_env == -2) {
    const char *e = getenv("SKB_PDL_LATE");
    late_env = e ? atoi(e) : -1;
  }
  ep.late_trigger = late_env >= 0 ? late_env : (conc > 1 ? 1 : 0);
#ifdef SKB_GEMM_TRACE
  {
    const char *e = getenv("SKB_SW_DBG");
    const int d = e ? atoi(e) : 0;
    cudaMemcpyToSymbol(g_dbg, &d, sizeof(int));
  }
#endif
  if (Na < 16 || Na > 256 || Na % 16 || !(CS == 1 || CS == 2 || CS == 4 || CS == 8 || CS == 16) ||
      (CS > 1 && Na % CS) || (CS == 16 && !push_small(Na, CS)))
    return fail(SKB_ERR_CONFIG, "gemm_sw: bad tile Na=%d CS=%d", Na, CS);
  if (i8 && (CS != 1 || ep.lnx || ep.ln_out || ep.kind == SKB_EPI_SSRU || ep.kind == SKB_EPI_LOGITS))
    return fail(SKB_ERR_CONFIG, "gemm_sw: the int8 path has no K split, LayerNorm, SSRU or LOGITS epilogue");
  CUtensorMap mw, mx;
  int rc = tc::make_map(&mw, W, N, K, ldw, 128, i8);
  if (rc) return rc;
  rc = tc::make_map(&mx, X, M, K, ldx, Na, i8);
  if (rc) return rc;
  const bool lnx = ep.lnx != nullptr;
  if (lnx && (K % 128 || K > 1024 || ep.kind == SKB_EPI_RESID || ep.kind == SKB_EPI_SSRU))
    return fail(SKB_ERR_CONFIG, "gemm_sw: prologue LayerNorm needs K %% 128 == 0 <= 1024");
  const int SB = lnx ? W_BYTES : W_BYTES + Na * 128;
  const int kbe = i8 ? 2 * tc::BK : tc::BK;
  const int nk = (K + kbe - 1) / kbe;
  const int nkc = (nk + CS - 1) / CS;
  const int panel_bytes = lnx ? nkc * Na * 128 : 0;  // this CTA's k-blocks
  const int arecv_bytes = push_small(Na, CS) ? Na * 512 : 0;  // st.async receive area
  const int smask_bytes = (ep.kind == SKB_EPI_LOGITS && ep.mask) ? Na * 16 : 0;  // staged mask words
  const int fixed = panel_bytes + arecv_bytes + smask_bytes + 1024 + 512;
  // TMA-store epilogue: the output tile is staged in the (drained) ring
  const bool f32o = ep.kind == SKB_EPI_RESID || ep.out_dtype == SKB_F32;
  const int es = f32o ? 4 : 2;
  // SSRU with whole-K tiles (mode 2): cells and relu(cells) staged, written
  // by a TMA store into the step's half of the cell buffer and a TMA
  // reduce-add into x (c_next rows = M; ld and pitches 16-byte aligned)
  const bool ssru_tma = ep.kind == SKB_EPI_SSRU && CS == 1 && ep.c_next &&
                        (reinterpret_cast<uintptr_t>(ep.out) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(ep.c_next) & 15) == 0 && ep.ldo % 4 == 0 &&
                        ep.ld_state % 4 == 0 && ep.state_stride % 4 == 0 && N % 2 == 0 && N / 2 <= ep.ld_state &&
                        (!ep.step || ep.state_stride >= (long long)M * ep.ld_state) && Na <= 256;
  const int tma_out = ssru_tma ? 2
                               : (ep.kind != SKB_EPI_SSRU && (reinterpret_cast<uintptr_t>(ep.out) & 15) == 0 &&
                                  ((long)ep.ldo * es) % 16 == 0);
  const int rows_box = CS == 1 ? Na : Na / CS;
  const int part_bytes = CS > 1 ? 2 * Na * 512 : 0;  // partial + receive slots
  const int stg_off = (part_bytes + 1023) & ~1023;
  const int need = ssru_tma ? Na * 512
                            : (tma_out ? stg_off + ((rows_box + 15) / 16 * 16) * 128 * es : part_bytes);
  // Ring budget: half the SM by default, so the next kernel's CTA (PDL)
  // can become resident beside this one and prefetch its weights while this
  // one drains; the per-SM TMA ingest (~80-120 GB/s) is already reached
  // with ~100 KB in flight.  SKB_SW_SMEM overrides (bytes).
  static int budget = -1;
  if (budget < 0) {
    const char *e = getenv("SKB_SW_SMEM");
    budget = e ? atoi(e) : 113 * 1024;
    if (budget > SMEM_MAX) budget = SMEM_MAX;
  }
  int stages = (budget - fixed) / SB;
  if (stages < 2) stages = 2;
  if (stages > nkc) stages = nkc;
  if (stages * SB < need) stages = (need + SB - 1) / SB;
  if (stages < 1 || stages * SB + fixed > SMEM_MAX)
    return fail(SKB_ERR_UNSUPPORTED, "gemm_sw: Na=%d CS=%d does not fit", Na, CS);
  const size_t smem = (size_t)stages * SB + fixed;
  OutMaps mo;
  mo.a = mo.b = mw;  // (unused unless set below)
  if (ssru_tma) {
    rc = make_map_ssru(&mo.a, ep.out, M, N / 2, ep.ldo, 1, 0, Na);
    if (rc) return rc;
    rc = make_map_ssru(&mo.b, ep.c_next, M, N / 2, ep.ld_state, ep.step ? 2 : 1, ep.state_stride, Na);
    if (rc) return rc;
  } else if (tma_out) {
    rc = make_map_out(&mo.a, ep.out, M, N, ep.ldo, f32o, rows_box);
    if (rc) return rc;
  }
  if (i8) {
    if (ep.kind == SKB_EPI_RELU)
      return launch_t<SKB_EPI_RELU, 1, false, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
    if (ep.kind == SKB_EPI_RESID)
      return launch_t<SKB_EPI_RESID, 1, false, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
    return launch_t<SKB_EPI_STORE, 1, false, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
  }
  switch (ep.kind) {
    case SKB_EPI_RELU:
      return launch_k2<SKB_EPI_RELU>(M, N, K, mw, mx, mo, Na, CS, stages, stg_off, tma_out, smem, ep, st);
    case SKB_EPI_RESID:
      return launch_k2<SKB_EPI_RESID>(M, N, K, mw, mx, mo, Na, CS, stages, stg_off, tma_out, smem, ep, st);
    case SKB_EPI_SSRU:
      return launch_k2<SKB_EPI_SSRU>(M, N, K, mw, mx, mo, Na, CS, stages, stg_off, tma_out, smem, ep, st);
    case SKB_EPI_LOGITS:
      if (CS != 1 || !tma_out) return fail(SKB_ERR_CONFIG, "gemm_sw: LOGITS needs CS=1 and TMA output");
      if (ep.lnx)
        return launch_t<SKB_EPI_LOGITS, 1, true>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep,
                                                 st);
      return launch_t<SKB_EPI_LOGITS, 1>(M, N, K, mw, mx, mo, Na, stages, stg_off, tma_out, smem, ep, st);
    default:
      return launch_k2<SKB_EPI_STORE>(M, N, K, mw, mx, mo, Na, CS, stages, stg_off, tma_out, smem, ep, st);
  }
}

// Cluster split CS from (N, K) only (numerics must not depend on M).
// Measured on B200 at M = 640 (tools/gemm_sweep.py): the bulk-copy
// reduction costs ~3-4 us, so only long-K shapes (FFN2, K = 4096) split.
static int pick_cs(int N, int K) {
  const int nk = (K + tc::BK - 1) / tc::BK;
  const int n_wt = (N + 127) / 128;
  // Long-K shapes (FFN2, K = 4096): whole-K tiles.  Measured on B200
  // (bench, 3 decode streams, profiles/r2_55_exp.txt, r2_56_exp.txt): split
  // 4 -> 5070, 2 -> 5400, 1 -> 5476 sentences/s, single stream 3131 / 3121 /
  // 2914; with the >= 128-row tiles under concurrency (pick_na), which a
  // cluster split cannot use (its partial buffers cap Na at 80), 5 streams
  // 5898 (split 2) -> 6190 (split 1), single stream 3160 -> 2944
  // (profiles/r2_149_longk_split_ab.txt).  A function of (N, K) only, as
  // batch invariance requires.  SKB_CS_LONGK overrides.
  static int long_k = -1;
  if (long_k < 0) {
    const char *e = getenv("SKB_CS_LONGK");
    long_k = e ? atoi(e) : 1;
  }
  if (nk >= 48 && n_wt <= 16) return long_k;
  // K = 2048-class shapes of narrow N (base FFN2: N 512, K 2048) split in
  // 2 as well: base beam-5 b64 +0.9 % at 5 streams, +3 % single stream
  // (profiles/r2_103_var.txt).  SKB_CS_MIDK overrides.
  static int mid_k = -1;
  if (mid_k < 0) {
    const char *e = getenv("SKB_CS_MIDK");
    mid_k = e ? atoi(e) : 2;
  }
  if (mid_k > 1 && nk >= 32 && n_wt <= 8) return mid_k;
  // SKB_CS_SMALLN=2|4 also splits the narrow K = 1024 shapes (wo, wo_c):
  // still a function of (N, K) only, a latency / throughput trade-off —
  // measured on B200: 4 gives batch-1 greedy 21.4 ms (from 23.5) but costs
  // 16 % of the multi-stream throughput (cluster reduction at M = 640).
  static int small_n = -1;
  if (small_n < 0) {
    const char *e = getenv("SKB_CS_SMALLN");
    small_n = e ? atoi(e) : 1;
  }
  if (small_n > 1 && n_wt <= 8 && nk >= 16) return small_n;
  return 1;
}

// Activation tile Na for the actual M (numerics do not depend on it).  Cost
// model fitted to the tools/gemm_sweep.py sweep on B200 (M = 64..1280): two
// CTAs co-reside per SM (113 KB ring), each streams (128 + Na) rows of K,
// plus a fixed per-CTA cost worth ~160 rows; CTA slots beyond one wave
// cost proportionally.

static int pick_na(int M, int N, int CS, int conc) {
  // with several decode streams in flight each GEMM gets a share of the SMs:
  // fewer, larger tiles ingest fewer bytes in total
  const int slots = 2 * tc::num_sms() / (conc > 0 ? conc : 1);
  const int n_wt = (N + 127) / 128;
  const int na_max = CS > 1 ? 80 : 160;  // split-K partial + receive slots fit the ring
  // Smallest tile worth issuing: a 128 x Na x 16 tcgen05.mma costs the same
  // ~71 cycles for every Na <= 128 (profiles/r2_136_gemm_mainloop_findings.txt),
  // so with several decode streams sharing the SMs (total tensor work, not
  // one GEMM's latency, is what counts) tiles of >= 128 rows issue 2-8x
  // fewer instructions for the same work: big 6-6 at 5 streams (M = 640)
  // 5703 -> 5791 sentences/s (r2_140).  One stream keeps the one-wave small
  // tiles (3160 vs 2893), and so do GEMMs of < 512 rows, whose few tiles
  // leave SMs idle (base b64 at M = 320 8096 -> 7943, SSRU greedy at
  // M = 128 20292 -> 19636 with the floor, r2_141).  Numerics do not depend
  // on Na.  SKB_SW_NA_MIN overrides.
  static int na_env = -2;
  if (na_env == -2) {
    const char *e = getenv("SKB_SW_NA_MIN");
    na_env = e ? atoi(e) : -1;
  }
  int na_floor = na_env >= 0 ? na_env : (conc > 1 && M >= 512 ? 128 : 16);
  if (na_floor > (M + 15) / 16 * 16) na_floor = (M + 15) / 16 * 16;
  int best = 16;
  double best_c = 1e30;
  for (int na = 16; na <= na_max; na += 16) {
    if (na < na_floor && na + 16 <= na_max && (long)n_wt * ((M + na - 1) / na) > 1) continue;
    if (CS > 1 && na % CS) continue;
    if (CS >= 8 && !push_small(na, CS)) continue;  // wide clusters: power-of-two slices only
    const double ctas = (double)n_wt * ((M + na - 1) / na) * CS;
    const double waves = ctas <= slots ? 1.0 : ctas / slots;
    const double c = waves * (128.0 + na + 160.0);
    if (c < best_c * 0.999) {
      best_c = c;
      best = na;
    }
  }
  return best;
}

// Largest M whose input LayerNorm runs in the GEMM prologue (every CTA
// normalises its own activation rows; beyond this the redundant row reads
// cost more than the LayerNorm launch they save).  SKB_LN_PROLOGUE_MAX.
static int lnx_max_rows() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("SKB_LN_PROLOGUE_MAX");
    v = e ? atoi(e) : 32;
  }
  return v;
}

thread_local int g_mode = -1, g_na = 0, g_cs = 0;  // test overrides; mode: 0 auto, 1 never, 2 always
void init_mode() {
  if (g_mode >= 0) return;
  const char *e = getenv("SKB_GEMM_SW");
  g_mode = e ? atoi(e) : 0;
}

}  // namespace sw

// ====================================== persistent CTA-pair GEMM (pc)
// The swap-AB layout of the sw kernel (weight rows on the MMA M side,
// activation rows on N) run by CTA pairs: tcgen05.mma.cta_group::2 with
// M = 256 weight rows (128 per SM, each from its own shared memory) and
// N = Na activation rows (Na/2 per SM, read by the MMA from both SMs), so a
// pair ingests (256 + Na) rows of K per tile instead of 2 x (128 + Na): the
// L2->SM bytes per FLOP drop by up to 2x, which is what bounds the decode
// GEMMs at M = 640 (per-SM TMA ingest).  The grid is
// persistent (a pair loops over tiles; M-tiles fastest so the pairs working
// at the same time share a weight tile in L2) and TMEM holds two
// accumulators, so the epilogue of tile i (TMEM -> registers -> 32-row
// staged chunks -> TMA store / TMA reduce-add) overlaps the MMAs of tile i+1
// and the per-CTA prologue is paid once per launch.
//   warp 0     : TMA producer (one lane) in both CTAs; the loads of both
//                CTAs complete on the leader's full barrier
//   warp 1     : MMA issuer (one lane of the leader CTA only)
//   warps 2..5 : epilogue in both CTAs (TMEM lane quarter = warp % 4)
// Every output element is one K-ordered tcgen05 accumulation, exactly as in
// the sw kernel with CS = 1, so the two kernels produce identical bits
// (tests/test_gemm_gpu.py::test_pair_kernel_bitwise_equal_sw) and the choice
// between them may depend on M without breaking batch invariance.
namespace pc {

using namespace tc;
#ifdef SKB_GEMM_TRACE
#define PC_STAMP(slot)                                                  \
  do {                                                                  \
    unsigned long long _t;                                              \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));              \
    if (blockIdx.x < 1024) sw::g_trace[blockIdx.x * 16 + (slot)] = _t;  \
  } while (0)
#else
#define PC_STAMP(slot) \
  do {                 \
  } while (0)
#endif
constexpr int CHUNK = 32;                       // activation rows per staged store
constexpr int STG_BYTES = CHUNK * 128 * 4;      // one fp32 staging buffer
constexpr uint16_t PAIR = 0x3;

__device__ __forceinline__ void tma_load_pair(void *dst, const CUtensorMap *map, int c0, int c1,
                                              uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}

__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// arrive on the barrier at the same offset in both CTAs of the pair once
// every MMA issued so far has completed
__device__ __forceinline__ void commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(PAIR)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
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
}

template <int KIND>
__global__ void __launch_bounds__(192, 1)
    k_gemm_pc(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
              const __grid_constant__ CUtensorMap tmO, int M, int N, int K, int Na, int stages,
              int tcols, int tma_out, EpiArgs ep) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int XB = (Na >> 1) * 128;  // this CTA's half of an activation k-block
  const int SB = sw::W_BYTES + XB;
  uint8_t *stg = smem + stages * SB;  // 2 staging buffers (1024-aligned: SB is)
  uint64_t *full = reinterpret_cast<uint64_t *>(stg + 2 * STG_BYTES);
  uint64_t *empty = full + stages;
  uint64_t *tfull = empty + stages;  // [2] accumulator ready (both CTAs)
  uint64_t *tempty = tfull + 2;      // [2] accumulator drained (leader: 8 arrivals)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = (int)blockIdx.x >> 1, npairs = (int)gridDim.x >> 1;
  const int n_at = (M + Na - 1) / Na;
  const int n_wt = (N + 255) / 256;
  const int tiles = n_at * n_wt;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    PC_STAMP(0);
#pragma unroll 1
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
    if (tma_out)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmO)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) PC_STAMP(1);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t lfull = sw::mapa(smem_u32(full), 0);  // leader's full[0]
      const uint32_t tx = 2u * (uint32_t)SB;
      // PDL prologue: the first tile's weight k-blocks do not depend on the
      // previous kernel; activations only after griddepcontrol.wait
      int pre = 0;
      if (pair < tiles) {
        const int n0 = (pair / n_at) * 256 + (int)rank * 128;
        pre = nk < stages ? nk : stages;
#pragma unroll 1
        for (int q = 0; q < pre; ++q) {
          if (rank == 0) mbar_expect_tx(&full[q], tx);
          tma_load_pair(smem + q * SB, &tmW, q * BK, n0, lfull + 8u * q);
        }
      }
      pdl_wait();
      pdl_trigger();
      PC_STAMP(2);
      int it = 0;
#pragma unroll 1
      for (int t = pair; t < tiles; t += npairs) {
        const int at = t % n_at, wt = t / n_at;
        const int n0 = wt * 256 + (int)rank * 128;
        const int mx = at * Na + (int)rank * (Na >> 1);
#pragma unroll 1
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % stages;
          uint8_t *st = smem + s * SB;
          if (it >= pre) {
            mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
            if (rank == 0) mbar_expect_tx(&full[s], tx);
            tma_load_pair(st, &tmW, kb * BK, n0, lfull + 8u * s);
          }
          tma_load_pair(st + sw::W_BYTES, &tmX, kb * BK, mx, lfull + 8u * s);
        }
      }
    } else {
      pdl_wait();
    }
  } else if (warp == 1) {
    pdl_wait();
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = idesc_bf16(256, Na);
      int it = 0, local = 0;
#pragma unroll 1
      for (int t = pair; t < tiles; t += npairs, ++local) {
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(acc * Na);
#pragma unroll 1
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(&full[s], (it / stages) & 1);
          if (it == 0) PC_STAMP(3);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t *st = smem + s * SB;
          const uint64_t da = umma_desc_sw128(st);
          const uint64_t db = umma_desc_sw128(st + sw::W_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_pair(d, da + 2 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          commit_pair(&empty[s]);
        }
        commit_pair(&tfull[acc]);
        if (local == 0) PC_STAMP(4);
      }
    }
  } else {
    // ---- epilogue warps 2..5: output column n (weight row) per thread
    pdl_wait();
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const bool leader = warp == 2 && lane == 0;
    const uint32_t stg0 = smem_u32(stg);
    const uint32_t ltempty = sw::mapa(smem_u32(tempty), 0);
    const bool bf16 = ep.out_dtype == SKB_BF16 && KIND != SKB_EPI_RESID;
    const float *cprev = nullptr;
    float *cnext = nullptr;
    if (KIND == SKB_EPI_SSRU) {
      cprev = ep.c_prev;
      cnext = ep.c_next;
      if (ep.step) {  // decode-loop double buffer selected by step parity
        const int t = *ep.step;
        cnext = ep.c_next + (t & 1) * ep.state_stride;
        cprev = t == 0 ? nullptr : ep.c_next + ((t + 1) & 1) * ep.state_stride;
      }
    }
    int local = 0, chunk = 0;
#pragma unroll 1
    for (int t = pair; t < tiles; t += npairs, ++local) {
      const int at = t % n_at, wt = t / n_at;
      const int m0 = at * Na;
      const int n0 = wt * 256 + (int)rank * 128;
      const int n = n0 + row;
      const bool nok = n < N;
      const float bn = (ep.bias && nok) ? __ldg(ep.bias + n) : 0.f;
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      if (local == 0 && leader) PC_STAMP(5);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tb = tmem + (uint32_t)(acc * Na) + ((uint32_t)(quarter * 32) << 16);
      const int rows = min(Na, M - m0);
#pragma unroll 1
      for (int c = 0; c < rows; c += CHUNK, ++chunk) {
        uint32_t r[32];
        tmem_ld32_nowait(tb + (uint32_t)c, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c + CHUNK >= rows) {  // last TMEM read of this tile: release the accumulator
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(ltempty + 8u * acc);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (KIND == SKB_EPI_SSRU || !tma_out) {
          sw::epi16<KIND>(ep, cprev, cnext, M, m0 + c, n, nok, bn, v);
          sw::epi16<KIND>(ep, cprev, cnext, M, m0 + c + 16, n, nok, bn, v + 16);
          continue;
        }
        // staging buffer chunk&1: the store issued from it two chunks ago
        // must have finished reading it
        if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const uint32_t sb = stg0 + (uint32_t)((chunk & 1) * STG_BYTES);
        sw::stage16<KIND>(sb, bf16, 0, row, bn, v);
        sw::stage16<KIND>(sb, bf16, 16, row, bn, v + 16);
        sw::flush_tile<KIND>(&tmO, sb, n0, m0 + c, leader, [] {}, false, true);
        if constexpr (KIND == SKB_EPI_LOGITS)
          sw::logits_stats(ep, sb, M, N, m0 + c, n0, CHUNK, warp - 2, lane);
      }
      if (local == 0 && leader) PC_STAMP(6);
    }
    if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (leader) PC_STAMP(8);
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // no MMA / remote arrive into a CTA that has left
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef SKB_GEMM_TRACE
  if (threadIdx.x == 0) {
    PC_STAMP(9);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (blockIdx.x < 1024) sw::g_trace[blockIdx.x * 16 + 7] = smid;
  }
#endif
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

thread_local int g_pairs = -1;  // SKB_PC_PAIRS: pairs per launch (0 = automatic)

template <int KIND>
static int launch_t(int M, int N, int K, const CUtensorMap &mw, const CUtensorMap &mx,
                    const CUtensorMap &mo, int Na, int stages, int tcols, int tma_out, size_t smem,
                    int pairs, EpiArgs ep, cudaStream_t st) {
  ensure_smem_fn(k_gemm_pc<KIND>, sw::SMEM_MAX);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  int na = 1;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k_gemm_pc<KIND>, mw, mx, mo, M, N, K, Na, stages, tcols, tma_out, ep);
  SKB_CHECK_LAUNCH("k_gemm_pc");
  return SKB_OK;
}

// Activation tile Na (numerics do not depend on it) and pairs per launch:
// a pair's tile time is max(MMA, TMA ingest of (256 + Na) rows of K) plus a
// fixed cost; tiles run in ceil(tiles / pairs) rounds on the pairs this
// call's share of the SMs provides.
static void pick(int M, int N, int K, int conc, int &Na, int &pairs) {
  const int nsm = tc::num_sms();
  int maxp = nsm / 2 / (conc > 0 ? conc : 1);
  if (maxp < 1) maxp = 1;
  if (g_pairs < 0) {
    const char *e = getenv("SKB_PC_PAIRS");
    g_pairs = e ? atoi(e) : 0;
  }
  if (g_pairs > 0) maxp = g_pairs < nsm / 2 ? g_pairs : nsm / 2;
  const int n_wt = (N + 255) / 256;
  double best = 1e30;
  Na = 256;
  for (int na = 32; na <= 256; na += 32) {
    const long tiles = (long)n_wt * ((M + na - 1) / na);
    const long p = tiles < maxp ? tiles : maxp;
    const long rounds = (tiles + p - 1) / p;
    // per SM per k-block: 16 KB weights + na/2 activation rows; MMA of a
    // 256 x na x 64 block on the pair ~ na/2 ns-equivalents
    const double ingest = 16384.0 + na * 64.0;
    const double mma = na * 128.0;  // bytes-equivalent at ~64 B/clk ingest
    const double c = rounds * ((ingest > mma ? ingest : mma) * ((K + 63) / 64) + 48.0 * 1024);
    if (c < best * 0.999) {
      best = c;
      Na = na;
    }
  }
  const long tiles = (long)n_wt * ((M + Na - 1) / Na);
  pairs = (int)(tiles < maxp ? tiles : maxp);
}

thread_local int g_mode = -1;   // SKB_GEMM_PC: 0 auto, 1 never, 2 always (where applicable)
thread_local int g_na = 0;      // forced activation tile (0 = automatic)
thread_local int g_min_m = -1;  // SKB_PC_MIN_M: smallest M the automatic choice sends here
void init_mode() {
  if (g_mode >= 0) return;
  const char *e = getenv("SKB_GEMM_PC");
  g_mode = e ? atoi(e) : 0;
  e = getenv("SKB_PC_MIN_M");
  g_min_m = e ? atoi(e) : 1024;
}

static int launch(int M, int N, int K, const void *X, int ldx, const void *W, int ldw, EpiArgs ep,
                  cudaStream_t st, int conc, int na_force) {
  ep.splits = 1;
  ep.late_trigger = 0;
  int Na, pairs;
  pick(M, N, K, conc, Na, pairs);
  if (na_force > 0) {
    Na = na_force;
    const long tiles = (long)((N + 255) / 256) * ((M + Na - 1) / Na);
    if (pairs > tiles) pairs = (int)tiles;
  }
  if (Na < 32 || Na > 256 || Na % 32) return fail(SKB_ERR_CONFIG, "gemm_pc: bad tile Na=%d", Na);
  CUtensorMap mw, mx, mo;
  int rc = tc::make_map(&mw, W, N, K, ldw, 128);
  if (rc) return rc;
  rc = tc::make_map(&mx, X, M, K, ldx, Na / 2);
  if (rc) return rc;
  const bool f32o = ep.kind == SKB_EPI_RESID || ep.out_dtype == SKB_F32;
  const int es = f32o ? 4 : 2;
  const int tma_out = ep.kind != SKB_EPI_SSRU && (reinterpret_cast<uintptr_t>(ep.out) & 15) == 0 &&
                      ((long)ep.ldo * es) % 16 == 0;
  if (ep.kind == SKB_EPI_LOGITS && !tma_out)
    return fail(SKB_ERR_CONFIG, "gemm_pc: LOGITS needs an aligned fp32 output");
  if (tma_out) {
    rc = sw::make_map_out(&mo, ep.out, M, N, ep.ldo, f32o, CHUNK);
    if (rc) return rc;
  } else {
    mo = mw;  // unused
  }
  const int SB = sw::W_BYTES + (Na / 2) * 128;
  const int nk = (K + tc::BK - 1) / tc::BK;
  const int fixed = 2 * STG_BYTES + 1024 + 256;
  static int budget = -1;  // SKB_PC_SMEM: shared-memory budget per CTA (bytes)
  if (budget < 0) {
    const char *e = getenv("SKB_PC_SMEM");
    budget = e ? atoi(e) : sw::SMEM_MAX;
    if (budget > sw::SMEM_MAX) budget = sw::SMEM_MAX;
  }
  int stages = (budget - fixed) / SB;
  if (stages < 2) return fail(SKB_ERR_UNSUPPORTED, "gemm_pc: Na=%d does not fit", Na);
  if (stages > nk) stages = nk;
  if (stages > 8) stages = 8;
  const size_t smem = (size_t)stages * SB + fixed;
  int tcols = 32;
  while (tcols < 2 * Na) tcols <<= 1;
  switch (ep.kind) {
    case SKB_EPI_RELU:
      return launch_t<SKB_EPI_RELU>(M, N, K, mw, mx, mo, Na, stages, tcols, tma_out, smem, pairs, ep, st);
    case SKB_EPI_RESID:
      return launch_t<SKB_EPI_RESID>(M, N, K, mw, mx, mo, Na, stages, tcols, tma_out, smem, pairs, ep, st);
    case SKB_EPI_SSRU:
      return launch_t<SKB_EPI_SSRU>(M, N, K, mw, mx, mo, Na, stages, tcols, tma_out, smem, pairs, ep, st);
    case SKB_EPI_LOGITS:
      return launch_t<SKB_EPI_LOGITS>(M, N, K, mw, mx, mo, Na, stages, tcols, tma_out, smem, pairs, ep, st);
    default:
      return launch_t<SKB_EPI_STORE>(M, N, K, mw, mx, mo, Na, stages, tcols, tma_out, smem, pairs, ep, st);
  }
}

}  // namespace pc

// ========================================================== SIMT kernel
// 64x64 output tile, BK=16, 256 threads, 4x4 outputs per thread.  Used for
// fp32 (parity) mode and for shapes TMA cannot describe.
template <typename T>
__global__ void __launch_bounds__(256) k_gemm_simt(int M, int N, int K, const T *__restrict__ A,
                                                   int lda, const T *__restrict__ W, int ldw,
                                                   EpiArgs ep) {
  PDL_ENTRY();
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
  a.splits = 1;
  a.ws = e->splitk_ws;
  a.counters = e->splitk_counters;
  a.ln_gain = e->ln_gain;
  a.ln_bias = e->ln_bias;
  a.ln_eps = e->ln_eps;
  a.ln_out = reinterpret_cast<__nv_bfloat16 *>(e->ln_out);
  a.ln_ldo = e->ln_ldo;
  a.ln_counter = e->ln_counter;
  if (e->kind != SKB_EPI_RESID) a.ln_out = nullptr;
  a.lnx = nullptr;  // set by gemm_impl when the prologue LayerNorm is used
  a.lnx_ld = e->ln_in_ld;
  a.lnx_g = e->ln_in_gain;
  a.lnx_b = e->ln_in_bias;
  a.lnx_eps = e->ln_in_eps;
  a.late_trigger = 0;
  a.a_scale = nullptr;
  a.w_scale = nullptr;
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
    launch_k(k_gemm_simt<float>, grid, 256, 0, st, M, N, K, (const float *)A, lda, (const float *)W, ldw, ep);
  else
    launch_k(k_gemm_simt<__nv_bfloat16>, grid, 256, 0, st, M, N, K, (const __nv_bfloat16 *)A, lda,
                                                     (const __nv_bfloat16 *)W, ldw, ep);
  SKB_CHECK_LAUNCH("k_gemm_simt");
  return SKB_OK;
}

}  // namespace skb

using namespace skb;

// A residual GEMM with a requested LayerNorm that did not run on the
// swap-AB kernel (which fuses it) is followed by the LN kernel.
static thread_local int g_last_launches = 0;

// A = LN(ln_in) as its own launch (large M, SIMT and tc paths)
static int ln_before(int in_dtype, int M, int K, const void *A, int lda, const skb_epilogue *epi,
                     void *stream) {
  ++g_last_launches;
  return skb_layernorm(M, K, epi->ln_in, epi->ln_in_ld, epi->ln_in_gain, epi->ln_in_bias,
                       epi->ln_in_eps, const_cast<void *>(A), lda, in_dtype, stream);
}

extern "C" int skb_last_launches(void) { return g_last_launches; }

static int ln_after(int M, int N, const skb_epilogue *epi, void *stream) {
  ++g_last_launches;
  return skb_layernorm(M, N, reinterpret_cast<const float *>(epi->out), epi->ldo, epi->ln_gain,
                       epi->ln_bias, epi->ln_eps, epi->ln_out, epi->ln_ldo, SKB_BF16, stream);
}

extern "C" int skb_tc_available(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0 && tc::encode_fn() != nullptr) ? 1 : 0;
}

extern "C" int skb_gemm_force(int bn, int cs, int splits) {
  tc::init_forces();
  tc::g_force_bn = bn;
  tc::g_force_cs = cs;
  tc::g_force_s = splits;
  return SKB_OK;
}

extern "C" int skb_gemm_force_sw(int mode, int na, int cs) {
  sw::init_mode();
  sw::g_mode = mode;
  sw::g_na = na;
  sw::g_cs = cs;
  return SKB_OK;
}

// int8 GEMM for the quantized feed-forward layers (quant.py:65-132):
// acc[m, n] = sum_k A[m, k] * W[n, k] exactly in int32 (tcgen05 kind::i8),
// then out = (float32(acc) * a_scale[m]) * w_scale[n] with the epilogue's
// bias / ReLU / residual add.  A, W int8 K-major; K % 16 == 0.
extern "C" int skb_gemm_i8(int M, int N, int K, const void *A, int lda, const float *a_scale,
                           const void *W, int ldw, const float *w_scale, const skb_epilogue *epi,
                           void *stream) {
  if (M < 0 || N <= 0 || K <= 0) return fail(SKB_ERR_SHAPE, "gemm_i8: bad shape M=%d N=%d K=%d", M, N, K);
  if (!A || !W || !a_scale || !w_scale || !epi || !epi->out) return fail(SKB_ERR_SHAPE, "gemm_i8: null operand");
  if (K % 16 || lda % 16 || ldw % 16 || (reinterpret_cast<uintptr_t>(A) & 15) ||
      (reinterpret_cast<uintptr_t>(W) & 15))
    return fail(SKB_ERR_CONFIG, "gemm_i8: K, leading dims and bases must be 16-byte aligned");
  if (K > (int)(2147483648LL / (127 * 127))) return fail(SKB_ERR_CONFIG, "gemm_i8: K=%d overflows int32", K);
  if (epi->kind != SKB_EPI_STORE && epi->kind != SKB_EPI_RELU && epi->kind != SKB_EPI_RESID)
    return fail(SKB_ERR_CONFIG, "gemm_i8: STORE, RELU or RESID epilogue only");
  if (epi->kind == SKB_EPI_RESID && epi->out_dtype != SKB_F32)
    return fail(SKB_ERR_CONFIG, "gemm_i8: residual target must be fp32");
  g_last_launches = 1;
  if (M == 0) return SKB_OK;
  EpiArgs ep = to_args(epi);
  ep.ln_out = nullptr;
  ep.a_scale = a_scale;
  ep.w_scale = w_scale;
  const int conc = epi->streams > 0 ? epi->streams : 1;
  const int na = sw::g_na > 0 ? sw::g_na : sw::pick_na(M, N, 1, conc);
  return sw::launch(M, N, K, A, lda, W, ldw, ep, as_stream(stream), na, 1, conc, true);
}

extern "C" int skb_gemm_force_pc(int mode, int na, int pairs) {
  if (mode < 0 || mode > 2 || na < 0 || na > 256 || na % 32 || pairs < 0)
    return fail(SKB_ERR_CONFIG, "gemm_force_pc: mode %d na %d pairs %d", mode, na, pairs);
  pc::init_mode();
  pc::g_mode = mode;
  pc::g_na = na;
  pc::g_pairs = pairs;
  return SKB_OK;
}

extern "C" int skb_debug_gemm_trace(unsigned long long *host) {
#ifdef SKB_GEMM_TRACE
  cudaMemcpyFromSymbol(host, sw::g_trace, sizeof(sw::g_trace));
  static unsigned long long zeros[1024 * 16];
  cudaMemcpyToSymbol(sw::g_trace, zeros, sizeof(zeros));  // read-and-clear
  return SKB_OK;
#else
  (void)host;
  return SKB_ERR_UNSUPPORTED;
#endif
}

extern "C" int skb_gemm_simt(int in_dtype, int M, int N, int K, const void *A, int lda,
                             const void *W, int ldw, const skb_epilogue *epi, void *stream) {
  int rc = check_args(in_dtype, M, N, K, A, W, epi);
  if (rc) return rc;
  if (M == 0) return SKB_OK;
  g_last_launches = 1;
  if (epi->ln_in) {
    rc = ln_before(in_dtype, M, K, A, lda, epi, stream);
    if (rc) return rc;
  }
  rc = gemm_simt(in_dtype, M, N, K, A, lda, W, ldw, to_args(epi), as_stream(stream));
  if (rc) return rc;
  if (epi->kind == SKB_EPI_RESID && epi->ln_out) return ln_after(M, N, epi, stream);
  return SKB_OK;
}

static int gemm_impl(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
                     int ldw, const skb_epilogue *epi, void *stream, bool &fused_ln);

extern "C" int skb_gemm(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
                        int ldw, const skb_epilogue *epi, void *stream) {
  bool fused = false;
  g_last_launches = 1;
  const int rc = gemm_impl(in_dtype, M, N, K, A, lda, W, ldw, epi, stream, fused);
  if (rc || M == 0) return rc;
  if (epi->kind == SKB_EPI_RESID && epi->ln_out && !fused) return ln_after(M, N, epi, stream);
  return SKB_OK;
}

static int gemm_impl(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
                     int ldw, const skb_epilogue *epi, void *stream, bool &fused_ln) {
  int rc = check_args(in_dtype, M, N, K, A, W, epi);
  if (rc) return rc;
  if (!(epi->k_split == 0 || epi->k_split == 1 || epi->k_split == 2 || epi->k_split == 4 ||
        epi->k_split == 8 || epi->k_split == 16))
    return fail(SKB_ERR_CONFIG, "gemm: k_split %d not in {0, 1, 2, 4, 8, 16}", epi->k_split);
  if (M == 0) return SKB_OK;
  EpiArgs ep = to_args(epi);
  cudaStream_t st = as_stream(stream);
  const bool tma_ok = in_dtype == SKB_BF16 && K % 8 == 0 && lda % 8 == 0 && ldw % 8 == 0 &&
                      (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(W) & 15) == 0;
  if (!tma_ok) {
    if (epi->ln_in) {
      rc = ln_before(in_dtype, M, K, A, lda, epi, stream);
      if (rc) return rc;
    }
    return gemm_simt(in_dtype, M, N, K, A, lda, W, ldw, ep, st);
  }
  // decode-sized M: swap-AB kernel (weights on the MMA M side)
  sw::init_mode();
  const bool logits_tma = epi->kind != SKB_EPI_LOGITS ||
                          ((reinterpret_cast<uintptr_t>(epi->out) & 15) == 0 && epi->ldo % 4 == 0);
  const bool ln_fused = epi->kind == SKB_EPI_RESID && epi->ln_out != nullptr;
  if (ln_fused && (!epi->ln_gain || !epi->ln_bias || !epi->ln_counter || N % 128 || N > 1024 ||
                   epi->ln_ldo % 4))
    return fail(SKB_ERR_CONFIG, "gemm: fused LayerNorm needs gain/bias/counter, N %% 128 == 0 <= 1024");
  // The swap-AB kernel serves every M (measured on B200, tools/tcsw_check.py:
  // 1.3-2x faster than the M-major kernel up to M = 3840, except the
  // K = 4096 residual GEMM beyond ~2.5k rows, 69 vs 51 us).  One kernel for
  // every M is what keeps a sentence's numbers independent of its batch:
  // the kernels' plain GEMM results are bitwise equal, but the swap-AB one
  // splits K = 4096 over a 4-CTA cluster (a different fp32 summation order)
  // and reduces the LOGITS partials in another order — with an M threshold
  // the encoder's FFN2 of a large batch (B*L rows) and the log-softmax of a
  // large decode batch took the other kernel (tools/invariance_check.py).
  const bool sw_pref = true;
  // Persistent CTA-pair kernel for the shapes whose sw plan has no cluster
  // K-split (identical bits, see namespace pc) once M is large enough that
  // its bigger tiles pay; below that the sw kernel's one-tile-per-CTA plan
  // (and its prologue LayerNorm) has the shorter critical path.
  pc::init_mode();
  const int conc = epi->streams > 0 ? epi->streams : 1;  // decode streams sharing the GPU
  // K split: the caller's (a function of the weight matrix, see
  // skb_epilogue.k_split) or the library's (N, K) rule
  int ksplit = epi->kind == SKB_EPI_LOGITS ? 1 : (epi->k_split > 0 ? epi->k_split : sw::pick_cs(N, K));
  while (ksplit > 1 && (K + tc::BK - 1) / tc::BK < ksplit) ksplit >>= 1;  // >= 1 k-block per partial
  {
    const int cs_sw = ksplit;
    const bool pc_ok = cs_sw == 1 && logits_tma && sw::g_mode == 0;
    // automatic: wide plain GEMMs of large M (the cross-attention K/V
    // projection of a batch, N = 2 d D); the LOGITS epilogue measured slower
    // on the pair kernel (126.6 vs 116.1 us at M = 1280, profiles/r2_05_*)
    static int pc_min_n = -1;  // SKB_PC_MIN_N: narrowest N the automatic choice sends here
    if (pc_min_n < 0) {
      const char *e = getenv("SKB_PC_MIN_N");
      pc_min_n = e ? atoi(e) : 8192;
    }
    const bool pc_auto = M >= pc::g_min_m && N >= pc_min_n && epi->kind != SKB_EPI_LOGITS;
    if (pc_ok && (pc::g_mode == 2 || (pc::g_mode == 0 && pc_auto))) {
      if (epi->ln_in) {
        rc = ln_before(in_dtype, M, K, A, lda, epi, stream);
        if (rc) return rc;
      }
      fused_ln = false;  // a requested output LayerNorm follows as its own launch
      return pc::launch(M, N, K, A, lda, W, ldw, ep, st, conc, pc::g_na);
    }
  }
  if (sw::g_mode != 1 && logits_tma && (sw::g_mode == 2 || sw_pref)) {
    const int cs = epi->kind == SKB_EPI_LOGITS ? 1 : (sw::g_cs > 0 ? sw::g_cs : ksplit);
    const int na = sw::g_na > 0 ? sw::g_na : sw::pick_na(M, N, cs, conc);
    // (instantiated: prologue LayerNorm for cs 1/4/8, fused LayerNorm-out for cs <= 8)
    fused_ln = epi->kind == SKB_EPI_RESID && epi->ln_out != nullptr && cs <= 8;
    if (!fused_ln) ep.ln_out = nullptr;
    if (epi->ln_in) {
      // input LayerNorm in the prologue while each CTA's share is small;
      // else one LayerNorm launch writes A first (identical bits)
      const long panel = (long)na * ((K / tc::BK + cs - 1) / cs) * 128;  // this CTA's k-blocks
      if ((cs == 1 || cs == 4 || cs == 8) && M <= sw::lnx_max_rows() && panel <= 64 * 1024 && K % 128 == 0 &&
          K <= 1024 && epi->kind != SKB_EPI_RESID &&
          epi->kind != SKB_EPI_SSRU && (reinterpret_cast<uintptr_t>(epi->ln_in) & 15) == 0 &&
          epi->ln_in_ld % 4 == 0) {
        ep.lnx = epi->ln_in;
      } else {
        rc = ln_before(in_dtype, M, K, A, lda, epi, stream);
        if (rc) return rc;
      }
    }
    return sw::launch(M, N, K, A, lda, W, ldw, ep, st, na, cs, conc);
  }
  if (epi->ln_in) {
    rc = ln_before(in_dtype, M, K, A, lda, epi, stream);
    if (rc) return rc;
  }
  // Tile width BN and split-K factor S from a bytes-per-SM cost model: every
  // work unit streams (BM + BN) x K/S bf16 operands (plus an fp32 partial
  // round trip when S > 1); units run in ceil(units / SMs) rounds.
  // S changes the fp32 summation order, so it is chosen from (N, K) alone
  // (cost evaluated at the reference decode batch of 640 rows): a row's
  // result never depends on how many other rows share the call, which keeps
  // translate() batch-composition invariant (test_search.py:400-405).  BN
  // does not affect numerics and is chosen for the actual M.
  const int nk = (K + tc::BK - 1) / tc::BK;
  const int nsm = tc::num_sms();
  const bool can_split = epi->splitk_ws != nullptr && epi->splitk_counters != nullptr;
  tc::init_forces();
  const int force_bn = tc::g_force_bn, force_s = tc::g_force_s;
  // BN <= 128: two accumulators of BN columns keep every CTA at <= 256 TMEM
  // columns, so the (at most two) TMEM-using CTAs an SM holds never block in
  // tcgen05.alloc — with several decode streams sharing the device a CTA
  // blocked there (holding shared memory) could otherwise stall the others.
  // BN = 256 stays available through skb_gemm_force.
  const int bns[3] = {force_bn == 256 ? 256 : 128, 128, 64};
  auto cost = [&](long m, int bn, int sp) {
    const long tiles = ((m + tc::BM - 1) / tc::BM) * ((N + bn - 1) / bn) * sp;
    const long rounds = (tiles + nsm - 1) / nsm;
    const double kb = (double)((nk + sp - 1) / sp) * tc::BK;
    const double bytes = (tc::BM + bn) * kb * 2.0 + (sp > 1 ? 2.0 * tc::BM * bn * 4 : 0.0);
    return rounds * (bytes + 96.0 * 1024);  // + fixed per-unit overhead
  };
  int best_s = 1;
  // Split-K is opt-in (SKB_GEMM_SPLITK=1): measured on B200 at the decode
  // shapes, the partial-tile round trip through L2 costs more than the extra
  // SMs gain (tools/bench_gemm.py sweep, profiles/r1_gemm_sweep.txt).
  static int splitk_on = -1;
  if (splitk_on < 0) {
    const char *e = getenv("SKB_GEMM_SPLITK");
    splitk_on = (e && e[0] == '1') ? 1 : 0;
  }
  if (can_split && splitk_on) {
    const int ss[6] = {1, 2, 3, 4, 6, 8};
    double best = 1e30;
    for (int si = 0; si < 6; ++si) {
      const int sp = ss[si];
      if (sp > 1 && nk < 2 * sp) continue;
      for (int bi = 0; bi < 3; ++bi) {
        const double c = cost(640, bns[bi], sp);
        if (c < best * 0.97) {
          best = c;
          best_s = sp;
        }
      }
    }
  }
  if (force_s) best_s = force_s;
  // Tile width BN and multicast cluster size CS (A shared by CS N tiles):
  // per-CTA bytes (BM/CS + BN) x K, units in ceil(CTAs / SMs) rounds.
  const int force_cs = tc::g_force_cs;
  int best_bn = 128, best_cs = 1;
  double best = 1e30;
  for (int bi = 0; bi < 3; ++bi) {
    const int bn = bns[bi];
    if (force_bn && bn != force_bn) continue;
    const int css[3] = {1, 2, 4};
    for (int ci = 0; ci < 3; ++ci) {
      const int cs = css[ci];
      if (force_cs && cs != force_cs) continue;
      if (cs > 1 && best_s > 1) continue;
      const long ntl = (N + bn - 1) / bn;
      const long ctas = ((M + tc::BM - 1) / tc::BM) * ((ntl + cs - 1) / cs) * cs * best_s;
      const long rounds = (ctas + nsm - 1) / nsm;
      const double kb = (double)((nk + best_s - 1) / best_s) * tc::BK;
      const double bytes = ((double)tc::BM / cs + bn) * kb * 2.0 +
                           (best_s > 1 ? 2.0 * tc::BM * bn * 4 : 0.0);
      const double c = rounds * (bytes + 96.0 * 1024);
      if (c < best * 0.97) {
        best = c;
        best_bn = bn;
        best_cs = cs;
      }
    }
  }
#define SKB_GEMM_GO(BNV)                                                               \
  do {                                                                                 \
    if (best_cs == 4) return tc::launch<BNV, 4>(M, N, K, A, lda, W, ldw, ep, st, 1);    \
    if (best_cs == 2) return tc::launch<BNV, 2>(M, N, K, A, lda, W, ldw, ep, st, 1);    \
    return tc::launch<BNV, 1>(M, N, K, A, lda, W, ldw, ep, st, best_s);                 \
  } while (0)
  if (best_bn == 256) SKB_GEMM_GO(256);
  if (best_bn == 128) SKB_GEMM_GO(128);
  SKB_GEMM_GO(64);
#undef SKB_GEMM_GO
}
