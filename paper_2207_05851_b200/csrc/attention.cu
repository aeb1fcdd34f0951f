// Attention kernels of the decode path (skiff kernels.py:510-547,
// model.py:414-430, 559-573).
//
//  * encoder self-attention: one warp per query row, keys/values of the
//    (sentence, head) streamed through shared memory in 64-key tiles with an
//    online softmax; padded keys (>= length) are skipped, which equals the
//    reference's additive -1e9 bias exactly (exp underflows to 0).
//  * incremental decoder self-attention: one warp per (row, head); the new
//    k/v are written into the preallocated cache at slot (row, t) and the
//    t earlier positions are read through the ancestor table, so the beam
//    reorder never copies cache bytes.
//  * cross-attention: one warp per (row, head) over the sentence's encoder
//    memory; all beam rows of a sentence read the same K/V (L2-resident).
// Scores are q.k * (1/sqrt(d_h)) in fp32 (kernels.py:512-514).

#include "common.cuh"

namespace skb {

constexpr int MAX_DH = 128;

// dot(q[0:dh], row[0:dh]) with row of dtype (fp32 / bf16), q in shared mem.
__device__ __forceinline__ float dot_row(const void *row, int dtype, const float *q, int dh) {
  float acc = 0.f;
  if (dtype == SKB_BF16) {
    const __nv_bfloat16 *r = reinterpret_cast<const __nv_bfloat16 *>(row);
    if ((dh & 7) == 0 && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
      for (int c = 0; c < dh; c += 8) {
        uint4 u = *reinterpret_cast<const uint4 *>(r + c);
        const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float2 f = __bfloat1622float2(p[h]);
          acc = fmaf(q[c + 2 * h], f.x, acc);
          acc = fmaf(q[c + 2 * h + 1], f.y, acc);
        }
      }
    } else {
      for (int c = 0; c < dh; ++c) acc = fmaf(q[c], __bfloat162float(r[c]), acc);
    }
  } else {
    const float *r = reinterpret_cast<const float *>(row);
    if ((dh & 3) == 0 && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
      for (int c = 0; c < dh; c += 4) {
        float4 f = *reinterpret_cast<const float4 *>(r + c);
        acc = fmaf(q[c], f.x, acc);
        acc = fmaf(q[c + 1], f.y, acc);
        acc = fmaf(q[c + 2], f.z, acc);
        acc = fmaf(q[c + 3], f.w, acc);
      }
    } else {
      for (int c = 0; c < dh; ++c) acc = fmaf(q[c], r[c], acc);
    }
  }
  return acc;
}

// Online-softmax accumulator owned by one warp; lane owns dims lane+32*j.
struct WarpSoftmax {
  float m, l;
  float o[MAX_DH / 32];
  __device__ void init() {
    m = -INFINITY;
    l = 0.f;
#pragma unroll
    for (int j = 0; j < MAX_DH / 32; ++j) o[j] = 0.f;
  }
};

// Process a chunk of up to 32 keys: lane k holds score s (or -inf if
// invalid) and a pointer to its value row; all lanes accumulate into o.
__device__ __forceinline__ void softmax_chunk(WarpSoftmax &st, float s, const void *vrow,
                                              int vdtype, int dh, int lane) {
  const float cmax = warp_max(s);
  if (cmax == -INFINITY) return;
  const float mnew = fmaxf(st.m, cmax);
  const float corr = st.m == -INFINITY ? 0.f : expf(st.m - mnew);
  const float p = s == -INFINITY ? 0.f : expf(s - mnew);
  st.l = st.l * corr + warp_sum(p);
#pragma unroll
  for (int j = 0; j < MAX_DH / 32; ++j) st.o[j] *= corr;
  st.m = mnew;
  for (int k = 0; k < 32; ++k) {
    const float pk = __shfl_sync(0xffffffffu, p, k);
    const unsigned long long vp =
        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(vrow), k);
    if (pk == 0.f) continue;
#pragma unroll
    for (int j = 0; j < MAX_DH / 32; ++j) {
      const int c = lane + 32 * j;
      if (c < dh) st.o[j] = fmaf(pk, load_f(reinterpret_cast<const void *>(vp), vdtype, c), st.o[j]);
    }
  }
}

__device__ __forceinline__ void write_ctx(const WarpSoftmax &st, void *ctx, int ctx_dtype,
                                          size_t base, int dh, int lane) {
  const float inv = 1.0f / st.l;
#pragma unroll
  for (int j = 0; j < MAX_DH / 32; ++j) {
    const int c = lane + 32 * j;
    if (c < dh) store_f(ctx, ctx_dtype, base + c, st.o[j] * inv);
  }
}

__device__ __forceinline__ const void *elem_ptr(const void *base, int dtype, size_t i) {
  return dtype == SKB_F32 ? (const void *)(reinterpret_cast<const float *>(base) + i)
                          : (const void *)(reinterpret_cast<const __nv_bfloat16 *>(base) + i);
}

// ------------------------------------------------------------ encoder
// grid (B*H, ceil(L/8)), 256 threads: warp w handles query l = blockIdx.y*8+w.
__global__ void __launch_bounds__(256) k_encoder_attention(int B, int L, int H, int dh,
                                                           const void *qkv, int ld_qkv, int qkv_dtype,
                                                           const int *lengths, float scale,
                                                           void *ctx, int ldc, int ctx_dtype) {
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.y * 8 + warp;
  const int D = H * dh;
  __shared__ float qs[8][MAX_DH];
  if (l >= L) return;
  const size_t qrow = (size_t)(b * L + l) * ld_qkv;
  for (int c = lane; c < dh; c += 32) qs[warp][c] = load_f(qkv, qkv_dtype, qrow + h * dh + c);
  __syncwarp();
  const int len = lengths[b];
  WarpSoftmax st;
  st.init();
  for (int k0 = 0; k0 < len; k0 += 32) {
    const int key = k0 + lane;
    float s = -INFINITY;
    const void *vrow = nullptr;
    if (key < len) {
      const size_t kr = (size_t)(b * L + key) * ld_qkv;
      s = dot_row(elem_ptr(qkv, qkv_dtype, kr + D + h * dh), qkv_dtype, qs[warp], dh) * scale;
      vrow = elem_ptr(qkv, qkv_dtype, kr + 2 * D + h * dh);
    }
    softmax_chunk(st, s, vrow, qkv_dtype, dh, lane);
  }
  write_ctx(st, ctx, ctx_dtype, (size_t)(b * L + l) * ldc + h * dh, dh, lane);
}

// ------------------------------------------------ decoder self-attention
// One warp per (row, head): 4 warps per block.
__global__ void __launch_bounds__(128) k_self_attention_step(
    int R, int H, int dh, const void *qkv, int ld_qkv, int qkv_dtype, void *kc, void *vc,
    int cache_dtype, int S_max, const int *anc, const int *step, float scale, void *ctx, int ldc,
    int ctx_dtype) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 4 + warp;
  __shared__ float qs[4][MAX_DH];
  if (gw >= R * H) return;
  const int r = gw / H, h = gw % H;
  const int D = H * dh;
  const int t = *step;
  const size_t qrow = (size_t)r * ld_qkv;
  // store this step's k, v at slot (r, t)
  const size_t cslot = ((size_t)r * S_max + t) * D + h * dh;
  for (int c = lane; c < dh; c += 32) {
    qs[warp][c] = load_f(qkv, qkv_dtype, qrow + h * dh + c);
    store_f(kc, cache_dtype, cslot + c, load_f(qkv, qkv_dtype, qrow + D + h * dh + c));
    store_f(vc, cache_dtype, cslot + c, load_f(qkv, qkv_dtype, qrow + 2 * D + h * dh + c));
  }
  __threadfence_block();
  __syncwarp();
  const int *arow = anc + ((size_t)(t & 1) * R + r) * S_max;
  WarpSoftmax st;
  st.init();
  for (int p0 = 0; p0 <= t; p0 += 32) {
    const int p = p0 + lane;
    float s = -INFINITY;
    const void *vrow = nullptr;
    if (p <= t) {
      const int slot = p == t ? r : arow[p];
      const size_t off = ((size_t)slot * S_max + p) * D + h * dh;
      s = dot_row(elem_ptr(kc, cache_dtype, off), cache_dtype, qs[warp], dh) * scale;
      vrow = elem_ptr(vc, cache_dtype, off);
    }
    softmax_chunk(st, s, vrow, cache_dtype, dh, lane);
  }
  write_ctx(st, ctx, ctx_dtype, (size_t)r * ldc + h * dh, dh, lane);
}

// -------------------------------------------------------- cross-attention
__global__ void __launch_bounds__(128) k_cross_attention_step(
    int R, int H, int dh, const void *q, int ldq, int q_dtype, const void *kv, int ld_kv,
    int kv_dtype, int koff, int voff, int L, const int *row_sent, const int *lengths, float scale,
    void *ctx, int ldc, int ctx_dtype) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * 4 + warp;
  __shared__ float qs[4][MAX_DH];
  if (gw >= R * H) return;
  const int r = gw / H, h = gw % H;
  const int b = row_sent[r];
  for (int c = lane; c < dh; c += 32) qs[warp][c] = load_f(q, q_dtype, (size_t)r * ldq + h * dh + c);
  __syncwarp();
  const int len = lengths[b];
  WarpSoftmax st;
  st.init();
  for (int k0 = 0; k0 < len; k0 += 32) {
    const int key = k0 + lane;
    float s = -INFINITY;
    const void *vrow = nullptr;
    if (key < len) {
      const size_t kr = (size_t)(b * L + key) * ld_kv;
      s = dot_row(elem_ptr(kv, kv_dtype, kr + koff + h * dh), kv_dtype, qs[warp], dh) * scale;
      vrow = elem_ptr(kv, kv_dtype, kr + voff + h * dh);
    }
    softmax_chunk(st, s, vrow, kv_dtype, dh, lane);
  }
  write_ctx(st, ctx, ctx_dtype, (size_t)r * ldc + h * dh, dh, lane);
}

static float attn_scale(int dh) { return (float)(1.0 / sqrt((double)dh)); }

}  // namespace skb

using namespace skb;

extern "C" int skb_encoder_attention(int B, int L, int H, int dh, const void *qkv, int ld_qkv,
                                     int qkv_dtype, const int *lengths, void *ctx, int ldc,
                                     int ctx_dtype, void *stream) {
  if (B <= 0 || L <= 0 || H <= 0 || dh <= 0) return fail(SKB_ERR_SHAPE, "encoder_attention: shape");
  if (dh > MAX_DH) return fail(SKB_ERR_UNSUPPORTED, "encoder_attention: head dim %d > %d", dh, MAX_DH);
  dim3 grid(B * H, (L + 7) / 8);
  k_encoder_attention<<<grid, 256, 0, as_stream(stream)>>>(B, L, H, dh, qkv, ld_qkv, qkv_dtype,
                                                           lengths, attn_scale(dh), ctx, ldc, ctx_dtype);
  SKB_CHECK_LAUNCH("k_encoder_attention");
  return SKB_OK;
}

extern "C" int skb_self_attention_step(int R, int H, int dh, const void *qkv, int ld_qkv,
                                       int qkv_dtype, void *kc, void *vc, int cache_dtype, int S_max,
                                       const int *anc, const int *step, void *ctx, int ldc,
                                       int ctx_dtype, void *stream) {
  if (R < 0 || H <= 0 || dh <= 0) return fail(SKB_ERR_SHAPE, "self_attention_step: shape");
  if (dh > MAX_DH) return fail(SKB_ERR_UNSUPPORTED, "self_attention_step: head dim %d", dh);
  if (R == 0) return SKB_OK;
  const int warps = R * H;
  k_self_attention_step<<<(warps + 3) / 4, 128, 0, as_stream(stream)>>>(
      R, H, dh, qkv, ld_qkv, qkv_dtype, kc, vc, cache_dtype, S_max, anc, step, attn_scale(dh), ctx,
      ldc, ctx_dtype);
  SKB_CHECK_LAUNCH("k_self_attention_step");
  return SKB_OK;
}

extern "C" int skb_cross_attention_step(int R, int H, int dh, const void *q, int ldq, int q_dtype,
                                        const void *kv, int ld_kv, int kv_dtype, int koff, int voff,
                                        int L, const int *row_sent, const int *lengths, void *ctx,
                                        int ldc, int ctx_dtype, void *stream) {
  if (R < 0 || H <= 0 || dh <= 0 || L <= 0) return fail(SKB_ERR_SHAPE, "cross_attention_step: shape");
  if (dh > MAX_DH) return fail(SKB_ERR_UNSUPPORTED, "cross_attention_step: head dim %d", dh);
  if (R == 0) return SKB_OK;
  const int warps = R * H;
  k_cross_attention_step<<<(warps + 3) / 4, 128, 0, as_stream(stream)>>>(
      R, H, dh, q, ldq, q_dtype, kv, ld_kv, kv_dtype, koff, voff, L, row_sent, lengths,
      attn_scale(dh), ctx, ldc, ctx_dtype);
  SKB_CHECK_LAUNCH("k_cross_attention_step");
  return SKB_OK;
}
