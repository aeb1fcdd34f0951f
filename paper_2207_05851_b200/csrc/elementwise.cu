// Row kernels of the decode path: layer norm, step/source embeddings, row
// gathers and the NVS max-pool.  All are HBM/L2-bound; one warp per row for
// the reductions, 16-byte vector access where the layout allows.

#include "common.cuh"

namespace skb {

// ------------------------------------------------------------ layer norm
// kernels.py:298-324: mu = mean(x); xc = x - mu; var = mean(xc*xc);
// out = xc * (1/sqrt(var + eps)) * gain + bias.  One warp per row.
__global__ void __launch_bounds__(256) k_layernorm(int rows, int d, const float *__restrict__ x,
                                                   int ldx, const float *__restrict__ gain,
                                                   const float *__restrict__ bias, float eps,
                                                   void *out, int ldo, int out_dtype) {
  PDL_ENTRY();
  const int warp = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float *xr = x + (size_t)warp * ldx;
  float s = 0.f;
  const bool vec = (d % 128 == 0) && (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (vec) {
    for (int c = lane * 4; c < d; c += 128) {
      float4 v = *reinterpret_cast<const float4 *>(xr + c);
      s += (v.x + v.y) + (v.z + v.w);
    }
  } else {
    for (int c = lane; c < d; c += 32) s += xr[c];
  }
  const float mu = warp_sum(s) / (float)d;
  float q = 0.f;
  if (vec) {
    for (int c = lane * 4; c < d; c += 128) {
      float4 v = *reinterpret_cast<const float4 *>(xr + c);
      float a = v.x - mu, b = v.y - mu, e = v.z - mu, f = v.w - mu;
      q += (a * a + b * b) + (e * e + f * f);
    }
  } else {
    for (int c = lane; c < d; c += 32) {
      float a = xr[c] - mu;
      q += a * a;
    }
  }
  const float var = warp_sum(q) / (float)d;
  const float inv = 1.0f / sqrtf(var + eps);
  if (out_dtype == SKB_F32) {
    float *o = reinterpret_cast<float *>(out) + (size_t)warp * ldo;
    for (int c = lane; c < d; c += 32) o[c] = ((xr[c] - mu) * inv) * gain[c] + bias[c];
  } else {
    __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(out) + (size_t)warp * ldo;
    if (vec && ldo % 4 == 0) {
      for (int c = lane * 4; c < d; c += 128) {
        float4 v = *reinterpret_cast<const float4 *>(xr + c);
        float4 g = *reinterpret_cast<const float4 *>(gain + c);
        float4 b = *reinterpret_cast<const float4 *>(bias + c);
        __nv_bfloat162 p0 = __floats2bfloat162_rn(((v.x - mu) * inv) * g.x + b.x,
                                                  ((v.y - mu) * inv) * g.y + b.y);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(((v.z - mu) * inv) * g.z + b.z,
                                                  ((v.w - mu) * inv) * g.w + b.w);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t *>(&p0);
        w.y = *reinterpret_cast<uint32_t *>(&p1);
        *reinterpret_cast<uint2 *>(o + c) = w;
      }
    } else {
      for (int c = lane; c < d; c += 32)
        o[c] = __float2bfloat16_rn(((xr[c] - mu) * inv) * gain[c] + bias[c]);
    }
  }
}

// Register-resident variant for d = NV * 128: one warp per row, each lane
// holds NV float4 of the row, so x is read from memory exactly once.
template <int NV>
__global__ void __launch_bounds__(256) k_layernorm_reg(int rows, const float *__restrict__ x,
                                                       int ldx, const float *__restrict__ gain,
                                                       const float *__restrict__ bias, float eps,
                                                       void *out, int ldo, int out_dtype) {
  constexpr int d = NV * 128;
  const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  // gain / bias are parameters: loaded before the grid-dependency wait
  float4 g[NV], bb[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    g[i] = __ldg(reinterpret_cast<const float4 *>(gain) + lane + 32 * i);
    bb[i] = __ldg(reinterpret_cast<const float4 *>(bias) + lane + 32 * i);
  }
  PDL_ENTRY();
  if (warp >= rows) return;
  const float4 *xr = reinterpret_cast<const float4 *>(x + (size_t)warp * ldx);
  float4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = xr[lane + 32 * i];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  const float mu = warp_sum(s) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a = v[i].x - mu, b = v[i].y - mu, e = v[i].z - mu, f = v[i].w - mu;
    q += (a * a + b * b) + (e * e + f * f);
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / (float)d + eps);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    const float o0 = ((v[i].x - mu) * inv) * g[i].x + bb[i].x, o1 = ((v[i].y - mu) * inv) * g[i].y + bb[i].y;
    const float o2 = ((v[i].z - mu) * inv) * g[i].z + bb[i].z, o3 = ((v[i].w - mu) * inv) * g[i].w + bb[i].w;
    if (out_dtype == SKB_F32) {
      reinterpret_cast<float4 *>(reinterpret_cast<float *>(out) + (size_t)warp * ldo)[c4] =
          make_float4(o0, o1, o2, o3);
    } else {
      __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t *>(&p0);
      w.y = *reinterpret_cast<uint32_t *>(&p1);
      reinterpret_cast<uint2 *>(reinterpret_cast<__nv_bfloat16 *>(out) + (size_t)warp * ldo)[c4] = w;
    }
  }
}

// ------------------------------------------------------- step embedding
// model.py:399-410 with offset = step (model.py:545-547).
__global__ void k_embed_target(int rows, int d, const int *__restrict__ tok,
                               const float *__restrict__ E, const float *__restrict__ pe,
                               const int *__restrict__ step, int n_factors,
                               const int *__restrict__ ftok, const float *const *__restrict__ ftables,
                               float *__restrict__ x) {
  PDL_ENTRY();
  const int r = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows || c >= d) return;
  const int t = *step;
  float v = E[(size_t)tok[r] * d + c] + pe[(size_t)t * d + c];
  for (int k = 0; k < n_factors; ++k) v = v + ftables[k][(size_t)ftok[k * rows + r] * d + c];
  x[(size_t)r * d + c] = v;
}

// Vectorised variant (d % 4 == 0, 16-byte aligned tables): one warp per row
// quarter-chunk, float4 per thread; several rows per CTA.
__global__ void __launch_bounds__(256) k_embed_target4(int rows, int d, const int *__restrict__ tok,
                                                       const float *__restrict__ E,
                                                       const float *__restrict__ pe,
                                                       const int *__restrict__ step, int n_factors,
                                                       const int *__restrict__ ftok,
                                                       const float *const *__restrict__ ftables,
                                                       float *__restrict__ x) {
  PDL_ENTRY();
  const int d4 = d >> 2;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)rows * d4) return;
  const int r = (int)(i / d4), c4 = (int)(i - (long)r * d4);
  const int t = *step;
  float4 v = reinterpret_cast<const float4 *>(E + (size_t)tok[r] * d)[c4];
  const float4 p = reinterpret_cast<const float4 *>(pe + (size_t)t * d)[c4];
  v.x = v.x + p.x; v.y = v.y + p.y; v.z = v.z + p.z; v.w = v.w + p.w;
  for (int k = 0; k < n_factors; ++k) {
    const float4 f = reinterpret_cast<const float4 *>(ftables[k] + (size_t)ftok[k * rows + r] * d)[c4];
    v.x = v.x + f.x; v.y = v.y + f.y; v.z = v.z + f.z; v.w = v.w + f.w;
  }
  reinterpret_cast<float4 *>(x + (size_t)r * d)[c4] = v;
}

// ----------------------------------------------------- source embedding
struct SrcFactors {
  int n;
  int dim[8];
  int combine[8];   // 0 sum, 1 concat
  int concat_off[8];
};

// model.py:370-397: surface + PE on the first ds columns; concat factors
// occupy [ds, d) in order; sum factors are added afterwards, in order.
__global__ void k_embed_source(int B, int L, int d, int ds, const int *__restrict__ ids,
                               const float *__restrict__ E, const float *__restrict__ pe,
                               SrcFactors f, const int *__restrict__ fids,
                               const float *const *__restrict__ ftables, float *__restrict__ x) {
  PDL_ENTRY();
  const int row = blockIdx.y;  // b*L + l
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= B * L || c >= d) return;
  const int l = row % L;
  const size_t n = (size_t)B * L;
  float v;
  if (c < ds) {
    v = E[(size_t)ids[row] * ds + c] + pe[(size_t)l * ds + c];
  } else {
    v = 0.f;
    for (int k = 0; k < f.n; ++k)
      if (f.combine[k] == 1 && c >= f.concat_off[k] && c < f.concat_off[k] + f.dim[k])
        v = ftables[k][(size_t)fids[k * n + row] * f.dim[k] + (c - f.concat_off[k])];
  }
  for (int k = 0; k < f.n; ++k)
    if (f.combine[k] == 0) v = v + ftables[k][(size_t)fids[k * n + row] * d + c];
  x[(size_t)row * d + c] = v;
}

// ---------------------------------------------------------------- gather
__global__ void k_gather_rows(int n, int w, const uint8_t *__restrict__ table, size_t ld_bytes,
                              const int *__restrict__ idx, uint8_t *__restrict__ out,
                              size_t ldo_bytes, int row_bytes) {
  PDL_ENTRY();
  const int i = blockIdx.x;
  if (i >= n) return;
  const uint8_t *src = table + (size_t)idx[i] * ld_bytes;
  uint8_t *dst = out + (size_t)i * ldo_bytes;
  if ((row_bytes % 16) == 0 && (ld_bytes % 16) == 0 && (ldo_bytes % 16) == 0 &&
      ((reinterpret_cast<uintptr_t>(table) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    for (int c = threadIdx.x * 16; c < row_bytes; c += blockDim.x * 16)
      *reinterpret_cast<uint4 *>(dst + c) = *reinterpret_cast<const uint4 *>(src + c);
  } else {
    for (int c = threadIdx.x; c < row_bytes; c += blockDim.x) dst[c] = src[c];
  }
}

// ---------------------------------------------------------- masked max
// model.py:496-500 (kernels.py masked_max): max over unpadded positions.
__global__ void k_masked_maxpool(int B, int L, int d, const float *__restrict__ enc,
                                 const int *__restrict__ lengths, float *__restrict__ out) {
  PDL_ENTRY();
  const int b = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || c >= d) return;
  const int n = lengths[b];
  float m = -INFINITY;
  for (int l = 0; l < n; ++l) m = fmaxf(m, enc[((size_t)b * L + l) * d + c]);
  out[(size_t)b * d + c] = m;
}

}  // namespace skb

using namespace skb;

extern "C" int skb_layernorm(int rows, int d, const float *x, int ldx, const float *gain,
                             const float *bias, float eps, void *out, int ldo, int out_dtype,
                             void *stream) {
  if (rows < 0 || d <= 0) return fail(SKB_ERR_SHAPE, "layernorm: rows=%d d=%d", rows, d);
  if (rows == 0) return SKB_OK;
  const bool aligned = ldx % 4 == 0 && ldo % 4 == 0 &&
                       ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) |
                         reinterpret_cast<uintptr_t>(gain) | reinterpret_cast<uintptr_t>(bias)) & 15) == 0;
  const int blocks = (rows + 7) / 8;
  cudaStream_t s = as_stream(stream);
  static int lw = -1;  // warps (rows) per CTA of the d = 1024 kernel, SKB_LN_WARPS
  if (lw < 0) {
    const char *e = getenv("SKB_LN_WARPS");
    lw = e ? atoi(e) : 4;  // 4 measured best at R = 640 (more SMs share the rows)
    if (lw < 1 || lw > 8) lw = 8;
  }
  if (aligned && d == 1024)
    launch_k(k_layernorm_reg<8>, (rows + lw - 1) / lw, 32 * lw, 0, s, rows, x, ldx, gain, bias, eps, out,
             ldo, out_dtype);
  else if (aligned && d == 512)
    launch_k(k_layernorm_reg<4>, blocks, 256, 0, s, rows, x, ldx, gain, bias, eps, out, ldo, out_dtype);
  else if (aligned && d == 256)
    launch_k(k_layernorm_reg<2>, blocks, 256, 0, s, rows, x, ldx, gain, bias, eps, out, ldo, out_dtype);
  else if (aligned && d == 2048)
    launch_k(k_layernorm_reg<16>, blocks, 256, 0, s, rows, x, ldx, gain, bias, eps, out, ldo, out_dtype);
  else
    launch_k(k_layernorm, blocks, 256, 0, s, rows, d, x, ldx, gain, bias, eps, out, ldo, out_dtype);
  SKB_CHECK_LAUNCH("k_layernorm");
  return SKB_OK;
}

extern "C" int skb_embed_target(int rows, int d, const int *tok, const float *E, const float *pe,
                                const int *step, int n_factors, const int *ftok,
                                const float *const *ftables, float *x, void *stream) {
  if (rows < 0 || d <= 0) return fail(SKB_ERR_SHAPE, "embed_target: rows=%d d=%d", rows, d);
  if (rows == 0) return SKB_OK;
  // (factor tables: device allocations with d-float rows, aligned like E)
  const bool vec = d % 4 == 0 && ((reinterpret_cast<uintptr_t>(E) | reinterpret_cast<uintptr_t>(pe) |
                                   reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  if (vec) {
    const long n4 = (long)rows * (d / 4);
    launch_k(k_embed_target4, (unsigned)((n4 + 255) / 256), 256, 0, as_stream(stream), rows, d, tok, E,
             pe, step, n_factors, ftok, ftables, x);
    SKB_CHECK_LAUNCH("k_embed_target4");
    return SKB_OK;
  }
  dim3 grid((d + 255) / 256, rows);
  launch_k(k_embed_target, grid, 256, 0, as_stream(stream), rows, d, tok, E, pe, step, n_factors, ftok,
                                                      ftables, x);
  SKB_CHECK_LAUNCH("k_embed_target");
  return SKB_OK;
}

extern "C" int skb_embed_source(int B, int L, int d, int ds, const int *ids, const float *E,
                                const float *pe, int n_factors, const int *fdims_host,
                                const int *fcombine_host, const int *fids,
                                const float *const *ftables, float *x, void *stream) {
  if (B <= 0 || L <= 0 || d <= 0 || ds <= 0 || ds > d)
    return fail(SKB_ERR_SHAPE, "embed_source: B=%d L=%d d=%d ds=%d", B, L, d, ds);
  if (n_factors > 8) return fail(SKB_ERR_CONFIG, "embed_source: at most 8 source factors");
  SrcFactors f{};
  f.n = n_factors;
  int off = ds;
  for (int k = 0; k < n_factors; ++k) {
    f.dim[k] = fdims_host[k];
    f.combine[k] = fcombine_host[k];
    if (f.combine[k] == 1) {
      f.concat_off[k] = off;
      off += f.dim[k];
    }
  }
  if (off != d) return fail(SKB_ERR_CONFIG, "embed_source: concat widths do not fill d");
  dim3 grid((d + 255) / 256, B * L);
  launch_k(k_embed_source, grid, 256, 0, as_stream(stream), B, L, d, ds, ids, E, pe, f, fids, ftables, x);
  SKB_CHECK_LAUNCH("k_embed_source");
  return SKB_OK;
}

extern "C" int skb_gather_rows(int n, int w, const void *table, int ld_table, const int *idx,
                               void *out, int ld_out, int dtype, void *stream) {
  if (n < 0 || w <= 0) return fail(SKB_ERR_SHAPE, "gather_rows: n=%d w=%d", n, w);
  if (n == 0) return SKB_OK;
  const size_t es = dtype == SKB_F32 ? 4 : 2;
  launch_k(k_gather_rows, n, 128, 0, as_stream(stream), n, w, (const uint8_t *)table, ld_table * es, idx,
                                                  (uint8_t *)out, ld_out * es, (int)(w * es));
  SKB_CHECK_LAUNCH("k_gather_rows");
  return SKB_OK;
}

extern "C" int skb_masked_maxpool(int B, int L, int d, const float *enc, const int *lengths,
                                  float *out, void *stream) {
  if (B <= 0 || L <= 0 || d <= 0) return fail(SKB_ERR_SHAPE, "masked_maxpool: bad shape");
  dim3 grid((d + 255) / 256, B);
  launch_k(k_masked_maxpool, grid, 256, 0, as_stream(stream), B, L, d, enc, lengths, out);
  SKB_CHECK_LAUNCH("k_masked_maxpool");
  return SKB_OK;
}

// ----------------------------------------------------- dtype conversion
namespace skb {
__global__ void k_convert(size_t n, const void *src, int sdt, void *dst, int ddt) {
  PDL_ENTRY();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    store_f(dst, ddt, i, load_f(src, sdt, i));
}

// NVS selection (model.py:511-517): bit c of row b set iff
// sigmoid(logit[b, c]) > threshold (threshold rounded to float32).
__global__ void k_nvs_mask(int B, int V, const float *logits, int ld, float thr, unsigned *mask) {
  PDL_ENTRY();
  const int b = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int words = (V + 31) >> 5;
  const bool on = c < V && sigmoid_ref(logits[(size_t)b * ld + c]) > thr;
  const unsigned bits = __ballot_sync(0xffffffffu, on);
  if ((threadIdx.x & 31) == 0 && (c >> 5) < words) mask[(size_t)b * words + (c >> 5)] = bits;
}
}  // namespace skb

extern "C" int skb_convert(long long n, const void *src, int src_dtype, void *dst, int dst_dtype,
                           void *stream) {
  if (n < 0) return fail(SKB_ERR_SHAPE, "convert: n=%lld", n);
  if (n == 0) return SKB_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(k_convert, blocks, 256, 0, as_stream(stream), (size_t)n, src, src_dtype, dst, dst_dtype);
  SKB_CHECK_LAUNCH("k_convert");
  return SKB_OK;
}

extern "C" int skb_nvs_mask(int B, int V, const float *logits, int ld, float threshold,
                            unsigned *mask, void *stream) {
  if (B <= 0 || V <= 0) return fail(SKB_ERR_SHAPE, "nvs_mask: bad shape");
  dim3 grid((V + 255) / 256, B);
  launch_k(k_nvs_mask, grid, 256, 0, as_stream(stream), B, V, logits, ld, threshold, mask);
  SKB_CHECK_LAUNCH("k_nvs_mask");
  return SKB_OK;
}

extern "C" int skb_set_device(int device) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(SKB_ERR_LAUNCH, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  return SKB_OK;
}

// ------------------------------------------------- int8 row quantization
// quant.py:40-53 (weights, offline) and :99-104 (activations, per call):
// scale = max|row| / 127 (1 for an all-zero row), q = clip(round half away
// from zero (x / scale), -127, 127).  Every operation is the reference's
// float32 operation (IEEE division, |v| + 0.5 rounded, then floor), so the
// integers and scales are bit-identical.  One CTA per row.
namespace skb {
__global__ void __launch_bounds__(128) k_quantize_rows(int rows, int k, const float *__restrict__ x,
                                                       int ldx, int8_t *__restrict__ q, int ldq,
                                                       float *__restrict__ scales) {
  PDL_ENTRY();
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float *xr = x + (size_t)r * ldx;
  float m = 0.f;
  for (int c = threadIdx.x; c < k; c += blockDim.x) m = fmaxf(m, fabsf(xr[c]));
  m = warp_max(m);
  __shared__ float wm[4];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  m = fmaxf(fmaxf(wm[0], wm[1]), fmaxf(wm[2], wm[3]));
  const float scale = m > 0.f ? __fdiv_rn(m, 127.0f) : 1.0f;
  if (threadIdx.x == 0) scales[r] = scale;
  int8_t *qr = q + (size_t)r * ldq;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    const float v = __fdiv_rn(xr[c], scale);
    float a = floorf(__fadd_rn(fabsf(v), 0.5f));
    a = fminf(a, 127.0f);
    qr[c] = (int8_t)(v < 0.f ? -(int)a : (int)a);
  }
}
}  // namespace skb

extern "C" int skb_quantize_rows(int rows, int k, const float *x, int ldx, void *q, int ldq,
                                 float *scales, void *stream) {
  if (rows < 0 || k <= 0 || ldx < k || ldq < k)
    return fail(SKB_ERR_SHAPE, "quantize_rows: rows=%d k=%d ldx=%d ldq=%d", rows, k, ldx, ldq);
  if (k > (int)(2147483648LL / (127 * 127)))
    return fail(SKB_ERR_CONFIG, "quantize_rows: inner extent %d would overflow int32 accumulation", k);
  if (rows == 0) return SKB_OK;
  launch_k(k_quantize_rows, rows, 128, 0, as_stream(stream), rows, k, x, ldx,
           reinterpret_cast<int8_t *>(q), ldq, scales);
  SKB_CHECK_LAUNCH("k_quantize_rows");
  return SKB_OK;
}

// --------------------------------------------------------- SSRU scan
// The SSRU recurrence over a whole target sequence (model.py:482-493
// _ssru_scan, cell model.py:268-272) for the teacher-forced pass: g is the
// fp32 [B*T, 2d] output of the interleaved [W_f; W] GEMM (column 2j = W_f h,
// 2j+1 = W h), bias the interleaved [2d] bias (b_f at even columns).  Per
// (sentence, column): c_0 = 0, f = sigmoid(W_f h + b_f), c = f c + (1 - f)
// W h, x += relu(c) — the arithmetic of the decode step's SSRU epilogue.
namespace skb {
__global__ void k_ssru_scan(int B, int T, int d, const float *__restrict__ g, int ldg,
                            const float *__restrict__ bias, float *__restrict__ x, int ldx) {
  PDL_ENTRY();
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || j >= d) return;
  const float bf = bias ? bias[2 * j] : 0.f;
  float c = 0.f;
  for (int t = 0; t < T; ++t) {
    const size_t r = (size_t)b * T + t;
    c = ssru_cell(g[r * ldg + 2 * j], bf, g[r * ldg + 2 * j + 1], c);
    float *xp = x + r * ldx + j;
    *xp = *xp + fmaxf(c, 0.f);
  }
}
}  // namespace skb

extern "C" int skb_ssru_scan(int B, int T, int d, const float *g, int ldg, const float *bias,
                             float *x, int ldx, void *stream) {
  if (B <= 0 || T <= 0 || d <= 0 || ldg < 2 * d || ldx < d)
    return fail(SKB_ERR_SHAPE, "ssru_scan: B=%d T=%d d=%d", B, T, d);
  dim3 grid((d + 127) / 128, B);
  launch_k(k_ssru_scan, grid, 128, 0, as_stream(stream), B, T, d, g, ldg, bias, x, ldx);
  SKB_CHECK_LAUNCH("k_ssru_scan");
  return SKB_OK;
}
