/*
 * skiff_b200.h — C ABI of the B200-native translation hot path.
 *
 * The reference (skiff, /root/reference/pkg/src/skiff) is pure Python/numpy:
 * it has no FFI.  Each entry point below replaces one numpy "kernel" or one
 * piece of search bookkeeping on the decode path; the citation names the
 * reference function it replaces (file:line).  The Python host package
 * (paper_2207_05851_b200) binds these with ctypes and mirrors the reference's
 * translate / Model.decode_init / decode_step interface on top.
 *
 * Conventions:
 *   - plain device pointers + int sizes; no torch types; every call is
 *     stream-ordered on the caller's cudaStream_t (passed as void*);
 *   - nothing here allocates or frees device memory; caller owns all buffers;
 *   - every function returns an int status (SKB_OK = 0).  The matching
 *     message is available from skb_last_error() (thread-local).  The host
 *     maps SKB_ERR_SHAPE -> ShapeError, SKB_ERR_CONFIG -> ConfigError,
 *     SKB_ERR_NUMERIC -> NumericError, others -> RuntimeError;
 *   - "step" arguments are device pointers so a whole decode step can be
 *     captured once into a CUDA graph and replayed.
 */
#ifndef SKIFF_B200_H
#define SKIFF_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SKB_OK 0
#define SKB_ERR_SHAPE 1
#define SKB_ERR_CONFIG 2
#define SKB_ERR_LAUNCH 3
#define SKB_ERR_NUMERIC 4
#define SKB_ERR_UNSUPPORTED 5

/* element types */
#define SKB_F32 0
#define SKB_BF16 1

/* GEMM epilogues */
#define SKB_EPI_STORE 0  /* out = acc (+bias)                                 */
#define SKB_EPI_RELU 1   /* out = relu(acc + bias)        (kernels.py:243-250) */
#define SKB_EPI_RESID 2  /* x  += acc (+bias), x fp32     (model.py:565-574)   */
#define SKB_EPI_SSRU 3   /* SSRU cell, columns interleaved (f_j, Wx_j)         */
                         /*                               (model.py:268-272)   */
#define SKB_EPI_LOGITS 4 /* fp32 logits + fused log-softmax partials          */
                         /* (kernels.py:287-295, search.py:294/347)            */

/* GEMM epilogue parameters (plain C struct, passed by pointer). */
typedef struct skb_epilogue {
  int kind;              /* SKB_EPI_*                                          */
  const float *bias;     /* [N] or NULL                                        */
  void *out;             /* STORE/RELU: [M, ldo] of out_dtype; RESID/SSRU: x   */
  int ldo;               /* leading dim of out (elements)                      */
  int out_dtype;         /* SKB_F32 / SKB_BF16 (RESID/SSRU: must be F32)       */
  /* SSRU only: cell state, fp32 [M, ld_state]; c_prev row = src_row[m]       */
  const float *c_prev;   /* NULL => zero previous cell (first step)            */
  float *c_next;
  const int *src_row;    /* NULL => identity                                   */
  int ld_state;
  /* Decode-loop mode (CUDA-graph friendly): if step != NULL, c_next is a    */
  /* [2, state_rows, ld_state] double buffer; step t writes half (t&1) and  */
  /* reads half ((t+1)&1) (zeros at t = 0); c_prev is ignored.              */
  const int *step;
  long long state_stride; /* elements between the two halves                 */
  /* SKB_EPI_LOGITS: besides storing fp32 logits in out, write for every row  */
  /* m and 32-column group g the partial (max, sum exp(x - max)) over the     */
  /* row's active columns as float2 lse_part[m * lse_ld + g]; the active set  */
  /* of row m is bit row (m / rows_per_group) of mask (NULL = all columns).   */
  float *lse_part;
  int lse_ld;
  const unsigned *mask;
  int mask_words;
  int rows_per_group;
  /* Optional split-K workspace (caller-owned; NULL disables split-K): fp32  */
  /* partial tiles and zero-initialised per-tile arrival counters.  Partial  */
  /* tiles are summed in split order by the last CTA to arrive, so results  */
  /* are deterministic and independent of scheduling.                       */
  float *splitk_ws;
  long long splitk_ws_elems;
  unsigned *splitk_counters;
  int splitk_counters_n;
  /* SKB_EPI_RESID only, optional fused LayerNorm of the updated rows        */
  /* (kernels.py:298-324; replaces the skb_layernorm launch that follows a   */
  /* residual GEMM, model.py:562-575): ln_out[m] = LN(x[m]) * gain + bias,   */
  /* bf16 [M, ln_ldo].  ln_counter: caller-owned, zero-initialised uint32    */
  /* [>= ceil(M / 16)] per call site, never reset (arrival tickets of the    */
  /* CTAs that finish an activation-row tile).  NULL ln_out disables it.     */
  const float *ln_gain;
  const float *ln_bias;
  float ln_eps;
  void *ln_out;
  int ln_ldo;
  unsigned *ln_counter;
  /* Optional LayerNorm of the GEMM input (kernels.py:298-324 feeding       */
  /* kernels.py:479-484; model.py:562-581): when ln_in != NULL the GEMM      */
  /* computes A[m] = LN(ln_in[m]) * ln_in_gain + ln_in_bias (eps ln_in_eps,  */
  /* fp32 [M, ln_in_ld] -> bf16 A) first.  Small M: inside the GEMM (every   */
  /* CTA normalises its activation rows into shared memory, A is not        */
  /* written); otherwise a LayerNorm launch writes A, then the GEMM runs.   */
  /* Bit-identical either way.  Not for RESID/SSRU (they update ln_in).     */
  const float *ln_in;
  int ln_in_ld;
  const float *ln_in_gain;
  const float *ln_in_bias;
  float ln_in_eps;
  /* Independent decode streams sharing the device while this call runs     */
  /* (0 or 1 = this call has the GPU to itself): tiles are sized for a      */
  /* 1/streams share of the SMs.  Never changes the numbers.                */
  int streams;
  /* K-split of the bf16 GEMM: 0 = the library's choice from (N, K) alone;  */
  /* 1, 2, 4, 8 or 16 = exactly that many K-partials, each one K-ordered    */
  /* tensor-core accumulation over a contiguous K range,                    */
  /* summed in partial order.  It fixes the fp32 summation order, so the    */
  /* caller must pass the same value for a weight matrix at every M to keep */
  /* a row's result independent of its batch (latency models: 8 / 16;      */
  /* DESIGN.md §4).  Ignored by LOGITS (always 1) and the int8 GEMM.        */
  int k_split;
} skb_epilogue;

/* Library identity / diagnostics */
const char *skb_version(void);
/* Kernels enqueued by the last skb_gemm / skb_gemm_simt call on this host  */
/* thread (1, or 2 when a LayerNorm launch accompanied the GEMM).           */
int skb_last_launches(void);
const char *skb_last_error(void);
/* 1 if the tcgen05 GEMM path is usable on the current device (sm_100). */
int skb_tc_available(void);

/*
 * C[M,N] = A[M,K] . W[N,K]^T with a fused epilogue.
 * Replaces kernels.py:479-484 (linear) / 167-195 (matmul, fp64-accumulated):
 * fp32 inputs use a SIMT FFMA kernel (fp32 accumulate); bf16 inputs use the
 * tcgen05/TMEM/TMA kernel (fp32 accumulate in TMEM).  A and W are K-major
 * (row-major), exactly the reference's (out, in) weight layout.
 */
int skb_gemm(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
             int ldw, const skb_epilogue *epi, void *stream);

/* Test / tuning overrides of the kernel choice (skb_gemm_force*): they hold
 * for later skb_gemm calls made from the calling host thread only
 * (thread-local); production callers never need them.
 *
 * Force the tcgen05 tile configuration of later skb_gemm calls (tests and
 * tuning): N-tile width bn in {64,128,256}, multicast cluster size cs in
 * {1,2,4}, split-K factor; 0 = choose automatically. */
int skb_gemm_force(int bn, int cs, int splits);

/* Select the swap-AB decode GEMM (weights on the MMA M side, one tile per
 * CTA, whole-smem TMA ring, K split across a cluster with a DSMEM
 * reduction): mode 0 = automatic (M <= 1024), 1 = never, 2 = always;
 * na = activation rows per tile (multiple of 16, <= 256), cs = cluster
 * K-split; 0 = choose automatically. */
int skb_gemm_force_sw(int mode, int na, int cs);

/* Select the persistent CTA-pair GEMM (tcgen05.mma.cta_group::2, 256 weight
 * rows x na activation rows per tile, two TMEM accumulators): mode 0 =
 * automatic (M >= 1024 and N >= 8192 outside the LOGITS epilogue, i.e. the
 * cross-attention K/V projection of a batch; shapes without a cluster
 * K-split), 1 = never,
 * 2 = always where applicable; na in {32..256} step 32, pairs = CTA pairs per
 * launch; 0 = choose automatically.  Bitwise equal to the swap-AB kernel. */
int skb_gemm_force_pc(int mode, int na, int pairs);

/*
 * INT8 feed-forward path (replaces skiff quant.py:40-53 quantize_rows,
 * :65-78 _gemm_i8_numba, :99-104 quantize_activations and :121-132
 * QuantizedLinear.__call__).
 *
 * skb_quantize_rows: per-row symmetric int8 quantization of fp32 rows,
 * scale = max|row| / 127 (1 for a zero row), q = clip(round-half-away(x /
 * scale), -127, 127); bit-identical to the reference's float32 arithmetic.
 * Used offline for weights and per step for activations.
 *
 * skb_gemm_i8: acc = A . W^T in exact int32 (tcgen05 kind::i8), then
 * out = (float(acc) * a_scale[m]) * w_scale[n] followed by the epilogue
 * (STORE / RELU with bias, or RESID x += ... + bias).  A [M, lda] and
 * W [N, ldw] int8 K-major, K % 16 == 0, 16-byte aligned.
 */
/*
 * Teacher-forced decoder pass (replaces skiff model.py:444-493
 * forward_sequence): all B x T target positions at once.
 * skb_causal_self_attention: multi-head self-attention of B sequences of T
 * positions over a fused [B*T, 3*H*dh] Q|K|V buffer, query t attending to
 * keys <= t (kernels.py:487-491 causal_mask); lengths [B] (device) bound the
 * keys of each sequence.
 * skb_ssru_scan: the SSRU recurrence along T (model.py:482-493) from the
 * fp32 [B*T, 2d] interleaved gate GEMM output g; x += relu(c_t).
 */
int skb_causal_self_attention(int B, int T, int H, int dh, const void *qkv, int ld_qkv,
                              int qkv_dtype, const int *lengths, void *ctx, int ldc, int ctx_dtype,
                              void *stream);
int skb_ssru_scan(int B, int T, int d, const float *g, int ldg, const float *bias, float *x, int ldx,
                  void *stream);

int skb_quantize_rows(int rows, int k, const float *x, int ldx, void *q, int ldq, float *scales,
                      void *stream);
int skb_gemm_i8(int M, int N, int K, const void *A, int lda, const float *a_scale, const void *W,
                int ldw, const float *w_scale, const skb_epilogue *epi, void *stream);


/* Same, forcing the SIMT path (for parity tests of the tcgen05 path). */
int skb_gemm_simt(int in_dtype, int M, int N, int K, const void *A, int lda, const void *W,
                  int ldw, const skb_epilogue *epi, void *stream);

/*
 * Pre-norm layer norm over rows of width d, population variance, eps.
 * Replaces kernels.py:298-324.  x fp32 [rows, ldx]; out [rows, ldo] out_dtype.
 */
int skb_layernorm(int rows, int d, const float *x, int ldx, const float *gain,
                  const float *bias, float eps, void *out, int ldo, int out_dtype,
                  void *stream);

/*
 * Target-side step embedding (model.py:399-410, 545-547):
 * x[r] = E[tok[r]] + PE[*step] + sum_k F_k[ftok[k*rows + r]].
 * pe: [max_steps, d] fp32 position table (float64 sin/cos cast to fp32).
 * ftables: array (device) of n_factors device pointers to [V_k, d] fp32.
 */
int skb_embed_target(int rows, int d, const int *tok, const float *E, const float *pe,
                     const int *step, int n_factors, const int *ftok,
                     const float *const *ftables, float *x, void *stream);

/*
 * Source embedding (model.py:370-397) for B x L padded ids:
 * surface E_src[id] + PE over the first ds = d - sum(concat dims) columns,
 * concat factor embeddings after it, then sum-combined factors added.
 * fdims[i] = factor dim, fcombine[i] = 0 sum / 1 concat (host arrays),
 * fids: device [n_factors, B*L]; ftables: device array of device pointers.
 */
int skb_embed_source(int B, int L, int d, int ds, const int *ids, const float *E,
                     const float *pe, int n_factors, const int *fdims_host,
                     const int *fcombine_host, const int *fids,
                     const float *const *ftables, float *x, void *stream);

/*
 * Encoder self-attention (kernels.py:510-547 with the pad bias of
 * model.py:174-179): qkv [B*L, ld_qkv] holds q | k | v (each d wide, dtype
 * qkv_dtype); lengths [B] int; ctx [B*L, ldc] in ctx_dtype.
 */
int skb_encoder_attention(int B, int L, int H, int dh, const void *qkv, int ld_qkv,
                          int qkv_dtype, const int *lengths, void *ctx, int ldc,
                          int ctx_dtype, void *stream);

/*
 * Incremental decoder self-attention for one step (model.py:559-567):
 * row r attends over positions 0..t (t = *step) of its hypothesis.  New k,v
 * (from qkv) are stored at cache slot (r, t); earlier positions p < t are
 * read from slot anc[(t&1)][r][p] (ancestor table) — the beam
 * reorder never moves cache bytes.  kc/vc: [R_cap, H, S_max, dh] cache_dtype.
 * rows_per_group G > 1 promises that rows [g*G, g*G+G) only reference slots
 * in that range (beam rows of one sentence): one CTA per (group, head) then
 * stages the group's cache tiles in shared memory.
 */
int skb_self_attention_step(int R, int H, int dh, const void *qkv, int ld_qkv, int qkv_dtype,
                            void *kc, void *vc, int cache_dtype, int S_max, const int *anc,
                            const int *step, int rows_per_group, void *ctx, int ldc,
                            int ctx_dtype, void *stream);

/*
 * Step plan for the self-attention of all decoder layers (model.py:559-566
 * reads the same per-row K/V history in every layer): for each group of
 * rows_per_group rows (a sentence's beam) the distinct (slot, position)
 * cache entries on the rows' ancestor paths at step *step, with a row mask
 * per entry.  plan: caller-owned device buffer of skb_attn_plan_bytes().
 */
size_t skb_attn_plan_bytes(int R, int rows_per_group, int S_max);
int skb_attn_plan(int R, int rows_per_group, int S_max, const int *anc, const int *step,
                  void *plan, void *stream);
/* Test override (calling host thread only) of the tensor-core attention's  */
/* heads per CTA: 2, 4 or 8; 0 = automatic (4, or 2 for small grids).      */
/* Never changes the numbers.                                               */
int skb_attn_force_heads(int hg);
/* skb_self_attention_step over a step plan instead of the ancestor table   */
/* (bitwise equal); bf16, d_h = 64, rows_per_group <= 16, else             */
/* SKB_ERR_UNSUPPORTED.                                                     */
int skb_self_attention_step_planned(int R, int H, int dh, const void *qkv, int ld_qkv,
                                    int qkv_dtype, void *kc, void *vc, int cache_dtype, int S_max,
                                    const void *plan, const int *step, int rows_per_group,
                                    void *ctx, int ldc, int ctx_dtype, void *stream);

/*
 * Cross-attention for one step (model.py:568-573): q [R, ldq]; row r reads
 * sentence row_sent[r] of the per-sentence encoder K/V memory
 * kv [B*L, ld_kv] (K at column offset koff, V at voff), masked past
 * lengths[sentence].  Rows [g*G, g*G+G) (G = rows_per_group, the beam) must
 * share one sentence: its K/V slice is staged in shared memory once per
 * (group, head) and read by all G rows.
 */
int skb_cross_attention_step(int R, int H, int dh, const void *q, int ldq, int q_dtype,
                             const void *kv, int ld_kv, int kv_dtype, int koff, int voff,
                             int L, const int *row_sent, const int *lengths, int rows_per_group,
                             void *ctx, int ldc, int ctx_dtype, void *stream);

/* Gather rows of a table: out[i] = table[idx[i]] (row width w, dtype). Used to
 * build the restricted output-projection operand E[active] (model.py:577-581). */
int skb_gather_rows(int n, int w, const void *table, int ld_table, const int *idx,
                    void *out, int ld_out, int dtype, void *stream);

/*
 * Beam search step state (all device memory, sized by the caller).
 * Rows are slots r = b*K + i (sentence b, beam position i).
 * Replaces the per-step body of search.py:345-393 (and greedy 292-312,
 * which is its beam = 1 special case, bit-identical per test_search.py:170).
 */
typedef struct skb_beam_state {
  int B, K, U;            /* sentences, beam, columns of the logits          */
  int S_max;              /* history capacity (steps)                        */
  int n_factors;          /* target factor streams                           */
  const double *len_pen;  /* [S_max+1] steps**alpha, computed on the host so */
                          /* it is bit-identical to search.py:74-75          */
  const int *step;        /* device: current step t                          */
  const int *col_token;   /* [U] token id of column (NULL: identity)         */
  const unsigned *mask;   /* [B, ceil(U/32)] active-column bits (NULL: all)  */
  int eos_col;            /* column of EOS                                    */
  const int *max_len;     /* [B] 2*L+10 per sentence (search.py:231)          */
  const int *prefix_len;  /* [B]                                              */
  const int *prefix_col;  /* [B, P] forced column per step (search.py:296)   */
  int P;
  const int *prefix_fac;  /* [B, n_factors, P] prefix factor ids or -1        */
  int *n_alive;           /* [B] alive rows (starts at 1)                     */
  int *done;              /* [B] sentence finished flag                       */
  double *score;          /* [R] alive hypothesis log-prob (float64), in place*/
  int *tok_next;          /* [R] token fed at the next step                   */
  int *ftok_next;         /* [n_factors, R] factor ids fed next step          */
  int *parent;            /* [R] parent slot of each new row                   */
  int *tok_hist;          /* [S_max, R] token appended at step t              */
  int *par_hist;          /* [S_max, R] parent beam index at step t           */
  int *fac_hist;          /* [S_max, n_factors, R] factor of the new row       */
  const float *fac_logits;/* [R, fac_ld] all factor heads side by side, or NULL*/
  int fac_ld;             /* row stride of fac_logits                          */
  const int *fac_off;     /* [n_factors+1] column offsets (device)            */
  const float *lse_part;  /* [R, lse_ld] float2 partials from SKB_EPI_LOGITS  */
                          /* (NULL: the step kernel reduces the row itself)  */
  int lse_ld;
  int prune;              /* 1: read only the 32-column groups whose partial  */
                          /* max can reach the top K (exact, see search.cu)  */
  int stage_partials;     /* set by the library (shared-memory staging)      */
  /* scratch */
  double *cand_score;     /* [R, K] */
  float *cand_lp;         /* [R, K] */
  int *cand_col;          /* [R, K] */
  int *cand_cnt;          /* [R]    */
  int *row_argmax;        /* [R]    */
  int *fac_choice;        /* [R, n_factors] */
  unsigned *counter;      /* [B] zero-initialised arrival counters            */
  /* best finished hypothesis per sentence (search.py:394) */
  double *best_norm;      /* [B] */
  double *best_logprob;   /* [B] */
  int *best_steps;        /* [B] 0 = none yet */
  int *best_forced;       /* [B] */
  int *best_parent;       /* [B] beam index of the parent row at step steps-1 */
  int *best_fac;          /* [B, n_factors] factor entry of the EOS step */
  int *n_done;            /* [1] sentences finished (for host polling)      */
} skb_beam_state;

/*
 * One beam step over fp32 logits [R, ld_logits]: per row masked
 * log-softmax (kernels.py:287-295), float64 candidate scores, exact
 * (score desc, token asc, parent asc) top-K per sentence (search.py:363),
 * EOS routing, forced prefix/EOS steps, finished-hypothesis tracking.
 * If lp_in is non-zero the logits are taken as already-normalised fp32
 * log-probs (bit-exact parity harness: "given identical scores").
 */
int skb_beam_step(const float *logits, int ld_logits, int lp_in, const skb_beam_state *st,
                  void *stream);

/*
 * Beam reorder (model.py:316-330 select_rows): ancestor table
 * anc[(t+1)&1][r][p] = anc[t&1][parent[r]][p] for p < t and = parent[r] at
 * p = t.  Also advances *step.  SSRU cells are gathered inside the SSRU GEMM
 * epilogue via src_row = parent.
 */
int skb_beam_reorder(int R, int S_max, int *anc, const int *parent, int *step, void *stream);

/*
 * Backtrack the best finished hypothesis of every sentence through the
 * per-step history: tokens_out [B, S_max] (EOS excluded), factors_out
 * [B, n_factors, S_max] (one entry per step incl. the EOS step).
 */
int skb_beam_finalize(const skb_beam_state *st, int *tokens_out, int *factors_out,
                      void *stream);

/* Debug: copy the beam kernel's per-row phase timestamps (only in builds
 * with -DSKB_PROFILE_PHASES; SKB_ERR_UNSUPPORTED otherwise). */
int skb_debug_beam_prof(unsigned long long *host_buf_4096x10);

/* Debug: per-CTA %globaltimer stamps of the last swap-AB GEMM launch
 * (entry, pre-wait, post-wait, first stage, last MMA, accumulator ready,
 * exit, smid, reduction phases) — builds with -DSKB_GEMM_TRACE only. */
int skb_debug_gemm_trace(unsigned long long *host_buf_1024x16);

/* Debug: per-CTA %globaltimer stamps of the last tensor-core self-attention
 * launch (entry, after PDL wait, walk, entries, staged, attended) — builds
 * with -DSKB_ATTN_TRACE only; read-and-clear. */
int skb_debug_attn_trace(unsigned long long *host_buf_4096x8);

/* out[r] = max over positions l < len[b] of enc[b, l, :] (model.py:496-500). */
int skb_masked_maxpool(int B, int L, int d, const float *enc, const int *lengths, float *out,
                       void *stream);

/* Element-wise dtype conversion (fp32 <-> bf16) of n elements. */
int skb_convert(long long n, const void *src, int src_dtype, void *dst, int dst_dtype,
                void *stream);

/* NVS vocabulary selection bits (model.py:511-517): bit c of row b is set iff
 * sigmoid(logits[b, c]) > threshold.  mask: [B, ceil(V/32)]. */
int skb_nvs_mask(int B, int V, const float *logits, int ld, float threshold, unsigned *mask,
                 void *stream);

/* Select the CUDA device used by this library's calls on the current thread
 * (one process per GPU; mirrors torch.cuda.set_device). */
int skb_set_device(int device);

#ifdef __cplusplus
}
#endif
#endif /* SKIFF_B200_H */
