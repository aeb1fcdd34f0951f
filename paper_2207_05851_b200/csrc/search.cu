// Beam search bookkeeping on the device (skiff search.py:275-394).
//
// skb_beam_step: one CTA per row slot r = b*K + i.  Pass 1/2 compute the
// masked row max and sum of exp (log_softmax over the sentence's active
// columns, kernels.py:287-295); pass 3 computes lp = (x - max) - log(sum)
// per column, the first-max column (np.argmax) and a per-thread top-K of the
// float64 candidate scores s_r + lp (search.py:353-358), merged across the
// CTA with warp shuffles.  The last CTA of a sentence to arrive (atomic
// counter) merges the <= K row lists in the exact order (score desc, token
// asc, parent asc) of np.lexsort (search.py:363), routes EOS candidates to
// the finished set, compacts survivors into new rows and records history
// for the final backtrack.  Forced steps (target prefix, final EOS) use the
// float32 candidate keys the reference builds there (python float +
// np.float32 -> float32 under NEP 50, search.py:353-355).

#include "common.cuh"

#include <cfloat>

namespace skb {

constexpr int BEAM_THREADS = 256;
constexpr int EOS = 3, PAD = 0;

struct Cand {
  double key;
  float lp;
  int col;
};

__device__ __forceinline__ bool better(double k1, int c1, double k2, int c2) {
  return k1 > k2 || (k1 == k2 && c1 < c2);
}

__device__ __forceinline__ bool col_active(const unsigned *mask, int c) {
  return mask == nullptr || ((mask[c >> 5] >> (c & 31)) & 1u);
}

template <int MAXK>
__device__ __forceinline__ void list_insert(double (&k)[MAXK], float (&l)[MAXK], int (&c)[MAXK],
                                            double key, float lp, int col) {
  // caller guarantees better(key, col, k[MAXK-1], c[MAXK-1])
  k[MAXK - 1] = key;
  l[MAXK - 1] = lp;
  c[MAXK - 1] = col;
#pragma unroll
  for (int j = MAXK - 1; j > 0; --j) {
    if (better(k[j], c[j], k[j - 1], c[j - 1])) {
      double tk = k[j]; k[j] = k[j - 1]; k[j - 1] = tk;
      float tl = l[j]; l[j] = l[j - 1]; l[j - 1] = tl;
      int tc = c[j]; c[j] = c[j - 1]; c[j - 1] = tc;
    }
  }
}


// K-th largest of the values held by a CTA (each thread passes its values
// through `feed`); K <= MAXK.  Exact; used to bound the beam threshold from
// the per-32-column group maxima the output GEMM wrote.
template <int MAXK>
__device__ __forceinline__ void warp_topk_vals(float (&v)[MAXK], int K, float *out_warp) {
  // v sorted descending per lane; K rounds of warp max with pop-one
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < K; ++j) {
    float b = v[0];
    int bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ob > b || (ob == b && ol < bl)) {
        b = ob;
        bl = ol;
      }
    }
    if (lane == 0) out_warp[j] = b;
    if (lane == bl) {
#pragma unroll
      for (int q = 0; q + 1 < MAXK; ++q) v[q] = v[q + 1];
      v[MAXK - 1] = -INFINITY;
    }
  }
}

template <int MAXK>
__device__ __forceinline__ void vals_insert(float (&v)[MAXK], float x) {
  v[MAXK - 1] = x;
#pragma unroll
  for (int j = MAXK - 1; j > 0; --j)
    if (v[j] > v[j - 1]) {
      const float t = v[j];
      v[j] = v[j - 1];
      v[j - 1] = t;
    }
}

template <int MAXK>
__global__ void __launch_bounds__(BEAM_THREADS) k_beam_step(const float *__restrict__ logits,
                                                            int ld, int lp_in, skb_beam_state st) {
  const int r = blockIdx.x;
  const int K = st.K, U = st.U;
  const int b = r / K, i = r % K;
  const int R = st.B * K;
  const int t = *st.step;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BEAM_THREADS / 32;

  __shared__ float red_f[NW];
  __shared__ int red_i[NW];
  __shared__ double wk[NW][MAXK];
  __shared__ float wl[NW][MAXK];
  __shared__ int wc[NW][MAXK];
  __shared__ int is_last;

  const bool live = !st.done[b] && i < st.n_alive[b];
  if (live) {
    const float *row = logits + (size_t)r * ld;
    const unsigned *mask = st.mask ? st.mask + (size_t)b * ((U + 31) >> 5) : nullptr;
    float mx = 0.f, lse = 0.f;
    if (!lp_in && st.lse_part) {
      // ---- fused path: combine the GEMM epilogue's per-32-column partials
      const float2 *part = reinterpret_cast<const float2 *>(st.lse_part) + (size_t)r * st.lse_ld;
      const int G = (U + 31) >> 5;
      float m = -INFINITY;
      for (int g = tid; g < G; g += BEAM_THREADS) m = fmaxf(m, part[g].x);
      m = warp_max(m);
      if (lane == 0) red_f[warp] = m;
      __syncthreads();
      mx = red_f[0];
      for (int w = 1; w < NW; ++w) mx = fmaxf(mx, red_f[w]);
      __syncthreads();
      float s = 0.f;
      for (int g = tid; g < G; g += BEAM_THREADS) {
        const float2 p = part[g];
        if (p.x != -INFINITY) s += p.y * expf(p.x - mx);
      }
      s = warp_sum(s);
      if (lane == 0) red_f[warp] = s;
      __syncthreads();
      s = 0.f;
      for (int w = 0; w < NW; ++w) s += red_f[w];
      __syncthreads();
      lse = logf(s);
    } else if (!lp_in) {
      // ---- pass 1: max over active columns
      mx = -INFINITY;
      for (int c = tid; c < U; c += BEAM_THREADS)
        if (col_active(mask, c)) mx = fmaxf(mx, row[c]);
      mx = warp_max(mx);
      if (lane == 0) red_f[warp] = mx;
      __syncthreads();
      mx = red_f[0];
      for (int w = 1; w < NW; ++w) mx = fmaxf(mx, red_f[w]);
      __syncthreads();
      // ---- pass 2: sum of exp(x - max)
      float s = 0.f;
      for (int c = tid; c < U; c += BEAM_THREADS)
        if (col_active(mask, c)) s += expf(row[c] - mx);
      s = warp_sum(s);
      if (lane == 0) red_f[warp] = s;
      __syncthreads();
      s = 0.f;
      for (int w = 0; w < NW; ++w) s += red_f[w];
      __syncthreads();
      lse = logf(s);
    }
    const int plen = st.prefix_len[b];
    const bool final_force = (t == st.max_len[b] - 1) && (t >= plen);
    const int fcol = t < plen ? st.prefix_col[(size_t)b * st.P + t] : (final_force ? st.eos_col : -1);
    const double s_r = st.score[r];

    // ---- single pass: lp = (x - max) - lse, first-max column, per-thread
    // top-K of the float64 scores.  A float32 prefilter (lp >= lp of the
    // list's last entry) skips the float64 work for almost every column;
    // it is exact because s_r + lp is monotone in lp and columns arrive in
    // increasing order per thread.
    double tk[MAXK];
    float tl[MAXK];
    int tc[MAXK];
#pragma unroll
    for (int j = 0; j < MAXK; ++j) {
      tk[j] = -DBL_MAX;
      tl[j] = -INFINITY;
      tc[j] = INT_MAX;
    }
    float amax = -INFINITY;
    int acol = INT_MAX;
    const bool need_argmax = final_force;
    const bool do_topk = fcol < 0;
    auto visit = [&](int c, float x) {
      if (mask && !col_active(mask, c)) return;
      const float lp = lp_in ? x : (x - mx) - lse;
      if (need_argmax && lp > amax) {
        amax = lp;
        acol = c;
      }
      if (do_topk && lp >= tl[MAXK - 1]) {
        const double key = s_r + (double)lp;
        if (key > tk[MAXK - 1]) list_insert<MAXK>(tk, tl, tc, key, lp, c);
      }
    };
    const bool pruned = !lp_in && st.lse_part != nullptr && st.prune;
    if (pruned && (do_topk || need_argmax)) {
      // ---- pruned scan: only 32-column groups whose maximum logit can reach
      // the top K are read.  T = K-th largest group maximum <= K-th largest
      // logit, and lp / the float64 key are monotone in x, so every column
      // that can enter the top K by (key desc, col asc) has
      // x >= T - delta, delta covering the float32 rounding of
      // (x - max) - lse and the float64 rounding of s_r + lp (so exact
      // ties are never lost).  At the final step the first-max column of lp
      // is searched the same way around the row maximum.
      __shared__ float wtop[NW][MAXK];
      __shared__ float thr_s;
      const float2 *part = reinterpret_cast<const float2 *>(st.lse_part) + (size_t)r * st.lse_ld;
      const int G = (U + 31) >> 5;
      float thr_top = INFINITY;
      if (do_topk) {
        float gv[MAXK];
#pragma unroll
        for (int j = 0; j < MAXK; ++j) gv[j] = -INFINITY;
        for (int g = tid; g < G; g += BEAM_THREADS) {
          const float v = part[g].x;
          if (v > gv[MAXK - 1]) vals_insert<MAXK>(gv, v);
        }
        const int kk = K < MAXK ? K : MAXK;
        warp_topk_vals<MAXK>(gv, kk, wtop[warp]);
        __syncthreads();
        if (warp == 0) {
          float w[MAXK];
#pragma unroll
          for (int j = 0; j < MAXK; ++j) w[j] = (lane < NW && j < kk) ? wtop[lane][j] : -INFINITY;
          __shared__ float fin[MAXK];
          warp_topk_vals<MAXK>(w, kk, fin);
          __syncwarp();
          if (lane == 0) {
            const float T = fin[kk - 1];
            const float delta = 4e-6f * (fabsf(T) + fabsf(mx) + fabsf(lse) + 1.0f) +
                                (float)(1e-15 * (fabs(s_r) + 1.0));
            thr_s = T == -INFINITY ? -INFINITY : T - delta;
          }
        }
        __syncthreads();
        thr_top = thr_s;
      }
      const float thr_arg =
          need_argmax ? mx - 4e-6f * (2.0f * fabsf(mx) + fabsf(lse) + 1.0f) : INFINITY;
      const float thr = fminf(thr_top, thr_arg);
      for (int g = tid; g < G; g += BEAM_THREADS) {
        if (!(part[g].x >= thr)) continue;
        const int c0 = g << 5;
        const int c1 = min(U, c0 + 32);
        for (int c = c0; c < c1; ++c) visit(c, row[c]);
      }
    } else if (do_topk || need_argmax) {
      const bool vec = (U & 3) == 0 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0;
      if (vec) {
        const float4 *row4 = reinterpret_cast<const float4 *>(row);
        const int U4 = U >> 2;
        int c4 = tid;
        for (; c4 + 3 * BEAM_THREADS < U4; c4 += 4 * BEAM_THREADS) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = __ldcs(row4 + c4 + u * BEAM_THREADS);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = 4 * (c4 + u * BEAM_THREADS);
            visit(c, v[u].x); visit(c + 1, v[u].y); visit(c + 2, v[u].z); visit(c + 3, v[u].w);
          }
        }
        for (; c4 < U4; c4 += BEAM_THREADS) {
          const float4 v = __ldcs(row4 + c4);
          const int c = 4 * c4;
          visit(c, v.x); visit(c + 1, v.y); visit(c + 2, v.z); visit(c + 3, v.w);
        }
      } else {
        for (int c = tid; c < U; c += BEAM_THREADS) visit(c, row[c]);
      }
    }
    // first max of lp across the CTA (ties -> lowest column)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float oa = __shfl_xor_sync(0xffffffffu, amax, o);
      const int oc = __shfl_xor_sync(0xffffffffu, acol, o);
      if (oa > amax || (oa == amax && oc < acol)) {
        amax = oa;
        acol = oc;
      }
    }
    if (lane == 0) {
      red_f[warp] = amax;
      red_i[warp] = acol;
    }
    // warp-level merge of the 32 thread lists -> top MAXK per warp
    if (fcol < 0) {
      int head = 0;
      for (int j = 0; j < MAXK; ++j) {
        double hk = head < MAXK ? tk[0] : -DBL_MAX;
        int hc = head < MAXK ? tc[0] : INT_MAX;
        double bk = hk;
        int bc = hc, bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
          if (better(ok, oc, bk, bc) || (ok == bk && oc == bc && ol < bl)) {
            bk = ok;
            bc = oc;
            bl = ol;
          }
        }
        const float blp = __shfl_sync(0xffffffffu, tl[0], bl);
        if (lane == 0) {
          wk[warp][j] = bk;
          wl[warp][j] = blp;
          wc[warp][j] = bc;
        }
        if (lane == bl) {  // pop the head of the winning lane's list
#pragma unroll
          for (int q = 0; q + 1 < MAXK; ++q) {
            tk[q] = tk[q + 1];
            tl[q] = tl[q + 1];
            tc[q] = tc[q + 1];
          }
          tk[MAXK - 1] = -DBL_MAX;
          tc[MAXK - 1] = INT_MAX;
          ++head;
        }
      }
    }
    __syncthreads();
    if (warp == 0) {
      // CTA-level first max
      float a = lane < NW ? red_f[lane] : -INFINITY;
      int ac = lane < NW ? red_i[lane] : INT_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float oa = __shfl_xor_sync(0xffffffffu, a, o);
        const int oc = __shfl_xor_sync(0xffffffffu, ac, o);
        if (oa > a || (oa == a && oc < ac)) {
          a = oa;
          ac = oc;
        }
      }
      if (lane == 0) st.row_argmax[r] = ac;
      if (fcol >= 0) {
        if (lane == 0) {
          const float x = row[fcol];
          const float lp = lp_in ? x : (x - mx) - lse;
          // forced steps: float32 key fl32(fl32(s) + lp) (NEP 50 promotion)
          const float key32 = (float)s_r + lp;
          st.cand_score[(size_t)r * K] = (double)key32;
          st.cand_lp[(size_t)r * K] = lp;
          st.cand_col[(size_t)r * K] = fcol;
          st.cand_cnt[r] = 1;
        }
      } else {
        // merge NW warp lists (each sorted) -> top K
        int head = 0;  // lane w (< NW) walks warp w's list
        const int kk = K < MAXK ? K : MAXK;
        for (int j = 0; j < kk; ++j) {
          const bool has = lane < NW && head < MAXK;
          double bk = has ? wk[lane][head] : -DBL_MAX;
          int bc = has ? wc[lane][head] : INT_MAX;
          const float my_lp = has ? wl[lane][head] : 0.f;
          int bl = lane;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
            const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
            if (better(ok, oc, bk, bc) || (ok == bk && oc == bc && ol < bl)) {
              bk = ok;
              bc = oc;
              bl = ol;
            }
          }
          const float blp = __shfl_sync(0xffffffffu, my_lp, bl);
          if (lane == 0) {
            st.cand_score[(size_t)r * K + j] = bk;
            st.cand_col[(size_t)r * K + j] = bc;
            st.cand_lp[(size_t)r * K + j] = blp;
          }
          if (lane == bl) ++head;
        }
        if (lane == 0) {
          int cnt = 0;
          for (int j = 0; j < kk; ++j) cnt += st.cand_col[(size_t)r * K + j] != INT_MAX;
          st.cand_cnt[r] = cnt;
        }
      }
      // factor choices of this row (search.py:261-272)
      if (lane == 0) {
        for (int k = 0; k < st.n_factors; ++k) {
          int choice = -1;
          if (t >= 1 && st.prefix_fac) {
            const int pf = t - 1 < st.P ? st.prefix_fac[((size_t)b * st.n_factors + k) * st.P + t - 1] : -1;
            choice = pf;
          }
          if (choice < 0) {
            const float *fr = st.fac_logits + (size_t)r * st.fac_ld;
            const int lo = st.fac_off[k], hi = st.fac_off[k + 1];
            float bm = -INFINITY;
            int bcol = 0;
            for (int c = lo; c < hi; ++c)
              if (fr[c] > bm) {
                bm = fr[c];
                bcol = c - lo;
              }
            choice = bcol;
          }
          st.fac_choice[(size_t)r * st.n_factors + k] = choice;
        }
      }
    }
  } else if (tid == 0) {
    st.cand_cnt[r] = 0;
  }

  // ---- arrival: the last row CTA of the sentence does the merge
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st.counter[b], 1u);
    is_last = prev == (unsigned)(K - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  __shared__ double m_key[MAXK * MAXK];
  __shared__ float m_lp[MAXK * MAXK];
  __shared__ int m_col[MAXK * MAXK];
  __shared__ int m_cnt[MAXK], m_arg[MAXK];
  __shared__ double m_s[MAXK];
  __shared__ int p_q[MAXK], p_c[MAXK], p_tok[MAXK];
  __shared__ float p_lp[MAXK];
  __shared__ int n_pick;
  const int base = b * K;
  const int nf = st.n_factors;
  if (__ldcg(st.done + b)) {
    if (tid == 0) st.counter[b] = 0;
    return;
  }
  const int nalive = __ldcg(st.n_alive + b);
  // stage every row list of the sentence in shared memory with one parallel
  // round of L2 reads (they were written by other CTAs of this launch)
  for (int idx = tid; idx < nalive * K; idx += BEAM_THREADS) {
    const int q = idx / K, j = idx % K;
    const size_t g = (size_t)(base + q) * K + j;
    m_key[q * MAXK + j] = __ldcg(st.cand_score + g);
    m_lp[q * MAXK + j] = __ldcg(st.cand_lp + g);
    m_col[q * MAXK + j] = __ldcg(st.cand_col + g);
  }
  if (tid < nalive) {
    m_cnt[tid] = __ldcg(st.cand_cnt + base + tid);
    m_s[tid] = __ldcg(st.score + base + tid);
    m_arg[tid] = __ldcg(st.row_argmax + base + tid);
  }
  __syncthreads();
  if (warp != 0) return;
  // ---- warp 0: K rounds of a warp-wide argmax over the row-list heads in the
  // exact order (score desc, token asc, parent asc); columns are sorted by
  // token, so token order is column order.
  int head = 0;
  int npk = 0;
  for (int sel = 0; sel < K; ++sel) {
    bool has = lane < nalive && head < m_cnt[lane];
    double bk = has ? m_key[lane * MAXK + head] : 0.0;
    int bc = has ? m_col[lane * MAXK + head] : 0;
    int bq = lane;
    bool bh = has;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
      const bool oh = __shfl_xor_sync(0xffffffffu, (int)bh, o) != 0;
      const bool take = oh && (!bh || ok > bk || (ok == bk && (oc < bc || (oc == bc && oq < bq))));
      if (take) {
        bk = ok;
        bc = oc;
        bq = oq;
        bh = true;
      }
    }
    if (!bh) break;
    if (lane == bq) {
      p_q[sel] = bq;
      p_c[sel] = bc;
      p_lp[sel] = m_lp[lane * MAXK + head];
      p_tok[sel] = st.col_token ? st.col_token[bc] : bc;
      ++head;
    }
    npk = sel + 1;
  }
  __syncwarp();
  if (lane != 0) return;
  // ---- sequential routing of the picks (search.py:370-386) from shared memory
  const int plen = st.prefix_len[b];
  const bool final_force = (t == st.max_len[b] - 1) && (t >= plen);
  const int steps = t + 1;
  const double pen = st.len_pen[steps];
  int best_steps = st.best_steps[b];
  double best_norm = st.best_norm[b];
  int n_new = 0;
  for (int sel = 0; sel < npk; ++sel) {
    const int q = p_q[sel], c = p_c[sel], token = p_tok[sel];
    const int rr = base + q;
    const double score = m_s[q] + (double)p_lp[sel];
    if (token == EOS) {
      const double norm = score / pen;
      if (best_steps == 0 || norm > best_norm) {
        best_norm = norm;
        best_steps = steps;
        st.best_norm[b] = norm;
        st.best_logprob[b] = score;
        st.best_steps[b] = steps;
        st.best_forced[b] = final_force && m_arg[q] != c;
        st.best_parent[b] = q;
        for (int k = 0; k < nf; ++k)
          st.best_fac[(size_t)b * nf + k] = __ldcg(st.fac_choice + (size_t)rr * nf + k);
      }
    } else {
      const int slot = base + n_new;
      st.tok_next[slot] = token;
      st.parent[slot] = rr;
      st.score[slot] = score;
      st.tok_hist[(size_t)t * R + slot] = token;
      st.par_hist[(size_t)t * R + slot] = q;
      for (int k = 0; k < nf; ++k) {
        const int f = __ldcg(st.fac_choice + (size_t)rr * nf + k);
        st.ftok_next[(size_t)k * R + slot] = f;
        st.fac_hist[((size_t)t * nf + k) * R + slot] = f;
      }
      ++n_new;
    }
  }
  for (int q = n_new; q < K; ++q) {
    st.tok_next[base + q] = PAD;
    st.parent[base + q] = base;
    for (int k = 0; k < nf; ++k) st.ftok_next[(size_t)k * R + base + q] = PAD;
  }
  st.n_alive[b] = n_new;
  st.counter[b] = 0;
  if (n_new == 0) {
    st.done[b] = 1;
    atomicAdd(st.n_done, 1);
  }
  (void)n_pick;
}

// ------------------------------------------------------------- reorder
__global__ void k_beam_reorder(int R, int S_max, int *anc, const int *parent, const int *step) {
  const int r = blockIdx.y;
  const int t = *step;
  const int p = parent[r];
  const int *src = anc + ((size_t)(t & 1) * R + p) * S_max;
  int *dst = anc + ((size_t)((t + 1) & 1) * R + r) * S_max;
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos <= t && pos < S_max;
       pos += gridDim.x * blockDim.x)
    dst[pos] = pos == t ? p : src[pos];
}

__global__ void k_step_advance(int *step) { *step += 1; }

// ------------------------------------------------------------ finalize
__global__ void k_beam_finalize(skb_beam_state st, int *tokens_out, int *factors_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= st.B) return;
  const int K = st.K, R = st.B * K, nf = st.n_factors;
  const int steps = st.best_steps[b];
  if (steps <= 0) return;
  const int tfin = steps - 1;
  int q = st.best_parent[b];
  for (int k = 0; k < nf; ++k)
    factors_out[((size_t)b * nf + k) * st.S_max + tfin] = st.best_fac[(size_t)b * nf + k];
  for (int pos = tfin - 1; pos >= 0; --pos) {
    const int slot = b * K + q;
    tokens_out[(size_t)b * st.S_max + pos] = st.tok_hist[(size_t)pos * R + slot];
    for (int k = 0; k < nf; ++k)
      factors_out[((size_t)b * nf + k) * st.S_max + pos] = st.fac_hist[((size_t)pos * nf + k) * R + slot];
    q = st.par_hist[(size_t)pos * R + slot];
  }
}

}  // namespace skb

using namespace skb;

extern "C" int skb_beam_step(const float *logits, int ld_logits, int lp_in, const skb_beam_state *st,
                             void *stream) {
  if (!st || st->B <= 0 || st->K <= 0 || st->U <= 0)
    return fail(SKB_ERR_SHAPE, "beam_step: bad state");
  if (st->K > 32) return fail(SKB_ERR_CONFIG, "beam size %d exceeds 32", st->K);
  const int R = st->B * st->K;
  cudaStream_t s = as_stream(stream);
  if (st->K <= 1)
    k_beam_step<1><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  else if (st->K <= 2)
    k_beam_step<2><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  else if (st->K <= 4)
    k_beam_step<4><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  else if (st->K <= 5)
    k_beam_step<5><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  else if (st->K <= 8)
    k_beam_step<8><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  else if (st->K <= 16)
    k_beam_step<16><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  else
    k_beam_step<32><<<R, BEAM_THREADS, 0, s>>>(logits, ld_logits, lp_in, *st);
  SKB_CHECK_LAUNCH("k_beam_step");
  return SKB_OK;
}

extern "C" int skb_beam_reorder(int R, int S_max, int *anc, const int *parent, int *step,
                                void *stream) {
  if (R <= 0 || S_max <= 0) return fail(SKB_ERR_SHAPE, "beam_reorder: bad shape");
  cudaStream_t s = as_stream(stream);
  dim3 grid((S_max + 127) / 128, R);
  k_beam_reorder<<<grid, 128, 0, s>>>(R, S_max, anc, parent, step);
  SKB_CHECK_LAUNCH("k_beam_reorder");
  k_step_advance<<<1, 1, 0, s>>>(step);
  SKB_CHECK_LAUNCH("k_step_advance");
  return SKB_OK;
}

extern "C" int skb_beam_finalize(const skb_beam_state *st, int *tokens_out, int *factors_out,
                                 void *stream) {
  if (!st || st->B <= 0) return fail(SKB_ERR_SHAPE, "beam_finalize: bad state");
  k_beam_finalize<<<(st->B + 127) / 128, 128, 0, as_stream(stream)>>>(*st, tokens_out, factors_out);
  SKB_CHECK_LAUNCH("k_beam_finalize");
  return SKB_OK;
}
