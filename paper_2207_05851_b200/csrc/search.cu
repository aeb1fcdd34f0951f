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


// Order-preserving integer images of fp32 / fp64 keys (no NaNs occur;
// -0 is folded into +0 so that equal keys map to equal images), so warp
// selections run on redux.sync instead of five-level shuffle trees.
__device__ __forceinline__ unsigned ord32(float v) {
  const unsigned u = __float_as_uint(v + 0.0f);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord32(unsigned o) {
  return __uint_as_float((o >> 31) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ unsigned long long ord64(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v + 0.0);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Lane holding the best entry of the warp in the order (key desc, col asc,
// lane asc) among lanes with `has`; -1 if none.
__device__ __forceinline__ int warp_best(double key, int col, bool has) {
  const unsigned long long o = ord64(key);
  const unsigned hi = has ? (unsigned)(o >> 32) : 0u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const bool h1 = has && hi == mh;
  const unsigned ml = __reduce_max_sync(0xffffffffu, h1 ? (unsigned)o : 0u);
  const bool h2 = h1 && (unsigned)o == ml;
  const unsigned mc = __reduce_min_sync(0xffffffffu, h2 ? (unsigned)col : 0xffffffffu);
  const unsigned who = __ballot_sync(0xffffffffu, h2 && (unsigned)col == mc);
  return who ? __ffs(who) - 1 : -1;
}

// First maximum (value desc, column asc) across the warp.
__device__ __forceinline__ void warp_argmax(float &v, int &col) {
  const unsigned m = __reduce_max_sync(0xffffffffu, ord32(v));
  const unsigned c = __reduce_min_sync(0xffffffffu, ord32(v) == m ? (unsigned)col : 0xffffffffu);
  v = unord32(m);
  col = (int)c;
}

// K rounds of "take the warp maximum of the lanes' sorted lists' heads";
// writes the K values (descending) through lane 0 when out != nullptr and
// returns the K-th largest.  Exact; used to bound the beam threshold from the
// per-32-column group maxima the output GEMM wrote.
template <int MAXK>
__device__ __forceinline__ float warp_kth(float (&v)[MAXK], int K, float *out = nullptr) {
  const int lane = threadIdx.x & 31;
  float last = -INFINITY;
  for (int j = 0; j < K; ++j) {
    const unsigned o = ord32(v[0]);
    const unsigned m = __reduce_max_sync(0xffffffffu, o);
    const int bl = __ffs(__ballot_sync(0xffffffffu, o == m)) - 1;
    last = unord32(m);
    if (out && lane == 0) out[j] = last;
    if (lane == bl) {
#pragma unroll
      for (int q = 0; q + 1 < MAXK; ++q) v[q] = v[q + 1];
      v[MAXK - 1] = -INFINITY;
    }
  }
  return last;
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

// Optional phase timestamps (build with SKB_NVCC_EXTRA=-DSKB_PROFILE_PHASES)
#ifdef SKB_PROFILE_PHASES
__device__ unsigned long long g_tprof[4096 * 10];
#define TP(k)                                                                         \
  do {                                                                                \
    unsigned long long _t;                                                            \
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(_t)::"memory");                   \
    if (lane == 0 && r < 1024 && s < 4) g_tprof[((s << 10) + r) * 10 + (k)] = _t;     \
  } while (0)
#else
// phase boundaries stay compiler scheduling fences: without them ptxas
// interleaves the phases of k_beam_step and the kernel runs ~1.7x slower
#define TP(k) asm volatile("" ::: "memory")
#endif

// Shared-memory layout of one sentence CTA (K rows x SUB warps).
template <int MAXK, int SUB>
struct BeamSmem {
  double key[MAXK][MAXK];   // row lists (row, rank)
  float lp[MAXK][MAXK];
  int col[MAXK][MAXK];
  int cnt[MAXK];
  int arg[MAXK];
  int cg[MAXK][SUB][64];    // per-warp candidate group list
  // per-warp partial results of a row, combined by the row's first warp
  double skey[MAXK][SUB][MAXK];
  float slp[MAXK][SUB][MAXK];
  int scol[MAXK][SUB][MAXK];
  int scnt[MAXK][SUB];
  float sav[MAXK][SUB];     // first-max argmax (value, column)
  int sac[MAXK][SUB];
  float rm[MAXK][SUB];      // row max / sum of exp partials
  float rs[MAXK][SUB];
  float rgv[MAXK][SUB * MAXK];  // top group maxima
};

#ifndef SKB_BEAM_SUB5
#define SKB_BEAM_SUB5 4  // warps per beam row at K = 5
#endif

// Barrier over the SUB warps of one beam row (named barrier 1 + row).
template <int SUB>
__device__ __forceinline__ void row_sync(int row) {
  __syncwarp();
#ifdef SKB_ROWSYNC_ALL
  __syncthreads();
#else
  if constexpr (SUB > 1) asm volatile("barrier.sync %0, %1;" ::"r"(1 + row), "r"(SUB * 32) : "memory");
#endif
}

// One CTA per sentence, SUB warps per beam row (slot r = b*K + i); the rows
// exchange their candidate lists through shared memory (one barrier), so
// there are no global atomics or fences.  Per row, each warp takes every
// SUB-th block of 32 columns (groups):
//   1. log-softmax statistics: combine the output GEMM's per-32-column
//      (max, sum exp) partials (staged in shared memory), or reduce the row;
//      the warps' max / sum partials are combined in warp order;
//   2. candidate columns: with partials, only 32-column groups whose max can
//      reach the top K (exact pruning: the margin covers the fp32 rounding
//      of (x - max) - lse and the fp64 rounding of s_r + lp, so ties are
//      never lost); otherwise every active column;
//   3. per-lane top-K of float64 keys s_r + lp (first-max argmax of lp at the
//      final step), merged across the warp with shuffles, then across the
//      row's warps (columns are disjoint, so the order stays exact);
// then warp 0 merges the <= K row lists in lexsort order (score desc, token
// asc, parent asc) and routes EOS / survivors (search.py:363-393).
template <int MAXK, int SUB>
__global__ void __launch_bounds__(MAXK * 32 * SUB)
    k_beam_step(const float *__restrict__ logits, int ld, int lp_in, skb_beam_state st) {
  extern __shared__ __align__(16) uint8_t beam_smem[];
  using Smem = BeamSmem<MAXK, SUB>;
  Smem &sm = *reinterpret_cast<Smem *>(beam_smem);
  float2 *part_s = reinterpret_cast<float2 *>(beam_smem + ((sizeof(Smem) + 15) & ~size_t(15)));
  constexpr int SW = 32 * SUB;  // threads per row
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = w / SUB, s = w % SUB;
  const int K = st.K, U = st.U;
  const int R = st.B * K;
  const int b = blockIdx.x;
  const int r = b * K + i;
  // The search state (step, done, alive count, scores; prefix tables) was
  // last written by this kernel / the step advance of the previous step,
  // grids long completed: read it through L2 before the grid-dependency
  // wait, which only the logits (preceding output GEMM) need.
  const int t = __ldcg(st.step);
  const int nf = st.n_factors;
  const int G = (U + 31) >> 5;
  TP(0);
  const int done = __ldcg(st.done + b);
  const int nalive = __ldcg(st.n_alive + b);
  const int plen = __ldcg(st.prefix_len + b);
  const int mlen = __ldcg(st.max_len + b);
  const double s_row = i < nalive ? __ldcg(st.score + b * K + i) : 0.0;
  if (done) return;
  PDL_ENTRY();
  const bool final_force = (t == mlen - 1) && (t >= plen);
  const int fcol = t < plen ? st.prefix_col[(size_t)b * st.P + t] : (final_force ? st.eos_col : -1);

  if (i < nalive) {
    const float *row = logits + (size_t)r * ld;
    const unsigned *mask = st.mask ? st.mask + (size_t)b * ((U + 31) >> 5) : nullptr;
    const bool do_topk = fcol < 0;
    const bool need_argmax = final_force;
    const int kk = K < MAXK ? K : MAXK;
    const double s_r = s_row;
    const bool use_part = !lp_in && st.lse_part != nullptr;
    const bool staged = use_part && st.stage_partials;
    const float2 *gpart = use_part ? reinterpret_cast<const float2 *>(st.lse_part) + (size_t)r * st.lse_ld
                                   : nullptr;
    const float2 *part = staged ? part_s + (size_t)i * G : gpart;

    // ---- 1. statistics (and the K-th largest group maximum for pruning)
    TP(1);
    float mx = 0.f, lse = 0.f, T = -INFINITY;
    if (use_part) {
      if (staged) {  // stage the row's partials: 16-byte loads, all in flight
        const float4 *src = reinterpret_cast<const float4 *>(gpart);
        float4 *dst = reinterpret_cast<float4 *>(part_s + (size_t)i * G);
        const bool al = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
        const int n4 = al ? (G >> 1) : 0;
        if (!al)
          for (int g = s * 32 + lane; g < G; g += SW) part_s[(size_t)i * G + g] = gpart[g];
        for (int q0 = s * 32 + lane; q0 < n4; q0 += SW * 8) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (q0 + SW * u < n4) v[u] = __ldcs(src + q0 + SW * u);
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (q0 + SW * u < n4) dst[q0 + SW * u] = v[u];
        }
        if (al && (G & 1) && s == 0 && lane == 0) part_s[(size_t)i * G + G - 1] = gpart[G - 1];
        row_sync<SUB>(i);
      }
      TP(2);
      float gv[MAXK];
#pragma unroll
      for (int j = 0; j < MAXK; ++j) gv[j] = -INFINITY;
      float m = -INFINITY;
      for (int g = s * 32 + lane; g < G; g += SW) {
        const float v = part[g].x;
        m = fmaxf(m, v);
        if (v > gv[MAXK - 1]) vals_insert<MAXK>(gv, v);
      }
      m = unord32(__reduce_max_sync(0xffffffffu, ord32(m)));
      if (do_topk) warp_kth<MAXK>(gv, kk, &sm.rgv[i][s * MAXK]);
      if (lane == 0) sm.rm[i][s] = m;
      row_sync<SUB>(i);
      mx = sm.rm[i][0];
#pragma unroll
      for (int q = 1; q < SUB; ++q) mx = fmaxf(mx, sm.rm[i][q]);
      float sum = 0.f;
      for (int g = s * 32 + lane; g < G; g += SW) {
        const float2 p = part[g];
        if (p.x != -INFINITY) sum += p.y * expf(p.x - mx);
      }
      sum = warp_sum(sum);
      if (lane == 0) sm.rs[i][s] = sum;
      if (do_topk) {  // K-th largest of the warps' top group maxima
        float v1[1];
        v1[0] = lane < SUB * kk ? sm.rgv[i][(lane / kk) * MAXK + lane % kk] : -INFINITY;
        T = warp_kth<1>(v1, kk);
      }
      row_sync<SUB>(i);
      float tot = sm.rs[i][0];
#pragma unroll
      for (int q = 1; q < SUB; ++q) tot += sm.rs[i][q];
      lse = logf(tot);
    } else if (!lp_in) {
      float m = -INFINITY;
      for (int c = s * 32 + lane; c < U; c += SW)
        if (col_active(mask, c)) m = fmaxf(m, row[c]);
      m = unord32(__reduce_max_sync(0xffffffffu, ord32(m)));
      if (lane == 0) sm.rm[i][s] = m;
      row_sync<SUB>(i);
      mx = sm.rm[i][0];
#pragma unroll
      for (int q = 1; q < SUB; ++q) mx = fmaxf(mx, sm.rm[i][q]);
      float sum = 0.f;
      for (int c = s * 32 + lane; c < U; c += SW)
        if (col_active(mask, c)) sum += expf(row[c] - mx);
      sum = warp_sum(sum);
      if (lane == 0) sm.rs[i][s] = sum;
      row_sync<SUB>(i);
      float tot = sm.rs[i][0];
#pragma unroll
      for (int q = 1; q < SUB; ++q) tot += sm.rs[i][q];
      lse = logf(tot);
    }

    TP(3);
    // ---- 2./3. candidates -> per-lane top-K and first-max argmax
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
    if (use_part && st.prune && (do_topk || need_argmax)) {
      const float thr_top = do_topk ? (T == -INFINITY ? -INFINITY
                                       : T - (4e-6f * (fabsf(T) + fabsf(mx) + fabsf(lse) + 1.0f) +
                                              (float)(1e-15 * (fabs(s_r) + 1.0))))
                                    : INFINITY;
      const float thr_arg =
          need_argmax ? mx - 4e-6f * (2.0f * fabsf(mx) + fabsf(lse) + 1.0f) : INFINITY;
      const float thr = fminf(thr_top, thr_arg);
      // collect this warp's candidate groups in increasing order (ballot per
      // 32 groups)
      int *cg = sm.cg[i][s];
      int ncg = 0;
      bool overflow = false;
      for (int g0 = s * 32; g0 < G; g0 += SW) {
        const int g = g0 + lane;
        unsigned cand = __ballot_sync(0xffffffffu, g < G && part[g].x >= thr);
        const int n = __popc(cand);
        if (ncg + n > 64) {
          overflow = true;
          break;
        }
        if ((cand >> lane) & 1u) cg[ncg + __popc(cand & ((1u << lane) - 1u))] = g;
        ncg += n;
      }
      __syncwarp();
      if (!overflow) {
        // lane = column inside the group: one coalesced 128-byte segment per
        // group; 8 groups' loads in flight before visiting them in order
        for (int q0 = 0; q0 < ncg; q0 += 8) {
          float xv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = q0 + u < ncg ? (cg[q0 + u] << 5) + lane : U;
            xv[u] = c < U ? __ldcs(row + c) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = q0 + u < ncg ? (cg[q0 + u] << 5) + lane : U;
            if (c < U) visit(c, xv[u]);
          }
        }
      } else {
        for (int g0 = s * 32; g0 < G; g0 += SW) {
          const int g = g0 + lane;
          unsigned cand = __ballot_sync(0xffffffffu, g < G && part[g].x >= thr);
          while (cand) {
            const int c = ((g0 + __ffs(cand) - 1) << 5) + lane;
            cand &= cand - 1;
            if (c < U) visit(c, __ldcs(row + c));
          }
        }
      }
    } else if (do_topk || need_argmax) {
      const bool vec = (U & 3) == 0 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0;
      if (vec) {
        const float4 *row4 = reinterpret_cast<const float4 *>(row);
        for (int c4 = s * 32 + lane; c4 < (U >> 2); c4 += SW) {
          const float4 v = __ldcs(row4 + c4);
          const int c = 4 * c4;
          visit(c, v.x); visit(c + 1, v.y); visit(c + 2, v.z); visit(c + 3, v.w);
        }
      } else {
        for (int c = s * 32 + lane; c < U; c += SW) visit(c, row[c]);
      }
    }
    TP(4);
    // first max of lp across the warp (ties -> lowest column)
    warp_argmax(amax, acol);
    if (lane == 0) {
      sm.sav[i][s] = amax;
      sm.sac[i][s] = acol;
    }
    __syncwarp();
    if (do_topk) {  // this warp's top kk, best first
      int cnt = 0;
      for (int j = 0; j < kk; ++j) {
        const int bl = warp_best(tk[0], tc[0], tc[0] != INT_MAX);
        if (bl < 0) break;
        if (lane == bl) {
          sm.skey[i][s][j] = tk[0];
          sm.slp[i][s][j] = tl[0];
          sm.scol[i][s][j] = tc[0];
#pragma unroll
          for (int q = 0; q + 1 < MAXK; ++q) {
            tk[q] = tk[q + 1];
            tl[q] = tl[q + 1];
            tc[q] = tc[q + 1];
          }
          tk[MAXK - 1] = -DBL_MAX;
          tl[MAXK - 1] = -INFINITY;
          tc[MAXK - 1] = INT_MAX;
        }
        ++cnt;
      }
      if (lane == 0) sm.scnt[i][s] = cnt;
    }
    row_sync<SUB>(i);
    if (s == 0) {
      if (lane == 0) {  // first max over the warps, in column order
        float ba = sm.sav[i][0];
        int bcol = sm.sac[i][0];
#pragma unroll
        for (int q = 1; q < SUB; ++q) {
          const float a = sm.sav[i][q];
          const int c = sm.sac[i][q];
          if (a > ba || (a == ba && c < bcol)) {
            ba = a;
            bcol = c;
          }
        }
        sm.arg[i] = bcol;
      }
      TP(8);
      if (!do_topk) {
        if (lane == 0) {
          const float x = row[fcol];
          const float lp = lp_in ? x : (x - mx) - lse;
          // forced steps: float32 key fl32(fl32(s) + lp) (NEP 50 promotion)
          const float key32 = (float)s_r + lp;
          sm.key[i][0] = (double)key32;
          sm.lp[i][0] = lp;
          sm.col[i][0] = fcol;
          sm.cnt[i] = 1;
        }
      } else {
        // merge the SUB sorted warp lists (disjoint columns): kk rounds of a
        // warp argmax over the list heads held by lanes 0..SUB-1
        __syncwarp();  // reconverge after the lane-0 section (shuffles below)
        const int my_cnt = lane < SUB ? sm.scnt[i][lane] : 0;
        int head = 0, cnt = 0;
        for (int j = 0; j < kk; ++j) {
          const bool has = head < my_cnt;
          const int bq = warp_best(has ? sm.skey[i][lane][head] : 0.0, has ? sm.scol[i][lane][head] : 0, has);
          if (bq < 0) break;
          if (lane == bq) {
            sm.key[i][j] = sm.skey[i][lane][head];
            sm.lp[i][j] = sm.slp[i][lane][head];
            sm.col[i][j] = sm.scol[i][lane][head];
            ++head;
          }
          ++cnt;
        }
        if (lane == 0) sm.cnt[i] = cnt;
      }
      TP(9);
      // factor choices of this row (search.py:261-272): prefix override at
      // t - 1, else first-max of the factor logits
      for (int k = 0; k < nf; ++k) {
        int choice = -1;
        if (t >= 1 && st.prefix_fac && t - 1 < st.P)
          choice = st.prefix_fac[((size_t)b * nf + k) * st.P + t - 1];
        if (choice < 0) {
          const float *fr = st.fac_logits + (size_t)r * st.fac_ld;
          const int lo = st.fac_off[k], hi = st.fac_off[k + 1];
          float bm = -INFINITY;
          int bcol = INT_MAX;
          for (int c = lo + lane; c < hi; c += 32)
            if (fr[c] > bm) {
              bm = fr[c];
              bcol = c - lo;
            }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, bm, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bcol, o);
            if (om > bm || (om == bm && oc < bcol)) {
              bm = om;
              bcol = oc;
            }
          }
          choice = bcol == INT_MAX ? 0 : bcol;
        }
        if (lane == 0) st.fac_choice[(size_t)r * nf + k] = choice;
      }
    }
  }
  TP(5);
  __syncthreads();
  TP(6);
  if (w != 0) return;

  // ---- warp 0: merge the row lists.  K rounds of a warp argmax over the
  // row-list heads in the exact order (score desc, token asc, parent asc);
  // columns are sorted by token.
  const int base = b * K;
  const int my_cnt = lane < nalive ? sm.cnt[lane] : 0;
  const double my_s = lane < nalive ? st.score[base + lane] : 0.0;
  const int my_arg = lane < nalive ? sm.arg[lane] : 0;
  int head = 0;
  int npk = 0;
  int pick_q = 0, pick_c = 0;  // lane j keeps pick j
  float pick_lp = 0.f;
  for (int sel = 0; sel < K; ++sel) {
    const bool has = lane < nalive && head < my_cnt;
    const int bq = warp_best(has ? sm.key[lane][head] : 0.0, has ? sm.col[lane][head] : 0, has);
    if (bq < 0) break;
    const int bc = __shfl_sync(0xffffffffu, has ? sm.col[lane][head] : 0, bq);
    const float plp = __shfl_sync(0xffffffffu, has ? sm.lp[lane][head] : 0.f, bq);
    if (lane == sel) {
      pick_q = bq;
      pick_c = bc;
      pick_lp = plp;
    }
    if (lane == bq) ++head;
    npk = sel + 1;
  }
  // scores and tokens of the picks (lane j = pick j)
  const double pick_score = __shfl_sync(0xffffffffu, my_s, pick_q) + (double)pick_lp;
  const int pick_arg = __shfl_sync(0xffffffffu, my_arg, pick_q);
  const int pick_tok = (lane < npk) ? (st.col_token ? st.col_token[pick_c] : pick_c) : -1;
  const int steps = t + 1;
  const double pen = st.len_pen[steps];
  // survivors take new rows in rank order
  const unsigned surv = __ballot_sync(0xffffffffu, lane < npk && pick_tok != EOS);
  const int n_new = __popc(surv);
  if (lane < npk && pick_tok != EOS) {
    const int slot = base + __popc(surv & ((1u << lane) - 1u));
    const int rr = base + pick_q;
    st.tok_next[slot] = pick_tok;
    st.parent[slot] = rr;
    st.score[slot] = pick_score;
    st.tok_hist[(size_t)t * R + slot] = pick_tok;
    st.par_hist[(size_t)t * R + slot] = pick_q;
    for (int k = 0; k < nf; ++k) {
      const int f = st.fac_choice[(size_t)rr * nf + k];
      st.ftok_next[(size_t)k * R + slot] = f;
      st.fac_hist[((size_t)t * nf + k) * R + slot] = f;
    }
  }
  if (lane >= n_new && lane < K) {
    st.tok_next[base + lane] = PAD;
    st.parent[base + lane] = base;
    for (int k = 0; k < nf; ++k) st.ftok_next[(size_t)k * R + base + lane] = PAD;
  }
  // finished hypotheses in rank order: keep the first maximum of
  // logprob / steps^alpha (search.py:394)
  unsigned f = __ballot_sync(0xffffffffu, lane < npk && pick_tok == EOS);
  int best_steps = st.best_steps[b];
  double best_norm = st.best_norm[b];
  while (f) {
    const int j = __ffs(f) - 1;
    f &= f - 1;
    const double sc = __shfl_sync(0xffffffffu, pick_score, j);
    const int q = __shfl_sync(0xffffffffu, pick_q, j);
    const int c = __shfl_sync(0xffffffffu, pick_c, j);
    const int ar = __shfl_sync(0xffffffffu, pick_arg, j);
    const double norm = sc / pen;
    if (best_steps == 0 || norm > best_norm) {
      best_steps = steps;
      best_norm = norm;
      if (lane == 0) {
        st.best_norm[b] = norm;
        st.best_logprob[b] = sc;
        st.best_steps[b] = steps;
        st.best_forced[b] = final_force && ar != c;
        st.best_parent[b] = q;
        for (int k = 0; k < nf; ++k)
          st.best_fac[(size_t)b * nf + k] = st.fac_choice[(size_t)(base + q) * nf + k];
      }
    }
  }
  if (lane == 0) {
    st.n_alive[b] = n_new;
    if (n_new == 0) {
      st.done[b] = 1;
      atomicAdd(st.n_done, 1);
    }
  }
  TP(7);
}

// ------------------------------------------------------------- reorder
__global__ void k_beam_reorder(int R, int S_max, int *anc, const int *parent, const int *step) {
  PDL_ENTRY();
  const int r = blockIdx.y;
  const int t = *step;
  const int p = parent[r];
  const int *src = anc + ((size_t)(t & 1) * R + p) * S_max;
  int *dst = anc + ((size_t)((t + 1) & 1) * R + r) * S_max;
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos <= t && pos < S_max;
       pos += gridDim.x * blockDim.x)
    dst[pos] = pos == t ? p : src[pos];
}

__global__ void k_step_advance(int *step) {
  PDL_ENTRY(); *step += 1; }

// ------------------------------------------------------------ finalize
__global__ void k_beam_finalize(skb_beam_state st, int *tokens_out, int *factors_out) {
  PDL_ENTRY();
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
  cudaStream_t s = as_stream(stream);
  skb_beam_state sv = *st;
  // stage the fused partials in shared memory when K rows x G groups fit
  const int G = (sv.U + 31) / 32;
  const size_t part_bytes = (size_t)sv.K * G * sizeof(float2);
  sv.stage_partials = (sv.lse_part != nullptr && part_bytes <= 160 * 1024) ? 1 : 0;
  auto go = [&](auto kern_ptr, size_t base_smem, int threads) {
    const size_t smem = ((base_smem + 15) & ~size_t(15)) + (sv.stage_partials ? part_bytes : 0);
    if (smem > 48 * 1024) ensure_smem_fn(kern_ptr, smem);
    launch_k(kern_ptr, sv.B, threads, smem, s, logits, ld_logits, lp_in, sv);
  };
  // SUB warps per beam row (<= 1024 threads, register budget of the
  // per-lane MAXK lists)
  if (sv.K <= 1)
    go(k_beam_step<1, 8>, sizeof(BeamSmem<1, 8>), sv.K * 32 * 8);
  else if (sv.K <= 2)
    go(k_beam_step<2, 8>, sizeof(BeamSmem<2, 8>), sv.K * 32 * 8);
  else if (sv.K <= 4)
    go(k_beam_step<4, 4>, sizeof(BeamSmem<4, 4>), sv.K * 32 * 4);
  else if (sv.K <= 5)
    go(k_beam_step<5, SKB_BEAM_SUB5>, sizeof(BeamSmem<5, SKB_BEAM_SUB5>), sv.K * 32 * SKB_BEAM_SUB5);
  else if (sv.K <= 8)
    go(k_beam_step<8, 2>, sizeof(BeamSmem<8, 2>), sv.K * 32 * 2);
  else if (sv.K <= 16)
    go(k_beam_step<16, 1>, sizeof(BeamSmem<16, 1>), sv.K * 32);
  else
    go(k_beam_step<32, 1>, sizeof(BeamSmem<32, 1>), sv.K * 32);
  SKB_CHECK_LAUNCH("k_beam_step");
  return SKB_OK;
}

extern "C" int skb_debug_beam_prof(unsigned long long *host) {
#ifdef SKB_PROFILE_PHASES
  return cudaMemcpyFromSymbol(host, skb::g_tprof, sizeof(unsigned long long) * 4096 * 10) == cudaSuccess
             ? 0 : 3;
#else
  (void)host;
  return SKB_ERR_UNSUPPORTED;
#endif
}

extern "C" int skb_beam_reorder(int R, int S_max, int *anc, const int *parent, int *step,
                                void *stream) {
  if (R <= 0 || S_max <= 0) return fail(SKB_ERR_SHAPE, "beam_reorder: bad shape");
  cudaStream_t s = as_stream(stream);
  dim3 grid((S_max + 127) / 128, R);
  launch_k(k_beam_reorder, grid, 128, 0, s, R, S_max, anc, parent, step);
  SKB_CHECK_LAUNCH("k_beam_reorder");
  launch_k(k_step_advance, 1, 1, 0, s, step);
  SKB_CHECK_LAUNCH("k_step_advance");
  return SKB_OK;
}

extern "C" int skb_beam_finalize(const skb_beam_state *st, int *tokens_out, int *factors_out,
                                 void *stream) {
  if (!st || st->B <= 0) return fail(SKB_ERR_SHAPE, "beam_finalize: bad state");
  launch_k(k_beam_finalize, (st->B + 127) / 128, 128, 0, as_stream(stream), *st, tokens_out, factors_out);
  SKB_CHECK_LAUNCH("k_beam_finalize");
  return SKB_OK;
}
