// beam.cuh — S3 SelectExperts (Alg. 1) for ONE token by ONE thread.
//
// Alg. 1 per token: beam := [()]; for every grid dimension i: expand each prefix p of the beam
// by j in [0, M) with score s_p + g_i(x, j) (Eq. 2's additive score), drop the candidates whose
// prefix has no alive expert (FilterAlive; reading X5), keep the best B
// (k at the last level) under the total order of reading X4 (score descending, then flat index
// ascending; -0.0 == +0.0).
//
// B200 design: a thread owns a token.  Its row of gate scores sits in shared memory (staged by
// coalesced loads, or written there by the gate GEMM's epilogue), the beam and the level's
// running top-W list live in registers as 64-bit keys  (order-preserving score bits << 32) |
// (2^32 - 1 - flat prefix index)  so "larger key" == "higher score, then lower index", and each
// candidate costs one fp32 add and one fp32 compare against the list's current W-th score; only
// the rare candidates that reach the list pay the unrolled compare-select insertion.  No warp
// shuffles, no divergence-bound merge rounds: the search is a short ALU loop per token, so a
// 128-token tile of the gate GEMM finishes it in its own epilogue.
#pragma once
#include <math.h>
#include <stdint.h>

namespace dmoe {

__device__ __forceinline__ uint32_t beam_ord(float s) {
  uint32_t u = __float_as_uint(s == 0.0f ? 0.0f : s);  // canonicalise -0.0 (reading X4)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float beam_unord(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t beam_key(float s, uint32_t p) {
  return ((uint64_t)beam_ord(s) << 32) | (uint64_t)(0xffffffffu - p);
}

// keep `top` sorted descending; the smallest entry falls off
template <int WMAX>
__device__ __forceinline__ void beam_insert(uint64_t (&top)[WMAX], uint64_t key) {
#pragma unroll
  for (int i = WMAX - 1; i >= 0; --i) {
    const uint64_t prev = (i > 0) ? top[i - 1] : ~0ull;
    if (key > top[i]) top[i] = (key > prev) ? prev : key;
  }
}

template <int WMAX>
__device__ __forceinline__ uint64_t beam_at(const uint64_t (&top)[WMAX], int i) {
  uint64_t v = 0;
#pragma unroll
  for (int q = 0; q < WMAX; ++q)
    if (q == i) v = top[q];
  return v;
}

// One token.  grow: its d*M gate scores G[t, i*M + j] (any memory, stride `gstride` floats
// between consecutive j — 1 for a contiguous row).  PA: prefix-alive bitmaps, level i at word
// offset pa_off[i] (level d-1 = the alive mask); read only when MASKED.  Writes sel[0..k) and
// score[0..k) (flat expert index / Eq. 2 score sum, best first; -1 / -inf pad, reading X6).
template <int WMAX, bool MASKED>
__device__ __forceinline__ void beam_search_row(const float* grow, int gstride, int d, int M, int k, int B,
                                                const uint32_t* PA, const int (&pa_off)[4], int32_t* sel,
                                                float* score) {
  uint64_t beam[WMAX];
#pragma unroll
  for (int q = 0; q < WMAX; ++q) beam[q] = 0ull;
  beam[0] = beam_key(0.0f, 0u);  // the empty prefix, score 0
  int nb = 1;
  for (int i = 0; i < d; ++i) {
    const int W = (i < d - 1) ? B : k;
    uint64_t top[WMAX];
#pragma unroll
    for (int q = 0; q < WMAX; ++q) top[q] = 0ull;
    uint64_t thr = 0ull;        // key of the W-th entry (0: fewer than W so far)
    float thr_s = -INFINITY;    // its score: a candidate below it cannot enter the list
    const float* gi = grow + (int64_t)i * M * gstride;
    const uint32_t* pa = nullptr;
    if (MASKED) pa = PA + (i == 0 ? pa_off[0] : i == 1 ? pa_off[1] : i == 2 ? pa_off[2] : pa_off[3]);
    // candidate (score s, flat prefix p): FilterAlive, then the exact key test and insertion
    auto consider = [&](float s, uint32_t p) {
      if (!(s >= thr_s)) return;  // below the W-th score (also drops NaN, undefined by X4)
      if (MASKED && !((pa[p >> 5] >> (p & 31)) & 1u)) return;  // FilterAlive
      const uint64_t key = beam_key(s, p);
      if (key > thr) {
        beam_insert<WMAX>(top, key);
        thr = beam_at<WMAX>(top, W - 1);
        if (thr) thr_s = beam_unord((uint32_t)(thr >> 32));
      }
    };
    // All experts alive (no FilterAlive): the level's candidates are prefix score + g_i(j), and
    // rounding is monotone, so prefix b's best W are among the best W of g_i -- the list L
    // (key: g desc, j asc) -- unless the (W+1)-th of L reaches the W-th's rounded sum (then
    // a j outside L could tie it and win on the lower flat index: that prefix is scanned in
    // full).  The union of the prefixes' best W holds the level's best W.
    uint64_t L[WMAX + 1];
    int nL = 0;
    if (!MASKED) {
#pragma unroll
      for (int q = 0; q <= WMAX; ++q) L[q] = 0ull;
      uint64_t lthr = 0ull;
      float lthr_g = -INFINITY;
      for (int j = 0; j < M; ++j) {
        const float g = gi[j * gstride];
        if (!(g >= lthr_g)) continue;
        const uint64_t key = beam_key(g, (uint32_t)j);
        if (key > lthr) {
          beam_insert<WMAX + 1>(L, key);
          lthr = beam_at<WMAX + 1>(L, W);   // the (W+1)-th entry
          if (lthr) lthr_g = beam_unord((uint32_t)(lthr >> 32));
        }
      }
      nL = M < W + 1 ? M : W + 1;
    }
#pragma unroll
    for (int b = 0; b < WMAX; ++b) {
      if (b < nb) {
        const uint32_t p0 = (0xffffffffu - (uint32_t)beam[b]) * (uint32_t)M;
        const float sp = beam_unord((uint32_t)(beam[b] >> 32));
        if (!MASKED) {
          bool full = false;
          if (nL == W + 1) {  // M > W: is the W-th rounded sum strictly above the (W+1)-th?
            const float sW = sp + beam_unord((uint32_t)(beam_at<WMAX + 1>(L, W - 1) >> 32));
            const float sN = sp + beam_unord((uint32_t)(beam_at<WMAX + 1>(L, W) >> 32));
            full = !(sW > sN);
          }
          if (!full) {
            const int nq = nL < W ? nL : W;
#pragma unroll
            for (int q = 0; q < WMAX; ++q) {
              if (q < nq) {
                const uint32_t jq = 0xffffffffu - (uint32_t)L[q];
                consider(sp + beam_unord((uint32_t)(L[q] >> 32)), p0 + jq);
              }
            }
            continue;
          }
        }
        int j = 0;
        // 4 candidates per step: four independent loads and adds, one combined test; the
        // rare step with a candidate at or above the W-th score walks its four in order
        for (; j + 4 <= M; j += 4) {
          const float s0 = sp + gi[(j + 0) * gstride], s1 = sp + gi[(j + 1) * gstride];
          const float s2 = sp + gi[(j + 2) * gstride], s3 = sp + gi[(j + 3) * gstride];
          if (!(fmaxf(fmaxf(s0, s1), fmaxf(s2, s3)) >= thr_s)) continue;
          consider(s0, p0 + (uint32_t)j);
          consider(s1, p0 + (uint32_t)j + 1u);
          consider(s2, p0 + (uint32_t)j + 2u);
          consider(s3, p0 + (uint32_t)j + 3u);
        }
        for (; j < M; ++j) consider(sp + gi[j * gstride], p0 + (uint32_t)j);
      }
    }
    nb = 0;
#pragma unroll
    for (int q = 0; q < WMAX; ++q) {
      const bool keep = q < W && top[q] != 0ull;
      beam[q] = keep ? top[q] : 0ull;
      nb += keep ? 1 : 0;
    }
  }
  for (int s = 0; s < k; ++s) {
    const uint64_t v = beam_at<WMAX>(beam, s);
    sel[s] = s < nb ? (int32_t)(0xffffffffu - (uint32_t)v) : -1;
    score[s] = s < nb ? beam_unord((uint32_t)(v >> 32)) : -INFINITY;
  }
}

// ---- unmasked fast path, split into per-dimension lists + a merge --------------------------
// With every expert alive, Alg. 1's level-i candidates are prefix score + g_i(j), so the work per
// token splits into d independent per-dimension lists (run by different threads) and a short
// sequential merge:
//   list_i = the best W_i + 1 of g_i(0..M) under the key (g desc, j asc)   (W_i = B, k at the end)
//   level 0: the beam is list_0's first W_0 (0 + g is exact: the order is g's own)
//   level i: prefix b's best W are among list_i's first W unless the (W+1)-th reaches the W-th's
//            rounded sum (then a j outside the list could tie it and win on the lower index: that
//            prefix is scanned in full); the union over prefixes holds the level's best W.
// Running best-n set of (score, index) under the order of reading X4, for a thread's scan:
// unsorted, with the worst member tracked, so a candidate costs one compare against it and an
// accepted one a slot replacement plus an n-step min scan (not a sorted-list shift of 64-bit
// keys); sorted once at the end.  Empty slots are (-inf, 0xffffffff), worse than any real key.
template <int N>
struct TopSet {
  float v[N];
  uint32_t i[N];
  float mv;     // the worst member
  uint32_t mi;
  int mpos;
  int n;        // active slots (<= N)
  __device__ __forceinline__ static bool better(float a, uint32_t ai, float b, uint32_t bi) {
    return a > b || (a == b && ai < bi);
  }
  __device__ __forceinline__ void init(int n_) {
    n = n_;
#pragma unroll
    for (int q = 0; q < N; ++q) { v[q] = -INFINITY; i[q] = 0xffffffffu; }
    mv = -INFINITY; mi = 0xffffffffu; mpos = 0;
  }
  __device__ __forceinline__ void rescan() {
    mv = v[0]; mi = i[0]; mpos = 0;
#pragma unroll
    for (int q = 1; q < N; ++q)
      if (q < n && better(mv, mi, v[q], i[q])) { mv = v[q]; mi = i[q]; mpos = q; }
  }
  __device__ __forceinline__ void offer(float s, uint32_t idx) {
    if (!better(s, idx, mv, mi)) return;  // NaN never enters (undefined, reading X4)
#pragma unroll
    for (int q = 0; q < N; ++q)
      if (q == mpos) { v[q] = s; i[q] = idx; }
    rescan();
  }
  // sort descending by key (odd-even transposition network), empty slots last
  __device__ __forceinline__ void sort() {
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int q = r & 1; q + 1 < N; q += 2)
        if (better(v[q + 1], i[q + 1], v[q], i[q])) {
          const float tv = v[q]; v[q] = v[q + 1]; v[q + 1] = tv;
          const uint32_t ti = i[q]; i[q] = i[q + 1]; i[q + 1] = ti;
        }
  }
  __device__ __forceinline__ uint64_t key(int q) const {  // 0 for an empty slot
    return i[q] == 0xffffffffu ? 0ull : beam_key(v[q], i[q]);
  }
};

template <int N>
__device__ __forceinline__ uint64_t beam_at_key(const TopSet<N>& ts, int q) {
  uint64_t v = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (i == q) v = ts.key(i);
  return v;
}

template <int WMAX>
__device__ __forceinline__ void beam_dim_list(const float* gi, int gstride, int M, int n, uint64_t* out) {
  TopSet<WMAX + 1> L;
  L.init(n);
  int j = 0;
  for (; j + 4 <= M; j += 4) {
    const float g0 = gi[(j + 0) * gstride], g1 = gi[(j + 1) * gstride];
    const float g2 = gi[(j + 2) * gstride], g3 = gi[(j + 3) * gstride];
    if (!(fmaxf(fmaxf(g0, g1), fmaxf(g2, g3)) >= L.mv)) continue;
    L.offer(g0, j); L.offer(g1, j + 1); L.offer(g2, j + 2); L.offer(g3, j + 3);
  }
  for (; j < M; ++j) L.offer(gi[j * gstride], j);
  L.sort();
#pragma unroll
  for (int q = 0; q <= WMAX; ++q)
    if (q < n) out[q] = L.key(q);
}

// the merge of one token: lists [d][WMAX + 1] (beam_dim_list outputs, n_i = W_i + 1 entries,
// 0 = missing); grow / gstride: the token's G row (read only by prefixes scanned in full)
template <int WMAX>
__device__ __forceinline__ void beam_merge_row(const float* grow, int gstride, int d, int M, int k, int B,
                                               const uint64_t* lists, int32_t* sel, float* score) {
  uint64_t beam[WMAX];
  int nb = 0;
  {
    const int W0 = d > 1 ? B : k;
#pragma unroll
    for (int q = 0; q < WMAX; ++q) {
      const uint64_t v = q < W0 ? lists[q] : 0ull;
      beam[q] = v;
      nb += v ? 1 : 0;
    }
  }
  for (int i = 1; i < d; ++i) {
    const int W = (i < d - 1) ? B : k;
    const uint64_t* Li = lists + i * (WMAX + 1);
    const int nL = M < W + 1 ? M : W + 1;
    const float* gi = grow + (int64_t)i * M * gstride;
    TopSet<WMAX> top;
    top.init(W);
    auto consider = [&](float s, uint32_t p) { top.offer(s == 0.0f ? 0.0f : s, p); };
    const float gW = nL >= W ? beam_unord((uint32_t)(Li[W - 1] >> 32)) : 0.0f;
    const float gN = nL == W + 1 ? beam_unord((uint32_t)(Li[W] >> 32)) : 0.0f;
#pragma unroll
    for (int b = 0; b < WMAX; ++b) {
      if (b < nb) {
        const uint32_t p0 = (0xffffffffu - (uint32_t)beam[b]) * (uint32_t)M;
        const float sp = beam_unord((uint32_t)(beam[b] >> 32));
        if (nL == W + 1 && !(sp + gW > sp + gN)) {  // rounding may let a j outside the list tie
          for (int j = 0; j < M; ++j) consider(sp + gi[j * gstride], p0 + (uint32_t)j);
        } else {
          const int nq = nL < W ? nL : W;
          for (int q = 0; q < nq; ++q) {
            const uint64_t v = Li[q];
            consider(sp + beam_unord((uint32_t)(v >> 32)), p0 + (0xffffffffu - (uint32_t)v));
          }
        }
      }
    }
    top.sort();
    nb = 0;
#pragma unroll
    for (int q = 0; q < WMAX; ++q) {
      const uint64_t kq = q < W ? top.key(q) : 0ull;
      beam[q] = kq;
      nb += kq ? 1 : 0;
    }
  }
  for (int s = 0; s < k; ++s) {
    const uint64_t v = beam_at<WMAX>(beam, s);
    sel[s] = s < nb ? (int32_t)(0xffffffffu - (uint32_t)v) : -1;
    score[s] = s < nb ? beam_unord((uint32_t)(v >> 32)) : -INFINITY;
  }
}

// any alive expert in [e0, e0 + span)
__device__ __forceinline__ bool span_any(const uint32_t* __restrict__ alive, int64_t e0, int64_t span) {
  const int64_t e1 = e0 + span;
  for (int64_t e = e0; e < e1;) {
    const uint32_t word = alive[e >> 5];
    const int sh = (int)(e & 31);
    int64_t take = 32 - sh;
    if (take > e1 - e) take = e1 - e;
    const uint32_t mask = (take == 32) ? 0xffffffffu : (((1u << take) - 1u) << sh);
    if (word & mask) return true;
    e += take;
  }
  return false;
}

// prefix bitmaps into `PA` (smem or global) by the whole CTA, one thread per prefix and a
// warp ballot per 32-bit word; the last level is the alive mask itself.  Same definition as
// k_prefix_alive (reading X5).
__device__ __forceinline__ void prefix_alive_block(const uint32_t* __restrict__ alive, int d, int M, int64_t E, uint32_t* PA) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t wo = 0, n = M;
  for (int i = 0; i < d; ++i) {
    const int64_t words = (n + 31) / 32, span = E / n;
    if (i == d - 1) {
      for (int64_t w = threadIdx.x; w < words; w += blockDim.x) PA[wo + w] = alive[w];
    } else {
      for (int64_t w = warp; w < words; w += nw) {
        const int64_t p = w * 32 + lane;
        const bool any = p < n && span_any(alive, p * span, span);
        const uint32_t bits = __ballot_sync(0xffffffffu, any);
        if (lane == 0) PA[wo + w] = bits;
      }
    }
    wo += words;
    n *= M;
  }
}

}  // namespace dmoe
