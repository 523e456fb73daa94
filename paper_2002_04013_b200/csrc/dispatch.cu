// dispatch.cu — S4 renormalised Eq. 3 weights + S5 stable counting-sort dispatch.
//
// PAPER.md:283-287 (Eq. 3, exclusion + renormalisation, batch drop) and PAPER.md:194,
// 327 (send inputs to the chosen experts; per-expert batching).  Deterministic
// without any ordering atomics:
//   1. k_weights_hist  — one warp per chunk of kChunkTok tokens: lane = token computes
//      ok / w / valid; ok pairs are counted into the chunk's private histogram row
//      hist[c][e] (integer atomics on a warp-private row: order-independent).
//   2. k_scan_chunks   — per expert, exclusive prefix over chunks (in place) -> counts[e]
//      (8-expert column blocks staged in shared memory: sector-coalesced both ways).
//   3. k_scan_experts  — one CTA: offsets = exclusive scan of counts, n_dropped, and the
//      grouped-GEMM tile plans (tiles of 128 and 64 rows per expert).
//   4. k_rank          — each warp re-walks its chunk 32 pairs at a time in pair order
//      t*k+s; __match_any_sync groups equal experts, rank = #earlier equal lanes +
//      running per-(chunk, expert) base.  Experts are distinct within a token, so pair
//      order == token order inside a segment (reading X18).
//   5. k_scatter       — xd[row_of_slot[t, s]] = x[t], token-parallel: x read once.
#include "common.cuh"

namespace dmoe {

constexpr int kDispWarps = 4;   // warps per CTA

// tokens per chunk (one warp per chunk): small enough for >= ~16 warps per SM on the
// rank/histogram passes, large enough that the per-chunk histograms stay <= 4M ints.
int64_t chunk_tokens(int64_t T, int64_t E) {
  int64_t nc = ceil_div(T, 16);
  const int64_t cap = (int64_t)(4 << 20) / (E > 0 ? E : 1);
  if (nc > cap) nc = cap;
  if (nc < 1) nc = 1;
  return ceil_div(T > 0 ? T : 1, nc);
}

__global__ void __launch_bounds__(kDispWarps * 32)
k_weights_hist(const int32_t* __restrict__ sel, const float* __restrict__ sel_score,
               const uint32_t* __restrict__ responded, int64_t T, int k, int64_t E,
               float* __restrict__ w, uint8_t* __restrict__ valid, int32_t* __restrict__ hist,
               int32_t* __restrict__ chunk_dropped, int64_t n_chunks, int64_t kChunkTok) {
  DMOE_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x * (int64_t)kDispWarps + (threadIdx.x >> 5);
  if (c >= n_chunks) return;
  int32_t* h = hist + c * E;
  for (int64_t e = lane; e < E; e += 32) h[e] = 0;
  __syncwarp();
  int dropped = 0;
  for (int64_t t0 = c * kChunkTok; t0 < (c + 1) * kChunkTok && t0 < T; t0 += 32) {
    const int64_t t = t0 + lane;
    if (t < T && t < (c + 1) * kChunkTok) {
      float m = -INFINITY;
      bool any = false;
      for (int s = 0; s < k; ++s) {
        int32_t e = sel[t * k + s];
        bool ok = e >= 0 && ((responded[e >> 5] >> (e & 31)) & 1u);
        if (ok) {
          any = true;
          m = fmaxf(m, sel_score[t * k + s]);
          atomicAdd(&h[e], 1);
        }
      }
      float z = 0.0f;
      for (int s = 0; s < k; ++s) {
        int32_t e = sel[t * k + s];
        bool ok = e >= 0 && ((responded[e >> 5] >> (e & 31)) & 1u);
        if (ok) z += __expf(sel_score[t * k + s] - m);
      }
      const float inv = any ? 1.0f / z : 0.0f;
      for (int s = 0; s < k; ++s) {
        int32_t e = sel[t * k + s];
        bool ok = e >= 0 && ((responded[e >> 5] >> (e & 31)) & 1u);
        w[t * k + s] = ok ? __expf(sel_score[t * k + s] - m) * inv : 0.0f;
      }
      valid[t] = any ? 1 : 0;
      dropped += any ? 0 : 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) dropped += __shfl_xor_sync(0xffffffffu, dropped, o);
  if (lane == 0) chunk_dropped[c] = dropped;
}

// per expert: exclusive prefix of hist[:, e] over chunks (in place) -> counts[e].  A CTA owns
// 8 consecutive experts and loads their columns for up to kScanBlk chunks into shared memory in
// one go (8 experts = one 32-byte sector per chunk row, every load in flight at once), warp w
// scans expert w along the chunks, and the block is written back the same way.
constexpr int kScanBlk = 1024;
__global__ void __launch_bounds__(256)
k_scan_chunks(int32_t* __restrict__ hist, int64_t n_chunks, int64_t E, int32_t* __restrict__ counts) {
  DMOE_PDL_ENTRY();
  __shared__ int32_t tile[kScanBlk][9];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t e0 = (int64_t)blockIdx.x * 8;
  int32_t carry = 0;  // warp w: expert e0 + w
  for (int64_t cb = 0; cb < n_chunks; cb += kScanBlk) {
    const int nb = (int)((n_chunks - cb) < kScanBlk ? (n_chunks - cb) : kScanBlk);
    for (int i = tid; i < nb * 8; i += 256) {
      const int cc = i >> 3, el = i & 7;
      tile[cc][el] = (e0 + el < E) ? hist[(cb + cc) * E + e0 + el] : 0;
    }
    __syncthreads();
    for (int c0 = 0; c0 < nb; c0 += 32) {
      const int cc = c0 + lane;
      const int32_t v = cc < nb ? tile[cc][w] : 0;
      int32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (cc < nb) tile[cc][w] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    __syncthreads();
    for (int i = tid; i < nb * 8; i += 256) {
      const int cc = i >> 3, el = i & 7;
      if (e0 + el < E) hist[(cb + cc) * E + e0 + el] = tile[cc][el];
    }
    __syncthreads();
  }
  if (lane == 0 && e0 + w < E) counts[e0 + w] = carry;
}

// block-wide exclusive scan helper (1024 threads), returns exclusive prefix and total
__device__ int32_t block_excl_scan(int32_t v, int32_t* sh, int32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  int32_t base = warp > 0 ? sh[warp - 1] : 0;
  *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

// offsets[e] = sum_{e'<e} counts[e'];  plan128/plan64[e] = sum_{e'<e} ceil(counts/128|64)
// (plans have E+1 entries).  Also folds chunk_dropped into n_dropped.
__global__ void __launch_bounds__(1024)
k_scan_experts(const int32_t* __restrict__ counts, int64_t E, int32_t* __restrict__ offsets,
               int32_t* __restrict__ plan128, int32_t* __restrict__ plan64,
               const int32_t* __restrict__ chunk_dropped, int64_t n_chunks,
               int32_t* __restrict__ n_dropped) {
  DMOE_PDL_ENTRY();
  __shared__ int32_t sh[32];
  int32_t carry = 0, carry128 = 0, carry64 = 0;
  for (int64_t e0 = 0; e0 < E; e0 += blockDim.x) {
    int64_t e = e0 + threadIdx.x;
    int32_t v = e < E ? counts[e] : 0;
    int32_t tot;
    int32_t ex = block_excl_scan(v, sh, &tot);
    if (e < E) offsets[e] = carry + ex;
    carry += tot;
    if (plan128) {
      int32_t v1 = (v + 127) / 128;
      int32_t ex1 = block_excl_scan(v1, sh, &tot);
      if (e < E) plan128[e] = carry128 + ex1;
      carry128 += tot;
      int32_t v2 = (v + 63) / 64;
      int32_t ex2 = block_excl_scan(v2, sh, &tot);
      if (e < E) plan64[e] = carry64 + ex2;
      carry64 += tot;
    }
  }
  if (threadIdx.x == 0) {
    offsets[E] = carry;
    if (plan128) { plan128[E] = carry128; plan64[E] = carry64; }
  }
  if (n_dropped) {
    int32_t d = 0;
    for (int64_t c = threadIdx.x; c < n_chunks; c += blockDim.x) d += chunk_dropped[c];
    int32_t tot;
    block_excl_scan(d, sh, &tot);
    if (threadIdx.x == 0) *n_dropped = tot;
  }
}

__global__ void __launch_bounds__(kDispWarps * 32)
k_rank(const int32_t* __restrict__ sel, const uint32_t* __restrict__ responded, int64_t T, int k,
       int64_t E, int32_t* __restrict__ hist, const int32_t* __restrict__ offsets,
       int32_t* __restrict__ row_of_slot, int32_t* __restrict__ token_of_row, int64_t n_chunks,
       int64_t kChunkTok) {
  DMOE_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x * (int64_t)kDispWarps + (threadIdx.x >> 5);
  if (c >= n_chunks) return;
  int32_t* base = hist + c * E;
  const int64_t q0 = c * kChunkTok * (int64_t)k;
  int64_t q1 = (c + 1) * kChunkTok * (int64_t)k;
  if (q1 > T * k) q1 = T * k;
  const uint32_t lt = (1u << lane) - 1u;
  for (int64_t qb = q0; qb < q1; qb += 32) {
    const int64_t q = qb + lane;
    int32_t e = -1;
    if (q < q1) {
      e = sel[q];
      if (e >= 0 && !((responded[e >> 5] >> (e & 31)) & 1u)) e = -1;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    int32_t b = 0;
    if (e >= 0 && lane == leader) b = base[e];
    b = __shfl_sync(0xffffffffu, b, leader);
    if (e >= 0) {
      const int32_t r = offsets[e] + b + __popc(peers & lt);
      row_of_slot[q] = r;
      token_of_row[r] = (int32_t)(q / k);
      if (lane == leader) base[e] = b + __popc(peers);
    } else if (q < q1) {
      row_of_slot[q] = -1;
    }
    __syncwarp();
  }
}

// xd[row_of_slot[t, s]] = x[t] for every ok slot: token-parallel (a warp per token), so each
// x row is read from HBM once and written to its <= k dispatched rows (a row-parallel gather
// re-reads it once per row); UNR 16-byte vectors per lane in flight before the stores.
template <typename T>
__global__ void __launch_bounds__(256)
k_scatter(const T* __restrict__ x, const int32_t* __restrict__ row_of_slot, int64_t Tn, int k, int32_t D,
          T* __restrict__ xd) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N, UNR = 4;
  const int lane = threadIdx.x & 31;
  const int vecs = D / V;  // D % V == 0 checked by the caller
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < Tn;
       t += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int32_t* ros = row_of_slot + t * k;
    for (int v0 = lane; v0 < vecs; v0 += UNR * 32) {
      uint4 u[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q)
        if (v0 + q * 32 < vecs) u[q] = ld_nc_v4(x + t * D + (int64_t)(v0 + q * 32) * V);
      for (int s = 0; s < k; ++s) {
        const int32_t r = ros[s];
        if (r < 0) continue;
#pragma unroll
        for (int q = 0; q < UNR; ++q)
          if (v0 + q * 32 < vecs) st_v4(xd + (int64_t)r * D + (int64_t)(v0 + q * 32) * V, u[q]);
      }
    }
  }
}

size_t dispatch_ws_bytes(int64_t T, int64_t E) {
  int64_t nc = ceil_div(T, chunk_tokens(T, E));
  return align_up((size_t)nc * E * 4, 256) + align_up((size_t)nc * 4, 256) + 1024;
}

dmoe_status dispatch(const void* x, dmoe_dtype dt, int64_t T, int32_t D, int64_t E, int32_t k,
                     const int32_t* sel, const float* sel_score, const uint32_t* responded,
                     float* w, uint8_t* valid, int32_t* n_dropped, int32_t* counts,
                     int32_t* offsets, int32_t* row_of_slot, int32_t* token_of_row, void* xd,
                     int32_t* plan128, int32_t* plan64, void* ws, size_t ws_bytes,
                     cudaStream_t s) {
  const int64_t kChunkTok = chunk_tokens(T, E);
  const int64_t nc = ceil_div(T, kChunkTok);
  Carver cv(ws, ws_bytes);
  int32_t* hist = cv.take<int32_t>((size_t)(nc > 0 ? nc : 1) * E);
  int32_t* cdrop = cv.take<int32_t>((size_t)(nc > 0 ? nc : 1));
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "dispatch: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  const unsigned blocks = (unsigned)ceil_div(nc, kDispWarps);
  if (nc > 0) {
    launch_pdl(k_weights_hist, blocks, kDispWarps * 32, 0, s, sel, sel_score, responded, T, k, E, w, valid,
                                                       hist, cdrop, nc, kChunkTok);
    DMOE_TRY(check_launch("dispatch.weights_hist"));
  }
  launch_pdl(k_scan_chunks, (unsigned)ceil_div(E, 8), 256, 0, s, hist, nc, E, counts);
  DMOE_TRY(check_launch("dispatch.scan_chunks"));
  launch_pdl(k_scan_experts, 1, 1024, 0, s, counts, E, offsets, plan128, plan64, cdrop, nc, n_dropped);
  DMOE_TRY(check_launch("dispatch.scan_experts"));
  if (nc > 0) {
    launch_pdl(k_rank, blocks, kDispWarps * 32, 0, s, sel, responded, T, k, E, hist, offsets, row_of_slot,
                                              token_of_row, nc, kChunkTok);
    DMOE_TRY(check_launch("dispatch.rank"));
    if (xd == nullptr) return DMOE_OK;  // gather fused into the peer exchange
    int64_t grid = ceil_div(T, 8);
    if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
    if (dt == DMOE_BF16)
      launch_pdl(k_scatter<__nv_bfloat16>, (unsigned)grid, 256, 0, s, (const __nv_bfloat16*)x, row_of_slot, T, k, D,
                 (__nv_bfloat16*)xd);
    else
      launch_pdl(k_scatter<float>, (unsigned)grid, 256, 0, s, (const float*)x, row_of_slot, T, k, D, (float*)xd);
    DMOE_TRY(check_launch("dispatch.scatter"));
  }
  return DMOE_OK;
}

// tile plan for a grouped GEMM over given offsets (used when the caller's offsets did not
// come from dmoe_dispatch in this process, e.g. after an all-to-all): plan[e] =
// sum_{e'<e} ceil((offsets[e'+1]-offsets[e'])/bm)
__global__ void __launch_bounds__(1024)
k_tile_plan(const int32_t* __restrict__ offsets, int64_t E, int bm, int32_t* __restrict__ plan) {
  DMOE_PDL_ENTRY();
  __shared__ int32_t sh[32];
  int32_t carry = 0;
  for (int64_t e0 = 0; e0 < E; e0 += blockDim.x) {
    int64_t e = e0 + threadIdx.x;
    int32_t v = e < E ? (offsets[e + 1] - offsets[e] + bm - 1) / bm : 0;
    int32_t tot;
    int32_t ex = block_excl_scan(v, sh, &tot);
    if (e < E) plan[e] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) plan[E] = carry;
}

dmoe_status tile_plan(const int32_t* offsets, int64_t E, int bm, int32_t* plan, cudaStream_t s) {
  launch_pdl(k_tile_plan, 1, 1024, 0, s, offsets, E, bm, plan);
  return check_launch("tile_plan");
}

}  // namespace dmoe

namespace dmoe {
// seg[s] = offsets[s * group], s = 0..E/group (reading X20: the tied-weight pool's slot segments)
__global__ void k_segment_offsets(const int32_t* __restrict__ offsets, int64_t n, int group,
                                  int32_t* __restrict__ seg) {
  DMOE_PDL_ENTRY();
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= n; s += (int64_t)gridDim.x * blockDim.x)
    seg[s] = offsets[s * group];
}

dmoe_status segment_offsets(const int32_t* offsets, int64_t E, int group, int32_t* seg, cudaStream_t s) {
  const int64_t n = E / group;
  int64_t blocks = ceil_div(n + 1, 256);
  if (blocks > 1024) blocks = 1024;
  launch_pdl(k_segment_offsets, (unsigned)blocks, 256, 0, s, offsets, n, group, seg);
  return check_launch("segment_offsets");
}
}  // namespace dmoe
