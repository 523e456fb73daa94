// exchange.cu — receive-side layout of the expert-parallel all-to-all (S11).
//
// The paper sends each token to the workers that own its selected experts and collects the
// outputs (§3.1; the runtime batches requests per expert).  On a
// B200 box the experts are sharded by contiguous flat index over G ranks, and one NCCL
// all-to-all moves the dispatched rows (already grouped by owner rank, dmoe_dispatch).
// A rank receives rows source-rank-major: [src 0: its experts' segments][src 1: ...].
// These kernels build the expert-major layout (expert e's rows from source 0, then source
// 1, ...).  Because every source holds a contiguous, increasing block of tokens, that is
// exactly the 1-GPU segment order (increasing global token, reading X18), so the grouped
// expert GEMMs produce results bitwise equal to the single-GPU run.
#include "common.cuh"

namespace dmoe {

__device__ int32_t xblock_excl_scan(int32_t v, int32_t* sh, int32_t* total) {
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
    int32_t t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sh[lane] = t;
  }
  __syncthreads();
  const int32_t base = warp > 0 ? sh[warp - 1] : 0;
  *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

// one CTA: counts[s][e] (G x El) -> src_off[s][e] (source-major exclusive scan),
// offsets[e] (expert-major segment starts, El+1) and dst_off[s][e] = offsets[e] +
// sum_{s'<s} counts[s'][e]
__global__ void __launch_bounds__(1024)
k_exchange_tables(const int32_t* __restrict__ counts, int G, int El, int64_t R_cap, int32_t* __restrict__ offsets,
                  int32_t* __restrict__ src_off, int32_t* __restrict__ dst_off) {
  DMOE_PDL_ENTRY();
  __shared__ int32_t sh[32];
  int32_t carry = 0, tot;
  for (int i0 = 0; i0 < G * El; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const int32_t v = i < G * El ? counts[i] : 0;
    const int32_t ex = xblock_excl_scan(v, sh, &tot);
    if (i < G * El) src_off[i] = carry + ex;
    carry += tot;
  }
  carry = 0;
  for (int e0 = 0; e0 < El; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    int32_t v = 0;
    if (e < El)
      for (int s = 0; s < G; ++s) v += counts[s * El + e];
    const int32_t ex = xblock_excl_scan(v, sh, &tot);
    if (e < El) {
      int32_t d = carry + ex;
      // capacity clamp: segments never extend past R_cap (offsets[El] < sum(counts) reports it)
      offsets[e] = (int64_t)d < R_cap ? d : (int32_t)R_cap;
      for (int s = 0; s < G; ++s) { dst_off[s * El + e] = d; d += counts[s * El + e]; }
    }
    carry += tot;
  }
  if (threadIdx.x == 0) offsets[El] = (int64_t)carry < R_cap ? carry : (int32_t)R_cap;
}

// src_of_dst[r] for every expert-major row r < offsets[El] (<= R_cap): expert by binary search
// over offsets, source by a scan over the <= G blocks of that expert
__global__ void k_exchange_index(const int32_t* __restrict__ counts, int G, int El,
                                 const int32_t* __restrict__ offsets, const int32_t* __restrict__ src_off,
                                 const int32_t* __restrict__ dst_off, int32_t* __restrict__ src_of_dst) {
  DMOE_PDL_ENTRY();
  const int32_t R = offsets[El];
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    int lo = 0, hi = El;
    while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (offsets[mid] <= r) lo = mid; else hi = mid; }
    const int e = lo;
    int s = 0;
    while (s + 1 < G && r >= dst_off[s * El + e] + counts[s * El + e]) ++s;
    src_of_dst[r] = src_off[s * El + e] + (r - dst_off[s * El + e]);
  }
}

// gather (inverse = 0): dst[r] = src[idx[r]];  scatter (inverse = 1): dst[idx[r]] = src[r]
// for r < *n_rows (device count), rows of D elements, 16-byte vectors
template <typename T>
__global__ void k_permute_rows(const T* __restrict__ src, const int32_t* __restrict__ idx,
                               const int32_t* __restrict__ n_rows, int32_t D, int inverse,
                               T* __restrict__ dst) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N;
  const int64_t R = *n_rows;
  const int vecs = D / V;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R * vecs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / vecs;
    const int v = (int)(i - r * vecs);
    const int64_t a = inverse ? r : idx[r], b = inverse ? idx[r] : r;
    st_v4(dst + b * D + (int64_t)v * V, ld_nc_v4(src + a * D + (int64_t)v * V));
  }
}

dmoe_status exchange_layout(const int32_t* counts, int G, int El, int32_t* offsets,
                            int32_t* src_of_dst, int64_t R_cap, void* ws, size_t ws_bytes, cudaStream_t s) {
  Carver cv(ws, ws_bytes);
  int32_t* src_off = cv.take<int32_t>((size_t)G * El);
  int32_t* dst_off = cv.take<int32_t>((size_t)G * El);
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "exchange_layout: workspace too small");
  launch_pdl(k_exchange_tables, 1, 1024, 0, s, counts, G, El, R_cap, offsets, src_off, dst_off);
  DMOE_TRY(check_launch("exchange_tables"));
  int64_t blocks = ceil_div(R_cap > 0 ? R_cap : 1, 256);
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  launch_pdl(k_exchange_index, (unsigned)blocks, 256, 0, s, counts, G, El, offsets, src_off, dst_off, src_of_dst);
  return check_launch("exchange_index");
}

dmoe_status permute_rows(const void* src, const int32_t* idx, const int32_t* n_rows, int32_t D,
                         dmoe_dtype dt, int inverse, void* dst, cudaStream_t s) {
  const int grid = num_sms() * 8;
  if (dt == DMOE_BF16)
    launch_pdl(k_permute_rows<__nv_bfloat16>, grid, 256, 0, s, (const __nv_bfloat16*)src, idx, n_rows, D, inverse,
                                                      (__nv_bfloat16*)dst);
  else
    launch_pdl(k_permute_rows<float>, grid, 256, 0, s, (const float*)src, idx, n_rows, D, inverse, (float*)dst);
  return check_launch("permute_rows");
}

}  // namespace dmoe
