// gate_bwd.cu — S10: undispatch (sum the expert-path input gradients back per token)
// and the gating gradient of Eq. 2 through the Eq. 3 softmax.
//
//   dG[t, i*M + u_i(sel_ts)] += dscore_ts            (sparse: <= k*d non-zeros per row)
//   dX_t  = sum_{ok s} dXd[row_ts] + sum_s dscore_ts sum_i W_g[:, i*M + u_i(sel_ts)]
//   dW_g  = X^T dG (fp32),  db_g = column sums of dG (fp32)
//
// W_g is transposed once into the workspace so the k*d gate columns a token touches are
// contiguous rows (coalesced, L2-resident).  dW_g is a split-K SIMT reduction over
// tokens with a fixed-order final sum (deterministic, no float atomics).
#include "common.cuh"

namespace dmoe {

template <typename T>
__global__ void k_transpose(const T* __restrict__ src, int64_t rows, int64_t cols,
                            T* __restrict__ dst) {
  DMOE_PDL_ENTRY();
  __shared__ float tile[32][33];
  const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = Elem<T>::load(src + r * cols + c);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) Elem<T>::store(dst + c * rows + r, tile[threadIdx.x][i]);
  }
}

dmoe_status transpose(const void* src, int64_t rows, int64_t cols, dmoe_dtype dt, void* dst,
                      cudaStream_t s) {
  dim3 tb(32, 8), tg((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  if (dt == DMOE_BF16)
    launch_pdl(k_transpose<__nv_bfloat16>, tg, tb, 0, s, (const __nv_bfloat16*)src, rows, cols, (__nv_bfloat16*)dst);
  else
    launch_pdl(k_transpose<float>, tg, tb, 0, s, (const float*)src, rows, cols, (float*)dst);
  return check_launch("transpose");
}

constexpr int kGbWarps = 4;

template <typename T, int kGbMaxK>
__global__ void __launch_bounds__(kGbWarps * 32)
k_gate_bwd_dx(const T* __restrict__ WgT, const int32_t* __restrict__ sel,
              const float* __restrict__ dscore, const T* __restrict__ dxd,
              const int32_t* __restrict__ row_of_slot, int64_t Tn, int32_t D, int d, int M, int k,
              T* __restrict__ dx, float* __restrict__ dG) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  const int dM = d * M;
  for (int64_t t = blockIdx.x * (int64_t)kGbWarps + (threadIdx.x >> 5); t < Tn;
       t += (int64_t)gridDim.x * kGbWarps) {
    int32_t rows[kGbMaxK], es[kGbMaxK];
    float ds[kGbMaxK];
#pragma unroll
    for (int s = 0; s < kGbMaxK; ++s) {
      rows[s] = s < k ? row_of_slot[t * k + s] : -1;
      es[s] = s < k ? sel[t * k + s] : -1;
      ds[s] = s < k ? dscore[t * k + s] : 0.0f;
    }
    // dense dG row (fp32) for dW_g / db_g
    for (int col = lane; col < dM; col += 32) {
      const int i = col / M, j = col - i * M;
      int div = 1;
      for (int q = i + 1; q < d; ++q) div *= M;
      float v = 0.0f;
#pragma unroll
      for (int s = 0; s < kGbMaxK; ++s)
        if (s < k && es[s] >= 0 && (es[s] / div) % M == j) v += ds[s];
      dG[t * dM + col] = v;
    }
    for (int c = lane * V; c < D; c += 32 * V) {
      float acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = 0.0f;
      {
        uint4 u[kGbMaxK];
#pragma unroll
        for (int s = 0; s < kGbMaxK; ++s)
          if (s < k && rows[s] >= 0) u[s] = ld_nc_v4(dxd + (int64_t)rows[s] * D + c);
#pragma unroll
        for (int s = 0; s < kGbMaxK; ++s) {
          if (s >= k || rows[s] < 0) continue;
          float f[V];
          unpack16(u[s], f, (const T*)nullptr);
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] += f[q];
        }
      }
#pragma unroll
      for (int s = 0; s < kGbMaxK; ++s) {
        if (s >= k || es[s] < 0 || ds[s] == 0.0f) continue;
        int e = es[s];
        for (int i = d - 1; i >= 0; --i) {
          const int col = i * M + (e % M);
          e /= M;
          float f[V];
          unpack16(ld_v4(WgT + (int64_t)col * D + c), f, (const T*)nullptr);
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = fmaf(ds[s], f[q], acc[q]);
        }
      }
      st_v4(dx + t * D + c, pack16(acc, (const T*)nullptr));
    }
  }
}

// partial[split][c][col] = sum_{t in split} X[t][c] dG[t][col]; pb[split][col] = sum dG[t][col]
// Tile: 128 columns of X (c) x 32 columns of dG (col) per CTA, 32 tokens per smem pass; thread
// (tc, tg) owns c = 4 tc .. 4 tc + 3 and col = 4 tg .. 4 tg + 3 (16 fp32 accumulators, two
// 16-byte shared loads per 16 FMAs), summing tokens in order.
constexpr int kDwgC = 128, kDwgCol = 32, kDwgTok = 32;
template <typename T>
__global__ void __launch_bounds__(256)
k_dwg_partial(const T* __restrict__ X, const float* __restrict__ dG, int64_t Tn, int32_t D, int dM,
              int64_t tok_per_split, float* __restrict__ partial, float* __restrict__ pb) {
  DMOE_PDL_ENTRY();
  __shared__ __align__(16) float xs[kDwgTok][kDwgC];
  __shared__ __align__(16) float gs[kDwgTok][kDwgCol];
  constexpr int V = Vec16<T>::N;
  const int tc = threadIdx.x & 31, tg = threadIdx.x >> 5;  // 32 x 8
  const int c0 = blockIdx.x * kDwgC, col0 = blockIdx.y * kDwgCol;
  const int64_t split = blockIdx.z;
  const int64_t t_begin = split * tok_per_split;
  int64_t t_end = t_begin + tok_per_split;
  if (t_end > Tn) t_end = Tn;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  const bool xvec = (c0 + kDwgC <= D);
  const bool gvec = (col0 + kDwgCol <= dM) && (dM % 4 == 0);
  for (int64_t tb = t_begin; tb < t_end; tb += kDwgTok) {
    // X tile: 32 tokens x 128 columns (fp32 in smem)
    for (int i = threadIdx.x; i < kDwgTok * (kDwgC / V); i += 256) {
      const int r = i / (kDwgC / V), cv = (i % (kDwgC / V)) * V;
      const int64_t t = tb + r;
      float f[V];
      if (t < t_end && xvec) {
        unpack16(ld_nc_v4(X + t * D + c0 + cv), f, (const T*)nullptr);
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) f[q] = (t < t_end && c0 + cv + q < D) ? Elem<T>::load(X + t * D + c0 + cv + q) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < V; ++q) xs[r][cv + q] = f[q];
    }
    // dG tile: 32 tokens x 32 columns
    {
      const int r = threadIdx.x >> 3, cv = (threadIdx.x & 7) * 4;
      const int64_t t = tb + r;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < t_end) {
        if (gvec) g = __ldg(reinterpret_cast<const float4*>(dG + t * dM + col0 + cv));
        else {
          g.x = col0 + cv + 0 < dM ? dG[t * dM + col0 + cv + 0] : 0.f;
          g.y = col0 + cv + 1 < dM ? dG[t * dM + col0 + cv + 1] : 0.f;
          g.z = col0 + cv + 2 < dM ? dG[t * dM + col0 + cv + 2] : 0.f;
          g.w = col0 + cv + 3 < dM ? dG[t * dM + col0 + cv + 3] : 0.f;
        }
      }
      *reinterpret_cast<float4*>(&gs[r][cv]) = g;
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < kDwgTok; ++r) {
      const float4 xa = *reinterpret_cast<const float4*>(&xs[r][tc * 4]);
      const float4 gb = *reinterpret_cast<const float4*>(&gs[r][tg * 4]);
      const float xv[4] = {xa.x, xa.y, xa.z, xa.w}, gv[4] = {gb.x, gb.y, gb.z, gb.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xv[a], gv[b], acc[a][b]);
      if (tc == 0) {
#pragma unroll
        for (int b = 0; b < 4; ++b) bsum[b] += gv[b];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int c = c0 + tc * 4 + a;
    if (c >= D) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int col = col0 + tg * 4 + b;
      if (col < dM) partial[(split * D + c) * dM + col] = acc[a][b];
    }
  }
  if (blockIdx.x == 0 && tc == 0)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int col = col0 + tg * 4 + b;
      if (col < dM) pb[split * dM + col] = bsum[b];
    }
}

// partial[split][c][col] = sum_{t in split} X[t][c] dG[t][col]; pb[split][col] = sum dG[t][col]
// Small gates (D * dM < 64K, e.g. 256 x 32): 64 columns of X (c) x 32 columns of dG (col) per
// CTA, 32 tokens per smem pass, each thread 8 outputs: more, shorter CTAs for a latency-bound size.
template <typename T>
__global__ void __launch_bounds__(256)
k_dwg_partial_small(const T* __restrict__ X, const float* __restrict__ dG, int64_t Tn, int32_t D, int dM,
              int64_t tok_per_split, float* __restrict__ partial, float* __restrict__ pb) {
  DMOE_PDL_ENTRY();
  __shared__ float xs[32][65];
  __shared__ float gs[32][33];
  constexpr int V = Vec16<T>::N;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty: 0..7
  const int c0 = blockIdx.x * 64, col0 = blockIdx.y * 32;
  const int64_t split = blockIdx.z;
  const int64_t t_begin = split * tok_per_split;
  int64_t t_end = t_begin + tok_per_split;
  if (t_end > Tn) t_end = Tn;
  float acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
  float bsum = 0.0f;
  const bool xvec = (c0 + 64 <= D);
  const bool gvec = (col0 + 32 <= dM) && (dM % 4 == 0);
  for (int64_t tb = t_begin; tb < t_end; tb += 32) {
    // X tile: 32 tokens x 64 columns
    for (int i = threadIdx.x; i < 32 * (64 / V); i += 256) {
      const int r = i / (64 / V), cv = (i % (64 / V)) * V;
      const int64_t t = tb + r;
      float f[V];
      if (t < t_end && xvec) {
        unpack16(ld_nc_v4(X + t * D + c0 + cv), f, (const T*)nullptr);
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) f[q] = (t < t_end && c0 + cv + q < D) ? Elem<T>::load(X + t * D + c0 + cv + q) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < V; ++q) xs[r][cv + q] = f[q];
    }
    // dG tile: 32 tokens x 32 columns (fp32)
    for (int i = threadIdx.x; i < 32 * 8; i += 256) {
      const int r = i / 8, cv = (i % 8) * 4;
      const int64_t t = tb + r;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < t_end) {
        if (gvec) g = __ldg(reinterpret_cast<const float4*>(dG + t * dM + col0 + cv));
        else {
          g.x = col0 + cv + 0 < dM ? dG[t * dM + col0 + cv + 0] : 0.f;
          g.y = col0 + cv + 1 < dM ? dG[t * dM + col0 + cv + 1] : 0.f;
          g.z = col0 + cv + 2 < dM ? dG[t * dM + col0 + cv + 2] : 0.f;
          g.w = col0 + cv + 3 < dM ? dG[t * dM + col0 + cv + 3] : 0.f;
        }
      }
      gs[r][cv] = g.x; gs[r][cv + 1] = g.y; gs[r][cv + 2] = g.z; gs[r][cv + 3] = g.w;
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const float g = gs[r][tx];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fmaf(xs[r][ty * 8 + q], g, acc[q]);
      if (ty == 0) bsum += g;
    }
    __syncthreads();
  }
  const int col = col0 + tx;
  if (col < dM) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = c0 + ty * 8 + q;
      if (c < D) partial[(split * D + c) * dM + col] = acc[q];
    }
    if (blockIdx.x == 0 && ty == 0) pb[split * dM + col] = bsum;
  }
}

// out[i] = sum over splits, 8 thread groups x (every 8th split) then a fixed-order combine
__global__ void __launch_bounds__(256)
k_dwg_reduce(const float* __restrict__ partial, const float* __restrict__ pb, int64_t nsplit, int32_t D, int dM,
             float* __restrict__ dWg, float* __restrict__ dbg) {
  DMOE_PDL_ENTRY();
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t n = (int64_t)D * dM;
  const int64_t i = blockIdx.x * 32 + lane;  // output index (dWg then dbg)
  float v = 0.0f;
  if (i < n + dM) {
    const float* src = i < n ? partial + i : pb + (i - n);
    const int64_t stride = i < n ? n : dM;
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t sidx = grp + 8 * j;
      a[j] = sidx < nsplit ? src[sidx * stride] : 0.0f;
    }
    for (int64_t s0 = grp + 64; s0 < nsplit; s0 += 64)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (s0 + 8 * j < nsplit) a[j] += src[(s0 + 8 * j) * stride];
    v = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  }
  red[grp][lane] = v;
  __syncthreads();
  if (grp == 0 && i < n + dM) {
    float t = 0.0f;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += red[g][lane];
    if (i < n) dWg[i] = t;
    else dbg[i - n] = t;
  }
}

// split-K over tokens: >= 64 tokens per split, partial sums capped at 8M floats
// split-K over tokens: one 32-token pass per split where the partial sums (capped at 8M floats)
// allow, so the CTAs stay short and many
static int64_t dwg_splits(int64_t T, int32_t D, int dM) {
  int64_t s = ceil_div(T, kDwgTok);
  const int64_t smax = ((int64_t)8 << 20) / ((int64_t)D * dM);
  if (s > smax) s = smax;
  return s < 1 ? 1 : s;
}

size_t gate_bwd_ws_bytes(int64_t T, int32_t D, int dM) {
  const int64_t S = dwg_splits(T, D, dM);
  return align_up((size_t)D * dM * 4, 256) + align_up((size_t)(T > 0 ? T : 1) * dM * 4, 256) +
         align_up((size_t)S * D * dM * 4, 256) + align_up((size_t)S * dM * 4, 256) + 1024;
}

dmoe_status gate_bwd(const void* x, const void* Wg, const int32_t* sel, const float* dscore,
                     const void* dxd, const int32_t* row_of_slot, int64_t T, int32_t D, int d, int M,
                     int k, dmoe_dtype dt, void* dx, float* dWg, float* dbg, void* ws,
                     size_t ws_bytes, cudaStream_t s) {
  const int dM = d * M;
  const int64_t S = dwg_splits(T, D, dM);
  const size_t esz = dt == DMOE_BF16 ? 2 : 4;
  Carver cv(ws, ws_bytes);
  void* WgT = cv.take<char>((size_t)D * dM * esz);
  float* dG = cv.take<float>((size_t)(T > 0 ? T : 1) * dM);
  float* part = cv.take<float>((size_t)S * D * dM);
  float* pb = cv.take<float>((size_t)S * dM);
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "gate_bwd: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  dim3 tb(32, 8), tg((unsigned)ceil_div(dM, 32), (unsigned)ceil_div(D, 32));
  if (dt == DMOE_BF16)
    launch_pdl(k_transpose<__nv_bfloat16>, tg, tb, 0, s, (const __nv_bfloat16*)Wg, D, dM, (__nv_bfloat16*)WgT);
  else
    launch_pdl(k_transpose<float>, tg, tb, 0, s, (const float*)Wg, D, dM, (float*)WgT);
  DMOE_TRY(check_launch("gate_bwd.transpose"));
  if (T > 0) {
    int64_t b = ceil_div(T, kGbWarps), cap = (int64_t)num_sms() * 16;
    unsigned grid = (unsigned)(b < cap ? b : cap);
#define DMOE_GBDX(KM)                                                                                   \
    if (dt == DMOE_BF16)                                                                                \
      launch_pdl(k_gate_bwd_dx<__nv_bfloat16, KM>, grid, kGbWarps * 32, 0, s, \
          (const __nv_bfloat16*)WgT, sel, dscore, (const __nv_bfloat16*)dxd, row_of_slot, T, D, d, M,   \
          k, (__nv_bfloat16*)dx, dG);                                                                   \
    else                                                                                                \
      launch_pdl(k_gate_bwd_dx<float, KM>, grid, kGbWarps * 32, 0, s, (const float*)WgT, sel, dscore,          \
                                                              (const float*)dxd, row_of_slot, T, D, d, \
                                                              M, k, (float*)dx, dG);
    if (k <= 4) { DMOE_GBDX(4) } else if (k <= 8) { DMOE_GBDX(8) } else { DMOE_GBDX(16) }
#undef DMOE_GBDX
    DMOE_TRY(check_launch("gate_bwd.dx"));
  }
  const int64_t tps = T > 0 ? ceil_div(T, S) : 1;
  if ((int64_t)D * dM < 65536) {
    dim3 pg((unsigned)ceil_div(D, 64), (unsigned)ceil_div(dM, 32), (unsigned)S);
    if (dt == DMOE_BF16)
      launch_pdl(k_dwg_partial_small<__nv_bfloat16>, pg, 256, 0, s, (const __nv_bfloat16*)x, dG, T, D, dM, tps,
                 part, pb);
    else
      launch_pdl(k_dwg_partial_small<float>, pg, 256, 0, s, (const float*)x, dG, T, D, dM, tps, part, pb);
  } else {
    dim3 pg((unsigned)ceil_div(D, kDwgC), (unsigned)ceil_div(dM, kDwgCol), (unsigned)S);
    if (dt == DMOE_BF16)
      launch_pdl(k_dwg_partial<__nv_bfloat16>, pg, 256, 0, s, (const __nv_bfloat16*)x, dG, T, D, dM, tps, part, pb);
    else
      launch_pdl(k_dwg_partial<float>, pg, 256, 0, s, (const float*)x, dG, T, D, dM, tps, part, pb);
  }
  DMOE_TRY(check_launch("gate_bwd.dwg_partial"));
  launch_pdl(k_dwg_reduce, (unsigned)ceil_div((int64_t)D * dM + dM, 32), 256, 0, s, part, pb, S, D, dM, dWg, dbg);
  return check_launch("gate_bwd.dwg_reduce");
}

}  // namespace dmoe
