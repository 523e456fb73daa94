// gate_bwd.cu — S10: undispatch (sum the expert-path input gradients back per token)
// and the gating gradient of Eq. 2 through the Eq. 3 softmax.
//
//   dG[t, i*M + u_i(sel_ts)] += dscore_ts            (sparse: <= k*d non-zeros per row)
//   dX_t  = sum_{ok s} dXd[row_ts] + sum_s dscore_ts sum_i W_g[:, i*M + u_i(sel_ts)]
//   dW_g  = X^T dG (fp32),  db_g = column sums of dG (fp32)
//
// W_g is transposed once into the workspace so the k*d gate columns a token touches are
// contiguous rows (coalesced, L2-resident).  k_gate_bwd_dx (warp per token) writes dX, the
// per-CTA bias partials and the token's dG row.  dW_g is a dense contraction over the tokens:
// on the bf16 path it runs on the tensor cores as a split-K weight-gradient GEMM (the SEGK
// engine of gemm_tc.cu, token chunks as segments, fp32 partial output) over dG split exactly
// into two bf16 halves (hi = bf16(dG), lo = bf16(dG - hi): 16 significant bits, and X is
// bf16 already), i.e. B = [dG_hi | dG_lo]; the fp32 path keeps a SIMT split-K.  Partials are
// summed over chunks (and hi + lo) in a fixed order: deterministic, no float atomics.
#include "gemm.cuh"

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


// dX (undispatch + gate path), the per-CTA partial bias gradient and the tokens' dG rows, one
// warp per token: every dxd row segment of the token's k dispatched rows is loaded before the
// first add (UNR 16-byte vectors per lane per row), the d*k gate rows come from W_g^T
// (transposed once, 2*d*M*D bytes: L2-resident), and the next token's routing record is fetched
// while this token's rows are in flight.  The token's dG row is written as exact bf16 hi | lo
// halves padded to ld2 columns (tensor-core dW_g) or as dense fp32 (SIMT dW_g), and the CTA's
// bias partial db_g = sum_t dG[t] (lane owns columns lane + 32 m; warps combined in a fixed order:
// deterministic).  Block 0 writes the token chunk bounds of the split-K dW_g GEMM.
constexpr int kGbWarps = 4;
// k <= 4: two 16-byte vectors per lane per row in flight and 5 CTAs (20 warps) per SM (93
// registers) beat four vectors at 3 CTAs per SM (transformer 295-358 -> 204 us, grid3d 1.2-1.6 ->
// 0.85-1.36 ms in one launch list)
#ifndef GBDX_UNR4
#define GBDX_UNR4 2
#endif
#ifndef GBDX_MINB
#define GBDX_MINB 5
#endif

template <int KMAX>
struct GbRec {  // a token's routing record: dispatched rows, dscore, gate columns (one byte per level)
  int32_t rows[KMAX];
  uint32_t cols[KMAX];  // byte i = i*M + u_i(e) (< d*M <= 256); 0xffffffff: no expert
  float ds[KMAX];
  __device__ __forceinline__ void load(const int32_t* __restrict__ row_of_slot, const int32_t* __restrict__ sel,
                                       const float* __restrict__ dscore, int64_t t, int64_t Tn, int d, int M,
                                       int mshift, int k) {
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      const bool on = s < k && t < Tn;
      rows[s] = on ? row_of_slot[t * k + s] : -1;
      const int32_t e = on ? sel[t * k + s] : -1;
      ds[s] = (on && e >= 0) ? dscore[t * k + s] : 0.0f;
      uint32_t pk = 0xffffffffu;
      if (e >= 0) {  // u_i(e) (reading X1): the last level is the lowest base-M digit
        pk = 0u;
        uint32_t ee = (uint32_t)e;
#pragma unroll
        for (int i = 3; i >= 0; --i) {
          if (i >= d) continue;
          uint32_t q, r;
          if (mshift >= 0) { q = ee >> mshift; r = ee & ((1u << mshift) - 1u); }
          else { q = ee / (uint32_t)M; r = ee - q * (uint32_t)M; }
          pk |= ((uint32_t)i * (uint32_t)M + r) << (8 * i);
          ee = q;
        }
      }
      cols[s] = pk;
    }
  }
};

template <typename T, int KMAX>
__global__ void __launch_bounds__(kGbWarps * 32, KMAX <= 4 ? GBDX_MINB : 1)
k_gate_bwd_dx(const T* __restrict__ WgT, const int32_t* __restrict__ sel,
              const float* __restrict__ dscore, const T* __restrict__ dxd,
              const int32_t* __restrict__ row_of_slot, int64_t Tn, int32_t D, int d, int M, int k,
              T* __restrict__ dx, float* __restrict__ pb, float* __restrict__ dG,
              __nv_bfloat16* __restrict__ dG2, int ld2, int32_t* __restrict__ chunk_off, int nchunk,
              int64_t tpc) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N;
  constexpr int UNR = KMAX <= 4 ? GBDX_UNR4 : (KMAX <= 8 ? 2 : 1);  // 16-byte vectors per lane per row in flight
  constexpr int NB = 8;                                      // gate columns per lane (d*M <= 256)
  __shared__ float bsh[kGbWarps][NB * 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int dM = d * M;
  const int mshift = (M & (M - 1)) == 0 ? __ffs(M) - 1 : -1;
  if (chunk_off && blockIdx.x == 0)
    for (int i = threadIdx.x; i <= nchunk; i += blockDim.x)
      chunk_off[i] = (int32_t)((int64_t)i * tpc < Tn ? (int64_t)i * tpc : Tn);
  float bpart[NB];
#pragma unroll
  for (int m = 0; m < NB; ++m) bpart[m] = 0.0f;
  const int64_t stride = (int64_t)gridDim.x * kGbWarps;
  int64_t t = (int64_t)blockIdx.x * kGbWarps + wib;
  GbRec<KMAX> cur, nxt;
  cur.load(row_of_slot, sel, dscore, t, Tn, d, M, mshift, k);
  for (; t < Tn; t += stride) {
    nxt.load(row_of_slot, sel, dscore, t + stride, Tn, d, M, mshift, k);  // in flight with this token's rows
    for (int c0 = lane * V; c0 < D; c0 += UNR * 32 * V) {
      uint4 u[KMAX][UNR];
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          const int c = c0 + q * 32 * V;
          u[s][q] = make_uint4(0u, 0u, 0u, 0u);  // a missing row reads as zeros
          if (cur.rows[s] >= 0 && c < D) u[s][q] = ld_nc_v4(dxd + (int64_t)cur.rows[s] * D + c);
        }
      float acc[UNR][V];
#pragma unroll
      for (int q = 0; q < UNR; ++q)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[q][j] = 0.0f;
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (s >= k) break;
#pragma unroll
        for (int q = 0; q < UNR; ++q) {
          float f[V];
          unpack16(u[s][q], f, (const T*)nullptr);
#pragma unroll
          for (int j = 0; j < V; ++j) acc[q][j] += f[j];
        }
      }
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (cur.ds[s] == 0.0f) continue;
#pragma unroll
        for (int i = 3; i >= 0; --i) {  // last level first
          if (i >= d) continue;
          const int64_t col = (cur.cols[s] >> (8 * i)) & 0xffu;
#pragma unroll
          for (int q = 0; q < UNR; ++q) {
            const int c = c0 + q * 32 * V;
            if (c >= D) continue;
            float f[V];
            unpack16(ld_v4(WgT + col * D + c), f, (const T*)nullptr);
#pragma unroll
            for (int j = 0; j < V; ++j) acc[q][j] = fmaf(cur.ds[s], f[j], acc[q][j]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int c = c0 + q * 32 * V;
        if (c < D) st_v4(dx + t * D + c, pack16(acc[q], (const T*)nullptr));
      }
    }
    // the token's dG row for the lane's columns lane + 32 m (fixed slot, level order; adding the
    // zeros of the other lanes' entries changes nothing)
    float g[NB];
#pragma unroll
    for (int m = 0; m < NB; ++m) g[m] = 0.0f;
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      if (cur.cols[s] == 0xffffffffu) continue;
#pragma unroll
      for (int i = 3; i >= 0; --i) {
        if (i >= d) continue;
        const int col = (int)((cur.cols[s] >> (8 * i)) & 0xffu);
        const float add = (col & 31) == lane ? cur.ds[s] : 0.0f;
#pragma unroll
        for (int m = 0; m < NB; ++m) g[m] += m == (col >> 5) ? add : 0.0f;
      }
    }
#pragma unroll
    for (int m = 0; m < NB; ++m) {
      const int col = lane + 32 * m;
      if (col >= dM) break;
      bpart[m] += g[m];
      if (dG) dG[t * dM + col] = g[m];
      if (dG2) {
        const __nv_bfloat16 hi = __float2bfloat16_rn(g[m]);
        dG2[t * ld2 + col] = hi;
        dG2[t * ld2 + dM + col] = __float2bfloat16_rn(g[m] - __bfloat162float(hi));
      }
    }
    if (dG2)
      for (int col = 2 * dM + lane; col < ld2; col += 32) dG2[t * ld2 + col] = __float2bfloat16_rn(0.0f);
    cur = nxt;
  }
#pragma unroll
  for (int m = 0; m < NB; ++m) bsh[wib][lane + 32 * m] = bpart[m];
  __syncthreads();
  for (int col = threadIdx.x; col < dM; col += blockDim.x) {
    float v = 0.0f;
#pragma unroll
    for (int w = 0; w < kGbWarps; ++w) v += bsh[w][col];
    pb[(int64_t)blockIdx.x * dM + col] = v;
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
  if (pb && blockIdx.x == 0 && tc == 0)
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
    if (pb && blockIdx.x == 0 && ty == 0) pb[split * dM + col] = bsum;
  }
}

// dWg[c][col] = sum over splits s of partial[s][c][col] (+ partial[s][c][dM + col]: the lo half
// on the tensor-core path; ld = the partial's row length), split order; dbg[col] = sum over the
// dx kernel's CTAs of pb[cta][col] (one warp per column, lane-strided then a fixed tree)
__global__ void __launch_bounds__(256)
k_gate_reduce(const float* __restrict__ partial, int64_t nsplit, int ld, int hilo, const float* __restrict__ pb,
              int64_t npb, int32_t D, int dM, float* __restrict__ dWg, float* __restrict__ dbg) {
  DMOE_PDL_ENTRY();
  const int64_t n = (int64_t)D * dM;
  const int64_t nblk_w = ceil_div_dev(n, 256);
  if (blockIdx.x < nblk_w) {
    const int64_t i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    const int64_t c = i / dM, col = i - c * dM;
    const float* src = partial + c * ld + col;
    const int64_t stride = (int64_t)D * ld;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    int64_t s = 0;
    for (; s + 4 <= nsplit; s += 4)
#pragma unroll
      for (int j = 0; j < 4; ++j) a[j] += hilo ? src[(s + j) * stride] + src[(s + j) * stride + dM] : src[(s + j) * stride];
    for (; s < nsplit; ++s) a[0] += hilo ? src[s * stride] + src[s * stride + dM] : src[s * stride];
    dWg[i] = (a[0] + a[1]) + (a[2] + a[3]);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t col = (blockIdx.x - nblk_w) * 8 + (threadIdx.x >> 5);
  if (col >= dM) return;
  float v = 0.0f;
  for (int64_t b = lane; b < npb; b += 32) v += pb[b * dM + col];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) dbg[col] = v;
}

static int64_t gbdx_grid(int64_t T) {
  const int64_t b = ceil_div(T > 0 ? T : 1, kGbWarps), cap = (int64_t)num_sms() * 16;
  return b < cap ? b : cap;
}
// SIMT split-K over tokens (fp32 path): one 32-token pass per split where the partial sums
// (capped at 8M floats) allow
static int64_t dwg_splits(int64_t T, int32_t D, int dM) {
  int64_t s = ceil_div(T, kDwgTok);
  const int64_t smax = ((int64_t)8 << 20) / ((int64_t)D * dM);
  if (s > smax) s = smax;
  return s < 1 ? 1 : s;
}
// tensor-core split-K: token chunks so that chunks x (D / 128) M-tiles ~ two tiles per SM
static int64_t tc_chunks(int64_t T, int32_t D) {
  const int64_t mt = D >= 128 ? (int64_t)D / 128 : 1;  // M tiles (the path needs D % 128 == 0)
  int64_t c = ceil_div((int64_t)num_sms() * 2, mt);
  const int64_t cmax = ceil_div(T > 0 ? T : 1, 256);  // >= 256 tokens (4 K blocks) per chunk
  if (c > cmax) c = cmax;
  return c < 1 ? 1 : c;
}
static int tc_ld2(int dM) { return (int)align_up((size_t)2 * dM, 128); }
static bool gate_bwd_tc(dmoe_dtype dt, int32_t D, int dM) {
  if (dt != DMOE_BF16) return false;
  GemmSegK g{};
  g.Mdim = D; g.N = tc_ld2(dM);
  return tc_segk_supported(g);
}

size_t gate_bwd_ws_bytes(int64_t T, int32_t D, int dM) {
  const size_t Tp = (size_t)(T > 0 ? T : 1);
  const size_t simt = align_up(Tp * dM * 4, 256) + align_up((size_t)dwg_splits(T, D, dM) * D * dM * 4, 256);
  const size_t tc = align_up(Tp * tc_ld2(dM) * 2, 256) + align_up((size_t)tc_chunks(T, D) * D * tc_ld2(dM) * 4, 256) +
                    align_up((size_t)(tc_chunks(T, D) + 1) * 4, 256);
  return align_up((size_t)D * dM * 4, 256) + (simt > tc ? simt : tc) + align_up((size_t)gbdx_grid(T) * dM * 4, 256) +
         1024;
}

dmoe_status gate_bwd(const void* x, const void* Wg, const int32_t* sel, const float* dscore,
                     const void* dxd, const int32_t* row_of_slot, int64_t T, int32_t D, int d, int M,
                     int k, dmoe_dtype dt, void* dx, float* dWg, float* dbg, void* ws,
                     size_t ws_bytes, cudaStream_t s) {
  const int dM = d * M;
  DMOE_REQUIRE(dM <= 256, DMOE_ERR_SHAPE, "gate_bwd: d*M=%d > 256", dM);
  const bool tc = gate_bwd_tc(dt, D, dM) && T > 0;
  const size_t esz = dt == DMOE_BF16 ? 2 : 4;
  const int64_t nb = gbdx_grid(T);
  Carver cv(ws, ws_bytes);
  void* WgT = cv.take<char>((size_t)D * dM * esz);
  float* pb = cv.take<float>((size_t)nb * dM);
  float* dG = nullptr;
  float* part = nullptr;
  __nv_bfloat16* dG2 = nullptr;
  int32_t* choff = nullptr;
  int64_t nsplit = 0;
  const int ld2 = tc_ld2(dM);
  if (tc) {
    nsplit = tc_chunks(T, D);
    dG2 = cv.take<__nv_bfloat16>((size_t)T * ld2);
    part = cv.take<float>((size_t)nsplit * D * ld2);
    choff = cv.take<int32_t>((size_t)nsplit + 1);
  } else {
    nsplit = T > 0 ? dwg_splits(T, D, dM) : 0;
    dG = cv.take<float>((size_t)(T > 0 ? T : 1) * dM);
    part = cv.take<float>((size_t)(nsplit > 0 ? nsplit : 1) * D * dM);
  }
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "gate_bwd: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  dim3 tb(32, 8), tg((unsigned)ceil_div(dM, 32), (unsigned)ceil_div(D, 32));
  if (dt == DMOE_BF16)
    launch_pdl(k_transpose<__nv_bfloat16>, tg, tb, 0, s, (const __nv_bfloat16*)Wg, D, dM, (__nv_bfloat16*)WgT);
  else
    launch_pdl(k_transpose<float>, tg, tb, 0, s, (const float*)Wg, D, dM, (float*)WgT);
  DMOE_TRY(check_launch("gate_bwd.transpose"));
  if (T > 0) {
    const int64_t tpc = tc ? ceil_div(T, nsplit) : 0;
#define DMOE_GBDX2(TT, KM)                                                                             \
    launch_pdl(k_gate_bwd_dx<TT, KM>, (unsigned)nb, kGbWarps * 32, 0, s, (const TT*)WgT, sel, dscore,   \
               (const TT*)dxd, row_of_slot, T, D, d, M, k, (TT*)dx, pb, dG, dG2, ld2, choff, (int)nsplit, tpc);
#define DMOE_GBDX(KM)                                                                                  \
    if (dt == DMOE_BF16) { DMOE_GBDX2(__nv_bfloat16, KM) } else { DMOE_GBDX2(float, KM) }
    if (k <= 4) { DMOE_GBDX(4) } else if (k <= 8) { DMOE_GBDX(8) } else { DMOE_GBDX(16) }
#undef DMOE_GBDX
#undef DMOE_GBDX2
    DMOE_TRY(check_launch("gate_bwd.dx"));
    if (tc) {
      // dW_g partials on the tensor cores: chunk c's [D][hi | lo] = X[chunk]^T [dG_hi | dG_lo]
      GemmSegK g{};
      g.A = x; g.B = dG2; g.C = part; g.offsets = choff; g.E = (int)nsplit; g.Mdim = D; g.N = ld2; g.R_cap = T;
      g.colsum = nullptr; g.out_f32 = true;
      DMOE_TRY(tc_gemm_segk(g, s));
    } else {
      const int64_t tps = ceil_div(T, nsplit);
      if ((int64_t)D * dM < 65536) {
        dim3 pg((unsigned)ceil_div(D, 64), (unsigned)ceil_div(dM, 32), (unsigned)nsplit);
        if (dt == DMOE_BF16)
          launch_pdl(k_dwg_partial_small<__nv_bfloat16>, pg, 256, 0, s, (const __nv_bfloat16*)x, dG, T, D, dM, tps,
                     part, (float*)nullptr);
        else
          launch_pdl(k_dwg_partial_small<float>, pg, 256, 0, s, (const float*)x, dG, T, D, dM, tps, part,
                     (float*)nullptr);
      } else {
        dim3 pg((unsigned)ceil_div(D, kDwgC), (unsigned)ceil_div(dM, kDwgCol), (unsigned)nsplit);
        if (dt == DMOE_BF16)
          launch_pdl(k_dwg_partial<__nv_bfloat16>, pg, 256, 0, s, (const __nv_bfloat16*)x, dG, T, D, dM, tps, part,
                     (float*)nullptr);
        else
          launch_pdl(k_dwg_partial<float>, pg, 256, 0, s, (const float*)x, dG, T, D, dM, tps, part, (float*)nullptr);
      }
      DMOE_TRY(check_launch("gate_bwd.dwg_partial"));
    }
  }
  const int64_t nw = ceil_div((int64_t)D * dM, 256), nbias = ceil_div(dM, 8);
  launch_pdl(k_gate_reduce, (unsigned)(nw + nbias), 256, 0, s, part, nsplit, tc ? ld2 : dM, tc ? 1 : 0, pb,
             T > 0 ? nb : 0, D, dM, dWg, dbg);
  return check_launch("gate_bwd.reduce");
}

}  // namespace dmoe
