// gemm_simt.cu — exact-fp32 SIMT grouped GEMMs for the fp32 parity configuration
// (BASELINE config 1) and for shapes the tcgen05 engine does not take.  No tensor cores,
// no TF32: every product and sum is an fp32 FMA, so fp32 parity holds at 1e-4.
//
// Two families, both over per-expert row segments [offsets[e], offsets[e+1]):
//   ROWS (the expert Forward/Backward-dx GEMMs):
//     C[r, n] = epi( sum_k A[r, k] * B_e(n, k) ),  B_e K-major [E][N][K] or MN-major [E][K][N]
//   SEGK (the expert weight-gradient GEMMs):
//     C_e[m, n] = sum_{r in seg e} A[r, m] * B[r, n]        (0 for an empty segment)
// Tile 64x64, BK 16, 256 threads x (4x4) outputs.  Row tiles are enumerated through the
// per-expert tile plan (exclusive prefix of ceil(m_e/64)).
#include "common.cuh"
#include "gemm.cuh"

namespace dmoe {

constexpr int SB = 64, SK = 16;

__device__ __forceinline__ int find_group(const int32_t* __restrict__ plan, int E, int tile) {
  int lo = 0, hi = E;  // plan[lo] <= tile < plan[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (plan[mid] <= tile) lo = mid; else hi = mid;
  }
  return lo;
}

template <typename T, typename TC, bool B_MN, int EPI>
__global__ void __launch_bounds__(256)
k_simt_rows(const T* __restrict__ A, const T* __restrict__ B, TC* __restrict__ C,
            const float* __restrict__ bias, const T* __restrict__ aux,
            const int32_t* __restrict__ offsets, const int32_t* __restrict__ plan, int E, int N,
            int K, int64_t rows_single) {
  DMOE_PDL_ENTRY();
  __shared__ float As[SK][SB + 1];
  __shared__ float Bs[SK][SB + 1];
  const int tile = blockIdx.x;
  int e = 0;
  int64_t r_begin, r_end;
  if (offsets) {
    if (tile >= plan[E]) return;
    e = find_group(plan, E, tile);
    r_begin = offsets[e] + (int64_t)(tile - plan[e]) * SB;
    r_end = offsets[e + 1];
  } else {
    r_begin = (int64_t)tile * SB;
    r_end = rows_single;
    if (r_begin >= r_end) return;
  }
  const int n0 = blockIdx.y * SB;
  const T* Be = B + (int64_t)e * N * K;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += SK) {
    for (int i = threadIdx.x; i < SB * SK; i += 256) {
      int r = i / SK, kk = i % SK;
      int64_t row = r_begin + r;
      As[kk][r] = (row < r_end && k0 + kk < K) ? Elem<T>::load(A + row * K + k0 + kk) : 0.0f;
      int n = i / SK;
      float bv = 0.0f;
      if (n0 + n < N && k0 + kk < K)
        bv = B_MN ? Elem<T>::load(Be + (int64_t)(k0 + kk) * N + n0 + n)
                  : Elem<T>::load(Be + (int64_t)(n0 + n) * K + k0 + kk);
      Bs[kk][n] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t row = r_begin + ty * 4 + i;
    if (row >= r_end) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (EPI == EPI_F32_BIAS || EPI == EPI_BIAS || EPI == EPI_BIAS_RELU) v += bias[(int64_t)e * N + n];
      if (EPI == EPI_BIAS_RELU) v = fmaxf(v, 0.0f);
      if (EPI == EPI_RELU_MASK) v = Elem<T>::load(aux + row * N + n) > 0.0f ? v : 0.0f;
      Elem<TC>::store(C + row * N + n, v);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_simt_segk(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
            const int32_t* __restrict__ offsets, int Mdim, int N) {
  DMOE_PDL_ENTRY();
  __shared__ float As[SK][SB + 1];
  __shared__ float Bs[SK][SB + 1];
  const int e = blockIdx.z;
  const int m0 = blockIdx.y * SB, n0 = blockIdx.x * SB;
  const int64_t r_begin = offsets[e], r_end = offsets[e + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int64_t r0 = r_begin; r0 < r_end; r0 += SK) {
    for (int i = threadIdx.x; i < SB * SK; i += 256) {
      int rr = i / SB, c = i % SB;
      int64_t row = r0 + rr;
      bool in = row < r_end;
      As[rr][c] = (in && m0 + c < Mdim) ? Elem<T>::load(A + row * Mdim + m0 + c) : 0.0f;
      Bs[rr][c] = (in && n0 + c < N) ? Elem<T>::load(B + row * N + n0 + c) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  T* Ce = C + (int64_t)e * Mdim * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= Mdim) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n < N) Elem<T>::store(Ce + (int64_t)m * N + n, acc[i][j]);
    }
  }
}

// segment column sums: out[e][n] = sum_{r in seg e} X[r][n] (fp32, row order) — db1 / db2
// Block = 8 warps over one expert and a 32-vector column strip; warp w sums rows
// r0+w, r0+w+8, ... (2 loads in flight), then the 8 partials are added in warp order
// (fixed order -> deterministic).
constexpr int kCsWarps = 8;
template <typename T>
__global__ void __launch_bounds__(kCsWarps * 32)
k_seg_colsum(const T* __restrict__ X, const int32_t* __restrict__ offsets, int N,
             float* __restrict__ out) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N;
  __shared__ float part[kCsWarps][32 * V + 1];
  const int e = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = (blockIdx.x * 32 + lane) * V;
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.0f;
  const int64_t r0 = offsets[e], r1 = offsets[e + 1];
  if (n < N) {
    int64_t r = r0 + warp;
    for (; r + kCsWarps < r1; r += 2 * kCsWarps) {
      const uint4 u0 = ld_nc_v4(X + r * N + n);
      const uint4 u1 = ld_nc_v4(X + (r + kCsWarps) * N + n);
      float f0[V], f1[V];
      unpack16(u0, f0, (const T*)nullptr);
      unpack16(u1, f1, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += f0[i] + f1[i];
    }
    if (r < r1) {
      float f[V];
      unpack16(ld_nc_v4(X + r * N + n), f, (const T*)nullptr);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += f[i];
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) part[warp][lane * V + i] = acc[i];
  __syncthreads();
  for (int c = threadIdx.x; c < 32 * V; c += kCsWarps * 32) {
    const int col = blockIdx.x * 32 * V + c;
    if (col >= N) continue;
    float v = 0.0f;
#pragma unroll
    for (int w = 0; w < kCsWarps; ++w) v += part[w][c];
    out[(int64_t)e * N + col] = v;
  }
}

template <typename T, typename TC>
static void launch_rows(const GemmRows& g, cudaStream_t s) {
  dim3 grid((unsigned)g.max_tiles, (unsigned)ceil_div(g.N, SB));
#define DMOE_ROWS(BMN, EPI_)                                                                   \
  launch_pdl(k_simt_rows<T, TC, BMN, EPI_>, grid, 256, 0, s, (const T*)g.A, (const T*)g.B, (TC*)g.C,     \
                                                      g.bias, (const T*)g.aux, g.offsets, g.plan, \
                                                      g.E, g.N, g.K, g.rows_single)
#define DMOE_ROWS_EPI(BMN)                                      \
  switch (g.epi) {                                              \
    case EPI_F32_BIAS: DMOE_ROWS(BMN, EPI_F32_BIAS); break;     \
    case EPI_BIAS_RELU: DMOE_ROWS(BMN, EPI_BIAS_RELU); break;   \
    case EPI_BIAS: DMOE_ROWS(BMN, EPI_BIAS); break;             \
    case EPI_RELU_MASK: DMOE_ROWS(BMN, EPI_RELU_MASK); break;   \
    default: DMOE_ROWS(BMN, EPI_PLAIN); break;                  \
  }
  if (g.b_mn) { DMOE_ROWS_EPI(true) } else { DMOE_ROWS_EPI(false) }
#undef DMOE_ROWS_EPI
#undef DMOE_ROWS
}

dmoe_status simt_gemm_rows(const GemmRows& g, dmoe_dtype dt, cudaStream_t s) {
  if (g.max_tiles <= 0) return DMOE_OK;
  if (dt == DMOE_BF16) {
    if (g.epi == EPI_F32_BIAS) launch_rows<__nv_bfloat16, float>(g, s);
    else launch_rows<__nv_bfloat16, __nv_bfloat16>(g, s);
  } else {
    launch_rows<float, float>(g, s);
  }
  __atomic_fetch_add(&g_counters[2], 1, __ATOMIC_RELAXED);
  return check_launch("simt_gemm_rows");
}

dmoe_status simt_gemm_segk(const GemmSegK& g, dmoe_dtype dt, cudaStream_t s) {
  dim3 grid((unsigned)ceil_div(g.N, SB), (unsigned)ceil_div(g.Mdim, SB), (unsigned)g.E);
  if (dt == DMOE_BF16)
    launch_pdl(k_simt_segk<__nv_bfloat16>, grid, 256, 0, s, (const __nv_bfloat16*)g.A, (const __nv_bfloat16*)g.B,
                                                    (__nv_bfloat16*)g.C, g.offsets, g.Mdim, g.N);
  else
    launch_pdl(k_simt_segk<float>, grid, 256, 0, s, (const float*)g.A, (const float*)g.B, (float*)g.C,
                                            g.offsets, g.Mdim, g.N);
  __atomic_fetch_add(&g_counters[2], 1, __ATOMIC_RELAXED);
  return check_launch("simt_gemm_segk");
}

dmoe_status seg_colsum(const void* X, dmoe_dtype dt, const int32_t* offsets, int E, int N,
                       float* out, cudaStream_t s) {
  const int V = dt == DMOE_BF16 ? 8 : 4;  // N % V == 0 is validated by the caller
  dim3 grid((unsigned)ceil_div(N, 32 * V), (unsigned)E);
  if (dt == DMOE_BF16)
    launch_pdl(k_seg_colsum<__nv_bfloat16>, grid, kCsWarps * 32, 0, s, (const __nv_bfloat16*)X, offsets, N, out);
  else
    launch_pdl(k_seg_colsum<float>, grid, kCsWarps * 32, 0, s, (const float*)X, offsets, N, out);
  return check_launch("seg_colsum");
}

}  // namespace dmoe
