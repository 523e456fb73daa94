// ffn3.cu — the row-wise stages of the paper's expert block (NEXT-2: "feedforward
// blocks 1024 -> 4096 -> 4096 -> 1024 with layer normalization and ReLU activations in between";
// reading X23): LayerNorm over the H features of a dispatched row with the row's expert's scale
// g / shift be (biased variance, eps), then ReLU, and its backward.  The three linears are the
// grouped tcgen05 GEMMs of gemm_tc.cu; these kernels sit between them.
//
//   forward  (one CTA per row):  a = relu(g * (z - mean) * rstd + be);  stats = (mean, rstd)
//   backward (one CTA per expert segment, rows in order, so dg / dbe accumulate
//             deterministically in registers):
//            dy = da * 1[g xhat + be > 0];  dg += dy xhat;  dbe += dy;  dxhat = dy g;
//            dz = rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat))
// z, a, da, dz are bf16 rows [R_cap, H]; statistics fp32 [R_cap][2]; g, be, dg, dbe fp32 [E, H].
#include "common.cuh"

namespace dmoe {

constexpr int kLnThreads = 256;

__device__ __forceinline__ float block_sum_ln(float v, float* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();  // sh reuse
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float t = 0.0f;
#pragma unroll
  for (int i = 0; i < kLnThreads / 32; ++i) t += sh[i];  // fixed order: deterministic
  return t;
}

__device__ __forceinline__ int expert_of_row(const int32_t* offsets, int E, int64_t r) {
  int lo = 0, hi = E;  // offsets[lo] <= r < offsets[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (offsets[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// VPT = H / (8 * kLnThreads) 16-byte vectors per thread (H <= 8192 -> VPT <= 4)
template <int VPT>
__global__ void __launch_bounds__(kLnThreads)
k_ln_relu_fwd(const __nv_bfloat16* __restrict__ z, const int32_t* __restrict__ offsets, int E, int H, float eps,
              const float* __restrict__ g, const float* __restrict__ be, __nv_bfloat16* __restrict__ a,
              float* __restrict__ stats) {
  DMOE_PDL_ENTRY();
  __shared__ float sh[kLnThreads / 32];
  const int64_t R = offsets[E];
  const int nvec = H / 8;
  for (int64_t r = blockIdx.x; r < R; r += gridDim.x) {
    const int e = expert_of_row(offsets, E, r);
    float v[VPT][8];
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int iv = threadIdx.x + q * kLnThreads;
      if (iv < nvec) {
        unpack16(ld_nc_v4(z + r * H + iv * 8), v[q], (const __nv_bfloat16*)nullptr);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[q][j];
      }
    }
    const float mean = block_sum_ln(s, sh) / H;
    float s2 = 0.0f;
#pragma unroll
    for (int q = 0; q < VPT; ++q)
      if (threadIdx.x + q * kLnThreads < nvec)
#pragma unroll
        for (int j = 0; j < 8; ++j) s2 += (v[q][j] - mean) * (v[q][j] - mean);
    const float rstd = rsqrtf(block_sum_ln(s2, sh) / H + eps);
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int iv = threadIdx.x + q * kLnThreads;
      if (iv >= nvec) continue;
      float o[8];
      const float* gg = g + (int64_t)e * H + iv * 8;
      const float* bb = be + (int64_t)e * H + iv * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = fmaxf(fmaf(gg[j], (v[q][j] - mean) * rstd, bb[j]), 0.0f);
      st_v4(a + r * H + iv * 8, pack16(o, (const __nv_bfloat16*)nullptr));
    }
    if (threadIdx.x == 0) { stats[2 * r] = mean; stats[2 * r + 1] = rstd; }
  }
}

template <int VPT>
__global__ void __launch_bounds__(kLnThreads)
k_ln_relu_bwd(const __nv_bfloat16* __restrict__ da, const __nv_bfloat16* __restrict__ z,
              const float* __restrict__ stats, const int32_t* __restrict__ offsets, int E, int H,
              const float* __restrict__ g, const float* __restrict__ be, __nv_bfloat16* __restrict__ dz,
              float* __restrict__ dg, float* __restrict__ dbe) {
  DMOE_PDL_ENTRY();
  __shared__ float sh[kLnThreads / 32];
  const int nvec = H / 8;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    float ag[VPT][8], ab[VPT][8], gv[VPT][8], bv[VPT][8];
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int iv = threadIdx.x + q * kLnThreads;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ag[q][j] = 0.0f; ab[q][j] = 0.0f;
        gv[q][j] = iv < nvec ? g[(int64_t)e * H + iv * 8 + j] : 0.0f;
        bv[q][j] = iv < nvec ? be[(int64_t)e * H + iv * 8 + j] : 0.0f;
      }
    }
    for (int64_t r = offsets[e]; r < offsets[e + 1]; ++r) {
      const float mean = stats[2 * r], rstd = stats[2 * r + 1];
      float xh[VPT][8], dx[VPT][8];
      float m1 = 0.0f, m2 = 0.0f;
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int iv = threadIdx.x + q * kLnThreads;
        if (iv >= nvec) continue;
        float zz[8], dd[8];
        unpack16(ld_nc_v4(z + r * H + iv * 8), zz, (const __nv_bfloat16*)nullptr);
        unpack16(ld_nc_v4(da + r * H + iv * 8), dd, (const __nv_bfloat16*)nullptr);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[q][j] = (zz[j] - mean) * rstd;
          const float dy = fmaf(gv[q][j], xh[q][j], bv[q][j]) > 0.0f ? dd[j] : 0.0f;  // ReLU'(0) = 0
          ag[q][j] = fmaf(dy, xh[q][j], ag[q][j]);
          ab[q][j] += dy;
          dx[q][j] = dy * gv[q][j];
          m1 += dx[q][j];
          m2 = fmaf(dx[q][j], xh[q][j], m2);
        }
      }
      m1 = block_sum_ln(m1, sh) / H;
      m2 = block_sum_ln(m2, sh) / H;
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        const int iv = threadIdx.x + q * kLnThreads;
        if (iv >= nvec) continue;
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rstd * (dx[q][j] - m1 - xh[q][j] * m2);
        st_v4(dz + r * H + iv * 8, pack16(o, (const __nv_bfloat16*)nullptr));
      }
    }
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int iv = threadIdx.x + q * kLnThreads;
      if (iv >= nvec) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dg[(int64_t)e * H + iv * 8 + j] = ag[q][j];
        dbe[(int64_t)e * H + iv * 8 + j] = ab[q][j];
      }
    }
  }
}

static int ln_vpt(int H) { return (int)ceil_div(H / 8, kLnThreads); }

dmoe_status ln_relu_fwd(const void* z, const int32_t* offsets, int E, int64_t R_cap, int H, float eps,
                        const float* g, const float* be, void* a, float* stats, cudaStream_t s) {
  int64_t grid = R_cap < (int64_t)num_sms() * 16 ? R_cap : (int64_t)num_sms() * 16;
  if (grid < 1) grid = 1;
  const int vpt = ln_vpt(H);
#define DMOE_LNF(V)                                                                                        \
  launch_pdl(k_ln_relu_fwd<V>, (unsigned)grid, kLnThreads, 0, s, (const __nv_bfloat16*)z, offsets, E, H, eps, g, \
             be, (__nv_bfloat16*)a, stats)
  if (vpt <= 1) DMOE_LNF(1); else if (vpt <= 2) DMOE_LNF(2); else DMOE_LNF(4);
#undef DMOE_LNF
  return check_launch("ln_relu_fwd");
}

dmoe_status ln_relu_bwd(const void* da, const void* z, const float* stats, const int32_t* offsets, int E, int H,
                        const float* g, const float* be, void* dz, float* dg, float* dbe, cudaStream_t s) {
  const int vpt = ln_vpt(H);
#define DMOE_LNB(V)                                                                                         \
  launch_pdl(k_ln_relu_bwd<V>, (unsigned)E, kLnThreads, 0, s, (const __nv_bfloat16*)da, (const __nv_bfloat16*)z, \
             stats, offsets, E, H, g, be, (__nv_bfloat16*)dz, dg, dbe)
  if (vpt <= 1) DMOE_LNB(1); else if (vpt <= 2) DMOE_LNB(2); else DMOE_LNB(4);
#undef DMOE_LNB
  return check_launch("ln_relu_bwd");
}

}  // namespace dmoe
