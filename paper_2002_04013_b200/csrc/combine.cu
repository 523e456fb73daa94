// combine.cu — S7 combine (Eq. 3 weighted average) and S8 combine backward.
//
// One warp per token; rows are read and written as 16-byte vectors (8 bf16 / 4 fp32
// per lane), accumulation in fp32.  Eq. 3; backward = softmax
// Jacobian over the ok slots (S8).
#include "common.cuh"

namespace dmoe {

constexpr int kCombWarps = 4;

template <typename T, int kMaxK>
__global__ void __launch_bounds__(kCombWarps * 32)
k_combine(const T* __restrict__ out, const int32_t* __restrict__ row_of_slot,
          const float* __restrict__ w, const uint8_t* __restrict__ valid, int64_t Tn, int32_t D,
          int k, T* __restrict__ y) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  for (int64_t t = blockIdx.x * (int64_t)kCombWarps + (threadIdx.x >> 5); t < Tn;
       t += (int64_t)gridDim.x * kCombWarps) {
    int32_t rows[kMaxK];
    float ws[kMaxK];
#pragma unroll
    for (int s = 0; s < kMaxK; ++s) {
      rows[s] = s < k ? row_of_slot[t * k + s] : -1;
      ws[s] = s < k ? w[t * k + s] : 0.0f;
    }
    const bool ok_tok = valid[t] != 0;
    for (int c = lane * V; c < D; c += 32 * V) {
      float acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.0f;
      if (ok_tok) {
        // issue every slot's row load before accumulating (k independent loads in flight)
        uint4 u[kMaxK];
#pragma unroll
        for (int s = 0; s < kMaxK; ++s)
          if (s < k && rows[s] >= 0) u[s] = ld_nc_v4(out + (int64_t)rows[s] * D + c);
#pragma unroll
        for (int s = 0; s < kMaxK; ++s) {
          if (s >= k || rows[s] < 0) continue;
          float f[V];
          unpack16(u[s], f, (const T*)nullptr);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] = fmaf(ws[s], f[i], acc[i]);
        }
      }
      st_v4(y + t * D + c, pack16(acc, (const T*)nullptr));
    }
  }
}

template <typename T, int kMaxK>
__global__ void __launch_bounds__(kCombWarps * 32)
k_combine_bwd(const T* __restrict__ dy, const T* __restrict__ out,
              const int32_t* __restrict__ row_of_slot, const float* __restrict__ w, int64_t Tn,
              int32_t D, int k, const int32_t* __restrict__ sel, const uint32_t* __restrict__ bwd_ok,
              T* __restrict__ dout, float* __restrict__ dscore) {
  DMOE_PDL_ENTRY();
  constexpr int V = Vec16<T>::N;
  const int lane = threadIdx.x & 31;
  for (int64_t t = blockIdx.x * (int64_t)kCombWarps + (threadIdx.x >> 5); t < Tn;
       t += (int64_t)gridDim.x * kCombWarps) {
    int32_t rows[kMaxK];
    float ws[kMaxK], a[kMaxK], wo[kMaxK];
#pragma unroll
    for (int s = 0; s < kMaxK; ++s) {
      rows[s] = s < k ? row_of_slot[t * k + s] : -1;
      ws[s] = s < k ? w[t * k + s] : 0.0f;
      a[s] = 0.0f;
      // backward-only failure (reading X22): the expert's Backward request is lost, so its
      // cotangent row is zero (no dx contribution, no parameter gradient); dscore is unchanged
      wo[s] = ws[s];
      if (bwd_ok && s < k && rows[s] >= 0) {
        const int32_t e = sel[t * k + s];
        if (!((bwd_ok[e >> 5] >> (e & 31)) & 1u)) wo[s] = 0.0f;
      }
    }
    // a_s = <dy_t, out_row>, and dout_row = w_s dy_t in the same pass over dy_t
    for (int c = lane * V; c < D; c += 32 * V) {
      float g[V];
      uint4 u[kMaxK];
      const uint4 gu = ld_nc_v4(dy + t * D + c);
#pragma unroll
      for (int s = 0; s < kMaxK; ++s)
        if (s < k && rows[s] >= 0) u[s] = ld_nc_v4(out + (int64_t)rows[s] * D + c);
      unpack16(gu, g, (const T*)nullptr);
#pragma unroll
      for (int s = 0; s < kMaxK; ++s) {
        if (s >= k || rows[s] < 0) continue;
        float f[V], o[V];
        unpack16(u[s], f, (const T*)nullptr);
        float pr = 0.0f;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          pr = fmaf(g[i], f[i], pr);
          o[i] = wo[s] * g[i];
        }
        a[s] += pr;
        st_v4(dout + (int64_t)rows[s] * D + c, pack16(o, (const T*)nullptr));
      }
    }
    float abar = 0.0f;
#pragma unroll
    for (int s = 0; s < kMaxK; ++s) {
      if (s >= k) break;
      a[s] = warp_sum(a[s]);
      if (rows[s] >= 0) abar = fmaf(ws[s], a[s], abar);
    }
    float mine = 0.0f;
#pragma unroll
    for (int s = 0; s < kMaxK; ++s)
      if (s == lane && s < k && rows[s] >= 0) mine = ws[s] * (a[s] - abar);
    if (lane < k) dscore[t * k + lane] = mine;
  }
}

static unsigned grid_tokens(int64_t T) {
  int64_t b = ceil_div(T, kCombWarps);
  int64_t cap = (int64_t)num_sms() * 16;
  return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}

dmoe_status combine(const void* out, const int32_t* row_of_slot, const float* w,
                    const uint8_t* valid, int64_t T, int32_t D, int32_t k, dmoe_dtype dt, void* y,
                    cudaStream_t s) {
  if (T == 0) return DMOE_OK;
#define DMOE_COMB(KM)                                                                              \
  if (dt == DMOE_BF16)                                                                             \
    launch_pdl(k_combine<__nv_bfloat16, KM>, grid_tokens(T), kCombWarps * 32, 0, s, \
        (const __nv_bfloat16*)out, row_of_slot, w, valid, T, D, k, (__nv_bfloat16*)y);            \
  else                                                                                             \
    launch_pdl(k_combine<float, KM>, grid_tokens(T), kCombWarps * 32, 0, s, (const float*)out, row_of_slot, w, \
                                                                    valid, T, D, k, (float*)y);
  if (k <= 4) { DMOE_COMB(4) } else if (k <= 8) { DMOE_COMB(8) } else { DMOE_COMB(16) }
#undef DMOE_COMB
  return check_launch("combine");
}

dmoe_status combine_bwd(const void* dy, const void* out, const int32_t* row_of_slot,
                        const float* w, int64_t T, int32_t D, int32_t k, dmoe_dtype dt, void* dout,
                        float* dscore, const int32_t* sel, const uint32_t* bwd_ok, cudaStream_t s) {
  if (T == 0) return DMOE_OK;
#define DMOE_COMBB(KM)                                                                             \
  if (dt == DMOE_BF16)                                                                             \
    launch_pdl(k_combine_bwd<__nv_bfloat16, KM>, grid_tokens(T), kCombWarps * 32, 0, s, \
        (const __nv_bfloat16*)dy, (const __nv_bfloat16*)out, row_of_slot, w, T, D, k, sel, bwd_ok, \
        (__nv_bfloat16*)dout, dscore);                                                             \
  else                                                                                             \
    launch_pdl(k_combine_bwd<float, KM>, grid_tokens(T), kCombWarps * 32, 0, s, \
        (const float*)dy, (const float*)out, row_of_slot, w, T, D, k, sel, bwd_ok, (float*)dout, dscore);
  if (k <= 4) { DMOE_COMBB(4) } else if (k <= 8) { DMOE_COMBB(8) } else { DMOE_COMBB(16) }
#undef DMOE_COMBB
  return check_launch("combine_bwd");
}

}  // namespace dmoe
