// routing.cu — S2 prefix liveness + S3 SelectExperts (Alg. 1).
//
// Layout: G [T, d*M] fp32 row-major (one 4*d*M-byte row per token).  One thread per token
// (the search itself is beam.cuh): 128-token tiles of G staged in shared memory by coalesced
// 16-byte loads, the prefix-alive bitmaps built in shared memory by every CTA (grids up to 64K
// prefix bits; larger grids: one k_prefix_alive pass into the workspace).
#include "beam.cuh"
#include "common.cuh"

namespace dmoe {

// ----------------------------------------------------------------- prefix bitmaps
// PA_i[p] = OR of alive bits over the M^(d-1-i) experts below prefix p (reading X5).
// Level i bitmap starts at word offset wo_i = sum_{l<i} ceil(M^(l+1)/32); level d-1
// is the alive mask itself (copied).
__global__ void k_prefix_alive(const uint32_t* __restrict__ alive, int d, int M, int64_t E,
                               uint32_t* __restrict__ PA) {
  DMOE_PDL_ENTRY();
  int64_t wo = 0, n = M;
  for (int i = 0; i < d; ++i) {
    int64_t words = (n + 31) / 32;
    int64_t span = E / n;  // experts per level-i prefix
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
         w += (int64_t)gridDim.x * blockDim.x) {
      uint32_t v = 0;
      for (int b = 0; b < 32; ++b) {
        int64_t p = w * 32 + b;
        if (p >= n) break;
        int64_t e0 = p * span, e1 = e0 + span;
        bool any = false;
        // scan the alive words covering [e0, e1)
        for (int64_t e = e0; e < e1 && !any;) {
          uint32_t word = alive[e >> 5];
          int sh = (int)(e & 31);
          int64_t take = 32 - sh;
          if (take > e1 - e) take = e1 - e;
          uint32_t mask = (take == 32) ? 0xffffffffu : (((1u << take) - 1u) << sh);
          any = (word & mask) != 0;
          e += take;
        }
        if (any) v |= 1u << b;
      }
      PA[wo + w] = v;
    }
    wo += words;
    n *= M;
  }
}

constexpr int kSmemPAWords = 2048;  // prefix bitmaps up to 64K bits live in smem
#ifndef DMOE_BEAM_TOK
#define DMOE_BEAM_TOK 128
#endif
#ifndef DMOE_BEAM_MINB
#define DMOE_BEAM_MINB 2
#endif
constexpr int kBeamTok = DMOE_BEAM_TOK;        // tokens per CTA tile
constexpr int kBeamThreads = 2 * kBeamTok;     // threads per CTA: (token, level) list tasks, then a merge per token

// Thread per token (beam.cuh): the CTA stages its 128 tokens' G rows in shared memory with
// coalesced 16-byte loads (row pitch d*M + 1 floats: the threads' column reads hit 32 distinct
// banks), builds the prefix-alive bitmaps in shared memory (small grids) and notes whether every
// expert is alive (then FilterAlive is a no-op and the unmasked search runs).
template <int WMAX>
__global__ void __launch_bounds__(kBeamThreads, DMOE_BEAM_MINB)
k_beam_topk(const float* __restrict__ G, int64_t T, int d, int M, int k, int B,
            const uint32_t* __restrict__ PA_global, const uint32_t* __restrict__ alive, int pa_words,
            int32_t* __restrict__ sel, float* __restrict__ sel_score) {
  DMOE_PDL_ENTRY();
  extern __shared__ float smem_f[];
  const int dM = d * M, pitch = dM + 1;
  float* gtile = smem_f;                                                     // [kBeamTok][pitch]
  uint64_t* lists = reinterpret_cast<uint64_t*>(smem_f + ((kBeamTok * pitch + 1) & ~1));  // [tok][d][WMAX+1]
  uint32_t* pa_s = reinterpret_cast<uint32_t*>(lists + (size_t)kBeamTok * d * (WMAX + 1));
  int64_t E = 1;
  for (int i = 0; i < d; ++i) E *= M;
  int pa_off[4] = {0, 0, 0, 0};
  {
    int64_t wo = 0, n = M;
    for (int i = 0; i < d; ++i) { pa_off[i] = (int)wo; wo += (n + 31) / 32; n *= M; }
  }
  // all alive?  (then FilterAlive removes nothing: per-dimension lists + merge)
  bool dead = false;
  const int64_t aw = (E + 31) / 32;
  for (int64_t w = threadIdx.x; w < aw; w += blockDim.x) {
    const uint32_t want = (w == aw - 1 && (E & 31)) ? ((1u << (E & 31)) - 1u) : 0xffffffffu;
    dead |= (alive[w] & want) != want;
  }
  const bool masked = __syncthreads_or(dead);
  const uint32_t* PA = PA_global;
  if (masked && PA_global == nullptr) {
    prefix_alive_block(alive, d, M, E, pa_s);
    PA = pa_s;
  }
  for (int64_t t0 = (int64_t)blockIdx.x * kBeamTok; t0 < T; t0 += (int64_t)gridDim.x * kBeamTok) {
    const int nt = (int)((T - t0) < kBeamTok ? (T - t0) : kBeamTok);
    __syncthreads();  // previous tile's rows and lists consumed (and the bitmaps built)
    const float* src = G + t0 * dM;
    if ((dM & 3) == 0) {
      const int n4 = nt * dM / 4, q = dM / 4;
#pragma unroll 4
      for (int i = threadIdx.x; i < n4; i += kBeamThreads) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
        const int r = i / q, c = (i - r * q) * 4;
        float* dst = gtile + r * pitch + c;
        dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
      }
    } else {
      for (int i = threadIdx.x; i < nt * dM; i += kBeamThreads) {
        const int r = i / dM;
        gtile[r * pitch + (i - r * dM)] = __ldg(src + i);
      }
    }
    __syncthreads();
    if (masked) {
      if ((int)threadIdx.x < nt) {
        const int64_t t = t0 + threadIdx.x;
        beam_search_row<WMAX, true>(gtile + threadIdx.x * pitch, 1, d, M, k, B, PA, pa_off, sel + t * k,
                                    sel_score + t * k);
      }
      continue;
    }
    // per-dimension lists, (token, level) tasks over all threads
    for (int task = threadIdx.x; task < nt * d; task += kBeamThreads) {
      const int r = task / d, i = task - r * d;
      const int W = (i < d - 1) ? B : k;
      beam_dim_list<WMAX>(gtile + r * pitch + i * M, 1, M, W + 1 < M ? W + 1 : M,
                          lists + ((size_t)r * d + i) * (WMAX + 1));
    }
    __syncthreads();
    if ((int)threadIdx.x < nt) {
      const int64_t t = t0 + threadIdx.x;
      beam_merge_row<WMAX>(gtile + threadIdx.x * pitch, 1, d, M, k, B, lists + (size_t)threadIdx.x * d * (WMAX + 1),
                           sel + t * k, sel_score + t * k);
    }
  }
}

size_t prefix_words(int d, int M) {
  size_t w = 0, n = M;
  for (int i = 0; i < d; ++i) { w += (n + 31) / 32; n *= M; }
  return w;
}

template <int WMAX>
static dmoe_status launch_beam(const float* G, int64_t T, dmoe_grid g, const uint32_t* PA_global,
                               const uint32_t* alive, int pa_words, int32_t* sel, float* sel_score,
                               cudaStream_t s) {
  const int dM = g.d * g.M;
  size_t smem = (((size_t)kBeamTok * (dM + 1) + 1) & ~(size_t)1) * sizeof(float) +
                (size_t)kBeamTok * g.d * (WMAX + 1) * 8;
  if (PA_global == nullptr) smem += (size_t)pa_words * 4;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(k_beam_topk<WMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  int64_t blocks = ceil_div(T, kBeamTok);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  launch_pdl(k_beam_topk<WMAX>, (unsigned)blocks, kBeamThreads, smem, s, G, T, g.d, g.M, g.k, g.beam, PA_global,
                                                                   alive, pa_words, sel, sel_score);
  return check_launch("beam_topk");
}

dmoe_status beam_topk(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive_bits,
                      int32_t* sel, float* sel_score, uint32_t* PA, cudaStream_t s) {
  int64_t E = 1;
  for (int i = 0; i < g.d; ++i) E *= g.M;
  const int64_t words = (int64_t)prefix_words(g.d, g.M);
  const uint32_t* PA_global = nullptr;
  if (words > kSmemPAWords) {  // big grids: one pass into the workspace, read through L1/L2
    int blocks = (int)(((E + 31) / 32 + 255) / 256);
    if (blocks > 1024) blocks = 1024;
    launch_pdl(k_prefix_alive, blocks, 256, 0, s, alive_bits, g.d, g.M, E, PA);
    DMOE_TRY(check_launch("prefix_alive"));
    PA_global = PA;
  }
  if (T == 0) return DMOE_OK;
  int w = g.beam > g.k ? g.beam : g.k;
  if (w <= 4) return launch_beam<4>(G, T, g, PA_global, alive_bits, (int)words, sel, sel_score, s);
  if (w <= 8) return launch_beam<8>(G, T, g, PA_global, alive_bits, (int)words, sel, sel_score, s);
  if (w <= 16) return launch_beam<16>(G, T, g, PA_global, alive_bits, (int)words, sel, sel_score, s);
  return launch_beam<32>(G, T, g, PA_global, alive_bits, (int)words, sel, sel_score, s);
}

// Exact top-k over the alive experts (NEXT-3; the north star's "exact top-k ... restricted to a
// liveness mask"): every alive expert e of the token is scored with the same level-order fp32
// additions Alg. 1 uses, s = ((0 + g_0(u_0)) + g_1(u_1)) + ..., and the best k kept under X4's
// order.  With every expert alive this equals Alg. 1 (SURVEY §8(c) X3 proof); with dead experts
// Alg. 1 with B = k may miss the true top-k, this does not.  Thread per token over all E experts,
// 128 tokens per CTA with their G rows staged in shared memory.
template <int KMAX>
__global__ void __launch_bounds__(kBeamTok)
k_topk_exact(const float* __restrict__ G, int64_t T, int d, int M, int k, const uint32_t* __restrict__ alive,
             int32_t* __restrict__ sel, float* __restrict__ sel_score) {
  DMOE_PDL_ENTRY();
  extern __shared__ float smem_f[];
  const int dM = d * M, pitch = dM + 1;
  float* gtile = smem_f;
  int64_t E = 1;
  for (int i = 0; i < d; ++i) E *= M;
  for (int64_t t0 = (int64_t)blockIdx.x * kBeamTok; t0 < T; t0 += (int64_t)gridDim.x * kBeamTok) {
    const int nt = (int)((T - t0) < kBeamTok ? (T - t0) : kBeamTok);
    __syncthreads();
    for (int i = threadIdx.x; i < nt * dM; i += kBeamTok) {
      const int r = i / dM;
      gtile[r * pitch + (i - r * dM)] = __ldg(G + t0 * dM + i);
    }
    __syncthreads();
    if ((int)threadIdx.x >= nt) continue;
    const float* g = gtile + threadIdx.x * pitch;
    TopSet<KMAX> top;
    top.init(k);
    for (int64_t w = 0; w < (E + 31) / 32; ++w) {
      uint32_t bits = alive[w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const int64_t e = w * 32 + b;
        if (e >= E) break;
        float s = 0.0f;
        int64_t rem = e, div = E / M;
        for (int i = 0; i < d; ++i) {  // u_i = (e / M^(d-1-i)) mod M, levels in order (X1)
          const int u = (int)(rem / div);
          rem -= (int64_t)u * div;
          div /= M;
          s = s + g[i * M + u];
        }
        top.offer(s == 0.0f ? 0.0f : s, (uint32_t)e);
      }
    }
    top.sort();
    const int64_t t = t0 + threadIdx.x;
    for (int q = 0; q < k; ++q) {
      const uint64_t kq = beam_at_key(top, q);
      sel[t * k + q] = kq ? (int32_t)(0xffffffffu - (uint32_t)kq) : -1;
      sel_score[t * k + q] = kq ? beam_unord((uint32_t)(kq >> 32)) : -INFINITY;
    }
  }
}

dmoe_status topk_exact(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive, int32_t* sel, float* sel_score,
                       cudaStream_t s) {
  if (T == 0) return DMOE_OK;
  const size_t smem = (size_t)kBeamTok * (g.d * g.M + 1) * sizeof(float);
  int64_t blocks = ceil_div(T, kBeamTok);
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
#define DMOE_TKX(KM)                                                                                   \
  {                                                                                                    \
    static bool attr = false;                                                                          \
    if (!attr && smem > 48 * 1024) {                                                                   \
      cudaFuncSetAttribute(k_topk_exact<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
      attr = true;                                                                                     \
    }                                                                                                  \
    launch_pdl(k_topk_exact<KM>, (unsigned)blocks, kBeamTok, smem, s, G, T, g.d, g.M, g.k, alive, sel, sel_score); \
  }
  if (g.k <= 4) DMOE_TKX(4) else if (g.k <= 8) DMOE_TKX(8) else DMOE_TKX(16)
#undef DMOE_TKX
  return check_launch("topk_exact");
}

}  // namespace dmoe

