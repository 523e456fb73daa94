// routing.cu — S2 prefix liveness + S3 SelectExperts (Alg. 1).
//
// Layout: G [T, d*M] fp32 row-major (one 4*d*M-byte row per token).  One warp per
// token; the row is staged in shared memory with coalesced 16-byte loads, every lane
// enumerates a strided subset of the level's candidates (beam entry b, column j),
// keeps a sorted register list of its best W under the total order of reading X4,
// and the warp merges the 32 lists with W rounds of a 64-bit shuffle argmax.
// The candidate key packs (order-preserving score bits << 32) | ~flat_index, so
// "larger key" == "higher score, then lower flat index".
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

__device__ __forceinline__ uint32_t ord_score(float s) {
  uint32_t u = __float_as_uint(s == 0.0f ? 0.0f : s);  // canonicalise -0.0 (reading X4)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_score(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}

template <int WMAX>
__device__ __forceinline__ void insert_sorted(uint64_t (&top)[WMAX], uint64_t key) {
#pragma unroll
  for (int i = WMAX - 1; i >= 0; --i) {
    uint64_t prev = (i > 0) ? top[i - 1] : ~0ull;
    if (key > top[i]) top[i] = (key > prev) ? prev : key;
  }
}

constexpr int kBeamWarps = 4;

// smem per warp: G row (dM floats) + beam (WMAX x {p, s})
constexpr int kSmemPAWords = 2048;  // prefix bitmaps up to 64K bits live in smem

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
__device__ void prefix_alive_cta(const uint32_t* __restrict__ alive, int d, int M, int64_t E, uint32_t* PA) {
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

template <int WMAX>
__global__ void __launch_bounds__(kBeamWarps * 32)
k_beam_topk(const float* __restrict__ G, int64_t T, int d, int M, int k, int B,
            const uint32_t* __restrict__ PA_global, const uint32_t* __restrict__ alive,
            int pa_words, int32_t* __restrict__ sel, float* __restrict__ sel_score) {
  DMOE_PDL_ENTRY();
  extern __shared__ float smem_f[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int dM = d * M;
  const uint32_t* PA = PA_global;
  if (PA_global == nullptr) {  // small grids: every CTA builds the bitmaps in smem
    uint32_t* pa_s = reinterpret_cast<uint32_t*>(smem_f + kBeamWarps * (dM + 2 * WMAX));
    int64_t E = 1;
    for (int i = 0; i < d; ++i) E *= M;
    prefix_alive_cta(alive, d, M, E, pa_s);
    __syncthreads();
    PA = pa_s;
  }
  float* grow = smem_f + warp * (dM + 2 * WMAX);
  int32_t* beam_p = reinterpret_cast<int32_t*>(grow + dM);
  float* beam_s = grow + dM + WMAX;

  for (int64_t t = blockIdx.x * (int64_t)kBeamWarps + warp; t < T;
       t += (int64_t)gridDim.x * kBeamWarps) {
    const float* g = G + t * dM;
    if ((dM & 3) == 0) {
      for (int c = lane * 4; c < dM; c += 128) {
        float4 v = __ldg(reinterpret_cast<const float4*>(g + c));
        grow[c] = v.x; grow[c + 1] = v.y; grow[c + 2] = v.z; grow[c + 3] = v.w;
      }
    } else {
      for (int c = lane; c < dM; c += 32) grow[c] = __ldg(g + c);
    }
    if (lane == 0) { beam_p[0] = 0; beam_s[0] = 0.0f; }
    __syncwarp();
    int nb = 1;
    int64_t wo = 0, npref = M;  // bit offset (words) and size of level-i prefix bitmap
    for (int i = 0; i < d; ++i) {
      const int W = (i < d - 1) ? B : k;
      uint64_t top[WMAX];
#pragma unroll
      for (int q = 0; q < WMAX; ++q) top[q] = 0ull;
      const int ncand = nb * M;
      const uint32_t* pa = PA + wo;
      for (int c = lane; c < ncand; c += 32) {
        int b = c / M, j = c - b * M;
        int64_t p = (int64_t)beam_p[b] * M + j;
        if (!((pa[p >> 5] >> (p & 31)) & 1u)) continue;  // FilterAlive
        float s = beam_s[b] + grow[i * M + j];
        uint64_t key = ((uint64_t)ord_score(s) << 32) | (uint64_t)(0xffffffffu - (uint32_t)p);
        insert_sorted<WMAX>(top, key);
      }
      __syncwarp();
      // merge: W rounds of warp argmax over the lanes' list heads
      int got = 0;
      for (int r = 0; r < W; ++r) {
        uint64_t best = top[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
          best = other > best ? other : best;
        }
        if (best == 0ull) break;  // fewer alive candidates than W (reading X6)
        if (top[0] == best) {      // unique owner pops its head
#pragma unroll
          for (int q = 0; q < WMAX - 1; ++q) top[q] = top[q + 1];
          top[WMAX - 1] = 0ull;
        }
        if (lane == 0) {
          beam_p[r] = (int32_t)(0xffffffffu - (uint32_t)(best & 0xffffffffu));
          beam_s[r] = unord_score((uint32_t)(best >> 32));
        }
        got = r + 1;
      }
      nb = got;
      __syncwarp();
      wo += (npref + 31) / 32;
      npref *= M;
    }
    for (int s = lane; s < k; s += 32) {
      sel[t * k + s] = s < nb ? beam_p[s] : -1;
      sel_score[t * k + s] = s < nb ? beam_s[s] : -INFINITY;
    }
    __syncwarp();
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
  size_t smem = (size_t)kBeamWarps * (dM + 2 * WMAX) * sizeof(float);
  if (PA_global == nullptr) smem += (size_t)pa_words * 4;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_beam_topk<WMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t blocks = ceil_div(T, kBeamWarps);
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  launch_pdl(k_beam_topk<WMAX>, (unsigned)blocks, kBeamWarps * 32, smem, s, G, T, g.d, g.M, g.k, g.beam, PA_global,
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

}  // namespace dmoe
