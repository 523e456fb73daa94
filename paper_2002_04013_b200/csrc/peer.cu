// peer.cu — expert-parallel exchange over NVLink peer memory (S11, fused form).
//
// The paper's trainer sends inputs to the experts' workers and collects their outputs
// (§3.1); on one B200 box the workers are GPUs behind NVSwitch, every one
// reachable by plain loads/stores to peer memory (CUDA IPC mappings).  Instead of
// all-to-all calls that need host-side split sizes, the dispatched rows are written straight
// into the owner's expert-major receive buffer and the expert outputs straight back into the
// source's dispatch-order buffer; completion is signalled by per-source epoch flags in the
// receiver's memory (st.release.sys / ld.acquire.sys).  Everything is device-side, so a
// whole multi-GPU layer step can be captured in one CUDA graph.
//
// Buffers are symmetric (same layout on every rank).  All pointer tables are device arrays of
// G peer pointers (entry `rank` is the local buffer).  Experts are owned by contiguous flat
// index: owner(e) = e / E_local.
//
// Ordering / reuse: every source signals phase p of step n with flag = 8n + p after its data
// writes; the receiver waits for all G flags >= 8n + p.  Buffers written in step n+1 were last
// read in step n before that rank's final phase signal, and the step ends with an all-reduce
// across ranks, so no write-after-read race exists across steps.
#include "common.cuh"

namespace dmoe {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// epoch[0] += 1 (start of a step)
__global__ void k_ep_begin(uint64_t* epoch) {
  DMOE_PDL_ENTRY(); epoch[0] += 1; }

// signal phase p to every peer: flags_j[rank] = 8*epoch + p (after all prior writes of this
// stream are complete: separate launch, then a system fence)
__global__ void k_ep_signal(uint64_t* const* peer_flags, int G, int rank, const uint64_t* epoch, int phase) {
  DMOE_PDL_ENTRY();
  __threadfence_system();
  const uint64_t v = epoch[0] * 8 + (uint64_t)phase;
  for (int j = threadIdx.x; j < G; j += blockDim.x) st_release_sys(peer_flags[j] + rank, v);
}

// wait until every source signalled phase p of this epoch; on timeout set err[0] |= 1 and go on
__global__ void k_ep_wait(const uint64_t* flags, int G, const uint64_t* epoch, int phase, uint64_t timeout_ns,
                          int32_t* err) {
  DMOE_PDL_ENTRY();
  const uint64_t want = epoch[0] * 8 + (uint64_t)phase;
  for (int s = threadIdx.x; s < G; s += blockDim.x) {
    const uint64_t t0 = now_ns();
    while (ld_acquire_sys(flags + s) < want) {
      if (now_ns() - t0 > timeout_ns) {
        atomicOr(err, 1);
        break;
      }
      __nanosleep(200);
    }
  }
}

// phase 0: broadcast this rank's per-expert counts into every peer's count matrix row `rank`
__global__ void k_ep_counts_push(const int32_t* __restrict__ counts, int E, int G, int rank,
                                 int32_t* const* peer_cnt) {
  DMOE_PDL_ENTRY();
  for (int j = 0; j < G; ++j) {
    int32_t* dst = peer_cnt[j] + (int64_t)rank * E;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) dst[e] = counts[e];
  }
}

// From the full count matrix cnt[s][e] (G x E, identical on every rank):
//   base[e]     (every global expert e): row in owner(e)'s expert-major buffer where THIS rank's
//               rows of e start = exp_off(e) + sum_{s < rank} cnt[s][e]
//   off_loc[el] (own experts, El+1): expert-major segment starts of this rank's receive buffer
//   src_off[s][el]: start of source s's rows of own expert el inside that source's dispatch order
//               (= sum_{e' < e0+el} cnt[s][e']) ; dst_off[s][el] = off_loc[el] + sum_{s'<s} cnt[s'][e]
// err[0] |= 2 if some owner would receive more than rin_cap rows.
__global__ void __launch_bounds__(1024)
k_ep_plan(const int32_t* __restrict__ cnt, int G, int rank, int E, int El, int64_t rin_cap,
          int32_t* __restrict__ base, int32_t* __restrict__ off_loc, int32_t* __restrict__ src_off,
          int32_t* __restrict__ dst_off, int32_t* __restrict__ err) {
  DMOE_PDL_ENTRY();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // per-expert totals and the exclusive scan within each owner's slice (one warp per owner)
  for (int j = warp; j < G; j += nw) {
    int32_t carry = 0;
    for (int i0 = 0; i0 < El; i0 += 32) {
      const int e = j * El + i0 + lane;
      int32_t tot = 0, mine = 0;
      if (i0 + lane < El)
        for (int s = 0; s < G; ++s) {
          const int32_t c = cnt[(int64_t)s * E + e];
          if (s < rank) mine += c;
          tot += c;
        }
      int32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const int32_t ex = carry + x - tot;
      if (i0 + lane < El) {
        base[e] = ex + mine;
        if (j == rank) {
          // clamped to the receive capacity: on overflow (err & 2) the expert GEMMs stay inside
          // the buffers (the step's results are then invalid and check() reports it)
          off_loc[i0 + lane] = ex < rin_cap ? ex : (int32_t)rin_cap;
          int32_t d = ex;
          for (int s = 0; s < G; ++s) {
            dst_off[s * El + i0 + lane] = d;
            d += cnt[(int64_t)s * E + e];
          }
        }
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) {
      if (j == rank) off_loc[El] = carry < rin_cap ? carry : (int32_t)rin_cap;
      if (carry > rin_cap) atomicOr(err, 2);
    }
  }
  // src_off[s][el]: exclusive scan of row s over all experts, read at this rank's experts
  for (int s = warp; s < G; s += nw) {
    int32_t carry = 0;
    for (int i0 = 0; i0 < E; i0 += 32) {
      const int e = i0 + lane;
      const int32_t v = e < E ? cnt[(int64_t)s * E + e] : 0;
      int32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (e < E && e / El == rank) src_off[s * El + (e - rank * El)] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

// Both row movers (err != 0, a plan overflow, skips all writes) run a warp per row over contiguous row chunks (rows are expert-major, so the
// row's expert advances linearly from one binary search per warp); a row is D/V 16-byte vectors,
// loaded 4 per lane before the first (NVLink peer) store.
template <typename T>
__device__ __forceinline__ void copy_row_warp(T* __restrict__ dst, const T* __restrict__ src, int vecs, int lane) {
  constexpr int V = Vec16<T>::N;
  for (int v = lane; v < vecs; v += 32 * 4) {
    uint4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v + 32 * u < vecs) a[u] = ld_nc_v4(src + (int64_t)(v + 32 * u) * V);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v + 32 * u < vecs) st_v4(dst + (int64_t)(v + 32 * u) * V, a[u]);
  }
}

// two rows at once (8 loads per lane in flight before the first store)
template <typename T>
__device__ __forceinline__ void copy_rows2_warp(T* __restrict__ d0, const T* __restrict__ s0, T* __restrict__ d1,
                                                const T* __restrict__ s1, int vecs, int lane) {
  constexpr int V = Vec16<T>::N;
  for (int v = lane; v < vecs; v += 32 * 4) {
    uint4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v + 32 * u < vecs) {
        a[u] = ld_nc_v4(s0 + (int64_t)(v + 32 * u) * V);
        b[u] = ld_nc_v4(s1 + (int64_t)(v + 32 * u) * V);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v + 32 * u < vecs) {
        st_v4(d0 + (int64_t)(v + 32 * u) * V, a[u]);
        st_v4(d1 + (int64_t)(v + 32 * u) * V, b[u]);
      }
  }
}

__device__ __forceinline__ int seg_of(const int32_t* __restrict__ offsets, int n, int64_t r) {
  int lo = 0, hi = n;  // offsets[lo] <= r < offsets[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (offsets[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// dispatch-order rows (expert-major over all E experts) -> owners' receive buffers: row r of
// expert e (owner e / El) goes to peer_dst[owner][base[e] + r - offsets[e]]; its source row is
// gidx[r] (the fused dispatch gather) or r.
template <typename T>
__global__ void __launch_bounds__(256)
k_ep_push_rows(const T* __restrict__ src, const int32_t* __restrict__ gidx, const int32_t* __restrict__ offsets,
               const int32_t* __restrict__ base, int E, int El, int32_t D, T* const* peer_dst,
               const int32_t* __restrict__ err) {
  DMOE_PDL_ENTRY();
  if (*err) return;
  constexpr int V = Vec16<T>::N;
  const int64_t R = offsets[E];
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t per = (R + nw - 1) / nw;
  const int64_t r0 = w * per, r1 = r0 + per < R ? r0 + per : R;
  if (r0 >= r1) return;
  int e = seg_of(offsets, E, r0);
  int64_t e_beg = offsets[e], e_end = offsets[e + 1];
  const int vecs = D / V;
  int64_t r = r0;
  for (; r + 1 < r1; r += 2) {
    while (r >= e_end) { ++e; e_beg = e_end; e_end = offsets[e + 1]; }
    T* d0 = peer_dst[e / El] + ((int64_t)base[e] + (r - e_beg)) * D;
    while (r + 1 >= e_end) { ++e; e_beg = e_end; e_end = offsets[e + 1]; }
    T* d1 = peer_dst[e / El] + ((int64_t)base[e] + (r + 1 - e_beg)) * D;
    const int64_t s0 = gidx ? (int64_t)gidx[r] : r, s1 = gidx ? (int64_t)gidx[r + 1] : r + 1;
    copy_rows2_warp(d0, src + s0 * D, d1, src + s1 * D, vecs, lane);
  }
  if (r < r1) {
    while (r >= e_end) { ++e; e_beg = e_end; e_end = offsets[e + 1]; }
    const int64_t srow = gidx ? (int64_t)gidx[r] : r;
    copy_row_warp(peer_dst[e / El] + ((int64_t)base[e] + (r - e_beg)) * D, src + srow * D, vecs, lane);
  }
}

// own experts' expert-major rows -> sources' dispatch-order buffers.  Local row q of own expert
// el from source s (dst_off[s][el] <= q < dst_off[s][el] + cnt[s][e]) goes to
// peer_dst[s][src_off[s][el] + q - dst_off[s][el]].
template <typename T>
__global__ void __launch_bounds__(256)
k_ep_return_rows(const T* __restrict__ src, const int32_t* __restrict__ cnt, const int32_t* __restrict__ off_loc,
                 const int32_t* __restrict__ src_off, const int32_t* __restrict__ dst_off, int G, int rank, int E,
                 int El, int32_t D, T* const* peer_dst, const int32_t* __restrict__ err) {
  DMOE_PDL_ENTRY();
  if (*err) return;
  constexpr int V = Vec16<T>::N;
  const int64_t R = off_loc[El];
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t per = (R + nw - 1) / nw;
  const int64_t q0 = w * per, q1 = q0 + per < R ? q0 + per : R;
  if (q0 >= q1) return;
  int el = seg_of(off_loc, El, q0);
  int64_t el_end = off_loc[el + 1];
  const int vecs = D / V;
  auto dst_of = [&](int64_t q) -> T* {
    while (q >= el_end) { ++el; el_end = off_loc[el + 1]; }
    const int e = rank * El + el;
    int sidx = 0;
    while (sidx + 1 < G && q >= dst_off[sidx * El + el] + cnt[(int64_t)sidx * E + e]) ++sidx;
    return peer_dst[sidx] + ((int64_t)src_off[sidx * El + el] + (q - dst_off[sidx * El + el])) * D;
  };
  int64_t q = q0;
  for (; q + 1 < q1; q += 2) {
    T* d0 = dst_of(q);
    T* d1 = dst_of(q + 1);
    copy_rows2_warp(d0, src + q * D, d1, src + (q + 1) * D, vecs, lane);
  }
  if (q < q1) copy_row_warp(dst_of(q), src + q * D, vecs, lane);
}

// ------------------------------------------------------------------ host entry points
static int rows_grid() { return num_sms() * 8; }

dmoe_status ep_begin(uint64_t* epoch, cudaStream_t s) {
  launch_pdl(k_ep_begin, 1, 1, 0, s, epoch);
  return check_launch("ep_begin");
}
dmoe_status ep_signal(uint64_t* const* peer_flags, int G, int rank, const uint64_t* epoch, int phase,
                      cudaStream_t s) {
  launch_pdl(k_ep_signal, 1, 32, 0, s, peer_flags, G, rank, epoch, phase);
  return check_launch("ep_signal");
}
dmoe_status ep_wait(const uint64_t* flags, int G, const uint64_t* epoch, int phase, uint64_t timeout_ns,
                    int32_t* err, cudaStream_t s) {
  launch_pdl(k_ep_wait, 1, 32, 0, s, flags, G, epoch, phase, timeout_ns, err);
  return check_launch("ep_wait");
}
dmoe_status ep_counts_push(const int32_t* counts, int E, int G, int rank, int32_t* const* peer_cnt,
                           cudaStream_t s) {
  launch_pdl(k_ep_counts_push, (unsigned)ceil_div(E, 256), 256, 0, s, counts, E, G, rank, peer_cnt);
  return check_launch("ep_counts_push");
}
dmoe_status ep_plan(const int32_t* cnt, int G, int rank, int E, int El, int64_t rin_cap, int32_t* base,
                    int32_t* off_loc, int32_t* src_off, int32_t* dst_off, int32_t* err, cudaStream_t s) {
  launch_pdl(k_ep_plan, 1, 1024, 0, s, cnt, G, rank, E, El, rin_cap, base, off_loc, src_off, dst_off, err);
  return check_launch("ep_plan");
}
dmoe_status ep_push_rows(const void* src, const int32_t* gidx, const int32_t* offsets, const int32_t* base,
                         int E, int El, int32_t D, dmoe_dtype dt, void* const* peer_dst, const int32_t* err,
                         cudaStream_t s) {
  if (dt == DMOE_BF16)
    launch_pdl(k_ep_push_rows<__nv_bfloat16>, rows_grid(), 256, 0, s, (const __nv_bfloat16*)src, gidx, offsets, base, E,
                                                             El, D, (__nv_bfloat16* const*)peer_dst, err);
  else
    launch_pdl(k_ep_push_rows<float>, rows_grid(), 256, 0, s, (const float*)src, gidx, offsets, base, E, El, D,
                                                     (float* const*)peer_dst, err);
  return check_launch("ep_push_rows");
}
dmoe_status ep_return_rows(const void* src, const int32_t* cnt, const int32_t* off_loc, const int32_t* src_off,
                           const int32_t* dst_off, int G, int rank, int E, int El, int32_t D, dmoe_dtype dt,
                           void* const* peer_dst, const int32_t* err, cudaStream_t s) {
  if (dt == DMOE_BF16)
    launch_pdl(k_ep_return_rows<__nv_bfloat16>, rows_grid(), 256, 0, s, (const __nv_bfloat16*)src, cnt, off_loc,
                                                               src_off, dst_off, G, rank, E, El, D,
                                                               (__nv_bfloat16* const*)peer_dst, err);
  else
    launch_pdl(k_ep_return_rows<float>, rows_grid(), 256, 0, s, (const float*)src, cnt, off_loc, src_off, dst_off, G,
                                                       rank, E, El, D, (float* const*)peer_dst, err);
  return check_launch("ep_return_rows");
}

}  // namespace dmoe
