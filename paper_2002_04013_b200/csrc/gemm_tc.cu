// gemm_tc.cu — grouped bf16 GEMM engine on the 5th-generation tensor cores (sm_100a).
//
// The expert FFNs are the dense contraction of the DMoE layer: the runtime "aggregates
// requests into batches for better GPU utilization" (§3.3); here every
// expert's batch is one row segment [offsets[e], offsets[e+1]) of a dispatched matrix
// and all experts run in ONE persistent launch.
//
// Structure (one CTA per SM, 256 threads, warp-specialised):
//   warp 0   TMA producer: cp.async.bulk.tensor tiles (128B-swizzled) into a smem ring
//   warp 1   MMA issuer: one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//            (M=128, N=BN, K=16) with fp32 accumulation in TMEM; tcgen05.commit frees
//            smem slots and hands finished accumulators to the epilogue
//   warp 2   TMEM allocator (2 accumulator buffers x BN columns)
//   warps 4-7 epilogue: tcgen05.ld 32x32b -> registers -> bias / ReLU / ReLU-mask ->
//            bf16 (or fp32) 16-byte global stores, rows masked to the segment
// Tile scheduler: static round robin over a device-side tile count (no host sync):
//   ROWS  tiles = (expert row tile from the plan) x (N tile); K = D or H (fixed)
//   SEGK  tiles = expert x (M tile) x (N tile); K = the expert's rows (variable). The
//         last K block's rows past the segment are zeroed in smem before the MMA.
// Operands are K-major (rows of A in ROWS; torch Linear weights in the forward) or
// MN-major (weights in the backward-dx GEMMs, both operands of the weight-gradient
// GEMMs); the UMMA descriptors encode either, so no transposed copy is ever made.
#include <cuda.h>
#include <stdlib.h>

#include "gemm.cuh"

namespace dmoe {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;  // one 128-byte swizzle atom of bf16


// --------------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait suspends the waiting warp until the phase completes (or this many ns pass): waiting
// roles then stop spinning and leave the issue slots to the epilogue warps
constexpr uint32_t kMbarSuspendNs = 1000000;
#if defined(DMOE_EXPERIMENTS)
__device__ uint32_t g_mbar_hint = kMbarSuspendNs;
#define DMOE_MBAR_HINT g_mbar_hint
#else
#define DMOE_MBAR_HINT kMbarSuspendNs
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(DMOE_MBAR_HINT)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// L2 eviction policies for the bulk copies (createpolicy): streamed-once data evict-first,
// re-read tiles evict-last
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_h(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_h(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                              int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// ---- CTA pair (cta_group::2): two SMs of a cluster run one M = 256 MMA, each CTA holding its
// own 128 rows of A and half of B's N columns, each CTA's TMEM its own 128 accumulator rows
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the same shared-memory offset in CTA 0 of the cluster (the pair's leader), as a cluster address
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// TMA into this CTA's smem, completion counted on the leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_c, int c0, int c1,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_c), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_c, int c0, int c1,
                                                 int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_c), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// MMA completion signalled on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"((uint16_t)3)
               : "memory");
}

#define TMEM_LD32(taddr, r)                                                                         \
  asm volatile(                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),        \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),    \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), \
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), \
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                         \
      : "r"(taddr))

// UMMA shared-memory descriptor, 128-byte swizzle (layout type 2), sm_100 version 1.
//   K-major operand: rows of 128 B (64 bf16 of K), 8-row atoms 1024 B apart (SBO).
//   MN-major operand: K rows of 128 B (64 bf16 of M/N), 8-row groups 1024 B apart (SBO),
//                     64-element M/N chunks LBO bytes apart.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::f16, A/B bf16, D fp32, M=128, N=BN, majors
__host__ __device__ constexpr uint32_t make_idesc(int bn, bool a_mn, bool b_mn, int m = TC_BM) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn ? 1u : 0u) << 15)      // A major
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(bn >> 3) << 17)   // N >> 3
         | ((uint32_t)(m >> 4) << 24);   // M >> 4 (256: the CTA pair's cta_group::2 MMA)
}

#define TMEM_LD16(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15}, [%16];"                                                                        \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), \
        "=r"(r[14]), "=r"(r[15])                                                               \
      : "r"(taddr))

// pipeline timeline probe (dbg & 8): CTA 0 records %globaltimer at role events of its
// first 32 tiles: [role][tile] with role 0 = producer first TMA issued, 1 = producer last TMA
// issued, 2 = MMA got first stage, 3 = MMA committed last stage, 4 = epilogue got the
// accumulator, 5 = epilogue done
// [launch % 8][role][tile]; roles 0 prod first load, 1 prod last load, 2 mma after the first
// full-wait, 3 mma commit, 4 epilogue start, 5 epilogue done, 6 mma before the first full-wait,
// 7 mma before issuing the last K block; role 8: [0] kernel id (BN<<8 | SEGK<<4 | EPI), [1] grid
constexpr int TC_PROBE_ROLES = 9;
__device__ unsigned long long g_tc_probe[8][TC_PROBE_ROLES][32];
// DMOE_TC_DEBUG=64: clock64 cycles per pipeline phase summed over all CTAs, [launch % 8][counter]:
// 0 producer empty-wait, 1 producer loop, 2 mma tempty-wait, 3 mma full-wait, 4 mma zeroing,
// 5 mma issue+commit, 6 mma loop, 7 epi tfull-wait (warp 4), 8 epi store-read wait, 9 epi loop,
// 10 mma tiles, 11 CTAs, 12 mma issue without the commits
__device__ unsigned long long g_tc_wait[8][20];
#define WT_T0(v) const long long v = (DMOE_DBG(p) & 64) ? clock64() : 0
#define WT_ADD(acc_, v) do { if (DMOE_DBG(p) & 64) acc_ += clock64() - v; } while (0)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROBE(role, i) \
  do { if ((DMOE_DBG(p) & 8) && blockIdx.x == 0 && (i) < 32) g_tc_probe[p.slot][role][i] = gtimer(); } while (0)

// n / d for a divisor fixed per launch (tile decode): multiply-high with a magic number
// (round-up method, valid for n < 2^31, which tile indices are)
struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ void init(uint32_t d_) {
    d = d_ > 0 ? d_ : 1;
    s = 0;
    while ((1u << s) < d) ++s;
    m = (uint32_t)(((uint64_t)1 << 32) * (((uint64_t)1 << s) - d) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

// Weight-gradient tail boxes: the last K block of an expert with at most `rows` rows left (e.g.
// the 1-16 rows of a 65-80-row expert at transformer) is loaded with these `rows`-row boxes
// instead of the 64-row ones (the MMA reads only the 16-row slices holding segment rows).
// rows == 0: none.
struct TcTail {
  CUtensorMap a, b, a2, b2;
  int rows;
};

// ------------------------------------------------------------------------- kernel
struct TcParams {
  const int32_t* offsets;  // [E+1] or nullptr (single group of rows_single rows)
  const int32_t* plan;     // ROWS: [E+1] row-tile prefix (128-row tiles)
  const float* bias;
  float* colsum;             // SEGK: optional [E][Mdim] column sums of A (the bias gradient)
  const __nv_bfloat16* aux;  // ReLU mask source [rows, N]
  uint32_t* hmask;           // packed ReLU mask [N/32][hmask_ld] (bit c of word (w,row) = h[row, 32w+c] > 0):
                             // written by EPI_BIAS_RELU, read instead of aux by EPI_RELU_MASK
  int64_t hmask_ld;
  // SEGK: an optional second problem over the same segments (offsets), tiles after the first's
  // (its A / B / C tensor maps are the kernel's tmA2 / tmB2 / tmC2)
  int Mdim2, N2;          // Mdim2 == 0: one problem
  float* colsum2;
  void* C;
  int E, N, K, Mdim;
  int64_t rows_single;
  int max_ctas;   // grid cap (0: all SMs)
  int stages;     // M-major engine: smem ring depth (runtime, <= TC_MAX_STAGES)
  int table_len;  // M-major engine: per-expert smem table entries (0: tables stay in global)
  float sgd_lr;    // SEGK bf16: != 0 -> C (and colsum) are the parameters, updated in place:
                   // C -= lr * acc (the dW tile never reaches HBM), colsum -= lr * column sums
  int segk_gs;    // weight-gradient tile walk: CTAs per expert group (<= 1: strided walk; see the kernel)
  int slot;  // probe slot (launch ordinal % 8)
  int dbg;  // experiment switches (DMOE_EXPERIMENTS builds only, env DMOE_TC_DEBUG): 1 skip stores,
            // 2 skip TMEM loads, 4 skip MMAs, 8 timeline probe, 16 L2 prefetch cursor, 32 no L2 hints,
            // 64 phase cycle counters, 128 no first-tile weight prefetch
};

constexpr int TC_SMEM_MAX = 227 * 1024 - 2048;   // opt-in maximum less the kernels' static smem (<= 2 KB)
constexpr int TC_STAGE_ROW = 144;              // staging row pitch: 128 B of data + 16 B pad
constexpr int TC_STAGE_WARP = 5 * 1024;           // one warp's 32-row staging tile (1 KB aligned)
constexpr int TC_TABLE_E = 2048;                  // experts whose offsets/plan live in smem

constexpr int TC_MAX_STAGES = 8;
#ifndef DMOE_TAIL_ROWS
#define DMOE_TAIL_ROWS 32
#endif
constexpr int kTailRows = DMOE_TAIL_ROWS;  // weight-gradient tail boxes (TcTail)

template <int BN, bool SEGK = false, bool PAIR = false> struct TcCfg {
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  // epilogue warps: 8 (two column halves) for tiles >= 128 wide.  4 warps on 256-wide tiles buy
  // a 4th ring stage but the epilogue then trails the mainloop (measured: mnist FFN fwd 78 -> 92 us)
  // weight-gradient tiles (~1 K block each) are epilogue-paced: 256-wide ones get 16 epilogue warps
  // (one 64-column box each) so TMEM drains at twice the rate (measured: the 8-warp epilogue was
  // busy ~70% of the tile time while the MMA waited for accumulators)
  static constexpr int EPI_WARPS = (SEGK && BN == 256) ? 16 : ((BN >= 128) ? 8 : 4);
  static constexpr int EPI_COLS = BN / (EPI_WARPS / 4);   // columns per epilogue warp
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;       // 16 KB
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * TC_BK * 2;   // a pair CTA holds half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // multiple of 1 KB (BN % 8 == 0)
  // fixed smem without the per-expert tables (those are sized at launch: 2 x table_len ints)
  // weight-gradient tiles (~1 K block each): a 3rd accumulator (when TMEM has room) lets the
  // MMA run two tiles ahead, and each warp double-buffers its 4 KB store box so the TMA
  // engine's read of one box overlaps the staging of the next
  static constexpr int NACC = (SEGK && BN <= 128) ? 3 : 2;
  static constexpr int STG_WARP = SEGK ? (EPI_WARPS == 16 ? 4 * 1024 : 8 * 1024) : TC_STAGE_WARP;
  static constexpr int NBOX = SEGK ? STG_WARP / 4096 : 1;   // SEGK store boxes per warp (4 KB each)
  static constexpr int FIXED = 1024 /*align*/ + 1024 /*barriers*/ + EPI_WARPS * STG_WARP + BN * 4 * 2;
  static int stages_for(int table_len) {
    const int st = (TC_SMEM_MAX - FIXED - 2 * table_len * 4) / STAGE_BYTES;
    return st > TC_MAX_STAGES ? TC_MAX_STAGES : st;
  }
  static int smem_for(int table_len) { return stages_for(table_len) * STAGE_BYTES + FIXED + 2 * table_len * 4; }
  static constexpr int pow2cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }
  static constexpr int TMEM_COLS = pow2cols(NACC * BN);                 // NACC accumulators
  static_assert(TMEM_COLS <= 512, "TMEM");
};

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// bf16 h > 0  <=>  sign bit clear and not +0
__device__ __forceinline__ bool bf16_pos(uint32_t b) { return b != 0 && !(b & 0x8000u); }

template <int BN, bool SEGK, bool B_MN, int EPI, bool PAIR = false>
__global__ void __launch_bounds__(TcCfg<BN, SEGK, PAIR>::THREADS, 1)
k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
          const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC2, const TcParams p,
          const __grid_constant__ TcTail tail) {
  using Cfg = TcCfg<BN, SEGK, PAIR>;
  static_assert(!PAIR || (!SEGK && BN == 256), "CTA pairs: 256-wide row GEMM tiles only");
  constexpr int RT = PAIR ? 2 * TC_BM : TC_BM;   // rows per row tile (a pair: 128 per CTA)
  // Before waiting for the previous kernel (programmatic dependent launch: this CTA may already
  // sit on an SM the previous grid freed while its last CTAs finish): pull the expert weights of
  // this CTA's first tile into L2.  Weights are parameters no kernel of the step writes, and a
  // prefetch never changes what the loads after the wait see, so this needs no ordering.  The
  // tile's expert is guessed as its row tile (one 128-row tile per expert); a wrong guess only
  // warms another expert's weights.
  if (!SEGK && p.offsets && (DMOE_DBG(p) & 128) == 0 && threadIdx.x == 0) {
    const int nt = (p.N + BN - 1) / BN;
    const int rt = (int)blockIdx.x / nt, n0 = ((int)blockIdx.x % nt) * BN;
    const int e = rt < p.E ? rt : p.E - 1;
    const int nkb = p.K / TC_BK;
    const int npf = nkb < 8 ? nkb : 8;
    for (int kb = 0; kb < npf; ++kb) {
      if (B_MN) {
        for (int c = 0; c < BN / 64; ++c) tma_prefetch_3d(&tmB, n0 + 64 * c, kb * TC_BK, e);
      } else {
        tma_prefetch_3d(&tmB, kb * TC_BK, n0, e);
      }
    }
  }
  DMOE_PDL_ENTRY();
  constexpr int NACC = Cfg::NACC;
  const int S = p.stages;
  constexpr bool A_MN = SEGK;  // A is MN-major exactly for the weight-gradient GEMMs
  constexpr bool OUT_F32 = (EPI == EPI_F32_BIAS || EPI == EPI_F32);
  constexpr bool STG_SWZ = Cfg::STG_WARP < 32 * TC_STAGE_ROW;  // 4 KB staging boxes: swizzled 128 B rows
  constexpr int OUT_ES = OUT_F32 ? 4 : 2;
  constexpr int SUB = 128 / OUT_ES;  // columns per staged sub-tile (128 bytes per row)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + S * Cfg::STAGE_BYTES);
  uint64_t* empty = full + TC_MAX_STAGES;
  uint64_t* tfull = empty + TC_MAX_STAGES;
  uint64_t* tempty = tfull + 4;
  uint64_t* ready = tempty + 4;  // SEGK: stage fixed up (tail rows zeroed) for the MMA
  uint64_t* wload = ready + TC_MAX_STAGES;  // SGD: per epilogue warp x box, parameter box landed
  uint32_t* tmem_slot = (uint32_t*)(wload + 16);
  uint8_t* stage_base = smem + S * Cfg::STAGE_BYTES + 1024;   // 1 KB aligned (128B-swizzled TMA stores)
  float* bias_s = (float*)(stage_base + Cfg::EPI_WARPS * Cfg::STG_WARP);  // [2][BN]
  int32_t* off_s = (int32_t*)(bias_s + 2 * BN);                             // [table_len]
  int32_t* plan_s = off_s + p.table_len;                                    // [table_len]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- per-expert tables in smem (every role decodes every tile: keep it off the L2 path).
  // ROWS with plan == nullptr: the row-tile plan (exclusive prefix of ceil(m_e/128)) is built
  // here with a block scan instead of a separate launch.
  const int32_t* offs = p.offsets;
  const int32_t* plan = p.plan;
  __shared__ int32_t scan_sh[33];
  if (p.offsets && p.table_len > 0) {
    for (int i = threadIdx.x; i <= p.E; i += blockDim.x) {
      off_s[i] = p.offsets[i];
      if (!SEGK && p.plan) plan_s[i] = p.plan[i];
    }
    offs = off_s;
    plan = plan_s;
    if (!SEGK && !p.plan) {
      __syncthreads();
      const int nw = blockDim.x >> 5;
      int32_t carry = 0;
      for (int e0 = 0; e0 < p.E; e0 += blockDim.x) {
        const int e = e0 + threadIdx.x;
        const int32_t v = e < p.E ? (off_s[e + 1] - off_s[e] + RT - 1) / RT : 0;
        int32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) scan_sh[warp] = x;
        __syncthreads();
        if (warp == 0) {
          int32_t t = lane < nw ? scan_sh[lane] : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
          }
          if (lane < nw) scan_sh[lane] = t;
        }
        __syncthreads();
        if (e < p.E) plan_s[e] = carry + (warp > 0 ? scan_sh[warp - 1] : 0) + x - v;
        carry += scan_sh[nw - 1];
        __syncthreads();
      }
      if (threadIdx.x == 0) plan_s[p.E] = carry;
    }
    __syncthreads();
  }

  // ---- tile space (identical walk in every role)
  const int NT = (p.N + BN - 1) / BN;
  const int MT = SEGK ? p.Mdim / TC_BM : 0;
  const bool two = SEGK && p.Mdim2 > 0;
  const int NT2 = two ? (p.N2 + BN - 1) / BN : 1;
  const int MT2 = two ? p.Mdim2 / TC_BM : 1;
  const int total0 = SEGK ? p.E * MT * NT : 0;
  int total;
  if (SEGK) total = total0 + (two ? p.E * MT2 * NT2 : 0);
  else if (p.offsets) total = plan[p.E] * NT;
  else total = (int)((p.rows_single + RT - 1) / RT) * NT;

  // tile walk: every role strides the grid.  (A contiguous chunk of SEGK tiles per CTA, which
  // would let consecutive tiles share the expert's operand rows, measured 45% slower on the
  // transformer dW2: the 148 CTAs then stream 148 experts' rows at once instead of sharing one
  // expert's rows through L2.)
  // a CTA pair (cluster of 2) walks one tile sequence; rank r takes rows [128 r, 128 r + 128) of it
  const int prank = PAIR ? (int)cluster_rank() : 0;
  const bool leader = prank == 0;
  const int t_begin = PAIR ? (int)blockIdx.x >> 1 : (int)blockIdx.x, t_end = total;
  const int t_step = PAIR ? (int)gridDim.x >> 1 : (int)gridDim.x;
  // Weight-gradient walk: groups of GS CTAs share one expert's tiles (both problems, interleaved
  // over the group's CTAs) and the NG = grid / GS groups take experts round-robin, so only NG
  // experts' operand rows are live at a time however far the groups drift apart; the host picks
  // GS so that they fit in ~40 MB of L2 (TcParams::segk_gs).  The strided walk over the flat tile
  // space (GS = 1) let drifting CTAs spread over hundreds of experts and re-read the operands
  // from HBM (transformer: 46-48 GB per call instead of ~5; 17 GB grouped, 22% faster).
  const int T0e = SEGK ? MT * NT : 0, T1e = (SEGK && two) ? MT2 * NT2 : 0, Te = T0e + T1e;
  const int GS = (SEGK && p.segk_gs > 1 && p.segk_gs <= (int)gridDim.x) ? p.segk_gs : 1;
  const int NG = (int)gridDim.x / GS, g_id = (int)blockIdx.x / GS, g_rk = (int)blockIdx.x % GS;
  const int per = (Te + GS - 1) / GS > 0 ? (Te + GS - 1) / GS : 1;
  FastDiv fd_per;
  fd_per.init(per);
  // the v-th tile of this CTA's walk: -1 past its end, -2 a slot of the group's last round that
  // has no tile (every role skips it alike)
  auto seq = [&](int v) -> int {
    if (GS == 1) {
      const int t = t_begin + v * t_step;
      return t < t_end ? t : -1;
    }
    if (g_id >= NG) return -1;  // CTAs past the last whole group idle
    const int j = (int)fd_per.div((uint32_t)v), w = v - j * per;
    const int e = g_id + j * NG;
    if (e >= p.E) return -1;
    const int lt = g_rk + w * GS;
    if (lt >= Te) return -2;
    return lt < T0e ? e * T0e + lt : total0 + e * T1e + (lt - T0e);
  };
  FastDiv fd_e, fd_n, fd_e2, fd_n2;  // SEGK: tiles per expert, N tiles (both problems); ROWS: N tiles
  fd_e.init(SEGK ? MT * NT : 1);
  fd_n.init(NT);
  fd_e2.init(SEGK ? MT2 * NT2 : 1);
  fd_n2.init(NT2);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if ((DMOE_DBG(p) & 8) && blockIdx.x == 0) {
    const unsigned long long t_entry = gtimer();
    for (int i = threadIdx.x; i < TC_PROBE_ROLES * 32; i += blockDim.x) (&g_tc_probe[p.slot][0][0])[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      g_tc_probe[p.slot][8][0] = (unsigned long long)((BN << 8) | (SEGK << 4) | EPI);
      g_tc_probe[p.slot][8][1] = gridDim.x;
      g_tc_probe[p.slot][8][2] = t_entry;
    }
  }
  if (warp == 1 && lane == 0) {
    // SEGK: a stage is released by the MMA commit and by the fix-up warp (column sums)
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], SEGK ? 2 : 1); mbar_init(&ready[i], 1); }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], (PAIR ? 2 : 1) * Cfg::EPI_WARPS);  // a pair: both CTAs' epilogues drain
    }
    for (int i = 0; i < 16; ++i) mbar_init(&wload[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t tmem_cols = Cfg::TMEM_COLS;
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the peer's barriers exist before any remote arrival
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if ((DMOE_DBG(p) & 8) && blockIdx.x == 0 && threadIdx.x == 0) g_tc_probe[p.slot][8][3] = gtimer();

  // decode a tile -> (group e, row0, row_end, m0, n0, number of K blocks).  SEGK caches the
  // expert's segment bounds per thread (tiles of one expert are consecutive in the walk).
  int c_e = -1;
  int64_t c_r0 = 0, c_r1 = 0;
  auto decode = [&](int tile, int& e, int64_t& row0, int64_t& row_end, int& m0, int& n0, int& nkb) -> int {
    int prob = 0;
    if (SEGK) {
      int mt = MT, nt = NT;
      const FastDiv* fe = &fd_e;
      const FastDiv* fn = &fd_n;
      if (tile >= total0) { prob = 1; tile -= total0; mt = MT2; nt = NT2; fe = &fd_e2; fn = &fd_n2; }
      e = (int)fe->div((uint32_t)tile);
      const int rem = tile - e * mt * nt;
      const int mi = (int)fn->div((uint32_t)rem);
      m0 = mi * TC_BM;
      n0 = (rem - mi * nt) * BN;
      if (e != c_e) {
        c_e = e;
        c_r0 = offs[e];
        c_r1 = offs[e + 1];
      }
      row0 = c_r0;
      row_end = c_r1;
      nkb = (int)((row_end - row0 + TC_BK - 1) / TC_BK);
    } else {
      const int rt = (int)fd_n.div((uint32_t)tile);
      n0 = (tile - rt * NT) * BN;
      m0 = 0;
      if (p.offsets) {
        int lo = 0, hi = p.E;
        while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (plan[mid] <= rt) lo = mid; else hi = mid; }
        e = lo;
        row0 = offs[e] + (int64_t)(rt - plan[e]) * RT + (int64_t)prank * TC_BM;
        row_end = offs[e + 1];
      } else {
        e = 0;
        row0 = (int64_t)rt * RT + (int64_t)prank * TC_BM;
        row_end = p.rows_single;
      }
      nkb = p.K / TC_BK;
    }
    return prob;
  };

  if (warp == 0) {
    // ======================= TMA producer =======================
    // An L2 prefetch cursor runs PF k-blocks ahead of the loads over the same (tile, kb)
    // sequence, so the loads into the smem ring mostly hit L2 (weights stream from HBM once).
    if (lane == 0) {
      constexpr int PF = SEGK ? 4 : 16;
      int ptile = t_begin, pkb = 0, pe = 0, pm0 = 0, pn0 = 0, pnkb = 0;
      int64_t prow0 = 0, prow_end = 0;
      auto pnext_tile = [&]() {
        while (ptile < total) {
          decode(ptile, pe, prow0, prow_end, pm0, pn0, pnkb);
          if (pnkb > 0) return;
          ptile += t_step;
        }
      };
      auto prefetch_one = [&]() {
        if (ptile >= t_end || !(DMOE_DBG(p) & 16) || GS > 1) return;  // opt-in (DMOE_TC_DEBUG=16): measured slower
        if (SEGK) {
          const int kr = (int)(prow0 + pkb * TC_BK);
          tma_prefetch_2d(&tmA, pm0, kr);
          tma_prefetch_2d(&tmA, pm0 + 64, kr);
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) tma_prefetch_2d(&tmB, pn0 + 64 * c, kr);
        } else if (B_MN) {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) tma_prefetch_3d(&tmB, pn0 + 64 * c, pkb * TC_BK, pe);
        } else {
          tma_prefetch_3d(&tmB, pkb * TC_BK, pn0, pe);
        }
        if (++pkb == pnkb) {
          pkb = 0;
          ptile += t_step;
          pnext_tile();
        }
      };
      pnext_tile();
      for (int i = 0; i < PF; ++i) prefetch_one();
      // expert weights stream through once (evict first); token / activation tiles are re-read
      // across N tiles (evict last).  DMOE_TC_DEBUG=32 disables the hints.
      const uint64_t pol_stream = (DMOE_DBG(p) & 32) ? l2_policy_last() : l2_policy_first();
      const uint64_t pol_keep = l2_policy_last();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      long long w_empty = 0, w_loop = 0;
      WT_T0(t_loop);
      for (int v = 0, tile; (tile = seq(v)) != -1; ++v, ++it) {
        if (tile < 0) continue;
        int e, m0, n0, nkb;
        int64_t row0, row_end;
        const int prob = decode(tile, e, row0, row_end, m0, n0, nkb);
        (void)prob;
        for (int kb = 0; kb < nkb; ++kb) {
          WT_T0(t_e);
          mbar_wait(&empty[stage], phase ^ 1);
          WT_ADD(w_empty, t_e);
          if (kb == 0) PROBE(0, it);
          if (kb == nkb - 1) PROBE(1, it);
          prefetch_one();
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (PAIR) {
            // both CTAs' loads complete on the leader's barrier, which expects the pair's bytes
            if (leader) mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
            const uint32_t fb = leader_addr(&full[stage]);
            tma_load_2d_pair(sa, &tmA, fb, kb * TC_BK, (int)row0, pol_keep);
            const int nh = n0 + prank * (BN / 2);  // this CTA's half of the N tile
            if (B_MN) {
#pragma unroll
              for (int c = 0; c < BN / 128; ++c)
                tma_load_3d_pair(sb + c * 8192, &tmB, fb, nh + 64 * c, kb * TC_BK, e, pol_stream);
            } else {
              tma_load_3d_pair(sb, &tmB, fb, kb * TC_BK, nh, e, pol_stream);
            }
            if (++stage == S) { stage = 0; phase ^= 1; }
            continue;
          }
          if (SEGK && (DMOE_DBG(p) & 512)) {  // experiments: no operand loads (pipeline skeleton)
            mbar_expect_tx(&full[stage], 0);
            if (++stage == S) { stage = 0; phase ^= 1; }
            continue;
          }
          if (SEGK) {
            const int kr = (int)(row0 + kb * TC_BK);
            const bool tl = tail.rows > 0 && row_end - kr <= tail.rows;  // a short last K block
            mbar_expect_tx(&full[stage], tl ? (2 + BN / 64) * tail.rows * 128 : Cfg::STAGE_BYTES);
            const CUtensorMap* mA = tl ? (prob ? &tail.a2 : &tail.a) : (prob ? &tmA2 : &tmA);
            const CUtensorMap* mB = tl ? (prob ? &tail.b2 : &tail.b) : (prob ? &tmB2 : &tmB);
            // one 2D box per 64 columns (a 3D {64, rows, chunks} view taking a whole operand per
            // command measured no faster and read 64% more DRAM bytes: 19.0 vs 11.6 GB per call)
            tma_load_2d_h(sa, mA, &full[stage], m0, kr, pol_keep);
            tma_load_2d_h(sa + 8192, mA, &full[stage], m0 + 64, kr, pol_keep);
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d_h(sb + c * 8192, mB, &full[stage], n0 + 64 * c, kr, pol_keep);
          } else {
            mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
            tma_load_2d_h(sa, &tmA, &full[stage], kb * TC_BK, (int)row0, pol_keep);
            if (B_MN) {
#pragma unroll
              for (int c = 0; c < BN / 64; ++c)
                tma_load_3d_h(sb + c * 8192, &tmB, &full[stage], n0 + 64 * c, kb * TC_BK, e, pol_stream);
            } else {
              tma_load_3d_h(sb, &tmB, &full[stage], kb * TC_BK, n0, e, pol_stream);
            }
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
      WT_ADD(w_loop, t_loop);
      if (DMOE_DBG(p) & 64) {
        atomicAdd(&g_tc_wait[p.slot][0], (unsigned long long)w_empty);
        atomicAdd(&g_tc_wait[p.slot][1], (unsigned long long)w_loop);
        atomicAdd(&g_tc_wait[p.slot][11], 1ull);
      }
    }
  } else if (warp == 1 && (!PAIR || leader)) {
    // ======================= MMA issuer =======================
    // (a pair: the leader issues M = 256 MMAs over both CTAs' smem into both CTAs' TMEM)
    constexpr uint32_t idesc = make_idesc(BN, A_MN, B_MN, PAIR ? 2 * TC_BM : TC_BM);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int it = 0;
    long long w_te = 0, w_full = 0, w_zero = 0, w_issue = 0, w_loop = 0, n_tiles = 0, w_mmaonly = 0;
    WT_T0(t_loop);
    for (int v = 0, tile; (tile = seq(v)) != -1; ++v, ++it) {
      if (tile < 0) continue;
      int e, m0, n0, nkb;
      int64_t row0, row_end;
      decode(tile, e, row0, row_end, m0, n0, nkb);
      if (nkb == 0) continue;  // empty segment: the epilogue writes zeros without TMEM
      ++n_tiles;
      WT_T0(t_te);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      WT_ADD(w_te, t_te);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        if (kb == 0 && lane == 0) PROBE(6, it);
        WT_T0(t_f);
        mbar_wait(SEGK ? &ready[stage] : &full[stage], phase);
        WT_ADD(w_full, t_f);
        tc_fence_after();
        WT_T0(t_z);
        if (kb == 0 && lane == 0) PROBE(2, it);
        uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        // SEGK: the last K block issues only the 16-row MMA slices that hold segment rows (the
        // fix-up warp has zeroed the rest of the last slice)
        int nk16 = TC_BK / 16;
        if (SEGK && kb == nkb - 1) nk16 = (int)((row_end - row0 - (int64_t)kb * TC_BK + 15) >> 4);
        WT_ADD(w_zero, t_z);
        WT_T0(t_i);
        if (lane == 0) {
          if (kb == nkb - 1) PROBE(7, it);
          const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            if ((DMOE_DBG(p) & 4) || k >= nk16) break;
            const uint64_t ad = A_MN ? make_desc(a0 + k * 2048, 8192, 1024) : make_desc(a0 + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(b0 + k * 2048, 8192, 1024) : make_desc(b0 + k * 32, 16, 1024);
            if (PAIR) tc_mma_pair(tmem_d, ad, bd, idesc, (kb | k) != 0);
            else tc_mma(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          WT_ADD(w_mmaonly, t_i);
          if (PAIR) {
            tc_commit_pair(&empty[stage]);
            if (kb == nkb - 1) tc_commit_pair(&tfull[acc]);
          } else if (DMOE_DBG(p) & 4096) {  // experiments (with MMAs skipped): plain arrivals
            mbar_arrive(&empty[stage]);
            if (kb == nkb - 1) mbar_arrive(&tfull[acc]);
          } else {
            tc_commit(&empty[stage]);
            if (kb == nkb - 1) { tc_commit(&tfull[acc]); PROBE(3, it); }
          }
        }
        __syncwarp();
        WT_ADD(w_issue, t_i);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
    }
    WT_ADD(w_loop, t_loop);
    if ((DMOE_DBG(p) & 64) && lane == 0) {
      atomicAdd(&g_tc_wait[p.slot][2], (unsigned long long)w_te);
      atomicAdd(&g_tc_wait[p.slot][3], (unsigned long long)w_full);
      atomicAdd(&g_tc_wait[p.slot][4], (unsigned long long)w_zero);
      atomicAdd(&g_tc_wait[p.slot][5], (unsigned long long)w_issue);
      atomicAdd(&g_tc_wait[p.slot][6], (unsigned long long)w_loop);
      atomicAdd(&g_tc_wait[p.slot][10], (unsigned long long)n_tiles);
      atomicAdd(&g_tc_wait[p.slot][12], (unsigned long long)w_mmaonly);
    }
  } else if (SEGK && warp == 3) {
    // ======================= fix-up (SEGK) =======================
    // Between the TMA landing a stage and the MMA reading it: zero the rows past the segment
    // end inside the last 16-row MMA slice (other experts' rows or uninitialised capacity rows,
    // <= 15 lines of every operand chunk), then release the stage to the MMA (ready).  On the
    // n0 == 0 tiles also sum A's columns over the segment rows (the bias gradient: db = sum
    // of the rows of dout / dh), in row order in fp32, before releasing the stage (empty).
    // Lane l owns A columns m0 + 4l .. 4l+3: chunk l/16, 16-byte unit (l%16)/2, half l%2.
    int stage = 0;
    uint32_t phase = 0;
    const int cchunk = lane >> 4, cunit = (lane & 15) >> 1, chalf = lane & 1;
    long long w_fw = 0, w_fl = 0, w_fc = 0;
    WT_T0(t_fl);
    for (int v = 0, tile; (tile = seq(v)) != -1; ++v) {
      if (tile < 0) continue;
      int e, m0, n0, nkb;
      int64_t row0, row_end;
      const int prob = decode(tile, e, row0, row_end, m0, n0, nkb);
      float* const colsum = prob ? p.colsum2 : p.colsum;
      const int mdim = prob ? p.Mdim2 : p.Mdim;
      const bool sums = colsum && n0 == 0;
      float cs[4] = {0.f, 0.f, 0.f, 0.f};
      for (int kb = 0; kb < nkb; ++kb) {
        WT_T0(t_fw);
        mbar_wait(&full[stage], phase);
        WT_ADD(w_fw, t_fw);
        uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        const int64_t left = row_end - row0 - (int64_t)kb * TC_BK;
        const int valid = left < TC_BK ? (int)left : TC_BK;
        const int lines = ((valid + 15) & ~15) - valid;
        if (lines > 0) {
          // 128-byte lines per K row: A's 2 chunks then B's BN / 64, 8 KB apart from sa on (a line
          // is zeroed whole, so the 128-byte swizzle inside it does not matter); lane = (row % 4,
          // 16-byte piece)
          constexpr int nchunk = 2 + BN / 64;
          const uint32_t z0 = smem_u32(sa) + (uint32_t)valid * 128 + (lane & 7) * 16;
#pragma unroll
          for (int c = 0; c < nchunk; ++c)
            for (int r = lane >> 3; r < lines; r += 4) sts_v4(z0 + c * 8192 + r * 128, make_uint4(0, 0, 0, 0));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[stage]);
        WT_T0(t_fc);
        if (sums) {
          // 16 rows' loads in flight per batch (shared memory is busy with TMA / MMA / stores)
          const uint8_t* col = sa + cchunk * 8192 + chalf * 8;
          int r = 0;
          for (; r + 16 <= valid; r += 16) {
            uint2 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              v[j] = *reinterpret_cast<const uint2*>(col + (r + j) * 128 + ((cunit ^ (j & 7)) << 4));
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              cs[0] += bf16lo(v[j].x); cs[1] += bf16hi(v[j].x); cs[2] += bf16lo(v[j].y); cs[3] += bf16hi(v[j].y);
            }
          }
          for (; r < valid; ++r) {
            const uint2 v = *reinterpret_cast<const uint2*>(col + r * 128 + ((cunit ^ (r & 7)) << 4));
            cs[0] += bf16lo(v.x); cs[1] += bf16hi(v.x); cs[2] += bf16lo(v.y); cs[3] += bf16hi(v.y);
          }
        }
        __syncwarp();
        WT_ADD(w_fc, t_fc);
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      if (sums)
      {
        float4* dst = reinterpret_cast<float4*>(colsum + (int64_t)e * mdim + m0 + 4 * lane);
        if (p.sgd_lr != 0.0f) {  // bias update in place (this tile is the only writer of these columns)
          const float4 b = *dst;
          *dst = make_float4(b.x - p.sgd_lr * cs[0], b.y - p.sgd_lr * cs[1], b.z - p.sgd_lr * cs[2],
                             b.w - p.sgd_lr * cs[3]);
        } else {
          *dst = make_float4(cs[0], cs[1], cs[2], cs[3]);
        }
      }
    }
    WT_ADD(w_fl, t_fl);
    if ((DMOE_DBG(p) & 64) && lane == 0) {
      atomicAdd(&g_tc_wait[p.slot][13], (unsigned long long)w_fw);
      atomicAdd(&g_tc_wait[p.slot][14], (unsigned long long)w_fl);
      atomicAdd(&g_tc_wait[p.slot][15], (unsigned long long)w_fc);
    }
  } else if (warp >= 4) {
    // ======================= epilogue =======================
    // warp -> TMEM lane quadrant q (rows 32q..32q+31) and column range [c_beg, c_beg+EPI_COLS).
    // Each 128-byte-wide sub-tile goes TMEM -> registers -> (bias/ReLU/mask) -> padded smem
    // staging -> coalesced 16-byte stores, 4 full rows (512 B) per warp instruction.
    const int ew = warp - 4;
    const int q = warp & 3;
    const int c_beg = (ew >> 2) * Cfg::EPI_COLS;
    const uint64_t pol_out = (DMOE_DBG(p) & 32) ? l2_policy_last() : l2_policy_first();  // dW: written once
    uint8_t* const stg_warp = stage_base + ew * Cfg::STG_WARP;
    uint8_t* stg = stg_warp;
    int stg_buf = 0;  // SEGK: which of the warp's two 4 KB store boxes
    uint32_t wph[2] = {0u, 0u};  // SGD: phase of each box's load barrier
    int acc = 0;
    uint32_t acc_phase = 0;
    int bias_buf = 0;
    int it = 0;
    long long w_tf = 0, w_st = 0, w_loop = 0, w_ld = 0, w_pk = 0, w_is = 0;
    WT_T0(t_loop);
    for (int v = 0, tile; (tile = seq(v)) != -1; ++v, ++it) {
      if (tile < 0) continue;
      int e, m0, n0, nkb;
      int64_t row0, row_end;
      const int prob = decode(tile, e, row0, row_end, m0, n0, nkb);
      const CUtensorMap* mC = prob ? &tmC2 : &tmC;
      const int mdim = prob ? p.Mdim2 : p.Mdim;
      const bool has_acc = !(SEGK && nkb == 0);
      bool released = false;  // accumulator handed back early (after the last TMEM load)
      // stage this tile's bias slice (double-buffered across tiles; one named barrier)
      constexpr bool HAS_BIAS = (EPI == EPI_F32_BIAS || EPI == EPI_BIAS || EPI == EPI_BIAS_RELU);
      float* bias_t = bias_s + bias_buf * BN;
      if (HAS_BIAS) {
        for (int c = threadIdx.x - 128; c < BN; c += 32 * Cfg::EPI_WARPS)
          bias_t[c] = (n0 + c < p.N) ? p.bias[(int64_t)e * p.N + n0 + c] : 0.0f;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * Cfg::EPI_WARPS) : "memory");
        bias_buf ^= 1;
      }
      // rows of this warp's quadrant: global row (ROWS) or output row m (SEGK)
      const int64_t qrow0 = SEGK ? (int64_t)(m0 + q * 32) : row0 + q * 32;
      int64_t live_rows;
      if (SEGK) live_rows = 32;
      else {
        const int64_t left = row_end - qrow0;
        live_rows = left < 0 ? 0 : (left > 32 ? 32 : left);
      }
      const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      // ReLU-mask source (h) for this warp's 32 rows x EPI_COLS columns: issue the coalesced
      // loads before waiting for the accumulator so their latency hides behind the MMA
      constexpr int NSUB = (Cfg::EPI_COLS + SUB - 1) / SUB;
      uint4 hreg[EPI == EPI_RELU_MASK ? NSUB : 1][8];
      constexpr int NW = Cfg::EPI_COLS >= 32 ? Cfg::EPI_COLS / 32 : 1;  // packed mask words of this warp's columns
      uint32_t mword[EPI == EPI_RELU_MASK ? NW : 1];
      if (EPI == EPI_RELU_MASK && p.hmask) {
        // one coalesced 4-byte load per 32 columns: lane = row (the TMEM row layout)
#pragma unroll
        for (int w = 0; w < NW; ++w)
          mword[w] = lane < live_rows ? __ldg(p.hmask + (int64_t)((n0 + c_beg) / 32 + w) * p.hmask_ld + qrow0 + lane) : 0u;
      } else if (EPI == EPI_RELU_MASK) {
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), piece = lane & 7;
            const int cs = c_beg + sb * SUB;
            hreg[sb][i] = make_uint4(0, 0, 0, 0);
            if (r < live_rows && cs + piece * 8 < c_beg + Cfg::EPI_COLS)
              hreg[sb][i] = __ldg(reinterpret_cast<const uint4*>(p.aux + (qrow0 + r) * p.N + n0 + cs + piece * 8));
          }
      }
      // fused SGD (SEGK bf16): the parameter boxes this warp will update are loaded by TMA into
      // its two store boxes while the MMA still runs (the box doubles as load and store buffer)
      const bool sgd = SEGK && !OUT_F32 && p.sgd_lr != 0.0f;
      if (sgd) {
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // both boxes free
#pragma unroll
          for (int sb = 0; sb < NSUB && sb < Cfg::NBOX; ++sb) {
            const int bx = (stg_buf + sb) % Cfg::NBOX;
            mbar_expect_tx(&wload[ew * Cfg::NBOX + bx], 4096);
            tma_load_2d(stg_warp + bx * 4096, mC, &wload[ew * Cfg::NBOX + bx], n0 + c_beg + sb * SUB,
                        (int)((int64_t)e * mdim + qrow0));
          }
        }
        __syncwarp();
      }
      if (has_acc) {
        WT_T0(t_tf);
        mbar_wait(&tfull[acc], acc_phase);
        WT_ADD(w_tf, t_tf);
        tc_fence_after();
      }
      if (ew == 0 && lane == 0) PROBE(4, it);
#pragma unroll
      for (int sb = 0; sb < NSUB; ++sb) {
        const int cs = c_beg + sb * SUB;
        const int ncols = (c_beg + Cfg::EPI_COLS - cs) < SUB ? (c_beg + Cfg::EPI_COLS - cs) : SUB;  // multiple of 16
        uint32_t hmask[SUB / 32] = {};
        if (EPI == EPI_RELU_MASK && p.hmask) {
#pragma unroll
          for (int w = 0; w < SUB / 32; ++w) hmask[w] = mword[sb * (SUB / 32) + w];
        } else if (EPI == EPI_RELU_MASK) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), piece = lane & 7;
            sts_v4(smem_u32(stg) + r * TC_STAGE_ROW + piece * 16, hreg[sb][i]);
          }
          __syncwarp();
          // this lane's row: one bit per column, 1 = h > 0
#pragma unroll
          for (int piece = 0; piece < 8; ++piece) {
            const uint4 hv = lds_v4(smem_u32(stg) + lane * TC_STAGE_ROW + piece * 16);
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int col = piece * 8 + 2 * i;
              if (bf16_pos(hw[i] & 0xFFFFu)) hmask[col >> 5] |= 1u << (col & 31);
              if (bf16_pos(hw[i] >> 16)) hmask[(col + 1) >> 5] |= 1u << ((col + 1) & 31);
            }
          }
          __syncwarp();
        }
        if (SEGK && !OUT_F32) {
          // this box was last stored two boxes ago: at most the newest store may still be reading
          stg = stg_warp + stg_buf * 4096;
          WT_T0(t_st);
          if (sgd) {
            mbar_wait(&wload[ew * Cfg::NBOX + stg_buf], wph[stg_buf]);  // the parameter box has landed
            wph[stg_buf] ^= 1u;
          } else if (lane == 0) {
            if (Cfg::NBOX == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          }
          __syncwarp();
          WT_ADD(w_st, t_st);
        }
        // TMEM -> registers -> epilogue math -> staging (row = lane).  The whole sub-tile's
        // columns are loaded with back-to-back tcgen05.ld and ONE wait (a wait per 16 columns
        // left the epilogue warps latency-bound on TMEM: the weight-gradient tiles, ~1 K block
        // each, are epilogue-paced)
        uint32_t mw_lo = 0;  // EPI_BIAS_RELU: packed-mask bits of the first 16 columns of a word
        (void)mw_lo;
        uint32_t racc[SUB];
        const bool tld = has_acc && !(DMOE_DBG(p) & 2);
        WT_T0(t_ld);
        if (tld) {
#pragma unroll
          for (int c16 = 0; c16 < SUB; c16 += 16) {
            if (c16 < ncols) {
              uint32_t* rp = racc + c16;
              TMEM_LD16(tq + cs + c16, rp);
            }
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (sb == NSUB - 1) {
            // the tile's last columns are in registers: hand the accumulator back to the MMA now,
            // before the staging and stores (the MMA of the tile after next needs it)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (PAIR) mbar_arrive_cluster(leader_addr(&tempty[acc]));
              else mbar_arrive(&tempty[acc]);
            }
            released = true;
          }
        }
        else {
#pragma unroll
          for (int j = 0; j < SUB; ++j) racc[j] = 0u;  // empty segment (or an experiment): zeros
        }
        WT_ADD(w_ld, t_ld);
        WT_T0(t_pk);
#pragma unroll
        for (int c16 = 0; c16 < SUB; c16 += 16) {
          if (c16 >= ncols) break;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(racc[c16 + j]);
          if (HAS_BIAS) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += bias_t[cs + c16 + j];
          }
          if (EPI == EPI_BIAS_RELU) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.0f);
            if (p.hmask) {
              // bit = (stored bf16 h > 0), the decision the backward would take from h: with
              // round-to-nearest-even a non-negative fp32 v rounds to a nonzero bf16 iff
              // v > 2^-134 (half the smallest bf16 subnormal; no flush-to-zero in this build)
              uint32_t bits = 0;
#pragma unroll
              for (int j = 0; j < 16; ++j) bits |= (v[j] > 0x1p-134f ? 1u : 0u) << j;
              const int col = n0 + cs + c16;  // multiple of 16
              if ((col & 31) == 0) mw_lo = bits;
              else if (lane < live_rows && !(DMOE_DBG(p) & 1))
                p.hmask[(int64_t)(col >> 5) * p.hmask_ld + qrow0 + lane] = mw_lo | (bits << 16);
            }
          }
          if (EPI == EPI_RELU_MASK) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = c16 + j;
              if (!((hmask[col >> 5] >> (col & 31)) & 1u)) v[j] = 0.0f;
            }
          }
          if (SEGK && !OUT_F32) {
            // 128B-swizzled box row (the TMA store layout): 16-byte chunk q of row `lane`
            // sits at chunk q ^ (lane & 7)
#pragma unroll
            for (int j = 0; j < 16; j += 8) {
              const int q = (c16 + j) >> 3;
              const uint32_t slot = smem_u32(stg) + lane * 128 + ((q ^ (lane & 7)) << 4);
              if (sgd) {  // W <- W - lr * dW (fp32 arithmetic, one bf16 rounding: reading X21)
                const uint4 wq = lds_v4(slot);
                const uint32_t ww[4] = {wq.x, wq.y, wq.z, wq.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  v[j + 2 * i] = bf16lo(ww[i]) - p.sgd_lr * v[j + 2 * i];
                  v[j + 2 * i + 1] = bf16hi(ww[i]) - p.sgd_lr * v[j + 2 * i + 1];
                }
              }
              sts_v4(slot, make_uint4(pack_bf16x2(v[j], v[j + 1]), pack_bf16x2(v[j + 2], v[j + 3]),
                                      pack_bf16x2(v[j + 4], v[j + 5]), pack_bf16x2(v[j + 6], v[j + 7])));
            }
            continue;
          }
          // staging row `lane`, 16-byte piece pc: padded rows (144 B pitch), or 128 B rows with the
          // pieces XOR-swizzled by the row when the warp's box is 4 KB (16-warp weight-gradient tiles)
          if (OUT_F32) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              const int pc = (c16 * 4 + j * 4) >> 4;
              const uint32_t dst = smem_u32(stg) + (STG_SWZ ? lane * 128 + ((pc ^ (lane & 7)) << 4) : lane * TC_STAGE_ROW + pc * 16);
              sts_v4(dst, make_uint4(__float_as_uint(v[j]), __float_as_uint(v[j + 1]), __float_as_uint(v[j + 2]),
                                     __float_as_uint(v[j + 3])));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; j += 8) {
              const int pc = (c16 * 2 + j * 2) >> 4;
              const uint32_t dst = smem_u32(stg) + (STG_SWZ ? lane * 128 + ((pc ^ (lane & 7)) << 4) : lane * TC_STAGE_ROW + pc * 16);
              sts_v4(dst, make_uint4(pack_bf16x2(v[j], v[j + 1]), pack_bf16x2(v[j + 2], v[j + 3]),
                                     pack_bf16x2(v[j + 4], v[j + 5]), pack_bf16x2(v[j + 6], v[j + 7])));
            }
          }
        }
        WT_ADD(w_pk, t_pk);
        if (SEGK && !OUT_F32) {
          // full 32 x 64 box: one bulk tensor store (double-buffered box, see above)
          WT_T0(t_is);
          if (!(DMOE_DBG(p) & 1024)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && !(DMOE_DBG(p) & 1)) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                    mC),
                "r"(smem_u32(stg)), "r"(n0 + cs), "r"((int)((int64_t)e * mdim + qrow0)), "l"(pol_out)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          stg_buf = (stg_buf + 1) % Cfg::NBOX;
          __syncwarp();
          WT_ADD(w_is, t_is);
          continue;
        }
        __syncwarp();
        // staging -> global: lane (r = i*4 + lane/8, piece = lane%8) -> 4 full rows per instruction
        const int row_bytes = ncols * OUT_ES;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + (lane >> 3), piece = lane & 7;
          if (r < live_rows && piece * 16 < row_bytes && !(DMOE_DBG(p) & 1)) {
            const uint4 v = lds_v4(smem_u32(stg) + (STG_SWZ ? r * 128 + ((piece ^ (r & 7)) << 4) : r * TC_STAGE_ROW + piece * 16));
            uint8_t* gdst;
            if (SEGK)
              gdst = (uint8_t*)p.C + (((int64_t)e * p.Mdim + qrow0 + r) * p.N + n0 + cs) * OUT_ES + piece * 16;
            else
              gdst = (uint8_t*)p.C + ((qrow0 + r) * p.N + n0 + cs) * OUT_ES + piece * 16;
            *reinterpret_cast<uint4*>(gdst) = v;
          }
        }
        __syncwarp();
      }
      if (ew == 0 && lane == 0) PROBE(5, it);
      if (has_acc) {
        if (!released) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR) mbar_arrive_cluster(leader_addr(&tempty[acc]));
            else mbar_arrive(&tempty[acc]);
          }
        }
        if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
      }
    }
    WT_ADD(w_loop, t_loop);
    if ((DMOE_DBG(p) & 64) && ew == 0 && lane == 0) {
      atomicAdd(&g_tc_wait[p.slot][7], (unsigned long long)w_tf);
      atomicAdd(&g_tc_wait[p.slot][8], (unsigned long long)w_st);
      atomicAdd(&g_tc_wait[p.slot][9], (unsigned long long)w_loop);
      atomicAdd(&g_tc_wait[p.slot][16], (unsigned long long)w_ld);
      atomicAdd(&g_tc_wait[p.slot][17], (unsigned long long)w_pk);
      atomicAdd(&g_tc_wait[p.slot][18], (unsigned long long)w_is);
    }
  }

  if (SEGK && warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if ((DMOE_DBG(p) & 8) && blockIdx.x == 0 && warp == 4 && lane == 0) g_tc_probe[p.slot][8][4] = gtimer();
  tc_fence_before();
  __syncthreads();
  if ((DMOE_DBG(p) & 8) && blockIdx.x == 0 && threadIdx.x == 0) g_tc_probe[p.slot][8][5] = gtimer();
  if (PAIR) cluster_sync_all();  // the peer is done with our barriers and our TMEM
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}

// ----------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  }
  return fn;
}

// bf16 tensor map, dims innermost first; box {64, box1, 1...}; 128-byte swizzle
static dmoe_status make_map(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims,
                            uint32_t box1) {
  EncodeTiledFn fn = encode_fn();
  DMOE_REQUIRE(fn != nullptr, DMOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[3], gstride[2];
  cuuint32_t box[3] = {64, box1, 1}, estr[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) gdim[i] = dims[i];
  gstride[0] = dims[0] * 2;
  if (rank == 3) gstride[1] = dims[0] * dims[1] * 2;
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DMOE_REQUIRE(r == CUDA_SUCCESS, DMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DMOE_OK;
}

// Weight-gradient walk group size (TcParams::segk_gs): NG = grid / GS experts in flight, their
// operand rows (R_cap / E rows x (A + B columns) per problem) within ~40 MB of L2.  Measured
// (ncu, one box, A/B): transformer (1.3 MB per expert, GS = 4) 22.5 -> 18.0 ms and 47 -> 17 GB
// of DRAM reads; but with a few MB per expert (grid3d 5.2 MB, 1024-row experts 21 MB) large
// groups were slower than the strided walk (32.5 vs 34.8 ms, 6.3 vs 8.6 ms), so the grouped
// walk is used only for small per-expert operands (>= 16 groups) and never when half the grid's
// experts already fit (the strided walk then keeps L2 anyway).
static int segk_group(int64_t R_cap, int E, int64_t cols, int max_ctas) {
  const int grid = (max_ctas > 0 && max_ctas < num_sms()) ? max_ctas : num_sms();
  const double bytes_e = E > 0 ? (double)R_cap / E * (double)cols * 2.0 : 0.0;
  if (bytes_e <= 0.0) return 1;
  const int ng = (int)(40e6 / bytes_e);
  if (ng < 16 || ng >= grid / 2) return 1;
  return grid / ng;
}

// N tile: 256 when it divides N, else 128; K-major B also takes any N = 16..256 in one tile
// (the gate, N = d*M) and MN-major B any multiple of 64 up to 256.
static int pick_bn(int N, bool b_mn) {
  static int force = -1;
  if (force < 0) {
    const char* e = dmoe_env("DMOE_TC_BN");  // experiment override: 128 / 256
    force = e ? atoi(e) : 0;
  }
  if ((force == 128 || force == 256) && N % force == 0) return force;
  if (N % 256 == 0) return 256;
  if (N % 128 == 0) return 128;
  if (N <= 256 && (b_mn ? N % 64 == 0 : N % 16 == 0)) return N;
  return 0;
}

// N tile of a grouped GEMM with `units` (row tiles or experts x M tiles) per N tile: 256 unless
// 128 balances the persistent grid markedly better (tiles per SM rounded up to whole waves)
static int pick_bn_balanced(int N, bool b_mn, int64_t units) {
  const int bn = pick_bn(N, b_mn);
  if (bn != 256 || dmoe_env("DMOE_TC_BN")) return bn;
  const int64_t sms = num_sms();
  auto eff = [&](int b) {
    const int64_t tiles = units * (N / b);
    const int64_t waves = (tiles + sms - 1) / sms;
    return (double)tiles / (double)(waves * sms);
  };
  return eff(128) > eff(256) + 0.08 ? 128 : 256;
}

int tc_plan_in_kernel_max() { return TC_TABLE_E; }
bool tc_rows_mmajor() { return true; }

// token rows per tile of the row GEMMs (the plan granularity)
// CTA pairs (cta_group::2, M = 256) for the grouped row GEMMs whose experts average >= 256 rows
// of capacity (the tensor-bound side of the ridge): each CTA loads half of the weight tile, so
// the L2 -> SM operand feed per MMA drops by a third
static bool rows_pair(const GemmRows& g) {
  static const bool off = dmoe_env("DMOE_TC_NOPAIR") != nullptr;  // A/B experiments
  return !off && g.offsets && g.epi != EPI_F32_BIAS && g.N % 256 == 0 && g.rows_cap >= (int64_t)2 * TC_BM * g.E;
}
int tc_rows_tile(const GemmRows& g) { return rows_pair(g) ? 2 * TC_BM : TC_BM; }

bool tc_rows_supported(const GemmRows& g) {
  if (g.K % TC_BK != 0 || g.K <= 0 || g.N % 16 != 0) return false;
  if (g.b_mn && g.N % 64 != 0) return false;
  if (pick_bn(g.N, g.b_mn) == 0) return false;
  if (g.epi == EPI_F32_BIAS && g.offsets != nullptr) return false;
  if (encode_fn() == nullptr) return false;
  return true;
}

bool tc_segk_supported(const GemmSegK& g) {
  return g.Mdim % TC_BM == 0 && g.N % 128 == 0 && encode_fn() != nullptr;
}
bool tc_segk_colsum_supported(const GemmSegK& g) { return tc_segk_supported(g); }

static int debug_flags() {
  static int f = -1;
  if (f < 0) {
    const char* e = dmoe_env("DMOE_TC_DEBUG");
    f = e ? atoi(e) : 0;
  }
  return f;
}
// the same flags for the weight-gradient (SEGK) launches only (their outputs feed nothing else)
static int debug_flags_segk() {
  static int f = -1;
  if (f < 0) {
    const char* e = dmoe_env("DMOE_TC_DEBUG_SEGK");
    f = e ? atoi(e) : 0;
  }
  return f;
}

template <int BN, bool SEGK, bool B_MN, int EPI, bool PAIR>
static dmoe_status launch_maps_p(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                                 const CUtensorMap& a2, const CUtensorMap& b2, const CUtensorMap& c2,
                                 const TcParams& p, int64_t max_tiles, cudaStream_t s,
                                 const TcTail* tail_in = nullptr) {
  TcTail tail;
  if (tail_in) tail = *tail_in;
  else { memset(&tail, 0, sizeof(tail)); }
  if (dmoe_env("DMOE_TC_NOTAIL")) tail.rows = 0;  // experiments: A/B of the tail boxes
  using Cfg = TcCfg<BN, SEGK, PAIR>;
  auto kern = k_tc_gemm<BN, SEGK, B_MN, EPI, PAIR>;
  const int table_len = (p.offsets && p.E <= TC_TABLE_E) ? ((p.E + 4) & ~3) : 0;
  const int smem = Cfg::smem_for(table_len);
  static int attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = smem;
  }
  int64_t ctas = (p.max_ctas > 0 && p.max_ctas < num_sms()) ? p.max_ctas : num_sms();
  int64_t grid = (PAIR ? 2 : 1) * max_tiles < ctas ? (PAIR ? 2 : 1) * max_tiles : ctas;
  if (PAIR) grid &= ~(int64_t)1;  // whole pairs
  if (grid < (PAIR ? 2 : 1)) grid = PAIR ? 2 : 1;
  TcParams pp = p;
  pp.dbg = debug_flags() | (SEGK ? debug_flags_segk() : 0);
#if defined(DMOE_EXPERIMENTS)
  static bool hint_set = false;
  if (!hint_set) {  // DMOE_MBAR_HINT=<ns>: the mbarrier try_wait suspend-time hint
    hint_set = true;
    if (const char* e = dmoe_env("DMOE_MBAR_HINT")) {
      const uint32_t v = (uint32_t)atoi(e);
      cudaMemcpyToSymbol(g_mbar_hint, &v, sizeof(v));
    }
  }
#endif
  pp.slot = (int)(__atomic_load_n(&g_counters[1], __ATOMIC_RELAXED) % 8);
  pp.stages = Cfg::stages_for(table_len);
  if (SEGK) {  // CTAs per expert group: NG = grid / GS experts' operands within ~40 MB of L2
    int gs = p.segk_gs;
    if (const char* e = dmoe_env("DMOE_SEGK_GS")) gs = atoi(e);  // experiments: A/B of the walk
    pp.segk_gs = gs;
  }
  if (const char* e = dmoe_env("DMOE_TC_STAGES")) {  // experiments: a shallower ring
    const int st = atoi(e);
    if (st >= 1 && st < pp.stages) pp.stages = st;
  }
  pp.table_len = table_len;
  if (PAIR)
    launch_pdl_cluster(kern, (unsigned)grid, Cfg::THREADS, smem, s, 2u, a, b, c, a2, b2, c2, pp, tail);
  else
    launch_pdl(kern, (unsigned)grid, Cfg::THREADS, smem, s, a, b, c, a2, b2, c2, pp, tail);
  __atomic_fetch_add(&g_counters[1], 1, __ATOMIC_RELAXED);
  return check_launch("tc_gemm");
}
template <int BN, bool SEGK, bool B_MN, int EPI>
static dmoe_status launch_maps(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                               const CUtensorMap& a2, const CUtensorMap& b2, const CUtensorMap& c2,
                               const TcParams& p, int64_t max_tiles, cudaStream_t s,
                               const TcTail* tail = nullptr) {
  return launch_maps_p<BN, SEGK, B_MN, EPI, false>(a, b, c, a2, b2, c2, p, max_tiles, s, tail);
}
template <int BN, bool SEGK, bool B_MN, int EPI>
static dmoe_status launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const TcParams& p,
                          int64_t max_tiles, cudaStream_t s, const TcTail* tail = nullptr) {
  return launch_maps<BN, SEGK, B_MN, EPI>(a, b, c, a, b, c, p, max_tiles, s, tail);
}

template <int BN>
static dmoe_status rows_bn(const GemmRows& g, const CUtensorMap& a, const CUtensorMap& b, const TcParams& p,
                           int64_t tiles, cudaStream_t s) {
#define DMOE_TC_ROWS(BMN, E_) return launch<BN, false, BMN, E_>(a, b, a, p, tiles, s)
#define DMOE_TC_EPI(BMN)                                   \
  switch (g.epi) {                                         \
    case EPI_F32_BIAS: DMOE_TC_ROWS(BMN, EPI_F32_BIAS);    \
    case EPI_BIAS_RELU: DMOE_TC_ROWS(BMN, EPI_BIAS_RELU);  \
    case EPI_BIAS: DMOE_TC_ROWS(BMN, EPI_BIAS);            \
    case EPI_RELU_MASK: DMOE_TC_ROWS(BMN, EPI_RELU_MASK);  \
    default: DMOE_TC_ROWS(BMN, EPI_PLAIN);                 \
  }
  if constexpr (BN % 64 == 0) {
    if (g.b_mn) { DMOE_TC_EPI(true) }
  }
  DMOE_TC_EPI(false)
#undef DMOE_TC_EPI
#undef DMOE_TC_ROWS
}

static dmoe_status tc_gemm_rows_mk(const GemmRows& g, cudaStream_t s) {
  if (g.max_tiles <= 0) return DMOE_OK;
  // expected row tiles ~ one per expert at <= 128 rows/expert, else rows/128
  const int64_t units = g.offsets ? (g.rows_cap / TC_BM > g.E ? g.rows_cap / TC_BM : g.E) : g.max_tiles;
  const bool pair = rows_pair(g);
  const int BN = pair ? 256 : pick_bn_balanced(g.N, g.b_mn, units);
  // A: [rows_cap, K] K-major; rows past the extent are zero-filled by TMA, rows past a
  // segment produce accumulator rows the epilogue never stores.
  CUtensorMap ta, tb;
  uint64_t adims[2] = {(uint64_t)g.K, (uint64_t)(g.rows_cap > 0 ? g.rows_cap : 1)};
  DMOE_TRY(make_map(&ta, g.A, 2, adims, TC_BM));
  if (g.b_mn) {
    uint64_t bdims[3] = {(uint64_t)g.N, (uint64_t)g.K, (uint64_t)g.E};
    DMOE_TRY(make_map(&tb, g.B, 3, bdims, 64));
  } else {
    uint64_t bdims[3] = {(uint64_t)g.K, (uint64_t)g.N, (uint64_t)g.E};
    DMOE_TRY(make_map(&tb, g.B, 3, bdims, (uint32_t)(pair ? BN / 2 : BN)));   // a pair CTA: half the N rows
  }
  TcParams p{};
  p.offsets = g.offsets; p.plan = g.plan; p.bias = g.bias; p.aux = (const __nv_bfloat16*)g.aux;
  p.C = g.C; p.E = g.E; p.N = g.N; p.K = g.K; p.Mdim = 0; p.rows_single = g.rows_single;
  p.max_ctas = g.max_ctas;
  p.hmask = g.hmask; p.hmask_ld = g.hmask_ld;
  const int64_t tiles = g.max_tiles * ((g.N + BN - 1) / BN);
  if (pair) {
#define DMOE_TC_PAIR(BMN, E_) return launch_maps_p<256, false, BMN, E_, true>(ta, tb, ta, ta, tb, ta, p, tiles, s)
#define DMOE_TC_PEPI(BMN)                                  \
    switch (g.epi) {                                       \
      case EPI_BIAS_RELU: DMOE_TC_PAIR(BMN, EPI_BIAS_RELU); \
      case EPI_BIAS: DMOE_TC_PAIR(BMN, EPI_BIAS);           \
      case EPI_RELU_MASK: DMOE_TC_PAIR(BMN, EPI_RELU_MASK); \
      default: DMOE_TC_PAIR(BMN, EPI_PLAIN);                \
    }
    if (g.b_mn) { DMOE_TC_PEPI(true) }
    DMOE_TC_PEPI(false)
#undef DMOE_TC_PEPI
#undef DMOE_TC_PAIR
  }
  switch (BN) {
    case 256: return rows_bn<256>(g, ta, tb, p, tiles, s);
    case 128: return rows_bn<128>(g, ta, tb, p, tiles, s);
    case 64: return rows_bn<64>(g, ta, tb, p, tiles, s);
    case 192: return rows_bn<192>(g, ta, tb, p, tiles, s);
    case 32: return rows_bn<32>(g, ta, tb, p, tiles, s);
    case 48: return rows_bn<48>(g, ta, tb, p, tiles, s);
    case 96: return rows_bn<96>(g, ta, tb, p, tiles, s);
    case 16: return rows_bn<16>(g, ta, tb, p, tiles, s);
    default: return set_error(DMOE_ERR_UNSUPPORTED, "tc_gemm_rows: N=%d", g.N);
  }
}


dmoe_status tc_gemm_rows(const GemmRows& g, cudaStream_t s) { return tc_gemm_rows_mk(g, s); }

dmoe_status tc_gemm_segk(const GemmSegK& g, cudaStream_t s) {
  // weight-gradient tiles have ~1 K block each and are bound by shared-memory traffic (TMA
  // in, MMA operand reads, staging, TMA store reads): a 256-wide tile reads its operands at
  // 96 B/clk instead of 128 and halves the per-tile control work (measured: transformer dW
  // 11.7 -> 8.3 ms per GEMM before the fix-up warp took the tail zeroing off the MMA path)
  const int BN = pick_bn(g.N, true);
  CUtensorMap ta, tb;
  // K rows past a segment end (other experts' rows, or capacity rows past R) are zeroed
  // in smem before the MMA; rows past R_cap are zero-filled by TMA.
  const uint64_t rc = (uint64_t)(g.R_cap > 0 ? g.R_cap : 1);
  uint64_t adims[2] = {(uint64_t)g.Mdim, rc};
  uint64_t bdims[2] = {(uint64_t)g.N, rc};
  DMOE_TRY(make_map(&ta, g.A, 2, adims, 64));
  DMOE_TRY(make_map(&tb, g.B, 2, bdims, 64));
  // output dW [E][Mdim][N] as a 2D [E*Mdim, N] map, 64 x 32 boxes (bulk tensor stores)
  CUtensorMap tc;
  if (!g.out_f32) {
    uint64_t cdims[2] = {(uint64_t)g.N, (uint64_t)g.E * g.Mdim};
    DMOE_TRY(make_map(&tc, g.C, 2, cdims, 32));
  }
  TcParams p{};
  p.offsets = g.offsets; p.C = g.C; p.E = g.E; p.N = g.N; p.Mdim = g.Mdim; p.colsum = g.colsum;
  p.max_ctas = g.max_ctas;
  p.sgd_lr = g.out_f32 ? 0.0f : g.sgd_lr;
  p.segk_gs = g.out_f32 ? 1 : segk_group(g.R_cap, g.E, (int64_t)g.Mdim + g.N, g.max_ctas);
  const int64_t tiles = (int64_t)g.E * (g.Mdim / TC_BM) * (g.N / BN);
  if (g.out_f32) {  // fp32 output through the padded staging (the C map is unused)
    if (BN == 256) return launch<256, true, true, EPI_F32>(ta, tb, ta, p, tiles, s);
    return launch<128, true, true, EPI_F32>(ta, tb, ta, p, tiles, s);
  }
  TcTail tail;
  memset(&tail, 0, sizeof(tail));
  DMOE_TRY(make_map(&tail.a, g.A, 2, adims, kTailRows));
  DMOE_TRY(make_map(&tail.b, g.B, 2, bdims, kTailRows));
  tail.a2 = tail.a; tail.b2 = tail.b;
  tail.rows = (g.E > 0 && g.R_cap <= (int64_t)2 * TC_BK * g.E) ? kTailRows : 0;  // see tc_gemm_segk2
  if (BN == 256) return launch<256, true, true, EPI_PLAIN>(ta, tb, tc, p, tiles, s, &tail);
  return launch<128, true, true, EPI_PLAIN>(ta, tb, tc, p, tiles, s, &tail);
}

// two weight-gradient GEMMs over the same segments in one persistent launch (the expert
// backward's dW2 and dW1): one ramp / drain instead of two
bool tc_segk2_supported(const GemmSegK& a, const GemmSegK& b) {
  return tc_segk_supported(a) && tc_segk_supported(b) && a.offsets == b.offsets && a.E == b.E &&
         a.sgd_lr == b.sgd_lr &&
         pick_bn(a.N, true) == 256 && pick_bn(b.N, true) == 256 && a.max_ctas == b.max_ctas;
}
dmoe_status tc_gemm_segk2(const GemmSegK& g, const GemmSegK& h, cudaStream_t s) {
  CUtensorMap m[6];
  TcTail tail;
  memset(&tail, 0, sizeof(tail));
  // tail boxes pay off for experts of ~1 K block (transformer, same-box A/B: 18.0 -> 17.6 ms,
  // 16.5 -> 14 GB read) and not at 256 rows (grid3d 32.7 -> 33.7 ms)
  tail.rows = (g.E > 0 && g.R_cap <= (int64_t)2 * TC_BK * g.E) ? kTailRows : 0;
  const GemmSegK* gs[2] = {&g, &h};
  for (int i = 0; i < 2; ++i) {
    const GemmSegK& x = *gs[i];
    const uint64_t rc = (uint64_t)(x.R_cap > 0 ? x.R_cap : 1);
    {
      uint64_t adims[2] = {(uint64_t)x.Mdim, rc};
      uint64_t bdims[2] = {(uint64_t)x.N, rc};
      DMOE_TRY(make_map(i ? &tail.a2 : &tail.a, x.A, 2, adims, kTailRows));
      DMOE_TRY(make_map(i ? &tail.b2 : &tail.b, x.B, 2, bdims, kTailRows));
    }
    uint64_t cdims[2] = {(uint64_t)x.N, (uint64_t)x.E * x.Mdim};
    uint64_t adims[2] = {(uint64_t)x.Mdim, rc};
    uint64_t bdims[2] = {(uint64_t)x.N, rc};
    DMOE_TRY(make_map(&m[3 * i + 0], x.A, 2, adims, 64));
    DMOE_TRY(make_map(&m[3 * i + 1], x.B, 2, bdims, 64));
    DMOE_TRY(make_map(&m[3 * i + 2], x.C, 2, cdims, 32));
  }
  TcParams p{};
  p.offsets = g.offsets; p.C = g.C; p.E = g.E; p.N = g.N; p.Mdim = g.Mdim; p.colsum = g.colsum;
  p.N2 = h.N; p.Mdim2 = h.Mdim; p.colsum2 = h.colsum;
  p.max_ctas = g.max_ctas;
  p.sgd_lr = g.sgd_lr;
  p.segk_gs = segk_group(g.R_cap, g.E, (int64_t)g.Mdim + g.N + h.Mdim + h.N, g.max_ctas);
  const int64_t tiles = (int64_t)g.E * ((g.Mdim / TC_BM) * (g.N / 256) + (h.Mdim / TC_BM) * (h.N / 256));
  return launch_maps<256, true, true, EPI_PLAIN>(m[0], m[1], m[2], m[3], m[4], m[5], p, tiles, s, &tail);
}

}  // namespace dmoe

extern "C" int dmoe_debug_tc_wait(unsigned long long* host, int reset) {
  cudaDeviceSynchronize();
  int r = (int)cudaMemcpyFromSymbol(host, dmoe::g_tc_wait, sizeof(dmoe::g_tc_wait));
  if (reset) {
    static unsigned long long zero[8 * 20] = {};
    r |= (int)cudaMemcpyToSymbol(dmoe::g_tc_wait, zero, sizeof(zero));
  }
  return r;
}
extern "C" int dmoe_debug_tc_probe(unsigned long long* host, int n) {
  if (n > 8 * dmoe::TC_PROBE_ROLES * 32) n = 8 * dmoe::TC_PROBE_ROLES * 32;
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(host, dmoe::g_tc_probe, n * sizeof(unsigned long long));
}
