// api.cu — the C ABI of include/dmoe.h: argument validation, workspace carving and the
// launch sequence of each call.  Every step of the hot path runs in this library's
// kernels; there is no host compute and no fallback outside the GPU.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "gemm.cuh"

namespace dmoe {

static thread_local char g_err[512] = "";

dmoe_status set_error(dmoe_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

int64_t g_counters[4] = {0, 0, 0, 0};  // launches: all kernels, tcgen05 GEMMs, SIMT GEMMs, -

dmoe_status check_launch(const char* what) {
  __atomic_fetch_add(&g_counters[0], 1, __ATOMIC_RELAXED);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(DMOE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return DMOE_OK;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = kNumSMs;
  }
  return n;
}

// declared in the kernel files
dmoe_status beam_topk(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive_bits,
                      int32_t* sel, float* sel_score, uint32_t* PA, cudaStream_t s);
size_t prefix_words(int d, int M);
size_t dispatch_ws_bytes(int64_t T, int64_t E);
dmoe_status dispatch(const void* x, dmoe_dtype dt, int64_t T, int32_t D, int64_t E, int32_t k,
                     const int32_t* sel, const float* sel_score, const uint32_t* responded,
                     float* w, uint8_t* valid, int32_t* n_dropped, int32_t* counts,
                     int32_t* offsets, int32_t* row_of_slot, int32_t* token_of_row, void* xd,
                     int32_t* plan128, int32_t* plan64, void* ws, size_t ws_bytes, cudaStream_t s);
dmoe_status combine(const void* out, const int32_t* row_of_slot, const float* w,
                    const uint8_t* valid, int64_t T, int32_t D, int32_t k, dmoe_dtype dt, void* y,
                    cudaStream_t s);
dmoe_status combine_bwd(const void* dy, const void* out, const int32_t* row_of_slot,
                        const float* w, int64_t T, int32_t D, int32_t k, dmoe_dtype dt, void* dout,
                        float* dscore, const int32_t* sel, const uint32_t* bwd_ok, cudaStream_t s);
size_t gate_bwd_ws_bytes(int64_t T, int32_t D, int dM);
dmoe_status transpose(const void* src, int64_t rows, int64_t cols, dmoe_dtype dt, void* dst,
                      cudaStream_t s);
dmoe_status gate_bwd(const void* x, const void* Wg, const int32_t* sel, const float* dscore,
                     const void* dxd, const int32_t* row_of_slot, int64_t T, int32_t D, int d, int M,
                     int k, dmoe_dtype dt, void* dx, float* dWg, float* dbg, void* ws,
                     size_t ws_bytes, cudaStream_t s);

dmoe_status segment_offsets(const int32_t* offsets, int64_t E, int group, int32_t* seg, cudaStream_t s);
dmoe_status topk_exact(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive, int32_t* sel, float* sel_score,
                       cudaStream_t s);
dmoe_status ln_relu_fwd(const void* z, const int32_t* offsets, int E, int64_t R_cap, int H, float eps,
                        const float* g, const float* be, void* a, float* stats, cudaStream_t s);
dmoe_status ln_relu_bwd(const void* da, const void* z, const float* stats, const int32_t* offsets, int E, int H,
                        const float* g, const float* be, void* dz, float* dg, float* dbe, cudaStream_t s);
dmoe_status exchange_layout(const int32_t* counts, int G, int El, int32_t* offsets,
                            int32_t* src_of_dst, int64_t R_cap, void* ws, size_t ws_bytes, cudaStream_t s);
dmoe_status permute_rows(const void* src, const int32_t* idx, const int32_t* n_rows, int32_t D,
                         dmoe_dtype dt, int inverse, void* dst, cudaStream_t s);

dmoe_status ep_begin(uint64_t* epoch, cudaStream_t s);
dmoe_status ep_signal(uint64_t* const* peer_flags, int G, int rank, const uint64_t* epoch, int phase,
                      cudaStream_t s);
dmoe_status ep_wait(const uint64_t* flags, int G, const uint64_t* epoch, int phase, uint64_t timeout_ns,
                    int32_t* err, cudaStream_t s);
dmoe_status ep_counts_push(const int32_t* counts, int E, int G, int rank, int32_t* const* peer_cnt,
                           cudaStream_t s);
dmoe_status ep_plan(const int32_t* cnt, int G, int rank, int E, int El, int64_t rin_cap, int32_t* base,
                    int32_t* off_loc, int32_t* src_off, int32_t* dst_off, int32_t* err, cudaStream_t s);
dmoe_status ep_push_rows(const void* src, const int32_t* gidx, const int32_t* offsets, const int32_t* base,
                         int E, int El, int32_t D, dmoe_dtype dt, void* const* peer_dst, const int32_t* err,
                         cudaStream_t s);
dmoe_status ep_return_rows(const void* src, const int32_t* cnt, const int32_t* off_loc, const int32_t* src_off,
                           const int32_t* dst_off, int G, int rank, int E, int El, int32_t D, dmoe_dtype dt,
                           void* const* peer_dst, const int32_t* err, cudaStream_t s);

static dmoe_status check_grid(dmoe_grid* g, int64_t* E) {
  if (g->beam == 0) g->beam = g->k;
  DMOE_REQUIRE(g->d >= 1 && g->d <= 4, DMOE_ERR_SHAPE, "grid: d=%d outside [1,4]", g->d);
  DMOE_REQUIRE(g->M >= 1 && g->M <= 1024, DMOE_ERR_SHAPE, "grid: M=%d outside [1,1024]", g->M);
  DMOE_REQUIRE(g->d * g->M <= 256, DMOE_ERR_SHAPE, "grid: d*M=%d > 256", g->d * g->M);
  DMOE_REQUIRE(g->k >= 1 && g->k <= 16, DMOE_ERR_SHAPE, "grid: k=%d outside [1,16]", g->k);
  DMOE_REQUIRE(g->beam >= g->k && g->beam <= 32, DMOE_ERR_SHAPE, "grid: beam=%d outside [k,32]", g->beam);
  DMOE_REQUIRE((int64_t)g->beam * g->M <= 8192, DMOE_ERR_SHAPE, "grid: beam*M > 8192");
  int64_t e = 1;
  for (int i = 0; i < g->d; ++i) e *= g->M;
  DMOE_REQUIRE(e < (1ll << 31), DMOE_ERR_SHAPE, "grid: M^d >= 2^31");
  *E = e;
  return DMOE_OK;
}

static dmoe_status check_dt(dmoe_dtype dt, int32_t D) {
  DMOE_REQUIRE(dt == DMOE_F32 || dt == DMOE_BF16, DMOE_ERR_ARG, "dtype %d unknown", (int)dt);
  const int v = dt == DMOE_BF16 ? 8 : 4;
  DMOE_REQUIRE(D >= v && D % v == 0, DMOE_ERR_SHAPE, "D=%d must be a positive multiple of %d", D, v);
  return DMOE_OK;
}

#define NN(p) DMOE_REQUIRE((p) != nullptr, DMOE_ERR_ARG, "%s: null pointer `%s`", __func__, #p)

static dmoe_status rows_gemm(const GemmRows& g, dmoe_dtype dt, cudaStream_t s) {
  if (dt == DMOE_BF16 && tc_rows_supported(g)) return tc_gemm_rows(g, s);
  return simt_gemm_rows(g, dt, s);
}
static dmoe_status segk_gemm(const GemmSegK& g, dmoe_dtype dt, cudaStream_t s) {
  if (dt == DMOE_BF16 && tc_segk_supported(g)) return tc_gemm_segk(g, s);
  return simt_gemm_segk(g, dt, s);
}
constexpr int kPlanBM_SIMT = 64;

// The packed ReLU record is produced by the forward's h GEMM and consumed by the backward's dh
// GEMM only when both run on the M-major tcgen05 engine; both calls evaluate this same test.
static bool hmask_path(dmoe_dtype dt, int32_t D, int32_t H, int32_t E, int64_t R_cap) {
  static const bool off = dmoe_env("DMOE_NO_HMASK") != nullptr;  // A/B experiments
  if (off || dt != DMOE_BF16 || H % 32 != 0 || !tc_rows_mmajor()) return false;
  GemmRows f{}, b{};
  f.E = b.E = E; f.N = b.N = H; f.K = b.K = D; f.rows_cap = b.rows_cap = R_cap;
  f.offsets = b.offsets = reinterpret_cast<const int32_t*>(16);  // grouped form (value unused)
  f.b_mn = false; f.epi = EPI_BIAS_RELU;
  b.b_mn = true; b.epi = EPI_RELU_MASK;
  return tc_rows_supported(f) && tc_rows_supported(b);
}

static int num_sms_api() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}
// CTAs of the weight-gradient chain in the expert backward (0: no split, every GEMM takes all
// SMs and the chains only fill each other's tails).  DMOE_BWD_SEGK_CTAS overrides.
static int bwd_segk_ctas() {
  static int v = -1;
  if (v < 0) {
    const char* e = dmoe_env("DMOE_BWD_SEGK_CTAS");
    v = e ? atoi(e) : 0;
    if (v >= num_sms_api()) v = 0;
  }
  return v;
}

// ------------------------------------------------------- library side stream (fork / join)
// One non-blocking side stream + 3 events per (device, caller stream), created on first use
// (setup, not hot path) and kept for the process: two host threads calling on different
// streams never share a side stream or an event, so one call can never wait on another call's
// fork point.  fork_stream(s): the side stream waits for everything enqueued on s so far;
// join_stream: s waits for the side stream.  Event record / wait are captured into CUDA graphs
// as edges.  DMOE_SERIAL=1 (experiment builds) disables the fork.
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
};
static std::mutex g_side_mu;
static std::map<std::pair<int, cudaStream_t>, SideStream> g_side;

static SideStream* side_for(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_side_mu);
  SideStream& ss = g_side[{dev, s}];
  if (!ss.st) {
    if (cudaStreamCreateWithFlags(&ss.st, cudaStreamNonBlocking) != cudaSuccess) { ss.st = nullptr; return nullptr; }
    for (auto& e : ss.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return &ss;
}

static cudaStream_t fork_stream(cudaStream_t s, SideStream** out) {
  static const bool serial = dmoe_env("DMOE_SERIAL") != nullptr;
  *out = nullptr;
  if (serial) return nullptr;
  SideStream* ss = side_for(s);
  if (!ss) return nullptr;
  if (cudaEventRecord(ss->ev[0], s) != cudaSuccess || cudaStreamWaitEvent(ss->st, ss->ev[0], 0) != cudaSuccess)
    return nullptr;
  *out = ss;
  return ss->st;
}
static dmoe_status fork_point(cudaStream_t s, SideStream* ss) {
  if (cudaEventRecord(ss->ev[1], s) != cudaSuccess || cudaStreamWaitEvent(ss->st, ss->ev[1], 0) != cudaSuccess)
    return set_error(DMOE_ERR_CUDA, "fork_point: %s", cudaGetErrorString(cudaGetLastError()));
  return DMOE_OK;
}
static dmoe_status join_stream(cudaStream_t s, SideStream* ss) {
  if (cudaEventRecord(ss->ev[2], ss->st) != cudaSuccess || cudaStreamWaitEvent(s, ss->ev[2], 0) != cudaSuccess)
    return set_error(DMOE_ERR_CUDA, "join_stream: %s", cudaGetErrorString(cudaGetLastError()));
  return DMOE_OK;
}

// row-tile plans only for the engines the two GEMMs of a call will use
static dmoe_status plans_for(GemmRows& a, GemmRows& b, const int32_t* offsets, int E,
                             int32_t* plan_tc, int32_t* plan_simt, cudaStream_t s) {
  // the tcgen05 M-major engine builds its plan in smem for E <= tc_plan_in_kernel_max()
  if (E <= tc_plan_in_kernel_max()) {
    if (a.plan == plan_tc) a.plan = nullptr;
    if (b.plan == plan_tc) b.plan = nullptr;
  }
  // both on the tensor-core engine with different row tiles (one CTA-pair GEMM, one not): the
  // second gets its own plan in the SIMT plan's buffer (unused then)
  if (a.plan == plan_tc && b.plan == plan_tc && tc_rows_tile(a) != tc_rows_tile(b)) {
    DMOE_TRY(tile_plan(offsets, E, tc_rows_tile(a), plan_tc, s));
    b.plan = plan_simt;
    return tile_plan(offsets, E, tc_rows_tile(b), plan_simt, s);
  }
  const bool need_tc = a.plan == plan_tc || b.plan == plan_tc;
  const bool need_simt = a.plan == plan_simt || b.plan == plan_simt;
  if (need_tc) DMOE_TRY(tile_plan(offsets, E, tc_rows_tile(a.plan == plan_tc ? a : b), plan_tc, s));
  if (need_simt) DMOE_TRY(tile_plan(offsets, E, kPlanBM_SIMT, plan_simt, s));
  return DMOE_OK;
}

}  // namespace dmoe

using namespace dmoe;

namespace {
// one NVTX range per ABI call (SURVEY §5 tracing): free when no profiler is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#define DMOE_NVTX() NvtxRange dmoe_nvtx_range_(__func__)

extern "C" {

const char* dmoe_last_error(void) { return g_err; }

int32_t dmoe_launch_counters(int64_t* out, int32_t n) {
  for (int i = 0; i < n && i < 4; ++i) out[i] = __atomic_load_n(&g_counters[i], __ATOMIC_RELAXED);
  return 4;
}
int32_t dmoe_version(void) { return 1; }

size_t dmoe_workspace_bytes(int64_t T, int32_t D, int32_t H, dmoe_grid g, int32_t E_local,
                            int64_t R_cap) {
  int64_t E = 1;
  for (int i = 0; i < g.d; ++i) E *= g.M;
  // gate / beam (dmoe_gate_topk's unfused form keeps G in the workspace when the caller passes none)
  size_t beam = align_up(prefix_words(g.d, g.M) * 4, 256) + align_up((size_t)g.d * g.M * D * 2, 256) +
                (size_t)T * g.d * g.M * 4 + 1024;
  size_t disp = dispatch_ws_bytes(T, E);
  // expert FFN: plans, dh (fp32 capacity), and the recomputed h + ReLU record of the SGD call
  size_t ffn = 2 * align_up((size_t)(E_local + 1) * 4, 256) + align_up((size_t)R_cap * H * 4, 256) +
               align_up((size_t)R_cap * H * 2, 256) + align_up((size_t)((H + 31) / 32) * R_cap * 4, 256) + 1024;
  size_t gate = gate_bwd_ws_bytes(T, D, g.d * g.M);
  size_t exch = (size_t)8 * E + 1024;  // exchange tables (G * E_local <= E)
  size_t m = beam;
  if (exch > m) m = exch;
  if (disp > m) m = disp;
  if (ffn > m) m = ffn;
  if (gate > m) m = gate;
  return align_up(m, 4096);
}

// ------------------------------------------------------- finiteness check (debug switch)
// Off by default (the hot path does not check finiteness); dmoe_set_check_finite(1)
// (or DMOE_CHECK_FINITE in experiments builds) makes the calls below scan their floating-point
// outputs after the launch, synchronise the stream and return DMOE_ERR_NONFINITE on a NaN / Inf.
static int g_check_finite = -1;
static bool finite_on() {
  if (g_check_finite < 0) g_check_finite = dmoe_env("DMOE_CHECK_FINITE") ? 1 : 0;
  return g_check_finite == 1;
}
__global__ void k_nonfinite(const void* p, int bf16, int64_t n, int* flag) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = bf16 ? __bfloat162float(((const __nv_bfloat16*)p)[i]) : ((const float*)p)[i];
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}
static dmoe_status finite_check(const char* call, const char* what, const void* p, dmoe_dtype dt, int64_t n,
                                cudaStream_t s) {
  if (!finite_on() || p == nullptr || n <= 0) return DMOE_OK;
  static int* dflag[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return set_error(DMOE_ERR_CUDA, "%s: finite check", call);
  if (!dflag[dev] && cudaMalloc(&dflag[dev], sizeof(int)) != cudaSuccess)
    return set_error(DMOE_ERR_CUDA, "%s: finite check flag", call);
  int h = 0;
  if (cudaMemsetAsync(dflag[dev], 0, sizeof(int), s) != cudaSuccess) return set_error(DMOE_ERR_CUDA, "%s", call);
  const int64_t blocks = ceil_div(n, (int64_t)256) < 4096 ? ceil_div(n, (int64_t)256) : 4096;
  k_nonfinite<<<(unsigned)blocks, 256, 0, s>>>(p, dt == DMOE_BF16, n, dflag[dev]);
  if (cudaMemcpyAsync(&h, dflag[dev], sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return set_error(DMOE_ERR_CUDA, "%s: finite check: %s", call, cudaGetErrorString(cudaGetLastError()));
  if (h) return set_error(DMOE_ERR_NONFINITE, "%s: non-finite value in %s", call, what);
  return DMOE_OK;
}
// rows [0, offsets[E]) of a capacity buffer (reads offsets[E] back: the check synchronises anyway)
static int64_t rows_used(const int32_t* offsets, int32_t E, cudaStream_t s) {
  if (!finite_on()) return 0;
  int32_t r = 0;
  if (cudaMemcpyAsync(&r, offsets + E, sizeof(r), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return 0;
  return r;
}
extern "C" void dmoe_set_check_finite(int on) { g_check_finite = on ? 1 : 0; }

dmoe_status dmoe_gate_scores(const void* x, dmoe_dtype dt, int64_t T, int32_t D, const void* Wg,
                             const float* bg, dmoe_grid g, float* G, void* ws, size_t ws_bytes,
                             dmoe_stream_t stream) {
  DMOE_NVTX();
  int64_t E = 0;
  DMOE_TRY(check_grid(&g, &E));
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0, DMOE_ERR_SHAPE, "T < 0");
  if (T == 0) return DMOE_OK;
  NN(x); NN(Wg); NN(bg); NN(G); NN(ws);
  cudaStream_t s = (cudaStream_t)stream;
  const int dM = g.d * g.M;
  GemmRows r{};
  r.A = x; r.B = Wg; r.C = G; r.bias = bg; r.aux = nullptr;
  r.offsets = nullptr; r.plan = nullptr;
  r.E = 1; r.N = dM; r.K = D; r.rows_single = T; r.rows_cap = T;
  r.b_mn = false; r.epi = EPI_F32_BIAS;
  if (dt == DMOE_BF16 && tc_rows_supported(r)) {
    // tensor-core path: W_g^T [d*M, D] (K-major B operand) staged in the workspace
    DMOE_REQUIRE(ws_bytes >= (size_t)dM * D * 2, DMOE_ERR_ARG, "gate_scores: workspace too small");
    DMOE_TRY(transpose(Wg, D, dM, dt, ws, s));
    r.B = ws;
    r.max_tiles = ceil_div(T, tc_rows_tile(r));
    DMOE_TRY(tc_gemm_rows(r, s));
  } else {
    r.b_mn = true;
    r.max_tiles = ceil_div(T, kPlanBM_SIMT);
    DMOE_TRY(simt_gemm_rows(r, dt, s));
  }
  return finite_check("gate_scores", "G", G, DMOE_F32, T * dM, s);
}

dmoe_status dmoe_gate_topk(const void* x, dmoe_dtype dt, int64_t T, int32_t D, const void* Wg, const float* bg,
                           dmoe_grid g, const uint32_t* alive_bits, float* G, int32_t* sel, float* sel_score,
                           void* ws, size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  int64_t E = 0;
  DMOE_TRY(check_grid(&g, &E));
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0, DMOE_ERR_SHAPE, "T < 0");
  NN(alive_bits); NN(ws); NN(Wg); NN(bg);
  if (T == 0) return DMOE_OK;
  NN(x); NN(sel); NN(sel_score);
  cudaStream_t s = (cudaStream_t)stream;
  const int dM = g.d * g.M;
  // The gate GEMM (tcgen05, W_g^T staged in the workspace) writes G, the thread-per-token search
  // reads it back (mostly from L2).  Running Alg. 1 in the GEMM's epilogue instead was built and
  // measured slower (transformer 107-128 us vs 44 + 52 us; grid3d 413 vs 234 us): a 128-token
  // tile's search needs more warps than the GEMM kernel's 8 epilogue warps, so it could not hide
  // behind the next tile's mainloop.
  Carver cv(ws, ws_bytes);
  uint32_t* pa = cv.take<uint32_t>(prefix_words(g.d, g.M));
  void* wgt = cv.take<char>((size_t)dM * D * 2);
  float* Gw = G ? G : cv.take<float>((size_t)T * dM);
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "gate_topk: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  DMOE_TRY(dmoe_gate_scores(x, dt, T, D, Wg, bg, g, Gw, wgt, (size_t)dM * D * 2, stream));
  return beam_topk(Gw, T, g, alive_bits, sel, sel_score, pa, s);
}

dmoe_status dmoe_beam_topk(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive_bits,
                           int32_t* sel, float* sel_score, void* ws, size_t ws_bytes,
                           dmoe_stream_t stream) {
  DMOE_NVTX();
  int64_t E = 0;
  DMOE_TRY(check_grid(&g, &E));
  DMOE_REQUIRE(T >= 0, DMOE_ERR_SHAPE, "T < 0");
  NN(alive_bits); NN(ws);
  if (T > 0) { NN(G); NN(sel); NN(sel_score); }
  DMOE_REQUIRE(ws_bytes >= prefix_words(g.d, g.M) * 4, DMOE_ERR_ARG, "beam_topk: workspace too small");
  return beam_topk(G, T, g, alive_bits, sel, sel_score, (uint32_t*)ws, (cudaStream_t)stream);
}

dmoe_status dmoe_topk_exact(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive_bits, int32_t* sel,
                            float* sel_score, dmoe_stream_t stream) {
  DMOE_NVTX();
  int64_t E = 0;
  DMOE_TRY(check_grid(&g, &E));
  DMOE_REQUIRE(T >= 0, DMOE_ERR_SHAPE, "T < 0");
  DMOE_REQUIRE(E <= (1 << 20), DMOE_ERR_SHAPE, "topk_exact: E=%lld > 2^20 (a per-token scan of every expert)",
               (long long)E);
  NN(alive_bits);
  if (T > 0) { NN(G); NN(sel); NN(sel_score); }
  return topk_exact(G, T, g, alive_bits, sel, sel_score, (cudaStream_t)stream);
}

dmoe_status dmoe_dispatch(const void* x, dmoe_dtype dt, int64_t T, int32_t D, dmoe_grid g,
                          const int32_t* sel, const float* sel_score,
                          const uint32_t* responded_bits, float* w, uint8_t* valid,
                          int32_t* n_dropped, int32_t* counts, int32_t* offsets,
                          int32_t* row_of_slot, int32_t* token_of_row, void* xd, void* ws,
                          size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  int64_t E = 0;
  DMOE_TRY(check_grid(&g, &E));
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0, DMOE_ERR_SHAPE, "T < 0");
  NN(responded_bits); NN(n_dropped); NN(counts); NN(offsets); NN(ws);
  if (T > 0) { NN(x); NN(sel); NN(sel_score); NN(w); NN(valid); NN(row_of_slot); NN(token_of_row); }
  return dispatch(x, dt, T, D, E, g.k, sel, sel_score, responded_bits, w, valid, n_dropped, counts,
                  offsets, row_of_slot, token_of_row, xd, nullptr, nullptr, ws, ws_bytes,
                  (cudaStream_t)stream);
}

dmoe_status dmoe_expert_ffn_fwd(const void* xd, const int32_t* offsets, int32_t E_local,
                                int64_t R_cap, int32_t D, int32_t H, dmoe_dtype dt,
                                const void* W1, const float* b1, const void* W2, const float* b2,
                                void* h, uint32_t* hmask, void* out, void* ws, size_t ws_bytes,
                                dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  DMOE_TRY(check_dt(dt, H));
  DMOE_REQUIRE(E_local >= 1 && R_cap >= 0, DMOE_ERR_SHAPE, "E_local=%d R_cap=%lld", E_local, (long long)R_cap);
  NN(offsets); NN(W1); NN(b1); NN(W2); NN(b2); NN(ws);
  if (R_cap > 0) { NN(xd); NN(h); NN(out); }
  cudaStream_t s = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  int32_t* plan_tc = cv.take<int32_t>(E_local + 1);
  int32_t* plan_simt = cv.take<int32_t>(E_local + 1);
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "expert_ffn_fwd: workspace too small");
  GemmRows g1{};
  g1.A = xd; g1.B = W1; g1.C = h; g1.bias = b1; g1.offsets = offsets;
  g1.E = E_local; g1.N = H; g1.K = D; g1.rows_cap = R_cap; g1.b_mn = false; g1.epi = EPI_BIAS_RELU;
  GemmRows g2 = g1;
  g2.A = h; g2.B = W2; g2.C = out; g2.bias = b2; g2.N = D; g2.K = H; g2.epi = EPI_BIAS;
  if (hmask && hmask_path(dt, D, H, E_local, R_cap)) { g1.hmask = hmask; g1.hmask_ld = R_cap; }
  for (GemmRows* g : {&g1, &g2}) {
    const bool tc = dt == DMOE_BF16 && tc_rows_supported(*g);
    const int bm = tc ? tc_rows_tile(*g) : kPlanBM_SIMT;
    g->plan = tc ? plan_tc : plan_simt;
    g->max_tiles = ceil_div(R_cap, bm) + E_local;
  }
  DMOE_TRY(plans_for(g1, g2, offsets, E_local, plan_tc, plan_simt, s));
  DMOE_TRY(rows_gemm(g1, dt, s));
  DMOE_TRY(rows_gemm(g2, dt, s));
  return finite_check("expert_ffn_fwd", "out", out, dt, rows_used(offsets, E_local, s) * D, s);
}

dmoe_status dmoe_combine(const void* out, const int32_t* row_of_slot, const float* w,
                         const uint8_t* valid, int64_t T, int32_t D, int32_t k, dmoe_dtype dt,
                         void* y, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0 && k >= 1 && k <= 16, DMOE_ERR_SHAPE, "T=%lld k=%d", (long long)T, k);
  if (T > 0) { NN(row_of_slot); NN(w); NN(valid); NN(y); }
  DMOE_TRY(combine(out, row_of_slot, w, valid, T, D, k, dt, y, (cudaStream_t)stream));
  return finite_check("combine", "y", y, dt, T * D, (cudaStream_t)stream);
}

dmoe_status dmoe_combine_bwd(const void* dy, const void* out, const int32_t* row_of_slot,
                             const float* w, int64_t T, int32_t D, int32_t k, dmoe_dtype dt,
                             void* dout, float* dscore, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0 && k >= 1 && k <= 16, DMOE_ERR_SHAPE, "T=%lld k=%d", (long long)T, k);
  if (T > 0) { NN(dy); NN(row_of_slot); NN(w); NN(dscore); }
  DMOE_TRY(combine_bwd(dy, out, row_of_slot, w, T, D, k, dt, dout, dscore, nullptr, nullptr, (cudaStream_t)stream));
  return finite_check("combine_bwd", "dscore", dscore, DMOE_F32, T * k, (cudaStream_t)stream);
}

dmoe_status dmoe_combine_bwd_failures(const void* dy, const void* out, const int32_t* row_of_slot,
                                      const float* w, const int32_t* sel, const uint32_t* responded_bwd_bits,
                                      int64_t T, int32_t D, int32_t k, dmoe_dtype dt, void* dout, float* dscore,
                                      dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0 && k >= 1 && k <= 16, DMOE_ERR_SHAPE, "T=%lld k=%d", (long long)T, k);
  NN(responded_bwd_bits);
  if (T > 0) { NN(dy); NN(row_of_slot); NN(w); NN(dscore); NN(sel); }
  return combine_bwd(dy, out, row_of_slot, w, T, D, k, dt, dout, dscore, sel, responded_bwd_bits,
                     (cudaStream_t)stream);
}

static dmoe_status expert_ffn_bwd_impl(const void* xd, const void* h, const uint32_t* hmask, const void* dout,
                                const int32_t* offsets, int32_t E_local, int64_t R_cap,
                                int32_t D, int32_t H, dmoe_dtype dt, const void* W1,
                                const void* W2, void* dxd, void* dW1, float* db1, void* dW2,
                                float* db2, void* ws, size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  DMOE_TRY(check_dt(dt, H));
  DMOE_REQUIRE(E_local >= 1 && R_cap >= 0, DMOE_ERR_SHAPE, "E_local=%d R_cap=%lld", E_local, (long long)R_cap);
  NN(offsets); NN(W1); NN(W2); NN(dW1); NN(db1); NN(dW2); NN(db2); NN(ws);
  if (R_cap > 0) { NN(xd); NN(h); NN(dout); NN(dxd); }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t esz = dt == DMOE_BF16 ? 2 : 4;
  Carver cv(ws, ws_bytes);
  int32_t* plan_tc = cv.take<int32_t>(E_local + 1);
  int32_t* plan_simt = cv.take<int32_t>(E_local + 1);
  void* dh = cv.take<char>((size_t)(R_cap > 0 ? R_cap : 1) * H * esz);
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "expert_ffn_bwd: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  // dh = (dout W2_e) * 1[h > 0];  dxd = dh W1_e
  GemmRows g3{};
  g3.A = dout; g3.B = W2; g3.C = dh; g3.aux = h; g3.offsets = offsets;
  g3.E = E_local; g3.N = H; g3.K = D; g3.rows_cap = R_cap; g3.b_mn = true; g3.epi = EPI_RELU_MASK;
  if (hmask && hmask_path(dt, D, H, E_local, R_cap)) { g3.hmask = const_cast<uint32_t*>(hmask); g3.hmask_ld = R_cap; }
  GemmRows g4 = g3;
  g4.A = dh; g4.B = W1; g4.C = dxd; g4.aux = nullptr; g4.N = D; g4.K = H; g4.epi = EPI_PLAIN;
  g4.hmask = nullptr;
  for (GemmRows* g : {&g3, &g4}) {
    const bool tc = dt == DMOE_BF16 && tc_rows_supported(*g);
    const int bm = tc ? tc_rows_tile(*g) : kPlanBM_SIMT;
    g->plan = tc ? plan_tc : plan_simt;
    g->max_tiles = ceil_div(R_cap, bm) + E_local;
  }
  DMOE_TRY(plans_for(g3, g4, offsets, E_local, plan_tc, plan_simt, s));
  // dW2_e = dout^T h;  dW1_e = dh^T xd;  db2 / db1 = segment column sums of dout / dh (on the
  // tensor-core path: an extra ones-MMA inside the same GEMMs)
  GemmSegK g5{dout, h, dW2, offsets, E_local, D, H, R_cap, db2};
  GemmSegK g6{dh, xd, dW1, offsets, E_local, H, D, R_cap, db1};
  static const bool no_fuse = dmoe_env("DMOE_NO_COLSUM_FUSE") != nullptr;  // A/B experiments
  const bool fused = !no_fuse && dt == DMOE_BF16 && tc_segk_colsum_supported(g5) && tc_segk_colsum_supported(g6);
  if (!fused) g5.colsum = g6.colsum = nullptr;
  // Dependency graph: dh (g3) -> dxd (g4); dh -> dW1 (g6); dW2 (g5) independent.  g5 and g6 run
  // on a library stream forked/joined with events (graph-capturable), so each persistent GEMM's
  // tail is filled by the other chain's tiles instead of idling SMs.
  // Both weight-gradient GEMMs in one persistent launch (one ramp / drain) once dh exists, on a
  // forked library stream next to the dxd GEMM.  DMOE_SEGK_SPLIT=1: the two-launch form below.
  static const bool segk_split = dmoe_env("DMOE_SEGK_SPLIT") != nullptr;
  if (!segk_split && fused && tc_segk2_supported(g5, g6)) {
    const int seg_ctas = bwd_segk_ctas();  // optional SM split with the dxd GEMM (experiments)
    if (seg_ctas > 0) {
      g5.max_ctas = g6.max_ctas = seg_ctas;
      g4.max_ctas = num_sms_api() - seg_ctas;
    }
    DMOE_TRY(rows_gemm(g3, dt, s));
    SideStream* ss2 = nullptr;
    cudaStream_t side2 = fork_stream(s, &ss2);
    DMOE_TRY(tc_gemm_segk2(g5, g6, side2 ? side2 : s));
    DMOE_TRY(rows_gemm(g4, dt, s));
    if (side2) DMOE_TRY(join_stream(s, ss2));
    return DMOE_OK;
  }
  SideStream* ss = nullptr;
  cudaStream_t side = fork_stream(s, &ss);
  if (side) {
    // SM split between the chains: the weight-gradient GEMMs are bound by HBM writes (dW), the
    // row GEMMs by HBM reads (W); run side by side on disjoint SMs the two mix into copy-like
    // traffic instead of alternating write-only and read-only phases.
    const int seg_ctas = bwd_segk_ctas();
    g5.max_ctas = g6.max_ctas = seg_ctas;
    g3.max_ctas = g4.max_ctas = seg_ctas > 0 ? num_sms_api() - seg_ctas : 0;
    DMOE_TRY(segk_gemm(g5, dt, side));
  }
  DMOE_TRY(rows_gemm(g3, dt, s));
  if (side) {
    DMOE_TRY(fork_point(s, ss));  // side waits for dh
    DMOE_TRY(segk_gemm(g6, dt, side));
  }
  DMOE_TRY(rows_gemm(g4, dt, s));
  if (side) {
    DMOE_TRY(join_stream(s, ss));
  } else {
    DMOE_TRY(segk_gemm(g5, dt, s));
    DMOE_TRY(segk_gemm(g6, dt, s));
  }
  if (fused) return DMOE_OK;
  DMOE_TRY(seg_colsum(dout, dt, offsets, E_local, D, db2, s));
  return seg_colsum(dh, dt, offsets, E_local, H, db1, s);
}

dmoe_status dmoe_expert_ffn_bwd(const void* xd, const void* h, const uint32_t* hmask, const void* dout,
                                const int32_t* offsets, int32_t E_local, int64_t R_cap,
                                int32_t D, int32_t H, dmoe_dtype dt, const void* W1,
                                const void* W2, void* dxd, void* dW1, float* db1, void* dW2,
                                float* db2, void* ws, size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_TRY(expert_ffn_bwd_impl(xd, h, hmask, dout, offsets, E_local, R_cap, D, H, dt, W1, W2, dxd, dW1, db1, dW2,
                               db2, ws, ws_bytes, stream));
  cudaStream_t s = (cudaStream_t)stream;
  DMOE_TRY(finite_check("expert_ffn_bwd", "dW1", dW1, dt, (int64_t)E_local * H * D, s));
  DMOE_TRY(finite_check("expert_ffn_bwd", "dW2", dW2, dt, (int64_t)E_local * D * H, s));
  DMOE_TRY(finite_check("expert_ffn_bwd", "db1", db1, DMOE_F32, (int64_t)E_local * H, s));
  DMOE_TRY(finite_check("expert_ffn_bwd", "db2", db2, DMOE_F32, (int64_t)E_local * D, s));
  return finite_check("expert_ffn_bwd", "dxd", dxd, dt, rows_used(offsets, E_local, s) * D, s);
}

dmoe_status dmoe_expert_ffn_bwd_sgd(const void* xd, const void* h, const uint32_t* hmask, const void* dout,
                                    const int32_t* offsets, int32_t E_local, int64_t R_cap, int32_t D,
                                    int32_t H, dmoe_dtype dt, void* W1, float* b1, void* W2, float* b2,
                                    float lr, void* dxd, void* ws, size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  DMOE_TRY(check_dt(dt, H));
  DMOE_REQUIRE(E_local >= 1 && R_cap >= 0, DMOE_ERR_SHAPE, "E_local=%d R_cap=%lld", E_local, (long long)R_cap);
  DMOE_REQUIRE(lr == lr, DMOE_ERR_ARG, "expert_ffn_bwd_sgd: lr is NaN");
  NN(offsets); NN(W1); NN(b1); NN(W2); NN(b2); NN(ws);
  if (R_cap > 0) { NN(xd); NN(dout); NN(dxd); }
  GemmSegK p5{}, p6{};
  p5.Mdim = D; p5.N = H; p6.Mdim = H; p6.N = D;
  DMOE_REQUIRE(dt == DMOE_BF16 && tc_segk_supported(p5) && tc_segk_supported(p6), DMOE_ERR_UNSUPPORTED,
               "expert_ffn_bwd_sgd: needs the bf16 tensor-core path (D, H multiples of 128)");
  cudaStream_t s = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  int32_t* plan_tc = cv.take<int32_t>(E_local + 1);
  int32_t* plan_simt = cv.take<int32_t>(E_local + 1);
  void* dh = cv.take<char>((size_t)(R_cap > 0 ? R_cap : 1) * H * 2);
  // h == NULL: the forward's hidden activation is recomputed here (gradient checkpointing:
  // the expert is "called twice per batch")
  void* hre = h ? nullptr : cv.take<char>((size_t)(R_cap > 0 ? R_cap : 1) * H * 2);
  uint32_t* mre = (h || !hmask_path(dt, D, H, E_local, R_cap)) ? nullptr
                                                                : cv.take<uint32_t>((size_t)((H + 31) / 32) * (R_cap > 0 ? R_cap : 1));
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "expert_ffn_bwd_sgd: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  const void* hh = h ? h : hre;
  const uint32_t* hm = h ? hmask : mre;
  GemmRows g1{};
  if (!h) {
    g1.A = xd; g1.B = W1; g1.C = hre; g1.bias = b1; g1.offsets = offsets;
    g1.E = E_local; g1.N = H; g1.K = D; g1.rows_cap = R_cap; g1.b_mn = false; g1.epi = EPI_BIAS_RELU;
    if (mre) { g1.hmask = mre; g1.hmask_ld = R_cap; }
  }
  GemmRows g3{};
  g3.A = dout; g3.B = W2; g3.C = dh; g3.aux = hh; g3.offsets = offsets;
  g3.E = E_local; g3.N = H; g3.K = D; g3.rows_cap = R_cap; g3.b_mn = true; g3.epi = EPI_RELU_MASK;
  if (hm && hmask_path(dt, D, H, E_local, R_cap)) { g3.hmask = const_cast<uint32_t*>(hm); g3.hmask_ld = R_cap; }
  GemmRows g4 = g3;
  g4.A = dh; g4.B = W1; g4.C = dxd; g4.aux = nullptr; g4.N = D; g4.K = H; g4.epi = EPI_PLAIN;
  g4.hmask = nullptr;
  for (GemmRows* g : {&g1, &g3, &g4}) {
    g->plan = plan_tc;
    g->max_tiles = ceil_div(R_cap, tc_rows_tile(*g)) + E_local;
  }
  DMOE_TRY(plans_for(g3, g4, offsets, E_local, plan_tc, plan_simt, s));
  if (!h) {
    g1.plan = g3.plan;
    DMOE_TRY(rows_gemm(g1, dt, s));
  }
  DMOE_TRY(rows_gemm(g3, dt, s));   // reads W2
  DMOE_TRY(rows_gemm(g4, dt, s));   // reads W1
  // then the parameter updates, in place, in one persistent launch (after both readers)
  GemmSegK g5{dout, hh, W2, offsets, E_local, D, H, R_cap, b2};
  GemmSegK g6{dh, xd, W1, offsets, E_local, H, D, R_cap, b1};
  g5.sgd_lr = g6.sgd_lr = lr;
  if (tc_segk2_supported(g5, g6)) return tc_gemm_segk2(g5, g6, s);
  DMOE_TRY(tc_gemm_segk(g5, s));
  return tc_gemm_segk(g6, s);
}

// ------------------------------------------------------------- NEXT-2: the §4.1 expert block
static dmoe_status ffn3_check(dmoe_dtype dt, int32_t D, int32_t H, int32_t E_local, int64_t R_cap) {
  DMOE_REQUIRE(dt == DMOE_BF16, DMOE_ERR_UNSUPPORTED, "expert_ffn3: bf16 only");
  DMOE_REQUIRE(E_local >= 1 && R_cap >= 0 && D % 128 == 0 && H % 128 == 0 && H <= 8192, DMOE_ERR_SHAPE,
               "expert_ffn3: E_local=%d D=%d H=%d (D, H multiples of 128, H <= 8192)", E_local, D, H);
  GemmRows g{};
  g.E = E_local; g.N = H; g.K = D; g.rows_cap = R_cap; g.offsets = reinterpret_cast<const int32_t*>(16);
  g.epi = EPI_BIAS;
  DMOE_REQUIRE(tc_rows_supported(g), DMOE_ERR_UNSUPPORTED, "expert_ffn3: tensor-core path unavailable");
  return DMOE_OK;
}

// plans: [2][E+1] row-tile plans for 128-row tiles and for CTA-pair 256-row tiles (host-built only
// when E exceeds the in-kernel plan's smem table)
static GemmRows rows_for(const void* A, const void* B, void* C, const float* bias, const int32_t* offsets, int E,
                         int N, int K, int64_t R_cap, bool b_mn, int epi, int32_t* plans) {
  GemmRows g{};
  g.A = A; g.B = B; g.C = C; g.bias = bias; g.aux = nullptr; g.offsets = offsets;
  g.E = E; g.N = N; g.K = K; g.rows_cap = R_cap; g.b_mn = b_mn; g.epi = epi;
  const int tile = tc_rows_tile(g);
  g.plan = E <= tc_plan_in_kernel_max() ? nullptr : plans + (tile == TC_ROWS_TILE_DEFAULT ? 0 : E + 1);
  g.max_tiles = ceil_div(R_cap, tile) + E;
  return g;
}
static dmoe_status ffn3_plans(const int32_t* offsets, int E, int32_t* plans, cudaStream_t s) {
  if (E <= tc_plan_in_kernel_max()) return DMOE_OK;
  DMOE_TRY(tile_plan(offsets, E, TC_ROWS_TILE_DEFAULT, plans, s));
  return tile_plan(offsets, E, 2 * TC_ROWS_TILE_DEFAULT, plans + E + 1, s);
}

dmoe_status dmoe_expert_ffn3_fwd(const void* xd, const int32_t* offsets, int32_t E_local, int64_t R_cap,
                                 int32_t D, int32_t H, dmoe_dtype dt, const void* W1, const float* b1,
                                 const float* g1, const float* be1, const void* W2, const float* b2,
                                 const float* g2, const float* be2, const void* W3, const float* b3, float eps,
                                 void* z1, void* a1, void* z2, void* a2, float* stats, void* out, void* ws,
                                 size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(ffn3_check(dt, D, H, E_local, R_cap));
  NN(offsets); NN(W1); NN(b1); NN(g1); NN(be1); NN(W2); NN(b2); NN(g2); NN(be2); NN(W3); NN(b3); NN(ws);
  if (R_cap > 0) { NN(xd); NN(z1); NN(a1); NN(z2); NN(a2); NN(stats); NN(out); }
  cudaStream_t s = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  int32_t* plan = cv.take<int32_t>(2 * ((size_t)E_local + 1));
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "expert_ffn3_fwd: workspace too small");
  DMOE_TRY(ffn3_plans(offsets, E_local, plan, s));
  // z1 = W1 x + b1 -> a1 = relu(LN1(z1)) -> z2 = W2 a1 + b2 -> a2 = relu(LN2(z2)) -> out = W3 a2 + b3
  DMOE_TRY(tc_gemm_rows(rows_for(xd, W1, z1, b1, offsets, E_local, H, D, R_cap, false, EPI_BIAS, plan), s));
  DMOE_TRY(ln_relu_fwd(z1, offsets, E_local, R_cap, H, eps, g1, be1, a1, stats, s));
  DMOE_TRY(tc_gemm_rows(rows_for(a1, W2, z2, b2, offsets, E_local, H, H, R_cap, false, EPI_BIAS, plan), s));
  DMOE_TRY(ln_relu_fwd(z2, offsets, E_local, R_cap, H, eps, g2, be2, a2, stats + 2 * (R_cap > 0 ? R_cap : 1), s));
  return tc_gemm_rows(rows_for(a2, W3, out, b3, offsets, E_local, D, H, R_cap, false, EPI_BIAS, plan), s);
}

dmoe_status dmoe_expert_ffn3_bwd(const void* xd, const void* z1, const void* a1, const void* z2, const void* a2,
                                 const float* stats, const void* dout, const int32_t* offsets, int32_t E_local,
                                 int64_t R_cap, int32_t D, int32_t H, dmoe_dtype dt, const void* W1,
                                 const float* g1, const float* be1, const void* W2, const float* g2,
                                 const float* be2, const void* W3, void* dxd, void* dW1, float* db1, float* dg1,
                                 float* dbe1, void* dW2, float* db2, float* dg2, float* dbe2, void* dW3,
                                 float* db3, void* ws, size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(ffn3_check(dt, D, H, E_local, R_cap));
  NN(offsets); NN(W1); NN(g1); NN(be1); NN(W2); NN(g2); NN(be2); NN(W3); NN(dW1); NN(db1); NN(dg1); NN(dbe1);
  NN(dW2); NN(db2); NN(dg2); NN(dbe2); NN(dW3); NN(db3); NN(ws);
  if (R_cap > 0) { NN(xd); NN(z1); NN(a1); NN(z2); NN(a2); NN(stats); NN(dout); NN(dxd); }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t Rc = R_cap > 0 ? R_cap : 1;
  Carver cv(ws, ws_bytes);
  int32_t* plan = cv.take<int32_t>(2 * ((size_t)E_local + 1));
  void* da = cv.take<char>((size_t)Rc * H * 2);
  void* dz = cv.take<char>((size_t)Rc * H * 2);
  DMOE_REQUIRE(cv.ok(), DMOE_ERR_ARG, "expert_ffn3_bwd: workspace too small (%zu < %zu)", ws_bytes, cv.used);
  DMOE_TRY(ffn3_plans(offsets, E_local, plan, s));
  // out = W3 a2 + b3:  da2 = dout W3;  dW3 = dout^T a2, db3 = sum dout
  DMOE_TRY(tc_gemm_rows(rows_for(dout, W3, da, nullptr, offsets, E_local, H, D, R_cap, true, EPI_PLAIN, plan), s));
  GemmSegK g3{dout, a2, dW3, offsets, E_local, D, H, R_cap, db3};
  DMOE_TRY(tc_gemm_segk(g3, s));
  // a2 = relu(LN2(z2)):  dz2, dg2, dbe2
  DMOE_TRY(ln_relu_bwd(da, z2, stats + 2 * Rc, offsets, E_local, H, g2, be2, dz, dg2, dbe2, s));
  // z2 = W2 a1 + b2:  da1 = dz2 W2;  dW2 = dz2^T a1, db2 = sum dz2
  GemmSegK g2s{dz, a1, dW2, offsets, E_local, H, H, R_cap, db2};
  DMOE_TRY(tc_gemm_segk(g2s, s));
  DMOE_TRY(tc_gemm_rows(rows_for(dz, W2, da, nullptr, offsets, E_local, H, H, R_cap, true, EPI_PLAIN, plan), s));
  // a1 = relu(LN1(z1)):  dz1, dg1, dbe1
  DMOE_TRY(ln_relu_bwd(da, z1, stats, offsets, E_local, H, g1, be1, dz, dg1, dbe1, s));
  // z1 = W1 x + b1:  dxd = dz1 W1;  dW1 = dz1^T xd, db1 = sum dz1
  GemmSegK g1s{dz, xd, dW1, offsets, E_local, H, D, R_cap, db1};
  DMOE_TRY(tc_gemm_segk(g1s, s));
  return tc_gemm_rows(rows_for(dz, W1, dxd, nullptr, offsets, E_local, D, H, R_cap, true, EPI_PLAIN, plan), s);
}

dmoe_status dmoe_gate_bwd(const void* x, const void* Wg, const int32_t* sel, const float* dscore,
                          const void* dxd, const int32_t* row_of_slot, int64_t T, int32_t D,
                          dmoe_grid g, dmoe_dtype dt, void* dx, float* dWg, float* dbg, void* ws,
                          size_t ws_bytes, dmoe_stream_t stream) {
  DMOE_NVTX();
  int64_t E = 0;
  DMOE_TRY(check_grid(&g, &E));
  DMOE_TRY(check_dt(dt, D));
  DMOE_REQUIRE(T >= 0, DMOE_ERR_SHAPE, "T < 0");
  NN(Wg); NN(dWg); NN(dbg); NN(ws);
  if (T > 0) { NN(x); NN(sel); NN(dscore); NN(row_of_slot); NN(dx); }
  cudaStream_t s = (cudaStream_t)stream;
  DMOE_TRY(gate_bwd(x, Wg, sel, dscore, dxd, row_of_slot, T, D, g.d, g.M, g.k, dt, dx, dWg, dbg, ws, ws_bytes, s));
  DMOE_TRY(finite_check("gate_bwd", "dWg", dWg, DMOE_F32, (int64_t)D * g.d * g.M, s));
  DMOE_TRY(finite_check("gate_bwd", "dbg", dbg, DMOE_F32, (int64_t)g.d * g.M, s));
  return finite_check("gate_bwd", "dx", dx, dt, T * D, s);
}

dmoe_status dmoe_segment_offsets(const int32_t* offsets, int32_t E, int32_t group, int32_t* seg,
                                 dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_REQUIRE(E >= 1 && group >= 1 && E % group == 0, DMOE_ERR_SHAPE, "segment_offsets: E=%d group=%d", E, group);
  NN(offsets); NN(seg);
  return segment_offsets(offsets, E, group, seg, (cudaStream_t)stream);
}

dmoe_status dmoe_exchange_layout(const int32_t* recv_counts, int32_t G, int32_t E_local, int64_t R_cap,
                                 int32_t* offsets, int32_t* src_of_dst, void* ws, size_t ws_bytes,
                                 dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_REQUIRE(G >= 1 && E_local >= 1 && R_cap >= 0, DMOE_ERR_SHAPE, "G=%d E_local=%d", G, E_local);
  NN(recv_counts); NN(offsets); NN(ws);
  if (R_cap > 0) NN(src_of_dst);
  return exchange_layout(recv_counts, G, E_local, offsets, src_of_dst, R_cap, ws, ws_bytes,
                         (cudaStream_t)stream);
}

dmoe_status dmoe_permute_rows(const void* src, dmoe_dtype dt, const int32_t* idx, const int32_t* n_rows,
                              int32_t D, int32_t inverse, void* dst, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_dt(dt, D));
  NN(src); NN(idx); NN(n_rows); NN(dst);
  DMOE_REQUIRE(inverse == 0 || inverse == 1, DMOE_ERR_ARG, "inverse must be 0 or 1");
  return permute_rows(src, idx, n_rows, D, dt, inverse, dst, (cudaStream_t)stream);
}

// ------------------------------------------------------------ peer-memory exchange
static dmoe_status check_ep(const dmoe_ep* ep) {
  DMOE_REQUIRE(ep != nullptr, DMOE_ERR_ARG, "ep: null");
  DMOE_REQUIRE(ep->G >= 1 && ep->rank >= 0 && ep->rank < ep->G && ep->E_local >= 1 &&
                   ep->E == ep->G * ep->E_local && ep->rin_cap >= 0,
               DMOE_ERR_SHAPE, "ep: G=%d rank=%d E=%d E_local=%d", ep->G, ep->rank, ep->E, ep->E_local);
  DMOE_REQUIRE(ep->epoch && ep->flags && ep->peer_flags && ep->cnt && ep->peer_cnt && ep->err && ep->base &&
                   ep->off_loc && ep->src_off && ep->dst_off,
               DMOE_ERR_ARG, "ep: null buffer");
  return DMOE_OK;
}

dmoe_status dmoe_ep_begin(const dmoe_ep* ep, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_ep(ep));
  return ep_begin(ep->epoch, (cudaStream_t)stream);
}

dmoe_status dmoe_ep_exchange_counts(const dmoe_ep* ep, const int32_t* counts, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_ep(ep));
  NN(counts);
  cudaStream_t s = (cudaStream_t)stream;
  DMOE_TRY(ep_counts_push(counts, ep->E, ep->G, ep->rank, ep->peer_cnt, s));
  DMOE_TRY(ep_signal(ep->peer_flags, ep->G, ep->rank, ep->epoch, 0, s));
  DMOE_TRY(ep_wait(ep->flags, ep->G, ep->epoch, 0, ep->timeout_ns, ep->err, s));
  return ep_plan(ep->cnt, ep->G, ep->rank, ep->E, ep->E_local, ep->rin_cap, ep->base, ep->off_loc, ep->src_off,
                 ep->dst_off, ep->err, s);
}

dmoe_status dmoe_ep_push_rows(const dmoe_ep* ep, const void* src, dmoe_dtype dt, const int32_t* gather_idx,
                              const int32_t* offsets, int32_t D, void* const* peer_dst, int32_t phase,
                              dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_ep(ep));
  DMOE_TRY(check_dt(dt, D));
  NN(src); NN(offsets); NN(peer_dst);
  DMOE_REQUIRE(phase >= 1 && phase <= 7, DMOE_ERR_ARG, "phase %d outside [1,7]", phase);
  cudaStream_t s = (cudaStream_t)stream;
  DMOE_TRY(ep_push_rows(src, gather_idx, offsets, ep->base, ep->E, ep->E_local, D, dt, peer_dst, ep->err, s));
  DMOE_TRY(ep_signal(ep->peer_flags, ep->G, ep->rank, ep->epoch, phase, s));
  return ep_wait(ep->flags, ep->G, ep->epoch, phase, ep->timeout_ns, ep->err, s);
}

dmoe_status dmoe_ep_return_rows(const dmoe_ep* ep, const void* src, dmoe_dtype dt, int32_t D,
                                void* const* peer_dst, int32_t phase, dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_TRY(check_ep(ep));
  DMOE_TRY(check_dt(dt, D));
  NN(src); NN(peer_dst);
  DMOE_REQUIRE(phase >= 1 && phase <= 7, DMOE_ERR_ARG, "phase %d outside [1,7]", phase);
  cudaStream_t s = (cudaStream_t)stream;
  DMOE_TRY(ep_return_rows(src, ep->cnt, ep->off_loc, ep->src_off, ep->dst_off, ep->G, ep->rank, ep->E,
                          ep->E_local, D, dt, peer_dst, ep->err, s));
  DMOE_TRY(ep_signal(ep->peer_flags, ep->G, ep->rank, ep->epoch, phase, s));
  return ep_wait(ep->flags, ep->G, ep->epoch, phase, ep->timeout_ns, ep->err, s);
}

dmoe_status dmoe_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  DMOE_NVTX();
  NN(ptr); NN(handle);
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle, *ptr);
  DMOE_REQUIRE(e == cudaSuccess, DMOE_ERR_CUDA, "ipc_alloc: %s", cudaGetErrorString(e));
  return DMOE_OK;
}

dmoe_status dmoe_ipc_open(const void* handle, void** ptr) {
  DMOE_NVTX();
  NN(handle); NN(ptr);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  DMOE_REQUIRE(e == cudaSuccess, DMOE_ERR_CUDA, "ipc_open: %s", cudaGetErrorString(e));
  return DMOE_OK;
}

dmoe_status dmoe_ipc_close(void* ptr) {
  DMOE_NVTX();
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  DMOE_REQUIRE(e == cudaSuccess, DMOE_ERR_CUDA, "ipc_close: %s", cudaGetErrorString(e));
  return DMOE_OK;
}

dmoe_status dmoe_ipc_free(void* ptr) {
  DMOE_NVTX();
  cudaError_t e = cudaFree(ptr);
  DMOE_REQUIRE(e == cudaSuccess, DMOE_ERR_CUDA, "ipc_free: %s", cudaGetErrorString(e));
  return DMOE_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ host-buffer layer step
namespace {
struct CopyStream {  // per (device, caller stream): the host step's copy stream and its events
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};
std::mutex g_copy_mu;
std::map<std::pair<int, cudaStream_t>, CopyStream> g_copy;
CopyStream* copy_for(cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_copy_mu);
  CopyStream& cs = g_copy[{dev, s}];
  if (!cs.st) {
    if (cudaStreamCreateWithFlags(&cs.st, cudaStreamNonBlocking) != cudaSuccess) { cs.st = nullptr; return nullptr; }
    for (auto& e : cs.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return &cs;
}
}  // namespace

extern "C" dmoe_status dmoe_layer_step_host(const dmoe_layer* L, int64_t T, const void* x_host,
                                            const void* dy_host, void* y_host, void* dx_host,
                                            dmoe_stream_t stream) {
  DMOE_NVTX();
  DMOE_REQUIRE(L && x_host && dy_host && y_host && dx_host, DMOE_ERR_ARG, "layer_step_host: null argument");
  DMOE_REQUIRE(T >= 0 && T <= L->T_max, DMOE_ERR_SHAPE, "layer_step_host: T=%lld outside [0, T_max=%lld]",
               (long long)T, (long long)L->T_max);
  DMOE_REQUIRE(L->tie >= 1, DMOE_ERR_ARG, "layer_step_host: tie=%d < 1", L->tie);
  cudaStream_t s = (cudaStream_t)stream;
  const dmoe_grid g = L->g;
  int64_t E = 1;
  for (int i = 0; i < g.d; ++i) E *= g.M;
  DMOE_REQUIRE(E % L->tie == 0, DMOE_ERR_SHAPE, "layer_step_host: tie=%d does not divide E=%lld", L->tie,
               (long long)E);
  const int32_t El = (int32_t)(E / L->tie);
  const int32_t* seg = L->tie > 1 ? L->seg : L->offsets;
  const size_t nbytes = (size_t)T * L->D * (L->dt == DMOE_BF16 ? 2 : 4);
  CopyStream* cs = copy_for(s);
  DMOE_REQUIRE(cs != nullptr, DMOE_ERR_CUDA, "layer_step_host: copy stream: %s",
               cudaGetErrorString(cudaGetLastError()));
#define DMOE_CU(x_)                                                                                 \
  do {                                                                                              \
    cudaError_t e_ = (x_);                                                                          \
    if (e_ != cudaSuccess) return set_error(DMOE_ERR_CUDA, "layer_step_host: %s", cudaGetErrorString(e_)); \
  } while (0)
  // x first (the forward waits for it), then dy on the copy stream while the forward runs (it
  // would otherwise share the host link with x)
  DMOE_CU(cudaMemcpyAsync(L->x, x_host, nbytes, cudaMemcpyHostToDevice, s));
  DMOE_CU(cudaEventRecord(cs->ev[0], s));
  DMOE_CU(cudaStreamWaitEvent(cs->st, cs->ev[0], 0));
  DMOE_CU(cudaMemcpyAsync(L->dy, dy_host, nbytes, cudaMemcpyHostToDevice, cs->st));
  DMOE_CU(cudaEventRecord(cs->ev[1], cs->st));
  // forward (S1-S7)
  DMOE_TRY(dmoe_gate_topk(L->x, L->dt, T, L->D, L->Wg, L->bg, g, L->alive_bits, L->G, L->sel, L->sel_score, L->ws,
                          L->ws_bytes, stream));
  DMOE_TRY(dmoe_dispatch(L->x, L->dt, T, L->D, g, L->sel, L->sel_score, L->responded_bits, L->w, L->valid,
                         L->n_dropped, L->counts, L->offsets, L->row_of_slot, L->token_of_row, L->xd, L->ws,
                         L->ws_bytes, stream));
  if (L->tie > 1) DMOE_TRY(dmoe_segment_offsets(L->offsets, (int32_t)E, L->tie, L->seg, stream));
  DMOE_TRY(dmoe_expert_ffn_fwd(L->xd, seg, El, L->R_cap, L->D, L->H, L->dt, L->W1, L->b1, L->W2, L->b2, L->h,
                               L->hmask, L->out, L->ws, L->ws_bytes, stream));
  DMOE_TRY(dmoe_combine(L->out, L->row_of_slot, L->w, L->valid, T, L->D, g.k, L->dt, L->y, stream));
  // y: downloaded on the copy stream while the backward runs
  DMOE_CU(cudaEventRecord(cs->ev[2], s));
  DMOE_CU(cudaStreamWaitEvent(cs->st, cs->ev[2], 0));
  DMOE_CU(cudaMemcpyAsync(y_host, L->y, nbytes, cudaMemcpyDeviceToHost, cs->st));
  // backward (S8-S10)
  DMOE_CU(cudaStreamWaitEvent(s, cs->ev[1], 0));
  DMOE_TRY(dmoe_combine_bwd(L->dy, L->out, L->row_of_slot, L->w, T, L->D, g.k, L->dt, L->dout, L->dscore, stream));
  DMOE_TRY(dmoe_expert_ffn_bwd(L->xd, L->h, L->hmask, L->dout, seg, El, L->R_cap, L->D, L->H, L->dt, L->W1, L->W2,
                               L->dxd, L->dW1, L->db1, L->dW2, L->db2, L->ws, L->ws_bytes, stream));
  DMOE_TRY(dmoe_gate_bwd(L->x, L->Wg, L->sel, L->dscore, L->dxd, L->row_of_slot, T, L->D, g, L->dt, L->dx, L->dWg,
                         L->dbg, L->ws, L->ws_bytes, stream));
  DMOE_CU(cudaMemcpyAsync(dx_host, L->dx, nbytes, cudaMemcpyDeviceToHost, s));
  DMOE_CU(cudaEventRecord(cs->ev[3], cs->st));
  DMOE_CU(cudaStreamWaitEvent(s, cs->ev[3], 0));  // the y download is part of this call's work
#undef DMOE_CU
  return DMOE_OK;
}
