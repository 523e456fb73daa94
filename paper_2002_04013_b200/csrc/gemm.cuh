// gemm.cuh — internal descriptors of the grouped GEMMs (SIMT fp32 and tcgen05 bf16).
#pragma once
#include "common.cuh"

namespace dmoe {

enum Epi {
  EPI_F32_BIAS = 0,   // fp32 out = acc + bias[n]                 (gate scores, Eq. 2)
  EPI_BIAS_RELU = 1,  // out = relu(acc + bias[e][n])             (expert hidden h)
  EPI_BIAS = 2,       // out = acc + bias[e][n]                   (expert output)
  EPI_RELU_MASK = 3,  // out = acc * 1[aux[r][n] > 0]             (dh, ReLU'(0) = 0)
  EPI_PLAIN = 4,      // out = acc                                (dxd)
  EPI_F32 = 6         // fp32 out = acc                           (SEGK split-K partials: dW_g)
};

// ROWS family: C[r, n] = epi(sum_k A[r, k] B_e(n, k)) for r in expert segments
struct GemmRows {
  const void* A;        // [rows, K] K-major
  const void* B;        // b_mn ? [E][K][N] : [E][N][K]
  void* C;              // [rows, N]
  const float* bias;    // [E][N] (EPI_F32_BIAS / BIAS / BIAS_RELU)
  const void* aux;      // [rows, N] (EPI_RELU_MASK)
  const int32_t* offsets;  // [E+1] device, or nullptr: one group of rows_single rows
  const int32_t* plan;     // [E+1] device tile plan for this engine's row-tile size
  int E, N, K;
  int64_t rows_single;
  int64_t rows_cap;        // allocated rows of A / C / aux (TMA tensor extent)
  int64_t max_tiles;       // host upper bound on plan[E] (grid size)
  bool b_mn;
  int epi;
  int max_ctas = 0;        // persistent grid cap (0: one CTA per SM); leaves SMs to a concurrent GEMM
  uint32_t* hmask = nullptr;  // packed ReLU mask [N/32][hmask_ld]: EPI_BIAS_RELU writes, EPI_RELU_MASK reads
  int64_t hmask_ld = 0;
};

// SEGK family: C_e[m, n] = sum_{r in seg e} A[r, m] B[r, n]  (K = segment rows)
struct GemmSegK {
  const void* A;  // [rows, Mdim]
  const void* B;  // [rows, N]
  void* C;        // [E][Mdim][N]
  const int32_t* offsets;
  int E, Mdim, N;
  int64_t R_cap;    // allocated rows of A and B
  float* colsum;    // optional [E][Mdim] fp32: sum over the segment's rows of A (bias gradient)
  int max_ctas = 0;  // persistent grid cap (0: one CTA per SM)
  bool out_f32 = false;  // C in fp32 (coalesced stores from the padded staging) instead of bf16
  float sgd_lr = 0.0f;   // != 0: C / colsum are the parameters W / b, updated in place
                         // (W -= lr * dW, b -= lr * db; bf16 tensor-core path only)
};

dmoe_status simt_gemm_rows(const GemmRows& g, dmoe_dtype dt, cudaStream_t s);
dmoe_status simt_gemm_segk(const GemmSegK& g, dmoe_dtype dt, cudaStream_t s);
dmoe_status seg_colsum(const void* X, dmoe_dtype dt, const int32_t* offsets, int E, int N,
                       float* out, cudaStream_t s);
dmoe_status tile_plan(const int32_t* offsets, int64_t E, int bm, int32_t* plan, cudaStream_t s);

// tcgen05 engine (bf16 in, fp32 accumulate in TMEM); returns DMOE_ERR_UNSUPPORTED for shapes
// it does not take (caller then uses the SIMT kernels)
dmoe_status tc_gemm_rows(const GemmRows& g, cudaStream_t s);
dmoe_status tc_gemm_segk(const GemmSegK& g, cudaStream_t s);
bool tc_rows_supported(const GemmRows& g);
int tc_rows_tile(const GemmRows& g);       // token rows per tile of the row engine (plan granularity)
constexpr int TC_ROWS_TILE_DEFAULT = 128;  // == tc_rows_tile() of the M-major row engine
int tc_plan_in_kernel_max();               // experts up to which the M-major engine plans row tiles itself
bool tc_rows_mmajor();                     // the M-major row engine (not the swap-AB experiment) runs them
bool tc_segk_supported(const GemmSegK& g);
bool tc_segk_colsum_supported(const GemmSegK& g);  // the SEGK engine also writes colsum
bool tc_segk2_supported(const GemmSegK& a, const GemmSegK& b);
dmoe_status tc_gemm_segk2(const GemmSegK& a, const GemmSegK& b, cudaStream_t s);  // both in one launch

}  // namespace dmoe
