/* include/dmoe.h — C ABI of the B200-native DMoE layer hot path (libdmoe.so).
 *
 * The calls follow the paper's statement of the layer (Ryabinin & Gusev,
 * "Learning@home", arXiv 2002.04013; line numbers refer to PAPER.md):
 *   - run the gating function to select k experts out of N       (§3.1)
 *       dmoe_gate_scores  (Eq. 2)
 *       dmoe_beam_topk    (Alg. 1 SelectExperts + FilterAlive)
 *   - send inputs to those experts and collect outputs           (§3.1)
 *       dmoe_dispatch     (renormalised Eq. 3 weights + per-expert batching)
 *       dmoe_expert_ffn_fwd (runtime Forward request)
 *   - aggregate expert outputs by weighted averaging             (Eq. 3)
 *       dmoe_combine
 *   - backward: runtime Backward request + gating gradient
 *       dmoe_combine_bwd, dmoe_expert_ffn_bwd, dmoe_gate_bwd
 *
 * Readings where the paper is silent or garbled (X1..X19):
 *   X1  expert uid (u_0..u_{d-1}) <-> flat index e = sum_i u_i M^(d-1-i), u_0 most significant.
 *   X2  Eq. 3's denominator is the standard softmax over the beam (index typo read as f_j).
 *   X3  beam width B >= k (B = k is the paper's Alg. 1); the last level keeps k.
 *   X4  ties broken by the total order (score descending, flat index ascending);
 *       -0.0 is treated as +0.0.
 *   X5  a prefix is alive iff at least one alive expert lies below it; FilterAlive runs
 *       before TopK at every level, including the last.
 *   X6  fewer than k alive experts: sel padded with -1, sel_score with -inf.
 *   X7  a token whose selected experts all failed is dropped: valid = 0, y = 0,
 *       zero gradient; counted in n_dropped (PAPER.md:287 footnote).
 *   X8  `responded` is known at dispatch time; non-responders are not dispatched.
 *   X11 the linear gate is affine (x W_g + b_g); logits G are fp32.
 *   X12 no gradient through the discrete selection.
 *   X13 ReLU'(0) = 0.
 *   X14 expert = 2-linear FFN D -> H -> D with bias and ReLU.
 *   X15 bf16 storage with fp32 accumulation; G, w, dscore, biases and all bias/gate
 *       gradients are fp32; H, Out, dW are stored in the parameter dtype.
 *   X18 rows inside an expert segment are in increasing token order.
 *
 * Conventions for every call:
 *   - All pointers are caller-owned DEVICE memory unless marked (host); row-major,
 *     contiguous; 16-byte aligned (the caller's cudaMalloc / torch allocations are).
 *   - Work is enqueued on `stream` (dmoe_expert_ffn_bwd forks its weight-gradient GEMMs onto a
 *     library stream with events and joins back before returning; CUDA-graph capturable); no call
 *     synchronises the host or allocates device memory.
 *     Scratch comes from the caller's workspace `ws` of at least
 *     dmoe_workspace_bytes(...) bytes (re-usable across calls on one stream).
 *   - Outputs are fully overwritten; callers never pre-zero (dW of an expert with no
 *     rows is written as 0; y and dX of dropped tokens are 0).
 *   - Argument/shape validation is synchronous and returns DMOE_ERR_* without
 *     enqueueing anything; launch failures return DMOE_ERR_CUDA; asynchronous kernel
 *     faults surface on a later CUDA call.  dmoe_last_error() gives a message.
 *   - Deterministic: no floating-point atomics; results are bitwise reproducible.
 *   - dtype DMOE_BF16 runs the tcgen05 tensor-core path for the contractions;
 *     DMOE_F32 runs exact fp32 SIMT kernels (no TF32), for the fp32 parity config.
 *   - "Batch dropped" is not an error (reported per token through valid/n_dropped).
 */
#ifndef DMOE_H
#define DMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dmoe_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  DMOE_OK = 0,
  DMOE_ERR_ARG = -1,         /* null pointer, negative size, bad enum */
  DMOE_ERR_SHAPE = -2,       /* dimension outside the supported envelope or inconsistent */
  DMOE_ERR_UNSUPPORTED = -3, /* valid request the library does not implement */
  DMOE_ERR_CUDA = -4,        /* a CUDA launch / driver call failed */
  DMOE_ERR_NONFINITE = -5    /* debug switch on (dmoe_set_check_finite): a NaN / Inf output */
} dmoe_status;

typedef enum { DMOE_F32 = 0, DMOE_BF16 = 1 } dmoe_dtype;

/* Expert grid of Eq. 1: E = M^d experts, k selected per token,
 * beam width `beam` (0 means k).  Envelope: 1 <= d <= 4, 1 <= M <= 1024, d*M <= 256,
 * M^d < 2^31, 1 <= k <= 16, k <= beam <= 32, beam*M <= 8192. */
typedef struct {
  int32_t d, M, k, beam;
} dmoe_grid;

const char* dmoe_last_error(void); /* thread-local text for the last non-OK status */
int32_t dmoe_version(void);

/* Host-side launch counters of this process (for tests and the bench's gpu_launches):
 * out[0] = all kernel launches, out[1] = tcgen05 GEMM launches, out[2] = SIMT GEMM
 * launches, out[3] reserved.  Writes min(n, 4) entries (host memory); returns 4. */
int32_t dmoe_launch_counters(int64_t* out, int32_t n);

/* Scratch needed by any call below for T tokens, d_model D, hidden H, E_local experts
 * on this rank and R_cap dispatched-row capacity (T*k on one GPU). */
size_t dmoe_workspace_bytes(int64_t T, int32_t D, int32_t H, dmoe_grid g, int32_t E_local,
                            int64_t R_cap);

/* S1 — gate scores, Eq. 2:
 *   G[t, i*M + j] = g_i(x_t, j) = b_g[i*M + j] + sum_c x[t, c] * W_g[c, i*M + j]
 * x [T, D] in dtype dt; W_g [D, d*M] in dt; b_g [d*M] fp32; G [T, d*M] fp32 (out).
 * bf16 with d*M % 16 == 0 runs on the tensor cores (W_g^T staged in `ws`). */
dmoe_status dmoe_gate_scores(const void* x, dmoe_dtype dt, int64_t T, int32_t D, const void* Wg,
                             const float* bg, dmoe_grid g, float* G, void* ws, size_t ws_bytes,
                             dmoe_stream_t stream);

/* S2+S3 — SelectExperts, Alg. 1 with FilterAlive,
 * per token: beam := [()]; for level i: expand every prefix p by j in [0,M) with score
 * s_p + G[t, i*M+j]; drop candidates whose prefix has no alive expert (X5); keep the
 * best B (k at the last level) under the order of X4.
 * G [T, d*M] fp32; alive_bits [ceil(E/32)] uint32, bit e%32 of word e/32 = expert e alive.
 * sel [T, k] int32 out: flat expert index per slot, best first, -1 pad (X6);
 * sel_score [T, k] fp32 out: the Eq. 2 score sum of the slot, -inf pad. */
dmoe_status dmoe_beam_topk(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive_bits,
                           int32_t* sel, float* sel_score, void* ws, size_t ws_bytes,
                           dmoe_stream_t stream);

/* S3, exact form (NEXT-3): the best k ALIVE experts by the Eq. 2 score, under X4's order — the
 * north star's "exact top-k ... restricted to a liveness mask".  Scores are the same level-order
 * fp32 sums Alg. 1 forms, so with every expert alive this equals dmoe_beam_topk bit for bit;
 * with dead experts Alg. 1 (beam B = k) may miss the true top-k, this does not (a per-token scan
 * of every alive expert: E <= 2^20).  Arguments as dmoe_beam_topk (g.beam is ignored). */
dmoe_status dmoe_topk_exact(const float* G, int64_t T, dmoe_grid g, const uint32_t* alive_bits, int32_t* sel,
                            float* sel_score, dmoe_stream_t stream);

/* S1+S2+S3 in one call — gate scores (Eq. 2) then SelectExperts (Alg. 1 + FilterAlive):
 * exactly dmoe_gate_scores followed by dmoe_beam_topk (same definitions, same results bit for
 * bit).  G [T, d*M] fp32 is optional: NULL keeps it in `ws` (the search reads it back from L2).
 * sel / sel_score as dmoe_beam_topk. */
dmoe_status dmoe_gate_topk(const void* x, dmoe_dtype dt, int64_t T, int32_t D, const void* Wg,
                           const float* bg, dmoe_grid g, const uint32_t* alive_bits, float* G,
                           int32_t* sel, float* sel_score, void* ws, size_t ws_bytes,
                           dmoe_stream_t stream);

/* S4+S5 — renormalised Eq. 3 weights and per-expert dispatch:
 *   ok[t,s]  = sel[t,s] >= 0 && responded(sel[t,s])                  (X8)
 *   w[t,s]   = exp(sel_score[t,s] - m_t) / sum_{ok r} exp(sel_score[t,r] - m_t), 0 if !ok
 *   valid[t] = any ok;  n_dropped = #tokens with !valid               (X7)
 *   rows of expert e = ok pairs with sel == e in increasing t (X18), segments by e;
 *   counts [E], offsets [E+1] (exclusive scan), row_of_slot [T,k] (-1 if !ok),
 *   token_of_row [R] (capacity T*k), xd [R, D] = x[token_of_row[r]] (capacity T*k rows).
 * x [T, D] in dt; responded_bits [ceil(E/32)] uint32; w [T,k] fp32; valid [T] uint8;
 * n_dropped [1] int32 (device).  xd may be NULL: the row gather is skipped (the peer exchange
 * gathers x while sending, dmoe_ep_push_rows). */
dmoe_status dmoe_dispatch(const void* x, dmoe_dtype dt, int64_t T, int32_t D, dmoe_grid g,
                          const int32_t* sel, const float* sel_score,
                          const uint32_t* responded_bits, float* w, uint8_t* valid,
                          int32_t* n_dropped, int32_t* counts, int32_t* offsets,
                          int32_t* row_of_slot, int32_t* token_of_row, void* xd, void* ws,
                          size_t ws_bytes, dmoe_stream_t stream);

/* S6 — grouped expert FFN forward, the runtime Forward request:
 * for expert e < E_local, rows r in [offsets[e], offsets[e+1]):
 *   h[r]   = relu(W1[e] xd[r] + b1[e])     (H outputs, stored in dt: saved for backward)
 *   out[r] = W2[e] h[r] + b2[e]            (D outputs, dt)
 * xd [R_cap, D] dt; offsets [E_local+1] int32 device, non-decreasing, offsets[E_local] <= R_cap;
 * W1 [E_local, H, D] dt; b1 [E_local, H] fp32; W2 [E_local, D, H] dt; b2 [E_local, D] fp32;
 * h [R_cap, H] dt (out); out [R_cap, D] dt (out).  bf16 needs D % 64 == 0, H % 64 == 0.
 * hmask: optional (NULL) packed ReLU record for the backward, [H/32][R_cap] uint32 (out):
 *   bit c of hmask[w * R_cap + r] = (stored h[r, 32w + c] > 0) — the bit X13's derivative
 *   needs — 1/16 of h's bytes; written for rows < offsets[E_local] when the bf16 tensor-core
 *   path runs (left untouched otherwise, and then the backward reads h). */
dmoe_status dmoe_expert_ffn_fwd(const void* xd, const int32_t* offsets, int32_t E_local,
                                int64_t R_cap, int32_t D, int32_t H, dmoe_dtype dt,
                                const void* W1, const float* b1, const void* W2, const float* b2,
                                void* h, uint32_t* hmask, void* out, void* ws, size_t ws_bytes,
                                dmoe_stream_t stream);

/* S7 — combine, Eq. 3: y[t] = sum_{ok s} w[t,s] out[row_of_slot[t,s]]
 * (fp32 accumulate), y[t] = 0 if !valid[t].  out [R, D] dt; y [T, D] dt (out). */
dmoe_status dmoe_combine(const void* out, const int32_t* row_of_slot, const float* w,
                         const uint8_t* valid, int64_t T, int32_t D, int32_t k, dmoe_dtype dt,
                         void* y, dmoe_stream_t stream);

/* S8 — combine backward (softmax Jacobian of Eq. 3 over the ok slots):
 *   a[t,s] = <dy[t], out[row]>;  dscore[t,s] = w[t,s] (a[t,s] - sum_{ok r} w[t,r] a[t,r]);
 *   dout[row] = w[t,s] dy[t]  (the Backward request's output gradient).
 * dy [T, D] dt; dout [R, D] dt (out); dscore [T, k] fp32 (out, 0 for !ok). */
dmoe_status dmoe_combine_bwd(const void* dy, const void* out, const int32_t* row_of_slot,
                             const float* w, int64_t T, int32_t D, int32_t k, dmoe_dtype dt,
                             void* dout, float* dscore, dmoe_stream_t stream);

/* S8 with backward-only failures (NEXT-3, reading X22; SPEC.md:300 spelling out PAPER.md:287 for
 * the Backward request): an expert that answered the Forward request but whose Backward request
 * fails (responded_bwd bit 0) is excluded from the gradient WITHOUT renormalisation: its
 * cotangent rows dout are written as 0, so the expert backward gives it no dx contribution and
 * no parameter gradient, while dscore (the gating gradient, formed locally from the forward's
 * record) is exactly dmoe_combine_bwd's.  sel [T, k] from the forward; responded_bwd_bits
 * [ceil(E/32)] uint32 (device).  Otherwise as dmoe_combine_bwd. */
dmoe_status dmoe_combine_bwd_failures(const void* dy, const void* out, const int32_t* row_of_slot,
                                      const float* w, const int32_t* sel, const uint32_t* responded_bwd_bits,
                                      int64_t T, int32_t D, int32_t k, dmoe_dtype dt, void* dout, float* dscore,
                                      dmoe_stream_t stream);

/* S9 — grouped expert FFN backward, the runtime Backward request:
 *   dh  = (dout W2[e]) * 1[h > 0]   (X13)
 *   dxd = dh W1[e]
 *   dW2[e] = sum_rows dout^T h;  db2[e] = sum_rows dout
 *   dW1[e] = sum_rows dh^T xd;   db1[e] = sum_rows dh      (0 for experts without rows)
 * dxd [R_cap, D] dt (out); dW1 [E_local, H, D] dt; dW2 [E_local, D, H] dt; db1 [E_local, H]
 * and db2 [E_local, D] fp32 (out).  hmask: optional (NULL), the packed ReLU record the forward
 * call wrote for these rows (same xd/offsets/h); when given, the dh GEMM reads its mask bits
 * instead of h (the same decisions, 1/16 of the bytes).  Contract: hmask is either NULL or the
 * buffer the last dmoe_expert_ffn_fwd call wrote for exactly these rows (same xd, offsets,
 * E_local, R_cap, D, H, dtype, with a non-NULL hmask); the library cannot check that the bits
 * are current, so a stale record gives a wrong dh mask without an error. */
dmoe_status dmoe_expert_ffn_bwd(const void* xd, const void* h, const uint32_t* hmask, const void* dout,
                                const int32_t* offsets, int32_t E_local, int64_t R_cap,
                                int32_t D, int32_t H, dmoe_dtype dt, const void* W1,
                                const void* W2, void* dxd, void* dW1, float* db1, void* dW2,
                                float* db2, void* ws, size_t ws_bytes, dmoe_stream_t stream);

/* S9 + the runtime's parameter update (NEXT-1): "compute gradients w.r.t. inputs and update
 * expert parameters by gradient descent" (§3.3), with optional gradient
 * checkpointing (the expert "called twice per batch").
 * The same gradients as dmoe_expert_ffn_bwd, applied in place instead of written out:
 *   dh  = (dout W2[e]) * 1[h > 0];   dxd = dh W1[e]          (with the weights BEFORE the update)
 *   W2[e] -= lr * dout^T h;  b2[e] -= lr * sum_rows dout;  W1[e] -= lr * dh^T xd;  b1[e] -= lr * sum_rows dh
 * The weight-gradient tiles are applied by the GEMM epilogue (TMA loads the parameter tile into
 * the store box, W - lr * dW in fp32, one bf16 rounding: reading X21), so no dW buffer exists and
 * dW never reaches HBM.  Experts without rows keep their parameters.
 * h: the saved hidden activation, or NULL to recompute it from xd, W1, b1 here (then hmask is
 * ignored).  W1, W2 in/out bf16; b1, b2 in/out fp32.  bf16 tensor-core path only (D, H multiples
 * of 128): DMOE_ERR_UNSUPPORTED otherwise. */
dmoe_status dmoe_expert_ffn_bwd_sgd(const void* xd, const void* h, const uint32_t* hmask, const void* dout,
                                    const int32_t* offsets, int32_t E_local, int64_t R_cap, int32_t D,
                                    int32_t H, dmoe_dtype dt, void* W1, float* b1, void* W2, float* b2,
                                    float lr, void* dxd, void* ws, size_t ws_bytes, dmoe_stream_t stream);

/* S6 / S9 with the paper's own expert block (NEXT-2, §4.1: "feedforward blocks
 * 1024 -> 4096 -> 4096 -> 1024 with layer normalization and ReLU activations in between";
 * reading X23): per expert e over its rows
 *   z1 = W1[e] x + b1[e];   a1 = relu(g1[e] * (z1 - mean z1) / sqrt(var z1 + eps) + be1[e])
 *   z2 = W2[e] a1 + b2[e];  a2 = relu(g2[e] * (z2 - mean z2) / sqrt(var z2 + eps) + be2[e])
 *   out = W3[e] a2 + b3[e]
 * (LayerNorm over the H features, biased variance.)  W1 [E_local, H, D], W2 [E_local, H, H],
 * W3 [E_local, D, H] bf16; b1, g1, be1, b2, g2, be2 [E_local, H] and b3 [E_local, D] fp32.
 * Saved for the backward: z1, a1, z2, a2 [R_cap, H] bf16 and stats [2][R_cap][2] fp32 (mean,
 * 1/std per row per LayerNorm).  The linears run on the grouped tcgen05 GEMMs, LayerNorm + ReLU
 * as row kernels between them.  bf16 only; D, H multiples of 128, H <= 8192. */
dmoe_status dmoe_expert_ffn3_fwd(const void* xd, const int32_t* offsets, int32_t E_local, int64_t R_cap,
                                 int32_t D, int32_t H, dmoe_dtype dt, const void* W1, const float* b1,
                                 const float* g1, const float* be1, const void* W2, const float* b2,
                                 const float* g2, const float* be2, const void* W3, const float* b3, float eps,
                                 void* z1, void* a1, void* z2, void* a2, float* stats, void* out, void* ws,
                                 size_t ws_bytes, dmoe_stream_t stream);
/* Its Backward request: dxd and every parameter gradient (dW1 [E_local, H, D], dW2 [E_local, H,
 * H], dW3 [E_local, D, H] bf16; db1, dg1, dbe1, db2, dg2, dbe2 [E_local, H], db3 [E_local, D]
 * fp32; zeros for experts without rows), from the saved z1, a1, z2, a2, stats. */
dmoe_status dmoe_expert_ffn3_bwd(const void* xd, const void* z1, const void* a1, const void* z2, const void* a2,
                                 const float* stats, const void* dout, const int32_t* offsets, int32_t E_local,
                                 int64_t R_cap, int32_t D, int32_t H, dmoe_dtype dt, const void* W1,
                                 const float* g1, const float* be1, const void* W2, const float* g2,
                                 const float* be2, const void* W3, void* dxd, void* dW1, float* db1, float* dg1,
                                 float* dbe1, void* dW2, float* db2, float* dg2, float* dbe2, void* dW3,
                                 float* db3, void* ws, size_t ws_bytes, dmoe_stream_t stream);

/* S10 — undispatch + gate backward (gradient of Eq. 2 through the Eq. 3 softmax):
 *   dG[t, i*M + u_i(sel[t,s])] += dscore[t,s]            (u_i per X1)
 *   dx[t]  = sum_{ok s} dxd[row_of_slot[t,s]] + sum_j dG[t,j] W_g[:, j]
 *   dWg    = sum_t x[t]^T dG[t]  ([D, d*M] fp32);  dbg = sum_t dG[t]  ([d*M] fp32)
 * x [T, D] dt; W_g [D, d*M] dt; dxd [R, D] dt; dx [T, D] dt (out). */
dmoe_status dmoe_gate_bwd(const void* x, const void* Wg, const int32_t* sel, const float* dscore,
                          const void* dxd, const int32_t* row_of_slot, int64_t T, int32_t D,
                          dmoe_grid g, dmoe_dtype dt, void* dx, float* dWg, float* dbg, void* ws,
                          size_t ws_bytes, dmoe_stream_t stream);

/* Tied-weight pool (reading X20): experts [s*group, (s+1)*group) share parameter
 * slot s, so the FFN calls run with E_local = E / group slots over the slot segments
 *   seg[s] = offsets[s * group],  s = 0 .. E/group        (seg [E/group + 1] int32, out)
 * Rows of tied experts are contiguous in the expert-major dispatch order, so a slot's rows are
 * one segment and its weight gradient (dW of the FFN backward) is the sum over its experts'
 * rows: the gradient of the tied parameters.  group = 1 copies offsets.
 * Fails with DMOE_ERR_SHAPE unless E % group == 0. */
dmoe_status dmoe_segment_offsets(const int32_t* offsets, int32_t E, int32_t group, int32_t* seg,
                                 dmoe_stream_t stream);

/* S11 — expert-parallel exchange, receive side ("send inputs to those workers
 * and collect outputs"; §3.3 the runtime batches requests per expert).  With experts sharded
 * over G ranks by contiguous flat index, a rank receives its experts' rows source-rank-major;
 * recv_counts [G][E_local] (device) gives the rows of local expert e from source s.
 *   offsets [E_local+1] (out): expert-major segment starts (expert e: source 0's rows, then
 *     source 1's, ... — the single-GPU token order when sources hold increasing token blocks);
 *   src_of_dst [R_cap] (out): source-major row index of every expert-major row.
 * Capacity: if sum(recv_counts) > R_cap the segments are clamped to R_cap (offsets[E_local] =
 * R_cap < sum(recv_counts) reports the overflow; rows past R_cap are never placed), so no kernel
 * downstream can run past the caller's buffers.
 * ws >= 8 * G * E_local bytes.  Fails with DMOE_ERR_SHAPE on G < 1 or E_local < 1. */
dmoe_status dmoe_exchange_layout(const int32_t* recv_counts, int32_t G, int32_t E_local, int64_t R_cap,
                                 int32_t* offsets, int32_t* src_of_dst, void* ws, size_t ws_bytes,
                                 dmoe_stream_t stream);

/* Row permutation for the exchange: inverse = 0 gathers dst[r] = src[idx[r]], inverse = 1
 * scatters dst[idx[r]] = src[r], for r < *n_rows (device int32).  Rows of D elements in dt. */
dmoe_status dmoe_permute_rows(const void* src, dmoe_dtype dt, const int32_t* idx, const int32_t* n_rows,
                              int32_t D, int32_t inverse, void* dst, dmoe_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * S11 fused form — expert-parallel exchange over NVLink peer memory ("send
 * inputs to those workers and collect outputs", one process per GPU on one node).
 * Rows are stored straight into the owner's expert-major receive buffer and outputs straight
 * back into the source's dispatch-order buffer; completion is signalled by per-source epoch
 * flags (release/acquire at system scope), so no host sync is needed and a whole step can be
 * captured in a CUDA graph.  Every buffer below is device memory; the peer-written ones
 * (flags, cnt and the row buffers passed as peer_dst) must be symmetric (same offsets on every
 * rank) and mapped on every peer (dmoe_ipc_alloc / dmoe_ipc_open).  A wait that does not
 * complete within timeout_ns sets err |= 1 and continues (no hang); a receive buffer
 * overflow (more than rin_cap rows for one owner) sets err |= 2 and skips all row writes.
 * Each push / return call is collective: every rank calls it with the same phase. */
typedef struct {
  int32_t G, rank, E, E_local;  /* E = G * E_local; rank owns experts [rank*E_local, +E_local) */
  int64_t rin_cap;              /* rows of each rank's expert-major receive buffers            */
  uint64_t timeout_ns;
  uint64_t* epoch;              /* [1] step counter (local)                                     */
  uint64_t* flags;              /* [G] flags written by the peers (symmetric)                   */
  uint64_t* const* peer_flags;  /* [G] every rank's `flags`                                      */
  int32_t* cnt;                 /* [G][E] count matrix, row s written by rank s (symmetric)      */
  int32_t* const* peer_cnt;     /* [G] every rank's `cnt`                                        */
  int32_t* err;                 /* [1] error word (local)                                        */
  int32_t* base;                /* [E] plan: this rank's first row in owner(e)'s receive buffer  */
  int32_t* off_loc;             /* [E_local+1] plan: expert-major segment starts (receive side)  */
  int32_t* src_off;             /* [G][E_local] plan: source s's rows of own expert, its order   */
  int32_t* dst_off;             /* [G][E_local] plan: where they sit in the receive buffer       */
} dmoe_ep;

dmoe_status dmoe_ep_begin(const dmoe_ep* ep, dmoe_stream_t stream); /* epoch += 1 */
/* C1: broadcast counts [E] (from dmoe_dispatch) into every peer's cnt row `rank`, wait for all
 * peers, then plan base / off_loc / src_off / dst_off. */
dmoe_status dmoe_ep_exchange_counts(const dmoe_ep* ep, const int32_t* counts, dmoe_stream_t stream);
/* C2 / C4: dispatch-order rows (offsets [E+1] from dmoe_dispatch) -> owners' receive buffers
 * peer_dst [G] (expert-major, off_loc layout).  Row r is src[gather_idx[r]] if gather_idx is
 * non-NULL (x with token_of_row: the dispatch gather fused with the send), else src[r]. */
dmoe_status dmoe_ep_push_rows(const dmoe_ep* ep, const void* src, dmoe_dtype dt, const int32_t* gather_idx,
                              const int32_t* offsets, int32_t D, void* const* peer_dst, int32_t phase,
                              dmoe_stream_t stream);
/* C3 / C5: own experts' expert-major rows src [off_loc[E_local], D] -> each source's
 * dispatch-order buffer peer_dst [G] (the rows it sent, same positions). */
dmoe_status dmoe_ep_return_rows(const dmoe_ep* ep, const void* src, dmoe_dtype dt, int32_t D,
                                void* const* peer_dst, int32_t phase, dmoe_stream_t stream);
/* plumbing: cudaMalloc'ed zeroed arena + its 64-byte IPC handle (host); open / close a peer's */
dmoe_status dmoe_ipc_alloc(size_t bytes, void** ptr, void* handle);
dmoe_status dmoe_ipc_open(const void* handle, void** ptr);
dmoe_status dmoe_ipc_close(void* ptr);
dmoe_status dmoe_ipc_free(void* ptr);

/* Debug switch (off by default; the hot path never checks finiteness): with on != 0, the calls
 * dmoe_gate_scores (G), dmoe_gate_topk (G), dmoe_expert_ffn_fwd (out rows [0, offsets[E_local])),
 * dmoe_combine (y), dmoe_combine_bwd (dscore), dmoe_expert_ffn_bwd (dW1, dW2, db1, db2, dxd rows)
 * and dmoe_gate_bwd (dWg, dbg, dx) scan their floating-point outputs after the launch,
 * SYNCHRONISE the stream and return DMOE_ERR_NONFINITE (message: call and output) on a NaN or
 * Inf — SPEC.md:40's "numeric error".  Process-wide; not for use inside graph capture. */
void dmoe_set_check_finite(int on);

/* One whole layer step from HOST buffers (the end-to-end unit): x and dy
 * are copied host -> device, S1-S10 run (forward: gate + beam search, dispatch, expert FFN,
 * combine; backward: combine backward, expert backward with dW written, gate backward), and y
 * and dX are copied device -> host, all on `stream` (x first; dy's upload then overlaps the
 * forward and y's download overlaps the backward on a library copy stream joined back into
 * `stream` before the call's work completes).  Every pointer in dmoe_layer is caller-owned DEVICE memory sized for
 * T_max tokens (the ones the per-call entry points above take); x_host, dy_host, y_host,
 * dx_host are host memory of [T, D] dt (pinned for asynchronous copies; pageable memory works
 * but the copies then synchronise).  tie > 1: the tied-weight pool (reading X20) with E / tie
 * parameter slots and seg [E/tie + 1]; tie == 1: seg is unused.  G, h and hmask may be NULL
 * (no scores kept / no saved-activation mask).  Errors: any entry point's status. */
typedef struct {
  dmoe_grid g;
  int32_t D, H, tie;
  dmoe_dtype dt;
  int64_t T_max, R_cap;                       /* R_cap = T_max * k capacity rows            */
  const void* Wg; const float* bg;            /* gate [D, d*M], [d*M]                        */
  const void* W1; const float* b1;            /* experts [E/tie, H, D], [E/tie, H]           */
  const void* W2; const float* b2;            /*         [E/tie, D, H], [E/tie, D]           */
  const uint32_t* alive_bits; const uint32_t* responded_bits;
  void* x; void* dy;                          /* [T_max, D] device staging                   */
  float* G;                                   /* [T_max, d*M] or NULL                        */
  int32_t* sel; float* sel_score; float* w; uint8_t* valid; int32_t* n_dropped;
  int32_t* counts; int32_t* offsets; int32_t* seg;
  int32_t* row_of_slot; int32_t* token_of_row;
  void* xd; void* h; uint32_t* hmask; void* out; void* y;
  void* dout; float* dscore; void* dxd;
  void* dW1; float* db1; void* dW2; float* db2;
  void* dx; float* dWg; float* dbg;
  void* ws; size_t ws_bytes;
} dmoe_layer;
dmoe_status dmoe_layer_step_host(const dmoe_layer* layer, int64_t T, const void* x_host, const void* dy_host,
                                 void* y_host, void* dx_host, dmoe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DMOE_H */
