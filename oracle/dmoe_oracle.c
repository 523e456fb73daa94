/* oracle/dmoe_oracle.c — float64 CPU oracle of the DMoE layer (forward + backward).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_2002_04013_b200/csrc/);
 * neither includes nor links the other.
 *
 * Plain loops, float64 throughout, no BLAS, no blocking or reordering beyond the
 * definitions below.  OpenMP only splits an outer loop whose iterations write
 * disjoint outputs (so results do not depend on the thread count).
 *
 * Citations are to /root/reference/PAPER.md line numbers + section/equation;
 * "reading Xn" refers to DESIGN.md §Readings (the paper is silent / garbled there).
 *
 * Pins (tests/test_oracle_*.py): gate scores vs an independent numpy float64 matmul
 * and the hand sum of SPEC.md:213; Alg. 1 vs brute-force top-k over all M^d experts
 * when all are alive (closed argument in DESIGN.md) and vs the masked worked example
 * SPEC.md:222 (+ its derived B=1 variant); softmax weights vs closed forms
 * (ln7/ln3 -> 0.7/0.3, equal scores -> mean, saturation, shift invariance, drop ==
 * renormalise without it); dispatch vs the stable-sort invariants; FFN vs
 * zero/identity/linear cases; the whole backward vs central finite differences of
 * the forward (routing held fixed).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ S1: Eq. 2
 * G[t][i*M+j] = g_i(x_t, j) = b_g[i*M+j] + sum_c X[t][c] * W_g[c][i*M+j]
 * PAPER.md:238-246 (§3.2, Eq. 2: "we use a linear gating function", "only needs to
 * predict d vectors of size M"); affine gate = reading X11.  dM = d*M columns. */
void oracle_gate_scores(const double* X, int64_t T, int32_t D, const double* Wg,
                        const double* bg, int32_t dM, double* G) {
  #pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int32_t col = 0; col < dM; ++col) {
      double acc = bg[col];
      for (int32_t c = 0; c < D; ++c) acc += X[t * D + c] * Wg[(int64_t)c * dM + col];
      G[t * dM + col] = acc;
    }
}

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

/* ------------------------------------------------------------ S2: FilterAlive
 * PA_i[p] = 1 iff some alive expert has uid_{0:i} == p, i = 0..d-1.
 * PAPER.md:278 (§3.2: experts "submit all prefixes of their identifier" and the
 * filter checks the prefix's record).  Reading X5: an alive expert announces every
 * prefix including the full uid; dead experts announce nothing.  Reading X1: flat
 * index e = sum_i u_i M^{d-1-i}, so the level-i prefix of e is e / M^{d-1-i}.
 * PA layout: level i at offset sum_{l<i} M^{l+1}, M^{i+1} entries. */
void oracle_prefix_alive(const uint8_t* alive, int32_t d, int32_t M, uint8_t* PA) {
  int64_t E = ipow(M, d), off = 0;
  for (int i = 0; i < d; ++i) {
    int64_t n = ipow(M, i + 1), div = ipow(M, d - 1 - i);
    memset(PA + off, 0, (size_t)n);
    for (int64_t e = 0; e < E; ++e)
      if (alive[e]) PA[off + e / div] = 1;
    off += n;
  }
}

typedef struct { int64_t p; double s; } cand_t;

/* total order of reading X4: score descending, then flat (prefix) index ascending */
static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  return (x->p < y->p) ? -1 : (x->p > y->p);
}

/* ------------------------------------------------------------ S3: Algorithm 1
 * SelectExperts, PAPER.md:250-274 (§3.2, Alg. 1), per token, literally:
 *   beam := [()], scores := [0]
 *   for i in 0..d-1:
 *     expand every (prefix, score) in the beam by j in [0, M): prefix (+) [j],
 *         score + g_i(x, j)
 *     beam := FilterAlive(beam)
 *     beam := TopK(beam, k)  "select at most k best prefixes"
 *   return beam
 * with beam width W = B at levels i < d-1 and k at the last level (reading X3;
 * B = k is the paper's algorithm), TopK under the total order of reading X4, and
 * fewer than k survivors returned as-is and padded with -1 / -inf (reading X6).
 * The prefix is carried as its flat index p (reading X1): p (+) [j] = p*M + j.
 *
 * gap[t] (optional, for the parity rule of DESIGN.md): min over levels i < d-1 of
 * (c_B - c_{B+1}) and over j = 1..k at the last level of (c_j - c_{j+1}), where
 * c_j is the j-th alive candidate (1-based, sorted); a term with no (j+1)-th
 * candidate is +inf. */
void oracle_select_experts(const double* G, int64_t T, int32_t d, int32_t M, int32_t k,
                           int32_t B, const uint8_t* PA, int32_t* sel, double* sel_score,
                           double* gap) {
  int32_t dM = d * M;
  #pragma omp parallel
  {
    int32_t maxw = B > k ? B : k;
    cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (size_t)maxw * (size_t)M);
    cand_t* beam = (cand_t*)malloc(sizeof(cand_t) * (size_t)maxw);
    #pragma omp for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      const double* g = G + t * dM;
      int32_t nb = 1;
      beam[0].p = 0;
      beam[0].s = 0.0;
      double gmin = INFINITY;
      int64_t off = 0;
      for (int32_t i = 0; i < d; ++i) {
        int32_t n = 0;
        for (int32_t b = 0; b < nb; ++b)
          for (int32_t j = 0; j < M; ++j) {
            int64_t p = beam[b].p * M + j;
            if (!PA[off + p]) continue; /* FilterAlive */
            cand[n].p = p;
            cand[n].s = beam[b].s + g[i * M + j];
            ++n;
          }
        qsort(cand, (size_t)n, sizeof(cand_t), cand_cmp);
        int32_t W = (i < d - 1) ? B : k;
        if (i < d - 1) {
          if (n > W) {
            double tgap = cand[W - 1].s - cand[W].s;
            if (tgap < gmin) gmin = tgap;
          }
        } else {
          for (int32_t j = 1; j <= k && j < n; ++j) {
            double tgap = cand[j - 1].s - cand[j].s;
            if (tgap < gmin) gmin = tgap;
          }
        }
        nb = n < W ? n : W;
        for (int32_t b = 0; b < nb; ++b) beam[b] = cand[b];
        off += ipow(M, i + 1);
      }
      for (int32_t s = 0; s < k; ++s) {
        sel[t * k + s] = s < nb ? (int32_t)beam[s].p : -1;
        sel_score[t * k + s] = s < nb ? beam[s].s : -INFINITY;
      }
      if (gap) gap[t] = gmin;
    }
    free(cand);
    free(beam);
  }
}

/* ------------------------------------------------- S4: Eq. 3 + renormalisation
 * ok[t][s] = sel >= 0 and the expert responded (experts that "crashed
 * or taken too long" are excluded; reading X8: `responded` known at dispatch time).
 * w[t][s] = exp(g_s) / sum_{ok r} exp(g_r) over ok slots, 0 otherwise: the softmax of
 * Eq. 3 (denominator index typo read as f_j, reading X2),
 * renormalised over the responders "so that they still add up to 1".
 * Evaluated with the max shift m = max_ok g (the same value mathematically).
 * valid[t] = any ok; if none, the token is dropped (PAPER.md:287 footnote, reading X7).
 * Returns the number of dropped tokens. */
int64_t oracle_weights(const int32_t* sel, const double* sel_score, int64_t T, int32_t k,
                       const uint8_t* responded, double* w, uint8_t* ok, uint8_t* valid) {
  int64_t dropped = 0;
  for (int64_t t = 0; t < T; ++t) {
    double m = -INFINITY;
    int any = 0;
    for (int32_t s = 0; s < k; ++s) {
      int32_t e = sel[t * k + s];
      uint8_t o = (e >= 0 && responded[e]) ? 1 : 0;
      ok[t * k + s] = o;
      if (o) {
        any = 1;
        if (sel_score[t * k + s] > m) m = sel_score[t * k + s];
      }
    }
    double z = 0.0;
    for (int32_t s = 0; s < k; ++s)
      if (ok[t * k + s]) z += exp(sel_score[t * k + s] - m);
    for (int32_t s = 0; s < k; ++s)
      w[t * k + s] = ok[t * k + s] ? exp(sel_score[t * k + s] - m) / z : 0.0;
    valid[t] = (uint8_t)any;
    if (!any) ++dropped;
  }
  return dropped;
}

/* ------------------------------------------------------------- S5: dispatch
 * "Send inputs to those workers" (§3.1); the runtime "aggregates
 * requests into batches" per expert (§3.3).  Rows of expert e are the
 * ok pairs (t, s) with sel[t][s] == e, in increasing t (reading X18), appended in
 * that order; expert segments laid out by increasing e (= owner-rank-major order for
 * contiguous expert ownership).  counts, offsets (exclusive prefix sum of counts,
 * E+1 entries), row_of_slot (-1 if not ok), token_of_row. Returns R. */
int64_t oracle_dispatch(const int32_t* sel, const uint8_t* ok, int64_t T, int32_t k,
                        int64_t E, int32_t* counts, int32_t* offsets, int32_t* row_of_slot,
                        int32_t* token_of_row) {
  for (int64_t e = 0; e < E; ++e) counts[e] = 0;
  for (int64_t q = 0; q < T * k; ++q)
    if (ok[q]) counts[sel[q]]++;
  offsets[0] = 0;
  for (int64_t e = 0; e < E; ++e) offsets[e + 1] = offsets[e] + counts[e];
  int32_t* fill = (int32_t*)calloc((size_t)E, sizeof(int32_t));
  for (int64_t t = 0; t < T; ++t)
    for (int32_t s = 0; s < k; ++s) {
      int64_t q = t * k + s;
      if (!ok[q]) {
        row_of_slot[q] = -1;
        continue;
      }
      int32_t e = sel[q];
      int32_t r = offsets[e] + fill[e]++;
      row_of_slot[q] = r;
      token_of_row[r] = (int32_t)t;
    }
  free(fill);
  return offsets[E];
}

/* --------------------------------------------------------- S6: expert forward
 * The runtime's Forward request: "given inputs, compute and return expert outputs"
 * (§3.3).  Expert = 2-linear FFN D -> H -> D with bias and ReLU
 * (reading X14; PAPER.md:370 names the block family):
 *   h = W1_e x + b1_e;  a = max(h, 0);  out = W2_e a + b2_e.
 * Rows are grouped by expert slot: rows of slot s are [seg[s], seg[s+1]).
 * W1 [S][H][D], b1 [S][H], W2 [S][D][H], b2 [S][D] (torch Linear [out, in] layout).
 * Writes a (the post-ReLU activation) [R][H] and out [R][D]. */
void oracle_ffn_fwd(const double* x, const int32_t* seg, int32_t S, int32_t D, int32_t H,
                    const double* W1, const double* b1, const double* W2, const double* b2,
                    double* a, double* out) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int32_t s = 0; s < S; ++s) {
    const double* w1 = W1 + (int64_t)s * H * D;
    const double* w2 = W2 + (int64_t)s * D * H;
    for (int64_t r = seg[s]; r < seg[s + 1]; ++r) {
      for (int32_t n = 0; n < H; ++n) {
        double h = b1[(int64_t)s * H + n];
        for (int32_t c = 0; c < D; ++c) h += w1[(int64_t)n * D + c] * x[r * D + c];
        a[r * H + n] = h > 0.0 ? h : 0.0;
      }
      for (int32_t c = 0; c < D; ++c) {
        double o = b2[(int64_t)s * D + c];
        for (int32_t n = 0; n < H; ++n) o += w2[(int64_t)c * H + n] * a[r * H + n];
        out[r * D + c] = o;
      }
    }
  }
}

/* --------------------------------------------------------------- S7: combine
 * DMoE(x) = sum_{ok s} w_s f_s(x)  (Eq. 3 with the renormalised
 * weights of S4); a dropped token (no ok slot) gives 0 (reading X7). */
void oracle_combine(const double* out, const int32_t* row_of_slot, const double* w,
                    int64_t T, int32_t D, int32_t k, double* y) {
  #pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int32_t c = 0; c < D; ++c) {
      double acc = 0.0;
      for (int32_t s = 0; s < k; ++s) {
        int32_t r = row_of_slot[t * k + s];
        if (r >= 0) acc += w[t * k + s] * out[(int64_t)r * D + c];
      }
      y[t * D + c] = acc;
    }
}

/* ------------------------------------------------------ S8: combine backward
 * Given dY: a_ts = <dY_t, out_ts>, abar_t = sum_{ok r} w_tr a_tr,
 * dscore_ts = w_ts (a_ts - abar_t)  — the softmax Jacobian dw_s/dg_r = w_s(delta_sr - w_r)
 * restricted to the ok slots over which Eq. 3 is renormalised;
 * selection itself has no gradient (reading X12).  The expert cotangent sent with the
 * Backward request is g_row = w_ts dY_t. */
void oracle_combine_bwd(const double* dy, const double* out, const int32_t* row_of_slot,
                        const double* w, int64_t T, int32_t D, int32_t k, double* g_rows,
                        double* dscore) {
  #pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    double abar = 0.0;
    double* av = (double*)malloc(sizeof(double) * (size_t)k);
    for (int32_t s = 0; s < k; ++s) {
      int32_t r = row_of_slot[t * k + s];
      av[s] = 0.0;
      if (r < 0) continue;
      for (int32_t c = 0; c < D; ++c) av[s] += dy[t * D + c] * out[(int64_t)r * D + c];
      abar += w[t * k + s] * av[s];
    }
    for (int32_t s = 0; s < k; ++s) {
      int32_t r = row_of_slot[t * k + s];
      dscore[t * k + s] = r >= 0 ? w[t * k + s] * (av[s] - abar) : 0.0;
      if (r >= 0)
        for (int32_t c = 0; c < D; ++c) g_rows[(int64_t)r * D + c] = w[t * k + s] * dy[t * D + c];
    }
    free(av);
  }
}

/* -------------------------------------------------------- S9: expert backward
 * The runtime's Backward request: "given inputs and gradients of some function w.r.t.
 * outputs, compute gradients w.r.t. inputs" and the expert parameters.
 * Chain rule through out = W2 a + b2, a = relu(W1 x + b1), per row with cotangent g:
 *   dW2 += g a^T;  db2 += g;  delta = (W2^T g) * 1[h > 0];  dW1 += delta x^T;
 *   db1 += delta;  dx = W1^T delta.
 * ReLU'(0) = 0 (reading X13); 1[h > 0] == 1[a > 0].  Rows accumulate in row order.
 * Slots with no rows get zero gradients. */
void oracle_ffn_bwd(const double* x, const double* a, const double* g, const int32_t* seg,
                    int32_t S, int32_t D, int32_t H, const double* W1, const double* W2,
                    double* dx, double* dW1, double* db1, double* dW2, double* db2) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int32_t s = 0; s < S; ++s) {
    const double* w1 = W1 + (int64_t)s * H * D;
    const double* w2 = W2 + (int64_t)s * D * H;
    double* gw1 = dW1 + (int64_t)s * H * D;
    double* gw2 = dW2 + (int64_t)s * D * H;
    double* gb1 = db1 + (int64_t)s * H;
    double* gb2 = db2 + (int64_t)s * D;
    memset(gw1, 0, sizeof(double) * (size_t)H * D);
    memset(gw2, 0, sizeof(double) * (size_t)D * H);
    memset(gb1, 0, sizeof(double) * (size_t)H);
    memset(gb2, 0, sizeof(double) * (size_t)D);
    double* delta = (double*)malloc(sizeof(double) * (size_t)H);
    for (int64_t r = seg[s]; r < seg[s + 1]; ++r) {
      const double* gr = g + r * D;
      const double* ar = a + r * H;
      const double* xr = x + r * D;
      for (int32_t c = 0; c < D; ++c) {
        gb2[c] += gr[c];
        for (int32_t n = 0; n < H; ++n) gw2[(int64_t)c * H + n] += gr[c] * ar[n];
      }
      for (int32_t n = 0; n < H; ++n) {
        double v = 0.0;
        for (int32_t c = 0; c < D; ++c) v += w2[(int64_t)c * H + n] * gr[c];
        delta[n] = ar[n] > 0.0 ? v : 0.0;
        gb1[n] += delta[n];
        for (int32_t c = 0; c < D; ++c) gw1[(int64_t)n * D + c] += delta[n] * xr[c];
      }
      for (int32_t c = 0; c < D; ++c) {
        double v = 0.0;
        for (int32_t n = 0; n < H; ++n) v += w1[(int64_t)n * D + c] * delta[n];
        dx[r * D + c] = v;
      }
    }
    free(delta);
  }
}

/* ------------------------------------------------ S10: gate backward + undispatch
 * dX_t = sum_{ok s} dx_row(t,s) + sum_s dscore_ts * sum_i W_g[:, i*M + u_i(sel_ts)]
 * dG[t][i*M+j] = sum_{s: sel_ts >= 0, u_i(sel_ts) = j} dscore_ts
 * dW_g = sum_t X_t (x) dG_t;  db_g = sum_t dG_t
 * — the gradient of Eq. 2 (g(x,f) = sum_i g_i(x, uid_i(f)), g_i affine; PAPER.md:
 * 238-246) composed with the softmax gradient of S8; the expert path returns dx rows
 * (PAPER.md:322).  u_i(e) = (e / M^{d-1-i}) mod M (reading X1). */
void oracle_gate_bwd(const double* X, const double* Wg, const int32_t* sel,
                     const double* dscore, const double* dx_rows, const int32_t* row_of_slot,
                     int64_t T, int32_t D, int32_t d, int32_t M, int32_t k, double* dX,
                     double* dWg, double* dbg) {
  int32_t dM = d * M;
  double* dG = (double*)calloc((size_t)T * dM, sizeof(double));
  for (int64_t t = 0; t < T; ++t)
    for (int32_t s = 0; s < k; ++s) {
      int32_t e = sel[t * k + s];
      if (e < 0) continue;
      for (int32_t i = 0; i < d; ++i) {
        int64_t u = (e / ipow(M, d - 1 - i)) % M;
        dG[t * dM + i * M + u] += dscore[t * k + s];
      }
    }
  #pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    for (int32_t c = 0; c < D; ++c) {
      double v = 0.0;
      for (int32_t s = 0; s < k; ++s) {
        int32_t r = row_of_slot[t * k + s];
        if (r >= 0) v += dx_rows[(int64_t)r * D + c];
      }
      for (int32_t col = 0; col < dM; ++col) v += dG[t * dM + col] * Wg[(int64_t)c * dM + col];
      dX[t * D + c] = v;
    }
  #pragma omp parallel for schedule(static)
  for (int32_t c = 0; c < D; ++c)
    for (int32_t col = 0; col < dM; ++col) {
      double v = 0.0;
      for (int64_t t = 0; t < T; ++t) v += X[t * D + c] * dG[t * dM + col];
      dWg[(int64_t)c * dM + col] = v;
    }
  for (int32_t col = 0; col < dM; ++col) {
    double v = 0.0;
    for (int64_t t = 0; t < T; ++t) v += dG[t * dM + col];
    dbg[col] = v;
  }
  free(dG);
}
