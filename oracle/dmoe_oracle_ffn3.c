/* dmoe_oracle_ffn3.c — float64 oracle of the paper's own expert block (NEXT-2).
 *
 * TEST INFRASTRUCTURE ONLY (see dmoe_oracle.c): plain loops, no BLAS, no code shared with the
 * CUDA path.  PAPER.md:370 (§4.1): the experts are "feedforward blocks 1024 -> 4096 -> 4096 ->
 * 1024 with layer normalization and ReLU activations in between" (§4.2, uses the
 * same block at 1/4 of the size).  Reading X23: three linears with bias, and between
 * them LayerNorm over the H features (learnable per-expert scale g and shift be, biased
 * variance, eps) followed by ReLU:
 *   z1 = W1 x + b1;   a1 = relu(g1 * (z1 - mean z1) / sqrt(var z1 + eps) + be1)
 *   z2 = W2 a1 + b2;  a2 = relu(g2 * (z2 - mean z2) / sqrt(var z2 + eps) + be2)
 *   out = W3 a2 + b3
 * W1 [S][H][D], W2 [S][H][H], W3 [S][D][H] (torch Linear [out, in]); b1, g1, be1, b2, g2, be2
 * [S][H]; b3 [S][D].  Rows of slot s are [seg[s], seg[s+1]).  ReLU'(0) = 0 (reading X13). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* y = LN(z) with scale g / shift be; also returns xhat and rstd */
static void ln_row(const double* z, const double* g, const double* be, int32_t H, double eps,
                   double* xhat, double* y, double* rstd) {
  double mu = 0.0, var = 0.0;
  for (int32_t n = 0; n < H; ++n) mu += z[n];
  mu /= H;
  for (int32_t n = 0; n < H; ++n) var += (z[n] - mu) * (z[n] - mu);
  var /= H;
  *rstd = 1.0 / sqrt(var + eps);
  for (int32_t n = 0; n < H; ++n) {
    xhat[n] = (z[n] - mu) * (*rstd);
    y[n] = g[n] * xhat[n] + be[n];
  }
}

void oracle_ffn3_fwd(const double* x, const int32_t* seg, int32_t S, int32_t D, int32_t H,
                     const double* W1, const double* b1, const double* g1, const double* be1,
                     const double* W2, const double* b2, const double* g2, const double* be2,
                     const double* W3, const double* b3, double eps,
                     double* z1, double* a1, double* z2, double* a2, double* out, double* y1, double* y2) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int32_t s = 0; s < S; ++s) {
    double* xh = (double*)malloc(sizeof(double) * (size_t)H);
    double* y = (double*)malloc(sizeof(double) * (size_t)H);
    const double* w1 = W1 + (int64_t)s * H * D;
    const double* w2 = W2 + (int64_t)s * H * H;
    const double* w3 = W3 + (int64_t)s * D * H;
    for (int64_t r = seg[s]; r < seg[s + 1]; ++r) {
      double rstd;
      for (int32_t n = 0; n < H; ++n) {
        double v = b1[(int64_t)s * H + n];
        for (int32_t c = 0; c < D; ++c) v += w1[(int64_t)n * D + c] * x[r * D + c];
        z1[r * H + n] = v;
      }
      ln_row(z1 + r * H, g1 + (int64_t)s * H, be1 + (int64_t)s * H, H, eps, xh, y, &rstd);
      for (int32_t n = 0; n < H; ++n) a1[r * H + n] = y[n] > 0.0 ? y[n] : 0.0;
      if (y1) memcpy(y1 + r * H, y, sizeof(double) * (size_t)H);
      for (int32_t m = 0; m < H; ++m) {
        double v = b2[(int64_t)s * H + m];
        for (int32_t n = 0; n < H; ++n) v += w2[(int64_t)m * H + n] * a1[r * H + n];
        z2[r * H + m] = v;
      }
      ln_row(z2 + r * H, g2 + (int64_t)s * H, be2 + (int64_t)s * H, H, eps, xh, y, &rstd);
      for (int32_t m = 0; m < H; ++m) a2[r * H + m] = y[m] > 0.0 ? y[m] : 0.0;
      if (y2) memcpy(y2 + r * H, y, sizeof(double) * (size_t)H);
      for (int32_t c = 0; c < D; ++c) {
        double v = b3[(int64_t)s * D + c];
        for (int32_t m = 0; m < H; ++m) v += w3[(int64_t)c * H + m] * a2[r * H + m];
        out[r * D + c] = v;
      }
    }
    free(xh);
    free(y);
  }
}

/* LayerNorm + ReLU backward for one row: dy = da * 1[y > 0]; dg += dy * xhat; dbe += dy;
 * dxhat = dy * g;  dz = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)).
 * mask (optional, NULL = 1[y > 0]): the ReLU decisions to take instead (forced-decision parity,
 * reading X23b: a decision within floating-point noise of y = 0 is taken from the kernel). */
static void ln_relu_bwd_row(const double* z, const double* g, const double* be, const double* da,
                            int32_t H, double eps, double* xh, double* y, double* dz, double* dg,
                            double* dbe, const uint8_t* mask) {
  double rstd;
  ln_row(z, g, be, H, eps, xh, y, &rstd);
  double m1 = 0.0, m2 = 0.0;
  for (int32_t n = 0; n < H; ++n) {
    const int on = mask ? mask[n] != 0 : y[n] > 0.0;
    const double dy = on ? da[n] : 0.0;
    dg[n] += dy * xh[n];
    dbe[n] += dy;
    dz[n] = dy * g[n];  /* dxhat */
    m1 += dz[n];
    m2 += dz[n] * xh[n];
  }
  m1 /= H;
  m2 /= H;
  for (int32_t n = 0; n < H; ++n) dz[n] = rstd * (dz[n] - m1 - xh[n] * m2);
}

/* The Backward request of the block, per row with cotangent gr [D]: the chain
 * rule through out, LN2 + ReLU, the middle linear, LN1 + ReLU and the first linear.  Gradients
 * accumulate over the slot's rows in row order; slots without rows get zeros. */
void oracle_ffn3_bwd(const double* x, const double* z1, const double* a1, const double* z2,
                     const double* a2, const double* gr, const int32_t* seg, int32_t S, int32_t D,
                     int32_t H, const double* W1, const double* g1, const double* be1,
                     const double* W2, const double* g2, const double* be2, const double* W3,
                     double eps, double* dx, double* dW1, double* db1, double* dg1, double* dbe1,
                     double* dW2, double* db2, double* dg2, double* dbe2, double* dW3, double* db3,
                     const uint8_t* m1, const uint8_t* m2) {
  #pragma omp parallel for schedule(dynamic, 1)
  for (int32_t s = 0; s < S; ++s) {
    const double* w1 = W1 + (int64_t)s * H * D;
    const double* w2 = W2 + (int64_t)s * H * H;
    const double* w3 = W3 + (int64_t)s * D * H;
    double* gW1 = dW1 + (int64_t)s * H * D;
    double* gW2 = dW2 + (int64_t)s * H * H;
    double* gW3 = dW3 + (int64_t)s * D * H;
    memset(gW1, 0, sizeof(double) * (size_t)H * D);
    memset(gW2, 0, sizeof(double) * (size_t)H * H);
    memset(gW3, 0, sizeof(double) * (size_t)D * H);
    memset(db1 + (int64_t)s * H, 0, sizeof(double) * (size_t)H);
    memset(dg1 + (int64_t)s * H, 0, sizeof(double) * (size_t)H);
    memset(dbe1 + (int64_t)s * H, 0, sizeof(double) * (size_t)H);
    memset(db2 + (int64_t)s * H, 0, sizeof(double) * (size_t)H);
    memset(dg2 + (int64_t)s * H, 0, sizeof(double) * (size_t)H);
    memset(dbe2 + (int64_t)s * H, 0, sizeof(double) * (size_t)H);
    memset(db3 + (int64_t)s * D, 0, sizeof(double) * (size_t)D);
    double* xh = (double*)malloc(sizeof(double) * (size_t)H);
    double* y = (double*)malloc(sizeof(double) * (size_t)H);
    double* da = (double*)malloc(sizeof(double) * (size_t)H);
    double* dz = (double*)malloc(sizeof(double) * (size_t)H);
    for (int64_t r = seg[s]; r < seg[s + 1]; ++r) {
      const double* g = gr + r * D;
      /* out = W3 a2 + b3 */
      for (int32_t c = 0; c < D; ++c) {
        db3[(int64_t)s * D + c] += g[c];
        for (int32_t m = 0; m < H; ++m) gW3[(int64_t)c * H + m] += g[c] * a2[r * H + m];
      }
      for (int32_t m = 0; m < H; ++m) {
        double v = 0.0;
        for (int32_t c = 0; c < D; ++c) v += w3[(int64_t)c * H + m] * g[c];
        da[m] = v;
      }
      ln_relu_bwd_row(z2 + r * H, g2 + (int64_t)s * H, be2 + (int64_t)s * H, da, H, eps, xh, y, dz,
                      dg2 + (int64_t)s * H, dbe2 + (int64_t)s * H, m2 ? m2 + r * H : NULL);
      /* z2 = W2 a1 + b2 */
      for (int32_t m = 0; m < H; ++m) {
        db2[(int64_t)s * H + m] += dz[m];
        for (int32_t n = 0; n < H; ++n) gW2[(int64_t)m * H + n] += dz[m] * a1[r * H + n];
      }
      for (int32_t n = 0; n < H; ++n) {
        double v = 0.0;
        for (int32_t m = 0; m < H; ++m) v += w2[(int64_t)m * H + n] * dz[m];
        da[n] = v;
      }
      ln_relu_bwd_row(z1 + r * H, g1 + (int64_t)s * H, be1 + (int64_t)s * H, da, H, eps, xh, y, dz,
                      dg1 + (int64_t)s * H, dbe1 + (int64_t)s * H, m1 ? m1 + r * H : NULL);
      /* z1 = W1 x + b1 */
      for (int32_t n = 0; n < H; ++n) {
        db1[(int64_t)s * H + n] += dz[n];
        for (int32_t c = 0; c < D; ++c) gW1[(int64_t)n * D + c] += dz[n] * x[r * D + c];
      }
      for (int32_t c = 0; c < D; ++c) {
        double v = 0.0;
        for (int32_t n = 0; n < H; ++n) v += w1[(int64_t)n * D + c] * dz[n];
        dx[r * D + c] = v;
      }
    }
    free(xh);
    free(y);
    free(da);
    free(dz);
  }
}
