/* gen/gen_host.c — host side of the counter-based input generator.
 * Fills caller-owned host arrays with elements [idx0, idx0+n) of a tensor.
 * Shared with nothing but gen/counter_gen.h (see that header). */
#include "counter_gen.h"
#include <stddef.h>

void gen_fill_f32(uint64_t seed, uint32_t tid, int dist, float scale,
                  uint64_t idx0, int64_t n, float* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = cg_value(seed, tid, idx0 + (uint64_t)i, dist, scale);
}

void gen_fill_bf16(uint64_t seed, uint32_t tid, int dist, float scale,
                   uint64_t idx0, int64_t n, uint16_t* out) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    out[i] = cg_f32_to_bf16(cg_value(seed, tid, idx0 + (uint64_t)i, dist, scale));
}

/* packed little-endian bit mask: bit e of word e/32 */
void gen_fill_mask(uint64_t seed, uint32_t tid, uint32_t thr, int64_t nbits, uint32_t* out) {
  int64_t nw = (nbits + 31) / 32;
  for (int64_t w = 0; w < nw; ++w) {
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      int64_t e = w * 32 + b;
      if (e < nbits && cg_keep_bit(seed, tid, (uint64_t)e, thr)) v |= 1u << b;
    }
    out[w] = v;
  }
}
