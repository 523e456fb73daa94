/* gen/counter_gen.h — counter-based synthetic input generator.
 *
 * This module is the ONE piece shared by the float64 oracle side (host, via
 * gen_host.c) and the GPU side (device, via gen_device.cu).  It holds none of
 * the DMoE method's arithmetic: it only maps (seed, tensor_id, flat_index) to
 * a value, so that either side can regenerate any element of any input tensor
 * without storing it.
 *
 * Every function is a pure integer hash followed by at most ONE IEEE fp32
 * multiply of an exactly representable integer, so host (x86-64 SSE) and
 * device (sm_100a) produce bit-identical floats.  No FMA contraction is
 * possible (there is no add after a multiply).  bf16 rounding is done here in
 * integer arithmetic (round-to-nearest-even, the same rule as
 * torch.Tensor.to(torch.bfloat16) / cvt.rn.bf16.f32).
 */
#ifndef DMOE_COUNTER_GEN_H
#define DMOE_COUNTER_GEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define CG_FN static __host__ __device__ __forceinline__
#else
#define CG_FN static inline
#endif

/* tensor ids (stable; part of the recipe) */
enum {
  CG_X = 1, CG_WG = 2, CG_BG = 3, CG_W1 = 4, CG_B1 = 5, CG_W2 = 6, CG_B2 = 7,
  CG_DY = 8, CG_ALIVE = 9, CG_RESPONDED = 10
};

/* distributions */
enum {
  CG_NORMAL = 0,     /* ~N(0,1): Irwin-Hall sum of four 16-bit uniforms, standardised */
  CG_UNIFORM = 1,    /* U(-a, a) with 24-bit resolution */
  CG_GRID8 = 2,      /* exact-grid mode: {-7..7}/8, exact in bf16 and fp32 */
  CG_ZERO = 3
};

CG_FN uint64_t cg_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

CG_FN uint64_t cg_hash(uint64_t seed, uint32_t tensor_id, uint64_t idx) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ULL + (uint64_t)tensor_id * 0xD1B54A32D192ED03ULL;
  z = cg_mix(z);
  return cg_mix(z + idx * 0x9E3779B97F4A7C15ULL + 0x632BE59BD9B4E019ULL);
}

/* value before any precision reduction.  `scale` multiplies the unit
 * distribution: NORMAL -> N(0, scale^2); UNIFORM -> U(-scale, scale);
 * GRID8 ignores scale. */
CG_FN float cg_value(uint64_t seed, uint32_t tensor_id, uint64_t idx, int dist, float scale) {
  uint64_t h = cg_hash(seed, tensor_id, idx);
  if (dist == CG_NORMAL) {
    int32_t s = (int32_t)(h & 0xFFFFu) + (int32_t)((h >> 16) & 0xFFFFu) +
                (int32_t)((h >> 32) & 0xFFFFu) + (int32_t)((h >> 48) & 0xFFFFu) - 131070;
    /* std of the centred sum = 65536/sqrt(3) (to 1e-9 relative); the
     * constant folds scale in with one fp32 multiply on each side. */
    float c = scale * (1.0f / 37837.22f);
    return (float)s * c;
  } else if (dist == CG_UNIFORM) {
    int32_t n = (int32_t)(h >> 40) - (1 << 23); /* in [-2^23, 2^23) */
    float c = scale * (1.0f / 8388608.0f);       /* exact power-of-two rescale of scale */
    return (float)n * c;
  } else if (dist == CG_GRID8) {
    int32_t q = (int32_t)((h >> 11) % 15u) - 7;
    return (float)q * 0.125f;
  }
  return 0.0f;
}

/* fp32 -> bf16 bits, round-to-nearest-even (NaN kept quiet). */
CG_FN uint16_t cg_f32_to_bf16(float f) {
  union { float f; uint32_t u; } v;
  v.f = f;
  uint32_t u = v.u;
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40u);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

CG_FN float cg_bf16_to_f32(uint16_t b) {
  union { float f; uint32_t u; } v;
  v.u = ((uint32_t)b) << 16;
  return v.f;
}

/* Bernoulli mask bit: 1 with probability 1 - thr/2^24 ("alive"/"responded"
 * drawn i.i.d. per expert; thr = round(f * 2^24) for failure fraction f). */
CG_FN uint32_t cg_keep_bit(uint64_t seed, uint32_t tensor_id, uint64_t idx, uint32_t thr) {
  uint64_t h = cg_hash(seed, tensor_id, idx);
  return (uint32_t)(h >> 40) >= thr ? 1u : 0u;
}

#endif
