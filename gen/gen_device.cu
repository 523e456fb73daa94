/* gen/gen_device.cu — device side of the counter-based input generator.
 * Same element formula as gen_host.c (both include counter_gen.h), used by
 * bench.py and the GPU tests to fill HBM-resident inputs without a host
 * round trip.  Not part of the DMoE library (libdmoe.so). */
#include "counter_gen.h"
#include <cuda_runtime.h>

__global__ void k_fill_f32(uint64_t seed, uint32_t tid, int dist, float scale,
                           uint64_t idx0, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cg_value(seed, tid, idx0 + (uint64_t)i, dist, scale);
}

__global__ void k_fill_bf16(uint64_t seed, uint32_t tid, int dist, float scale,
                            uint64_t idx0, int64_t n, uint16_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cg_f32_to_bf16(cg_value(seed, tid, idx0 + (uint64_t)i, dist, scale));
}

__global__ void k_fill_mask(uint64_t seed, uint32_t tid, uint32_t thr, int64_t nbits, uint32_t* out) {
  int64_t nw = (nbits + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      int64_t e = w * 32 + b;
      if (e < nbits && cg_keep_bit(seed, tid, (uint64_t)e, thr)) v |= 1u << b;
    }
    out[w] = v;
  }
}

static int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

extern "C" int gen_dev_fill_f32(uint64_t seed, uint32_t tid, int dist, float scale,
                                uint64_t idx0, int64_t n, float* out, cudaStream_t s) {
  if (n <= 0) return 0;
  k_fill_f32<<<grid_for(n), 256, 0, s>>>(seed, tid, dist, scale, idx0, n, out);
  return (int)cudaGetLastError();
}
extern "C" int gen_dev_fill_bf16(uint64_t seed, uint32_t tid, int dist, float scale,
                                 uint64_t idx0, int64_t n, uint16_t* out, cudaStream_t s) {
  if (n <= 0) return 0;
  k_fill_bf16<<<grid_for(n), 256, 0, s>>>(seed, tid, dist, scale, idx0, n, out);
  return (int)cudaGetLastError();
}
extern "C" int gen_dev_fill_mask(uint64_t seed, uint32_t tid, uint32_t thr, int64_t nbits,
                                 uint32_t* out, cudaStream_t s) {
  if (nbits <= 0) return 0;
  k_fill_mask<<<grid_for((nbits + 31) / 32), 256, 0, s>>>(seed, tid, thr, nbits, out);
  return (int)cudaGetLastError();
}
