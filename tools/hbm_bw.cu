// HBM bandwidth ceilings for the access patterns the layer's kernels use: pure 16-byte writes
// (plain / streaming), bulk-async writes from shared memory (the weight-gradient epilogue's
// path), pure 16-byte reads, and copies.  CUDA events, best of 10, 4 GiB buffers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_bw tools/hbm_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void k_write(uint4* p, size_t n, int cs) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    if (cs) __stcs(p + i, v);
    else p[i] = v;
  }
}
__global__ void k_read(const uint4* p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_copy(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
// bulk async stores (cp.async.bulk global <- shared), CHUNK bytes each, DEPTH in flight per warp
template <int CHUNK, int DEPTH>
__global__ void k_bulk_write(char* p, size_t bytes) {
  extern __shared__ __align__(128) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  char* buf = sm + warp * CHUNK;
  for (int i = lane * 16; i < CHUNK; i += 512) *reinterpret_cast<uint4*>(buf + i) = make_uint4(1, 2, 3, 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    const size_t nchunks = bytes / CHUNK;
    for (size_t c = (size_t)blockIdx.x * nw + warp; c < nchunks; c += (size_t)gridDim.x * nw) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * CHUNK),
                   "r"((uint32_t)__cvta_generic_to_shared(buf)), "r"(CHUNK)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// the weight-gradient epilogue's store pattern: 128 x 128 bf16 tiles of an [R, N] matrix, each
// as 8 boxes of 32 rows x 64 columns (one per warp, 128B-swizzled), double-buffered per warp
__global__ void k_tile_store(const __grid_constant__ CUtensorMap tm, int MT, int NT, int hint) {
  extern __shared__ __align__(128) char sm[];
  char* base = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* buf = base + warp * 8192;
  for (int i = lane * 16; i < 8192; i += 512) *reinterpret_cast<uint4*>(buf + i) = make_uint4(1, 2, 3, 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int b = 0;
  if (lane == 0)
    for (int t = blockIdx.x; t < MT * NT; t += gridDim.x) {
      const int mt = t / NT, nt = t % NT;
      const int col = nt * 128 + (warp >> 2) * 64, row = mt * 128 + (warp & 3) * 32;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(buf + b * 4096);
      if (hint)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(&tm),
                     "r"(src), "r"(col), "r"(row), "l"(pol) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                     "r"(src), "r"(col), "r"(row) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      b ^= 1;
    }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA loads into an S-stage ring of 32 KB stages (4 boxes of 64 x 64 bf16), consumer warp only
// waits full / arrives empty: the operand-load ceiling of one SM without any math.
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}
__global__ void k_tma_ring(const __grid_constant__ CUtensorMap tm, int S, int iters, int rows) {
  extern __shared__ __align__(128) char sm2[];
  char* base = (char*)(((uintptr_t)sm2 + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + S * 32768);
  uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(empty + i)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      mb_wait((uint32_t)__cvta_generic_to_shared(empty + st), ph ^ 1);
      const uint32_t fb = (uint32_t)__cvta_generic_to_shared(full + st);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(32768) : "memory");
      const int row = (int)(((unsigned)(blockIdx.x * 7919 + it * 131) * 64u) % (unsigned)(rows - 64));
      for (int c = 0; c < 4; ++c) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(base + st * 32768 + c * 8192);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
                     "l"(&tm), "r"(fb), "r"(c * 64), "r"(row) : "memory");
      }
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      mb_wait((uint32_t)__cvta_generic_to_shared(full + st), ph);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(empty + st)) : "memory");
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <class F>
float best_ms(F f) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  f();
  cudaDeviceSynchronize();
  float best = 1e9f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(s);
    f();
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const size_t bytes = (size_t)4 << 30, n = bytes / 16;
  char *a, *b;
  unsigned* o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&o, 4);
  cudaMemset(a, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {2, 4, 8}) {
    const int g = sms * per;
    float w = best_ms([&] { k_write<<<g, 512>>>((uint4*)b, n, 0); });
    float wc = best_ms([&] { k_write<<<g, 512>>>((uint4*)b, n, 1); });
    float r = best_ms([&] { k_read<<<g, 512>>>((const uint4*)a, n, o); });
    float c = best_ms([&] { k_copy<<<g, 512>>>((const uint4*)a, (uint4*)b, n); });
    printf("grid %4d x512: write %6.0f  write.cs %6.0f  read %6.0f  copy %6.0f (read+write) GB/s\n", g,
           bytes / w / 1e6, bytes / wc / 1e6, bytes / r / 1e6, 2 * bytes / c / 1e6);
  }
  {
    auto k = k_bulk_write<4096, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096);
    float t = best_ms([&] { k<<<sms, 256, 8 * 4096>>>(b, bytes); });
    printf("bulk store 4 KB x 2 in flight, 8 warps/SM: %6.0f GB/s\n", bytes / t / 1e6);
    auto k2 = k_bulk_write<4096, 4>;
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096);
    t = best_ms([&] { k2<<<sms, 512, 16 * 4096>>>(b, bytes); });
    printf("bulk store 4 KB x 4 in flight, 16 warps/SM: %6.0f GB/s\n", bytes / t / 1e6);
    auto k3 = k_bulk_write<16384, 2>;
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    t = best_ms([&] { k3<<<sms, 256, 8 * 16384>>>(b, bytes); });
    printf("bulk store 16 KB x 2 in flight, 8 warps/SM: %6.0f GB/s\n", bytes / t / 1e6);
  }
  {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)f;
    cudaFuncSetAttribute(k_tile_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192 + 1024);
    for (int N : {256, 1024, 4096}) {
      const uint64_t R = bytes / (2 * (uint64_t)N);
      CUtensorMap tm;
      cuuint64_t gdim[2] = {(cuuint64_t)N, R}, gstr[1] = {(cuuint64_t)N * 2};
      cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int hint : {0, 1}) {
        for (int per : {1, 2}) {
          float t = best_ms([&] { k_tile_store<<<sms * per, 256, 8 * 8192 + 1024>>>(tm, (int)(R / 128), N / 128, hint); });
          printf("tile store N=%4d (128x128 tiles, 8 boxes 32x64): hint %d, %d CTA/SM: %6.0f GB/s\n", N, hint, per,
                 bytes / t / 1e6);
        }
      }
    }
  }
  {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)f;
    cudaFuncSetAttribute(k_tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 2048);
    for (size_t mb : {(size_t)32, (size_t)4096}) {
      const uint64_t N = 256, R = (mb << 20) / (N * 2);
      CUtensorMap tm;
      cuuint64_t gdim[2] = {N, R}, gstr[1] = {N * 2};
      cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int S : {2, 4, 6}) {
        const int iters = 4000;
        float t = best_ms([&] { k_tma_ring<<<sms, 64, S * 32768 + 2048>>>(tm, S, iters, (int)R); });
        printf("TMA ring loads from a %5zu MB buffer, %d x 32 KB stages: %6.0f GB/s (%.2f us per stage per SM)\n", mb, S,
               (double)sms * iters * 32768 / t / 1e6, t * 1e3 / iters);
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
