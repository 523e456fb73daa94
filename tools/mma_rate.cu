// tcgen05.mma issue/execution rate on one SM per CTA: cycles per MMA (M=128, K=16, bf16 -> fp32,
// both operands in 128B-swizzled smem) for K-major / MN-major operands and N = 128 / 256, as a
// back-to-back burst and in the weight-gradient pattern (4 MMAs, commit, wait, repeat).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (uint64_t)((lbo >> 4) & 0x3FFF) << 16 |
         (uint64_t)((sbo >> 4) & 0x3FFF) << 32 | (uint64_t)1 << 46 | (uint64_t)2 << 61;
}
__host__ __device__ constexpr uint32_t idesc(int n, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(s32(bar)),
               "r"(ph) : "memory");
}

template <int N, bool MN>
__global__ void k_rate(int mode, int iters, long long* out) {
  extern __shared__ __align__(128) char sm[];
  char* base = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  char* A = base;                 // 128 x 64 bf16 (16 KB)
  char* B = base + 16384;         // N x 64 bf16
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x * 16; i < 16384 + N * 128; i += blockDim.x * 16) *(uint4*)(base + i) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc(N, MN, MN);
    uint32_t ph = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = MN ? desc(s32(A) + k * 2048, 8192, 1024) : desc(s32(A) + k * 32, 16, 1024);
        const uint64_t bd = MN ? desc(s32(B) + k * 2048, 8192, 1024) : desc(s32(B) + k * 32, 16, 1024);
        mma(tm + (it & 1) * N, ad, bd, id, k != 0);
      }
      if (mode == 1) {  // per-tile commit + wait (serialised tiles)
        commit(&bar);
        wait(&bar, ph);
        ph ^= 1;
      } else if (mode == 2) {  // commit per tile, no wait (like the empty-slot commits)
        commit(&bar);
      }
    }
    commit(&bar2);
    wait(&bar2, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, bool MN>
void run(const char* name, int sms, long long* d) {
  auto k = k_rate<N, MN>;
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<sms, 128, smem>>>(mode, iters, d);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-22s mode %d (%s): %6.1f cyc per MMA (floor %d)\n", name, mode,
           mode == 0 ? "burst" : mode == 1 ? "commit+wait per 4" : "commit per 4, no wait", (double)mx / (iters * 4),
           128 * N / 256);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 256);
  run<128, false>("N=128 K-major", sms, d);
  run<128, true>("N=128 MN-major", sms, d);
  run<256, false>("N=256 K-major", sms, d);
  run<256, true>("N=256 MN-major", sms, d);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
