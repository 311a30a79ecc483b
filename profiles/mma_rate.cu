// Micro-benchmark: issue rate of tcgen05.mma.kind::tf32 (cta_group::1, M = 128)
// for K-major / MN-major operands and several N, one CTA per SM, operands in
// shared memory (contents irrelevant).  Prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate profiles/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)lay << 61);
}

// mode 0: one shape; mode 1: alternate N and N/2 on the same accumulator;
// mode 2: mode 1 + a commit every 8 MMAs
__global__ void bench(int n, int mn, int kind, int iters, long long* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x * 4; i < 96 * 1024; i += blockDim.x * 4) *(float*)(sm + i) = 0.f;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    uint32_t idesc;
    if (kind == 0)  // tf32
      idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) |
              ((uint32_t)(n >> 3) << 17) | (8u << 24);
    else  // bf16
      idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) |
              ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    uint64_t ad, bd;
    if (mn) {
      ad = sdesc(a, 4096, 512, 1);
      bd = sdesc(b, 4096, 512, 1);
    } else {
      ad = sdesc(a, 16, 1024, 2);
      bd = sdesc(b, 16, 1024, 2);
    }
    const uint32_t idesc2 = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(n >> 4) << 17);
    __shared__ __align__(8) uint64_t bar2;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t id = (mode && (i & 1)) ? idesc2 : idesc;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tbase),
          "l"(ad), "l"(bd), "r"(id), "r"(1));
      if (mode == 2 && (i & 7) == 7)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int mn = 0; mn < 2; ++mn)
      for (int n : {64, 128, 256}) {
        if (mode && n == 64) continue;
        bench<<<148, 128, 96 * 1024>>>(n, mn, 0, iters, d, mode);
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        printf("mode %d tf32 %s N=%3d: %.1f cycles/MMA  %s\n", mode, mn ? "MN-major" : "K-major ", n,
               (double)c / iters, cudaGetErrorString(e));
      }
  return 0;
}
