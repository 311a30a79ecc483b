// Micro-benchmark: HBM read bandwidth through TMA 2-D tiled loads into a
// shared-memory ring (one CTA per SM, one producer thread, the consumer
// releases each stage as soon as it lands).  Varies box rows, ring depth and
// the matrix row pitch, to size the tensor-core GEMMs' stage rings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate profiles/tma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait(uint64_t* bar, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(bar)),
      "r"(ph)
      : "memory");
}

// each stage = `boxes` boxes of (32 fp32 x rows) stacked along the columns
__global__ void bench(const __grid_constant__ CUtensorMap map, int64_t nrow_blocks, int rows,
                      int boxes, int stages) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t box_bytes = rows * 128, stage_bytes = box_bytes * boxes;
  const int64_t mine = nrow_blocks > blockIdx.x ? (nrow_blocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    int slot = 0;
    unsigned ph = 0;
    int64_t blk = blockIdx.x;
    for (int64_t i = 0; i < mine; ++i, blk += gridDim.x) {
      wait(&empty[slot], ph ^ 1u);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])),
                   "r"(stage_bytes));
      for (int g = 0; g < boxes; ++g)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                "r"(su32(sm + slot * stage_bytes + g * box_bytes)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(g * 32), "r"((int)(blk * rows)),
            "r"(su32(&full[slot]))
            : "memory");
      if (++slot == stages) slot = 0, ph ^= 1u;
    }
  } else if (threadIdx.x == 32) {
    int slot = 0;
    unsigned ph = 0;
    for (int64_t i = 0; i < mine; ++i) {
      wait(&full[slot], ph);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
      if (++slot == stages) slot = 0, ph ^= 1u;
    }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  const int64_t F = 1600000;
  float* buf;
  cudaMalloc(&buf, F * 256 * 4);
  cudaMemset(buf, 0, F * 256 * 4);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int cols, rows, stages, l2; } cfgs[] = {
      {64, 128, 6, 3},  {64, 128, 3, 3},  {64, 64, 6, 3},   {64, 32, 6, 3},  {64, 128, 12, 3},
      {64, 256, 3, 3},  {64, 128, 6, 0},  {64, 128, 6, 2},  {256, 32, 4, 3}, {256, 16, 8, 3},
      {256, 64, 2, 3},  {256, 32, 6, 3},  {256, 16, 12, 3}, {128, 64, 6, 3}, {128, 128, 3, 3}};
  for (auto c : cfgs) {
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)c.cols, (cuuint64_t)F};
    const cuuint64_t str[1] = {(cuuint64_t)c.cols * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)c.rows};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     (CUtensorMapL2promotion)c.l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int boxes = c.cols / 32;
    const int64_t nb = F / c.rows;
    const size_t smem = (size_t)c.rows * 128 * boxes * c.stages;
    if (smem > 200 * 1024 || r != CUDA_SUCCESS) {
      printf("skip cols=%d rows=%d stages=%d\n", c.cols, c.rows, c.stages);
      continue;
    }
    bench<<<148, 64, smem>>>(map, nb, c.rows, boxes, c.stages);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) bench<<<148, 64, smem>>>(map, nb, c.rows, boxes, c.stages);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const double bytes = (double)nb * c.rows * c.cols * 4;
    printf("cols=%3d box_rows=%3d stages=%2d stage=%3zuKB ring=%3zuKB l2promo=%d: %.0f GB/s  %s\n", c.cols,
           c.rows, c.stages, (size_t)c.rows * 128 * boxes / 1024, smem / 1024, c.l2, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
