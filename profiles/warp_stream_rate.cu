// Access-pattern probe for the GAE kernel (DESIGN.md §8 item 1): does HBM
// bandwidth drop when every warp streams its own contiguous region (the
// segmented GAE's per-warp trajectory ranges: ~2,400 warps x 2 read + 2 write
// streams, ~1.5 KB per chunk) instead of the grid sweeping memory together?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wsr profiles/warp_stream_rate.cu
//   /tmp/wsr
//
// Both kernels move the same bytes (2 reads + 2 writes of 4 B per element,
// 25.5 M elements = the 64 K-trajectory cfg2 batch) with 4-byte coalesced warp
// rows.  "sweep": grid-stride rows (neighbouring warps touch neighbouring
// addresses at the same time); "private": warp w owns elements
// [w*N/W, (w+1)*N/W) and walks them in chunk-sized steps.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void sweep(const float* __restrict__ a, const float* __restrict__ b,
                      float* __restrict__ x, float* __restrict__ y, long n) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float u = __ldcs(a + i), v = __ldcs(b + i);
    __stcs(x + i, u + v);
    __stcs(y + i, u - v);
  }
}

template <int kRows>
__global__ void priv(const float* __restrict__ a, const float* __restrict__ b,
                     float* __restrict__ x, float* __restrict__ y, long n) {
  const int lane = threadIdx.x & 31;
  const long W = (long)gridDim.x * (blockDim.x / 32);
  const long w = (long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const long lo = w * n / W, hi = (w + 1) * n / W;
  for (long c = lo; c < hi; c += 32 * kRows) {
    float u[kRows], v[kRows];
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
      const long i = c + 32 * j + lane;
      u[j] = i < hi ? __ldcs(a + i) : 0.f;
      v[j] = i < hi ? __ldcs(b + i) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
      const long i = c + 32 * j + lane;
      if (i < hi) {
        __stcs(x + i, u[j] + v[j]);
        __stcs(y + i, u[j] - v[j]);
      }
    }
  }
}

template <typename F>
float time_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 20;
}

int main() {
  const long n = 25549837;
  float *a, *b, *x, *y;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMalloc(&x, n * 4);
  cudaMalloc(&y, n * 4);
  cudaMemset(a, 0, n * 4);
  cudaMemset(b, 0, n * 4);
  const double bytes = 16.0 * n;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {2, 4, 8}) {
    const int g = sms * per_sm;
    float ms = time_ms([&] { sweep<<<g, 256>>>(a, b, x, y, n); });
    printf("{\"kernel\": \"sweep\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", per_sm,
           ms, bytes / ms / 1e6);
  }
  for (int per_sm : {2, 3, 4}) {
    const int g = sms * per_sm;
    float ms1 = time_ms([&] { priv<12><<<g, 256>>>(a, b, x, y, n); });
    printf("{\"kernel\": \"private_rows12\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
           per_sm, ms1, bytes / ms1 / 1e6);
    float ms2 = time_ms([&] { priv<4><<<g, 256>>>(a, b, x, y, n); });
    printf("{\"kernel\": \"private_rows4\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
           per_sm, ms2, bytes / ms2 / 1e6);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
