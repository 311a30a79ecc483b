// Policy backbone/head glue around the library GEMMs (cuBLAS via torch).
//
// Reference: PolicyModel.forward_teacher (models.py:165-184) and
// backward_teacher (models.py:186-209).  The GEMMs x@W0^T, h1@W1^T, c@Wh^T,
// dlogits^T@c, dlogits@Wh, dz2^T@h1, dz2@W1, dz1^T@x stay plain library
// GEMMs; everything between them is here, fused so each activation is read
// once:
//   bias_tanh         h = tanh(z + b)                       (models.py:176-177)
//   build_c           c = h2[frame] + e_prev[prev] + e_pos   (models.py:178-181)
//   dc_reduce         dh2 = sum_k dc; de_pos partials; dz2 = dh2 (1 - h2^2);
//                     db1 partials                          (models.py:196-200)
//   tanh_grad_colsum  dz1 = dh1 (1 - h1^2); db0 partials     (models.py:202-204)
// Column sums are written as per-CTA partials and reduced in fixed order
// (accel_reduce_segments) so results are bitwise deterministic.
#include "common.cuh"

namespace accel {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 16;

__global__ void bias_tanh_kernel(float* __restrict__ z, const float* __restrict__ b,
                                 int64_t total, int cols) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    z[i] = tanhf(z[i] + __ldg(b + i % cols));
}

__global__ void bias_tanh4_kernel(float4* __restrict__ z, const float* __restrict__ b,
                                  int64_t total4, int cols4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += stride) {
    const int c = (int)(i % cols4) * 4;
    float4 v = z[i];
    v.x = tanhf(v.x + __ldg(b + c));
    v.y = tanhf(v.y + __ldg(b + c + 1));
    v.z = tanhf(v.z + __ldg(b + c + 2));
    v.w = tanhf(v.w + __ldg(b + c + 3));
    z[i] = v;
  }
}

// c[i*K + k, :] = h2[frame_of[i], :] + e_prev[prev, :] + e_pos[k, :]
__global__ void build_c4_kernel(const float4* __restrict__ h2, const int32_t* __restrict__ frame_of,
                                const int32_t* __restrict__ tokens,
                                const float4* __restrict__ e_prev, const float4* __restrict__ e_pos,
                                int64_t M, int K, int A, int D4, float4* __restrict__ c) {
  const int64_t total = M * D4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t row = idx / D4;
    const int d = (int)(idx - row * D4);
    const int64_t i = row / K;
    const int k = (int)(row - i * K);
    int prev = k == 0 ? A : __ldg(tokens + row - 1);
    prev = min(max(prev, 0), A);
    const float4 a = __ldg(h2 + (int64_t)__ldg(frame_of + i) * D4 + d);
    const float4 p = __ldg(e_prev + (int64_t)prev * D4 + d);
    const float4 q = __ldg(e_pos + (int64_t)k * D4 + d);
    __stcs(c + idx, make_float4(a.x + p.x + q.x, a.y + p.y + q.y, a.z + p.z + q.z, a.w + p.w + q.w));
  }
}

__global__ void build_c_kernel(const float* __restrict__ h2, const int32_t* __restrict__ frame_of,
                               const int32_t* __restrict__ tokens, const float* __restrict__ e_prev,
                               const float* __restrict__ e_pos, int64_t M, int K, int A, int D,
                               float* __restrict__ c) {
  const int64_t total = M * D;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int64_t row = idx / D;
    const int d = (int)(idx - row * D);
    const int64_t i = row / K;
    const int k = (int)(row - i * K);
    int prev = k == 0 ? A : __ldg(tokens + row - 1);
    prev = min(max(prev, 0), A);
    c[idx] = __ldg(h2 + (int64_t)__ldg(frame_of + i) * D + d) + __ldg(e_prev + (int64_t)prev * D + d) +
             __ldg(e_pos + (int64_t)k * D + d);
  }
}

// Thread layout shared by the column-reduction kernels: the CTA's 256 threads
// are `sub` row-lanes x `span` columns (span = min(D, 256) with 256 % span == 0
// when D <= 256, else span = 256 and the kernel loops over column blocks).
struct ColLayout {
  int span, sub;
  __host__ __device__ static ColLayout make(int D) {
    ColLayout l;
    if (D <= kThreads && kThreads % D == 0) {
      l.span = D;
      l.sub = kThreads / D;
    } else {
      l.span = kThreads;
      l.sub = 1;
    }
    return l;
  }
};

// One CTA per contiguous range of transitions; per-CTA partials:
//   pos_part[blk][k][d] = sum over its transitions of dc[i,k,d]
//   db1_part[blk][d]    = sum of dz2[i,d]
__global__ void __launch_bounds__(kThreads)
dc_reduce_kernel(const float* __restrict__ dc, const float* __restrict__ h2,
                 const int32_t* __restrict__ frame_of, int64_t N, int K, int D,
                 float* __restrict__ dz2, float* __restrict__ pos_part,
                 float* __restrict__ db1_part) {
  extern __shared__ float s_acc[];  // [sub][K+1][span]
  const ColLayout L = ColLayout::make(D);
  const int lane_row = threadIdx.x / L.span, lane_col = threadIdx.x % L.span;
  const int64_t per = ceil_div(N, (int64_t)gridDim.x);
  const int64_t i_begin = (int64_t)blockIdx.x * per, i_end = min(N, i_begin + per);
  for (int d0 = 0; d0 < D; d0 += L.span) {
    const int d = d0 + lane_col;
    float pos[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) pos[k] = 0.f;
    float db1 = 0.f;
    if (d < D) {
      for (int64_t i = i_begin + lane_row; i < i_end; i += L.sub) {
        const float* row = dc + i * K * D + d;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < kMaxK; ++k)
          if (k < K) {
            const float v = __ldcs(row + (int64_t)k * D);
            acc += v;
            pos[k] += v;
          }
        const int64_t f = __ldg(frame_of + i);
        const float h = __ldg(h2 + f * D + d);
        const float g = acc * (1.f - h * h);
        dz2[f * D + d] = g;
        db1 += g;
      }
    }
    float* mine = s_acc + (size_t)lane_row * (K + 1) * L.span;
#pragma unroll
    for (int k = 0; k < kMaxK; ++k)
      if (k < K) mine[k * L.span + lane_col] = pos[k];
    mine[K * L.span + lane_col] = db1;
    __syncthreads();
    for (int e = threadIdx.x; e < (K + 1) * L.span; e += kThreads) {
      const int k = e / L.span, c = e % L.span;
      if (d0 + c < D) {
        float acc = 0.f;
        for (int s = 0; s < L.sub; ++s) acc += s_acc[(size_t)s * (K + 1) * L.span + e];
        if (k < K) pos_part[((int64_t)blockIdx.x * K + k) * D + d0 + c] = acc;
        else db1_part[(int64_t)blockIdx.x * D + d0 + c] = acc;
      }
    }
    __syncthreads();
  }
}

// g <- g * (1 - h^2) in place over [R, C]; per-CTA column sums of the result.
__global__ void __launch_bounds__(kThreads)
tanh_grad_colsum_kernel(float* __restrict__ g, int64_t ldg, const float* __restrict__ h,
                        int64_t ldh, int64_t R, int C, float* __restrict__ col_part) {
  extern __shared__ float s_acc[];  // [sub][span]
  const ColLayout L = ColLayout::make(C);
  const int lane_row = threadIdx.x / L.span, lane_col = threadIdx.x % L.span;
  const int64_t per = ceil_div(R, (int64_t)gridDim.x);
  const int64_t r_begin = (int64_t)blockIdx.x * per, r_end = min(R, r_begin + per);
  for (int c0 = 0; c0 < C; c0 += L.span) {
    const int c = c0 + lane_col;
    float acc = 0.f;
    if (c < C) {
      for (int64_t r = r_begin + lane_row; r < r_end; r += L.sub) {
        const float hv = __ldg(h + r * ldh + c);
        const float v = g[r * ldg + c] * (1.f - hv * hv);
        g[r * ldg + c] = v;
        acc += v;
      }
    }
    s_acc[lane_row * L.span + lane_col] = acc;
    __syncthreads();
    for (int e = threadIdx.x; e < L.span; e += kThreads) {
      if (c0 + e < C) {
        float a = 0.f;
        for (int s = 0; s < L.sub; ++s) a += s_acc[s * L.span + e];
        col_part[(int64_t)blockIdx.x * C + c0 + e] = a;
      }
    }
    __syncthreads();
  }
}

// float4 variant (C % 4 == 0, 256 % (C/4) == 0): same fixed summation order
// per (row-lane, column), four rows in flight per thread.
__global__ void __launch_bounds__(kThreads)
tanh_grad_colsum4_kernel(float4* __restrict__ g, int64_t ldg4, const float4* __restrict__ h,
                         int64_t ldh4, int64_t R, int C4, float* __restrict__ col_part) {
  extern __shared__ float4 s_acc4[];  // [sub][C4]
  const int sub = kThreads / C4;
  const int lr = threadIdx.x / C4, lc = threadIdx.x % C4;
  const int64_t per = ceil_div(R, (int64_t)gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(R, r0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int64_t r = r0 + lr;
  for (; r + 3 * sub < r1; r += 4 * sub) {
    float4 gv[4], hv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      gv[u] = g[(r + u * sub) * ldg4 + lc];
      hv[u] = __ldg(h + (r + u * sub) * ldh4 + lc);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float4 v;
      v.x = gv[u].x * (1.f - hv[u].x * hv[u].x);
      v.y = gv[u].y * (1.f - hv[u].y * hv[u].y);
      v.z = gv[u].z * (1.f - hv[u].z * hv[u].z);
      v.w = gv[u].w * (1.f - hv[u].w * hv[u].w);
      g[(r + u * sub) * ldg4 + lc] = v;
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  for (; r < r1; r += sub) {
    const float4 gv = g[r * ldg4 + lc], hv = __ldg(h + r * ldh4 + lc);
    float4 v;
    v.x = gv.x * (1.f - hv.x * hv.x);
    v.y = gv.y * (1.f - hv.y * hv.y);
    v.z = gv.z * (1.f - hv.z * hv.z);
    v.w = gv.w * (1.f - hv.w * hv.w);
    g[r * ldg4 + lc] = v;
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  s_acc4[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < C4) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < sub; ++s) {
      const float4 y = s_acc4[s * C4 + threadIdx.x];
      a.x += y.x; a.y += y.y; a.z += y.z; a.w += y.w;
    }
    reinterpret_cast<float4*>(col_part + (int64_t)blockIdx.x * C4 * 4)[threadIdx.x] = a;
  }
}

int row_grid(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)kNumSMs * 4));
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_bias_tanh(float* z, const float* b, int64_t rows, int cols, void* stream) {
  if (rows < 0 || cols < 1) return fail(kDimension, "bias_tanh: bad sizes");
  if (rows == 0) return kOk;
  if (!z || !b) return fail(kDimension, "bias_tanh: NULL buffer");
  cudaStream_t s = as_stream(stream);
  const int64_t total = rows * cols;
  if (cols % 4 == 0 && (reinterpret_cast<uintptr_t>(z) & 15) == 0) {
    const int64_t t4 = total / 4;
    const int grid = (int)std::min<int64_t>(ceil_div(t4, kThreads), (int64_t)kNumSMs * 8);
    bias_tanh4_kernel<<<grid, kThreads, 0, s>>>(reinterpret_cast<float4*>(z), b, t4, cols / 4);
  } else {
    const int grid = (int)std::min<int64_t>(ceil_div(total, kThreads), (int64_t)kNumSMs * 8);
    bias_tanh_kernel<<<grid, kThreads, 0, s>>>(z, b, total, cols);
  }
  return post_launch("bias_tanh_kernel");
}

extern "C" int accel_build_c(const float* h2, const int32_t* frame_of, const int32_t* tokens,
                             const float* e_prev, const float* e_pos, int64_t N, int K, int A,
                             int D, float* c_out, void* stream) {
  if (N < 0 || K < 1 || A < 1 || D < 1) return fail(kDimension, "build_c: bad sizes");
  if (N == 0) return kOk;
  if (!h2 || !frame_of || !tokens || !e_prev || !e_pos || !c_out)
    return fail(kDimension, "build_c: NULL buffer");
  cudaStream_t s = as_stream(stream);
  const int64_t M = N * K;
  const uintptr_t al = reinterpret_cast<uintptr_t>(h2) | reinterpret_cast<uintptr_t>(e_prev) |
                       reinterpret_cast<uintptr_t>(e_pos) | reinterpret_cast<uintptr_t>(c_out);
  if (D % 4 == 0 && (al & 15) == 0) {
    const int64_t total = M * (D / 4);
    const int grid = (int)std::min<int64_t>(ceil_div(total, kThreads), (int64_t)kNumSMs * 16);
    build_c4_kernel<<<grid, kThreads, 0, s>>>(
        reinterpret_cast<const float4*>(h2), frame_of, tokens,
        reinterpret_cast<const float4*>(e_prev), reinterpret_cast<const float4*>(e_pos), M, K, A,
        D / 4, reinterpret_cast<float4*>(c_out));
  } else {
    const int grid = (int)std::min<int64_t>(ceil_div(M * D, kThreads), (int64_t)kNumSMs * 16);
    build_c_kernel<<<grid, kThreads, 0, s>>>(h2, frame_of, tokens, e_prev, e_pos, M, K, A, D,
                                             c_out);
  }
  return post_launch("build_c_kernel");
}

extern "C" int accel_rows_grid(int64_t rows) { return row_grid(rows); }

extern "C" int accel_dc_reduce(const float* dc, const float* h2, const int32_t* frame_of,
                               int64_t N, int K, int D, float* dz2, float* pos_part,
                               float* db1_part, int grid, void* stream) {
  if (N < 0 || K < 1 || K > kMaxK || D < 1)
    return fail(kDimension, "dc_reduce: bad sizes (chunk_len must be <= %d)", kMaxK);
  if (N == 0) return kOk;
  if (!dc || !h2 || !frame_of || !dz2 || !pos_part || !db1_part)
    return fail(kDimension, "dc_reduce: NULL buffer");
  if (grid < 1) return fail(kDimension, "dc_reduce: grid < 1");
  const ColLayout L = ColLayout::make(D);
  const size_t smem = sizeof(float) * (size_t)L.sub * (K + 1) * L.span;
  dc_reduce_kernel<<<grid, kThreads, smem, as_stream(stream)>>>(dc, h2, frame_of, N, K, D, dz2,
                                                                pos_part, db1_part);
  return post_launch("dc_reduce_kernel");
}

extern "C" int accel_tanh_grad_colsum(float* g, int64_t ldg, const float* h, int64_t ldh,
                                      int64_t R, int C, float* col_part, int grid, void* stream) {
  if (R < 0 || C < 1 || ldg < C || ldh < C) return fail(kDimension, "tanh_grad_colsum: bad sizes");
  if (R == 0) return kOk;
  if (!g || !h || !col_part) return fail(kDimension, "tanh_grad_colsum: NULL buffer");
  if (grid < 1) return fail(kDimension, "tanh_grad_colsum: grid < 1");
  const uintptr_t al = reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(h) |
                       reinterpret_cast<uintptr_t>(col_part);
  if (C % 4 == 0 && C / 4 <= kThreads && kThreads % (C / 4) == 0 && (al & 15) == 0 &&
      ldg % 4 == 0 && ldh % 4 == 0) {
    tanh_grad_colsum4_kernel<<<grid, kThreads, kThreads * sizeof(float4), as_stream(stream)>>>(
        reinterpret_cast<float4*>(g), ldg / 4, reinterpret_cast<const float4*>(h), ldh / 4, R,
        C / 4, col_part);
    return post_launch("tanh_grad_colsum4_kernel");
  }
  const ColLayout L = ColLayout::make(C);
  const size_t smem = sizeof(float) * (size_t)L.sub * L.span;
  tanh_grad_colsum_kernel<<<grid, kThreads, smem, as_stream(stream)>>>(g, ldg, h, ldh, R, C,
                                                                      col_part);
  return post_launch("tanh_grad_colsum_kernel");
}

// ---- small products -------------------------------------------------------------
// C[M, N] = sum_k A(m, k) B(n, k) for the handful of tiny products around the
// factorized head (e_prev / e_pos times W_head and their gradients: <= 264
// rows, models.py:181-182, :191-197): 32 x 32 output tiles through shared
// memory, fp32 FMA in a fixed k order (exact like a SIMT library GEMM, and
// one short launch instead of a persistent tensor-core kernel's prologue).
namespace accel {
namespace {

constexpr int kSgT = 32;

__global__ void __launch_bounds__(256)
small_gemm_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
                  int M, int N, int K, int64_t lda, int64_t ldb, int64_t ldc, int a_trans,
                  int b_trans, int kper) {
  __shared__ float sa[kSgT][kSgT + 1], sb[kSgT][kSgT + 1];  // [k][m], [k][n]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int m0 = blockIdx.y * kSgT, n0 = blockIdx.x * kSgT;
  // split-K: slice blockIdx.z covers k in [z kper, (z + 1) kper) and writes its
  // own [M, N] partial (C + z M ldc); the caller sums the slices in order
  const int kb = blockIdx.z * kper, ke = min(K, kb + kper);
  C += (int64_t)blockIdx.z * M * ldc;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};  // rows ty, ty + 8, ty + 16, ty + 24; column tx
  for (int k0 = kb; k0 < ke; k0 += kSgT) {
    for (int i = threadIdx.x; i < kSgT * kSgT; i += 256) {
      const int r = i >> 5, c = i & 31;  // loads walk the contiguous dimension
      // A tile: element (m0 + mm, k0 + kk)
      {
        const int mm = a_trans ? c : r, kk = a_trans ? r : c;
        const int m = m0 + mm, k = k0 + kk;
        sa[kk][mm] = (m < M && k < ke) ? (a_trans ? A[(int64_t)k * lda + m] : A[(int64_t)m * lda + k])
                                      : 0.f;
      }
      {
        const int nn = b_trans ? c : r, kk = b_trans ? r : c;
        const int n = n0 + nn, k = k0 + kk;
        sb[kk][nn] = (n < N && k < ke) ? (b_trans ? B[(int64_t)k * ldb + n] : B[(int64_t)n * ldb + k])
                                      : 0.f;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kSgT; ++kk) {
      const float b = sb[kk][tx];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fmaf(sa[kk][ty + 8 * r], b, acc[r]);
    }
    __syncthreads();
  }
  const int n = n0 + tx;
  if (n < N)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int m = m0 + ty + 8 * r;
      if (m < M) C[(int64_t)m * ldc + n] = acc[r];
    }
}

// C[m, n] = sum_z part[z][m][n] (slices in order: deterministic)
__global__ void small_gemm_sum_kernel(const float* __restrict__ part, int ks, int M, int N,
                                      float* __restrict__ C, int64_t ldc) {
  const int64_t total = (int64_t)M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int z = 0; z < ks; ++z) a += part[z * total + e];
    C[(e / N) * ldc + e % N] = a;
  }
}

// k slices of a small product: when its output tiles leave SMs idle and the
// reduction is long, split k (>= 128 per slice) until ~2 waves of blocks
int small_gemm_slices(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(M, (int64_t)kSgT) * ceil_div(N, (int64_t)kSgT);
  if (tiles >= kNumSMs || K < 256) return 1;
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(K, (int64_t)128),
                                                     2 * kNumSMs / tiles));
}

}  // namespace
}  // namespace accel

// C[M, N] = op(A) op(B)^T: A(m, k) = a_trans ? A[k][m] : A[m][k], B(n, k) =
// b_trans ? B[k][n] : B[n][k]; fp32, fixed order, for small products.
extern "C" int64_t accel_small_gemm_ws_floats(int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  const int ks = accel::small_gemm_slices(M, N, K);
  return ks > 1 ? (int64_t)ks * M * N : 0;
}

extern "C" int accel_small_gemm(const float* A, const float* B, float* C, int64_t M, int64_t N,
                                int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int a_trans,
                                int b_trans, float* ws, int64_t ws_floats, void* stream) {
  if (M < 0 || N < 0 || K < 0 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return accel::fail(accel::kDimension, "small_gemm: bad sizes");
  if (M == 0 || N == 0) return accel::kOk;
  if (!A || !B || !C) return accel::fail(accel::kDimension, "small_gemm: NULL buffer");
  cudaStream_t s = accel::as_stream(stream);
  int ks = accel::small_gemm_slices(M, N, K);
  if (ks > 1 && (!ws || ws_floats < (int64_t)ks * M * N)) ks = 1;  // no workspace: one slice
  const int kper = (int)(accel::ceil_div(accel::ceil_div(K, (int64_t)ks), (int64_t)accel::kSgT) *
                         accel::kSgT);
  ks = (int)accel::ceil_div(K, (int64_t)kper);
  dim3 grid((unsigned)accel::ceil_div(N, accel::kSgT), (unsigned)accel::ceil_div(M, accel::kSgT),
            (unsigned)ks);
  if (ks == 1) {
    accel::small_gemm_kernel<<<grid, 256, 0, s>>>(A, B, C, (int)M, (int)N, (int)K, lda, ldb, ldc,
                                                  a_trans, b_trans, (int)K);
    return accel::post_launch("small_gemm_kernel");
  }
  accel::small_gemm_kernel<<<grid, 256, 0, s>>>(A, B, ws, (int)M, (int)N, (int)K, lda, ldb, N,
                                                a_trans, b_trans, kper);
  int rc = accel::post_launch("small_gemm_kernel");
  if (rc != accel::kOk) return rc;
  const int g2 = (int)std::min<int64_t>(accel::ceil_div(M * N, (int64_t)256), 1184);
  accel::small_gemm_sum_kernel<<<g2, 256, 0, s>>>(ws, ks, (int)M, (int)N, C, ldc);
  return accel::post_launch("small_gemm_sum_kernel");
}
