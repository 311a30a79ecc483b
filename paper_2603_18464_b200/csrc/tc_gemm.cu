// fp32-accurate tensor-core GEMM for the trainer's tall-skinny products (tcgen05, 3xTF32).
//
//   C[M, N] (+)= A[M, K] . B[N, K]^T  (+ bias[N], tanh)       "row transform"
//
// The policy/value heads' dense products (models.py:176-182 forward, :191-204
// backward; value head :283-314) are GEMMs with one huge dimension (frames,
// ~1.6 M at the bench size) and the others <= 256.  The 1e-4 gradient
// tolerance rules out plain TF32 (10-bit mantissa), so each fp32 operand is
// split in shared memory into a TF32 head (low 13 mantissa bits cleared) and
// an fp32 tail, and every k-step issues three tcgen05.mma.kind::tf32:
// A_hi.B_hi + A_hi.B_lo + A_lo.B_hi (the dropped A_lo.B_lo term is ~2^-22
// relative), accumulating in TMEM (fp32).
//
// Structure (one 128-row M tile per CTA, 128 threads):
//   * all threads stage the next K block (32 fp32) of A and B from global
//     memory (coalesced float4 loads; A may be given transposed, i.e. with M
//     contiguous, for the weight-gradient products) and write the hi/lo
//     halves straight into the canonical no-swizzle K-major UMMA layout
//     (8-row x 16-byte core matrices, LBO = 128 B, SBO = BK*32 B);
//   * thread 0 issues the MMAs and commits them to an mbarrier; the next
//     block's loads are issued before waiting on it, so global loads overlap
//     the tensor-core work; two CTAs per SM overlap further;
//   * epilogue: tcgen05.ld 32x32b rows -> bias / tanh -> global stores.
// Split-K (`kslices` > 1) writes per-slice partial tiles that the caller
// reduces in fixed order (deterministic), for the reduction-over-frames
// products dW = dY^T X.
#include "common.cuh"

namespace accel {
namespace {

constexpr int BM = 128;      // rows per CTA (UMMA M)
constexpr int BK = 32;       // fp32 elements per K block (4 UMMA k-steps of 8)
constexpr int kTC = 128;     // threads per CTA

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// kind::tf32, D fp32, A/B tf32 K-major, M = 128, N = n
__device__ __forceinline__ uint32_t make_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// x = hi + lo exactly; hi is x rounded to nearest TF32 (the tensor core reads
// only its top 19 bits), lo the (fp32-exact) remainder
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}

// byte offset of element (r, k) in a canonical K-major no-swizzle tile of BK columns
__device__ __forceinline__ uint32_t canon_off(int r, int k) {
  return (uint32_t)((r >> 3) * (BK * 32) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

struct TcArgs {
  const float* A;  // [M, K] row-major (a_trans == 0) or [K, M] (a_trans == 1)
  const float* B;  // [N, K] row-major (b_trans == 0) or [K, N] (b_trans == 1)
  float* C;        // [M, N] (ldc), or partials [kslices][M][N] when kslices > 1
  const float* bias;
  int64_t M, K;
  int N, Npad;     // Npad: N rounded up to 16 (UMMA N), TMEM columns = pow2 >= Npad
  int64_t lda, ldb, ldc;
  int a_trans, b_trans, act_tanh, accumulate, kslices;
  int tmem_cols;
};

// stage rows [r0, r0 + R) x K block [k0, k0 + BK) of X into hi/lo canonical tiles
__device__ __forceinline__ void stage(const float* __restrict__ X, int64_t ld, int trans,
                                      int64_t rows_total, int64_t k_total, int64_t r0, int R,
                                      int64_t k0, unsigned char* hi, unsigned char* lo) {
  if (!trans) {
    // R rows x 8 float4 per row
    for (int idx = threadIdx.x; idx < R * (BK / 4); idx += kTC) {
      const int r = idx / (BK / 4), c4 = (idx % (BK / 4)) * 4;
      const int64_t gr = r0 + r, gk = k0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < rows_total) {
        const float* src = X + gr * ld + gk;
        if (gk + 3 < k_total && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          v.x = gk < k_total ? __ldg(src) : 0.f;
          v.y = gk + 1 < k_total ? __ldg(src + 1) : 0.f;
          v.z = gk + 2 < k_total ? __ldg(src + 2) : 0.f;
          v.w = gk + 3 < k_total ? __ldg(src + 3) : 0.f;
        }
      }
      float4 h, l;
      split_tf32(v.x, h.x, l.x);
      split_tf32(v.y, h.y, l.y);
      split_tf32(v.z, h.z, l.z);
      split_tf32(v.w, h.w, l.w);
      const uint32_t off = canon_off(r, c4);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) = l;
    }
  } else {
    // X[k][r] with r contiguous: threads walk r (coalesced), scatter 4 k's? no: one element
    for (int idx = threadIdx.x; idx < R * BK; idx += kTC) {
      const int k = idx / R, r = idx % R;
      const int64_t gr = r0 + r, gk = k0 + k;
      const float v = (gr < rows_total && gk < k_total) ? __ldg(X + gk * ld + gr) : 0.f;
      float h, l;
      split_tf32(v, h, l);
      const uint32_t off = canon_off(r, k);
      *reinterpret_cast<float*>(hi + off) = h;
      *reinterpret_cast<float*>(lo + off) = l;
    }
  }
}

__global__ void __launch_bounds__(kTC)
tc_gemm_kernel(TcArgs p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int Npad = p.Npad;
  const uint32_t a_bytes = BM * BK * 4, b_bytes = (uint32_t)Npad * BK * 4;
  unsigned char* a_hi = smem;
  unsigned char* a_lo = a_hi + a_bytes;
  unsigned char* b_hi = a_lo + a_bytes;
  unsigned char* b_lo = b_hi + b_bytes;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int slice = blockIdx.y;
  const int64_t kb_total = ceil_div(p.K, (int64_t)BK);
  const int64_t kb_per = ceil_div(kb_total, (int64_t)p.kslices);
  const int64_t kb_begin = slice * kb_per, kb_end = min(kb_total, kb_begin + kb_per);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc(Npad);
  const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo);
  const uint32_t sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
  const uint32_t SBO = BK * 32, LBO = 128;

  unsigned phase = 0;
  bool any = false;
  for (int64_t kb = kb_begin; kb < kb_end; ++kb) {
    if (any) {  // the previous block's MMAs must finish reading smem
      mbar_wait(&bar, phase);
      phase ^= 1u;
    }
    stage(p.A, p.lda, p.a_trans, p.M, p.K, m0, BM, kb * BK, a_hi, a_lo);
    stage(p.B, p.ldb, p.b_trans, p.N, p.K, 0, Npad, kb * BK, b_hi, b_lo);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int s = 0; s < BK / 8; ++s) {
        const uint32_t koff = s * 2 * 128;
        const uint64_t ah = make_sdesc(sa_hi + koff, LBO, SBO), al = make_sdesc(sa_lo + koff, LBO, SBO);
        const uint64_t bh = make_sdesc(sb_hi + koff, LBO, SBO), bl = make_sdesc(sb_lo + koff, LBO, SBO);
        const uint32_t acc0 = (kb > kb_begin || s > 0) ? 1u : 0u;
        mma_tf32(tmem, ah, bh, idesc, acc0);
        mma_tf32(tmem, ah, bl, idesc, 1u);
        mma_tf32(tmem, al, bh, idesc, 1u);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    any = true;
  }
  if (any) mbar_wait(&bar, phase);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: warp w owns TMEM lanes [32w, 32w + 32) = tile rows
  const int64_t row = m0 + warp * 32 + lane;
  float* out = p.kslices > 1 ? p.C + ((int64_t)slice * p.M + row) * p.N : p.C + row * p.ldc;
  for (int c0 = 0; c0 < Npad; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < p.M && any) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = c0 + j;
        if (c < p.N) {
          float v = __uint_as_float(r[j]);
          if (p.kslices == 1) {
            if (p.bias) v += __ldg(p.bias + c);
            if (p.act_tanh) v = tanhf(v);
            if (p.accumulate) v += out[c];
          }
          out[c] = v;
        }
      }
    } else if (row < p.M && !any) {
      for (int j = 0; j < 16; ++j) {
        const int c = c0 + j;
        if (c < p.N) out[c] = 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(p.tmem_cols)
                 : "memory");
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" size_t accel_tc_gemm_smem(int N) {
  const int Npad = (N + 15) / 16 * 16;
  return (size_t)2 * BM * BK * 4 + (size_t)2 * Npad * BK * 4;
}

// C[M, N] = act(A . B^T + bias) (+ C if accumulate).  a_trans: A stored [K, M];
// b_trans: B stored [K, N].  kslices > 1: C receives [kslices][M][N] partial
// products (no bias / act / accumulate) to be reduced by the caller.
extern "C" int accel_tc_gemm(const float* A, const float* B, float* C, const float* bias,
                             int64_t M, int64_t K, int N, int64_t lda, int64_t ldb, int64_t ldc,
                             int a_trans, int b_trans, int act_tanh, int accumulate, int kslices,
                             void* stream) {
  if (M < 0 || K < 1 || N < 1 || N > 256 || kslices < 1)
    return fail(kDimension, "tc_gemm: bad sizes M=%lld K=%lld N=%d", (long long)M, (long long)K, N);
  if (M == 0) return kOk;
  if (!A || !B || !C) return fail(kDimension, "tc_gemm: NULL buffer");
  TcArgs p;
  p.A = A; p.B = B; p.C = C; p.bias = bias;
  p.M = M; p.K = K; p.N = N;
  p.Npad = (N + 15) / 16 * 16;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc;
  p.a_trans = a_trans; p.b_trans = b_trans; p.act_tanh = act_tanh; p.accumulate = accumulate;
  p.kslices = kslices;
  int cols = 32;
  while (cols < p.Npad) cols <<= 1;
  p.tmem_cols = cols;
  const size_t smem = accel_tc_gemm_smem(N);
  cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return fail(kCuda, "tc_gemm smem: %s", cudaGetErrorString(e));
  dim3 grid((unsigned)ceil_div(M, (int64_t)BM), (unsigned)kslices);
  tc_gemm_kernel<<<grid, kTC, smem, as_stream(stream)>>>(p);
  return post_launch("tc_gemm_kernel");
}
