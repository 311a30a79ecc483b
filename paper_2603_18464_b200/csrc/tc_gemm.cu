// fp32-accurate tensor-core GEMMs for the trainer's tall-skinny products (tcgen05, 3xTF32).
//
// The policy/value heads' dense products (models.py:176-182 forward, :191-204
// backward; value head :283-314) have one huge dimension (frame rows, ~1.6 M
// at the bench size) and the others <= 256, so they are HBM-bound: the job is
// to stream the big operand once at full bandwidth while the tensor cores do
// the (small) math.  The 1e-4 gradient tolerance rules out plain TF32, so each
// fp32 operand x is used as x_hi + x_lo and every k-step accumulates
// x_hi.y_hi + x_hi.y_lo + x_lo.y_hi in TMEM (the dropped lo.lo term is
// ~2^-21 relative).  The tensor core reads only the top 19 bits of an fp32
// word, so the raw fp32 tile that TMA lands in shared memory IS the hi
// operand (truncated); converter warps only compute lo = x - trunc19(x).
//
// Two persistent, warp-specialised kernels (one CTA per SM, 320 threads):
//
//   tc_rows    Y[M, N] = act(X[M, K] . W^T + bias) (+ Y)       "row transform"
//              W ([N, K] or [K, N]) is split (round-to-nearest hi, lo) once per
//              CTA and stays resident in shared memory as [W_hi; W_lo] (2N
//              rows, K-major, no swizzle), so one MMA with N' = 2N computes
//              X_hi.W_hi and X_hi.W_lo side by side in TMEM and a second one
//              adds X_lo.W_hi; the epilogue sums the two halves.  X streams
//              through TMA (128 rows x 32 fp32, SWIZZLE_128B, K-major).
//   tc_wgrad   C[Mc, Nc] = sum_f P[f, :Mc]^T Q[f, :Nc]          "weight gradient"
//              the reduction runs over the frame rows; both operands stream
//              through TMA as MN-major SWIZZLE_128B_ATOM_32B slabs (32 columns
//              x SR rows), again with [Q_hi | Q_lo] concatenated along N.  Each
//              CTA accumulates its share of row blocks in TMEM and flushes to a
//              per-CTA fp32 partial every 512 rows (bounds the fp32
//              accumulation error); the caller reduces the partials in fixed
//              order: deterministic.
//
// Roles: warp 0 lane 0 issues TMA loads into a stage ring; warps 2-5 compute
// the lo halves; warp 1 lane 0 issues the MMAs and commits them to mbarriers;
// warps 6-9 drain the double-buffered TMEM accumulators (tcgen05.ld) while the
// next tile is being multiplied.  TMA bulk loads do not allocate in L1, so the
// bytes in flight are bounded by the stage ring, not by the ~23 KB of L1 left
// beside 229 KB of shared memory (the limit a register-staged loader hits).
#include <cuda.h>

#include <algorithm>

#include "tc_common.cuh"

namespace accel {
namespace {

using namespace tc;

constexpr int BM = 128;                    // UMMA M: rows per tile / accumulator
constexpr int BK = 32;                     // row kernel: fp32 K elements per stage
constexpr int kThreads = 320;              // 10 warps
constexpr int kConvWarp0 = 2, kConvWarps = 4, kConv = kConvWarps * 32;
constexpr int kEpiWarp0 = 6, kEpiWarps = 4;
// tc_rows may run 8 epilogue warps (two per TMEM lane quarter, each draining
// half of the column chunks) when its ring keeps enough stages: its epilogue
// (bias, tanh, swizzled staging, TMA stores) is the longer pole at narrow K
constexpr int kRowsEpiMax = 8;
constexpr int kRowsThreads = (kEpiWarp0 + kRowsEpiMax) * 32;  // 14 warps
constexpr int kMaxRaw = 12;                // raw (TMA) ring slots
constexpr int kNL = 2;                     // lo ring slots
#ifndef ACCEL_ROWS_HDIRECT_WBYTES
#define ACCEL_ROWS_HDIRECT_WBYTES (96 * 1024)  // dtanh: H from global memory from this weight size
#endif
constexpr size_t kSmemBudget = 225 * 1024;  // dynamic shared memory (wgrad)
constexpr size_t kRowsBudget = 224 * 1024;  // tc_rows also holds ~2 KB of static smem (<= 227 KB)
constexpr uint32_t kTile = BM * BK * 4;    // one 128 x 32 fp32 tile (16 KB)
constexpr int kFlushRows = 512;            // wgrad: TMEM flush period (rows)

// lo = x - trunc19(x): the part of x the tensor core drops when it reads x as TF32
__device__ __forceinline__ float4 tf32_lo(float4 v) {
  float4 l;
  l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
  l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
  l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
  l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
  return l;
}

// x = hi + lo exactly, hi = x rounded to nearest TF32 (resident weights)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}

// tanh via one ex2 and one fast divide: |error| ~1e-7 (the products' own error is ~1e-6)
__device__ __forceinline__ float fast_tanh(float x) {
  const float t = __expf(2.f * x);
  return 1.f - __fdividef(2.f, t + 1.f);
}

// byte offset of element (r, k) in a K-major no-swizzle tile of BK columns
__device__ __forceinline__ uint32_t canon_k(int r, int k) {
  return (uint32_t)((r >> 3) * (BK * 32) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// converters: lo[i] = tf32_lo(raw[i]) over `bytes` (multiple of 16) of a stage
__device__ __forceinline__ void convert_lo(const unsigned char* raw, unsigned char* lo,
                                           uint32_t bytes, int t) {
  constexpr uint32_t kStep = kConv * 16;
  uint32_t i = (uint32_t)t * 16;
  for (; i + 3 * kStep < bytes; i += 4 * kStep) {  // four shared loads in flight
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(raw + i + u * kStep);
#pragma unroll
    for (int u = 0; u < 4; ++u) *reinterpret_cast<float4*>(lo + i + u * kStep) = tf32_lo(v[u]);
  }
  for (; i < bytes; i += kStep)
    *reinterpret_cast<float4*>(lo + i) = tf32_lo(*reinterpret_cast<const float4*>(raw + i));
}

__device__ __forceinline__ unsigned nonfinite4(float4 v) {
  auto bad = [](float x) { return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u ? 1u : 0u; };
  return bad(v.x) + bad(v.y) + bad(v.z) + bad(v.w);
}

// the same, also counting non-finite inputs (the streamed operand is read anyway)
__device__ __forceinline__ unsigned convert_lo_count(const unsigned char* raw, unsigned char* lo,
                                                     uint32_t bytes, int t) {
  constexpr uint32_t kStep = kConv * 16;
  unsigned n = 0;
  uint32_t i = (uint32_t)t * 16;
  for (; i + 3 * kStep < bytes; i += 4 * kStep) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(raw + i + u * kStep);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      n += nonfinite4(v[u]);
      *reinterpret_cast<float4*>(lo + i + u * kStep) = tf32_lo(v[u]);
    }
  }
  for (; i < bytes; i += kStep) {
    const float4 v = *reinterpret_cast<const float4*>(raw + i);
    n += nonfinite4(v);
    *reinterpret_cast<float4*>(lo + i) = tf32_lo(v);
  }
  return n;
}

// Pipeline state of one ring: slot index and mbarrier phase of the current stage.
struct Ring {
  int slot = 0, n;
  unsigned ph = 0;
  __device__ explicit Ring(int n_) : n(n_) {}
  __device__ void next() {
    if (++slot == n) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

// Barriers: raw ring (TMA -> converters, MMA), lo ring (converters -> MMA),
// double-buffered TMEM accumulators (MMA -> epilogue).
struct Bars {
  uint64_t raw_full[kMaxRaw], raw_empty[kMaxRaw], lo_full[kNL], lo_empty[kNL], tfull[2], tempty[2];
  uint64_t hbar[kRowsEpiMax][2];  // dtanh epilogue: per-warp H box loads
};

__device__ __forceinline__ void init_bars(Bars& b, int nraw, int nepi = kEpiWarps) {
  for (int s = 0; s < nraw; ++s) {
    mbar_init(&b.raw_full[s], 1);
    mbar_init(&b.raw_empty[s], 1);
  }
  for (int s = 0; s < kNL; ++s) {
    mbar_init(&b.lo_full[s], kConv);
    mbar_init(&b.lo_empty[s], 1);
  }
  for (int s = 0; s < 2; ++s) {
    mbar_init(&b.tfull[s], 1);
    mbar_init(&b.tempty[s], nepi);
  }
  for (int w = 0; w < nepi; ++w) {
    mbar_init(&b.hbar[w][0], 1);
    mbar_init(&b.hbar[w][1], 1);
  }
  fence_mbar_init();
}

// ============================================================================
// row transform

struct RowArgs {
  const float* W;
  float* Y;
  const float* bias;
  int64_t M, ntiles, ldw, ldy;
  int K, N, Npad, kblocks, last_ksteps, concat;
  int w_trans, act_tanh, accumulate, y_vec, nraw, tma_store, nstg, has_bias;
  int dtanh;          // Y = (X.W^T) * (1 - H^2), per-CTA column sums of Y into col_part
  float* col_part;    // [gridDim.x][N]
  unsigned* nonfinite;  // optional: += number of non-finite elements of X
  uint32_t tmem_cols, acc_cols;
  int nepi;           // epilogue warps: 4 (warps 6-9) or 8 (6-13)
  // dtanh with H read straight from global memory by the epilogue lanes (no H
  // boxes in shared memory: a large resident weight keeps its ring), column sums
  // in lane registers (<= 2 chunks per warp); hdirect needs N % 32 == 0
  int hdirect;
  const float* Hp;
  int64_t ldh;
};

__global__ void __launch_bounds__(kRowsThreads, 1)
tc_rows_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap ymap,
               const __grid_constant__ CUtensorMap hmap, RowArgs p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ Bars bars;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float s_bias[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Npad = p.Npad;
  if (smem_u32(smem) & 1023) __trap();  // SWIZZLE_128B atoms need 1 KB alignment
  const uint32_t wblk = (uint32_t)Npad * BK * 4 * 2;  // one K block of [W_hi; W_lo]
  unsigned char* wres = smem;
  unsigned char* raw_ring = smem + (size_t)p.kblocks * wblk;
  unsigned char* lo_ring = raw_ring + (size_t)p.nraw * kTile;
  unsigned char* staging = lo_ring + (size_t)kNL * kTile;  // epilogue: nstg boxes per warp
  const int nepi = p.nepi;
  // dtanh only: per-epilogue-warp column sums [nepi][256] after the staging boxes
  float (*s_csum)[256] = reinterpret_cast<float (*)[256]>(staging + (size_t)nepi * p.nstg * 4096);

  // W resident: split once, K-major, [hi rows | lo rows] per K block
  const int Kpad = p.kblocks * BK;
  for (int idx = threadIdx.x; idx < Npad * Kpad; idx += kRowsThreads) {
    const int n = idx / Kpad, k = idx - n * Kpad;
    float v = 0.f;
    if (n < p.N && k < p.K)
      v = p.w_trans ? __ldg(p.W + (int64_t)k * p.ldw + n) : __ldg(p.W + (int64_t)n * p.ldw + k);
    float h, l;
    split_tf32(v, h, l);
    unsigned char* blk = wres + (size_t)(k / BK) * wblk;
    *reinterpret_cast<float*>(blk + canon_k(n, k % BK)) = h;
    *reinterpret_cast<float*>(blk + canon_k(Npad + n, k % BK)) = l;
  }
  for (int c = threadIdx.x; c < 256; c += kRowsThreads)
    s_bias[c] = (p.bias && c < p.N) ? __ldg(p.bias + c) : 0.f;
  if (warp == 1) tmem_alloc(&tmem_base, p.tmem_cols);
  if (threadIdx.x == 0) {
    init_bars(bars, p.nraw, nepi);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int64_t my_tiles =
      p.ntiles > (int64_t)blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * p.kblocks;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      Ring r(p.nraw);
      int64_t tile = blockIdx.x;
      int kb = 0;
      for (int64_t s = 0; s < total; ++s, r.next()) {
        mbar_wait(&bars.raw_empty[r.slot], r.ph ^ 1u);
        mbar_expect_tx(&bars.raw_full[r.slot], kTile);
        tma_load_2d(raw_ring + (size_t)r.slot * kTile, &xmap, kb * BK, (int)(tile * BM),
                    &bars.raw_full[r.slot]);
        if (++kb == p.kblocks) {
          kb = 0;
          tile += gridDim.x;
        }
      }
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer (warp-wide loop, one elected lane issues)
      const int n1 = p.concat ? 2 * Npad : Npad;
      const uint32_t id1 = make_idesc(n1, 0, 0), id2 = make_idesc(Npad, 0, 0);
      Ring r(p.nraw), l(kNL);
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int b = (int)(t & 1);
        mbar_wait(&bars.tempty[b], ((unsigned)(t >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)b * p.acc_cols;
        for (int kb = 0; kb < p.kblocks; ++kb, r.next(), l.next()) {
          mbar_wait(&bars.raw_full[r.slot], r.ph);
          mbar_wait(&bars.lo_full[l.slot], l.ph);
          tc_fence_after();
          const uint32_t a_raw = smem_u32(raw_ring + (size_t)r.slot * kTile);
          const uint32_t a_lo = smem_u32(lo_ring + (size_t)l.slot * kTile);
          const uint32_t wb = smem_u32(wres + (size_t)kb * wblk);
          const int nsteps = kb == p.kblocks - 1 ? p.last_ksteps : BK / 8;
          for (int s = 0; s < nsteps; ++s) {
            const uint64_t ar = make_sdesc(a_raw + s * 32, 16, 1024, 2);
            const uint64_t al = make_sdesc(a_lo + s * 32, 16, 1024, 2);
            const uint64_t wh = make_sdesc(wb + s * 256, 128, 1024, 0);
            const uint32_t acc = (kb > 0 || s > 0) ? 1u : 0u;
            if (p.concat) {
              mma_tf32_w(d, ar, wh, id1, acc);  // [X.W_hi | X.W_lo]
            } else {
              const uint64_t wl = make_sdesc(wb + (uint32_t)Npad * 128 + s * 256, 128, 1024, 0);
              mma_tf32_w(d, ar, wh, id2, acc);
              mma_tf32_w(d, ar, wl, id2, 1u);
            }
            mma_tf32_w(d, al, wh, id2, 1u);  // + X_lo.W_hi
          }
          mma_commit_w(&bars.raw_empty[r.slot]);
          mma_commit_w(&bars.lo_empty[l.slot]);
        }
        mma_commit_w(&bars.tfull[b]);
      }
    }
  } else if (warp < kEpiWarp0) {
    // ---- converters
    const int t = threadIdx.x - kConvWarp0 * 32;
    Ring r(p.nraw), l(kNL);
    unsigned nbad = 0;
    for (int64_t s = 0; s < total; ++s, r.next(), l.next()) {
      mbar_wait(&bars.raw_full[r.slot], r.ph);
      mbar_wait(&bars.lo_empty[l.slot], l.ph ^ 1u);
      if (p.nonfinite)  // (TMA zero-fills rows and columns past the matrix)
        nbad += convert_lo_count(raw_ring + (size_t)r.slot * kTile, lo_ring + (size_t)l.slot * kTile,
                                 kTile, t);
      else
        convert_lo(raw_ring + (size_t)r.slot * kTile, lo_ring + (size_t)l.slot * kTile, kTile, t);
      fence_proxy_async();
      mbar_arrive(&bars.lo_full[l.slot]);
    }
    if (p.nonfinite) {
      nbad = __reduce_add_sync(0xffffffffu, nbad);
      if (lane == 0 && nbad) atomicAdd(p.nonfinite, nbad);  // integer: order-independent
    }
  } else if (warp - kEpiWarp0 < nepi) {
    // ---- epilogue: warp q drains TMEM lanes [32q, 32q + 32) = tile rows, 32
    // columns at a time (with 8 epilogue warps, warps 6-9 take the even and
    // warps 10-13 the odd 32-column chunks); rows go out through a swizzled
    // staging box + TMA store.
    // dtanh: the box is first filled with the matching H box by TMA, read back
    // (same swizzle), overwritten with y = acc (1 - h^2), stored; column sums of
    // y are read column-wise from the box (conflict-free) into lane registers.
    const int q = warp & 3, ew = warp - kEpiWarp0;
    const int cfirst = nepi == 8 ? (ew >> 2) * 32 : 0, cstep = nepi == 8 ? 64 : 32;
    const int nch = Npad > cfirst ? (Npad - cfirst + cstep - 1) / cstep : 0;  // this warp's chunks
    unsigned char* stg0 = staging + (size_t)ew * p.nstg * 4096;
    int sb = 0;
    unsigned hph = 0;  // per-box H barrier phases
    if (p.dtanh && !p.hdirect)
      for (int c = lane; c < 256; c += 32) s_csum[ew][c] = 0.f;  // dtanh column sums
    // dtanh with all of a tile's chunks fitting the boxes: H boxes of the next
    // tile are loaded as soon as this tile's stores have read the boxes, so the
    // load latency hides behind the MMAs instead of stalling every chunk
    const bool hdir = p.dtanh && p.hdirect;
    const bool hpre = p.dtanh && !hdir && nch == p.nstg;
    float cs_acc[2] = {0.f, 0.f};  // hdirect: this lane's column sums of chunks 0 and 1
    auto load_h = [&](int64_t tt) {
      const int64_t r0h = (blockIdx.x + tt * gridDim.x) * BM + q * 32;
      for (int c = 0; c < nch; ++c) {
        mbar_expect_tx(&bars.hbar[ew][c], 4096);
        tma_load_2d(stg0 + c * 4096, &hmap, cfirst + c * cstep, (int)r0h, &bars.hbar[ew][c]);
      }
    };
    if (hpre && my_tiles > 0 && lane == 0) load_h(0);
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int b = (int)(t & 1);
      mbar_wait(&bars.tfull[b], (unsigned)(t >> 1) & 1u);
      tc_fence_after();
      const int64_t row0 = (blockIdx.x + t * gridDim.x) * BM + q * 32;
      const int64_t row = row0 + lane;
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)b * p.acc_cols;
#pragma unroll 1
      for (int c0 = cfirst; c0 < Npad; c0 += cstep) {
        unsigned char* stg = stg0 + sb * 4096;
        if (p.tma_store) {
          if (lane == 0 && !hpre) tma_store_wait_read();  // this box's previous store has read it
          __syncwarp();
          if (p.dtanh && !hdir && !hpre && lane == 0) {
            mbar_expect_tx(&bars.hbar[ew][sb], 4096);
            tma_load_2d(stg, &hmap, c0, (int)row0, &bars.hbar[ew][sb]);
          }
        }
        float4 hv[8];  // hdirect: this lane's row of H, columns c0 .. c0 + 31 (loads in flight
                       // while the accumulator is read)
        if (hdir) {
          if (row < p.M) {
            const float4* hp = reinterpret_cast<const float4*>(p.Hp + row * p.ldh + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j) hv[j] = __ldg(hp + j);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) hv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        uint32_t r[32];
        float v[32];
        tmem_ld32(tb + c0, r);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (p.concat) {
          tmem_ld32(tb + Npad + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(r[j]);
        }
        if (p.has_bias) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(&s_bias[c0 + j]);
            v[j] += bb.x;
            v[j + 1] += bb.y;
            v[j + 2] += bb.z;
            v[j + 3] += bb.w;
          }
        }
        if (p.act_tanh) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fast_tanh(v[j]);
        }
        if (p.tma_store) {
          if (p.dtanh) {
            if (!hdir) {
              mbar_wait(&bars.hbar[ew][sb], (hph >> sb) & 1u);
              hph ^= 1u << sb;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 h =
                  hdir ? hv[j]
                       : *reinterpret_cast<const float4*>(stg + lane * 128 + ((j ^ (lane & 7)) * 16));
              v[4 * j] *= 1.f - h.x * h.x;
              v[4 * j + 1] *= 1.f - h.y * h.y;
              v[4 * j + 2] *= 1.f - h.z * h.z;
              v[4 * j + 3] *= 1.f - h.w * h.w;
            }
            if (row >= p.M) {  // rows past M (zero-filled H) must not enter the sums
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0.f;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(stg + lane * 128 + ((j ^ (lane & 7)) * 16)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) tma_store_2d(&ymap, c0, (int)row0, stg);
          if (p.dtanh) {  // column c0 + lane of this box: 32 rows, fixed order
            float cs = 0.f;
            for (int rr = 0; rr < 32; ++rr)
              cs += *reinterpret_cast<const float*>(stg + rr * 128 + ((((lane >> 2) ^ (rr & 7)) * 16) + (lane & 3) * 4));
            if (hdir) {
              if (c0 == cfirst) cs_acc[0] += cs; else cs_acc[1] += cs;
            } else {
              s_csum[ew][c0 + lane] += cs;  // lane-owned slot
            }
          }
          if (++sb == p.nstg) sb = 0;
        } else if (row < p.M) {
          float* out = p.Y + row * p.ldy;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < p.N) out[c0 + j] = p.accumulate ? out[c0 + j] + v[j] : v[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.tempty[b]);
      if (hpre && t + 1 < my_tiles && lane == 0) {
        tma_store_wait_read();  // every box's store has read it
        load_h(t + 1);
      }
    }
    if (p.tma_store && lane == 0) tma_store_wait_all();
    if (hdir) {  // the warp's column sums into its (drained) staging box
      __syncwarp();
      float* sc = reinterpret_cast<float*>(stg0);
      if (nch > 0) sc[cfirst + lane] = cs_acc[0];
      if (nch > 1) sc[cfirst + cstep + lane] = cs_acc[1];
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (p.dtanh) {  // the CTA's column sums, epilogue warps in fixed order
    for (int c = threadIdx.x; c < p.N; c += kRowsThreads) {
      float a = 0.f;
      for (int w = 0; w < nepi; ++w)
        a += p.hdirect ? reinterpret_cast<const float*>(staging + (size_t)w * p.nstg * 4096)[c]
                       : s_csum[w][c];
      p.col_part[(int64_t)blockIdx.x * p.N + c] = a;
    }
  }
  if (warp == 1) tmem_dealloc(tmem, p.tmem_cols);
}

// ============================================================================
// weight gradient (reduction over rows), MN-major operands

struct WgArgs {
  float* C;  // partials [2 * gridDim.x][Mc][Nc] (or [..][Nc][Mc] when out_t)
  int64_t F, nblocks;
  int Mc, Nc, Mt, MSl, NSl, SR, Npad, concat, stacked, out_t, nraw, nbuf, flush_blocks, sum_col;
  int p_full, q_full;  // slabs loaded by the 3-D maps (the rest: one 2-D box each)
  uint32_t tmem_cols, acc_cols;
};

// Two operand arrangements (one 32-column slab = SR rows x 128 B, MN-major):
//  * stacked (Mc <= 64): raw slot [P raw (2 slabs) | P lo (2) | Q raw (NSl) | Q lo (NSl)];
//    the M = 128 A operand is [P_raw ; P_lo] and B is [Q_raw | Q_lo], so ONE
//    MMA per k-step yields all four products (incl. the tiny lo.lo); accumulator
//    rows 64.. hold the P_lo products and go to the CTA's second partial slice.
//  * split (Mc > 64, Mt <= 2 M tiles): raw slot [P raw (MSl) | Q raw | Q lo], lo ring
//    slot [P lo (MSl)]; per M tile and k-step P_raw.[Q_raw | Q_lo] + P_lo.Q_raw.
//    An M tile's MMA reads 4 slabs from its start: rows past Mc come from the
//    following regions (or the tail pad) and only feed rows that are never stored.
__global__ void __launch_bounds__(kThreads, 1)
tc_wgrad_kernel(const __grid_constant__ CUtensorMap pmap3, const __grid_constant__ CUtensorMap qmap3,
                const __grid_constant__ CUtensorMap pmap, const __grid_constant__ CUtensorMap qmap,
                WgArgs p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ Bars bars;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Mt = p.Mt;
  if (smem_u32(smem) & 1023) __trap();
  const uint32_t slab = (uint32_t)p.SR * 128;
  const uint32_t a_bytes = (uint32_t)(p.stacked ? 4 : p.MSl) * slab;  // A region in the raw slot
  const uint32_t b_bytes = (uint32_t)p.NSl * slab;
  const uint32_t lo_bytes = p.stacked ? 0u : (uint32_t)p.MSl * slab;  // lo ring slot
  const uint32_t raw_bytes = a_bytes + 2 * b_bytes;
  unsigned char* raw_ring = smem;
  unsigned char* lo_ring = smem + (size_t)p.nraw * raw_bytes;

  if (warp == 1) tmem_alloc(&tmem_base, p.tmem_cols);
  if (threadIdx.x == 0) {
    init_bars(bars, p.nraw);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pmap3)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&qmap3)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const int64_t my_blocks =
      p.nblocks > (int64_t)blockIdx.x ? (p.nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t rounds = (my_blocks + p.flush_blocks - 1) / p.flush_blocks;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      const uint32_t tx = (uint32_t)(p.MSl + p.NSl) * slab;
      Ring r(p.nraw);
      int64_t blk = blockIdx.x;
      for (int64_t s = 0; s < my_blocks; ++s, blk += gridDim.x, r.next()) {
        mbar_wait(&bars.raw_empty[r.slot], r.ph ^ 1u);
        unsigned char* base = raw_ring + (size_t)r.slot * raw_bytes;
        uint64_t* bar = &bars.raw_full[r.slot];
        mbar_expect_tx(bar, tx);
        const int r0 = (int)(blk * p.SR);
        // full 32-column slabs: one 3-D box per operand; a partial last slab: one 2-D box
        if (p.p_full) tma_load_3d(base, &pmap3, 0, r0, 0, bar);
        if (p.p_full < p.MSl) tma_load_2d(base + p.p_full * slab, &pmap, p.p_full * 32, r0, bar);
        unsigned char* bq = base + a_bytes;
        if (p.q_full) tma_load_3d(bq, &qmap3, 0, r0, 0, bar);
        if (p.q_full < p.NSl) tma_load_2d(bq + p.q_full * slab, &qmap, p.q_full * 32, r0, bar);
      }
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer (warp-wide loop, one elected lane issues)
      const int nq = p.NSl * 32;
      const uint32_t id1 = make_idesc(p.concat ? 2 * nq : p.Npad, 1, 1), id2 = make_idesc(p.Npad, 1, 1);
      Ring r(p.nraw), l(kNL);
      int64_t blk = 0;
      for (int64_t rd = 0; rd < rounds; ++rd) {
        const int b = p.nbuf == 2 ? (int)(rd & 1) : 0;
        const unsigned use = p.nbuf == 2 ? (unsigned)(rd >> 1) & 1u : (unsigned)rd & 1u;
        mbar_wait(&bars.tempty[b], use ^ 1u);
        tc_fence_after();
        const int64_t blk_end = blk + p.flush_blocks < my_blocks ? blk + p.flush_blocks : my_blocks;
        const int64_t blk0 = blk;
        for (; blk < blk_end; ++blk, r.next(), l.next()) {
          mbar_wait(&bars.raw_full[r.slot], r.ph);
          mbar_wait(&bars.lo_full[l.slot], l.ph);
          tc_fence_after();
          const uint32_t a_raw = smem_u32(raw_ring + (size_t)r.slot * raw_bytes);
          const uint32_t a_lo = smem_u32(lo_ring + (size_t)l.slot * lo_bytes);
          const uint32_t b_raw = a_raw + a_bytes, b_lo = b_raw + b_bytes;
          for (int s = 0; s < p.SR / 8; ++s) {
            const uint32_t ko = s * 1024;  // two 4-row K atoms per k-step
            const uint64_t br = make_sdesc(b_raw + ko, slab, 512, 1);
            const uint32_t acc = (blk > blk0 || s > 0) ? 1u : 0u;
            if (p.stacked) {
              const uint32_t d = tmem + (uint32_t)(b * p.acc_cols);
              const uint64_t ar = make_sdesc(a_raw + ko, slab, 512, 1);  // [P_raw ; P_lo]
              if (p.concat) {
                mma_tf32_w(d, ar, br, id1, acc);
              } else {
                mma_tf32_w(d, ar, br, id2, acc);
                mma_tf32_w(d, ar, make_sdesc(b_lo + ko, slab, 512, 1), id2, 1u);
              }
              continue;
            }
            for (int t = 0; t < Mt; ++t) {
              const uint32_t d = tmem + (uint32_t)((b * Mt + t) * p.acc_cols);
              const uint32_t ao = (uint32_t)t * 4 * slab + ko;
              const uint64_t ar = make_sdesc(a_raw + ao, slab, 512, 1);
              const uint64_t al = make_sdesc(a_lo + ao, slab, 512, 1);
              if (p.concat) {
                mma_tf32_w(d, ar, br, id1, acc);  // [P.Q_hi | P.Q_lo]
              } else {
                mma_tf32_w(d, ar, br, id2, acc);
                mma_tf32_w(d, ar, make_sdesc(b_lo + ko, slab, 512, 1), id2, 1u);
              }
              mma_tf32_w(d, al, br, id2, 1u);  // + P_lo.Q_hi
            }
          }
          mma_commit_w(&bars.raw_empty[r.slot]);
          mma_commit_w(&bars.lo_empty[l.slot]);
        }
        mma_commit_w(&bars.tfull[b]);
      }
    }
  } else if (warp < kEpiWarp0) {
    // ---- converters: lo halves (P lo into the raw slot when stacked, else the lo ring)
    const int t = threadIdx.x - kConvWarp0 * 32;
    Ring r(p.nraw), l(kNL);
    for (int64_t s = 0; s < my_blocks; ++s, r.next(), l.next()) {
      mbar_wait(&bars.raw_full[r.slot], r.ph);
      mbar_wait(&bars.lo_empty[l.slot], l.ph ^ 1u);
      unsigned char* base = raw_ring + (size_t)r.slot * raw_bytes;
      if (p.stacked)
        convert_lo(base, base + 2 * slab, 2 * slab, t);
      else
        convert_lo(base, lo_ring + (size_t)l.slot * lo_bytes, lo_bytes, t);
      convert_lo(base + a_bytes, base + a_bytes + b_bytes, b_bytes, t);
      fence_proxy_async();
      mbar_arrive(&bars.lo_full[l.slot]);
    }
  } else {
    // ---- epilogue: fold each flushed accumulator into a running fp32 sum kept
    // in TMEM (columns sum_col..), write this CTA's partials once at the end
    const int q = warp & 3;
    const int nq = p.NSl * 32;
    const int tiles = p.stacked ? 1 : Mt;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    for (int64_t rd = 0; rd < rounds; ++rd) {
      const int b = p.nbuf == 2 ? (int)(rd & 1) : 0;
      const unsigned use = p.nbuf == 2 ? (unsigned)(rd >> 1) & 1u : (unsigned)rd & 1u;
      mbar_wait(&bars.tfull[b], use);
      tc_fence_after();
      for (int t = 0; t < tiles; ++t) {
        const uint32_t tb = lane_base + (uint32_t)((b * tiles + t) * p.acc_cols);
        const uint32_t sb = lane_base + p.sum_col + (uint32_t)(t * p.Npad);
        for (int c0 = 0; c0 < p.Npad; c0 += 16) {
          uint32_t r[16], r2[16], acc[16];
          tmem_ld16(tb + c0, r);
          if (p.concat) tmem_ld16(tb + nq + c0, r2);
          if (rd > 0) tmem_ld16(sb + c0, acc);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float v = __uint_as_float(r[j]) + (p.concat ? __uint_as_float(r2[j]) : 0.f);
            if (rd > 0) v += __uint_as_float(acc[j]);
            acc[j] = __float_as_uint(v);
          }
          tmem_st16(sb + c0, acc);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.tempty[b]);
    }
    // this CTA's two partial slices, fixed order (deterministic): stacked rows
    // 64.. (the P_lo products) go to the second slice, otherwise it is zero
    const int64_t slice = (int64_t)p.Mc * p.Nc;
    float* part = p.C + (int64_t)blockIdx.x * 2 * slice;
    if (!p.stacked)
      for (int i = (warp - kEpiWarp0) * 32 + lane; i < slice; i += kEpiWarps * 32) part[slice + i] = 0.f;
    for (int t = 0; t < tiles; ++t) {
      const int lrow = t * BM + q * 32 + lane;
      const int m = p.stacked ? (lrow & 63) : lrow;
      float* dstp = part + (p.stacked && lrow >= 64 ? slice : 0);
      const uint32_t sb = lane_base + p.sum_col + (uint32_t)(t * p.Npad);
      for (int c0 = 0; c0 < p.Npad; c0 += 16) {
        uint32_t acc[16];
        if (rounds > 0) {
          tmem_ld16(sb + c0, acc);
          tmem_wait_ld();
        }
        if (m < p.Mc) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int c = c0 + j;
            if (c < p.Nc)
              dstp[p.out_t ? (int64_t)c * p.Mc + m : (int64_t)m * p.Nc + c] =
                  rounds > 0 ? __uint_as_float(acc[j]) : 0.f;
          }
        }
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, p.tmem_cols);
}

// ---- host ---------------------------------------------------------------------

int launch_rows(const float* X, const float* W, float* Y, const float* bias, int64_t M, int64_t K,
                int N, int64_t ldx, int64_t ldw, int64_t ldy, int w_trans, int act_tanh,
                int accumulate, cudaStream_t st, const float* H = nullptr, int64_t ldh = 0,
                float* col_part = nullptr, unsigned* nonfinite = nullptr) {
  const int Npad = (N + 31) / 32 * 32;  // the epilogue drains 32 columns at a time
  const int kblocks = (int)ceil_div(K, BK);
  const size_t wbytes = (size_t)kblocks * Npad * BK * 4 * 2;
  const size_t fixed = (size_t)kNL * kTile + (size_t)kEpiWarps * 4096;  // lo ring + 1 staging box
  if (wbytes + fixed + 2 * kTile > kRowsBudget && N > 32 && !H) {
    // resident [W_hi; W_lo] too large for a useful ring: split the output columns
    const int n1 = (N / 2 + 31) / 32 * 32;
    const float* W2 = w_trans ? W + n1 : W + (int64_t)n1 * ldw;
    if (int e = launch_rows(X, W, Y, bias, M, K, n1, ldx, ldw, ldy, w_trans, act_tanh, accumulate, st,
                            nullptr, 0, nullptr, nonfinite))
      return e;
    return launch_rows(X, W2, Y + n1, bias ? bias + n1 : nullptr, M, K, N - n1, ldx, ldw, ldy,
                       w_trans, act_tanh, accumulate, st);
  }
  if (wbytes + fixed + 2 * kTile > kRowsBudget)
    return fail(kDimension, "tc_gemm: resident weight %d x %lld too large", N, (long long)K);
  CUtensorMap xmap, ymap;
  if (int e = make_map(&xmap, X, M, K, ldx, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B)) return e;
  RowArgs p;
  p.W = W; p.Y = Y; p.bias = bias;
  p.has_bias = bias ? 1 : 0;
  p.M = M; p.K = (int)K; p.N = N;
  p.Npad = Npad;
  p.concat = 2 * Npad <= 256 ? 1 : 0;
  p.kblocks = kblocks;
  p.last_ksteps = (int)ceil_div(K - (int64_t)(kblocks - 1) * BK, 8);
  p.ldw = ldw; p.ldy = ldy;
  p.w_trans = w_trans; p.act_tanh = act_tanh; p.accumulate = accumulate;
  p.y_vec = (ldy % 4 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0) ? 1 : 0;
  p.tma_store = (p.y_vec && !accumulate) ? 1 : 0;
  if (p.tma_store) {
    if (int e = make_map(&ymap, Y, M, N, ldy, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)) return e;
  } else {
    ymap = xmap;  // unused
  }
  CUtensorMap hmap = xmap;  // unused unless dtanh (H boxes)
  p.dtanh = H ? 1 : 0;
  p.col_part = col_part;
  p.nonfinite = nonfinite;
  // a large resident weight: H straight from global memory, no H boxes (the ring
  // keeps the stages the plain product has)
  p.hdirect = (H && wbytes >= (size_t)ACCEL_ROWS_HDIRECT_WBYTES && Npad <= 64 && N % 32 == 0 &&
               ldh % 4 == 0 && (reinterpret_cast<uintptr_t>(H) & 15) == 0) ? 1 : 0;
  p.Hp = H;
  p.ldh = ldh;
  if (H) {
    if (!p.tma_store || !col_part || act_tanh || bias || N > 256)
      return fail(kDimension, "tc_gemm dtanh: needs an aligned output, col_part, no bias/act");
    if (!p.hdirect)
      if (int e = make_map(&hmap, H, M, N, ldh, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)) return e;
  }
  p.ntiles = ceil_div(M, BM);
  p.acc_cols = p.concat ? 2 * Npad : Npad;
  p.tmem_cols = tmem_cols_for(2 * (int)p.acc_cols);
  // epilogue warps: 8 when the ring still keeps >= 6 slots beside their two
  // staging boxes each (narrow K: the epilogue is the longer pole), else 4;
  // staging: two boxes per epilogue warp when the raw ring keeps >= 6 slots
  const bool hbox = H && !p.hdirect;  // H boxes + shared-memory column sums
  auto ring_left = [&](int nepi, int nstg) -> int64_t {
    const size_t sb = (size_t)nepi * nstg * 4096 + (hbox ? (size_t)nepi * 256 * 4 : 0);
    const size_t used = wbytes + (size_t)kNL * kTile + sb;
    return used > kRowsBudget ? -1 : (int64_t)((kRowsBudget - used) / kTile);
  };
  // (with 8 warps a warp drains ceil(Npad / 64) chunks per tile: one box each, up to two)
  const int nstg8 = std::min(2, (Npad + 63) / 64);
  p.nepi = (p.tma_store && !p.hdirect && Npad >= 64 && ring_left(kRowsEpiMax, nstg8) >= 4)
               ? kRowsEpiMax
               : kEpiWarps;
  p.nstg = p.tma_store ? (p.nepi == kRowsEpiMax ? nstg8 : 2) : 0;
  if (p.tma_store && p.nstg == 2 && ring_left(p.nepi, 2) < 6) p.nstg = 1;
  const size_t sbytes = (size_t)p.nepi * p.nstg * 4096 + (hbox ? (size_t)p.nepi * 256 * 4 : 0);
  p.nraw = (int)std::min<size_t>(kMaxRaw, (kRowsBudget - wbytes - sbytes - kNL * kTile) / kTile);
  const size_t smem = wbytes + (size_t)(p.nraw + kNL) * kTile + sbytes;
  cudaError_t e = cudaFuncSetAttribute(tc_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return fail(kCuda, "tc_rows smem: %s", cudaGetErrorString(e));
  const int grid = (int)std::min<int64_t>(p.ntiles, sm_count());
  tc_rows_kernel<<<grid, kRowsThreads, smem, st>>>(xmap, ymap, hmap, p);
  return post_launch("tc_rows_kernel");
}

// C partials [2 * slices][n][k] of dY[F, n]^T X[F, k]
int launch_wgrad(const float* dY, const float* X, float* C, int64_t F, int n, int k,
                 int64_t ldy, int64_t ldx, int slices, cudaStream_t st) {
  // pick orientation (which side is the UMMA M side) and arrangement by the
  // tensor-core cycles per k-step (measured: an M = 128 MMA of N columns takes
  // max(48, N / 2) cycles)
  auto mma = [](int nc) { return std::max(48, nc / 2); };
  auto plan = [&](int mc, int nc, bool stacked) -> int {
    const int nsl = (nc + 31) / 32, npad = (nc + 15) / 16 * 16;
    const bool concat = 2 * nsl * 32 <= 256;
    if (stacked) return mc <= 64 ? (concat ? mma(2 * nsl * 32) : 2 * mma(npad)) : 1 << 30;
    const int mt = (mc + BM - 1) / BM;
    if (mt > 2 || nsl > 8) return 1 << 30;
    const int c = mt * (concat ? mma(2 * nsl * 32) + mma(npad) : 3 * mma(npad));
    // two M tiles also convert and stage the wide P's lo halves through the lo
    // ring: measured slower than the MMA count says (G^T h2, 256 x 64: split 543 us,
    // stacked with the operands swapped 480 us)
    return mt == 2 ? c + c / 4 : c;
  };
  int best = 1 << 30;
  bool swap = false, stacked = false;
  for (int sw = 0; sw < 2; ++sw)
    for (int stk = 1; stk >= 0; --stk) {
      const int c = sw ? plan(k, n, stk) : plan(n, k, stk);
      if (c < best) best = c, swap = sw, stacked = stk;
    }
  if (best == 1 << 30) return fail(kDimension, "tc_wgrad: output %d x %d too large", n, k);
  WgArgs p;
  const float* P = swap ? X : dY;
  const float* Q = swap ? dY : X;
  const int64_t ldp = swap ? ldx : ldy, ldq = swap ? ldy : ldx;
  p.Mc = swap ? k : n;
  p.Nc = swap ? n : k;
  p.out_t = swap ? 1 : 0;
  p.stacked = stacked ? 1 : 0;
  p.C = C;
  p.F = F;
  p.Mt = stacked ? 1 : (p.Mc + BM - 1) / BM;
  p.MSl = (p.Mc + 31) / 32;
  p.NSl = (p.Nc + 31) / 32;
  p.Npad = (p.Nc + 15) / 16 * 16;
  p.concat = 2 * p.NSl * 32 <= 256 ? 1 : 0;
  p.acc_cols = p.concat ? 2 * p.NSl * 32 : p.Npad;
  // TMEM: nbuf x Mt accumulators, then Mt running sums of Npad columns
  const int acc_total = p.Mt * (int)p.acc_cols, sum_total = p.Mt * p.Npad;
  if (acc_total + sum_total > 512) return fail(kDimension, "tc_wgrad: accumulator exceeds TMEM");
  p.nbuf = 2 * acc_total + sum_total <= 512 ? 2 : 1;
  p.sum_col = p.nbuf * acc_total;
  p.tmem_cols = tmem_cols_for(p.nbuf * acc_total + sum_total);
  // stage rows: the largest of 64 / 32 / 16 that leaves >= 3 raw slots
  const int a_slabs = stacked ? 4 : p.MSl, lo_slabs = stacked ? 0 : p.MSl;
  auto raw_of = [&](int sr) { return (size_t)(a_slabs + 2 * p.NSl) * sr * 128; };
  auto lo_of = [&](int sr) { return (size_t)lo_slabs * sr * 128; };
  // split mode: the last lo slot's M-tile reads may run (4 * Mt - MSl) slabs past the ring
  auto pad_of = [&](int sr) { return stacked ? (size_t)0 : (size_t)(4 * p.Mt - p.MSl) * sr * 128; };
  p.SR = 16;
  for (int sr : {64, 32}) {
    if ((kSmemBudget - kNL * lo_of(sr) - pad_of(sr)) / raw_of(sr) >= 3) {
      p.SR = sr;
      break;
    }
  }
  p.nraw = (int)std::min<size_t>(kMaxRaw, (kSmemBudget - kNL * lo_of(p.SR) - pad_of(p.SR)) / raw_of(p.SR));
  if (p.nraw < 2) return fail(kDimension, "tc_wgrad: stage too large");
  p.nblocks = ceil_div(F, p.SR);
  p.flush_blocks = kFlushRows / p.SR;
  p.p_full = p.Mc / 32;
  p.q_full = p.Nc / 32;
  CUtensorMap pmap3, qmap3, pmap, qmap;
  if (int e = make_map(&pmap, P, F, p.Mc, ldp, 32, p.SR, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return e;
  if (int e = make_map(&qmap, Q, F, p.Nc, ldq, 32, p.SR, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return e;
  pmap3 = pmap;
  qmap3 = qmap;
  if (p.p_full)
    if (int e = make_map3(&pmap3, P, F, p.p_full, ldp, p.SR)) return e;
  if (p.q_full)
    if (int e = make_map3(&qmap3, Q, F, p.q_full, ldq, p.SR)) return e;
  const size_t smem = (size_t)p.nraw * raw_of(p.SR) + kNL * lo_of(p.SR) + pad_of(p.SR);
  cudaError_t e = cudaFuncSetAttribute(tc_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return fail(kCuda, "tc_wgrad smem: %s", cudaGetErrorString(e));
  const int grid = std::max(1, slices);
  tc_wgrad_kernel<<<grid, kThreads, smem, st>>>(pmap3, qmap3, pmap, qmap, p);
  return post_launch("tc_wgrad_kernel");
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_tc_sm_count(void) { return sm_count(); }

// accel_tc_gemm's row transform (a_trans = 0, B [N, K]) that also adds the
// number of non-finite elements of A to *nonfinite (the frame check of
// build_train_batch, trainer.py:392-396, folded into the first layer's read).
extern "C" int accel_tc_linear_checked(const float* A, const float* B, float* C, const float* bias,
                                       int64_t M, int64_t K, int N, int64_t lda, int64_t ldb,
                                       int64_t ldc, int act_tanh, unsigned* nonfinite,
                                       void* stream) {
  if (M < 0 || K < 1 || N < 1 || N > 256) return fail(kDimension, "tc_linear_checked: bad sizes");
  if (M == 0) return kOk;
  if (!A || !B || !C || !nonfinite) return fail(kDimension, "tc_linear_checked: NULL buffer");
  if (K > INT32_MAX || M > INT32_MAX) return fail(kDimension, "tc_linear_checked: too large");
  return launch_rows(A, B, C, bias, M, K, N, lda, ldb, ldc, 0, act_tanh, 0, as_stream(stream),
                     nullptr, 0, nullptr, nonfinite);
}

extern "C" int accel_tc_rows_grid(int64_t M) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(M, BM), sm_count()));
}

// C[M, N] = (A[M, K] . B^T) * (1 - H[M, N]^2) -- a GEMM fused with the tanh
// derivative of its output rows -- and col_part[accel_tc_rows_grid(M)][N] = the
// per-CTA column sums of C (fixed order; the caller reduces them).
extern "C" int accel_tc_gemm_dtanh(const float* A, const float* B, float* C, const float* H,
                                   float* col_part, int64_t M, int64_t K, int N, int64_t lda,
                                   int64_t ldb, int64_t ldc, int64_t ldh, int b_trans,
                                   void* stream) {
  if (M < 0 || K < 1 || N < 1 || N > 256) return fail(kDimension, "tc_gemm_dtanh: bad sizes");
  if (M == 0) return kOk;
  if (!A || !B || !C || !H || !col_part) return fail(kDimension, "tc_gemm_dtanh: NULL buffer");
  if (K > INT32_MAX || M > INT32_MAX) return fail(kDimension, "tc_gemm_dtanh: too large");
  return launch_rows(A, B, C, nullptr, M, K, N, lda, ldb, ldc, b_trans, 0, 0, as_stream(stream), H,
                     ldh, col_part);
}

// C[M, N] = act(A . B^T + bias) (+ C if accumulate).  a_trans: A stored [K, M];
// b_trans: B stored [K, N].  a_trans && b_trans (weight gradient, reduction over
// the K rows): C receives [2 * kslices][M][N] fp32 partials, two per persistent CTA.
extern "C" int accel_tc_gemm(const float* A, const float* B, float* C, const float* bias,
                             int64_t M, int64_t K, int N, int64_t lda, int64_t ldb, int64_t ldc,
                             int a_trans, int b_trans, int act_tanh, int accumulate, int kslices,
                             void* stream) {
  if (M < 0 || K < 1 || N < 1 || N > 256 || kslices < 1)
    return fail(kDimension, "tc_gemm: bad sizes M=%lld K=%lld N=%d", (long long)M, (long long)K, N);
  if (M == 0) return kOk;
  if (!A || !B || !C) return fail(kDimension, "tc_gemm: NULL buffer");
  if (K > INT32_MAX) return fail(kDimension, "tc_gemm: K too large");
  if (a_trans && b_trans) {
    if (M > 256 || bias || act_tanh || accumulate)
      return fail(kDimension, "tc_gemm: weight-gradient mode takes M <= 256, no epilogue");
    return launch_wgrad(A, B, C, K, (int)M, N, lda, ldb, kslices, as_stream(stream));
  }
  if (a_trans || kslices != 1)
    return fail(kDimension, "tc_gemm: unsupported operand layout");
  if (M > INT32_MAX) return fail(kDimension, "tc_gemm: M too large");
  return launch_rows(A, B, C, bias, M, K, N, lda, ldb, ldc, b_trans, act_tanh, accumulate,
                     as_stream(stream));
}
