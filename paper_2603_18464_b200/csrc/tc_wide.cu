// Wide fp32-accurate GEMMs on tcgen05 (cfg4: the OpenVLA-7B-shaped heads, O = D = 4096).
//
// The row kernels of tc_gemm.cu keep the whole (<= 256 x 256) weight resident in
// shared memory; at cfg4 every product of the policy / value heads has two
// dimensions of 4096 (models.py:176-182 forward, :191-204 backward; value head
// :283-314), so here both operands stream through a TMA ring, tile by tile:
//
//   C[M, N] = A[M, K] . B[N, K]^T      (UMMA: D[m, n] = sum_k A[m, k] B[n, k])
//
// with each operand K-major (k contiguous: activations in a forward product,
// weights [out, in]) or MN-major (m / n contiguous: a weight used as [in, out],
// or both operands of a weight gradient, whose reduction runs over the rows).
//
// Accuracy (the 1e-4 gradient tolerance rules out plain TF32).  Every fp32 x is
// x = hi + lo with hi = trunc19(x), the value the tensor core reads from a raw
// fp32 word.  Per 8-wide k step the kernel issues TWO MMAs into one fp32 TMEM
// accumulator:
//   kind::tf32  A_raw . B_raw                       = A_hi B_hi
//   kind::f16   [bf16(A_hi) x8 | bf16(A_lo) x8] . [bf16(B_lo) x8 | bf16(B_hi) x8]
//                                                   = A_hi B_lo + A_lo B_hi
// The correction terms are ~2^-10 of the main term, so rounding them to bf16
// costs ~2^-19 relative (the dropped lo.lo is ~2^-20): fp32-class accuracy for
// two tensor-core passes instead of 3xTF32's three (a K = 16 bf16 MMA takes the
// cycles of a K = 8 tf32 one).  The bf16 "pair" operands are written by
// accel_tf32_pairs (one HBM-bound elementwise pass per operand).
//
// Persistent, warp-specialised (192 threads, one CTA per SM): warp 0 lane 0
// issues the TMA loads of a 4..8-stage ring (16 k per stage: raw fp32 tiles
// with 64 B-swizzled K-major rows or 128 B-swizzled MN-major slabs, bf16 pair
// tiles alike); warp 1 issues the MMAs (one elected lane) into double-buffered
// TMEM accumulators (128 x BN fp32, BN <= 256); warps 2-5 drain them
// (tcgen05.ld, 32 columns at a time) through the epilogue: plain store, bias +
// tanh, the tanh derivative (Y = acc (1 - H^2)) with per-tile column sums for
// the bias gradient, or split-K partial slices (reduced by the caller in fixed
// order: deterministic).  Work units (m tile, n tile, k slice) are dealt n-tile
// fastest, so CTAs running together share the A tile rows through L2.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "tc_common.cuh"

namespace accel {
namespace {

using namespace tc;

constexpr int kWThreads = 192;  // 6 warps
constexpr int kWEpi0 = 2;       // epilogue warps 2..5
constexpr int kBK = 16;         // fp32 k per stage (two 8-k MMA steps)
constexpr int kMaxStages = 8;
// k blocks per accumulation chunk; 0 = one chunk per work unit.  Chunking only
// shrinks the fp32 truncation drift by sqrt(#chunks) and costs an output
// read-modify-write per chunk, so it is off by default (drift ~ n_mma 2^-25
// relative: 2e-5 at K = 4096, the same accumulator cuBLAS's TF32 GEMMs use).
int g_chunk_kb = 0;
int g_wide_multicast = 2;  // 2-CTA clusters: 2 = 2-SM UMMA, 1 = B multicast, 0 = off
constexpr size_t kWideSmem = 222 * 1024;  // dynamic (ring); + ~5 KB static

enum Epi : int { kStore = 0, kBiasTanh = 1, kDtanh = 2, kPartial = 3 };

struct WideArgs {
  float* C;
  const float* bias;
  const float* H;
  float* col_part;  // kDtanh: [m_tiles][N] column sums of Y (per m tile, fixed order)
  int64_t M, N, ldc, ldh;
  int BN, m_tiles, n_tiles, kslices, kblocks, a_mn, b_mn, epi, nstages, vec, hvec;
  int chunk_kb;      // k blocks per accumulation chunk (bounds the truncating fp32 sum)
  int mc;            // 2-CTA clusters: m tiles 2g, 2g + 1 share (multicast) each B tile
  int a_3d, b_3d;    // MN-major operand loaded by one 3-D box per stage (MN % 64 == 0)
  uint32_t stage_bytes, a_pair_off, b_raw_off, b_pair_off, tx_bytes, tmem_cols;
};

__device__ __forceinline__ void mma_bf16_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// ---- 2-CTA clusters sharing the B tile (TMA multicast) ----
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, int c0, int c1,
                                               int c2, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// the MMAs of this CTA that read a stage are done: arrive on that stage's empty
// barrier in every CTA of `mask` (the peer's B half lives in this stage too)
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}\n" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// ---- 2-SM UMMA (cta_group::2): the pair computes one 256 x BN tile ----
// The leader (cluster rank 0) issues every MMA; each CTA holds its own 128 A
// rows and half of the B tile in its shared memory and its 128 accumulator rows
// in its TMEM.  TMA loads of both CTAs complete on the LEADER's full barrier (the
// peer's barrier address with the cluster-rank bit cleared).
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, int c0, int c1,
                                                uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_cg2(void* dst, const CUtensorMap* map, int c0, int c1,
                                                int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar) & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_w2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_bf16_w2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc));
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {  // both CTAs' barrier at this offset
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}\n" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   smem_u32(bar) & kPeerMask)
               : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols)
               : "memory");
}
// instruction descriptor with an explicit M (256 for cta_group::2); bf16: kind::f16 / BF16
__device__ __forceinline__ uint32_t make_idesc_m(int n, int m, int a_mn, int b_mn, int bf16) {
  const uint32_t fmt = bf16 ? 1u : 2u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// This CTA's share of a 2-SM B tile (rows r0, rows of them) into its own B region;
// completes on the leader's barrier.
__device__ __forceinline__ void load_operand_cg2(unsigned char* raw, unsigned char* pair,
                                                 const CUtensorMap* rmap, const CUtensorMap* pmap,
                                                 int mn, int three_d, int r0, int rows, int kb,
                                                 uint64_t* bar) {
  if (mn && three_d) {
    tma_load_3d_cg2(raw, rmap, 0, kb * kBK, r0 / 32, bar);
    tma_load_3d_cg2(pair, pmap, 0, kb * 2 * kBK, r0 / 64, bar);
  } else if (mn) {
    for (int j = 0; j < rows / 32; ++j)
      tma_load_2d_cg2(raw + j * (kBK * 128), rmap, r0 + 32 * j, kb * kBK, bar);
    for (int j = 0; j < rows / 64; ++j)
      tma_load_2d_cg2(pair + j * (2 * kBK * 128), pmap, r0 + 64 * j, kb * 2 * kBK, bar);
  } else {
    tma_load_2d_cg2(raw, rmap, kb * kBK, r0, bar);
    tma_load_2d_cg2(pair, pmap, kb * 2 * kBK, r0, bar);
  }
}

// kind::f16 with bf16 A/B, fp32 D, M = 128, N = n
__device__ __forceinline__ uint32_t make_idesc_bf16(int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ float tanh_fast(float x) {
  const float t = __expf(2.f * x);
  return 1.f - __fdividef(2.f, t + 1.f);
}

// operand descriptors at k step s of a stage (see the layouts in launch_wide)
__device__ __forceinline__ uint64_t raw_desc(uint32_t base, int mn, int s) {
  return mn ? make_sdesc(base + s * 1024, kBK * 128, 512, 1)   // 32-col slabs of 16 rows
            : make_sdesc(base + s * 32, 16, 512, 4);           // 64 B rows, SWIZZLE_64B
}
__device__ __forceinline__ uint64_t pair_desc(uint32_t base, int mn, int s) {
  return mn ? make_sdesc(base + s * 2048, 2 * kBK * 128, 1024, 2)  // 64-col atoms of 32 rows
            : make_sdesc(base + s * 32, 16, 512, 4);
}

// TMA loads of one operand tile (rows r0.. of the MN dimension, k block kb).
// MN-major: 32-column fp32 slabs of 16 k rows and 64-column bf16 atoms of 32
// pair rows, slab / atom-major in shared memory -- one 3-D box each when the
// MN extent is a multiple of 64 (three_d), else one 2-D box per slab / atom.
__device__ __forceinline__ void load_operand(unsigned char* raw, unsigned char* pair,
                                             const CUtensorMap* rmap, const CUtensorMap* pmap,
                                             int mn, int three_d, int r0, int rows, int kb,
                                             uint64_t* bar) {
  if (mn && three_d) {
    tma_load_3d(raw, rmap, 0, kb * kBK, r0 / 32, bar);
    tma_load_3d(pair, pmap, 0, kb * 2 * kBK, r0 / 64, bar);
  } else if (mn) {
    for (int j = 0; j < rows / 32; ++j)
      tma_load_2d(raw + j * (kBK * 128), rmap, r0 + 32 * j, kb * kBK, bar);
    for (int j = 0; j < rows / 64; ++j)
      tma_load_2d(pair + j * (2 * kBK * 128), pmap, r0 + 64 * j, kb * 2 * kBK, bar);
  } else {
    tma_load_2d(raw, rmap, kb * kBK, r0, bar);        // rows x 16 fp32
    tma_load_2d(pair, pmap, kb * 2 * kBK, r0, bar);   // rows x 32 bf16
  }
}

// One CTA's half of a cluster-shared B tile (rows r0 + half * rows/2 ..), written
// into both CTAs' shared memory at the half's offset (TMA multicast, mask 0b11).
__device__ __forceinline__ void load_operand_half(unsigned char* raw, unsigned char* pair,
                                                  const CUtensorMap* rmap,
                                                  const CUtensorMap* pmap, int mn, int three_d,
                                                  int r0, int rows, int kb, int half,
                                                  uint64_t* bar) {
  const int hr = rows / 2;
  const uint32_t hoff = (uint32_t)hr * kBK * 4;  // bytes of half a tile (raw == pair)
  raw += half * hoff;
  pair += half * hoff;
  r0 += half * hr;
  if (mn && three_d) {
    tma_load_3d_mc(raw, rmap, 0, kb * kBK, r0 / 32, bar, 3);
    tma_load_3d_mc(pair, pmap, 0, kb * 2 * kBK, r0 / 64, bar, 3);
  } else if (mn) {
    for (int j = 0; j < hr / 32; ++j)
      tma_load_2d_mc(raw + j * (kBK * 128), rmap, r0 + 32 * j, kb * kBK, bar, 3);
    for (int j = 0; j < hr / 64; ++j)
      tma_load_2d_mc(pair + j * (2 * kBK * 128), pmap, r0 + 64 * j, kb * 2 * kBK, bar, 3);
  } else {
    tma_load_2d_mc(raw, rmap, kb * kBK, r0, bar, 3);
    tma_load_2d_mc(pair, pmap, kb * 2 * kBK, r0, bar, 3);
  }
}

struct WideBars {
  uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2];
};

template <int MODE>  // 0 one CTA per tile, 1 B multicast pairs, 2 2-SM UMMA pairs
__global__ void __launch_bounds__(kWThreads, 1)
tc_wide_kernel(const __grid_constant__ CUtensorMap a_raw, const __grid_constant__ CUtensorMap a_pair,
               const __grid_constant__ CUtensorMap b_raw, const __grid_constant__ CUtensorMap b_pair,
               WideArgs p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ WideBars bars;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float s_col[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (smem_u32(smem) & 1023) __trap();
  const int BN = p.BN;
  constexpr bool cg2 = MODE == 2;  // 2-SM UMMA; MODE 1: 1-SM MMAs, B tile multicast
  if (warp == 1) {
    if constexpr (cg2)
      tmem_alloc2(&tmem_base, p.tmem_cols);
    else
      tmem_alloc(&tmem_base, p.tmem_cols);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstages; ++s) {
      mbar_init(&bars.full[s], 1);
      mbar_init(&bars.empty[s], MODE == 1 ? 2 : 1);  // multicast: both CTAs' MMAs read it
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.tfull[b], 1);
      mbar_init(&bars.tempty[b], cg2 ? 8 : 4);  // cg2: both CTAs' epilogue warps (leader's)
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a_raw)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&b_raw)) : "memory");
  }
  tc_fence_before();
  if constexpr (MODE != 0)
    cluster_sync_all();  // the peer's barriers exist before anything is multicast into them
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  // work units (k slice, m group, n tile), n fastest; an m group is one m tile, or
  // the two m tiles of a cluster (rank r takes tile 2g + r, both share B)
  const int mstep = MODE ? 2 : 1, rank = MODE ? (int)(blockIdx.x & 1) : 0;
  const int64_t worker = MODE ? blockIdx.x >> 1 : blockIdx.x;
  const int64_t nworkers = MODE ? gridDim.x >> 1 : gridDim.x;
  const int64_t m_groups = (p.m_tiles + mstep - 1) / mstep;
  const int64_t units = m_groups * p.n_tiles * p.kslices;
  const int64_t my_units = units > worker ? (units - 1 - worker) / nworkers + 1 : 0;
  auto decode = [&](int64_t t, int& ks, int& mt, int& nt, int& kb0, int& kb1) {
    const int64_t u = worker + t * nworkers;
    const int64_t mn = m_groups * p.n_tiles;
    ks = (int)(u / mn);
    const int64_t r = u - (int64_t)ks * mn;
    const int mg = (int)(r / p.n_tiles);
    nt = (int)(r - (int64_t)mg * p.n_tiles);
    mt = mg * mstep + rank;
    kb0 = (int)((int64_t)ks * p.kblocks / p.kslices);
    kb1 = (int)((int64_t)(ks + 1) * p.kblocks / p.kslices);
  };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int slot = 0;
      unsigned ph = 0;
      for (int64_t t = 0; t < my_units; ++t) {
        int ks, mt, nt, kb0, kb1;
        decode(t, ks, mt, nt, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&bars.empty[slot], ph ^ 1u);
          unsigned char* st = smem + (size_t)slot * p.stage_bytes;
          uint64_t* bar = &bars.full[slot];
          if constexpr (cg2) {  // both CTAs' loads complete on the leader's barrier
            if (rank == 0) mbar_expect_tx(bar, p.tx_bytes);
            load_operand_cg2(st, st + p.a_pair_off, &a_raw, &a_pair, p.a_mn, p.a_3d, mt * kBM,
                             kBM, kb, bar);
            load_operand_cg2(st + p.b_raw_off, st + p.b_pair_off, &b_raw, &b_pair, p.b_mn,
                             p.b_3d, nt * BN + rank * (BN / 2), BN / 2, kb, bar);
            if (++slot == p.nstages) {
              slot = 0;
              ph ^= 1u;
            }
            continue;
          }
          mbar_expect_tx(bar, p.tx_bytes);
          load_operand(st, st + p.a_pair_off, &a_raw, &a_pair, p.a_mn, p.a_3d, mt * kBM, kBM, kb,
                       bar);
          if constexpr (MODE == 1)
            load_operand_half(st + p.b_raw_off, st + p.b_pair_off, &b_raw, &b_pair, p.b_mn,
                              p.b_3d, nt * BN, BN, kb, rank, bar);
          else
            load_operand(st + p.b_raw_off, st + p.b_pair_off, &b_raw, &b_pair, p.b_mn, p.b_3d,
                         nt * BN, BN, kb, bar);
          if (++slot == p.nstages) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (warp-wide loop, one elected lane issues); under cg2 the
    // leader issues the pair's MMAs (M = 256) and the peer's MMA warp idles
    const uint32_t id_tf = cg2 ? make_idesc_m(BN, 256, p.a_mn, p.b_mn, 0)
                               : make_idesc(BN, p.a_mn, p.b_mn);
    const uint32_t id_bf = cg2 ? make_idesc_m(BN, 256, p.a_mn, p.b_mn, 1)
                               : make_idesc_bf16(BN, p.a_mn, p.b_mn);
    int slot = 0;
    unsigned ph = 0;
    int64_t c = 0;  // accumulation chunks issued by this CTA (TMEM buffer c & 1)
    for (int64_t t = 0; t < (cg2 && rank != 0 ? 0 : my_units); ++t) {
      int ks, mt, nt, kb0, kb1;
      decode(t, ks, mt, nt, kb0, kb1);
      for (int cb0 = kb0; cb0 < kb1; cb0 += p.chunk_kb, ++c) {
        const int cb1 = min(kb1, cb0 + p.chunk_kb);
        const int b = (int)(c & 1);
        mbar_wait(&bars.tempty[b], ((unsigned)(c >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        for (int kb = cb0; kb < cb1; ++kb) {
          mbar_wait(&bars.full[slot], ph);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + (size_t)slot * p.stage_bytes);
          if constexpr (cg2) {
#pragma unroll
            for (int s = 0; s < kBK / 8; ++s) {
              mma_tf32_w2(d, raw_desc(st, p.a_mn, s), raw_desc(st + p.b_raw_off, p.b_mn, s),
                          id_tf, (kb > cb0 || s > 0) ? 1u : 0u);
              mma_bf16_w2(d, pair_desc(st + p.a_pair_off, p.a_mn, s),
                          pair_desc(st + p.b_pair_off, p.b_mn, s), id_bf);
            }
            commit2_mc(&bars.empty[slot]);  // both CTAs' slot is free
          } else {
#pragma unroll
            for (int s = 0; s < kBK / 8; ++s) {
              mma_tf32_w(d, raw_desc(st, p.a_mn, s), raw_desc(st + p.b_raw_off, p.b_mn, s),
                         id_tf, (kb > cb0 || s > 0) ? 1u : 0u);
              mma_bf16_w(d, pair_desc(st + p.a_pair_off, p.a_mn, s),
                         pair_desc(st + p.b_pair_off, p.b_mn, s), id_bf, 1u);
            }
            if constexpr (MODE == 1)
              mma_commit_mc(&bars.empty[slot], 3);
            else
              mma_commit_w(&bars.empty[slot]);
          }
          if (++slot == p.nstages) {
            slot = 0;
            ph ^= 1u;
          }
        }
        if constexpr (cg2)
          commit2_mc(&bars.tfull[b]);  // both CTAs' epilogues
        else
          mma_commit_w(&bars.tfull[b]);
      }
    }
  } else {
    // ---- epilogue: warp q drains TMEM lanes [32q, 32q + 32) = tile rows.  The
    // tensor core accumulates in fp32 with truncation, so a unit's k range is
    // cut into chunks of chunk_kb k blocks, each in a fresh accumulator; the
    // epilogue adds them in order (round to nearest) through the output itself
    // (chunk 0 stores, later chunks read back, the last applies the epilogue op).
    const int q = warp & 3, ew = warp - kWEpi0;
    int64_t c = 0;
    for (int64_t t = 0; t < my_units; ++t) {
      int ks, mt, nt, kb0, kb1;
      decode(t, ks, mt, nt, kb0, kb1);
      const int64_t row = (int64_t)mt * kBM + q * 32 + lane;
      const bool row_ok = row < p.M;
      const int64_t n0 = (int64_t)nt * BN;
      float* out = p.epi == kPartial ? p.C + (int64_t)ks * p.M * p.N + row * p.N
                                     : p.C + row * p.ldc;
      for (int cb0 = kb0; cb0 < kb1; cb0 += p.chunk_kb, ++c) {
        const bool first = cb0 == kb0, last = cb0 + p.chunk_kb >= kb1;
        const int epi = last ? p.epi : kPartial;  // intermediate chunks: raw sums
        const int b = (int)(c & 1);
        mbar_wait(&bars.tfull[b], (unsigned)(c >> 1) & 1u);
        tc_fence_after();
        const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          float v[32];
          tmem_ld32(tb + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          const int64_t cb = n0 + c0;
          const bool full = p.vec && cb + 32 <= p.N;
          if (!first && row_ok) {  // the previous chunks' sum
            if (full) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 o = *reinterpret_cast<const float4*>(out + cb + j);
                v[j] += o.x;
                v[j + 1] += o.y;
                v[j + 2] += o.z;
                v[j + 3] += o.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (cb + j < p.N) v[j] += out[cb + j];
            }
          }
          if (epi == kBiasTanh) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              v[j] = tanh_fast(v[j] + (cb + j < p.N ? __ldg(p.bias + cb + j) : 0.f));
          } else if (epi == kDtanh) {
            const float* h = p.H + row * p.ldh + cb;
            if (row_ok && p.hvec && cb + 32 <= p.N) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 hv = __ldg(reinterpret_cast<const float4*>(h + j));
                v[j] *= 1.f - hv.x * hv.x;
                v[j + 1] *= 1.f - hv.y * hv.y;
                v[j + 2] *= 1.f - hv.z * hv.z;
                v[j + 3] *= 1.f - hv.w * hv.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float hv = (row_ok && cb + j < p.N) ? __ldg(h + j) : 0.f;
                v[j] = row_ok ? v[j] * (1.f - hv * hv) : 0.f;
              }
            }
          }
          if (row_ok) {
            if (full) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(out + cb + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (cb + j < p.N) out[cb + j] = v[j];
            }
          }
          if (epi == kDtanh) {
            // column sums of this warp's 32 rows: transposed butterfly, lane j ends
            // with column c0 + j (31 shuffles; fixed order)
#pragma unroll
            for (int sft = 16; sft >= 1; sft >>= 1) {
              const bool up = (lane & sft) != 0;
#pragma unroll
              for (int i = 0; i < sft; ++i) {
                const float send = up ? v[i] : v[i + sft];
                const float keep = up ? v[i + sft] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
              }
            }
            s_col[ew][c0 + lane] = v[0];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (cg2)
            arrive_leader(&bars.tempty[b]);  // the leader's MMA reuses the pair's buffer
          else
            mbar_arrive(&bars.tempty[b]);
        }
        if (epi == kDtanh) {  // the tile's column sums, epilogue warps in fixed order
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int e = threadIdx.x - kWEpi0 * 32;
          // (a 2-SM pair's second tile can lie wholly past M: col_part has no row for it)
          const bool tile_ok = (int64_t)mt * kBM < p.M;
          for (int cc = e; cc < BN; cc += 128)
            if (tile_ok && n0 + cc < p.N)
              p.col_part[(int64_t)mt * p.N + n0 + cc] =
                  ((s_col[0][cc] + s_col[1][cc]) + s_col[2][cc]) + s_col[3][cc];
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  if constexpr (MODE != 0)
    cluster_sync_all();  // no multicast or remote arrive still targets this CTA
  else
    __syncthreads();
  if (warp == 1) {
    if constexpr (cg2)
      tmem_dealloc2(tmem, p.tmem_cols);
    else
      tmem_dealloc(tmem, p.tmem_cols);
  }
}

// ---- bf16 pair operands --------------------------------------------------------

__device__ __forceinline__ void split_pair(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  hi = __float2bfloat16_rn(h);
  lo = __float2bfloat16_rn(x - h);
}

// K along the columns: out[r, 16 g + j] = first(x[r, 8 g + j]), out[r, 16 g + 8 + j] = second
__global__ void pairs_col_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                                 __nv_bfloat16* __restrict__ out, int64_t ldo, int lo_first) {
  const int64_t groups = (cols + 7) / 8;
  const int64_t n = rows * groups;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / groups, g = i - r * groups;
    const float* src = X + r * ld + g * 8;
    float x[8];
    if (g * 8 + 8 <= cols && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
      const float4 u = *reinterpret_cast<const float4*>(src);
      const float4 w = *reinterpret_cast<const float4*>(src + 4);
      x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
      x[4] = w.x; x[5] = w.y; x[6] = w.z; x[7] = w.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = g * 8 + j < cols ? src[j] : 0.f;
    }
    __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_pair(x[j], hi[j], lo[j]);
    uint4* dst = reinterpret_cast<uint4*>(out + r * ldo + g * 16);
    dst[0] = *reinterpret_cast<const uint4*>(lo_first ? lo : hi);
    dst[1] = *reinterpret_cast<const uint4*>(lo_first ? hi : lo);
  }
}

// K along the rows: out[16 g + j, c] = first(x[8 g + j, c]), out[16 g + 8 + j, c] = second
__global__ void pairs_row_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                                 __nv_bfloat16* __restrict__ out, int64_t ldo, int lo_first) {
  const int64_t groups = (rows + 7) / 8;
  const int64_t cq = (cols + 3) / 4;  // 4 columns per thread
  const int64_t n = groups * cq;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i / cq, c = (i - g * cq) * 4;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t r = g * 8 + j;
      float x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = (r < rows && c + u < cols) ? X[r * ld + c + u] : 0.f;
      __align__(8) __nv_bfloat16 hi[4], lo[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) split_pair(x[u], hi[u], lo[u]);
      __nv_bfloat16* d0 = out + (g * 16 + j) * ldo + c;
      __nv_bfloat16* d1 = out + (g * 16 + 8 + j) * ldo + c;
      *reinterpret_cast<uint2*>(d0) = *reinterpret_cast<const uint2*>(lo_first ? lo : hi);
      *reinterpret_cast<uint2*>(d1) = *reinterpret_cast<const uint2*>(lo_first ? hi : lo);
    }
  }
}

// ---- host ------------------------------------------------------------------------

int launch_wide(const float* A, const void* Ap, const float* B, const void* Bp, float* C,
                const float* bias, const float* H, float* col_part, int64_t M, int64_t N, int64_t K,
                int64_t lda, int64_t ldap, int64_t ldb, int64_t ldbp, int64_t ldc, int64_t ldh,
                int a_mn, int b_mn, int epi, int kslices, cudaStream_t st) {
  WideArgs p{};
  p.BN = (int)std::min<int64_t>(256, (N + 31) / 32 * 32);
  if (b_mn) p.BN = (p.BN + 63) / 64 * 64;  // MN-major pair tiles come in 64-column atoms
  p.C = C; p.bias = bias; p.H = H; p.col_part = col_part;
  p.M = M; p.N = N; p.ldc = ldc; p.ldh = ldh;
  p.m_tiles = (int)ceil_div(M, kBM);
  p.n_tiles = (int)ceil_div(N, p.BN);
  p.kblocks = (int)ceil_div(K, kBK);
  p.kslices = kslices;
  p.a_mn = a_mn; p.b_mn = b_mn; p.epi = epi;
  const bool c_al = (reinterpret_cast<uintptr_t>(C) & 15) == 0;
  p.vec = (c_al && (epi == kPartial ? N % 4 == 0 : ldc % 4 == 0)) ? 1 : 0;
  p.hvec = (H && (reinterpret_cast<uintptr_t>(H) & 15) == 0 && ldh % 4 == 0) ? 1 : 0;
  // stage layout: [A raw | A pair | B raw | B pair], each region 1 KB aligned
  auto al = [](uint32_t x) { return (x + 1023u) / 1024u * 1024u; };
  // mode: 2 = 2-SM UMMA pairs (each CTA holds half the B tile), 1 = B multicast, 0 = single
  const int m_tiles = (int)ceil_div(M, kBM);
  p.mc = (g_wide_multicast && p.BN == 256 && m_tiles >= 2 && sm_count() >= 2) ? g_wide_multicast
                                                                                : 0;
  const uint32_t a_bytes = kBM * kBK * 4;  // raw == pair bytes
  const uint32_t b_bytes = (uint32_t)(p.mc == 2 ? p.BN / 2 : p.BN) * kBK * 4;
  p.a_pair_off = al(a_bytes);
  p.b_raw_off = p.a_pair_off + al(a_bytes);
  p.b_pair_off = p.b_raw_off + al(b_bytes);
  p.stage_bytes = p.b_pair_off + al(b_bytes);
  p.tx_bytes = (p.mc == 2 ? 4 : 2) * (a_bytes + b_bytes);  // cg2: both CTAs' loads
  p.nstages = (int)std::min<size_t>(kMaxStages, kWideSmem / p.stage_bytes);
  if (p.nstages < 2) return fail(kDimension, "tc_wide: stage too large");
  p.tmem_cols = tmem_cols_for(2 * p.BN);
  // tensor maps: K-major operands as [rows = M|N, cols = K] with 64 B-swizzled
  // boxes; MN-major ones as [rows = K, cols = M|N] in 128 B-swizzled slabs / atoms
  const int64_t K8 = (K + 7) / 8 * 8;
  CUtensorMap am, apm, bm, bpm;
  auto mk = [&](CUtensorMap* raw, CUtensorMap* pair, const float* X, const void* Xp, int64_t mnrows,
                int64_t ld, int64_t ldp, int mn, int tile_rows, int three_d) -> int {
    if (mn && three_d) {  // {32 | 64 columns, k rows, slabs | atoms}: one box per stage
      EncodeFn fn = encode_fn();
      if (!fn) return fail(kCuda, "tc_wide: cuTensorMapEncodeTiled unavailable");
      if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(Xp) & 15) ||
          (ld % 4) || (ldp % 8))
        return fail(kDimension, "tc_wide: MN-major operands need 16-byte aligned rows");
      const cuuint32_t estr[3] = {1, 1, 1};
      const cuuint64_t rd[3] = {32, (cuuint64_t)K, (cuuint64_t)(mnrows / 32)};
      const cuuint64_t rs[2] = {(cuuint64_t)ld * 4, 128};
      const cuuint32_t rb[3] = {32, (cuuint32_t)kBK, (cuuint32_t)(tile_rows / 32)};
      CUresult r = fn(raw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(X), rd, rs, rb,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(kCuda, "tc_wide: 3-D map encode failed (%d)", (int)r);
      const cuuint64_t pd[3] = {64, (cuuint64_t)(2 * K8), (cuuint64_t)(mnrows / 64)};
      const cuuint64_t ps[2] = {(cuuint64_t)ldp * 2, 128};
      const cuuint32_t pb[3] = {64, (cuuint32_t)(2 * kBK), (cuuint32_t)(tile_rows / 64)};
      r = fn(pair, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(Xp), pd, ps, pb, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(kCuda, "tc_wide: 3-D pair map encode failed (%d)", (int)r);
      return kOk;
    }
    if (mn) {
      if (int e = make_map_dt(raw, X, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, K, mnrows, ld, 32, kBK,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
        return e;
      return make_map_dt(pair, Xp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2 * K8, mnrows, ldp, 64,
                         2 * kBK, CU_TENSOR_MAP_SWIZZLE_128B);
    }
    if (int e = make_map_dt(raw, X, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, mnrows, K, ld, kBK, tile_rows,
                            CU_TENSOR_MAP_SWIZZLE_64B))
      return e;
    return make_map_dt(pair, Xp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mnrows, 2 * K8, ldp, 2 * kBK,
                       tile_rows, CU_TENSOR_MAP_SWIZZLE_64B);
  };
  // 3-D boxes need whole slabs / atoms inside the matrix: MN % 64 == 0 and, for
  // A, a full 128-row tile span (the box covers the tile's whole MN extent)
  p.a_3d = (a_mn && M % 64 == 0 && M % kBM == 0) ? 1 : 0;
  p.b_3d = (b_mn && N % 64 == 0 && N % p.BN == 0) ? 1 : 0;
  p.chunk_kb = g_chunk_kb > 0 ? g_chunk_kb : (1 << 30);
  // 2-CTA clusters share each 256-wide B tile: each CTA loads half of it and
  // multicasts it to both (1/3 less L2 -> SM traffic per stage); used when the
  // halves are whole 64-column atoms and there are m tiles to pair
  if (int e = mk(&am, &apm, A, Ap, M, lda, ldap, a_mn, kBM, p.a_3d)) return e;
  if (int e = mk(&bm, &bpm, B, Bp, N, ldb, ldbp, b_mn, p.mc ? p.BN / 2 : p.BN, p.b_3d)) return e;
  const size_t smem = (size_t)p.nstages * p.stage_bytes;
  auto kern = p.mc == 2 ? tc_wide_kernel<2> : p.mc == 1 ? tc_wide_kernel<1> : tc_wide_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return fail(kCuda, "tc_wide smem: %s", cudaGetErrorString(e));
  if (!p.mc) {
    const int64_t units = (int64_t)p.m_tiles * p.n_tiles * p.kslices;
    const int grid = (int)std::min<int64_t>(units, sm_count());
    kern<<<grid, kWThreads, smem, st>>>(am, apm, bm, bpm, p);
    return post_launch("tc_wide_kernel");
  }
  const int64_t pairs = ceil_div(p.m_tiles, 2) * p.n_tiles * p.kslices;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(pairs, sm_count() / 2)));
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, am, apm, bm, bpm, p);
  if (e != cudaSuccess) return fail(kCuda, "tc_wide cluster launch: %s", cudaGetErrorString(e));
  return post_launch(p.mc == 2 ? "tc_wide_kernel<2> (2-SM UMMA)" : "tc_wide_kernel<1> (multicast)");
}

}  // namespace
}  // namespace accel

using namespace accel;

// C = A . B^T over fp32 operands with fp32-class accuracy (see the file comment).
//   a_mn = 0: A is [M, K] (row pitch lda), else [K, M];  b_mn = 0: B is [N, K], else [K, N].
//   Ap / Bp: the operands' bf16 pair arrays (accel_tf32_pairs: A with lo_first = 0,
//   B with lo_first = 1; column pairs for K-major, row pairs for MN-major), pitch in
//   elements.  epi: 0 store C[M, N] (ldc); 1 tanh(acc + bias); 2 acc (1 - H^2) with
//   col_part[ceil(M / 128)][N] = per-128-row-tile column sums of C; 3 split-K:
//   C = [kslices][M][N] partial slices (the caller sums them in order).
extern "C" int accel_tc_gemm_wide(const float* A, const void* Ap, const float* B, const void* Bp,
                                  float* C, const float* bias, const float* H, float* col_part,
                                  int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldap,
                                  int64_t ldb, int64_t ldbp, int64_t ldc, int64_t ldh, int a_mn,
                                  int b_mn, int epi, int kslices, void* stream) {
  if (M < 0 || N < 1 || K < 1 || kslices < 1 || epi < 0 || epi > 3)
    return fail(kDimension, "tc_gemm_wide: bad sizes M=%lld N=%lld K=%lld", (long long)M,
                (long long)N, (long long)K);
  if (M == 0) return kOk;
  if (!A || !Ap || !B || !Bp || !C) return fail(kDimension, "tc_gemm_wide: NULL operand");
  if (epi == kBiasTanh && !bias) return fail(kDimension, "tc_gemm_wide: bias+tanh needs bias");
  if (epi == kDtanh && (!H || !col_part)) return fail(kDimension, "tc_gemm_wide: dtanh needs H, col_part");
  if (epi != kPartial && kslices != 1) return fail(kDimension, "tc_gemm_wide: split-K needs epi 3");
  if (kslices > ceil_div(K, kBK))  // every slice owns >= one 16-k block (else its slice is unwritten)
    return fail(kDimension, "tc_gemm_wide: kslices %d > ceil(K / 16) = %lld", kslices,
                (long long)ceil_div(K, kBK));
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return fail(kDimension, "tc_gemm_wide: too large");
  return launch_wide(A, Ap, B, Bp, C, bias, H, col_part, M, N, K, lda, ldap, ldb, ldbp, ldc, ldh,
                     a_mn, b_mn, epi, kslices, as_stream(stream));
}

// Tuning knob: k blocks (16 k each) per fp32 accumulation chunk (>= 1).
extern "C" void accel_tc_wide_set_chunk(int kblocks) { g_chunk_kb = kblocks < 0 ? 0 : kblocks; }

// Tuning knob: 2 (default) = 2-SM UMMA pairs (cta_group::2), 1 = 1-SM MMAs with the
// shared B tile multicast, 0 = one CTA per tile.
extern "C" void accel_tc_wide_set_multicast(int mode) {
  g_wide_multicast = mode < 0 ? 0 : (mode > 2 ? 2 : mode);
}

extern "C" int accel_tc_wide_tiles(int64_t M, int64_t N, int b_mn) {
  int bn = (int)std::min<int64_t>(256, (N + 31) / 32 * 32);
  if (b_mn) bn = (bn + 63) / 64 * 64;
  return (int)(ceil_div(M, kBM) * ceil_div(N, bn));
}

// bf16 pair operand of an fp32 matrix X [rows, cols] (pitch ld): per 8-element group
// along K, [bf16(hi) x8 | bf16(lo) x8] (lo_first: [lo | hi]), hi = trunc19(x), lo = x - hi.
// row_pair = 0 (K = cols): out [rows, 2 * ceil8(cols)], pitch ldo >= 2 * ceil8(cols);
// row_pair = 1 (K = rows): out [2 * ceil8(rows), cols], pitch ldo >= cols (ldo % 8 == 0).
extern "C" int accel_tf32_pairs(const float* X, int64_t rows, int64_t cols, int64_t ld, void* out,
                                int64_t ldo, int row_pair, int lo_first, void* stream) {
  if (rows < 0 || cols < 1 || ld < cols) return fail(kDimension, "tf32_pairs: bad sizes");
  if (rows == 0) return kOk;
  if (!X || !out) return fail(kDimension, "tf32_pairs: NULL buffer");
  if ((reinterpret_cast<uintptr_t>(out) & 15) || ldo % 8)
    return fail(kDimension, "tf32_pairs: output needs 16-byte aligned rows");
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  cudaStream_t st = as_stream(stream);
  const int threads = 256;
  if (row_pair) {
    if (ldo < cols) return fail(kDimension, "tf32_pairs: ldo < cols");
    const int64_t n = (rows + 7) / 8 * ((cols + 3) / 4);
    const int grid = (int)std::min<int64_t>(ceil_div(n, threads), 148 * 16);
    pairs_row_kernel<<<grid, threads, 0, st>>>(X, rows, cols, ld, o, ldo, lo_first);
  } else {
    if (ldo < 2 * ((cols + 7) / 8 * 8)) return fail(kDimension, "tf32_pairs: ldo too small");
    const int64_t n = rows * ((cols + 7) / 8);
    const int grid = (int)std::min<int64_t>(ceil_div(n, threads), 148 * 16);
    pairs_col_kernel<<<grid, threads, 0, st>>>(X, rows, cols, ld, o, ldo, lo_first);
  }
  return post_launch("tf32_pairs");
}
