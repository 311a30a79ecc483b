// Deterministic grouped row sums (the reference's np.add.at scatter-adds).
//
// Reference: `np.add.at(de_prev, prev.ravel(), dc)` (models.py:195) and
// `np.add.at(de_step, t, du)` (models.py:305).  Float atomics would make the
// result depend on scheduling; instead the keys of a batch (previous-token
// ids x chunk positions, step ids — fixed per TrainBatch) are counting-sorted
// once, stably, at batch build time, and every later grouped sum is a
// segmented reduction in that fixed order:
//   1. chunk histograms (one warp per 16K-row chunk, smem int atomics),
//   2. exclusive scan of the key-major [key][chunk] counts (CUB DeviceScan),
//   3. stable scatter: each warp walks its chunk 32 rows at a time, ranking
//      equal keys with __match_any_sync,
//   4. grouped sums: each key segment is cut into <=256-row pieces; one CTA
//      sums a piece (gathered rows, coalesced within a row) in fixed order, a
//      second pass sums the pieces of each key in order.
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace accel {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 4096;   // rows per block unit (the caller's cpb counts these)
// rows per warp chunk of the histogram / scatter: 4096, or fewer for small R so
// that enough warps take part (a chunk is walked serially by one warp)
inline int chunk_rows(int64_t R) {
  int c = kChunk;
  while (c > 256 && ceil_div(R, (int64_t)c) < (int64_t)kNumSMs * 8) c >>= 1;
  return c;
}
constexpr int kPiece = 256;    // rows per grouped-sum piece

// key = prev (with_pos == 0) or prev * K + k (with_pos == 1); prev = A at k == 0
__global__ void prev_keys_kernel(const int32_t* __restrict__ tokens, int64_t M, int K, int A,
                                 int with_pos, int32_t* __restrict__ keys) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < M; r += stride) {
    const int k = (int)(r % K);
    int prev = k == 0 ? A : __ldg(tokens + r - 1);
    prev = min(max(prev, 0), A);
    keys[r] = with_pos ? prev * K + k : prev;
  }
}

__global__ void step_keys_kernel(const int32_t* __restrict__ steps,
                                 const int32_t* __restrict__ frame_of, int64_t R, int n_steps,
                                 int32_t* __restrict__ keys, unsigned* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned nbad = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    const int64_t f = frame_of ? __ldg(frame_of + r) : r;
    const int s = __ldg(steps + f);
    nbad += (s < 0 || s >= n_steps);
    keys[r] = min(max(s, 0), n_steps - 1);
  }
  if (nbad) atomicAdd(bad, nbad);  // integer count: order-independent
}

// counts[((chunk / cpb) * nkeys + key) * cpb + chunk % cpb]: the row range is cut
// into blocks of cpb chunks and the scan order is block-major, key-minor, chunk
// last (cpb = n_chunks: plain key-major order).  Composite key = block * nkeys + key.
// optional sorted per-row metadata written by the scatter (pos == nullptr: off)
struct SortedRows {
  const int32_t* frame_of;
  const int32_t* tokens;
  int K;
  int32_t* row_frame;
  int32_t* row_tok;
  int32_t* pos;
};

__device__ __forceinline__ int64_t count_idx(int64_t chunk, int key, int nkeys, int64_t cpb) {
  return ((chunk / cpb) * nkeys + key) * cpb + chunk % cpb;
}

__global__ void __launch_bounds__(kThreads)
chunk_hist_kernel(const int32_t* __restrict__ keys, int64_t R, int nkeys, int64_t n_chunks,
                  int64_t cpb, int crows, int* __restrict__ counts) {
  extern __shared__ int s_hist[];  // [kWarps][nkeys]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* h = s_hist + warp * nkeys;
  for (int j = lane; j < nkeys; j += 32) h[j] = 0;
  __syncwarp();
  const int64_t chunk = (int64_t)blockIdx.x * kWarps + warp;
  if (chunk < n_chunks) {
    const int64_t r0 = chunk * crows, r1 = min(R, r0 + crows);
    for (int64_t r = r0 + lane; r < r1; r += 32 * 8) {  // eight key loads in flight per lane
      int kk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kk[u] = r + 32 * u < r1 ? __ldg(keys + r + 32 * u) : -1;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (kk[u] >= 0) atomicAdd(h + kk[u], 1);
    }
    __syncwarp();
    for (int j = lane; j < nkeys; j += 32) counts[count_idx(chunk, j, nkeys, cpb)] = h[j];
  }
}

// seg_off / piece_off from the scanned counts: one 1024-thread block, each
// thread owns a contiguous run of keys; a fixed-order scan of the per-thread
// piece totals gives the piece offsets.
__global__ void __launch_bounds__(1024)
segment_offsets_kernel(const int* __restrict__ base, int nkeys, int64_t n_chunks, int64_t R,
                       int64_t* __restrict__ seg_off, int64_t* __restrict__ piece_off) {
  // (composite keys: nkeys = blocks * keys, n_chunks = chunks per block)
  __shared__ int64_t s_warp[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (nkeys + blockDim.x - 1) / blockDim.x;
  const int j0 = min(nkeys, t * per), j1 = min(nkeys, j0 + per);
  int64_t mine = 0;
  for (int j = j0; j < j1; ++j) {
    const int64_t a = base[(int64_t)j * n_chunks];
    const int64_t b = j + 1 < nkeys ? (int64_t)base[(int64_t)(j + 1) * n_chunks] : R;
    seg_off[j] = a;
    mine += ceil_div(b - a, (int64_t)kPiece);
  }
  // exclusive block scan of the per-thread piece totals (integers: exact in any
  // order): warp scans, then a scan of the 32 warp totals
  int64_t x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  if (t == 0) {
    seg_off[nkeys] = R;
    piece_off[nkeys] = s_warp[(blockDim.x >> 5) - 1];
  }
  int64_t p = (x - mine) + (warp > 0 ? s_warp[warp - 1] : 0);
  for (int j = j0; j < j1; ++j) {
    piece_off[j] = p;
    const int64_t a = seg_off[j];
    const int64_t b = j + 1 < nkeys ? (int64_t)base[(int64_t)(j + 1) * n_chunks] : R;
    p += ceil_div(b - a, (int64_t)kPiece);
  }
}

__global__ void __launch_bounds__(kThreads)
stable_scatter_kernel(const int32_t* __restrict__ keys, int64_t R, int nkeys, int64_t n_chunks,
                      int64_t cpb, int crows, const int* __restrict__ base,
                      int32_t* __restrict__ perm, SortedRows sr) {
  extern __shared__ int s_ctr[];  // [kWarps][nkeys]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunk = (int64_t)blockIdx.x * kWarps + warp;
  if (chunk >= n_chunks) return;
  int* ctr = s_ctr + warp * nkeys;
  for (int j0 = lane; j0 < nkeys; j0 += 32 * 8) {  // eight strided loads in flight per lane
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + 32 * u;
      v[u] = j < nkeys ? __ldg(base + count_idx(chunk, j, nkeys, cpb)) : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + 32 * u < nkeys) ctr[j0 + 32 * u] = v[u];
  }
  __syncwarp();
  const int64_t r0 = chunk * crows, r1 = min(R, r0 + crows);
  const unsigned lt = (1u << lane) - 1u;
  const int kbits = nkeys > 1 ? 32 - __clz(nkeys - 1) : 1;  // bits of the largest key
  for (int64_t g0 = r0; g0 < r1; g0 += 32 * 8) {
    int kk[8];  // the keys of eight 32-row groups, loaded together (latency once per 256 rows)
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = g0 + 32 * u + lane;
      kk[u] = r < r1 ? __ldg(keys + r) : -1 - lane;  // dead lanes never match
    }
    // peer masks (lanes holding the same key) from one ballot per key bit:
    // cheaper than MATCH.ANY, whose cost grows with the number of distinct
    // keys in the group (here nearly all 32 differ)
    unsigned pm[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int key = kk[u];
      const bool live = key >= 0;
      unsigned m = __ballot_sync(0xffffffffu, live);
      m = live ? m : ~m;
      for (int b = 0; b < kbits; ++b) {
        const bool bit = (key >> b) & 1;
        const unsigned bb = __ballot_sync(0xffffffffu, bit);
        m &= bit ? bb : ~bb;
      }
      pm[u] = live ? m : (1u << lane);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t g = g0 + 32 * u;
      if (g >= r1) break;  // warp-uniform
      const int64_t r = g + lane;
      const bool live = r < r1;
      const int key = kk[u];
      const unsigned peers = pm[u];
      if (live) {
        const int rank = __popc(peers & lt);
        const int32_t dst = ctr[key] + rank;
        perm[dst] = (int32_t)r;
        if (sr.pos != nullptr) sr.pos[r] = dst;  // inverse permutation (coalesced writes)
        if (sr.row_frame != nullptr) {           // sorted per-row metadata (scattered writes)
          sr.row_frame[dst] = __ldg(sr.frame_of + r / sr.K);
          sr.row_tok[dst] = __ldg(sr.tokens + r);
        }
      }
      __syncwarp();
      if (live && (peers & lt) == 0) ctr[key] += __popc(peers);
      __syncwarp();
    }
  }
}

// piece sums: one CTA per piece, rows gathered through perm.
__global__ void __launch_bounds__(kThreads)
piece_sum_kernel(const float* __restrict__ vals, const int32_t* __restrict__ perm,
                 const int64_t* __restrict__ seg_off, const int64_t* __restrict__ piece_off,
                 const int32_t* __restrict__ piece_key, int nkeys, int D,
                 float* __restrict__ piece_out) {
  extern __shared__ float s_acc[];
  const int64_t piece = blockIdx.x;
  if (piece >= piece_off[nkeys]) return;  // grid is sized for the worst case
  int key;
  if (piece_key != nullptr) {  // one load instead of a dependent binary search
    key = __ldg(piece_key + piece);
  } else {  // last j with piece_off[j] <= piece
    int lo = 0, hi = nkeys;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (piece_off[mid] <= piece) lo = mid; else hi = mid;
    }
    key = lo;
  }
  const int64_t r0 = seg_off[key] + (piece - piece_off[key]) * kPiece;
  const int64_t r1 = min(seg_off[key + 1], r0 + kPiece);
  if ((D & 3) == 0) {
    // float4 columns: a row is D/4 lanes wide; the piece's row ids are staged in
    // shared memory first so four independent row loads per lane stay in flight
    __shared__ int s_rows[kPiece];
    const int nr = (int)(r1 - r0);
    for (int r = threadIdx.x; r < nr; r += kThreads) s_rows[r] = __ldg(perm + r0 + r);
    __syncthreads();
    const int D4 = D >> 2;
    const int span = (D4 <= kThreads && kThreads % D4 == 0) ? D4 : kThreads;
    const int sub = kThreads / span;
    const int lr = threadIdx.x / span, lc = threadIdx.x % span;
    float4* s4 = reinterpret_cast<float4*>(s_acc);
    const float4* v4 = reinterpret_cast<const float4*>(vals);
    for (int d0 = 0; d0 < D4; d0 += span) {
      const int d = d0 + lc;
      float4 acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (d < D4) {
        int r = lr;
        for (; r + 3 * sub < nr; r += 4 * sub) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 x = __ldg(v4 + (int64_t)s_rows[r + u * sub] * D4 + d);
            acc[u].x += x.x; acc[u].y += x.y; acc[u].z += x.z; acc[u].w += x.w;
          }
        }
        for (; r < nr; r += sub) {
          const float4 x = __ldg(v4 + (int64_t)s_rows[r] * D4 + d);
          acc[0].x += x.x; acc[0].y += x.y; acc[0].z += x.z; acc[0].w += x.w;
        }
      }
      float4 t = acc[0];
#pragma unroll
      for (int u = 1; u < 4; ++u) { t.x += acc[u].x; t.y += acc[u].y; t.z += acc[u].z; t.w += acc[u].w; }
      s4[threadIdx.x] = t;
      __syncthreads();
      if (threadIdx.x < span && d0 + threadIdx.x < D4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s2 = 0; s2 < sub; ++s2) {
          const float4 y = s4[s2 * span + threadIdx.x];
          a.x += y.x; a.y += y.y; a.z += y.z; a.w += y.w;
        }
        reinterpret_cast<float4*>(piece_out + piece * D)[d0 + threadIdx.x] = a;
      }
      __syncthreads();
    }
    return;
  }
  const int span = (D <= kThreads && kThreads % D == 0) ? D : kThreads;
  const int sub = kThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  for (int d0 = 0; d0 < D; d0 += span) {
    const int d = d0 + lc;
    float acc = 0.f;
    if (d < D)
      for (int64_t r = r0 + lr; r < r1; r += sub)
        acc += __ldg(vals + (int64_t)__ldg(perm + r) * D + d);
    s_acc[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D) {
      float a = 0.f;
      for (int s = 0; s < sub; ++s) a += s_acc[s * span + threadIdx.x];
      piece_out[piece * D + d0 + threadIdx.x] = a;
    }
    __syncthreads();
  }
}

// One CTA per key: `sub` row-lanes split the key's pieces round-robin (fixed
// order), then the row-lanes are combined in order.  A key with thousands of
// pieces (the chunk-start token holds one row per transition) is summed by a
// whole CTA instead of one serial thread per column.
__global__ void __launch_bounds__(kThreads)
key_sum_kernel(const float* __restrict__ piece_out, const int64_t* __restrict__ piece_off,
               int nkeys, int D, float* __restrict__ out) {
  extern __shared__ float s_acc[];
  const int key = blockIdx.x;
  const int64_t p0 = piece_off[key], p1 = piece_off[key + 1];
  const int span = (D <= kThreads && kThreads % D == 0) ? D : kThreads;
  const int sub = kThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  for (int d0 = 0; d0 < D; d0 += span) {
    const int d = d0 + lc;
    float acc = 0.f;
    if (d < D)
      for (int64_t p = p0 + lr; p < p1; p += sub) acc += piece_out[p * D + d];
    s_acc[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D) {
      float a = 0.f;
      for (int s = 0; s < sub; ++s) a += s_acc[s * span + threadIdx.x];
      out[(int64_t)key * D + d0 + threadIdx.x] = a;
    }
    __syncthreads();
  }
}

// float4 columns, 1024 threads: `sub` = 1024 / (D / 4) row-lanes, each with 4
// independent partial sums (fixed assignment, fixed combine order).  The
// chunk-start key holds one row per transition (thousands of pieces): this
// keeps ~64 loads in flight per column group instead of a serial chain.
constexpr int kKeyThreads = 1024;
__global__ void __launch_bounds__(kKeyThreads)
key_sum4_kernel(const float4* __restrict__ piece_out, const int64_t* __restrict__ piece_off,
                int nkeys, int D4, float4* __restrict__ out) {
  extern __shared__ float4 s4[];
  const int key = blockIdx.x;
  const int64_t p0 = piece_off[key], p1 = piece_off[key + 1];
  const int span = D4 <= kKeyThreads && kKeyThreads % D4 == 0 ? D4 : kKeyThreads;
  const int sub = kKeyThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  for (int d0 = 0; d0 < D4; d0 += span) {
    const int d = d0 + lc;
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d < D4) {
      int64_t p = p0 + lr;
      for (; p + 3 * sub < p1; p += 4 * sub) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 x = __ldg(piece_out + (p + u * sub) * D4 + d);
          a[u].x += x.x; a[u].y += x.y; a[u].z += x.z; a[u].w += x.w;
        }
      }
      for (int u = 0; p < p1; p += sub, ++u) {
        const float4 x = __ldg(piece_out + p * D4 + d);
        a[u & 3].x += x.x; a[u & 3].y += x.y; a[u & 3].z += x.z; a[u & 3].w += x.w;
      }
    }
    float4 t = a[0];
    for (int u = 1; u < 4; ++u) { t.x += a[u].x; t.y += a[u].y; t.z += a[u].z; t.w += a[u].w; }
    s4[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D4) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s2 = 0; s2 < sub; ++s2) {
        const float4 y = s4[s2 * span + threadIdx.x];
        r.x += y.x; r.y += y.y; r.z += y.z; r.w += y.w;
      }
      out[(int64_t)key * D4 + d0 + threadIdx.x] = r;
    }
    __syncthreads();
  }
}

// Blocked grouping: Dk[key] = sum over blocks b (in order) of the pieces of the
// composite key b * nkeys + key (in order).  Grid (key, split): CTA (key, q)
// folds the contiguous block range q of the key into part[q][key] (64 float4
// columns x 4 block-lanes, four loads in flight, lanes combined in order);
// fold_parts_kernel then sums the kFoldSplit parts in order.  One key may be
// heavy (the factorized head's chunk-start key holds every transition's token 0:
// a piece per 256 of them in every block); it is skipped here and folded by
// fold_heavy_parts_kernel over ~kHeavySplit CTAs instead.
constexpr int kFoldThreads = 256;
constexpr int kFoldSplit = 2;
constexpr int kHeavySplit = 64;
constexpr int kHeavyMaxParts = 2 * kHeavySplit;
__global__ void __launch_bounds__(kFoldThreads)
fold_blocked_pieces_kernel(const float4* __restrict__ piece_out,
                           const int64_t* __restrict__ piece_off, int nkeys, int nblocks, int D4,
                           int heavy_key, float4* __restrict__ part) {
  __shared__ float4 s4[kFoldThreads];
  const int key = blockIdx.x, q = blockIdx.y, split = gridDim.y;
  if (key == heavy_key) return;
  const int b0 = (int)((int64_t)nblocks * q / split);
  const int b1 = (int)((int64_t)nblocks * (q + 1) / split);
  const int span = D4 <= kFoldThreads && kFoldThreads % D4 == 0 ? D4 : kFoldThreads;
  const int sub = kFoldThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  for (int d0 = 0; d0 < D4; d0 += span) {
    const int d = d0 + lc;
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d < D4) {
      for (int b = b0 + lr; b < b1; b += sub) {
        const int64_t ck = (int64_t)b * nkeys + key;
        const int64_t p0 = __ldg(piece_off + ck), p1 = __ldg(piece_off + ck + 1);
        int64_t p = p0;
        for (; p + 3 < p1; p += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 x = __ldg(piece_out + (p + u) * D4 + d);
            a[u].x += x.x; a[u].y += x.y; a[u].z += x.z; a[u].w += x.w;
          }
        }
        for (int u = 0; p < p1; ++p, ++u) {
          const float4 x = __ldg(piece_out + p * D4 + d);
          a[u].x += x.x; a[u].y += x.y; a[u].z += x.z; a[u].w += x.w;
        }
      }
    }
    s4[threadIdx.x] = make_float4(((a[0].x + a[1].x) + a[2].x) + a[3].x,
                                  ((a[0].y + a[1].y) + a[2].y) + a[3].y,
                                  ((a[0].z + a[1].z) + a[2].z) + a[3].z,
                                  ((a[0].w + a[1].w) + a[2].w) + a[3].w);
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D4) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s2 = 0; s2 < sub; ++s2) {
        const float4 y = s4[s2 * span + threadIdx.x];
        r.x += y.x; r.y += y.y; r.z += y.z; r.w += y.w;
      }
      part[((int64_t)q * nkeys + key) * D4 + d0 + threadIdx.x] = r;
    }
    __syncthreads();
  }
}

// The heavy key: nq CTAs; with nblocks >= kHeavySplit CTA q takes a contiguous
// block range, else (r = ceil(kHeavySplit / nblocks) CTAs per block) sub-range
// q % r of block q / r's pieces.  The 4 lane-rows take every 4th piece of the
// range (four loads in flight each); lanes combined in order into hpart[q].
__global__ void __launch_bounds__(kFoldThreads)
fold_heavy_parts_kernel(const float4* __restrict__ piece_out, const int64_t* __restrict__ piece_off,
                        int nkeys, int nblocks, int D4, int key, int r, float4* __restrict__ hpart) {
  __shared__ float4 s4[kFoldThreads];
  const int q = blockIdx.x, nq = gridDim.x;
  const int b0 = r == 1 ? (int)((int64_t)nblocks * q / nq) : q / r;
  const int b1 = r == 1 ? (int)((int64_t)nblocks * (q + 1) / nq) : b0 + 1;
  const int j = q % r;
  const int span = D4 <= kFoldThreads && kFoldThreads % D4 == 0 ? D4 : kFoldThreads;
  const int sub = kFoldThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  for (int d0 = 0; d0 < D4; d0 += span) {
    const int d = d0 + lc;
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d < D4) {
      for (int b = b0; b < b1; ++b) {
        const int64_t ck = (int64_t)b * nkeys + key;
        const int64_t p0 = __ldg(piece_off + ck), p1 = __ldg(piece_off + ck + 1), n = p1 - p0;
        const int64_t pa = p0 + n * j / r, pb = p0 + n * (j + 1) / r;
        int64_t p = pa + lr;
        for (; p + 3 * sub < pb; p += 4 * sub) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 x = __ldg(piece_out + (p + u * sub) * D4 + d);
            a[u].x += x.x; a[u].y += x.y; a[u].z += x.z; a[u].w += x.w;
          }
        }
        for (int u = 0; p < pb; p += sub, ++u) {
          const float4 x = __ldg(piece_out + p * D4 + d);
          a[u].x += x.x; a[u].y += x.y; a[u].z += x.z; a[u].w += x.w;
        }
      }
    }
    s4[threadIdx.x] = make_float4(((a[0].x + a[1].x) + a[2].x) + a[3].x,
                                  ((a[0].y + a[1].y) + a[2].y) + a[3].y,
                                  ((a[0].z + a[1].z) + a[2].z) + a[3].z,
                                  ((a[0].w + a[1].w) + a[2].w) + a[3].w);
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D4) {
      float4 rr = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s2 = 0; s2 < sub; ++s2) {
        const float4 y = s4[s2 * span + threadIdx.x];
        rr.x += y.x; rr.y += y.y; rr.z += y.z; rr.w += y.w;
      }
      hpart[(int64_t)q * D4 + d0 + threadIdx.x] = rr;
    }
    __syncthreads();
  }
}

// out[key] = the heavy key's nq parts: column group i's parts in 4 strided
// accumulators per lane-row, lane-rows and accumulators combined in a fixed order
__global__ void __launch_bounds__(kFoldThreads)
fold_heavy_kernel(const float4* __restrict__ hpart, int nq, int D4, int key,
                  float4* __restrict__ out) {
  __shared__ float4 s4[kFoldThreads];
  const int span = D4 <= kFoldThreads && kFoldThreads % D4 == 0 ? D4 : kFoldThreads;
  const int sub = kFoldThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  for (int d0 = 0; d0 < D4; d0 += span) {
    const int d = d0 + lc;
    float4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d < D4) {
      int q = lr;
      for (; q + 3 * sub < nq; q += 4 * sub) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 y = hpart[(int64_t)(q + u * sub) * D4 + d];
          a[u].x += y.x; a[u].y += y.y; a[u].z += y.z; a[u].w += y.w;
        }
      }
      for (int u = 0; q < nq; q += sub, ++u) {
        const float4 y = hpart[(int64_t)q * D4 + d];
        a[u].x += y.x; a[u].y += y.y; a[u].z += y.z; a[u].w += y.w;
      }
    }
    s4[threadIdx.x] = make_float4(((a[0].x + a[1].x) + a[2].x) + a[3].x,
                                  ((a[0].y + a[1].y) + a[2].y) + a[3].y,
                                  ((a[0].z + a[1].z) + a[2].z) + a[3].z,
                                  ((a[0].w + a[1].w) + a[2].w) + a[3].w);
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D4) {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s2 = 0; s2 < sub; ++s2) {
        const float4 y = s4[s2 * span + threadIdx.x];
        r.x += y.x; r.y += y.y; r.z += y.z; r.w += y.w;
      }
      out[(int64_t)key * D4 + d0 + threadIdx.x] = r;
    }
    __syncthreads();
  }
}

// (skip: [skip_lo, skip_hi) float4s -- the heavy key's row, folded separately)
__global__ void fold_parts_kernel(const float4* __restrict__ part, int64_t n4, int64_t stride4,
                                  int split, float4* __restrict__ out, int64_t skip_lo = 0,
                                  int64_t skip_hi = 0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4 || (i >= skip_lo && i < skip_hi)) return;
  float4 r = part[i];
  for (int q = 1; q < split; ++q) {
    const float4 y = part[q * stride4 + i];
    r.x += y.x; r.y += y.y; r.z += y.z; r.w += y.w;
  }
  out[i] = r;
}

// piece_key[p] = the composite key owning piece p
__global__ void piece_keys_kernel(const int64_t* __restrict__ piece_off, int64_t nk,
                                  int32_t* __restrict__ piece_key) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nk) return;
  for (int64_t p = piece_off[j]; p < piece_off[j + 1]; ++p) piece_key[p] = (int32_t)j;
}

// Parallel segment offsets (many composite keys): seg_off[j] = base[j * cpb],
// pcount[j] = pieces of key j; piece_off = exclusive scan of pcount (CUB).
__global__ void seg_counts_kernel(const int* __restrict__ base, int64_t nk, int64_t cpb, int64_t R,
                                  int64_t* __restrict__ seg_off, int64_t* __restrict__ pcount) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nk) return;
  if (j == nk) {
    seg_off[nk] = R;
    pcount[nk] = 0;
    return;
  }
  const int64_t a = base[j * cpb];
  const int64_t b = j + 1 < nk ? (int64_t)base[(j + 1) * cpb] : R;
  seg_off[j] = a;
  pcount[j] = ceil_div(b - a, (int64_t)kPiece);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t cub_scan_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const int*>(nullptr),
                                static_cast<int*>(nullptr), (int)std::max<int64_t>(n, 1));
  return bytes;
}

size_t cub_scan64_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const int64_t*>(nullptr),
                                static_cast<int64_t*>(nullptr), (int)std::max<int64_t>(n, 1));
  return bytes;
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_prev_keys(const int32_t* tokens, int64_t N, int K, int A, int with_pos,
                               int32_t* keys, void* stream) {
  if (N < 0 || K < 1 || A < 1) return fail(kDimension, "prev_keys: bad sizes");
  if (N == 0) return kOk;
  const int64_t M = N * K;
  const int grid = (int)std::min<int64_t>(ceil_div(M, kThreads), (int64_t)kNumSMs * 8);
  prev_keys_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(tokens, M, K, A, with_pos, keys);
  return post_launch("prev_keys_kernel");
}

extern "C" int accel_step_keys(const int32_t* steps, const int32_t* frame_of, int64_t R,
                               int n_steps, int32_t* keys, unsigned* bad_count, void* stream) {
  if (R < 0 || n_steps < 1) return fail(kDimension, "step_keys: bad sizes");
  if (R == 0) return kOk;
  if (!steps || !keys || !bad_count) return fail(kDimension, "step_keys: NULL buffer");
  const int grid = (int)std::min<int64_t>(ceil_div(R, kThreads), (int64_t)kNumSMs * 8);
  step_keys_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(steps, frame_of, R, n_steps, keys,
                                                             bad_count);
  return post_launch("step_keys_kernel");
}

namespace {
// the caller's cpb counts 4096-row units; internally a block is cpb * (4096 /
// chunk_rows) warp chunks (the same rows)
int64_t blocks_of(int64_t R, int64_t cpb) {
  const int64_t n_chunks = std::max<int64_t>(1, ceil_div(R, (int64_t)chunk_rows(R)));
  return cpb <= 0 ? 1 : ceil_div(n_chunks, cpb);
}
int64_t cpb_of(int64_t R, int64_t cpb) {
  const int64_t n_chunks = std::max<int64_t>(1, ceil_div(R, (int64_t)chunk_rows(R)));
  return cpb <= 0 ? n_chunks : std::min(cpb * (kChunk / chunk_rows(R)), n_chunks);
}
}  // namespace

extern "C" size_t accel_group_workspace_size_blocked(int64_t R, int nkeys, int64_t cpb) {
  const int64_t c = cpb_of(R, cpb), nb = blocks_of(R, c);
  const int64_t n = (int64_t)nkeys * nb * c;
  const int64_t nk = (int64_t)nkeys * nb + 1;
  return 2 * align256(sizeof(int) * (size_t)n) +
         std::max(align256(cub_scan_bytes(n)),
                  align256(sizeof(int64_t) * (size_t)nk) + align256(cub_scan64_bytes(nk))) + 256;
}

extern "C" size_t accel_group_workspace_size(int64_t R, int nkeys) {
  return accel_group_workspace_size_blocked(R, nkeys, 0);
}

extern "C" int64_t accel_group_blocks(int64_t R, int64_t cpb) { return blocks_of(R, cpb_of(R, cpb)); }

extern "C" int64_t accel_group_max_pieces_blocked(int64_t R, int nkeys, int64_t cpb) {
  return ceil_div(R, kPiece) + (int64_t)nkeys * blocks_of(R, cpb_of(R, cpb));
}

extern "C" int64_t accel_group_max_pieces(int64_t R, int nkeys) {
  return accel_group_max_pieces_blocked(R, nkeys, 0);
}

// perm[R]: row ids sorted stably by composite key (block of cpb 4096-row chunks,
// key); seg_off / piece_off [blocks * nkeys + 1].  cpb <= 0: one block.
extern "C" int accel_group_by_key_blocked(const int32_t* keys, int64_t R, int nkeys, int64_t cpb,
                                          int32_t* perm, int64_t* seg_off, int64_t* piece_off,
                                          int32_t* piece_key, const int32_t* frame_of,
                                          const int32_t* tokens, int K, int32_t* row_frame,
                                          int32_t* row_tok, int32_t* pos, void* workspace,
                                          size_t workspace_bytes, void* stream) {
  if (R < 0 || nkeys < 1) return fail(kDimension, "group_by_key: bad sizes");
  if (nkeys * (size_t)kWarps * sizeof(int) > 200 * 1024)
    return fail(kDimension, "group_by_key: %d keys exceed the shared-memory histogram", nkeys);
  if (R >= ((int64_t)1 << 31)) return fail(kDimension, "group_by_key: R exceeds int32 range");
  if (!keys || !perm || !seg_off || !piece_off || !workspace)
    return fail(kDimension, "group_by_key: NULL buffer");
  if (workspace_bytes < accel_group_workspace_size_blocked(R, nkeys, cpb))
    return fail(kDimension, "group_by_key: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int crows = chunk_rows(R);
  const int64_t n_chunks = std::max<int64_t>(1, ceil_div(R, (int64_t)crows));
  const int64_t c = cpb_of(R, cpb), nb = blocks_of(R, c);
  const int64_t n = (int64_t)nkeys * nb * c;
  if (n >= ((int64_t)1 << 31) || nkeys * nb >= ((int64_t)1 << 31))
    return fail(kDimension, "group_by_key: too many counters");
  char* ws = static_cast<char*>(workspace);
  int* counts = reinterpret_cast<int*>(ws);
  int* base = reinterpret_cast<int*>(ws + align256(sizeof(int) * (size_t)n));
  void* cub_tmp = ws + 2 * align256(sizeof(int) * (size_t)n);
  size_t cub_bytes = cub_scan_bytes(n);
  const size_t smem = sizeof(int) * (size_t)nkeys * kWarps;
  const int grid = (int)ceil_div(n_chunks, kWarps);
  int st;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(chunk_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(stable_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  }
  if (nb * c != n_chunks) {  // the last block's missing chunks count zero rows
    if ((st = check_cuda(cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)n, s), "group memset")))
      return st;
  }
  chunk_hist_kernel<<<grid, kThreads, smem, s>>>(keys, R, nkeys, n_chunks, c, crows, counts);
  if ((st = post_launch("chunk_hist_kernel"))) return st;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, counts, base, (int)n, s);
  if (e != cudaSuccess) return fail(kCuda, "DeviceScan: %s", cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (nb == 1) {
    segment_offsets_kernel<<<1, 1024, 0, s>>>(base, nkeys, c, R, seg_off, piece_off);
    if ((st = post_launch("segment_offsets_kernel"))) return st;
  } else {  // many composite keys: parallel counts + a CUB scan of the piece counts
    const int64_t nk = (int64_t)nkeys * nb;
    int64_t* pcount = reinterpret_cast<int64_t*>(cub_tmp);
    void* tmp2 = static_cast<char*>(cub_tmp) + align256(sizeof(int64_t) * (size_t)(nk + 1));
    size_t b2 = cub_scan64_bytes(nk + 1);
    seg_counts_kernel<<<(unsigned)ceil_div(nk + 1, 256), 256, 0, s>>>(base, nk, c, R, seg_off,
                                                                       pcount);
    if ((st = post_launch("seg_counts_kernel"))) return st;
    e = cub::DeviceScan::ExclusiveSum(tmp2, b2, pcount, piece_off, (int)(nk + 1), s);
    if (e != cudaSuccess) return fail(kCuda, "DeviceScan: %s", cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (piece_key != nullptr) {
    const int64_t nk = (int64_t)nkeys * nb;
    piece_keys_kernel<<<(unsigned)ceil_div(nk, 256), 256, 0, s>>>(piece_off, nk, piece_key);
    if ((st = post_launch("piece_keys_kernel"))) return st;
  }
  if (R == 0) return kOk;
  SortedRows sr{frame_of, tokens, K, row_frame, row_tok, pos};
  if (row_frame != nullptr && (!frame_of || !tokens || !row_tok || K < 1))
    return fail(kDimension, "group_by_key: sorted rows need frame_of, tokens, outputs, K");
  if ((row_frame == nullptr) != (row_tok == nullptr))
    return fail(kDimension, "group_by_key: row_frame and row_tok go together");
  stable_scatter_kernel<<<grid, kThreads, smem, s>>>(keys, R, nkeys, n_chunks, c, crows, base, perm,
                                                     sr);
  return post_launch("stable_scatter_kernel");
}

// perm[R]: row ids sorted stably by key; seg_off[nkeys+1]; piece_off[nkeys+1]
extern "C" int accel_group_by_key(const int32_t* keys, int64_t R, int nkeys, int32_t* perm,
                                  int64_t* seg_off, int64_t* piece_off, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  return accel_group_by_key_blocked(keys, R, nkeys, 0, perm, seg_off, piece_off, nullptr, nullptr,
                                    nullptr, 1, nullptr, nullptr, nullptr, workspace,
                                    workspace_bytes, stream);
}

extern "C" size_t accel_fold_workspace_size(int nkeys, int D) {
  return sizeof(float) * ((size_t)kFoldSplit * nkeys + kHeavyMaxParts) * D;
}

// out[nkeys, D] = sum over blocks of the piece sums of composite keys b * nkeys + key
extern "C" int accel_fold_blocked_pieces(const float* piece_buf, const int64_t* piece_off,
                                         int nkeys, int nblocks, int D, int heavy_key, float* out,
                                         void* workspace, void* stream) {
  if (nkeys < 1 || nblocks < 1 || D < 4 || (D & 3) || heavy_key < -1 || heavy_key >= nkeys)
    return fail(kDimension, "fold_blocked: bad sizes");
  if (!piece_buf || !piece_off || !out || !workspace)
    return fail(kDimension, "fold_blocked: NULL buffer");
  if ((reinterpret_cast<uintptr_t>(piece_buf) | reinterpret_cast<uintptr_t>(out) |
       reinterpret_cast<uintptr_t>(workspace)) & 15)
    return fail(kDimension, "fold_blocked: buffers must be 16B aligned");
  cudaStream_t s = as_stream(stream);
  const int D4 = D / 4;
  float4* part = static_cast<float4*>(workspace);
  float4* hpart = part + (size_t)kFoldSplit * nkeys * D4;
  // every split is fixed by nblocks and the caller's heavy key: deterministic
  const int split = std::min(kFoldSplit, nblocks);
  float4* dst = split == 1 ? reinterpret_cast<float4*>(out) : part;
  const auto pieces = reinterpret_cast<const float4*>(piece_buf);
  fold_blocked_pieces_kernel<<<dim3(nkeys, split), kFoldThreads, 0, s>>>(
      pieces, piece_off, nkeys, nblocks, D4, nblocks > 1 ? heavy_key : -1, dst);
  int st = post_launch("fold_blocked_pieces_kernel");
  if (st) return st;
  // (a single block: the plain pass already runs every key on its own CTAs)
  const int heavy = nblocks > 1 ? heavy_key : -1;
  if (split > 1) {
    const int64_t n4 = (int64_t)nkeys * D4;
    const int64_t h0 = heavy >= 0 ? (int64_t)heavy * D4 : 0;
    fold_parts_kernel<<<(unsigned)ceil_div(n4, 256), 256, 0, s>>>(
        part, n4, n4, split, reinterpret_cast<float4*>(out), h0, heavy >= 0 ? h0 + D4 : 0);
    if ((st = post_launch("fold_parts_kernel"))) return st;
  }
  if (heavy >= 0) {
    const int r = nblocks >= kHeavySplit ? 1 : (kHeavySplit + nblocks - 1) / nblocks;
    const int nq = r == 1 ? kHeavySplit : nblocks * r;  // <= kHeavyMaxParts
    fold_heavy_parts_kernel<<<nq, kFoldThreads, 0, s>>>(pieces, piece_off, nkeys, nblocks, D4,
                                                        heavy, r, hpart);
    if ((st = post_launch("fold_heavy_parts_kernel"))) return st;
    fold_heavy_kernel<<<1, kFoldThreads, 0, s>>>(hpart, nq, D4, heavy,
                                                 reinterpret_cast<float4*>(out));
    st = post_launch("fold_heavy_kernel");
  }
  return st;
}

// out[nkeys, D] = grouped sums of vals[R, D] rows; piece_buf holds
// accel_group_max_pieces(R, nkeys) * D floats.
extern "C" int accel_grouped_rows_sum(const float* vals, int64_t R, int D, const int32_t* perm,
                                      const int64_t* seg_off, const int64_t* piece_off,
                                      const int32_t* piece_key, int nkeys, int64_t n_pieces,
                                      float* piece_buf, float* out, void* stream) {
  if (R < 0 || D < 1 || nkeys < 1 || n_pieces < 0) return fail(kDimension, "grouped_rows_sum: bad sizes");
  if (!perm || !seg_off || !piece_off || !piece_buf || !out)
    return fail(kDimension, "grouped_rows_sum: NULL buffer");
  if ((D & 3) == 0 && ((reinterpret_cast<uintptr_t>(vals) | reinterpret_cast<uintptr_t>(piece_buf)) & 15))
    return fail(kDimension, "grouped_rows_sum: vals/piece_buf must be 16B aligned");
  cudaStream_t s = as_stream(stream);
  int st;
  if (vals && n_pieces > 0) {  // vals == NULL: piece_buf already holds the piece sums
    piece_sum_kernel<<<(unsigned)n_pieces, kThreads, kThreads * sizeof(float4), s>>>(
        vals, perm, seg_off, piece_off, piece_key, nkeys, D, piece_buf);
    if ((st = post_launch("piece_sum_kernel"))) return st;
  }
  if ((D & 3) == 0 && ((reinterpret_cast<uintptr_t>(piece_buf) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
    key_sum4_kernel<<<nkeys, kKeyThreads, kKeyThreads * sizeof(float4), s>>>(
        reinterpret_cast<const float4*>(piece_buf), piece_off, nkeys, D / 4,
        reinterpret_cast<float4*>(out));
    return post_launch("key_sum4_kernel");
  }
  key_sum_kernel<<<nkeys, kThreads, kThreads * sizeof(float), s>>>(piece_buf, piece_off, nkeys, D,
                                                                   out);
  return post_launch("key_sum_kernel");
}
