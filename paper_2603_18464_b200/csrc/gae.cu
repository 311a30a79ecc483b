// (a) Segmented reverse-scan GAE + pooled-normalization statistics.
//
// Reference: trainer.py:79-101 (compute_gae, one Python loop per
// trajectory), trainer.py:128-158 (shard sums -> pooled mean/std).
//
// Design (single pass over HBM, 16 B/transition + 13 B/trajectory):
//   * The ragged batch is one flat array of N transitions; trajectory s
//     owns transitions [off[s], off[s+1]) and value frames
//     [off[s]+s, off[s+1]+s] (T+1 values, bootstrap last).
//   * A_t = delta_t + c_t * A_{t+1} with c_t = gamma*lam, or 0 at the last
//     step of a trajectory, is a linear recurrence; the scan operator is the
//     affine map (b, c): A_left = b + c * A_right.
//   * Each CTA owns a 2048-transition tile; tiles are claimed right-to-left
//     via an atomic ticket and chained with decoupled look-back, so every
//     element is read once.  A tile containing a trajectory end has c = 0
//     and publishes its inclusive value immediately (no waiting chain).
//   * Arithmetic is float64 (HBM-bound kernel, fp64 is free here); the
//     per-tile (sum A, sum A^2) partials feed the pooled statistics in
//     fixed order, so results are bitwise deterministic.
#include "common.cuh"

namespace accel {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;

struct Map {
  double b, c;
};

// l covers the earlier (left) range, r the later one.
__device__ __forceinline__ Map compose(const Map& l, const Map& r) {
  return {fma(l.c, r.b, l.b), l.c * r.c};
}

__device__ __forceinline__ Map shfl_down_map(const Map& m, int d) {
  return {__shfl_down_sync(0xffffffffu, m.b, d), __shfl_down_sync(0xffffffffu, m.c, d)};
}

// index of the trajectory containing transition t: last s with off[s] <= t
__device__ __forceinline__ int64_t find_traj(const int64_t* off, int64_t n_traj, int64_t t) {
  int64_t lo = 0, hi = n_traj;  // invariant off[lo] <= t < off[hi]
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

struct Workspace {
  unsigned* counter;
  unsigned* flags;
  Map* agg;
  double* inc;
  double* partials;  // [tiles][3]
  size_t reset_bytes;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

Workspace carve(void* base, int64_t tiles) {
  char* p = static_cast<char*>(base);
  Workspace w;
  w.counter = reinterpret_cast<unsigned*>(p);
  w.flags = reinterpret_cast<unsigned*>(p + 16);
  size_t o = align_up(16 + 4 * (size_t)tiles, 16);
  w.reset_bytes = o;
  w.agg = reinterpret_cast<Map*>(p + o);
  o += sizeof(Map) * (size_t)tiles;
  w.inc = reinterpret_cast<double*>(p + o);
  o += sizeof(double) * (size_t)tiles;
  w.partials = reinterpret_cast<double*>(p + o);
  return w;
}

size_t workspace_bytes(int64_t tiles) {
  size_t o = align_up(16 + 4 * (size_t)tiles, 16);
  o += (sizeof(Map) + sizeof(double) + 3 * sizeof(double)) * (size_t)tiles;
  return o + 16;
}

__global__ void __launch_bounds__(kThreads)
gae_scan_kernel(const float* __restrict__ rewards, const float* __restrict__ vals,
                const int64_t* __restrict__ off, const uint8_t* __restrict__ done,
                int64_t n_traj, int64_t n, double gamma, double decay,
                float* __restrict__ adv_out, float* __restrict__ ret_out,
                int32_t* __restrict__ frame_out, Workspace ws, int num_tiles) {
  __shared__ int s_tile;
  __shared__ int64_t s_lo, s_hi;
  __shared__ int s_end[kTile + 1];
  __shared__ float s_val[2 * kTile + 2];
  __shared__ Map s_warp[kWarps];
  __shared__ double s_carry;
  __shared__ double s_red[kWarps * 3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = num_tiles - 1 - (int)atomicAdd(ws.counter, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int64_t t0 = (int64_t)tile * kTile;
  const int64_t t1 = min(t0 + (int64_t)kTile, n);
  const int len = (int)(t1 - t0);

  if (tid == 0) s_lo = find_traj(off, n_traj, t0);
  if (tid == 32) s_hi = find_traj(off, n_traj, t1 - 1);
  __syncthreads();
  const int64_t lo = s_lo;
  const int ns = (int)(s_hi - lo + 1);
  for (int j = tid; j < ns; j += kThreads) {
    int64_t e = __ldg(off + lo + j + 1) - t0;
    s_end[j] = (int)min(e, (int64_t)kTile + 1);
  }
  const int cnt = len + ns;
  const float* vbase = vals + t0 + lo;
  for (int k = tid; k < cnt; k += kThreads) s_val[k] = __ldg(vbase + k);

  // rewards: 8 consecutive transitions per thread (two 16-byte loads)
  const int i0 = tid * kItems;
  float r[kItems];
  if (t0 + i0 + kItems <= n) {
    const float4* rp = reinterpret_cast<const float4*>(rewards + t0 + i0);
    float4 a = __ldcs(rp), b = __ldcs(rp + 1);
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < kItems; ++k) r[k] = (i0 + k < len) ? rewards[t0 + i0 + k] : 0.f;
  }
  __syncthreads();

  // per-item deltas and continuation masks
  double delta[kItems];
  float vcur[kItems];
  unsigned cont = 0;  // bit k set: c_k = decay
  int j = 0;
  if (i0 < len) {
    int a = 0, b = ns - 1;  // first j with s_end[j] > i0
    while (a < b) {
      int m = (a + b) >> 1;
      if (s_end[m] > i0) b = m; else a = m + 1;
    }
    j = a;
  }
  const int j_first = j;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int i = i0 + k;
    if (i < len) {
      while (s_end[j] <= i) ++j;
      const bool last = (s_end[j] == i + 1);
      const float vc = s_val[i + j];
      float vn = s_val[i + j + 1];
      if (last && __ldg(done + lo + j)) vn = 0.f;
      delta[k] = fma(gamma, (double)vn, (double)r[k]) - (double)vc;
      vcur[k] = vc;
      if (!last) cont |= 1u << k;
    } else {
      delta[k] = 0.0;
      vcur[k] = 0.f;
      cont |= 1u << k;  // identity map past the end
    }
  }

  // thread map over its 8 items (right to left)
  Map m{0.0, 1.0};
#pragma unroll
  for (int k = kItems - 1; k >= 0; --k) {
    const double c = (cont >> k & 1u) ? decay : 0.0;
    m.b = fma(c, m.b, delta[k]);
    m.c *= c;
  }
  // warp suffix scan
  Map incl = m;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Map o = shfl_down_map(incl, d);
    if (lane + d < 32) incl = compose(incl, o);
  }
  Map excl = shfl_down_map(incl, 1);
  if (lane == 31) excl = Map{0.0, 1.0};
  if (lane == 0) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    Map w = lane < kWarps ? s_warp[lane] : Map{0.0, 1.0};
    Map wi = w;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
      Map o = shfl_down_map(wi, d);
      if (lane + d < kWarps) wi = compose(wi, o);
    }
    Map we = shfl_down_map(wi, 1);
    if (lane >= kWarps - 1) we = Map{0.0, 1.0};
    __syncwarp();
    if (lane < kWarps) s_warp[lane] = we;  // exclusive suffix of warps to the right

    if (lane == 0) {
      const Map agg = wi;  // whole-tile map
      double carry = 0.0;
      if (tile == num_tiles - 1) {
        ws.inc[tile] = agg.b;
        st_release_u32(ws.flags + tile, 2u);
      } else {
        if (agg.c == 0.0) {
          ws.inc[tile] = agg.b;
          st_release_u32(ws.flags + tile, 2u);
        } else {
          ws.agg[tile] = agg;
          st_release_u32(ws.flags + tile, 1u);
        }
        Map acc{0.0, 1.0};
        for (int q = tile + 1;; ++q) {
          unsigned f;
          do { f = ld_acquire_u32(ws.flags + q); } while (f == 0u);
          if (f == 2u) {
            carry = fma(acc.c, __ldcg(ws.inc + q), acc.b);
            break;
          }
          Map st{__ldcg(&ws.agg[q].b), __ldcg(&ws.agg[q].c)};
          acc = compose(acc, st);
          if (acc.c == 0.0) { carry = acc.b; break; }
        }
        if (agg.c != 0.0) {
          ws.inc[tile] = fma(agg.c, carry, agg.b);
          st_release_u32(ws.flags + tile, 2u);
        }
      }
      s_carry = carry;
    }
  }
  __syncthreads();

  // resolve this thread's right-hand context and emit
  const Map right = compose(excl, s_warp[warp]);
  double A = fma(right.c, s_carry, right.b);
  double S = 0.0, Q = 0.0, bad = 0.0;
  float a_out[kItems], r_out[kItems];
#pragma unroll
  for (int k = kItems - 1; k >= 0; --k) {
    const double c = (cont >> k & 1u) ? decay : 0.0;
    A = fma(c, A, delta[k]);
    const float af = (float)A;
    const float rf = (float)(A + (double)vcur[k]);
    a_out[k] = af;
    r_out[k] = rf;
    if (i0 + k < len) {
      S += A;
      Q = fma(A, A, Q);
      if (!isfinite(af) || !isfinite(rf)) bad += 1.0;
    }
  }
  if (t0 + i0 + kItems <= n) {
    float4* ap = reinterpret_cast<float4*>(adv_out + t0 + i0);
    float4* rp = reinterpret_cast<float4*>(ret_out + t0 + i0);
    __stcs(ap, make_float4(a_out[0], a_out[1], a_out[2], a_out[3]));
    __stcs(ap + 1, make_float4(a_out[4], a_out[5], a_out[6], a_out[7]));
    __stcs(rp, make_float4(r_out[0], r_out[1], r_out[2], r_out[3]));
    __stcs(rp + 1, make_float4(r_out[4], r_out[5], r_out[6], r_out[7]));
  } else {
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (i0 + k < len) {
        adv_out[t0 + i0 + k] = a_out[k];
        ret_out[t0 + i0 + k] = r_out[k];
      }
  }
  if (frame_out != nullptr && i0 < len) {
    int jj = j_first;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int i = i0 + k;
      if (i < len) {
        while (s_end[jj] <= i) ++jj;
        frame_out[t0 + i] = (int32_t)(t0 + i + lo + jj);
      }
    }
  }

  double v3[3] = {S, Q, bad};
  block_sum_d<3>(v3, s_red);
  if (tid == 0) {
    ws.partials[3 * (int64_t)tile + 0] = v3[0];
    ws.partials[3 * (int64_t)tile + 1] = v3[1];
    ws.partials[3 * (int64_t)tile + 2] = v3[2];
  }
}

// Fixed-order reduction of the per-tile partials -> {S, Q, N, bad}.
__global__ void __launch_bounds__(1024)
gae_sums_kernel(const double* __restrict__ partials, int tiles, int64_t n, double* sums) {
  __shared__ double s_red[32 * 3];
  double v[3] = {0.0, 0.0, 0.0};
  for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
    v[0] += partials[3 * (int64_t)t + 0];
    v[1] += partials[3 * (int64_t)t + 1];
    v[2] += partials[3 * (int64_t)t + 2];
  }
  block_sum_d<3>(v, s_red);
  if (threadIdx.x == 0) {
    sums[0] = v[0];
    sums[1] = v[1];
    sums[2] = (double)n;
    sums[3] = v[2];
  }
}

__global__ void normalize_finalize_kernel(const double* sums, double eps, double* stats) {
  const double S = sums[0], Q = sums[1], N = sums[2];
  double flags = 0.0, mean = 0.0, var = 0.0;
  if (N == 0.0) {
    flags = 1.0;
  } else {
    mean = S / N;
    var = Q / N - mean * mean;
    if (var < -1e-12) flags = 2.0;
    var = fmax(var, 0.0);
  }
  const double sd = sqrt(var);
  stats[0] = mean;
  stats[1] = sd;
  stats[2] = sd + eps;
  stats[3] = flags;
}

__global__ void normalize_apply_kernel(const float* __restrict__ adv, int64_t n,
                                       const double* __restrict__ stats,
                                       float* __restrict__ out) {
  const double mean = stats[0], denom = stats[2];
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = __ldcs(reinterpret_cast<const float4*>(adv) + i);
    float4 o;
    o.x = (float)(((double)a.x - mean) / denom);
    o.y = (float)(((double)a.y - mean) / denom);
    o.z = (float)(((double)a.z - mean) / denom);
    o.w = (float)(((double)a.w - mean) / denom);
    reinterpret_cast<float4*>(out)[i] = o;
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (float)(((double)adv[i] - mean) / denom);
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" size_t accel_gae_workspace_size(int64_t n_transitions) {
  if (n_transitions <= 0) return 16;
  return workspace_bytes(ceil_div(n_transitions, kTile));
}

extern "C" int accel_gae_segmented(const float* rewards, const float* values_frames,
                                   const int64_t* traj_off, const uint8_t* done,
                                   int64_t n_traj, int64_t n_transitions, double gamma,
                                   double lam, float* adv_out, float* ret_out,
                                   int32_t* frame_of_out, double* sums_out, void* workspace,
                                   size_t workspace_bytes_, void* stream) {
  if (!(gamma > 0.0 && gamma <= 1.0))
    return fail(kDomain, "gamma must be in (0, 1], got %g", gamma);
  if (!(lam >= 0.0 && lam <= 1.0)) return fail(kDomain, "lam must be in [0, 1], got %g", lam);
  if (n_traj < 0 || n_transitions < 0)
    return fail(kDimension, "negative sizes (n_traj=%lld, N=%lld)", (long long)n_traj,
                (long long)n_transitions);
  if (n_transitions > 0 && n_traj == 0)
    return fail(kDimension, "transitions without trajectories");
  if (n_transitions >= (int64_t)1 << 31)
    return fail(kDimension, "N=%lld exceeds the int32 frame index range",
                (long long)n_transitions);
  if (!sums_out) return fail(kDimension, "sums_out is NULL");
  cudaStream_t s = as_stream(stream);
  if (n_transitions == 0) {
    return check_cuda(cudaMemsetAsync(sums_out, 0, 4 * sizeof(double), s), "gae memset");
  }
  if (!rewards || !values_frames || !traj_off || !done || !adv_out || !ret_out || !workspace)
    return fail(kDimension, "NULL buffer passed to accel_gae_segmented");
  if ((reinterpret_cast<uintptr_t>(rewards) | reinterpret_cast<uintptr_t>(adv_out) |
       reinterpret_cast<uintptr_t>(ret_out)) & 15)
    return fail(kDimension, "GAE needs 16-byte aligned rewards/adv/ret buffers");
  const int64_t tiles = ceil_div(n_transitions, kTile);
  if (workspace_bytes_ < workspace_bytes(tiles))
    return fail(kDimension, "GAE workspace too small (%zu < %zu)", workspace_bytes_,
                workspace_bytes(tiles));
  Workspace ws = carve(workspace, tiles);
  int st = check_cuda(cudaMemsetAsync(workspace, 0, ws.reset_bytes, s), "gae reset");
  if (st) return st;
  gae_scan_kernel<<<(unsigned)tiles, kThreads, 0, s>>>(
      rewards, values_frames, traj_off, done, n_traj, n_transitions, gamma, gamma * lam,
      adv_out, ret_out, frame_of_out, ws, (int)tiles);
  if ((st = post_launch("gae_scan_kernel"))) return st;
  gae_sums_kernel<<<1, 1024, 0, s>>>(ws.partials, (int)tiles, n_transitions, sums_out);
  return post_launch("gae_sums_kernel");
}

extern "C" int accel_normalize_finalize(const double* sums, double eps, double* stats_out,
                                        void* stream) {
  if (!sums || !stats_out) return fail(kDimension, "NULL buffer passed to normalize_finalize");
  normalize_finalize_kernel<<<1, 1, 0, as_stream(stream)>>>(sums, eps, stats_out);
  return post_launch("normalize_finalize_kernel");
}

extern "C" int accel_normalize_apply(const float* adv, int64_t n, const double* stats,
                                     float* adv_norm_out, void* stream) {
  if (n < 0) return fail(kDimension, "negative length");
  if (n == 0) return kOk;
  if (!adv || !stats || !adv_norm_out) return fail(kDimension, "NULL buffer to normalize_apply");
  if ((reinterpret_cast<uintptr_t>(adv) | reinterpret_cast<uintptr_t>(adv_norm_out)) & 15)
    return fail(kDimension, "normalize_apply needs 16-byte aligned buffers");
  int64_t blocks = std::min<int64_t>(ceil_div(n / 4 + 1, 256), (int64_t)kNumSMs * 8);
  normalize_apply_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(adv, n, stats,
                                                                          adv_norm_out);
  return post_launch("normalize_apply_kernel");
}
