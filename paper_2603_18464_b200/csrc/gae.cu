// (a) Segmented reverse-scan GAE + pooled-normalization statistics.
//
// Reference: trainer.py:79-101 (compute_gae, one Python loop per
// trajectory), trainer.py:128-158 (shard sums -> pooled mean/std).
//
// Design (single pass over HBM, 20 B/transition + 17 B/trajectory):
//   * The ragged batch is one flat array of N transitions; trajectory s
//     owns transitions [off[s], off[s+1]) and value frames
//     [off[s]+s, off[s+1]+s] (T+1 values, bootstrap last).
//   * A_t = delta_t + c_t * A_{t+1} with c_t = gamma*lam, or 0 at the last
//     step of a trajectory, is a linear recurrence; its scan operator is the
//     affine map (b, c): A_left = b + c * A_right.
//   * A warp owns a contiguous range of whole trajectories: the ones whose
//     start cost (transitions + kTrajCost per trajectory) falls in its 1/W share
//     (found by a 16-ary half-warp search on the offsets; fixed for a given
//     grid, so the pooled sums are bitwise deterministic).
//   * A trajectory is one chunk when it has <= 544 steps (longer ones: 544-step
//     chunks from the right, carry between them).  The chunk's r and v land in
//     shared memory by 4-byte cp.async copies (coalesced rows), double-buffered
//     one chunk ahead; lane l then owns kd = ceil(T / 32) consecutive steps:
//     a serial right-to-left fold of its affine maps, ONE 5-level shuffle
//     suffix scan of the 32 lane maps, a serial resolve, and the outputs go
//     back through shared memory to coalesced row stores.  No block barriers,
//     no inter-CTA traffic.
//   * The recurrence runs in fp32; the TD error is formed with gamma split into
//     two floats (see the kernel), so rounding stays relative to the TD error
//     and the advantage, never to |v|.  Per-CTA (sum A, sum A^2) partials in
//     float64 feed the pooled statistics in CTA order.
#include <cfloat>

#include "common.cuh"

namespace accel {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 17;                 // max consecutive steps per lane
constexpr int kChunkSteps = 32 * kItems;   // max steps per warp chunk (one chunk per
                                           // trajectory up to 544 steps)
constexpr int kPitch = kChunkSteps + 4;
#ifndef ACCEL_GAE_GRP
#define ACCEL_GAE_GRP 4
#endif
constexpr int kGrp = ACCEL_GAE_GRP;  // steps per group in the fold / resolve
constexpr int kMaxGrid = 148 * 8;          // persistent grid bound (partials capacity)

struct Workspace {
  double* partials;   // [grid][3]
  unsigned* counter;  // [1] arrival ticket (zeroed before the launch)
};

size_t workspace_bytes() { return 3 * sizeof(double) * kMaxGrid + 16; }

constexpr size_t kGaeSmem = sizeof(float) * kWarps * 2 * 2 * kPitch;

Workspace carve(void* base) {
  Workspace w;
  w.partials = static_cast<double*>(base);
  w.counter = reinterpret_cast<unsigned*>(static_cast<char*>(base) +
                                          3 * sizeof(double) * kMaxGrid);
  return w;
}

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

// First s in [0, n] with off[s] + kTrajCost*s >= target, searched by the
// 16 lanes of a half-warp: 16-ary narrowing, one dependent load per round.  The
// two half-warps search different targets; the loop runs until both are done.
// Warp ranges balance transitions + kTrajCost per trajectory: a chunk's fixed
// cost (offsets, staging setup, the shuffle scan, the partial rows) is worth
// about that many steps of the serial scan, so ranges of short trajectories
// would otherwise finish last.
#ifndef ACCEL_GAE_TRAJ_COST
#define ACCEL_GAE_TRAJ_COST 256
#endif
constexpr int64_t kTrajCost = ACCEL_GAE_TRAJ_COST;

__device__ __forceinline__ int64_t half_warp_lower_bound(const int64_t* __restrict__ off,
                                                         int64_t n, int64_t target, int hl,
                                                         unsigned hmask, int hshift) {
  int64_t lo = 0, hi = n;
  bool fin = lo >= hi;
  while (__any_sync(0xffffffffu, !fin)) {
    int64_t q = hi, step = 1;
    bool ge = true;
    if (!fin) {
      step = (hi - lo + 16) / 16;  // ceil((hi - lo + 1) / 16)
      q = min(lo + (int64_t)(hl + 1) * step - 1, hi);
      ge = __ldg(off + q) + kTrajCost * q >= target;
    }
    const unsigned m = (__ballot_sync(0xffffffffu, ge) & hmask) >> hshift;
    const int f = __ffs(m) - 1;  // lane 15 probes hi: always set
    const int64_t qf = __shfl_sync(0xffffffffu, q, hshift + f);
    const int64_t qp = __shfl_sync(0xffffffffu, q, hshift + max(f - 1, 0));
    if (!fin) {
      const int64_t nlo = f == 0 ? lo : qp + 1;
      if (qf == nlo || step == 1) {
        lo = hi = qf;
        fin = true;
      } else {
        lo = nlo;
        hi = qf;
      }
    }
  }
  return lo;
}

__global__ void __launch_bounds__(kThreads, 2)
gae_warp_kernel(const float* __restrict__ rewards, const float* __restrict__ vals,
                const int64_t* __restrict__ off, const uint8_t* __restrict__ done,
                int64_t n_traj, float g_hi, float g_lo, float decay,
                float* __restrict__ adv_out, float* __restrict__ ret_out,
                int32_t* __restrict__ frame_out, Workspace ws, int64_t n_transitions,
                double* __restrict__ sums_out) {
  __shared__ double s_red[kWarps * 3];
  extern __shared__ __align__(16) float s_dyn[];  // [warp][buffer][r | v][kPitch]
  auto s_buf = reinterpret_cast<float (*)[2][2][kPitch]>(s_dyn);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t W = (int64_t)gridDim.x * kWarps;
  const int64_t w = (int64_t)blockIdx.x * kWarps + warp;
  // this warp's trajectories [sa, sb): the ones starting in its 1/W share of
  // the cost (transitions + kTrajCost per trajectory, fixed for a given grid)
  int64_t sa, sb;
  {
    const int half = lane >> 4, hl = lane & 15;
    const int64_t target =
        (int64_t)(((__int128)(w + half) * (n_transitions + kTrajCost * n_traj) + W - 1) / W);
    const int64_t x = half_warp_lower_bound(off, n_traj, target, hl,
                                            half ? 0xffff0000u : 0x0000ffffu, half ? 16 : 0);
    sa = __shfl_sync(0xffffffffu, x, 0);
    sb = w + 1 == W ? n_traj : __shfl_sync(0xffffffffu, x, 16);
  }
  double S = 0.0, Q = 0.0;
  int nbad = 0;

  // chunk sequence: trajectory s from its end leftwards, chunks [cb, e), e -= 256.
  // Offsets and the done flag are prefetched one trajectory ahead (off[s+1]
  // is already known when s starts, so one new load per trajectory).
  struct Ck { int64_t s, t0, T, cb, e; bool dn; };
  int64_t pf_t0 = 0, pf_t1 = 0;
  int pf_dn = 0;
  if (sa < sb) {
    pf_t0 = __ldg(off + sa);
    pf_t1 = __ldg(off + sa + 1);
    pf_dn = __ldg(done + sa);
  }
  auto first_chunk = [&](int64_t s) -> Ck {  // s = the prefetched trajectory
    Ck c{s, 0, 0, 0, 0, false};
    if (s < sb) {
      c.t0 = pf_t0;
      c.T = pf_t1 - pf_t0;
      c.dn = pf_dn != 0;
      c.e = c.T;
      c.cb = c.e > kChunkSteps ? c.e - kChunkSteps : 0;
      if (s + 1 < sb) {
        pf_t0 = pf_t1;
        pf_t1 = __ldg(off + s + 2);
        pf_dn = __ldg(done + s + 1);
      }
    }
    return c;
  };
  auto next_chunk = [&](const Ck& c) -> Ck {
    if (c.cb > 0) {
      Ck n = c;
      n.e = c.cb;
      n.cb = n.e > kChunkSteps ? n.e - kChunkSteps : 0;
      return n;
    }
    return first_chunk(c.s + 1);
  };
  // stage chunk c (r[cb, e), v[cb, e]) into buffer b: 4-byte async copies,
  // step i at slot i (rows coalesced), the value after the chunk at slot nv
  auto stage = [&](const Ck& c, int b) {
    if (c.s >= sb) return;
    const int nv = (int)(c.e - c.cb);
    const float* rc = rewards + c.t0 + c.cb + lane;
    const float* vc = vals + c.t0 + c.s + c.cb;
    float* sr = s_buf[warp][b][0] + lane;
    float* sv = s_buf[warp][b][1] + lane;
    const float* vl = vc + lane;
    // full rows without a lane predicate, then the partial row
    const int nfull = nv >> 5;
#pragma unroll 4
    for (int j = 0; j < nfull; ++j) {
      cp_async4(sr + 32 * j, rc + 32 * j);
      cp_async4(sv + 32 * j, vl + 32 * j);
    }
    if (32 * nfull + lane < nv) {
      cp_async4(sr + 32 * nfull, rc + 32 * nfull);
      cp_async4(sv + 32 * nfull, vl + 32 * nfull);
    }
    // the value after the chunk; a successful trajectory's bootstrap value is 0
    // (trainer.py:92-93), written here so the scan needs no last-step test
    if (lane == 0) {
      if (c.dn && c.e == c.T)
        s_buf[warp][b][1][nv] = 0.f;
      else
        cp_async4(s_buf[warp][b][1] + nv, vc + nv);
    }
  };

  Ck cur = first_chunk(sa);
  stage(cur, 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  float carry = 0.f;  // A right of the current chunk (0 past a trajectory's end)
  for (int it = 0; cur.s < sb; ++it) {
    const int b = it & 1;
    const Ck nxt = next_chunk(cur);
    stage(nxt, b ^ 1);  // its buffer was drained by the previous chunk
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const int nv = (int)(cur.e - cur.cb);
    const int kd = (nv + 31) >> 5;  // steps per lane (warp-uniform)
    float* sr = s_buf[warp][b][0] + kd * lane;  // this lane's steps kd*l .. kd*l + kd - 1
    float* sv = s_buf[warp][b][1] + kd * lane;
    const int nl = nv - kd * lane;  // this lane's valid steps
    // A chunk never spans two trajectories and the carry into a trajectory's
    // last chunk is 0, so the last step needs no special map: (d, decay)
    // applied to A = 0 is d, as the reference's zero continuation gives.
    float dl[kItems];
    float vnext = sv[min(kd, max(nl, 0))];  // v after the lane's last valid step
    float B = 0.f, C = 1.f;  // the lane's composed map (right to left)
    // steps in groups of kGrp (a warp-uniform test per group, the group's shared-memory
    // loads issued together); steps past the lane's last valid one are identities
#pragma unroll
    for (int g = (kItems - 1) / kGrp; g >= 0; --g) {
      const int k0 = kGrp * g;
      if (k0 < kd) {
        float vv[kGrp], rr[kGrp];
#pragma unroll
        for (int u = kGrp - 1; u >= 0; --u)
          if (k0 + u < kItems) {
            vv[u] = sv[k0 + u];
            rr[u] = sr[k0 + u];
          }
#pragma unroll
        for (int u = kGrp - 1; u >= 0; --u) {
          const int k = k0 + u;
          if (k < kItems) {
            const bool ok = k < nl && k < kd;
            // delta = r + gamma v' - v with gamma = g_hi + g_lo: fma(g_hi, v', -v) is
            // exact before its one rounding, so the error is relative to the TD
            // error, not to |v|
            const float d = fmaf(g_lo, vnext, fmaf(g_hi, vnext, -vv[u])) + rr[u];
            dl[k] = ok ? d : 0.f;
            const float ck = ok ? decay : 1.f;
            vnext = ok ? vv[u] : vnext;
            B = fmaf(ck, B, dl[k]);
            C *= ck;
          }
        }
      }
    }
    // exclusive suffix scan of the lane maps: the map of lanes (lane, 31]
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float ob = __shfl_down_sync(0xffffffffu, B, o);
      const float oc = __shfl_down_sync(0xffffffffu, C, o);
      if (lane + o < 32) {
        B = fmaf(C, ob, B);
        C *= oc;
      }
    }
    float eb = __shfl_down_sync(0xffffffffu, B, 1), ec = __shfl_down_sync(0xffffffffu, C, 1);
    if (lane == 31) { eb = 0.f; ec = 1.f; }
    float A = fmaf(ec, carry, eb);
    __syncwarp();  // every lane has read its neighbour's v before slots turn into outputs
    float Sf = 0.f, Qf = 0.f, Rf = 0.f;
#pragma unroll
    for (int g = (kItems - 1) / kGrp; g >= 0; --g) {
      const int k0 = kGrp * g;
      if (k0 < kd) {
        float vv[kGrp];
#pragma unroll
        for (int u = kGrp - 1; u >= 0; --u)
          if (k0 + u < kItems) vv[u] = sv[k0 + u];
#pragma unroll
        for (int u = kGrp - 1; u >= 0; --u) {
          const int k = k0 + u;
          if (k < kItems && k < kd && k < nl) {
            A = fmaf(decay, A, dl[k]);
            const float rt = A + vv[u];
            sr[k] = A;
            sv[k] = rt;
            Sf += A;
            Qf = fmaf(A, A, Qf);
            Rf += rt;
          }
        }
      }
    }
    // non-finite outputs: a finite sum has only finite terms, so the per-step
    // test runs only when a lane's sums are not finite (an inf / NaN output, or
    // an overflowing sum of finite ones: the recount then finds none)
    if (!(fabsf(Sf) <= FLT_MAX && fabsf(Rf) <= FLT_MAX)) {
      for (int k = 0; k < min(kd, nl); ++k)
        nbad += (fabsf(sr[k]) <= FLT_MAX && fabsf(sv[k]) <= FLT_MAX) ? 0 : 1;
    }
    S += (double)Sf;
    Q += (double)Qf;
    carry = __shfl_sync(0xffffffffu, A, 0);  // A at the chunk's first step
    __syncwarp();
    // coalesced write-back of the chunk
    const float* sr0 = s_buf[warp][b][0] + lane;
    const float* sv0 = s_buf[warp][b][1] + lane;
    float* ac = adv_out + cur.t0 + cur.cb + lane;
    float* rtc = ret_out + cur.t0 + cur.cb + lane;
    // full rows without a lane predicate, then the partial row
    const int nfull = nv >> 5;
#pragma unroll 4
    for (int j = 0; j < nfull; ++j) {
      __stcs(ac + 32 * j, sr0[32 * j]);
      __stcs(rtc + 32 * j, sv0[32 * j]);
    }
    const bool part = 32 * nfull + lane < nv;
    if (part) {
      __stcs(ac + 32 * nfull, sr0[32 * nfull]);
      __stcs(rtc + 32 * nfull, sv0[32 * nfull]);
    }
    if (frame_out != nullptr) {
      int32_t* fc = frame_out + cur.t0 + cur.cb + lane;
      const int32_t fb = (int32_t)(cur.t0 + cur.s + cur.cb) + lane;
#pragma unroll 4
      for (int j = 0; j < nfull; ++j) __stcs(fc + 32 * j, fb + 32 * j);
      if (part) __stcs(fc + 32 * nfull, fb + 32 * nfull);
    }
    __syncwarp();  // the buffer is restaged two chunks on
    if (nxt.s != cur.s) carry = 0.f;  // next chunk starts a new trajectory at its end
    cur = nxt;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");

  // statistics: one partial per CTA (its warps' trajectories in a fixed order),
  // then the last CTA to arrive sums the partials in CTA order -- the grid size
  // is fixed for a device, so the pooled sums are bitwise deterministic
  __shared__ bool s_last;
  double v3[3] = {S, Q, (double)nbad};
  block_sum_d<3>(v3, s_red);
  if (tid == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) ws.partials[3 * blockIdx.x + c] = v3[c];
    __threadfence();
    s_last = atomicAdd(ws.counter, 1u) == gridDim.x - 1u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double z[3] = {0.0, 0.0, 0.0};
  for (int t = tid; t < (int)gridDim.x; t += kThreads)
#pragma unroll
    for (int c = 0; c < 3; ++c) z[c] += __ldcg(ws.partials + 3 * t + c);
  block_sum_d<3>(z, s_red);
  if (tid == 0) {
    sums_out[0] = z[0];
    sums_out[1] = z[1];
    sums_out[2] = (double)n_transitions;
    sums_out[3] = z[2];
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

extern "C" size_t accel_gae_workspace_size(int64_t n_traj, int64_t n_transitions) {
  (void)n_traj;
  (void)n_transitions;
  return workspace_bytes();
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
  if (workspace_bytes_ < workspace_bytes())
    return fail(kDimension, "GAE workspace too small (%zu < %zu)", workspace_bytes_,
                workspace_bytes());
  Workspace ws = carve(workspace);
  int st = check_cuda(cudaMemsetAsync(ws.counter, 0, sizeof(unsigned), s), "gae counter");
  if (st) return st;
  // grid per device (a process may drive several GPUs)
  static int grids[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return fail(kDimension, "gae: device ordinal %d", dev);
  int& grid = grids[dev];
  if (grid == 0) {
    st = check_cuda(cudaFuncSetAttribute(gae_warp_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kGaeSmem), "gae smem");
    if (st) return st;
    int per_sm = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    st = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_warp_kernel,
                                                                  kThreads, kGaeSmem),
                    "gae occupancy");
    if (st) return st;
    grid = std::max(1, std::min(per_sm * sms, kMaxGrid));
  }
  const int64_t need = ceil_div(ceil_div(n_transitions, 64), kWarps);  // >= 64 steps per warp
  gae_warp_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(grid, need)), kThreads, kGaeSmem, s>>>(
      rewards, values_frames, traj_off, done, n_traj, (float)gamma,
      (float)(gamma - (double)(float)gamma), (float)(gamma * lam), adv_out, ret_out,
      frame_of_out, ws, n_transitions, sums_out);
  return post_launch("gae_warp_kernel");
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
