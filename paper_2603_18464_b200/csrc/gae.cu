// (a) Segmented reverse-scan GAE + pooled-normalization statistics.
//
// Reference: trainer.py:79-101 (compute_gae, one Python loop per
// trajectory), trainer.py:128-158 (shard sums -> pooled mean/std).
//
// Design (single pass over HBM, 20 B/transition + 13 B/trajectory):
//   * The ragged batch is one flat array of N transitions; trajectory s
//     owns transitions [off[s], off[s+1]) and value frames
//     [off[s]+s, off[s+1]+s] (T+1 values, bootstrap last).
//   * A_t = delta_t + c_t * A_{t+1} with c_t = gamma*lam, or 0 at the last
//     step of a trajectory, is a linear recurrence; the scan operator is the
//     affine map (b, c): A_left = b + c * A_right.
//   * Work is cut in value-frame space into segments of whole trajectories
//     (those whose first frame falls in a 2560-frame stride), swept by
//     persistent CTAs: a segment ends on a trajectory end, so no carry
//     crosses CTAs -- no look-back, no ticket, no inter-CTA wait.  Inside a
//     CTA the affine maps are suffix-scanned (thread, warp, block); a
//     trajectory reaching past a pass (3328 frames) is swept in several
//     right-to-left passes with the carry in shared memory.
//   * Loads are 16-B cp.async copies of aligned runs (segments start at
//     arbitrary offsets), all in flight at once; stores are staged through
//     shared memory into coalesced 16-B vectors.
//   * The issue budget is the limit (~20 B of HBM per transition), so the
//     recurrence runs in fp32; the TD error is formed with gamma split into
//     two floats (see the kernel), so rounding stays relative to the TD error
//     and the advantage, never to |v|.  Per-CTA (sum A, sum A^2) partials
//     feed the pooled statistics (float64) in a fixed order: bitwise
//     deterministic for a given device.
#include <cfloat>

#include "common.cuh"

namespace accel {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 13;                // odd: item-strided smem reads are conflict-free
constexpr int kChunk = kThreads * kItems;  // value frames per pass (3328)
constexpr int kSeg = 2560;                 // segment stride in frame space (single pass
                                           // while trajectories stay under 769 frames)
constexpr int kPad = 8;                    // float4 alignment slack in the staging arrays
constexpr int kVec = (kChunk + kPad + 4 + 4 * kThreads - 1) / (4 * kThreads);  // float4 / thread
constexpr size_t kSegSmem = sizeof(float) * (3 * (kChunk + kPad) + 4);
constexpr int kDoneBit = 1 << 30;          // packed beside a trajectory end in s_end
constexpr int kEndMask = kDoneBit - 1;

struct Map {
  float b, c;
};

// l covers the earlier (left) range, r the later one.
__device__ __forceinline__ Map compose(const Map& l, const Map& r) {
  return {fmaf(l.c, r.b, l.b), l.c * r.c};
}

__device__ __forceinline__ Map shfl_down_map(const Map& m, int d) {
  return {__shfl_down_sync(0xffffffffu, m.b, d), __shfl_down_sync(0xffffffffu, m.c, d)};
}

// first frame of trajectory s (g is strictly increasing: T_s + 1 >= 1 frames)
__device__ __forceinline__ int64_t first_frame(const int64_t* off, int64_t s) {
  return __ldg(off + s) + s;
}

// async 16-B copy of elements [e, e + 4) of x into shared memory, zero-filled
// past `end` (e < end; x + e is 16-B aligned)
__device__ __forceinline__ void copy4(float* dst, const float* x, int64_t e, int64_t end) {
  const int bytes = e + 4 <= end ? 16 : 4 * (int)(end - e);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)),
               "l"(x + e), "r"(bytes)
               : "memory");
}

constexpr int kMaxGrid = 148 * 8;  // persistent grid bound (partials capacity)

struct Workspace {
  double* partials;     // [grid][3]
  unsigned* counters;   // [1] arrival ticket (zeroed by the index kernel)
  int64_t* seg_first;   // [segs + 1]: first trajectory of each segment
  int64_t* seg_frame;   // [segs + 1]: its first value frame
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

Workspace carve(void* base, int64_t segs) {
  char* p = static_cast<char*>(base);
  Workspace w;
  w.partials = reinterpret_cast<double*>(p);
  size_t o = 3 * sizeof(double) * kMaxGrid;
  w.counters = reinterpret_cast<unsigned*>(p + o);
  o += 16;
  w.seg_first = reinterpret_cast<int64_t*>(p + o);
  o += align_up(sizeof(int64_t) * (size_t)(segs + 1), 16);
  w.seg_frame = reinterpret_cast<int64_t*>(p + o);
  return w;
}

size_t workspace_bytes(int64_t segs) {
  return 3 * sizeof(double) * kMaxGrid + 16 +
         2 * align_up(sizeof(int64_t) * (size_t)(segs + 1), 16);
}

// Segment k = the trajectories whose first value frame g(s) = off[s] + s lies
// in [k kSeg, (k+1) kSeg): seg_first[k] = min{s : g(s) >= k kSeg}.  Thread s
// (0..n_traj; s = n_traj is the end sentinel, g = F) writes the k in
// (g(s-1) / kSeg, g(s) / kSeg]; every k < segs is written exactly once.
__global__ void gae_segment_index_kernel(const int64_t* __restrict__ off, int64_t n_traj,
                                         int64_t segs, Workspace ws) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) ws.counters[0] = 0u;
  if (s > n_traj) return;
  int64_t* seg_first = ws.seg_first;
  int64_t* seg_frame = ws.seg_frame;
  const int64_t g = first_frame(off, s);
  const int64_t k0 = s == 0 ? 0 : first_frame(off, s - 1) / kSeg + 1;
  const int64_t k1 = min(g / kSeg, segs - 1);
  for (int64_t k = k0; k <= k1; ++k) {
    seg_first[k] = s;
    seg_frame[k] = g;
  }
  if (s == n_traj) {
    seg_first[segs] = n_traj;
    seg_frame[segs] = g;
  }
}

// Persistent CTAs stride over the segments.  A segment holds whole
// trajectories, so its right edge is a trajectory end (A = 0 beyond it) and
// no carry crosses CTAs: there is no look-back, ticket or inter-CTA wait.
// The segment is swept right to left in passes of <= kChunk value frames (one
// pass unless a trajectory straddles more than kChunk - kSeg frames past the
// stride), the carry between passes held in shared memory.
//
// Frame-space items: frame f of trajectory s is transition t = f - s, except
// the trajectory's last frame (the bootstrap value), which is the map (0, 0).
// Transition t has delta = r[t] + gamma * v[f+1] * (1 - last * done) - v[f]
// and c = gamma * lam, or 0 at the trajectory's last transition.
__global__ void __launch_bounds__(kThreads, 4)
gae_segment_kernel(const float* __restrict__ rewards, const float* __restrict__ vals,
                   const int64_t* __restrict__ off, const uint8_t* __restrict__ done,
                   int64_t n_frames, float g_hi, float g_lo, float decay,
                   float* __restrict__ adv_out, float* __restrict__ ret_out,
                   int32_t* __restrict__ frame_out, Workspace ws,
                   int64_t segs, int64_t n_transitions, double* __restrict__ sums_out) {
  extern __shared__ __align__(16) float s_dyn[];
  float* s_r = s_dyn;                    // rewards, then advantages
  float* s_v = s_r + kChunk + kPad;      // values [f0, f1], then frame ids
  float* s_ret = s_v + kChunk + kPad + 4;
  int* s_end = reinterpret_cast<int*>(s_ret);  // trajectory ends (| done bit), then returns
  __shared__ Map s_warp[kWarps];
  __shared__ float s_carry;
  __shared__ double s_red[kWarps * 3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double S = 0.0, Q = 0.0, bad = 0.0;
  // persistent: segments blockIdx.x, + gridDim.x, ...; the next segment's
  // bounds are fetched while the current one is processed
  int64_t seg = blockIdx.x;
  int64_t nxt[4] = {0, 0, 0, 0};
  if (seg < segs) {
    nxt[0] = __ldcg(ws.seg_first + seg);
    nxt[1] = __ldcg(ws.seg_first + seg + 1);
    nxt[2] = __ldcg(ws.seg_frame + seg);
    nxt[3] = __ldcg(ws.seg_frame + seg + 1);
  }
  for (; seg < segs; seg += gridDim.x) {
    const int64_t a = nxt[0], b = nxt[1], Fa = nxt[2], Fb = nxt[3];
    if (seg + gridDim.x < segs) {
      const int64_t sn = seg + gridDim.x;
      nxt[0] = __ldcg(ws.seg_first + sn);
      nxt[1] = __ldcg(ws.seg_first + sn + 1);
      nxt[2] = __ldcg(ws.seg_frame + sn);
      nxt[3] = __ldcg(ws.seg_frame + sn + 1);
    }
    if (tid == 0) s_carry = 0.f;
    int64_t f1 = Fb, jb = b;
    while (f1 > Fa) {
      const int64_t f0 = max(Fa, f1 - (int64_t)kChunk);
      int64_t ja = a;
      if (f0 > Fa) {  // long-trajectory pass: last s in [a, jb) with g(s) <= f0
        int64_t lo = a, hi = jb;
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) >> 1;
          if (first_frame(off, mid) <= f0) lo = mid; else hi = mid;
        }
        ja = lo;
      }
      const int nf = (int)(f1 - f0);
      const int nt = (int)(jb - ja);
      const int64_t t_first = f0 - ja;
      const int64_t t_end = (f1 == Fb || f1 == first_frame(off, jb)) ? f1 - jb : f1 - jb + 1;
      // (f1 on a trajectory start: frame f1 - 1 is jb-1's bootstrap, else a transition)
      // stage values [f0, f1] and rewards as aligned 16-B async copies: every
      // load of the pass is in flight at once (one HBM round trip per pass)
      const int64_t vb = f0 & ~3ll, ve = min(f1 + 1, n_frames);
      const int vsh = (int)(f0 - vb);
      const int nv4 = (int)((ve - vb + 3) >> 2);
      const int64_t rb = t_first & ~3ll;
      const int rsh = (int)(t_first - rb);
      const int nr4 = (int)((t_end - rb + 3) >> 2);
  #pragma unroll
      for (int u = 0; u < kVec; ++u) {
        const int q = tid + u * kThreads;
        if (q < nv4) copy4(s_v + 4 * q, vals, vb + 4 * (int64_t)q, ve);
        if (q < nr4) copy4(s_r + 4 * q, rewards, rb + 4 * (int64_t)q, t_end);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      // trajectory frame ends (clipped past the pass: never 'last' inside it)
      for (int j = tid; j < nt; j += kThreads)
        s_end[j] = (int)min(first_frame(off, ja + j + 1) - f0, (int64_t)kChunk + 2) |
                   (__ldg(done + ja + j) ? kDoneBit : 0);
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();

      // pass 1: this thread's items [i0, i0 + kItems).  j0 = trajectories
      // ending before i0 = bootstrap frames before i0, so transition index
      // (relative to t_first) of item i is i - j0 - (bootstraps in [i0, i)).
      const int i0 = tid * kItems;
      int j0 = 0;
      unsigned boot = 0, last = 0, zero_next = 0;
      const unsigned all = (1u << kItems) - 1u;
      const unsigned pad = i0 >= nf ? all
                                    : (i0 + kItems > nf ? all & ~((1u << (nf - i0)) - 1u) : 0u);
      if (i0 < nf) {
        int lo = 0, hi = nt - 1;  // first j with end(j) > i0
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if ((s_end[m] & kEndMask) > i0) hi = m; else lo = m + 1;
        }
        j0 = lo;
        // the (few) trajectory ends touching this thread's window
        for (int j = j0; j < nt; ++j) {
          const int ed = s_end[j], e = ed & kEndMask;
          if (e - 2 >= i0 + kItems) break;
          if (e - 1 < i0 + kItems) boot |= 1u << (e - 1 - i0);
          if (e - 2 >= i0) {
            last |= 1u << (e - 2 - i0);
            if (ed & kDoneBit) zero_next |= 1u << (e - 2 - i0);
          }
        }
      }
      // deltas and the thread's map.  delta = r + gamma v' - v with gamma split
      // into two floats: fma(g_hi, v', -v) is exact before its one rounding, so
      // the result carries fp32 rounding relative to the TD error itself, not to
      // |v| (values much larger than the advantages lose nothing).
      const unsigned cz = boot | last;  // c = 0 (bootstrap and last steps), else decay
      float dl[kItems], vc[kItems];
      Map m{0.f, 1.f};
      if (i0 < nf) {
        float vn = s_v[vsh + min(i0 + kItems, nf)];  // unused when frame f1 is past the end
        // live items hold consecutive transition indices [i0 - j0, i0 - j0 + L)
        int tr = i0 - j0 + kItems - __popc(boot) - __popc(pad);
  #pragma unroll
        for (int k = kItems - 1; k >= 0; --k) {
          const unsigned bit = 1u << k;
          const bool live = !((boot | pad) & bit);
          tr -= live ? 1 : 0;
          const float vi = (pad & bit) ? vn : s_v[vsh + i0 + k];
          const float vnext = (zero_next & bit) ? 0.f : vn;
          const float d = fmaf(g_lo, vnext, fmaf(g_hi, vnext, -vi)) + s_r[rsh + tr];
          dl[k] = live ? d : 0.f;
          vc[k] = vi;
          vn = vi;
          const float c = (pad & bit) ? 1.f : ((cz & bit) ? 0.f : decay);
          m.b = fmaf(c, m.b, dl[k]);
          m.c *= c;
        }
      }
      // suffix scan of the maps: warp, then block (warp 0)
      Map incl = m;
  #pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const Map o = shfl_down_map(incl, d);
        if (lane + d < 32) incl = compose(incl, o);
      }
      Map excl = shfl_down_map(incl, 1);
      if (lane == 31) excl = Map{0.f, 1.f};
      if (lane == 0) s_warp[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const Map w = lane < kWarps ? s_warp[lane] : Map{0.f, 1.f};
        Map wi = w;
  #pragma unroll
        for (int d = 1; d < kWarps; d <<= 1) {
          const Map o = shfl_down_map(wi, d);
          if (lane + d < kWarps) wi = compose(wi, o);
        }
        Map we = shfl_down_map(wi, 1);
        if (lane >= kWarps - 1) we = Map{0.f, 1.f};
        __syncwarp();
        if (lane < kWarps) s_warp[lane] = we;  // exclusive suffix of the warps to the right
      }
      __syncthreads();

      // pass 2: resolve the right-hand context and emit into shared memory
      // (advantages over the reward slots, returns over the trajectory ends,
      // frame ids over the values -- each slot is read back by its owner only)
      const Map right = compose(excl, s_warp[warp]);
      float A = fmaf(right.c, s_carry, right.b);
      float Sf = 0.f, Qf = 0.f;
      int nbad = 0;
      if (i0 < nf) {
        int tr = i0 - j0 + kItems - __popc(boot) - __popc(pad);
  #pragma unroll
        for (int k = kItems - 1; k >= 0; --k) {
          const unsigned bit = 1u << k;
          // bootstrap: c = 0, delta = 0 -> A = 0; padding: c = 1, delta = 0
          const float c = (pad & bit) ? 1.f : ((cz & bit) ? 0.f : decay);
          A = fmaf(c, A, dl[k]);
          if (!((boot | pad) & bit)) {
            --tr;
            const float rf = A + vc[k];
            s_r[rsh + tr] = A;
            s_ret[rsh + tr] = rf;
            reinterpret_cast<int*>(s_v)[rsh + tr] = (int)(f0 + i0 + k);
            Sf += A;
            Qf = fmaf(A, A, Qf);
            nbad += (fabsf(A) <= FLT_MAX && fabsf(rf) <= FLT_MAX) ? 0 : 1;
          }
        }
      }
      S += (double)Sf;
      Q += (double)Qf;
      bad += (double)nbad;
      __syncthreads();
      if (tid == 0) s_carry = A;  // A at frame f0, carried into the pass to the left

      // coalesced write-back of [t_first, t_end): aligned float4 body, scalar edges
      const int64_t body0 = (t_first + 3) & ~3ll, body1 = t_end & ~3ll;
      if (body0 < body1) {
        const int q0 = (int)((body0 - rb) >> 2), q1 = (int)((body1 - rb) >> 2);
        for (int q = q0 + tid; q < q1; q += kThreads) {
          const int64_t e = rb + 4 * (int64_t)q;
          __stcs(reinterpret_cast<float4*>(adv_out + e), reinterpret_cast<const float4*>(s_r)[q]);
          __stcs(reinterpret_cast<float4*>(ret_out + e), reinterpret_cast<const float4*>(s_ret)[q]);
          if (frame_out != nullptr)
            __stcs(reinterpret_cast<int4*>(frame_out + e), reinterpret_cast<const int4*>(s_v)[q]);
        }
        int64_t e = -1;
        if (tid < body0 - t_first) e = t_first + tid;
        else if (tid >= 4 && tid - 4 < t_end - body1) e = body1 + tid - 4;
        if (e >= 0) {
          const int x = (int)(e - rb);
          adv_out[e] = s_r[x];
          ret_out[e] = s_ret[x];
          if (frame_out != nullptr) frame_out[e] = reinterpret_cast<const int*>(s_v)[x];
        }
      } else {
        for (int64_t e = t_first + tid; e < t_end; e += kThreads) {
          const int x = (int)(e - rb);
          adv_out[e] = s_r[x];
          ret_out[e] = s_ret[x];
          if (frame_out != nullptr) frame_out[e] = reinterpret_cast<const int*>(s_v)[x];
        }
      }
      // next pass to the left
      const int64_t gja = first_frame(off, ja);
      jb = gja == f0 ? ja : ja + 1;
      f1 = f0;
      __syncthreads();
    }
  }

  // statistics: one partial per CTA (its segments in a fixed order), then the
  // last CTA to arrive sums the partials in CTA order -- the grid size is
  // fixed for a device, so the pooled sums are bitwise deterministic
  __shared__ bool s_last;
  double v3[3] = {S, Q, bad};
  block_sum_d<3>(v3, s_red);
  if (tid == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) ws.partials[3 * blockIdx.x + c] = v3[c];
    __threadfence();
    s_last = atomicAdd(ws.counters, 1u) == gridDim.x - 1u;
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
  if (n_transitions <= 0 || n_traj <= 0) return 16;
  return workspace_bytes(ceil_div(n_transitions + n_traj, kSeg));
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
       reinterpret_cast<uintptr_t>(ret_out) | reinterpret_cast<uintptr_t>(values_frames) |
       reinterpret_cast<uintptr_t>(frame_of_out)) & 15)
    return fail(kDimension, "GAE needs 16-byte aligned rewards/values/adv/ret/frame buffers");
  const int64_t n_frames = n_transitions + n_traj;
  const int64_t segs = ceil_div(n_frames, kSeg);
  if (workspace_bytes_ < workspace_bytes(segs))
    return fail(kDimension, "GAE workspace too small (%zu < %zu)", workspace_bytes_,
                workspace_bytes(segs));
  Workspace ws = carve(workspace, segs);
  gae_segment_index_kernel<<<(unsigned)ceil_div(n_traj + 1, 256), 256, 0, s>>>(traj_off, n_traj,
                                                                            segs, ws);
  int st = post_launch("gae_segment_index_kernel");
  if (st) return st;
  static int grid = 0;
  if (grid == 0) {
    st = check_cuda(cudaFuncSetAttribute(gae_segment_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSegSmem), "gae smem");
    if (st) return st;
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    st = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gae_segment_kernel,
                                                                  kThreads, kSegSmem),
                    "gae occupancy");
    if (st) return st;
    grid = std::max(1, std::min(per_sm * sms, kMaxGrid));
  }
  gae_segment_kernel<<<(unsigned)std::min<int64_t>(grid, segs), kThreads, kSegSmem, s>>>(
      rewards, values_frames, traj_off, done, n_frames, (float)gamma,
      (float)(gamma - (double)(float)gamma), (float)(gamma * lam), adv_out, ret_out,
      frame_of_out, ws, segs, n_transitions, sums_out);
  return post_launch("gae_segment_kernel");
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
