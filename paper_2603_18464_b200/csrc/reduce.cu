// Fixed-order reductions of per-CTA partials, the step's scalar record, and
// the Adam update.
//
//   reduce_segments  dst[j] = sum_p src[p][j] for up to 16 (src, dst) pairs
//                    in one launch (bias/embedding gradients, value-head
//                    parameter gradients) — float64 accumulation, p order.
//   reduce_f64       sum or max over double partial records.
//   step_finalize    the train_step record (trainer.py:417-464): policy loss
//                    = -sum/m, entropy mean, value MSE, total_loss (:254-256),
//                    ratio/trust/clip diagnostics, and the device-side skip
//                    flag (dropped batch :420-424, non-finite logits or
//                    attention -> DomainError, non-finite grads -> NonFiniteError).
//   adam             bias-corrected Adam (numerics.py:95-126) over one flat
//                    fp32 buffer holding two parameter groups (policy, value),
//                    ping-pong (reads *_in, writes *_out) so a rejected update
//                    leaves the live parameters untouched; float64 math.
#include <math_constants.h>

#include "common.cuh"

namespace accel {
namespace {

constexpr int kMaxSegs = 16;

struct Segs {
  const float* src[kMaxSegs];
  float* dst[kMaxSegs];
  int64_t parts[kMaxSegs];
  int64_t len[kMaxSegs];
  int64_t pitch[kMaxSegs];
};

// Two fixed-order schedules (chosen by the segment's part count only, so every
// launch of a segment sums in the same order):
//  * few parts (< 16): a lane owns 4 columns and adds the parts in order;
//  * many parts (the per-CTA weight-gradient partials): the 16 warps of a block
//    each add a fixed 1/16 of the parts for the same 128 columns (eight rows in
//    flight), then the warp sums are added in warp order.
__device__ __forceinline__ void load4(const float* p, bool vec, int64_t j, int64_t len, double* a) {
  if (vec && j + 3 < len) {
    const float4 x = __ldcs(reinterpret_cast<const float4*>(p + j));
    a[0] += (double)x.x;
    a[1] += (double)x.y;
    a[2] += (double)x.z;
    a[3] += (double)x.w;
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (j + c < len) a[c] += (double)p[j + c];
  }
}

__device__ __forceinline__ void store4(float* p, bool vec, int64_t j, int64_t len, const double* a) {
  if (vec && j + 3 < len) {
    *reinterpret_cast<float4*>(p + j) = make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (j + c < len) p[j + c] = (float)a[c];
  }
}

constexpr int kSegThreads = 512;
constexpr int kSegWarps = kSegThreads / 32;
__global__ void __launch_bounds__(kSegThreads) reduce_segments_kernel(Segs s) {
  __shared__ double red[kSegWarps][32][4];
  const int seg = blockIdx.y;
  const int64_t len = s.len[seg], parts = s.parts[seg], pitch = s.pitch[seg];
  const float* src = s.src[seg];
  float* dst = s.dst[seg];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool vec = ((pitch & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (parts < 16) {
    for (int64_t j = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); j < len;
         j += 4 * (int64_t)gridDim.x * blockDim.x) {
      double a[4] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t p = 0; p < parts; ++p) load4(src + p * pitch, vec, j, len, a);
      store4(dst, vec, j, len, a);
    }
    return;
  }
  const int64_t p0 = warp * parts / kSegWarps, p1 = (warp + 1) * parts / kSegWarps;
  for (int64_t c0 = (int64_t)blockIdx.x * 128; c0 < len; c0 += (int64_t)gridDim.x * 128) {
    const int64_t j = c0 + 4 * lane;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t p = p0;
    for (; p + 8 <= p1; p += 8) {  // eight independent rows in flight
#pragma unroll
      for (int u = 0; u < 8; ++u) load4(src + (p + u) * pitch, vec, j, len, a);
    }
    for (; p < p1; ++p) load4(src + p * pitch, vec, j, len, a);
#pragma unroll
    for (int c = 0; c < 4; ++c) red[warp][lane][c] = a[c];
    __syncthreads();
    if (warp == 0) {
      double t[4] = {0.0, 0.0, 0.0, 0.0};
      for (int w = 0; w < kSegWarps; ++w)
#pragma unroll
        for (int c = 0; c < 4; ++c) t[c] += red[w][lane][c];
      store4(dst, vec, j, len, t);
    }
    __syncthreads();
  }
}

// moments[s] = {sum x, sum x^2, count} of x[off[s]:off[s+1]] (float64, fixed order)
__global__ void __launch_bounds__(256)
segment_moments_kernel(const float* __restrict__ x, const int64_t* __restrict__ off,
                       double* __restrict__ out) {
  __shared__ double s_red[8 * 2];
  const int64_t a = off[blockIdx.x], b = off[blockIdx.x + 1];
  double v[2] = {0.0, 0.0};
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    const double y = x[i];
    v[0] += y;
    v[1] = fma(y, y, v[1]);
  }
  block_sum_d<2>(v, s_red);
  if (threadIdx.x == 0) {
    out[3 * blockIdx.x] = v[0];
    out[3 * blockIdx.x + 1] = v[1];
    out[3 * blockIdx.x + 2] = (double)(b - a);
  }
}

// count of rows r (row index rows[r] of x[*, C]) holding a non-finite value
__global__ void count_nonfinite_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows,
                                            int64_t R, int C, int64_t ld, unsigned* __restrict__ count) {
  unsigned c = 0;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += warps) {
    const int64_t f = rows ? __ldg(rows + r) : r;
    bool bad = false;
    for (int j = lane; j < C; j += 32) bad |= !isfinite(__ldg(x + f * ld + j));
    c += __any_sync(0xffffffffu, bad) && lane == 0;
  }
  if (c) atomicAdd(count, c);
}

__global__ void __launch_bounds__(1024)
reduce_f64_kernel(const double* __restrict__ part, int64_t parts, int width, int mode,
                  double* __restrict__ out) {
  __shared__ double s[1024];
  if (width <= 8) {  // every column at once: thread rows, warp trees, warps in order
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = mode ? -CUDART_INF : 0.0;
    for (int64_t p = threadIdx.x; p < parts; p += blockDim.x) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < width) {
          const double v = __ldg(part + p * width + c);
          acc[c] = mode ? fmax(acc[c], v) : acc[c] + v;
        }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double y = __shfl_down_sync(0xffffffffu, acc[c], o);
        acc[c] = mode ? fmax(acc[c], y) : acc[c] + y;
      }
    double* s8 = s;  // [warp][8]
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 8; ++c) s8[warp * 8 + c] = acc[c];
    __syncthreads();
    if ((int)threadIdx.x < width) {
      double r = mode ? -CUDART_INF : 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        r = mode ? fmax(r, s8[w * 8 + threadIdx.x]) : r + s8[w * 8 + threadIdx.x];
      out[threadIdx.x] = r;
    }
    return;
  }
  for (int c = 0; c < width; ++c) {
    double acc = mode ? -CUDART_INF : 0.0;
    for (int64_t p = threadIdx.x; p < parts; p += blockDim.x) {
      const double v = part[p * width + c];
      acc = mode ? fmax(acc, v) : acc + v;
    }
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o)
        s[threadIdx.x] = mode ? fmax(s[threadIdx.x], s[threadIdx.x + o])
                              : s[threadIdx.x] + s[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = s[0];
    __syncthreads();
  }
}

// Level 1 of the two-level reduction for many partial rows: CTA b folds the
// contiguous rows [b per, (b+1) per) (all <= 8 columns per pass, thread order
// fixed, warp shuffle trees, warps in order) into tmp[b][width].
constexpr int kRedThreads = 256;
constexpr int kRedMaxCtas = 296;

__global__ void __launch_bounds__(kRedThreads)
reduce_f64_rows_kernel(const double* __restrict__ part, int64_t parts, int width, int mode,
                       int64_t per, double* __restrict__ tmp) {
  __shared__ double s[kRedThreads];
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(parts, r0 + per);
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = mode ? -CUDART_INF : 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += kRedThreads) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < width) {
        const double v = __ldg(part + r * width + c);
        acc[c] = mode ? fmax(acc[c], v) : acc[c] + v;
      }
    }
  }
  // warp trees, then the warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_down_sync(0xffffffffu, acc[c], o);
      acc[c] = mode ? fmax(acc[c], y) : acc[c] + y;
    }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < 8; ++c) s[warp * 8 + c] = acc[c];
  __syncthreads();
  if ((int)threadIdx.x < width) {
    double r = mode ? -CUDART_INF : 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w)
      r = mode ? fmax(r, s[w * 8 + threadIdx.x]) : r + s[w * 8 + threadIdx.x];
    tmp[(int64_t)blockIdx.x * width + threadIdx.x] = r;
  }
}

struct FinalizeParams {
  int algo;
  double lambda_v, lambda_h, n_tokens, n_transitions;
};

// loss_sums: token_loss kStat layout; loss_max: [ratio_max, -w_min];
// value_sums: [sum err^2, non-finite v]; bad_counts: [attn, steps, grads]
__global__ void step_finalize_kernel(const double* __restrict__ ls, const double* __restrict__ lm,
                                     const double* __restrict__ vs,
                                     const unsigned* __restrict__ bad_counts,
                                     const double* __restrict__ attn_bad, FinalizeParams p,
                                     double* __restrict__ rec, int* __restrict__ skip) {
  const double excluded = ls[5];
  const double m = p.n_tokens - excluded;
  const bool dropped = !(m > 0.0);
  const double policy_loss = dropped ? 0.0 : -ls[0] / m;
  const double entropy = ls[1] / p.n_tokens;
  const double value_loss = vs[0] / p.n_transitions;
  rec[0] = policy_loss + p.lambda_v * value_loss - p.lambda_h * entropy;
  rec[1] = policy_loss;
  rec[2] = value_loss;
  rec[3] = entropy;
  rec[4] = excluded;
  rec[5] = dropped ? 0.0 : ls[2] / m;                 // ratio_mean
  rec[6] = lm[0];                                     // ratio_max
  rec[7] = dropped ? 0.0 : ls[3] / m;                 // trust_weight_mean
  rec[8] = -lm[1];                                    // trust_weight_min
  rec[9] = dropped ? 0.0 : ls[4] / m;                 // clipped_fraction
  rec[10] = dropped ? 1.0 : 0.0;
  rec[11] = ls[6];                                    // rows with non-finite logits
  rec[12] = ls[7];                                    // tokens outside [0, A)
  rec[13] = attn_bad[0];                              // non-finite attention scores
  rec[14] = (double)bad_counts[0];                    // non-finite gradients
  rec[15] = attn_bad[1] + (double)bad_counts[1];      // step index out of range
  const bool s = dropped || ls[6] > 0 || ls[7] > 0 || attn_bad[0] > 0 || rec[15] > 0 ||
                 bad_counts[0] > 0;
  rec[16] = s ? 1.0 : 0.0;
  *skip = s ? 1 : 0;
}

__global__ void count_nonfinite_kernel(const float* __restrict__ x, int64_t n,
                                       unsigned* __restrict__ count) {
  unsigned c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += !isfinite(x[i]);
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

struct AdamGroup {
  double lr, beta1, beta2, eps, bc1, bc2;  // bc = 1 - beta^t
};

__global__ void adam_kernel(const float* __restrict__ p_in, const float* __restrict__ g,
                            const float* __restrict__ m_in, const float* __restrict__ v_in,
                            float* __restrict__ p_out, float* __restrict__ m_out,
                            float* __restrict__ v_out, int64_t n, int64_t n0, AdamGroup g0,
                            AdamGroup g1, const double* __restrict__ hyper,
                            const int* __restrict__ skip, unsigned* __restrict__ bad) {
  if (*skip) return;
  if (hyper) {  // {group 0, group 1} from device memory (graph-replayable steps)
    g0 = AdamGroup{hyper[0], hyper[1], hyper[2], hyper[3], hyper[4], hyper[5]};
    g1 = AdamGroup{hyper[6], hyper[7], hyper[8], hyper[9], hyper[10], hyper[11]};
  }
  unsigned nb = 0;
  auto one = [&](int64_t i, float pi, float gi, float mi, float vi, float& po, float& mo,
                 float& vo) {
    const AdamGroup& G = i < n0 ? g0 : g1;
    const double gr = gi;
    const double m = G.beta1 * (double)mi + (1.0 - G.beta1) * gr;
    const double v = G.beta2 * (double)vi + (1.0 - G.beta2) * gr * gr;
    const double mh = m / G.bc1, vh = v / G.bc2;
    const double w = (double)pi - G.lr * mh / (sqrt(vh) + G.eps);
    po = (float)w;
    mo = (float)m;
    vo = (float)v;
    nb += !isfinite(po);
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = (n & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(p_in) | reinterpret_cast<uintptr_t>(g) |
                     reinterpret_cast<uintptr_t>(m_in) | reinterpret_cast<uintptr_t>(v_in) |
                     reinterpret_cast<uintptr_t>(p_out) | reinterpret_cast<uintptr_t>(m_out) |
                     reinterpret_cast<uintptr_t>(v_out)) & 15) == 0;
  if (vec) {  // 16-byte loads / stores, the same float64 math per element
    for (int64_t i = 4 * t0; i < n; i += 4 * stride) {
      const float4 p4 = __ldcs(reinterpret_cast<const float4*>(p_in + i));
      const float4 g4 = __ldcs(reinterpret_cast<const float4*>(g + i));
      const float4 m4 = __ldcs(reinterpret_cast<const float4*>(m_in + i));
      const float4 v4 = __ldcs(reinterpret_cast<const float4*>(v_in + i));
      float4 po, mo, vo;
      one(i, p4.x, g4.x, m4.x, v4.x, po.x, mo.x, vo.x);
      one(i + 1, p4.y, g4.y, m4.y, v4.y, po.y, mo.y, vo.y);
      one(i + 2, p4.z, g4.z, m4.z, v4.z, po.z, mo.z, vo.z);
      one(i + 3, p4.w, g4.w, m4.w, v4.w, po.w, mo.w, vo.w);
      *reinterpret_cast<float4*>(p_out + i) = po;
      *reinterpret_cast<float4*>(m_out + i) = mo;
      *reinterpret_cast<float4*>(v_out + i) = vo;
    }
  } else {
    for (int64_t i = t0; i < n; i += stride) {
      float po, mo, vo;
      one(i, p_in[i], g[i], m_in[i], v_in[i], po, mo, vo);
      p_out[i] = po;
      m_out[i] = mo;
      v_out[i] = vo;
    }
  }
  nb = __reduce_add_sync(0xffffffffu, nb);
  if ((threadIdx.x & 31) == 0 && nb) atomicAdd(bad, nb);
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_reduce_segments(const void* const* srcs, void* const* dsts,
                                     const int64_t* parts, const int64_t* lens,
                                     const int64_t* pitches, int nseg, void* stream) {
  if (nseg < 0 || nseg > kMaxSegs) return fail(kDimension, "reduce_segments: 0..16 segments");
  if (nseg == 0) return kOk;
  Segs s{};
  int64_t maxlen = 1;
  for (int i = 0; i < nseg; ++i) {
    if (!srcs[i] || !dsts[i] || parts[i] < 0 || lens[i] < 0)
      return fail(kDimension, "reduce_segments: bad segment %d", i);
    s.src[i] = static_cast<const float*>(srcs[i]);
    s.dst[i] = static_cast<float*>(dsts[i]);
    s.parts[i] = parts[i];
    s.len[i] = lens[i];
    s.pitch[i] = pitches ? pitches[i] : lens[i];
    if (s.pitch[i] < lens[i]) return fail(kDimension, "reduce_segments: pitch < len");
    maxlen = std::max(maxlen, lens[i]);
  }
  // enough CTAs to stream the largest segment at full bandwidth (wide weight
  // gradients are 16.7 M floats at cfg4)
  dim3 grid((unsigned)std::min<int64_t>(ceil_div(maxlen, 128), std::max(64, 2368 / nseg)),
            (unsigned)nseg);
  reduce_segments_kernel<<<grid, kSegThreads, 0, as_stream(stream)>>>(s);
  return post_launch("reduce_segments_kernel");
}

extern "C" size_t accel_reduce_f64_scratch_size(int64_t parts, int width) {
  return (parts > 8192 && width <= 8) ? (size_t)kRedMaxCtas * 8 * sizeof(double) : 0;
}

// single-block reduction width: <= 8 columns run warp trees (any warp count: about
// two rows per thread, short rows on one warp); wider rows keep the 1024-thread tree
static int red_threads(int64_t parts, int width) {
  if (width > 8) return 1024;
  return (int)std::min<int64_t>(1024, std::max<int64_t>(32, ceil_div(ceil_div(parts, 2), 32) * 32));
}

extern "C" int accel_reduce_f64(const double* part, int64_t parts, int width, int mode,
                                double* out, double* scratch, void* stream) {
  if (parts < 0 || width < 1 || (mode != 0 && mode != 1))
    return fail(kDimension, "reduce_f64: bad arguments");
  if (!part || !out) return fail(kDimension, "reduce_f64: NULL buffer");
  cudaStream_t s = as_stream(stream);
  if (parts > 8192 && width <= 8) {  // many rows: two levels, both in a fixed order
    const int ctas = (int)std::min<int64_t>(kRedMaxCtas, ceil_div(parts, 4096));
    const int64_t per = ceil_div(parts, ctas);
    double* tmp = scratch;  // level-1 partials, caller workspace
    if (!tmp) return fail(kDimension, "reduce_f64: %lld rows need the level-1 scratch",
                          (long long)parts);
    int st;
    reduce_f64_rows_kernel<<<ctas, kRedThreads, 0, s>>>(part, parts, width, mode, per, tmp);
    if ((st = post_launch("reduce_f64_rows_kernel"))) return st;
    reduce_f64_kernel<<<1, red_threads(ctas, width), 0, s>>>(tmp, ctas, width, mode, out);
    return post_launch("reduce_f64_kernel");
  }
  reduce_f64_kernel<<<1, red_threads(parts, width), 0, s>>>(part, parts, width, mode, out);
  return post_launch("reduce_f64_kernel");
}

extern "C" int accel_step_finalize(const double* loss_sums, const double* loss_max,
                                   const double* value_sums, const unsigned* bad_counts,
                                   const double* attn_bad, int algo, double lambda_v,
                                   double lambda_h, double n_tokens, double n_transitions,
                                   double* record, int* skip, void* stream) {
  if (!loss_sums || !loss_max || !value_sums || !bad_counts || !attn_bad || !record || !skip)
    return fail(kDimension, "step_finalize: NULL buffer");
  FinalizeParams p{algo, lambda_v, lambda_h, n_tokens, n_transitions};
  step_finalize_kernel<<<1, 1, 0, as_stream(stream)>>>(loss_sums, loss_max, value_sums,
                                                       bad_counts, attn_bad, p, record, skip);
  return post_launch("step_finalize_kernel");
}

extern "C" int accel_count_nonfinite(const float* x, int64_t n, unsigned* count, void* stream) {
  if (n < 0 || !count) return fail(kDimension, "count_nonfinite: bad arguments");
  if (n == 0) return kOk;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)kNumSMs * 4);
  count_nonfinite_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, n, count);
  return post_launch("count_nonfinite_kernel");
}

extern "C" int accel_adam(const float* p_in, const float* g, const float* m_in, const float* v_in,
                          float* p_out, float* m_out, float* v_out, int64_t n, int64_t n0,
                          const double* group0, const double* group1, const int* skip,
                          unsigned* bad, void* stream) {
  if (n < 0 || n0 < 0 || n0 > n) return fail(kDimension, "adam: bad sizes");
  if (!group0 || !group1 || !skip || !bad) return fail(kDimension, "adam: NULL buffer");
  AdamGroup a{group0[0], group0[1], group0[2], group0[3], group0[4], group0[5]};
  AdamGroup b{group1[0], group1[1], group1[2], group1[3], group1[4], group1[5]};
  for (const AdamGroup* G : {&a, &b}) {
    if (!(G->bc1 > 0 && G->bc2 > 0)) return fail(kDomain, "adam: bias correction must be > 0");
  }
  if (n == 0) return kOk;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 1024), (int64_t)kNumSMs * 16);
  adam_kernel<<<grid, 256, 0, as_stream(stream)>>>(p_in, g, m_in, v_in, p_out, m_out, v_out, n,
                                                   n0, a, b, nullptr, skip, bad);
  return post_launch("adam_kernel");
}

// accel_adam with the two groups' {lr, beta1, beta2, eps, 1 - beta1^t, 1 - beta2^t}
// read from DEVICE memory (hyper f64[12]) at run time, so a captured CUDA graph
// replays successive optimizer steps (the host refreshes hyper before each replay).
extern "C" int accel_adam_dev(const float* p_in, const float* g, const float* m_in,
                              const float* v_in, float* p_out, float* m_out, float* v_out,
                              int64_t n, int64_t n0, const double* hyper, const int* skip,
                              unsigned* bad, void* stream) {
  if (n < 0 || n0 < 0 || n0 > n) return fail(kDimension, "adam: bad sizes");
  if (!hyper || !skip || !bad) return fail(kDimension, "adam: NULL buffer");
  if (n == 0) return kOk;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 1024), (int64_t)kNumSMs * 16);
  adam_kernel<<<grid, 256, 0, as_stream(stream)>>>(p_in, g, m_in, v_in, p_out, m_out, v_out, n,
                                                   n0, AdamGroup{}, AdamGroup{}, hyper, skip, bad);
  return post_launch("adam_kernel");
}

extern "C" int accel_segment_moments(const float* x, const int64_t* off, int64_t nseg,
                                     double* out, void* stream) {
  if (nseg < 0 || !x || !off || !out) return fail(kDimension, "segment_moments: bad arguments");
  if (nseg == 0) return kOk;
  segment_moments_kernel<<<(unsigned)nseg, 256, 0, as_stream(stream)>>>(x, off, out);
  return post_launch("segment_moments_kernel");
}

extern "C" int accel_count_nonfinite_rows(const float* x, const int32_t* rows, int64_t R, int C,
                                          int64_t ld, unsigned* count, void* stream) {
  if (R < 0 || C < 1 || ld < C || !x || !count)
    return fail(kDimension, "count_nonfinite_rows: bad arguments");
  if (R == 0) return kOk;
  const int grid = (int)std::min<int64_t>(ceil_div(R, 8), (int64_t)kNumSMs * 8);
  count_nonfinite_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, rows, R, C, ld, count);
  return post_launch("count_nonfinite_rows_kernel");
}

// ---- 3xTF32 operand split for the wide-layer library GEMMs ------------------
// hi = x rounded to TF32 (10-bit mantissa, round-half-away on the magnitude
// bits), lo = x - hi (exact in fp32).  A product then runs as three TF32
// tensor-core GEMMs, hi.hi + hi.lo + lo.hi, accumulated in fp32: about fp32
// accuracy (the dropped lo.lo term and the TF32 truncation of lo are below
// 2^-20 relative) at tensor-core rate.  Non-finite inputs pass through hi.
namespace accel {
namespace {
__global__ void split_tf32_kernel(const float4* __restrict__ x, int64_t n4, float4* __restrict__ hi,
                                  float4* __restrict__ lo) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = x[i];
    float h[4];
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned b = __float_as_uint(e[j]);
      const bool fin = (b & 0x7f800000u) != 0x7f800000u;
      h[j] = fin ? __uint_as_float((b + 0x1000u) & 0xffffe000u) : e[j];
    }
    hi[i] = make_float4(h[0], h[1], h[2], h[3]);
    lo[i] = make_float4(isfinite(e[0]) ? e[0] - h[0] : 0.f, isfinite(e[1]) ? e[1] - h[1] : 0.f,
                        isfinite(e[2]) ? e[2] - h[2] : 0.f, isfinite(e[3]) ? e[3] - h[3] : 0.f);
  }
}
}  // namespace
}  // namespace accel

extern "C" int accel_split_tf32(const float* x, int64_t n, float* hi, float* lo, void* stream) {
  using namespace accel;
  if (n < 0 || (n & 3)) return fail(kDimension, "split_tf32: n must be a multiple of 4");
  if (n == 0) return kOk;
  if (!x || !hi || !lo) return fail(kDimension, "split_tf32: NULL buffer");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) |
       reinterpret_cast<uintptr_t>(lo)) & 15)
    return fail(kDimension, "split_tf32: buffers must be 16B aligned");
  const int64_t n4 = n / 4;
  const int grid = (int)std::min<int64_t>(ceil_div(n4, 256), (int64_t)kNumSMs * 8);
  split_tf32_kernel<<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(x), n4,
                                                         reinterpret_cast<float4*>(hi),
                                                         reinterpret_cast<float4*>(lo));
  return post_launch("split_tf32_kernel");
}
