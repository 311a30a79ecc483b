// Value head: attention pooling over detached (h1, h2), step embedding,
// tanh MLP to a scalar; MSE loss and its backward.
//
// Reference: ValueHead.forward_batch (models.py:273-290), backward_batch
// (models.py:292-314), value loss in train_step (trainer.py:438-443), and
// revaluation `state_values_batch` (models.py:411-415, trainer.py:352-356).
// The two GEMMs u@W0v^T and dzm^T@u / dzm@W0v are library GEMMs; the
// row-wise parts are here:
//   value_pool        e_j = h_j.w_attn + b, alpha = softmax(e), u = sum_j alpha_j h_j + e_step[t]
//   value_head        m = tanh(z + b0v), v = w1v.m + b1v; err, dv = lambda_v 2 err / N;
//                     dzm = dv w1v (1 - m^2); partial sums for dw1v, db0v, db1v, sum err^2
//   value_attn_grad   dalpha_j = du.h_j; de = alpha (dalpha - sum alpha dalpha)
//   value_attn_wgrad  dw_attn = sum_i sum_j de_ij h_ij (column layout)
// Rows may be transitions (row_frame maps them to frame rows of h1/h2/steps)
// or frames (row_frame == NULL).
#include "common.cuh"

namespace accel {
namespace {

// MSE (trainer.py:438-443) or, with v_old, the PPO value-clip loss of the north
// star: max((v - R)^2, (v_old + clip(v - v_old, +-eps) - R)^2).  Returns the loss
// term (float64) and dL/dv.
__device__ __forceinline__ double value_loss_term(float v, float t, const float* v_old, int64_t r,
                                                  float eps, double& g) {
  const double e = (double)v - (double)t;
  if (!v_old) {
    g = 2.0 * e;
    return e * e;
  }
  const float vo = __ldg(v_old + r);
  const float d = v - vo;
  const double vc = (double)vo + (double)fminf(fmaxf(d, -eps), eps);
  const double ec = vc - (double)t;
  const double l1 = e * e, l2 = ec * ec;
  g = l1 >= l2 ? 2.0 * e : (fabsf(d) < eps ? 2.0 * ec : 0.0);
  return fmax(l1, l2);
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxHPL = 4;  // mlp_hidden <= 128

__global__ void __launch_bounds__(kThreads)
value_pool_kernel(const float* __restrict__ h1, const float* __restrict__ h2,
                  const int32_t* __restrict__ row_frame, const int32_t* __restrict__ steps,
                  int64_t R, int D, int n_steps, const float* __restrict__ w_attn,
                  const float* __restrict__ b_attn, const float* __restrict__ e_step,
                  float* __restrict__ U, float* __restrict__ alpha, double* __restrict__ bad_part) {
  __shared__ double s_bad[kWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float b = __ldg(b_attn);
  double bad_attn = 0.0, bad_step = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kWarps;
  for (int64_t r = (int64_t)blockIdx.x * kWarps + warp; r < R; r += stride) {
    const int64_t f = row_frame ? __ldg(row_frame + r) : r;
    const float* a = h1 + f * D;
    const float* c = h2 + f * D;
    float e0 = 0.f, e1 = 0.f;
    for (int d = lane; d < D; d += 32) {
      const float w = __ldg(w_attn + d);
      e0 = fmaf(__ldg(a + d), w, e0);
      e1 = fmaf(__ldg(c + d), w, e1);
    }
    e0 = warp_sum(e0) + b;
    e1 = warp_sum(e1) + b;
    const bool bad = !isfinite(e0) || !isfinite(e1);
    const float mx = fmaxf(e0, e1);
    const float x0 = __expf(e0 - mx), x1 = __expf(e1 - mx);
    const float inv = 1.f / (x0 + x1);
    const float a0 = x0 * inv, a1 = x1 * inv;
    int st = __ldg(steps + f);
    const bool bst = st < 0 || st >= n_steps;
    st = min(max(st, 0), n_steps - 1);
    const float* es = e_step + (int64_t)st * D;
    float* u = U + r * D;
    for (int d = lane; d < D; d += 32) u[d] = fmaf(a0, __ldg(a + d), fmaf(a1, __ldg(c + d), __ldg(es + d)));
    if (lane == 0) {
      alpha[2 * r] = a0;
      alpha[2 * r + 1] = a1;
    }
    bad_attn += bad;
    bad_step += bst;
  }
  if (lane == 0) {
    s_bad[warp][0] = bad_attn;
    s_bad[warp][1] = bad_step;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < kWarps; ++w) {
      x += s_bad[w][0];
      y += s_bad[w][1];
    }
    bad_part[2 * (int64_t)blockIdx.x] = x;
    bad_part[2 * (int64_t)blockIdx.x + 1] = y;
  }
}

// Vectorized variant for D = 4 * LPR (LPR lanes per row, 32 / LPR rows per
// warp, two row groups in flight): same arithmetic as value_pool_kernel.
template <int LPR>
__global__ void __launch_bounds__(kThreads)
value_pool4_kernel(const float* __restrict__ h1, const float* __restrict__ h2,
                   const int32_t* __restrict__ row_frame, const int32_t* __restrict__ steps,
                   int64_t R, int n_steps, const float* __restrict__ w_attn,
                   const float* __restrict__ b_attn, const float* __restrict__ e_step,
                   float* __restrict__ U, float* __restrict__ alpha, double* __restrict__ bad_part) {
  constexpr int RPW = 32 / LPR;
  constexpr int D4 = LPR;
  __shared__ double s_bad[kWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sl = lane % LPR;
  const float4 w = __ldg(reinterpret_cast<const float4*>(w_attn) + sl);
  const float b = __ldg(b_attn);
  int bad_attn = 0, bad_step = 0;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t step = (int64_t)gridDim.x * kWarps * RPW * 2;
  for (int64_t r0 = gw * RPW * 2; r0 < R; r0 += step) {
    int64_t r[2] = {r0 + slot, r0 + RPW + slot};
    float4 a[2], c[2];
    float e0[2], e1[2];
    int64_t f[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const bool ok = r[q] < R;
      f[q] = ok ? (row_frame ? __ldg(row_frame + r[q]) : r[q]) : 0;
      a[q] = __ldg(reinterpret_cast<const float4*>(h1 + f[q] * 4 * D4) + sl);
      c[q] = __ldg(reinterpret_cast<const float4*>(h2 + f[q] * 4 * D4) + sl);
      e0[q] = a[q].x * w.x + a[q].y * w.y + a[q].z * w.z + a[q].w * w.w;
      e1[q] = c[q].x * w.x + c[q].y * w.y + c[q].z * w.z + c[q].w * w.w;
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        e0[q] += __shfl_xor_sync(0xffffffffu, e0[q], o);
        e1[q] += __shfl_xor_sync(0xffffffffu, e1[q], o);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (r[q] >= R) continue;
      const float x0 = e0[q] + b, x1 = e1[q] + b;
      const bool bad = !isfinite(x0) || !isfinite(x1);
      const float mx = fmaxf(x0, x1);
      const float p0 = __expf(x0 - mx), p1 = __expf(x1 - mx);
      const float inv = 1.f / (p0 + p1);
      const float a0 = p0 * inv, a1 = p1 * inv;
      int st = __ldg(steps + f[q]);
      const bool bst = st < 0 || st >= n_steps;
      st = min(max(st, 0), n_steps - 1);
      const float4 es = __ldg(reinterpret_cast<const float4*>(e_step + (int64_t)st * 4 * D4) + sl);
      float4 u;
      u.x = fmaf(a0, a[q].x, fmaf(a1, c[q].x, es.x));
      u.y = fmaf(a0, a[q].y, fmaf(a1, c[q].y, es.y));
      u.z = fmaf(a0, a[q].z, fmaf(a1, c[q].z, es.z));
      u.w = fmaf(a0, a[q].w, fmaf(a1, c[q].w, es.w));
      reinterpret_cast<float4*>(U + r[q] * 4 * D4)[sl] = u;
      if (sl == 0) {
        alpha[2 * r[q]] = a0;
        alpha[2 * r[q] + 1] = a1;
        bad_attn += bad;
        bad_step += bst;
      }
    }
  }
  bad_attn = __reduce_add_sync(0xffffffffu, bad_attn);
  bad_step = __reduce_add_sync(0xffffffffu, bad_step);
  if (lane == 0) {
    s_bad[warp][0] = bad_attn;
    s_bad[warp][1] = bad_step;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) {
      x += s_bad[w2][0];
      y += s_bad[w2][1];
    }
    bad_part[2 * (int64_t)blockIdx.x] = x;
    bad_part[2 * (int64_t)blockIdx.x + 1] = y;
  }
}

// Vectorized attention backward for D = 4 * LPR (see value_attn_grad_kernel).
template <int LPR>
__global__ void __launch_bounds__(kThreads)
value_attn_grad4_kernel(const float* __restrict__ dU, const float* __restrict__ h1,
                        const float* __restrict__ h2, const int32_t* __restrict__ row_frame,
                        const float* __restrict__ alpha, int64_t R, float* __restrict__ de,
                        float* __restrict__ part) {
  constexpr int RPW = 32 / LPR;
  constexpr int D4 = LPR;
  __shared__ float s_b[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sl = lane % LPR;
  float gb = 0.f;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t step = (int64_t)gridDim.x * kWarps * RPW * 2;
  for (int64_t r0 = gw * RPW * 2; r0 < R; r0 += step) {
    int64_t r[2] = {r0 + slot, r0 + RPW + slot};
    float d0[2], d1[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const bool ok = r[q] < R;
      const int64_t rr = ok ? r[q] : 0;
      const int64_t f = row_frame ? __ldg(row_frame + rr) : rr;
      const float4 g = __ldg(reinterpret_cast<const float4*>(dU + rr * 4 * D4) + sl);
      const float4 a = __ldg(reinterpret_cast<const float4*>(h1 + f * 4 * D4) + sl);
      const float4 c = __ldg(reinterpret_cast<const float4*>(h2 + f * 4 * D4) + sl);
      d0[q] = g.x * a.x + g.y * a.y + g.z * a.z + g.w * a.w;
      d1[q] = g.x * c.x + g.y * c.y + g.z * c.z + g.w * c.w;
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        d0[q] += __shfl_xor_sync(0xffffffffu, d0[q], o);
        d1[q] += __shfl_xor_sync(0xffffffffu, d1[q], o);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (r[q] >= R || sl != 0) continue;
      const float a0 = __ldg(alpha + 2 * r[q]), a1 = __ldg(alpha + 2 * r[q] + 1);
      const float s = a0 * d0[q] + a1 * d1[q];
      const float x0 = a0 * (d0[q] - s), x1 = a1 * (d1[q] - s);
      de[2 * r[q]] = x0;
      de[2 * r[q] + 1] = x1;
      gb += x0 + x1;
    }
  }
  // fixed-order warp reduction (xor butterfly), then warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gb += __shfl_xor_sync(0xffffffffu, gb, o);
  if (lane == 0) s_b[warp] = gb;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int w2 = 0; w2 < kWarps; ++w2) a += s_b[w2];
    part[blockIdx.x] = a;
  }
}

// Fused attention backward (value_attn_grad4 + value_attn_wgrad4 in one pass):
// the row's h1 / h2 chunks are already in registers for dalpha, so the score
// gradients de feed the dw_attn sums directly instead of a second pass over
// h1, h2 and de.  Every lane of a row group holds the butterfly totals, so
// each accumulates de_0 h1 + de_1 h2 for its float4 of columns; the block's
// lanes are then summed in thread order (deterministic for a fixed grid).
// wpart f32[grid][4 LPR], bpart f32[grid]; de (optional) f32[R, 2].
template <int LPR>
__global__ void __launch_bounds__(kThreads)
value_attn_bwd4_kernel(const float* __restrict__ dU, const float* __restrict__ h1,
                       const float* __restrict__ h2, const int32_t* __restrict__ row_frame,
                       const float* __restrict__ alpha, int64_t R, float* __restrict__ de,
                       float* __restrict__ bpart, float* __restrict__ wpart) {
  constexpr int RPW = 32 / LPR;
  constexpr int D4 = LPR;
  __shared__ float s_b[kWarps];
  __shared__ float4 s_w[kThreads];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / LPR, sl = lane % LPR;
  float gb = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t step = (int64_t)gridDim.x * kWarps * RPW * 2;
  for (int64_t r0 = gw * RPW * 2; r0 < R; r0 += step) {
    int64_t r[2] = {r0 + slot, r0 + RPW + slot};
    float d0[2], d1[2];
    float4 a[2], c[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const bool ok = r[q] < R;
      const int64_t rr = ok ? r[q] : 0;
      const int64_t f = row_frame ? __ldg(row_frame + rr) : rr;
      const float4 g = __ldg(reinterpret_cast<const float4*>(dU + rr * 4 * D4) + sl);
      a[q] = __ldg(reinterpret_cast<const float4*>(h1 + f * 4 * D4) + sl);
      c[q] = __ldg(reinterpret_cast<const float4*>(h2 + f * 4 * D4) + sl);
      d0[q] = g.x * a[q].x + g.y * a[q].y + g.z * a[q].z + g.w * a[q].w;
      d1[q] = g.x * c[q].x + g.y * c[q].y + g.z * c[q].z + g.w * c[q].w;
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        d0[q] += __shfl_xor_sync(0xffffffffu, d0[q], o);
        d1[q] += __shfl_xor_sync(0xffffffffu, d1[q], o);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (r[q] >= R) continue;
      const float a0 = __ldg(alpha + 2 * r[q]), a1 = __ldg(alpha + 2 * r[q] + 1);
      const float s = a0 * d0[q] + a1 * d1[q];
      const float x0 = a0 * (d0[q] - s), x1 = a1 * (d1[q] - s);
      acc.x = fmaf(x0, a[q].x, fmaf(x1, c[q].x, acc.x));
      acc.y = fmaf(x0, a[q].y, fmaf(x1, c[q].y, acc.y));
      acc.z = fmaf(x0, a[q].z, fmaf(x1, c[q].z, acc.z));
      acc.w = fmaf(x0, a[q].w, fmaf(x1, c[q].w, acc.w));
      if (sl == 0) {
        if (de) {
          de[2 * r[q]] = x0;
          de[2 * r[q] + 1] = x1;
        }
        gb += x0 + x1;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gb += __shfl_xor_sync(0xffffffffu, gb, o);
  if (lane == 0) s_b[warp] = gb;
  s_w[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int w2 = 0; w2 < kWarps; ++w2) b += s_b[w2];
    bpart[blockIdx.x] = b;
  }
  if (threadIdx.x < D4) {  // column group t: the block's row lanes in thread order
    float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int u = threadIdx.x; u < kThreads; u += D4) {
      const float4 y = s_w[u];
      w.x += y.x; w.y += y.y; w.z += y.z; w.w += y.w;
    }
    reinterpret_cast<float4*>(wpart + (int64_t)blockIdx.x * D4 * 4)[threadIdx.x] = w;
  }
}

// part layout per block: [dw1v (H) | db0v (H) | db1v (1)]; dpart: [sum err^2, non-finite v]
__global__ void __launch_bounds__(kThreads)
value_head_kernel(float* __restrict__ zm, const int32_t* __restrict__ row_frame,
                  const float* __restrict__ b0v,
                  const float* __restrict__ w1v, const float* __restrict__ b1v, int64_t R, int H,
                  const float* __restrict__ targets, const float* __restrict__ v_old, float vclip,
                  float lambda_v, double inv_n, float* __restrict__ values_out,
                  float* __restrict__ part, double* __restrict__ dpart) {
  __shared__ float s_part[kWarps][2 * 32 * kMaxHPL + 1];
  __shared__ double s_err[kWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float bias1 = __ldg(b1v);
  float bz[kMaxHPL], w1[kMaxHPL], gw1[kMaxHPL], gb0[kMaxHPL];
#pragma unroll
  for (int j = 0; j < kMaxHPL; ++j) {
    const int h = lane + 32 * j;
    bz[j] = h < H ? __ldg(b0v + h) : 0.f;
    w1[j] = h < H ? __ldg(w1v + h) : 0.f;
    gw1[j] = 0.f;
    gb0[j] = 0.f;
  }
  float gb1 = 0.f;
  double err2 = 0.0, bad = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kWarps;
  for (int64_t r = (int64_t)blockIdx.x * kWarps + warp; r < R; r += stride) {
    float m[kMaxHPL];
    float acc = 0.f;
    const int64_t zr = row_frame ? __ldg(row_frame + r) : r;
#pragma unroll
    for (int j = 0; j < kMaxHPL; ++j) {
      const int h = lane + 32 * j;
      m[j] = h < H ? tanhf(zm[zr * H + h] + bz[j]) : 0.f;
      acc = fmaf(w1[j], m[j], acc);
    }
    const float v = warp_sum(acc) + bias1;
    if (values_out && lane == 0) values_out[r] = v;
    if (targets) {
      double gl;
      err2 += value_loss_term(v, __ldg(targets + r), v_old, r, vclip, gl);
      const float dv = (float)((double)lambda_v * gl * inv_n);
      bad += !isfinite(v);
      gb1 += dv;
#pragma unroll
      for (int j = 0; j < kMaxHPL; ++j) {
        const int h = lane + 32 * j;
        if (h < H) {
          const float g = dv * w1[j] * (1.f - m[j] * m[j]);
          zm[zr * H + h] = g;
          gw1[j] = fmaf(dv, m[j], gw1[j]);
          gb0[j] += g;
        }
      }
    }
  }
  if (!targets) return;
#pragma unroll
  for (int j = 0; j < kMaxHPL; ++j) {
    s_part[warp][lane + 32 * j] = gw1[j];
    s_part[warp][32 * kMaxHPL + lane + 32 * j] = gb0[j];
  }
  if (lane == 0) {
    s_part[warp][2 * 32 * kMaxHPL] = gb1;
    s_err[warp][0] = err2;
    s_err[warp][1] = bad;
  }
  __syncthreads();
  float* out = part + (int64_t)blockIdx.x * (2 * H + 1);
  for (int e = threadIdx.x; e < 2 * H + 1; e += kThreads) {
    int src;
    if (e < H) src = e;
    else if (e < 2 * H) src = 32 * kMaxHPL + (e - H);
    else src = 2 * 32 * kMaxHPL;
    float a = 0.f;
    for (int w = 0; w < kWarps; ++w) a += s_part[w][src];
    out[e] = a;
  }
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < kWarps; ++w) {
      x += s_err[w][0];
      y += s_err[w][1];
    }
    dpart[2 * (int64_t)blockIdx.x] = x;
    dpart[2 * (int64_t)blockIdx.x + 1] = y;
  }
}

// de[r] = alpha * (dalpha - sum alpha dalpha); part[blk] = sum of de over rows (db_attn)
__global__ void __launch_bounds__(kThreads)
value_attn_grad_kernel(const float* __restrict__ dU, const float* __restrict__ h1,
                       const float* __restrict__ h2, const int32_t* __restrict__ row_frame,
                       const float* __restrict__ alpha, int64_t R, int D, float* __restrict__ de,
                       float* __restrict__ part) {
  __shared__ float s_b[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float gb = 0.f;
  const int64_t stride = (int64_t)gridDim.x * kWarps;
  for (int64_t r = (int64_t)blockIdx.x * kWarps + warp; r < R; r += stride) {
    const int64_t f = row_frame ? __ldg(row_frame + r) : r;
    const float* du = dU + r * D;
    float d0 = 0.f, d1 = 0.f;
    for (int d = lane; d < D; d += 32) {
      const float g = __ldg(du + d);
      d0 = fmaf(g, __ldg(h1 + f * D + d), d0);
      d1 = fmaf(g, __ldg(h2 + f * D + d), d1);
    }
    d0 = warp_sum(d0);
    d1 = warp_sum(d1);
    const float a0 = __ldg(alpha + 2 * r), a1 = __ldg(alpha + 2 * r + 1);
    const float s = a0 * d0 + a1 * d1;
    const float e0 = a0 * (d0 - s), e1 = a1 * (d1 - s);
    if (lane == 0) {
      de[2 * r] = e0;
      de[2 * r + 1] = e1;
    }
    gb += e0 + e1;
  }
  if (lane == 0) s_b[warp] = gb;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int w = 0; w < kWarps; ++w) a += s_b[w];
    part[blockIdx.x] = a;
  }
}

// part[blk][d] = sum over the block's rows of de0 h1[f, d] + de1 h2[f, d]
__global__ void __launch_bounds__(kThreads)
value_attn_wgrad_kernel(const float* __restrict__ de, const float* __restrict__ h1,
                        const float* __restrict__ h2, const int32_t* __restrict__ row_frame,
                        int64_t R, int D, float* __restrict__ part) {
  extern __shared__ float s_acc[];
  const int span = (D <= kThreads && kThreads % D == 0) ? D : kThreads;
  const int sub = kThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  const int64_t per = ceil_div(R, (int64_t)gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(R, r0 + per);
  for (int d0 = 0; d0 < D; d0 += span) {
    const int d = d0 + lc;
    float acc = 0.f;
    if (d < D)
      for (int64_t r = r0 + lr; r < r1; r += sub) {
        const int64_t f = row_frame ? __ldg(row_frame + r) : r;
        acc = fmaf(__ldg(de + 2 * r), __ldg(h1 + f * D + d),
                   fmaf(__ldg(de + 2 * r + 1), __ldg(h2 + f * D + d), acc));
      }
    s_acc[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < span && d0 + threadIdx.x < D) {
      float a = 0.f;
      for (int s = 0; s < sub; ++s) a += s_acc[s * span + threadIdx.x];
      part[(int64_t)blockIdx.x * D + d0 + threadIdx.x] = a;
    }
    __syncthreads();
  }
}

// value_head with LPR lanes per row (CPL = H / LPR columns each, float4 I/O):
// the row's dot product is an LPR-lane reduction instead of a full-warp one,
// the column sums stay in registers, tanh uses one ex2 + one fast divide.
template <int LPR, int CPL>
__global__ void __launch_bounds__(kThreads)
value_head4_kernel(float* __restrict__ zm, const int32_t* __restrict__ row_frame,
                   const float* __restrict__ b0v,
                   const float* __restrict__ w1v, const float* __restrict__ b1v, int64_t R,
                   const float* __restrict__ targets, const float* __restrict__ v_old,
                   float vclip, float lambda_v, double inv_n, float* __restrict__ values_out,
                   float* __restrict__ part, double* __restrict__ dpart) {
  constexpr int H = LPR * CPL, RPW = 32 / LPR, Q = CPL / 4;
  __shared__ float s_part[kWarps][2 * H + 1];
  __shared__ double s_err[kWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rsub = lane / LPR, lc = lane % LPR;
  const float bias1 = __ldg(b1v);
  float bz[CPL], w1[CPL], gw1[CPL], gb0[CPL];
#pragma unroll
  for (int j = 0; j < CPL; ++j) {
    bz[j] = __ldg(b0v + lc * CPL + j);
    w1[j] = __ldg(w1v + lc * CPL + j);
    gw1[j] = 0.f;
    gb0[j] = 0.f;
  }
  float gb1 = 0.f;
  double err2 = 0.0, bad = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kWarps * RPW;
  for (int64_t r = ((int64_t)blockIdx.x * kWarps + warp) * RPW + rsub; r - rsub < R; r += stride) {
    const bool act = r < R;
    float m[CPL];
    float acc = 0.f;
    const int64_t zr = act && row_frame ? __ldg(row_frame + r) : r;
    float4* row = reinterpret_cast<float4*>(zm + zr * H + lc * CPL);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const float4 z = act ? row[q] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float x = zz[u] + bz[4 * q + u];
        const float t = __expf(2.f * x);
        m[4 * q + u] = 1.f - __fdividef(2.f, t + 1.f);
        acc = fmaf(w1[4 * q + u], m[4 * q + u], acc);
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const float v = acc + bias1;
    if (act && values_out && lc == 0) values_out[r] = v;
    if (targets && act) {
      double gl;
      const double lterm = value_loss_term(v, __ldg(targets + r), v_old, r, vclip, gl);
      const float dv = (float)((double)lambda_v * gl * inv_n);
      if (lc == 0) {
        err2 += lterm;
        bad += !isfinite(v);
        gb1 += dv;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        float g4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          g4[u] = dv * w1[j] * (1.f - m[j] * m[j]);
          gw1[j] = fmaf(dv, m[j], gw1[j]);
          gb0[j] += g4[u];
        }
        row[q] = make_float4(g4[0], g4[1], g4[2], g4[3]);
      }
    }
  }
  if (!targets) return;
  // rows of the warp -> one set of column sums (fixed xor order), then warps in order
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      gw1[j] += __shfl_xor_sync(0xffffffffu, gw1[j], o);
      gb0[j] += __shfl_xor_sync(0xffffffffu, gb0[j], o);
    }
  }
  gb1 = warp_sum(gb1);
  err2 = warp_sum_d(err2);
  bad = warp_sum_d(bad);
  if (rsub == 0) {
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      s_part[warp][lc * CPL + j] = gw1[j];
      s_part[warp][H + lc * CPL + j] = gb0[j];
    }
  }
  if (lane == 0) {
    s_part[warp][2 * H] = gb1;
    s_err[warp][0] = err2;
    s_err[warp][1] = bad;
  }
  __syncthreads();
  float* out = part + (int64_t)blockIdx.x * (2 * H + 1);
  for (int e = threadIdx.x; e < 2 * H + 1; e += kThreads) {
    float a = 0.f;
    for (int w = 0; w < kWarps; ++w) a += s_part[w][e];
    out[e] = a;
  }
  if (threadIdx.x < 2) {
    double a = 0.0;
    for (int w = 0; w < kWarps; ++w) a += s_err[w][threadIdx.x];
    dpart[(int64_t)blockIdx.x * 2 + threadIdx.x] = a;
  }
}

// dw_attn partials with float4 columns and four independent row accumulators
template <int D4>
__global__ void __launch_bounds__(kThreads)
value_attn_wgrad4_kernel(const float* __restrict__ de, const float4* __restrict__ h1,
                         const float4* __restrict__ h2, const int32_t* __restrict__ row_frame,
                         int64_t R, float* __restrict__ part) {
  constexpr int SUB = kThreads / D4;
  __shared__ float4 s_acc[kThreads];
  const int lr = threadIdx.x / D4, lc = threadIdx.x % D4;
  const int64_t per = ceil_div(R, (int64_t)gridDim.x);
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(R, r0 + per);
  float4 acc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  auto one = [&](int64_t r, float4& a) {
    const int64_t f = row_frame ? __ldg(row_frame + r) : r;
    const float2 d = __ldg(reinterpret_cast<const float2*>(de) + r);
    const float4 x = __ldg(h1 + f * D4 + lc), y = __ldg(h2 + f * D4 + lc);
    a.x = fmaf(d.x, x.x, fmaf(d.y, y.x, a.x));
    a.y = fmaf(d.x, x.y, fmaf(d.y, y.y, a.y));
    a.z = fmaf(d.x, x.z, fmaf(d.y, y.z, a.z));
    a.w = fmaf(d.x, x.w, fmaf(d.y, y.w, a.w));
  };
  int64_t r = r0 + lr;
  for (; r + 3 * SUB < r1; r += 4 * SUB) {
#pragma unroll
    for (int u = 0; u < 4; ++u) one(r + u * SUB, acc[u]);
  }
  for (; r < r1; r += SUB) one(r, acc[0]);
  float4 t = acc[0];
#pragma unroll
  for (int u = 1; u < 4; ++u) { t.x += acc[u].x; t.y += acc[u].y; t.z += acc[u].z; t.w += acc[u].w; }
  s_acc[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x < D4) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s2 = 0; s2 < SUB; ++s2) {
      const float4 y = s_acc[s2 * D4 + threadIdx.x];
      a.x += y.x; a.y += y.y; a.z += y.z; a.w += y.w;
    }
    reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * D4 * 4)[threadIdx.x] = a;
  }
}

// CTAs of the warp-per-row value kernels: >= 8 rows per warp (fewer partial rows
// to reduce at small batches), at most 8 CTAs per SM
int warp_grid(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, kWarps * 8), (int64_t)kNumSMs * 8));
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_warp_grid(int64_t rows) { return warp_grid(rows); }

extern "C" int accel_value_pool(const float* h1, const float* h2, const int32_t* row_frame,
                                const int32_t* steps, int64_t R, int D, int n_steps,
                                const float* w_attn, const float* b_attn, const float* e_step,
                                float* U, float* alpha, double* bad_part, int grid, void* stream) {
  if (R < 0 || D < 1 || n_steps < 1 || grid < 1) return fail(kDimension, "value_pool: bad sizes");
  if (R == 0) return kOk;
  if (!h1 || !h2 || !steps || !w_attn || !b_attn || !e_step || !U || !alpha || !bad_part)
    return fail(kDimension, "value_pool: NULL buffer");
  const uintptr_t al = reinterpret_cast<uintptr_t>(h1) | reinterpret_cast<uintptr_t>(h2) |
                       reinterpret_cast<uintptr_t>(w_attn) | reinterpret_cast<uintptr_t>(e_step) |
                       reinterpret_cast<uintptr_t>(U);
  if ((al & 15) == 0 && (D == 16 || D == 32 || D == 64 || D == 128)) {
    cudaStream_t s = as_stream(stream);
    switch (D / 4) {
      case 4: value_pool4_kernel<4><<<grid, kThreads, 0, s>>>(h1, h2, row_frame, steps, R, n_steps, w_attn, b_attn, e_step, U, alpha, bad_part); break;
      case 8: value_pool4_kernel<8><<<grid, kThreads, 0, s>>>(h1, h2, row_frame, steps, R, n_steps, w_attn, b_attn, e_step, U, alpha, bad_part); break;
      case 16: value_pool4_kernel<16><<<grid, kThreads, 0, s>>>(h1, h2, row_frame, steps, R, n_steps, w_attn, b_attn, e_step, U, alpha, bad_part); break;
      default: value_pool4_kernel<32><<<grid, kThreads, 0, s>>>(h1, h2, row_frame, steps, R, n_steps, w_attn, b_attn, e_step, U, alpha, bad_part); break;
    }
    return post_launch("value_pool4_kernel");
  }
  value_pool_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(
      h1, h2, row_frame, steps, R, D, n_steps, w_attn, b_attn, e_step, U, alpha, bad_part);
  return post_launch("value_pool_kernel");
}

extern "C" int accel_value_head(float* zm, const int32_t* row_frame, const float* b0v,
                                const float* w1v, const float* b1v,
                                int64_t R, int H, const float* targets, const float* v_old,
                                double vclip, double lambda_v,
                                double n_global, float* values_out, float* part, double* dpart,
                                int grid, void* stream) {
  if (R < 0 || H < 1 || grid < 1) return fail(kDimension, "value_head: bad sizes");
  if (H > 32 * kMaxHPL) return fail(kDimension, "value mlp_hidden=%d exceeds %d", H, 32 * kMaxHPL);
  if (R == 0) return kOk;
  if (!zm || !b0v || !w1v || !b1v || (targets && (!part || !dpart)))
    return fail(kDimension, "value_head: NULL buffer");
  if (v_old && !(vclip > 0)) return fail(kDomain, "value clip epsilon must be > 0");
  const double inv_n = n_global > 0 ? 1.0 / n_global : 0.0;
  cudaStream_t st = as_stream(stream);
  if ((reinterpret_cast<uintptr_t>(zm) & 15) == 0 && (H == 32 || H == 64 || H == 128)) {
    if (H == 32)
      value_head4_kernel<8, 4><<<grid, kThreads, 0, st>>>(zm, row_frame, b0v, w1v, b1v, R, targets, v_old, (float)vclip,
                                                          (float)lambda_v, inv_n, values_out, part, dpart);
    else if (H == 64)
      value_head4_kernel<8, 8><<<grid, kThreads, 0, st>>>(zm, row_frame, b0v, w1v, b1v, R, targets, v_old, (float)vclip,
                                                          (float)lambda_v, inv_n, values_out, part, dpart);
    else
      value_head4_kernel<16, 8><<<grid, kThreads, 0, st>>>(zm, row_frame, b0v, w1v, b1v, R, targets, v_old, (float)vclip,
                                                           (float)lambda_v, inv_n, values_out, part, dpart);
    return post_launch("value_head4_kernel");
  }
  value_head_kernel<<<grid, kThreads, 0, st>>>(zm, row_frame, b0v, w1v, b1v, R, H, targets, v_old,
                                               (float)vclip, (float)lambda_v,
                                               inv_n, values_out, part, dpart);
  return post_launch("value_head_kernel");
}

extern "C" int accel_value_attn_grad(const float* dU, const float* h1, const float* h2,
                                     const int32_t* row_frame, const float* alpha, int64_t R,
                                     int D, float* de, float* part, int grid, void* stream) {
  if (R < 0 || D < 1 || grid < 1) return fail(kDimension, "value_attn_grad: bad sizes");
  if (R == 0) return kOk;
  const uintptr_t al = reinterpret_cast<uintptr_t>(h1) | reinterpret_cast<uintptr_t>(h2) |
                       reinterpret_cast<uintptr_t>(dU);
  if ((al & 15) == 0 && (D == 16 || D == 32 || D == 64 || D == 128)) {
    cudaStream_t s = as_stream(stream);
    switch (D / 4) {
      case 4: value_attn_grad4_kernel<4><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, part); break;
      case 8: value_attn_grad4_kernel<8><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, part); break;
      case 16: value_attn_grad4_kernel<16><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, part); break;
      default: value_attn_grad4_kernel<32><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, part); break;
    }
    return post_launch("value_attn_grad4_kernel");
  }
  value_attn_grad_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(dU, h1, h2, row_frame, alpha,
                                                                   R, D, de, part);
  return post_launch("value_attn_grad_kernel");
}

extern "C" int accel_value_attn_wgrad(const float* de, const float* h1, const float* h2,
                                      const int32_t* row_frame, int64_t R, int D, float* part,
                                      int grid, void* stream) {
  if (R < 0 || D < 1 || grid < 1) return fail(kDimension, "value_attn_wgrad: bad sizes");
  if (R == 0) return kOk;
  const uintptr_t al = reinterpret_cast<uintptr_t>(h1) | reinterpret_cast<uintptr_t>(h2) |
                       reinterpret_cast<uintptr_t>(de) | reinterpret_cast<uintptr_t>(part);
  cudaStream_t st = as_stream(stream);
  if ((al & 15) == 0 && (D == 32 || D == 64 || D == 128)) {
    const float4* a4 = reinterpret_cast<const float4*>(h1);
    const float4* b4 = reinterpret_cast<const float4*>(h2);
    if (D == 32) value_attn_wgrad4_kernel<8><<<grid, kThreads, 0, st>>>(de, a4, b4, row_frame, R, part);
    else if (D == 64) value_attn_wgrad4_kernel<16><<<grid, kThreads, 0, st>>>(de, a4, b4, row_frame, R, part);
    else value_attn_wgrad4_kernel<32><<<grid, kThreads, 0, st>>>(de, a4, b4, row_frame, R, part);
    return post_launch("value_attn_wgrad4_kernel");
  }
  value_attn_wgrad_kernel<<<grid, kThreads, kThreads * sizeof(float), st>>>(de, h1, h2, row_frame,
                                                                             R, D, part);
  return post_launch("value_attn_wgrad_kernel");
}

extern "C" int accel_value_attn_backward(const float* dU, const float* h1, const float* h2,
                                         const int32_t* row_frame, const float* alpha, int64_t R,
                                         int D, float* de, float* bpart, float* wpart, int grid,
                                         void* stream) {
  if (R < 0 || D < 1 || grid < 1) return fail(kDimension, "value_attn_backward: bad sizes");
  if (R == 0) return kOk;
  if (!dU || !h1 || !h2 || !alpha || !bpart || !wpart)
    return fail(kDimension, "value_attn_backward: NULL buffer");
  const uintptr_t al = reinterpret_cast<uintptr_t>(h1) | reinterpret_cast<uintptr_t>(h2) |
                       reinterpret_cast<uintptr_t>(dU) | reinterpret_cast<uintptr_t>(wpart);
  if ((al & 15) != 0 || !(D == 16 || D == 32 || D == 64 || D == 128)) {
    // general widths: the two-pass kernels (they need the de rows)
    if (!de) return fail(kDimension, "value_attn_backward: de buffer needed at this width");
    const int rc = accel_value_attn_grad(dU, h1, h2, row_frame, alpha, R, D, de, bpart, grid, stream);
    if (rc != kOk) return rc;
    return accel_value_attn_wgrad(de, h1, h2, row_frame, R, D, wpart, grid, stream);
  }
  cudaStream_t s = as_stream(stream);
  switch (D / 4) {
    case 4: value_attn_bwd4_kernel<4><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, bpart, wpart); break;
    case 8: value_attn_bwd4_kernel<8><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, bpart, wpart); break;
    case 16: value_attn_bwd4_kernel<16><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, bpart, wpart); break;
    default: value_attn_bwd4_kernel<32><<<grid, kThreads, 0, s>>>(dU, h1, h2, row_frame, alpha, R, de, bpart, wpart); break;
  }
  return post_launch("value_attn_bwd4_kernel");
}

