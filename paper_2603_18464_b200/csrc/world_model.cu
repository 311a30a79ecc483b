// World-model training sub-steps: one optimizer step of the
// observation model (MSE on (o_t, a_t) -> o_{t+1}) or the reward model (binary
// cross-entropy on frames), both 2-layer tanh MLPs.
//
// Reference: train_obs_model_step / train_reward_model_step (trainer.py:469-535),
// mlp_forward / mlp_backward (numerics.py:174-220), adam_step (numerics.py:95-126).
// The reference computes in float64 and so does this file (the sub-steps are
// small -- <= wm_max_transitions rows -- and latency-bound, so float64 costs
// nothing and keeps parity at round-off level).  Every reduction runs in a
// fixed order (rows ascending), so a sub-step is bitwise reproducible.
//
// Layout: x f64[n, din], hidden f64[n, dh], out / grad f64[n, dout]; parameters
// one flat f64 buffer {w0 [dh, din], b0 [dh], w1 [dout, dh], b1 [dout]}.
#include <math_constants.h>

#include "common.cuh"

namespace accel {
namespace {

constexpr int kWmThreads = 256;

struct Mlp2 {
  const double* w0;
  const double* b0;
  const double* w1;
  const double* b1;
};

// h[r, j] = tanh(x[r] . w0[j] + b0[j])
__global__ void wm_hidden_kernel(const double* __restrict__ x, int64_t n, int din, int dh,
                                 Mlp2 p, double* __restrict__ h) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * dh) return;
  const int64_t r = e / dh;
  const int j = (int)(e % dh);
  const double* xr = x + r * din;
  const double* wj = p.w0 + (int64_t)j * din;
  double z = 0.0;
  for (int i = 0; i < din; ++i) z = fma(xr[i], wj[i], z);
  h[e] = tanh(z + p.b0[j]);
}

// out = h . w1^T + b1; kind 0 (MSE vs target[n, dout]): g = 2 (out - t) / (n dout),
// loss term (out - t)^2; kind 1 (BCE from logits, dout = 1, target = labels):
// g = (sigmoid(z) - y) / n, loss term softplus(z) - y z (trainer.py:520-523).
// One partial per block (threads in order).
__global__ void wm_out_loss_kernel(const double* __restrict__ h, const double* __restrict__ target,
                                   int64_t n, int dh, int dout, int kind, Mlp2 p,
                                   double* __restrict__ g, double* __restrict__ loss_part) {
  __shared__ double s_l[kWmThreads];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double term = 0.0;
  if (e < n * dout) {
    const int64_t r = e / dout;
    const int o = (int)(e % dout);
    const double* hr = h + r * dh;
    const double* wo = p.w1 + (int64_t)o * dh;
    double z = 0.0;
    for (int j = 0; j < dh; ++j) z = fma(hr[j], wo[j], z);
    z += p.b1[o];
    const double t = target[e];
    if (kind == 0) {
      const double err = z - t;
      term = err * err;
      g[e] = 2.0 * err / (double)(n * dout);
    } else {
      // logaddexp(0, z) = max(z, 0) + log1p(exp(-|z|))
      term = fmax(z, 0.0) + log1p(exp(-fabs(z))) - t * z;
      const double prob = 1.0 / (1.0 + exp(-z));
      g[e] = (prob - t) / (double)n;
    }
  }
  s_l[threadIdx.x] = term;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kWmThreads; ++i) s += s_l[i];
    loss_part[blockIdx.x] = s;
  }
}

// dh[r, j] = (sum_o g[r, o] w1[o, j]) (1 - h[r, j]^2)   (numerics.py:216-218)
__global__ void wm_dhidden_kernel(const double* __restrict__ g, const double* __restrict__ h,
                                  int64_t n, int dh, int dout, Mlp2 p, double* __restrict__ dh_out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * dh) return;
  const int64_t r = e / dh;
  const int j = (int)(e % dh);
  double s = 0.0;
  for (int o = 0; o < dout; ++o) s = fma(g[r * dout + o], p.w1[(int64_t)o * dh + j], s);
  const double hv = h[e];
  dh_out[e] = s * (1.0 - hv * hv);
}

// dw[o, i] = sum_r g[r, o] a[r, i] for i < din, db[o] = sum_r g[r, o]   (rows in order)
__global__ void wm_wgrad_kernel(const double* __restrict__ g, const double* __restrict__ a,
                                int64_t n, int dout, int din, double* __restrict__ dw,
                                double* __restrict__ db) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)dout * (din + 1)) return;
  const int o = (int)(e / (din + 1));
  const int i = (int)(e % (din + 1));
  double s = 0.0;
  if (i < din) {
    for (int64_t r = 0; r < n; ++r) s = fma(g[r * dout + o], a[r * din + i], s);
    dw[(int64_t)o * din + i] = s;
  } else {
    for (int64_t r = 0; r < n; ++r) s += g[r * dout + o];
    db[o] = s;
  }
}

__global__ void wm_sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out,
                              double scale) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    out[0] = s * scale;
  }
}

__global__ void wm_count_nonfinite_kernel(const double* __restrict__ x, int64_t n,
                                          unsigned* __restrict__ count) {
  unsigned c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += isfinite(x[i]) ? 0u : 1u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);  // integer: order-independent
}

// Adam (numerics.py:109-116) in float64; bad += non-finite new parameters.
__global__ void wm_adam_kernel(double* __restrict__ p, const double* __restrict__ g,
                               double* __restrict__ m, double* __restrict__ v, int64_t n,
                               double lr, double b1, double b2, double eps, double bc1,
                               double bc2, unsigned* __restrict__ bad) {
  unsigned c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
    const double mh = mi / bc1, vh = vi / bc2;
    const double pi = p[i] - lr * mh / (sqrt(vh) + eps);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
    c += isfinite(pi) ? 0u : 1u;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}

unsigned blocks_for(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, kWmThreads)); }

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" size_t accel_wm_workspace_size(int64_t n, int dh, int dout) {
  // hidden [n, dh] + dhidden [n, dh] + grad [n, dout] + loss partials
  return sizeof(double) * (size_t)(2 * n * dh + n * dout + ceil_div(n * dout, kWmThreads) + 8);
}

extern "C" int accel_wm_mlp2_grad(const double* x, const double* target, int64_t n, int din,
                                  int dh, int dout, int kind, const double* params,
                                  double* grads, double* loss_out, unsigned* nonfinite,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 1 || din < 1 || dh < 1 || dout < 1) return fail(kDimension, "wm_mlp2_grad: bad sizes");
  if (kind != 0 && kind != 1) return fail(kDomain, "wm_mlp2_grad: unknown loss kind %d", kind);
  if (kind == 1 && dout != 1) return fail(kDimension, "wm_mlp2_grad: BCE needs one output");
  if (!x || !target || !params || !grads || !loss_out || !nonfinite || !workspace)
    return fail(kDimension, "wm_mlp2_grad: NULL buffer");
  if (workspace_bytes < accel_wm_workspace_size(n, dh, dout))
    return fail(kDimension, "wm_mlp2_grad: workspace too small");
  cudaStream_t s = as_stream(stream);
  Mlp2 p{params, params + (int64_t)dh * din, params + (int64_t)dh * din + dh,
         params + (int64_t)dh * din + dh + (int64_t)dout * dh};
  double* h = static_cast<double*>(workspace);
  double* dhid = h + n * dh;
  double* g = dhid + n * dh;
  double* loss_part = g + n * dout;
  double* gw0 = grads;
  double* gb0 = grads + (int64_t)dh * din;
  double* gw1 = gb0 + dh;
  double* gb1 = gw1 + (int64_t)dout * dh;
  int st;
  wm_hidden_kernel<<<blocks_for(n * dh), kWmThreads, 0, s>>>(x, n, din, dh, p, h);
  if ((st = post_launch("wm_hidden_kernel"))) return st;
  const unsigned lb = blocks_for(n * dout);
  wm_out_loss_kernel<<<lb, kWmThreads, 0, s>>>(h, target, n, dh, dout, kind, p, g, loss_part);
  if ((st = post_launch("wm_out_loss_kernel"))) return st;
  wm_sum_kernel<<<1, 32, 0, s>>>(loss_part, (int)lb, loss_out,
                                  kind == 0 ? 1.0 / (double)(n * dout) : 1.0 / (double)n);
  if ((st = post_launch("wm_sum_kernel"))) return st;
  wm_wgrad_kernel<<<blocks_for((int64_t)dout * (dh + 1)), kWmThreads, 0, s>>>(g, h, n, dout, dh,
                                                                             gw1, gb1);
  if ((st = post_launch("wm_wgrad_kernel"))) return st;
  wm_dhidden_kernel<<<blocks_for(n * dh), kWmThreads, 0, s>>>(g, h, n, dh, dout, p, dhid);
  if ((st = post_launch("wm_dhidden_kernel"))) return st;
  wm_wgrad_kernel<<<blocks_for((int64_t)dh * (din + 1)), kWmThreads, 0, s>>>(dhid, x, n, dh, din,
                                                                           gw0, gb0);
  if ((st = post_launch("wm_wgrad_kernel"))) return st;
  const int64_t np_ = (int64_t)dh * din + dh + (int64_t)dout * dh + dout;
  if ((st = check_cuda(cudaMemsetAsync(nonfinite, 0, sizeof(unsigned), s), "wm memset")))
    return st;
  wm_count_nonfinite_kernel<<<std::min<unsigned>(blocks_for(np_), 64), kWmThreads, 0, s>>>(
      grads, np_, nonfinite);
  return post_launch("wm_count_nonfinite_kernel");
}

extern "C" int accel_wm_adam(double* params, const double* grads, double* m, double* v,
                             int64_t n, double lr, double beta1, double beta2, double eps,
                             int64_t t, unsigned* bad, void* stream) {
  if (n < 1 || t < 1) return fail(kDimension, "wm_adam: bad sizes");
  if (!params || !grads || !m || !v || !bad) return fail(kDimension, "wm_adam: NULL buffer");
  cudaStream_t s = as_stream(stream);
  int st;
  if ((st = check_cuda(cudaMemsetAsync(bad, 0, sizeof(unsigned), s), "wm memset"))) return st;
  const double bc1 = 1.0 - pow(beta1, (double)t), bc2 = 1.0 - pow(beta2, (double)t);
  wm_adam_kernel<<<std::min<unsigned>(blocks_for(n), 148 * 4), kWmThreads, 0, s>>>(
      params, grads, m, v, n, lr, beta1, beta2, eps, bc1, bc2, bad);
  return post_launch("wm_adam_kernel");
}
