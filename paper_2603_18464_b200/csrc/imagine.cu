// (c) World-model imagination: H imagined steps for N trajectories in ONE launch.
//
// Reference: RolloutWorker.imagine_episode (rollout.py:295-362), whose every
// step makes three round trips through the inference service
// (rollout.py:312, :313, :324 -> inference.run_batch, inference.py:146-159):
//   policy   PolicyModel.sample_chunk (models.py:135-150) + state_value (:406-408)
//   obs      ObsModel.predict (models.py:349-355) -> GridTaskSuite.snap_observation (env.py:259-283)
//   reward   RewardModel.predict (models.py:375-377); r = p' - p (telescoping), done-hat at p' >= thr
// Here each warp owns one trajectory and loops over the horizon on the device
// (no host round trip per step).  Arithmetic is float64 like the reference, so
// sampled tokens (searchsorted of the float64 cumsum against the request's
// uniforms) match it; uniforms are injected (parity) or drawn from Philox keyed
// by (seed, trajectory, request).  Weights are stored transposed ([in][out]) so a
// warp's matrix-vector products read 32 consecutive outputs per input element
// (coalesced, L1/L2-resident); activations live in per-warp shared memory.
#include <curand_kernel.h>
#include <math_constants.h>

#include "common.cuh"

namespace accel {
namespace {

struct ImagineWeights {
  // policy backbone and head (transposed: [in][out]) — models.py:103-109
  const double *w0t, *b0, *w1t, *b1, *e_prev, *e_pos, *w_headt, *b_head;
  // value head — models.py:247-255 (w0vt transposed)
  const double *w_attn, *b_attn, *e_step, *w0vt, *b0v, *w1v, *b1v;
  // world model: obs MLP [O + K*A -> HO -> O], reward MLP [O -> HR -> 1]
  const double *ow0t, *ob0, *ow1t, *ob1, *rw0t, *rb0, *rw1, *rb1;
};

struct ImagineDims {
  int O, D, K, A, S, HV, HO, HR, GH, GW, snap;
  int H;
  double threshold;
  unsigned long long seed;
};

// y[j] = act(sum_i Wt[i][j] x[i] + b[j]) for j in [0, out); lanes over j.
__device__ __forceinline__ void warp_matvec(const double* __restrict__ Wt, const double* x, int in,
                                            int out, const double* __restrict__ b, double* y,
                                            bool tanh_act, int lane) {
  for (int j0 = 0; j0 < out; j0 += 32) {
    const int j = j0 + lane;
    if (j < out) {
      double acc = 0.0;
      for (int i = 0; i < in; ++i) acc = fma(__ldg(Wt + (int64_t)i * out + j), x[i], acc);
      acc += b ? __ldg(b + j) : 0.0;
      y[j] = tanh_act ? tanh(acc) : acc;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// first index of the maximum of x[0..n) (np.argmax tie rule)
__device__ __forceinline__ int warp_argmax(const double* x, int n, int lane) {
  double best = -CUDART_INF;
  int bi = 0x7fffffff;
  for (int i = lane; i < n; i += 32) {
    const double v = x[i];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  return bi;
}

// V(o): value head over (h1, h2) at `step` (models.py:273-290 for one row)
__device__ double state_value(const ImagineWeights& w, const ImagineDims& d, const double* h1,
                              const double* h2, int step, double* u, double* m, int lane) {
  double e0 = 0.0, e1 = 0.0;
  for (int i = lane; i < d.D; i += 32) {
    const double wa = __ldg(w.w_attn + i);
    e0 = fma(h1[i], wa, e0);
    e1 = fma(h2[i], wa, e1);
  }
  e0 = warp_sum_f64(e0) + __ldg(w.b_attn);
  e1 = warp_sum_f64(e1) + __ldg(w.b_attn);
  const double mx = fmax(e0, e1);
  const double x0 = exp(e0 - mx), x1 = exp(e1 - mx);
  const double a0 = x0 / (x0 + x1), a1 = x1 / (x0 + x1);
  const int st = min(max(step, 0), d.S - 1);
  for (int i = lane; i < d.D; i += 32)
    u[i] = a0 * h1[i] + a1 * h2[i] + __ldg(w.e_step + (int64_t)st * d.D + i);
  __syncwarp();
  warp_matvec(w.w0vt, u, d.D, d.HV, w.b0v, m, true, lane);
  double v = 0.0;
  for (int i = lane; i < d.HV; i += 32) v = fma(__ldg(w.w1v + i), m[i], v);
  return warp_sum_f64(v) + __ldg(w.b1v);
}

__device__ double reward_prob(const ImagineWeights& w, const ImagineDims& d, const double* x,
                              double* hr, int lane) {
  warp_matvec(w.rw0t, x, d.O, d.HR, w.rb0, hr, true, lane);
  double z = 0.0;
  for (int i = lane; i < d.HR; i += 32) z = fma(__ldg(w.rw1 + i), hr[i], z);
  z = warp_sum_f64(z) + __ldg(w.rb1);
  return 1.0 / (1.0 + exp(-z));
}

// K autoregressive tokens from h2 (models.py:135-150): logits of token k from
// c = h2 + e_prev[prev] + e_pos[k], softmax, sequential cumsum, searchsorted
// against the k-th uniform (u_k injected, else Philox), clamped to A - 1.
// Writes toks[K] and the K x A logits (logits_out).
__device__ void policy_chunk(const ImagineWeights& w, const ImagineDims& d, const double* h2,
                             double* cvec, double* lg, const double* __restrict__ u_k,
                             curandStatePhilox4_32_10_t* rng, int* toks,
                             double* __restrict__ logits_out, int lane) {
  const int K = d.K, A = d.A;
  int prev = A;
  for (int k = 0; k < K; ++k) {
    for (int i = lane; i < d.D; i += 32)
      cvec[i] = h2[i] + __ldg(w.e_prev + (int64_t)prev * d.D + i) +
                __ldg(w.e_pos + (int64_t)k * d.D + i);
    __syncwarp();
    warp_matvec(w.w_headt, cvec, d.D, A, w.b_head, lg, false, lane);
    double mx = -CUDART_INF;
    for (int a = lane; a < A; a += 32) mx = fmax(mx, lg[a]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double u = u_k ? u_k[k] : (lane == 0 ? curand_uniform_double(rng) : 0.0);
    int tok = 0;
    if (lane == 0) {  // softmax + sequential cumsum + searchsorted (models.py:145-147)
      double s = 0.0;
      for (int a = 0; a < A; ++a) s += exp(lg[a] - mx);
      double cum = 0.0;
      tok = A;
      for (int a = 0; a < A; ++a) {
        cum += exp(lg[a] - mx) / s;
        if (u <= cum) { tok = a; break; }
      }
      tok = min(tok, A - 1);
    }
    tok = __shfl_sync(0xffffffffu, tok, 0);
    toks[k] = tok;
    double* lo = logits_out + (int64_t)k * A;
    for (int a = lane; a < A; a += 32) lo[a] = lg[a];
    prev = tok;
    __syncwarp();
  }
}

// next observation of the obs model for (x, chunk tokens) (models.py:349-355),
// the one-hot part of the input read as K weight rows
__device__ void obs_predict(const ImagineWeights& w, const ImagineDims& d, const double* x,
                            const int* toks, double* ho, double* nx, int lane) {
  const int O = d.O;
  for (int j0 = 0; j0 < d.HO; j0 += 32) {
    const int j = j0 + lane;
    if (j < d.HO) {
      double acc = 0.0;
      for (int i = 0; i < O; ++i) acc = fma(__ldg(w.ow0t + (int64_t)i * d.HO + j), x[i], acc);
      for (int k = 0; k < d.K; ++k)
        acc += __ldg(w.ow0t + (int64_t)(O + k * d.A + toks[k]) * d.HO + j);
      ho[j] = tanh(acc + __ldg(w.ob0 + j));
    }
  }
  __syncwarp();
  warp_matvec(w.ow1t, ho, d.HO, O, w.ob1, nx, false, lane);
}

__global__ void __launch_bounds__(128)
imagine_kernel(ImagineWeights w, ImagineDims d, const double* __restrict__ start_obs,
               const int32_t* __restrict__ start_step, const double* __restrict__ uniforms,
               int64_t n, double* __restrict__ obs_out, int32_t* __restrict__ steps_out,
               int32_t* __restrict__ tokens_out, double* __restrict__ logits_out,
               double* __restrict__ values_out, double* __restrict__ rewards_out,
               double* __restrict__ boot_out, int32_t* __restrict__ len_out,
               uint8_t* __restrict__ done_out, int32_t* __restrict__ status_out) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_warp = 2 * d.O + 3 * d.D + d.HO + d.HR + d.HV + d.A + d.D;
  double* x = sm + (size_t)warp * per_warp;  // current observation
  double* nx = x + d.O;                       // next observation (prediction / snapped)
  double* h1 = nx + d.O;
  double* h2 = h1 + d.D;
  double* cvec = h2 + d.D;                    // h2 + e_prev[prev] + e_pos[k]
  double* ho = cvec + d.D;                    // obs-model hidden
  double* hr = ho + d.HO;                     // reward-model hidden
  double* mv = hr + d.HR;                     // value-head hidden
  double* lg = mv + d.HV;                     // one token's logits
  double* uv = lg + d.A;                      // value-head pooled input
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
  if (t >= n) return;
  const int O = d.O, K = d.K, A = d.A;
  for (int i = lane; i < O; i += 32) x[i] = start_obs[t * O + i];
  __syncwarp();
  int step = start_step[t];
  double* obs_t = obs_out + t * (int64_t)(d.H + 1) * O;
  for (int i = lane; i < O; i += 32) obs_t[i] = x[i];
  if (lane == 0) steps_out[t * (d.H + 1)] = step;
  double p_cur = reward_prob(w, d, x, hr, lane);
  curandStatePhilox4_32_10_t rng;
  if (uniforms == nullptr) curand_init(d.seed, (unsigned long long)t, 0, &rng);
  int req = 0, len = 0, status = 0;
  bool done = false;
  for (int h = 0; h < d.H; ++h) {
    // ---- policy request: backbone, AR token sampling, value ----------------------
    warp_matvec(w.w0t, x, O, d.D, w.b0, h1, true, lane);
    warp_matvec(w.w1t, h1, d.D, d.D, w.b1, h2, true, lane);
    int toks[32];
    policy_chunk(w, d, h2, cvec, lg, uniforms ? uniforms + (t * (d.H + 1) + req) * K : nullptr,
                 &rng, toks, logits_out + (t * d.H + h) * K * (int64_t)A, lane);
    const double val = state_value(w, d, h1, h2, step, uv, mv, lane);
    ++req;
    // ---- obs request: [o, onehot(chunk)] -> HO -> O ------------------------------------
    obs_predict(w, d, x, toks, ho, nx, lane);
    bool finite = true;
    for (int i = lane; i < O; i += 32) finite &= isfinite(nx[i]);
    if (!__all_sync(0xffffffffu, finite)) { status = 1; break; }
    if (d.snap) {  // env.py:259-283
      const int cells = d.GH * d.GW;
      const int agent = warp_argmax(nx, cells, lane);
      const int obj = warp_argmax(nx + cells, cells, lane);
      const bool carried = nx[cells + obj] > 1.5;
      const int goal = warp_argmax(nx + 2 * cells, cells, lane);
      const int kind = warp_argmax(nx + 3 * cells, O - 3 * cells, lane);
      __syncwarp();
      for (int i = lane; i < O; i += 32) nx[i] = 0.0;
      __syncwarp();
      if (lane == 0) {
        nx[agent] = 1.0;
        if (carried) nx[cells + agent] = 2.0; else nx[cells + obj] = 1.0;
        nx[2 * cells + goal] = 1.0;
        nx[3 * cells + kind] = 1.0;
      }
      __syncwarp();
    }
    // ---- reward request --------------------------------------------------------------
    const double p_next = reward_prob(w, d, nx, hr, lane);
    if (!isfinite(p_next)) { status = 2; break; }
    if (lane == 0) {
      for (int k = 0; k < K; ++k) tokens_out[(t * d.H + h) * K + k] = toks[k];
      values_out[t * d.H + h] = val;
      rewards_out[t * d.H + h] = p_next - p_cur;
      steps_out[t * (d.H + 1) + h + 1] = step + 1;
    }
    for (int i = lane; i < O; i += 32) {
      x[i] = nx[i];
      obs_t[(int64_t)(h + 1) * O + i] = nx[i];
    }
    __syncwarp();
    p_cur = p_next;
    ++step;
    ++len;
    if (p_next >= d.threshold) { done = true; break; }
  }
  double boot = 0.0;
  if (status == 0) {  // tail policy request: bootstrap value of the last frame (rollout.py:345)
    warp_matvec(w.w0t, x, O, d.D, w.b0, h1, true, lane);
    warp_matvec(w.w1t, h1, d.D, d.D, w.b1, h2, true, lane);
    boot = state_value(w, d, h1, h2, step, uv, mv, lane);
  }
  if (lane == 0) {
    boot_out[t] = boot;
    len_out[t] = len;
    done_out[t] = done ? 1 : 0;
    status_out[t] = status;
  }
}

// Batched inference service evaluation (inference.py:129-160, run_batch): one
// warp per request, all of one kind.  kind 0 policy: sample_chunk + state_value
// (uniforms u[n, K] drawn by the host from the request's ticket substream, so
// tokens equal the reference's whatever the batch composition); kind 1 obs
// model: predict(o, chunk); kind 2 reward model: sigmoid probability.
__global__ void __launch_bounds__(128)
serve_kernel(ImagineWeights w, ImagineDims d, int kind, const double* __restrict__ obs,
             const int32_t* __restrict__ steps, const int32_t* __restrict__ chunks,
             const double* __restrict__ uniforms, int64_t n, int32_t* __restrict__ tokens_out,
             double* __restrict__ logits_out, double* __restrict__ values_out,
             double* __restrict__ next_obs_out, double* __restrict__ probs_out) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per_warp = 2 * d.O + 3 * d.D + d.HO + d.HR + d.HV + d.A + d.D;
  double* x = sm + (size_t)warp * per_warp;
  double* nx = x + d.O;
  double* h1 = nx + d.O;
  double* h2 = h1 + d.D;
  double* cvec = h2 + d.D;
  double* ho = cvec + d.D;
  double* hr = ho + d.HO;
  double* mv = hr + d.HR;
  double* lg = mv + d.HV;
  double* uv = lg + d.A;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
  if (r >= n) return;
  for (int i = lane; i < d.O; i += 32) x[i] = obs[r * d.O + i];
  __syncwarp();
  if (kind == 0) {
    warp_matvec(w.w0t, x, d.O, d.D, w.b0, h1, true, lane);
    warp_matvec(w.w1t, h1, d.D, d.D, w.b1, h2, true, lane);
    int toks[32];
    policy_chunk(w, d, h2, cvec, lg, uniforms + r * d.K, nullptr, toks,
                 logits_out + r * d.K * (int64_t)d.A, lane);
    const double val = state_value(w, d, h1, h2, steps[r], uv, mv, lane);
    if (lane == 0) {
      for (int k = 0; k < d.K; ++k) tokens_out[r * d.K + k] = toks[k];
      values_out[r] = val;
    }
  } else if (kind == 1) {
    int toks[32];
    for (int k = 0; k < d.K; ++k) toks[k] = min(max(chunks[r * d.K + k], 0), d.A - 1);
    obs_predict(w, d, x, toks, ho, nx, lane);
    for (int i = lane; i < d.O; i += 32) next_obs_out[r * d.O + i] = nx[i];
  } else {
    const double pr = reward_prob(w, d, x, hr, lane);
    if (lane == 0) probs_out[r] = pr;
  }
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" size_t accel_imagine_smem_bytes(int O, int D, int A, int HV, int HO, int HR) {
  return sizeof(double) * 4 * (size_t)(2 * O + 4 * D + HO + HR + HV + A);
}

// weights: 23 device pointers in ImagineWeights order; dims: 11 ints
// {O, D, K, A, S, HV, HO, HR, GH, GW, snap}.
extern "C" int accel_imagine(const void* const* weights, const int* dims, int H, double threshold,
                             unsigned long long seed, const double* start_obs,
                             const int32_t* start_step, const double* uniforms, int64_t n,
                             double* obs_out, int32_t* steps_out, int32_t* tokens_out,
                             double* logits_out, double* values_out, double* rewards_out,
                             double* boot_out, int32_t* len_out, uint8_t* done_out,
                             int32_t* status_out, void* stream) {
  if (!weights || !dims) return fail(kDimension, "imagine: NULL weights/dims");
  ImagineDims d;
  d.O = dims[0]; d.D = dims[1]; d.K = dims[2]; d.A = dims[3]; d.S = dims[4]; d.HV = dims[5];
  d.HO = dims[6]; d.HR = dims[7]; d.GH = dims[8]; d.GW = dims[9]; d.snap = dims[10];
  d.H = H;
  d.threshold = threshold;
  d.seed = seed;
  if (d.O < 1 || d.D < 1 || d.K < 1 || d.K > 32 || d.A < 1 || d.S < 1 || d.HV < 1 || d.HO < 1 ||
      d.HR < 1 || H < 1 || n < 0)
    return fail(kDimension, "imagine: bad dimensions");
  if (d.snap && (d.GH < 1 || d.GW < 1 || 3 * d.GH * d.GW >= d.O))
    return fail(kDimension, "imagine: grid %dx%d does not fit obs_dim %d", d.GH, d.GW, d.O);
  if (!(threshold > 0.0 && threshold <= 1.0))
    return fail(kDomain, "success_threshold must be in (0, 1]");
  if (n == 0) return kOk;
  const void* const* p = weights;
  for (int i = 0; i < 23; ++i)
    if (!p[i]) return fail(kDimension, "imagine: weight %d is NULL", i);
  ImagineWeights w{
      (const double*)p[0], (const double*)p[1], (const double*)p[2], (const double*)p[3],
      (const double*)p[4], (const double*)p[5], (const double*)p[6], (const double*)p[7],
      (const double*)p[8], (const double*)p[9], (const double*)p[10], (const double*)p[11],
      (const double*)p[12], (const double*)p[13], (const double*)p[14], (const double*)p[15],
      (const double*)p[16], (const double*)p[17], (const double*)p[18], (const double*)p[19],
      (const double*)p[20], (const double*)p[21], (const double*)p[22]};
  const size_t smem = accel_imagine_smem_bytes(d.O, d.D, d.A, d.HV, d.HO, d.HR);
  if (smem > 200 * 1024) return fail(kDimension, "imagine: activations exceed shared memory");
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(imagine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(kCuda, "imagine smem: %s", cudaGetErrorString(e));
  }
  const int grid = (int)ceil_div(n, 4);
  imagine_kernel<<<grid, 128, smem, as_stream(stream)>>>(
      w, d, start_obs, start_step, uniforms, n, obs_out, steps_out, tokens_out, logits_out,
      values_out, rewards_out, boot_out, len_out, done_out, status_out);
  return post_launch("imagine_kernel");
}

extern "C" int accel_serve(const void* const* weights, const int* dims, int kind, const double* obs,
                           const int32_t* steps, const int32_t* chunks, const double* uniforms,
                           int64_t n, int32_t* tokens_out, double* logits_out, double* values_out,
                           double* next_obs_out, double* probs_out, void* stream) {
  if (n < 0 || kind < 0 || kind > 2) return fail(kDimension, "serve: bad kind / size");
  if (n == 0) return kOk;
  if (!weights || !dims || !obs) return fail(kDimension, "serve: NULL buffer");
  ImagineDims d{};
  d.O = dims[0]; d.D = dims[1]; d.K = dims[2]; d.A = dims[3]; d.S = dims[4]; d.HV = dims[5];
  d.HO = dims[6]; d.HR = dims[7];
  if (d.O < 1 || d.D < 1 || d.K < 1 || d.K > 32 || d.A < 1 || d.S < 1)
    return fail(kDimension, "serve: bad dims");
  if (kind == 0 && (!steps || !uniforms || !tokens_out || !logits_out || !values_out))
    return fail(kDimension, "serve: policy batch needs steps, uniforms and outputs");
  if (kind == 1 && (!chunks || !next_obs_out)) return fail(kDimension, "serve: obs batch buffers");
  if (kind == 2 && !probs_out) return fail(kDimension, "serve: reward batch buffers");
  const double* const* p = reinterpret_cast<const double* const*>(weights);
  ImagineWeights w{p[0],  p[1],  p[2],  p[3],  p[4],  p[5],  p[6],  p[7],
                   p[8],  p[9],  p[10], p[11], p[12], p[13], p[14],
                   p[15], p[16], p[17], p[18], p[19], p[20], p[21], p[22]};
  const size_t smem = accel_imagine_smem_bytes(d.O, d.D, d.A, d.HV, d.HO, d.HR);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(serve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(kCuda, "serve smem: %s", cudaGetErrorString(e));
  }
  serve_kernel<<<(unsigned)ceil_div(n, 4), 128, smem, as_stream(stream)>>>(
      w, d, kind, obs, steps, chunks, uniforms, n, tokens_out, logits_out, values_out,
      next_obs_out, probs_out);
  return post_launch("serve_kernel");
}
