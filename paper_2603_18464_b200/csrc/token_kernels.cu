// (b) Token-level loss over action-vocabulary logits.
//
//   K3 token_logp  — behavior_log_probs (trainer.py:289-293):
//                    log_softmax(mu)[token] per token row.
//   K4 token_loss  — log_prob_chunk (models.py:219-223) + policy_surrogate
//                    (trainer.py:183-239, GIPO "trust" and PPO "clip") +
//                    entropy_bonus (:242-251) + the dlogits assembly of
//                    train_step (:425-435), forward AND backward in one pass:
//                    each logit row is read once and its dlogits row written
//                    once (2*A*4 + 12 B/token, HBM-bound).
//
// Layout: warp-per-row; each lane holds VPL logits of the row.  When rows
// are 16-byte multiples (A % 4 == 0, A >= 128) the rows are streamed into a
// per-warp shared-memory ring by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier complete_tx, STAGES rows in flight per warp), so
// memory-level parallelism does not cost registers; otherwise rows are
// loaded straight into registers.  Row statistics use xor-shuffle
// butterflies (deterministic).  exp(z - max) is evaluated once per logit and
// reused for the partition function, the entropy and the gradient:
//   H = log s - (sum e d)/s,  dz = p (lambda_h/NK (d - sum e d / s) - c) + c [a == tok]
// with d = z - max, e = exp(d), p = e / s, c = the token's surrogate coefficient.
// Per-token scalar algebra is float except the rare tails (|log-ratio| >= 60
// or a trust weight below e^-75), which switch to float64 so ratio
// overflow/underflow follows the reference's float64 exclusion rule
// (isfinite(r) & r > 0, trainer.py:204-205).
//
// The surrogate gradient carries 1/m, m = #included tokens — a GLOBAL count
// (all ranks).  The kernel writes dlogits with the optimistic m0 = M_global
// (no exclusions); the same kernel launched in FIXUP mode reads the reduced
// excluded count on the device and rewrites dlogits only when 0 < excluded
// < M_global, so the common case costs a single pass and no host sync.
#include <math_constants.h>

#include "common.cuh"

namespace accel {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRows = 2;     // rows in flight per warp (register path)
constexpr int kStages = 4;   // rows in flight per warp (TMA path)

// per-block float64 partial sums (layout documented in accel.h)
enum : int {
  kLossNum = 0,    // sum over included tokens of w*r*a (trust) or min(r a, clip(r) a)
  kEntSum = 1,     // sum of per-token entropy over ALL tokens
  kRatioSum = 2,   // sum of r over included tokens
  kWSum = 3,       // sum of trust weights over included tokens
  kOutside = 4,    // included tokens with r outside [1-eps, 1+eps]
  kExcluded = 5,   // tokens with non-finite or zero ratio
  kBadRows = 6,    // rows with non-finite logits
  kBadTok = 7,     // tokens outside [0, A)
  kNumStat = 8
};
enum : int { kRatioMax = 0, kNegWMin = 1, kNumMax = 2 };

struct LossParams {
  int algo;  // 0 trust (GIPO), 1 clip (PPO)
  float sigma, clip_lo, clip_hi, lambda_h;
  double inv_nk;    // 1 / global token count (entropy mean)
  double m_global;  // global token count
};

template <int VPL, bool VEC>
struct RowLayout {
  __device__ __forceinline__ static int col(int lane, int v) {
    if (VEC) return (v >> 2) * 128 + lane * 4 + (v & 3);
    return v * 32 + lane;
  }
  __device__ __forceinline__ static void locate(int tok, int& lane, int& v) {
    if (VEC) {
      const int w = tok & 127;
      lane = w >> 2;
      v = (tok >> 7) * 4 + (w & 3);
    } else {
      lane = tok & 31;
      v = tok >> 5;
    }
  }
  // global or shared source (generic pointers)
  __device__ __forceinline__ static void load(const float* __restrict__ row, int lane, int A,
                                              float (&z)[VPL], bool streaming) {
    if (VEC) {
#pragma unroll
      for (int q = 0; q < VPL / 4; ++q) {
        const int c = q * 128 + lane * 4;
        const float4* p = reinterpret_cast<const float4*>(row + c);
        float4 x = c < A ? (streaming ? __ldcs(p) : *p) : make_float4(0.f, 0.f, 0.f, 0.f);
        z[4 * q] = x.x; z[4 * q + 1] = x.y; z[4 * q + 2] = x.z; z[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = v * 32 + lane;
        z[v] = c < A ? (streaming ? __ldcs(row + c) : row[c]) : 0.f;
      }
    }
  }
  __device__ __forceinline__ static void store(float* __restrict__ row, int lane, int A,
                                               const float (&d)[VPL]) {
    if (VEC) {
#pragma unroll
      for (int q = 0; q < VPL / 4; ++q) {
        const int c = q * 128 + lane * 4;
        if (c < A)
          __stcs(reinterpret_cast<float4*>(row + c),
                 make_float4(d[4 * q], d[4 * q + 1], d[4 * q + 2], d[4 * q + 3]));
      }
    } else {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = v * 32 + lane;
        if (c < A) __stcs(row + c, d[v]);
      }
    }
  }
};

// Row statistics; on return z[] holds d = z - max and e[] holds exp(d).
struct RowStats {
  float log_s, inv_s, sd_over_s, H, d_tok;
  bool bad;
};

template <int VPL, bool VEC>
__device__ __forceinline__ RowStats row_stats(float (&z)[VPL], float (&e)[VPL], int lane, int A,
                                              int tok, bool with_entropy) {
  using L = RowLayout<VPL, VEC>;
  RowStats s;
  float mx = -CUDART_INF_F;
  bool bad = false;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    if (L::col(lane, v) < A) {
      mx = fmaxf(mx, z[v]);
      bad |= !isfinite(z[v]);
    }
  }
  s.bad = __any_sync(0xffffffffu, bad);
  mx = warp_max(mx);
  float sum = 0.f, sed = 0.f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const bool ok = L::col(lane, v) < A;
    z[v] = ok ? z[v] - mx : 0.f;
    e[v] = ok ? __expf(z[v]) : 0.f;
    sum += e[v];
    sed = fmaf(e[v], z[v], sed);
  }
  if (with_entropy) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      sed += __shfl_xor_sync(0xffffffffu, sed, o);
    }
  } else {
    sum = warp_sum(sum);
  }
  s.inv_s = 1.f / sum;
  s.log_s = __logf(sum);
  s.sd_over_s = sed * s.inv_s;
  s.H = s.log_s - s.sd_over_s;
  int tl, tv;
  L::locate(tok, tl, tv);
  float pick = 0.f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) pick = (v == tv) ? z[v] : pick;
  s.d_tok = __shfl_sync(0xffffffffu, pick, tl);
  return s;
}

// Per-token surrogate algebra (trainer.py:204-236) in precision T.
template <typename T>
__device__ __forceinline__ void token_scalars(T delta, T a, const LossParams& p, T& coef, T& term,
                                              T& r, T& w, bool& outside) {
  r = exp(delta);
  outside = false;
  if (p.algo == 0) {
    const T q = delta / (T)p.sigma;
    w = exp((T)-0.5 * q * q);  // trust_weight, trainer.py:174 (stop-gradient)
    term = w * r * a;
    coef = -term;              // d(-w r a)/dlogp, trainer.py:222
  } else {
    w = (T)1;
    const T lo = (T)p.clip_lo, hi = (T)p.clip_hi;
    const T rc = r < lo ? lo : (r > hi ? hi : r);
    const T ra = r * a, rca = rc * a;
    term = ra < rca ? ra : rca;
    coef = (ra <= rca) ? -ra : (T)0;  // trainer.py:232-233
    outside = (r < lo) || (r > hi);
  }
}

template <int VPL>
struct LossAcc {
  float dbias[VPL];
  double loss_num, ent_sum, ratio_sum, w_sum, rmax, negwmin;
  int n_out, n_excl, n_bad, n_badtok;
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int v = 0; v < VPL; ++v) dbias[v] = 0.f;
    loss_num = ent_sum = ratio_sum = w_sum = 0.0;
    rmax = negwmin = -CUDART_INF;
    n_out = n_excl = n_bad = n_badtok = 0;
  }
};

struct RowCtx {
  LossParams prm;
  float inv_m, ent_scale;
  double inv_m_d;
  bool fixup;
};

// Everything after the logits of one row are in registers (bias not yet added).
template <int VPL, bool VEC>
__device__ __forceinline__ void loss_row(float (&z)[VPL], const float* __restrict__ s_bias,
                                         int64_t row, int lane, int A, int K,
                                         const int32_t* __restrict__ tokens,
                                         const float* __restrict__ lp_old,
                                         const float* __restrict__ adv, const RowCtx& cx,
                                         float* __restrict__ dlogits, float* __restrict__ lp_new,
                                         LossAcc<VPL>& acc) {
  using L = RowLayout<VPL, VEC>;
#pragma unroll
  for (int v = 0; v < VPL; ++v) z[v] += s_bias[L::col(lane, v)];
  int tok = __ldg(tokens + row);
  const bool bad_tok = tok < 0 || tok >= A;
  if (bad_tok) tok = 0;
  float e[VPL];
  const RowStats rs = row_stats<VPL, VEC>(z, e, lane, A, tok, true);
  const float lpn = rs.d_tok - rs.log_s;
  const float dlt = lpn - __ldg(lp_old + row);
  const float a = __ldg(adv + row / K);
  // reference exclusion: exp(delta) in float64 finite and > 0
  const bool inc = !bad_tok && !rs.bad && dlt <= 709.78271289f && dlt >= -745.13321910f;
  float coef = 0.f;
  double term_d = 0.0, r_d = 1.0, w_d = 1.0;
  bool outside = false;
  if (inc) {
    const float qq = dlt / cx.prm.sigma;
    if (fabsf(dlt) < 60.f && (cx.prm.algo != 0 || qq * qq < 150.f)) {
      float cf, tf, rf, wf;
      token_scalars<float>(dlt, a, cx.prm, cf, tf, rf, wf, outside);
      coef = cf * cx.inv_m;
      term_d = tf; r_d = rf; w_d = wf;
    } else {
      double cd;
      token_scalars<double>((double)dlt, (double)a, cx.prm, cd, term_d, r_d, w_d, outside);
      coef = (float)(cd * cx.inv_m_d);
    }
  }
  // dz = p (ent_scale (d - sd/s) - coef) + coef [a == tok]
  float g[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int c = L::col(lane, v);
    const float p = e[v] * rs.inv_s;
    const float t = fmaf(cx.ent_scale, z[v] - rs.sd_over_s, -coef);
    float x = fmaf(p, t, c == tok ? coef : 0.f);
    x = c < A ? x : 0.f;
    g[v] = x;
    acc.dbias[v] += x;
  }
  L::store(dlogits + row * A, lane, A, g);
  if (!cx.fixup) {
    if (lane == 0) lp_new[row] = lpn;
    acc.ent_sum += (double)rs.H;
    acc.n_bad += rs.bad;
    acc.n_badtok += bad_tok;
    if (inc) {
      acc.loss_num += term_d;
      acc.ratio_sum += r_d;
      acc.w_sum += w_d;
      acc.n_out += outside;
      acc.rmax = fmax(acc.rmax, r_d);
      acc.negwmin = fmax(acc.negwmin, -w_d);
    } else {
      ++acc.n_excl;
    }
  }
}

__device__ __forceinline__ bool setup_ctx(const LossParams& prm, const double* fix_stats,
                                          RowCtx& cx) {
  cx.prm = prm;
  cx.fixup = fix_stats != nullptr;
  double m_eff = prm.m_global;
  if (cx.fixup) {
    const double excl = fix_stats[kExcluded];
    if (excl == 0.0 || excl >= prm.m_global) return false;  // uniform early exit
    m_eff = prm.m_global - excl;
  }
  cx.inv_m = (float)(1.0 / m_eff);
  cx.inv_m_d = 1.0 / m_eff;
  cx.ent_scale = prm.lambda_h * (float)prm.inv_nk;
  return true;
}

// fixed-order block reduction of the bias gradient and the token statistics
template <int VPL, bool VEC>
__device__ __forceinline__ void loss_epilogue(const LossAcc<VPL>& acc, int A, bool fixup,
                                              float* s_dbias /*[kWarps][VPL*32]*/,
                                              double* s_stat /*[kWarps][10]*/,
                                              float* __restrict__ dbias_part,
                                              double* __restrict__ stat_part,
                                              double* __restrict__ max_part) {
  using L = RowLayout<VPL, VEC>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NS = kNumStat + kNumMax;
#pragma unroll
  for (int v = 0; v < VPL; ++v) s_dbias[warp * VPL * 32 + v * 32 + lane] = acc.dbias[v];
  if (!fixup && lane == 0) {
    double* st = s_stat + warp * NS;
    st[kLossNum] = acc.loss_num;
    st[kEntSum] = acc.ent_sum;
    st[kRatioSum] = acc.ratio_sum;
    st[kWSum] = acc.w_sum;
    st[kOutside] = acc.n_out;
    st[kExcluded] = acc.n_excl;
    st[kBadRows] = acc.n_bad;
    st[kBadTok] = acc.n_badtok;
    st[kNumStat + kRatioMax] = acc.rmax;
    st[kNumStat + kNegWMin] = acc.negwmin;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < VPL * 32; idx += kThreads) {
    const int v = idx >> 5, ln = idx & 31;
    const int c = L::col(ln, v);
    if (c < A) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += s_dbias[w * VPL * 32 + idx];
      dbias_part[(int64_t)blockIdx.x * A + c] = s;
    }
  }
  if (!fixup && threadIdx.x == 0) {
    double sum[NS];
#pragma unroll
    for (int i = 0; i < kNumStat; ++i) sum[i] = 0.0;
    sum[kNumStat + kRatioMax] = -CUDART_INF;
    sum[kNumStat + kNegWMin] = -CUDART_INF;
    for (int w = 0; w < kWarps; ++w) {
#pragma unroll
      for (int i = 0; i < kNumStat; ++i) sum[i] += s_stat[w * NS + i];
#pragma unroll
      for (int i = kNumStat; i < NS; ++i) sum[i] = fmax(sum[i], s_stat[w * NS + i]);
    }
#pragma unroll
    for (int i = 0; i < kNumStat; ++i) stat_part[(int64_t)blockIdx.x * kNumStat + i] = sum[i];
    max_part[(int64_t)blockIdx.x * kNumMax + kRatioMax] = sum[kNumStat + kRatioMax];
    max_part[(int64_t)blockIdx.x * kNumMax + kNegWMin] = sum[kNumStat + kNegWMin];
  }
}

// ---- register path (any A <= 1024) -----------------------------------------------
template <int VPL, bool VEC>
__global__ void __launch_bounds__(kThreads, 3)
token_loss_kernel(const float* __restrict__ logits, const float* __restrict__ bias,
                  const int32_t* __restrict__ tokens, const float* __restrict__ lp_old,
                  const float* __restrict__ adv, int64_t M, int K, int A, LossParams prm,
                  const double* __restrict__ fix_stats, float* __restrict__ dlogits,
                  float* __restrict__ lp_new, float* __restrict__ dbias_part,
                  double* __restrict__ stat_part, double* __restrict__ max_part) {
  using L = RowLayout<VPL, VEC>;
  __shared__ float s_dbias[kWarps * VPL * 32];
  __shared__ double s_stat[kWarps * (kNumStat + kNumMax)];
  __shared__ float s_bias[VPL * 32];
  RowCtx cx;
  if (!setup_ctx(prm, fix_stats, cx)) return;
  for (int c = threadIdx.x; c < VPL * 32; c += kThreads) s_bias[c] = c < A ? __ldg(bias + c) : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  LossAcc<VPL> acc;
  acc.init();
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t stride = (int64_t)gridDim.x * kWarps * kRows;
  for (int64_t base = gw * kRows; base < M; base += stride) {
    float z[kRows][VPL];
#pragma unroll
    for (int r = 0; r < kRows; ++r)
      if (base + r < M) L::load(logits + (base + r) * A, lane, A, z[r], true);
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (base + r >= M) break;
      loss_row<VPL, VEC>(z[r], s_bias, base + r, lane, A, K, tokens, lp_old, adv, cx, dlogits,
                         lp_new, acc);
    }
  }
  loss_epilogue<VPL, VEC>(acc, A, cx.fixup, s_dbias, s_stat, dbias_part, stat_part, max_part);
}

// ---- TMA bulk-copy path (A % 4 == 0, 128 <= A <= 1024) ----------------------------
// dynamic smem: [kWarps][kStages][VPL*32] floats, then [kWarps][kStages] mbarriers
template <int VPL>
__global__ void __launch_bounds__(kThreads, 3)
token_loss_tma_kernel(const float* __restrict__ logits, const float* __restrict__ bias,
                      const int32_t* __restrict__ tokens, const float* __restrict__ lp_old,
                      const float* __restrict__ adv, int64_t M, int K, int A, LossParams prm,
                      const double* __restrict__ fix_stats, float* __restrict__ dlogits,
                      float* __restrict__ lp_new, float* __restrict__ dbias_part,
                      double* __restrict__ stat_part, double* __restrict__ max_part) {
  using L = RowLayout<VPL, true>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ float s_dbias[kWarps * VPL * 32];
  __shared__ double s_stat[kWarps * (kNumStat + kNumMax)];
  __shared__ float s_bias[VPL * 32];
  RowCtx cx;
  if (!setup_ctx(prm, fix_stats, cx)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ring = reinterpret_cast<float*>(smem) + (size_t)warp * kStages * VPL * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * kStages * VPL * 32 * 4) +
                   warp * kStages;
  for (int c = threadIdx.x; c < VPL * 32; c += kThreads) s_bias[c] = c < A ? __ldg(bias + c) : 0.f;
  const unsigned row_bytes = (unsigned)A * 4u;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      const int64_t row = gw + s * nw;
      if (row < M) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(ring + s * VPL * 32, logits + row * A, row_bytes, &bars[s]);
      }
    }
  }
  __syncthreads();
  LossAcc<VPL> acc;
  acc.init();
  int j = 0;
  for (int64_t row = gw; row < M; row += nw, ++j) {
    const int s = j % kStages;
    mbar_wait(&bars[s], (unsigned)(j / kStages) & 1u);
    float z[VPL];
    L::load(ring + s * VPL * 32, lane, A, z, false);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      const int64_t next = row + kStages * nw;
      if (next < M) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(ring + s * VPL * 32, logits + next * A, row_bytes, &bars[s]);
      }
    }
    loss_row<VPL, true>(z, s_bias, row, lane, A, K, tokens, lp_old, adv, cx, dlogits, lp_new,
                        acc);
  }
  loss_epilogue<VPL, true>(acc, A, cx.fixup, s_dbias, s_stat, dbias_part, stat_part, max_part);
}

// ---- full-row fast path helpers (A == VPL * 32, VEC layout) -----------------------------
// No per-element column masks; a non-finite logit is detected through the
// FMA pipe: 0 * z is NaN for z = +-inf or NaN, so `chk` (and the entropy sum
// sum e*d) turns NaN exactly when the reference's log_softmax would raise.
// warp max of floats in one CREDUX (sm_100a), NaN-propagating
__device__ __forceinline__ float warp_max_nan(float v) {
  float r;
  asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

template <int VPL>
__device__ __forceinline__ RowStats row_stats_full(float (&z)[VPL], float (&e)[VPL],
                                                   bool with_entropy) {
  RowStats s;
  float mx = z[0];
#pragma unroll
  for (int v = 1; v < VPL; ++v) mx = fmaxf(mx, z[v]);
  mx = warp_max_nan(mx);  // NaN logit -> NaN max; +inf -> inf - inf = NaN below
  float sum = 0.f, sed = 0.f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const float zo = z[v];
    z[v] = zo - mx;
    e[v] = __expf(z[v]);
    sum += fmaf(zo, 0.f, e[v]);  // 0 * (-inf) = NaN: a -inf logit poisons the sum
    if (with_entropy) sed = fmaf(e[v], z[v], sed);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (with_entropy) sed += __shfl_xor_sync(0xffffffffu, sed, o);
  }
  s.inv_s = 1.f / sum;
  s.log_s = __logf(sum);
  s.sd_over_s = sed * s.inv_s;
  s.H = s.log_s - s.sd_over_s;
  s.bad = !isfinite(sum) || !isfinite(mx);
  s.d_tok = mx;  // caller subtracts: d_tok = z_tok - mx
  return s;
}

// Per-token coefficient c (= dloss/dlogp * m) and the statistics terms.
__device__ __forceinline__ float token_coef(float dlt, float a, bool inc, const RowCtx& cx,
                                            double& term_d, double& r_d, double& w_d,
                                            bool& outside) {
  float coef = 0.f;
  term_d = 0.0; r_d = 1.0; w_d = 1.0;
  outside = false;
  if (inc) {
    const float qq = dlt / cx.prm.sigma;
    if (fabsf(dlt) < 60.f && (cx.prm.algo != 0 || qq * qq < 150.f)) {
      float cf, tf, rf, wf;
      token_scalars<float>(dlt, a, cx.prm, cf, tf, rf, wf, outside);
      coef = cf * cx.inv_m;
      term_d = tf; r_d = rf; w_d = wf;
    } else {
      double cd;
      token_scalars<double>((double)dlt, (double)a, cx.prm, cd, term_d, r_d, w_d, outside);
      coef = (float)(cd * cx.inv_m_d);
    }
  }
  return coef;
}

template <int VPL>
__device__ __forceinline__ void acc_token(LossAcc<VPL>& acc, bool inc, bool bad, bool bad_tok,
                                          float H, double term_d, double r_d, double w_d,
                                          bool outside) {
  acc.ent_sum += (double)H;
  acc.n_bad += bad;
  acc.n_badtok += bad_tok;
  if (inc) {
    acc.loss_num += term_d;
    acc.ratio_sum += r_d;
    acc.w_sum += w_d;
    acc.n_out += outside;
    acc.rmax = fmax(acc.rmax, r_d);
    acc.negwmin = fmax(acc.negwmin, -w_d);
  } else {
    ++acc.n_excl;
  }
}

template <int VPL>
__device__ __forceinline__ void stats_epilogue(const LossAcc<VPL>& acc, double* s_stat,
                                               double* __restrict__ stat_part,
                                               double* __restrict__ max_part) {
  constexpr int NS = kNumStat + kNumMax;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    double* st = s_stat + warp * NS;
    st[kLossNum] = acc.loss_num;
    st[kEntSum] = acc.ent_sum;
    st[kRatioSum] = acc.ratio_sum;
    st[kWSum] = acc.w_sum;
    st[kOutside] = acc.n_out;
    st[kExcluded] = acc.n_excl;
    st[kBadRows] = acc.n_bad;
    st[kBadTok] = acc.n_badtok;
    st[kNumStat + kRatioMax] = acc.rmax;
    st[kNumStat + kNegWMin] = acc.negwmin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum[NS];
#pragma unroll
    for (int q = 0; q < kNumStat; ++q) sum[q] = 0.0;
    sum[kNumStat + kRatioMax] = -CUDART_INF;
    sum[kNumStat + kNegWMin] = -CUDART_INF;
    for (int w = 0; w < kWarps; ++w) {
#pragma unroll
      for (int q = 0; q < kNumStat; ++q) sum[q] += s_stat[w * NS + q];
#pragma unroll
      for (int q = kNumStat; q < NS; ++q) sum[q] = fmax(sum[q], s_stat[w * NS + q]);
    }
#pragma unroll
    for (int q = 0; q < kNumStat; ++q) stat_part[(int64_t)blockIdx.x * kNumStat + q] = sum[q];
    max_part[(int64_t)blockIdx.x * kNumMax + kRatioMax] = sum[kNumStat + kRatioMax];
    max_part[(int64_t)blockIdx.x * kNumMax + kNegWMin] = sum[kNumStat + kNegWMin];
  }
}

template <int VPL>
__device__ __forceinline__ void load_row4(const float* __restrict__ row, int lane, int A,
                                          float (&x)[VPL], bool full) {
#pragma unroll
  for (int q = 0; q < VPL / 4; ++q) {
    const int c = q * 128 + lane * 4;
    float4 y = (full || c < A) ? __ldg(reinterpret_cast<const float4*>(row + c))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    x[4 * q] = y.x; x[4 * q + 1] = y.y; x[4 * q + 2] = y.z; x[4 * q + 3] = y.w;
  }
}

// ---- factorized head: logits never materialized ----------------------------------------
// logits[i, k] = H2W[frame_of[i]] + EP[prev(i, k)] + PP[k] + b_head, with
//   H2W = h2 @ W_head^T (frame rows), EP = e_prev @ W_head^T, PP = e_pos @ W_head^T
// (models.py:181-182 distributed over the sum c = h2 + e_prev[prev] + e_pos).
// One warp owns a whole transition (K consecutive token rows): the H2W row is
// streamed once into the warp's smem ring by the bulk-copy engine (kStages
// transitions in flight), EP rows come from L2 (prefetched one token ahead),
// PP + bias sit in smem.  The chosen-token column is handled once per row
// (scalar re-evaluation + single-lane fix-up store), not per element.
// Outputs:
//   dz      f32[M, A]  per-token dlogits (token-major), consumed by the
//                      (prev, k)-grouped row sum for the e_prev / e_pos / W_head terms
//   g_frame f32[F, A]  G = sum_k dz[i, k] written to the transition's frame row
//                      (bootstrap rows are left untouched: pre-zero), consumed
//                      by dW_head += G^T h2 and dh2 = G W_head.
template <int VPL, bool FULL>
__global__ void __launch_bounds__(kThreads, 2)
token_loss_fact_kernel(const float* __restrict__ h2w, const float* __restrict__ ep,
                       const float* __restrict__ pp, const float* __restrict__ bias,
                       const int32_t* __restrict__ frame_of, const int32_t* __restrict__ tokens,
                       const float* __restrict__ lp_old, const float* __restrict__ adv, int64_t N,
                       int K, int A, LossParams prm, const double* __restrict__ fix_stats,
                       float* __restrict__ dz, float* __restrict__ g_frame,
                       float* __restrict__ lp_new, double* __restrict__ stat_part,
                       double* __restrict__ max_part) {
  using L = RowLayout<VPL, true>;
  constexpr int W = VPL * 32;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_stat[kWarps * (kNumStat + kNumMax)];
  RowCtx cx;
  if (!setup_ctx(prm, fix_stats, cx)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // smem: ring [kWarps][kStages][W] | s_pp [K][W] | s_oh [kWarps][W] | bars [kWarps][kStages]
  float* ring = reinterpret_cast<float*>(smem) + (size_t)warp * kStages * W;
  float* s_pp = reinterpret_cast<float*>(smem) + (size_t)kWarps * kStages * W;
  float* s_oh = s_pp + (size_t)K * W + (size_t)warp * W;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_pp + (size_t)K * W + (size_t)kWarps * W) +
                   warp * kStages;
  for (int e = threadIdx.x; e < K * W; e += kThreads) {
    const int k = e / W, c = e % W;
    s_pp[e] = c < A ? __ldg(pp + (int64_t)k * A + c) + __ldg(bias + c) : 0.f;
  }
  for (int c = lane; c < W; c += 32) s_oh[c] = 0.f;
  const unsigned row_bytes = (unsigned)A * 4u;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      const int64_t i = gw + s * nw;
      if (i < N) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(ring + s * W, h2w + (int64_t)__ldg(frame_of + i) * A, row_bytes, &bars[s]);
      }
    }
  }
  __syncthreads();
  LossAcc<VPL> acc;
  acc.init();
  // per-transition scalars are prefetched one transition ahead (lane k < K holds
  // token k and its behavior log-prob)
  int j = 0;
  int fi_n = 0, tok_n = 0;
  float lpo_n = 0.f, a_n = 0.f;
  if (gw < N) {
    fi_n = __ldg(frame_of + gw);
    tok_n = lane < K ? __ldg(tokens + gw * K + lane) : 0;
    lpo_n = lane < K ? __ldg(lp_old + gw * K + lane) : 0.f;
    a_n = __ldg(adv + gw);
  }
  for (int64_t i = gw; i < N; i += nw, ++j) {
    const int s = j % kStages;
    const float* hrow = ring + s * W;
    const int fi = fi_n, tok_l = tok_n;
    const float lpo_l = lpo_n, a = a_n;
    const int64_t next = i + kStages * nw;
    const int f_next = (lane == 0 && next < N) ? __ldg(frame_of + next) : 0;
    if (i + nw < N) {
      const int64_t i2 = i + nw;
      fi_n = __ldg(frame_of + i2);
      tok_n = lane < K ? __ldg(tokens + i2 * K + lane) : 0;
      lpo_n = lane < K ? __ldg(lp_old + i2 * K + lane) : 0.f;
      a_n = __ldg(adv + i2);
    }
    mbar_wait(&bars[s], (unsigned)(j / kStages) & 1u);
    float h[VPL], epn[VPL], g[VPL];
    L::load(hrow, lane, A, h, false);
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] = 0.f;
    load_row4<VPL>(ep + (int64_t)A * A, lane, A, epn, FULL);  // k = 0: chunk-start row
    int tok0 = __shfl_sync(0xffffffffu, tok_l, 0);
    float ep_tok_n = __ldg(ep + (int64_t)A * A + min(max(tok0, 0), A - 1));
    float coef_l = 0.f;  // lane k keeps token k's coefficient for the G one-hot pass
    for (int k = 0; k < K; ++k) {
      const int tok_raw = __shfl_sync(0xffffffffu, tok_l, k);
      const float lpo = __shfl_sync(0xffffffffu, lpo_l, k);
      float z[VPL];
      const float* ppk = s_pp + k * W;
#pragma unroll
      for (int v = 0; v < VPL; ++v) z[v] = (h[v] + epn[v]) + ppk[L::col(lane, v)];
      const bool bad_tok = tok_raw < 0 || tok_raw >= A;
      const int tok = bad_tok ? 0 : tok_raw;
      // the chosen column, evaluated exactly as z[] is: (h + ep) + pp
      const float z_tok = (hrow[tok] + ep_tok_n) + ppk[tok];
      if (k + 1 < K) {  // prefetch the next token's EP row (prev = this token) and column
        const int tn = __shfl_sync(0xffffffffu, tok_l, k + 1);
        const float* er = ep + (int64_t)tok * A;
        load_row4<VPL>(er, lane, A, epn, FULL);
        ep_tok_n = __ldg(er + min(max(tn, 0), A - 1));
      }
      float e[VPL];
      RowStats rs;
      if (FULL) {
        rs = row_stats_full<VPL>(z, e, true);
        rs.d_tok = z_tok - rs.d_tok;
      } else {
        rs = row_stats<VPL, true>(z, e, lane, A, tok, true);
      }
      const int64_t row = i * K + k;
      const float lpn = rs.d_tok - rs.log_s;
      const float dlt = lpn - lpo;
      const bool inc = !bad_tok && !rs.bad && dlt <= 709.78271289f && dlt >= -745.13321910f;
      double term_d, r_d, w_d;
      bool outside;
      const float coef = token_coef(dlt, a, inc, cx, term_d, r_d, w_d, outside);
      // dz = p (ent_scale (d - sd/s) - coef); the +coef at the token column is applied below
      float d[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const float p = e[v] * rs.inv_s;
        float x = p * fmaf(cx.ent_scale, z[v] - rs.sd_over_s, -coef);
        if (!FULL) x = L::col(lane, v) < A ? x : 0.f;
        d[v] = x;
        g[v] += x;
      }
      float* drow = dz + row * A;
      L::store(drow, lane, A, d);
      if (lane == k) coef_l = coef;
      __syncwarp();
      if (lane == 0) {
        const float p_tok = __expf(rs.d_tok) * rs.inv_s;
        drow[tok] = fmaf(p_tok, fmaf(cx.ent_scale, rs.d_tok - rs.sd_over_s, -coef), coef);
        if (!cx.fixup) lp_new[row] = lpn;
      }
      if (!cx.fixup) acc_token(acc, inc, rs.bad, bad_tok, rs.H, term_d, r_d, w_d, outside);
    }
    // slot s is free: refill it with the transition kStages ahead
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      if (next < N) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(ring + s * W, h2w + (int64_t)f_next * A, row_bytes, &bars[s]);
      }
    }
    // one-hot contributions (serial over k in lane order: duplicates accumulate)
    for (int k = 0; k < K; ++k) {
      const int tk = __shfl_sync(0xffffffffu, tok_l, k);
      const float ck = __shfl_sync(0xffffffffu, coef_l, k);
      if (lane == 0 && tk >= 0 && tk < A) s_oh[tk] += ck;
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] += s_oh[L::col(lane, v)];
    L::store(g_frame + (int64_t)fi * A, lane, A, g);
    __syncwarp();
    if (lane < K && tok_l >= 0 && tok_l < A) s_oh[tok_l] = 0.f;
    __syncwarp();
  }
  if (!cx.fixup) stats_epilogue<VPL>(acc, s_stat, stat_part, max_part);
}

// Dprev[j] = sum_k Dpk[j, k], Dpos[k] = sum_j Dpk[j, k]  (Dpk f32[(A+1), K, A])
__global__ void pk_marginals_kernel(const float* __restrict__ dpk, int K, int A, int nprev,
                                    float* __restrict__ dprev, float* __restrict__ dpos) {
  const int64_t total = (int64_t)(nprev + K) * A;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e % A);
    const int64_t r = e / A;
    float s = 0.f;
    if (r < nprev) {
      for (int k = 0; k < K; ++k) s += dpk[(r * K + k) * A + a];
      dprev[r * A + a] = s;
    } else {
      const int k = (int)(r - nprev);
      for (int jj = 0; jj < nprev; ++jj) s += dpk[((int64_t)jj * K + k) * A + a];
      dpos[(int64_t)k * A + a] = s;
    }
  }
}

// ---- behavior log-probs ---------------------------------------------------------------
__device__ __forceinline__ void logp_block_epilogue(int bad_rows, int bad_tok,
                                                    double* __restrict__ bad_part) {
  __shared__ int s_bad[kWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    s_bad[warp][0] = bad_rows;
    s_bad[warp][1] = bad_tok;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int w = 0; w < kWarps; ++w) {
      a += s_bad[w][0];
      b += s_bad[w][1];
    }
    bad_part[2 * (int64_t)blockIdx.x] = a;
    bad_part[2 * (int64_t)blockIdx.x + 1] = b;
  }
}

template <int VPL, bool VEC>
__device__ __forceinline__ void logp_row(float (&z)[VPL], int64_t row, int lane, int A,
                                         const int32_t* __restrict__ tokens,
                                         float* __restrict__ lp_out, int& bad_rows, int& bad_tok) {
  int tok = __ldg(tokens + row);
  const bool bt = tok < 0 || tok >= A;
  if (bt) tok = 0;
  float e[VPL];
  const RowStats rs = row_stats<VPL, VEC>(z, e, lane, A, tok, false);
  if (lane == 0) lp_out[row] = rs.d_tok - rs.log_s;
  bad_rows += rs.bad;
  bad_tok += bt;
}

template <int VPL, bool VEC>
__global__ void __launch_bounds__(kThreads)
token_logp_kernel(const float* __restrict__ mu, const int32_t* __restrict__ tokens, int64_t M,
                  int A, float* __restrict__ lp_out, double* __restrict__ bad_part) {
  using L = RowLayout<VPL, VEC>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int bad_rows = 0, bad_tok = 0;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t stride = (int64_t)gridDim.x * kWarps * kRows;
  for (int64_t base = gw * kRows; base < M; base += stride) {
    float z[kRows][VPL];
#pragma unroll
    for (int r = 0; r < kRows; ++r)
      if (base + r < M) L::load(mu + (base + r) * A, lane, A, z[r], true);
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (base + r >= M) break;
      logp_row<VPL, VEC>(z[r], base + r, lane, A, tokens, lp_out, bad_rows, bad_tok);
    }
  }
  logp_block_epilogue(bad_rows, bad_tok, bad_part);
}

template <int VPL, bool FULL>
__global__ void __launch_bounds__(kThreads, 3)
token_logp_tma_kernel(const float* __restrict__ mu, const int32_t* __restrict__ tokens, int64_t M,
                      int A, float* __restrict__ lp_out, double* __restrict__ bad_part) {
  using L = RowLayout<VPL, true>;
  constexpr int W = VPL * 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ring = reinterpret_cast<float*>(smem) + (size_t)warp * kStages * W;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * kStages * W * 4) +
                   warp * kStages;
  const unsigned row_bytes = (unsigned)A * 4u;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      const int64_t row = gw + s * nw;
      if (row < M) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(ring + s * W, mu + row * A, row_bytes, &bars[s]);
      }
    }
  }
  __syncwarp();
  int bad_rows = 0, bad_tok = 0, j = 0;
  int tok_next = gw < M ? __ldg(tokens + gw) : 0;  // token ids prefetched one row ahead
  for (int64_t row = gw; row < M; row += nw, ++j) {
    const int s = j % kStages;
    const float* slot = ring + s * W;
    const int tok_raw = tok_next;
    if (row + nw < M) tok_next = __ldg(tokens + row + nw);
    mbar_wait(&bars[s], (unsigned)(j / kStages) & 1u);
    float z[VPL], e[VPL];
    L::load(slot, lane, A, z, false);
    const bool bt = tok_raw < 0 || tok_raw >= A;
    const int tok = bt ? 0 : tok_raw;
    RowStats rs;
    if (FULL) {
      rs = row_stats_full<VPL>(z, e, false);
      rs.d_tok = slot[tok] - rs.d_tok;
    } else {
      rs = row_stats<VPL, true>(z, e, lane, A, tok, false);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      lp_out[row] = rs.d_tok - rs.log_s;
      const int64_t next = row + kStages * nw;
      if (next < M) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(ring + s * W, mu + next * A, row_bytes, &bars[s]);
      }
    }
    bad_rows += rs.bad;
    bad_tok += bt;
  }
  logp_block_epilogue(bad_rows, bad_tok, bad_part);
}

// ---- launch plumbing -------------------------------------------------------------------
int grid_for_rows(int64_t M) {
  const int64_t warps_needed = ceil_div(M, kRows);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps_needed, kWarps),
                                                     (int64_t)kNumSMs * 3));
}

size_t tma_smem(int VPL) {
  return (size_t)kWarps * kStages * (VPL * 32 * 4 + sizeof(uint64_t));
}

template <template <int, bool> class Launch, typename... Args>
int dispatch_vpl(int A, Args... args) {
  const bool vec = (A % 4) == 0;
  if (A <= 32) return Launch<1, false>::run(args...);
  if (A <= 64) return Launch<2, false>::run(args...);
  if (A <= 128) return vec ? Launch<4, true>::run(args...) : Launch<4, false>::run(args...);
  if (A <= 256) return vec ? Launch<8, true>::run(args...) : Launch<8, false>::run(args...);
  if (A <= 512) return vec ? Launch<16, true>::run(args...) : Launch<16, false>::run(args...);
  if (A <= 1024) return vec ? Launch<32, true>::run(args...) : Launch<32, false>::run(args...);
  return fail(kDimension, "n_actions=%d exceeds the supported maximum of 1024", A);
}

template <typename KernelT>
int launch_tma(KernelT kernel, int VPL, int grid, cudaStream_t s, const char* name,
               auto... args) {
  const size_t smem = tma_smem(VPL);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(kCuda, "%s smem attribute: %s", name, cudaGetErrorString(e));
  }
  kernel<<<grid, kThreads, smem, s>>>(args...);
  return post_launch(name);
}

template <int VPL, bool VEC>
struct LossLaunch {
  static int run(const float* logits, const float* bias, const int32_t* tokens,
                 const float* lp_old, const float* adv, int64_t M, int K, int A,
                 LossParams prm, const double* fix, float* dlogits, float* lp_new,
                 float* dbias_part, double* stat_part, double* max_part, int grid,
                 cudaStream_t s) {
    if constexpr (VEC && VPL >= 4) {
      return launch_tma(token_loss_tma_kernel<VPL>, VPL, grid, s, "token_loss_tma_kernel",
                        logits, bias, tokens, lp_old, adv, M, K, A, prm, fix, dlogits, lp_new,
                        dbias_part, stat_part, max_part);
    } else {
      token_loss_kernel<VPL, VEC><<<grid, kThreads, 0, s>>>(logits, bias, tokens, lp_old, adv, M,
                                                            K, A, prm, fix, dlogits, lp_new,
                                                            dbias_part, stat_part, max_part);
      return post_launch("token_loss_kernel");
    }
  }
};

template <int VPL, bool VEC>
struct LogpLaunch {
  static int run(const float* mu, const int32_t* tokens, int64_t M, int A, float* lp,
                 double* bad_part, int grid, cudaStream_t s) {
    if constexpr (VEC && VPL >= 4) {
      if (A == VPL * 32)
        return launch_tma(token_logp_tma_kernel<VPL, true>, VPL, grid, s,
                          "token_logp_tma_kernel", mu, tokens, M, A, lp, bad_part);
      return launch_tma(token_logp_tma_kernel<VPL, false>, VPL, grid, s, "token_logp_tma_kernel",
                        mu, tokens, M, A, lp, bad_part);
    } else {
      token_logp_kernel<VPL, VEC><<<grid, kThreads, 0, s>>>(mu, tokens, M, A, lp, bad_part);
      return post_launch("token_logp_kernel");
    }
  }
};

bool misaligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) & 15; }

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_token_grid(int64_t M) { return M > 0 ? grid_for_rows(M) : 1; }

extern "C" int accel_fact_grid(int64_t N) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(N, kWarps), (int64_t)kNumSMs * 2));
}

extern "C" int accel_token_loss_fact(const float* h2w, const float* ep, const float* pp,
                                     const float* bias, const int32_t* frame_of,
                                     const int32_t* tokens, const float* lp_old, const float* adv,
                                     int64_t N, int K, int A, int algo, double sigma,
                                     double clip_eps, double lambda_h, double m_global,
                                     const double* fix_stats, float* dz, float* g_frame,
                                     float* lp_new, double* stat_part, double* max_part,
                                     void* stream) {
  if (algo != 0 && algo != 1) return fail(kDomain, "unknown algorithm %d", algo);
  if (!(sigma > 0)) return fail(kDomain, "sigma must be > 0, got %g", sigma);
  if (!(clip_eps > 0 && clip_eps < 1)) return fail(kDomain, "clip_eps must be in (0, 1)");
  if (lambda_h < 0) return fail(kDomain, "loss coefficients must be >= 0");
  if (N < 0 || K < 1 || K > 32 || A < 1) return fail(kDimension, "token_loss_fact: bad sizes");
  if (A % 4 != 0 || A < 128 || A > 1024)
    return fail(kDimension, "token_loss_fact needs 128 <= A <= 1024, A %% 4 == 0 (got %d)", A);
  if (N == 0) return kOk;
  if (!(m_global >= (double)(N * K))) return fail(kDimension, "m_global < local token count");
  if (!h2w || !ep || !pp || !bias || !frame_of || !tokens || !lp_old || !adv || !dz || !g_frame ||
      (!fix_stats && (!lp_new || !stat_part || !max_part)))
    return fail(kDimension, "token_loss_fact: NULL buffer");
  if (misaligned16(h2w) || misaligned16(ep) || misaligned16(dz) || misaligned16(g_frame))
    return fail(kDimension, "token_loss_fact: buffers must be 16B aligned");
  LossParams prm;
  prm.algo = algo;
  prm.sigma = (float)sigma;
  prm.clip_lo = (float)(1.0 - clip_eps);
  prm.clip_hi = (float)(1.0 + clip_eps);
  prm.lambda_h = (float)lambda_h;
  prm.inv_nk = 1.0 / m_global;
  prm.m_global = m_global;
  cudaStream_t s = as_stream(stream);
  const int grid = accel_fact_grid(N);
  auto go = [&](auto kernel, int VPL) -> int {
    const size_t smem = (size_t)kWarps * kStages * (VPL * 32 * 4 + sizeof(uint64_t)) +
                        (size_t)K * VPL * 32 * 4 + (size_t)kWarps * VPL * 32 * 4 + 16;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return fail(kCuda, "token_loss_fact smem: %s", cudaGetErrorString(e));
    }
    kernel<<<grid, kThreads, smem, s>>>(h2w, ep, pp, bias, frame_of, tokens, lp_old, adv, N, K, A,
                                        prm, fix_stats, dz, g_frame, lp_new, stat_part, max_part);
    return post_launch("token_loss_fact_kernel");
  };
  const bool full = A == 128 || A == 256 || A == 512 || A == 1024;
  if (A <= 128) return full ? go(token_loss_fact_kernel<4, true>, 4) : go(token_loss_fact_kernel<4, false>, 4);
  if (A <= 256) return full ? go(token_loss_fact_kernel<8, true>, 8) : go(token_loss_fact_kernel<8, false>, 8);
  if (A <= 512) return full ? go(token_loss_fact_kernel<16, true>, 16) : go(token_loss_fact_kernel<16, false>, 16);
  return full ? go(token_loss_fact_kernel<32, true>, 32) : go(token_loss_fact_kernel<32, false>, 32);
}

extern "C" int accel_pk_marginals(const float* dpk, int K, int A, float* dprev, float* dpos,
                                  void* stream) {
  if (K < 1 || A < 1 || !dpk || !dprev || !dpos) return fail(kDimension, "pk_marginals: bad args");
  const int nprev = A + 1;
  const int64_t total = (int64_t)(nprev + K) * A;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)kNumSMs * 4);
  pk_marginals_kernel<<<grid, 256, 0, as_stream(stream)>>>(dpk, K, A, nprev, dprev, dpos);
  return post_launch("pk_marginals_kernel");
}

extern "C" int accel_token_logp(const float* mu, const int32_t* tokens, int64_t M, int A,
                                float* lp_out, double* bad_part, void* stream) {
  if (M < 0 || A < 1) return fail(kDimension, "token_logp: bad sizes M=%lld A=%d",
                                  (long long)M, A);
  if (M == 0) return kOk;
  if (!mu || !tokens || !lp_out || !bad_part) return fail(kDimension, "token_logp: NULL buffer");
  if (A % 4 == 0 && misaligned16(mu)) return fail(kDimension, "token_logp: mu not 16B aligned");
  return dispatch_vpl<LogpLaunch>(A, mu, tokens, M, A, lp_out, bad_part, grid_for_rows(M),
                                  as_stream(stream));
}

extern "C" int accel_token_loss(const float* logits, const float* bias, const int32_t* tokens,
                                const float* lp_old, const float* adv, int64_t M, int K, int A,
                                int algo, double sigma, double clip_eps, double lambda_h,
                                double m_global, const double* fix_stats, float* dlogits,
                                float* lp_new, float* dbias_part, double* stat_part,
                                double* max_part, void* stream) {
  if (algo != 0 && algo != 1) return fail(kDomain, "unknown algorithm %d", algo);
  if (!(sigma > 0)) return fail(kDomain, "sigma must be > 0, got %g", sigma);
  if (!(clip_eps > 0 && clip_eps < 1)) return fail(kDomain, "clip_eps must be in (0, 1)");
  if (lambda_h < 0) return fail(kDomain, "loss coefficients must be >= 0");
  if (M < 0 || K < 1 || A < 1 || M % K) return fail(kDimension, "token_loss: bad sizes");
  if (M == 0) return kOk;
  if (!(m_global >= (double)M)) return fail(kDimension, "m_global < local token count");
  if (!logits || !bias || !tokens || !lp_old || !adv || !dlogits || !dbias_part ||
      (!fix_stats && (!lp_new || !stat_part || !max_part)))
    return fail(kDimension, "token_loss: NULL buffer");
  if (A % 4 == 0 && (misaligned16(logits) || misaligned16(dlogits)))
    return fail(kDimension, "token_loss: logits/dlogits not 16B aligned");
  LossParams prm;
  prm.algo = algo;
  prm.sigma = (float)sigma;
  prm.clip_lo = (float)(1.0 - clip_eps);
  prm.clip_hi = (float)(1.0 + clip_eps);
  prm.lambda_h = (float)lambda_h;
  prm.inv_nk = 1.0 / m_global;
  prm.m_global = m_global;
  return dispatch_vpl<LossLaunch>(A, logits, bias, tokens, lp_old, adv, M, K, A, prm, fix_stats,
                                  dlogits, lp_new, dbias_part, stat_part, max_part,
                                  grid_for_rows(M), as_stream(stream));
}
