// Shared device code of the token-row kernels (token_loss.cu, token_fact.cu).
//
// Reference semantics implemented here: log_softmax / softmax (numerics.py:133-151),
// the surrogate per-token algebra of policy_surrogate (trainer.py:183-239), and
// the entropy term of entropy_bonus (trainer.py:242-251).
#pragma once

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
  float inv_m, ent_scale, inv_sigma;
  double inv_m_d;
  bool fixup;
};

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
  cx.inv_sigma = 1.f / prm.sigma;
  return true;
}

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

// Log-partition of a full row for the behavior log-prob pass (no entropy):
// log2 domain (one FFMA folds the shift and the log2(e) scale), packed fp32x2
// arithmetic, SFU exponentials.  A -inf logit still poisons the sum (0 * -inf).
template <int VPL>
__device__ __forceinline__ RowStats row_stats_logp(const float (&z)[VPL]) {
  static_assert(VPL % 2 == 0, "pairs");
  constexpr float kL2e = 1.4426950408889634f, kLn2f = 0.6931471805599453f;
  RowStats s;
  float mx = z[0];
#pragma unroll
  for (int v = 1; v < VPL; ++v) mx = fmaxf(mx, z[v]);
  mx = warp_max_nan(mx);  // NaN logit -> NaN max; +inf -> inf - inf = NaN below
  const float2 l2 = make_float2(kL2e, kL2e), n2 = make_float2(-mx * kL2e, -mx * kL2e);
  const float2 zero2 = make_float2(0.f, 0.f);
  float2 s2 = zero2;
#pragma unroll
  for (int p = 0; p < VPL / 2; ++p) {
    const float2 zz = make_float2(z[2 * p], z[2 * p + 1]);
    const float2 d = __ffma2_rn(zz, l2, n2);
    float2 e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(d.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(d.y));
    s2 = __fadd2_rn(__ffma2_rn(zz, zero2, s2), e);
  }
  float sum = s2.x + s2.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(sum));
  s.log_s = lg * kLn2f;
  s.inv_s = 0.f;
  s.sd_over_s = 0.f;
  s.H = 0.f;
  s.bad = !isfinite(sum) || !isfinite(mx);
  s.d_tok = mx;  // caller subtracts: d_tok = z_tok - mx
  return s;
}

// The rare float64 tail of token_coef, kept out of line so its register
// footprint does not size the hot loop; results come back by value (taking the
// callers' addresses would push their statistics to local memory every token).
struct CoefTail {
  double term, r, w;
  float coef;
  int outside;
};
__device__ __noinline__ CoefTail token_coef_f64(float dlt, float a, LossParams prm, double inv_m_d) {
  CoefTail o;
  double cd;
  bool out;
  token_scalars<double>((double)dlt, (double)a, prm, cd, o.term, o.r, o.w, out);
  o.coef = (float)(cd * inv_m_d);
  o.outside = out;
  return o;
}

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp)
__device__ __forceinline__ float ex2_sfu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Per-token coefficient c (= dloss/dlogp * m) and the statistics terms.  The
// common path is float with SFU exponentials (r = e^dlt, w = e^(-q^2/2)); the
// float64 tail takes |dlt| >= 60 or trust weights below e^-75.
__device__ __forceinline__ float token_coef(float dlt, float a, bool inc, const RowCtx& cx,
                                            double& term_d, double& r_d, double& w_d,
                                            bool& outside) {
  constexpr float kL2e = 1.4426950408889634f;
  float coef = 0.f;
  term_d = 0.0; r_d = 1.0; w_d = 1.0;
  outside = false;
  if (inc) {
    const float qq = dlt * cx.inv_sigma;
    if (fabsf(dlt) < 60.f && (cx.prm.algo != 0 || qq * qq < 150.f)) {
      const float r = ex2_sfu(dlt * kL2e);
      float w = 1.f, term, cf;
      if (cx.prm.algo == 0) {
        w = ex2_sfu(-0.5f * kL2e * qq * qq);
        term = w * r * a;
        cf = -term;
      } else {
        const float rc = fminf(fmaxf(r, cx.prm.clip_lo), cx.prm.clip_hi);
        const float ra = r * a, rca = rc * a;
        term = fminf(ra, rca);
        cf = ra <= rca ? -ra : 0.f;
        outside = r < cx.prm.clip_lo || r > cx.prm.clip_hi;
      }
      coef = cf * cx.inv_m;
      term_d = term; r_d = r; w_d = w;
    } else {
      const CoefTail o = token_coef_f64(dlt, a, cx.prm, cx.inv_m_d);
      coef = o.coef;
      term_d = o.term; r_d = o.r; w_d = o.w;
      outside = o.outside;
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

__host__ __device__ __forceinline__ bool misaligned16(const void* p) {
  return reinterpret_cast<uintptr_t>(p) & 15;
}

}  // namespace
}  // namespace accel
