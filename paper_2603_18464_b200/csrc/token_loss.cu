// (b) Token-level loss over action-vocabulary logits.
//
//   K3 token_logp  — behavior_log_probs (trainer.py:289-293):
//                    log_softmax(mu)[token] per token row.
//   K4 token_loss  — log_prob_chunk (models.py:219-223) + policy_surrogate
//                    (trainer.py:183-239, GIPO "trust" and PPO "clip") +
//                    entropy_bonus (:242-251) + the dlogits assembly of
//                    train_step (:425-435), forward AND backward in one pass:
//                    each logit row is read once and its dlogits row written
//                    once (2*A*4 + 13 B/token, HBM-bound).
//
// Layout: warp-per-row; each lane holds VPL logits of the row (float4 loads
// when A % 4 == 0).  Row statistics (max, sum-exp, entropy) use xor-shuffle
// butterflies (deterministic).  Per-token scalar algebra is float except the
// rare tails (|log-ratio| >= 60 or a trust weight below e^-75) which switch
// to float64 so ratio overflow/underflow follows the reference's float64
// exclusion rule (isfinite(r) & r > 0, trainer.py:204-205).
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
constexpr int kRows = 2;  // rows in flight per warp

// per-block float64 partial sums (order matters: see accel.h LOSS_STAT_*)
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
  __device__ __forceinline__ static void load(const float* __restrict__ row, int lane, int A,
                                              float (&z)[VPL]) {
    if (VEC) {
#pragma unroll
      for (int q = 0; q < VPL / 4; ++q) {
        const int c = q * 128 + lane * 4;
        float4 x = c < A ? __ldcs(reinterpret_cast<const float4*>(row + c))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        z[4 * q] = x.x; z[4 * q + 1] = x.y; z[4 * q + 2] = x.z; z[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = v * 32 + lane;
        z[v] = c < A ? __ldcs(row + c) : 0.f;
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

struct RowStats {
  float mx, lse, inv_s, H, z_tok;
  bool bad;
};

// log-sum-exp, softmax denominator, entropy and the chosen-token logit.
template <int VPL, bool VEC>
__device__ __forceinline__ RowStats row_stats(const float (&z)[VPL], int lane, int A, int tok,
                                              bool with_entropy) {
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
  float sum = 0.f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) sum += L::col(lane, v) < A ? __expf(z[v] - mx) : 0.f;
  sum = warp_sum(sum);
  s.mx = mx;
  s.inv_s = 1.f / sum;
  s.lse = mx + __logf(sum);
  s.H = 0.f;
  if (with_entropy) {
    float acc = 0.f;
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      if (L::col(lane, v) < A) {
        const float p = __expf(z[v] - mx) * s.inv_s;
        acc = fmaf(p, z[v] - s.lse, acc);
      }
    s.H = -warp_sum(acc);
  }
  int tl, tv;
  L::locate(tok, tl, tv);
  float pick = 0.f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) pick = (v == tv) ? z[v] : pick;
  s.z_tok = __shfl_sync(0xffffffffu, pick, tl);
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

template <int VPL, bool VEC>
__global__ void __launch_bounds__(kThreads, 3)
token_loss_kernel(const float* __restrict__ logits, const float* __restrict__ bias,
                  const int32_t* __restrict__ tokens, const float* __restrict__ lp_old,
                  const float* __restrict__ adv, int64_t M, int K, int A, LossParams prm,
                  const double* __restrict__ fix_stats, float* __restrict__ dlogits,
                  float* __restrict__ lp_new, float* __restrict__ dbias_part,
                  double* __restrict__ stat_part, double* __restrict__ max_part) {
  using L = RowLayout<VPL, VEC>;
  __shared__ float s_dbias[kWarps][VPL * 32];
  __shared__ double s_stat[kWarps][kNumStat + kNumMax];

  const bool fixup = fix_stats != nullptr;
  double m_eff = prm.m_global;
  if (fixup) {
    const double excl = fix_stats[kExcluded];
    if (excl == 0.0 || excl >= prm.m_global) return;  // uniform early exit
    m_eff = prm.m_global - excl;
  }
  const float inv_m = (float)(1.0 / m_eff);
  const double inv_m_d = 1.0 / m_eff;
  const float ent_scale = prm.lambda_h * (float)prm.inv_nk;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float s_bias[VPL * 32];
  for (int c = threadIdx.x; c < VPL * 32; c += kThreads) s_bias[c] = c < A ? __ldg(bias + c) : 0.f;
  __syncthreads();
  float dbias[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) dbias[v] = 0.f;
  // float64 sums; integer counters
  double loss_num = 0.0, ent_sum = 0.0, ratio_sum = 0.0, w_sum = 0.0;
  int n_out = 0, n_excl = 0, n_bad = 0, n_badtok = 0;
  double rmax = -CUDART_INF, negwmin = -CUDART_INF;

  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t stride = (int64_t)gridDim.x * kWarps * kRows;
  for (int64_t base = gw * kRows; base < M; base += stride) {
    float z[kRows][VPL];
#pragma unroll
    for (int r = 0; r < kRows; ++r)
      if (base + r < M) L::load(logits + (base + r) * A, lane, A, z[r]);
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int64_t row = base + r;
      if (row >= M) break;
#pragma unroll
      for (int v = 0; v < VPL; ++v) z[r][v] += s_bias[L::col(lane, v)];
      int tok = __ldg(tokens + row);
      const bool bad_tok = tok < 0 || tok >= A;
      if (bad_tok) tok = 0;
      const RowStats rs = row_stats<VPL, VEC>(z[r], lane, A, tok, true);
      const float lpn = rs.z_tok - rs.lse;
      const float dlt = lpn - __ldg(lp_old + row);
      const float a = __ldg(adv + row / K);
      // reference exclusion: exp(delta) in float64 finite and > 0
      const bool inc = !bad_tok && !rs.bad && dlt <= 709.78271289f && dlt >= -745.13321910f;
      float coef = 0.f;
      double term_d = 0.0, r_d = 1.0, w_d = 1.0;
      bool outside = false;
      if (inc) {
        const float qq = dlt / prm.sigma;
        if (fabsf(dlt) < 60.f && (prm.algo != 0 || qq * qq < 150.f)) {
          float cf, tf, rf, wf;
          token_scalars<float>(dlt, a, prm, cf, tf, rf, wf, outside);
          coef = cf * inv_m;
          term_d = tf; r_d = rf; w_d = wf;
        } else {
          double cd;
          token_scalars<double>((double)dlt, (double)a, prm, cd, term_d, r_d, w_d, outside);
          coef = (float)(cd * inv_m_d);
        }
      }
      // dlogits = dlogp (onehot - p) + lambda_h p (lp + H) / (N K)
      float d[VPL];
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = L::col(lane, v);
        const float p = __expf(z[r][v] - rs.mx) * rs.inv_s;
        const float lp = z[r][v] - rs.lse;
        float g = coef * ((c == tok ? 1.f : 0.f) - p) + ent_scale * p * (lp + rs.H);
        g = c < A ? g : 0.f;
        d[v] = g;
        dbias[v] += g;
      }
      L::store(dlogits + row * A, lane, A, d);
      if (!fixup) {
        if (lane == 0) lp_new[row] = lpn;
        ent_sum += (double)rs.H;
        n_bad += rs.bad;
        n_badtok += bad_tok;
        if (inc) {
          loss_num += term_d;
          ratio_sum += r_d;
          w_sum += w_d;
          n_out += outside;
          rmax = fmax(rmax, r_d);
          negwmin = fmax(negwmin, -w_d);
        } else {
          ++n_excl;
        }
      }
    }
  }

  // fixed-order block reduction of the bias gradient
#pragma unroll
  for (int v = 0; v < VPL; ++v) s_dbias[warp][v * 32 + lane] = dbias[v];
  if (!fixup && lane == 0) {
    s_stat[warp][kLossNum] = loss_num;
    s_stat[warp][kEntSum] = ent_sum;
    s_stat[warp][kRatioSum] = ratio_sum;
    s_stat[warp][kWSum] = w_sum;
    s_stat[warp][kOutside] = n_out;
    s_stat[warp][kExcluded] = n_excl;
    s_stat[warp][kBadRows] = n_bad;
    s_stat[warp][kBadTok] = n_badtok;
    s_stat[warp][kNumStat + kRatioMax] = rmax;
    s_stat[warp][kNumStat + kNegWMin] = negwmin;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < VPL * 32; idx += kThreads) {
    const int v = idx >> 5, ln = idx & 31;
    const int c = L::col(ln, v);
    if (c < A) {
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) acc += s_dbias[w][idx];
      dbias_part[(int64_t)blockIdx.x * A + c] = acc;
    }
  }
  if (!fixup && threadIdx.x == 0) {
    double acc[kNumStat + kNumMax];
#pragma unroll
    for (int i = 0; i < kNumStat; ++i) acc[i] = 0.0;
    acc[kNumStat + kRatioMax] = -CUDART_INF;
    acc[kNumStat + kNegWMin] = -CUDART_INF;
    for (int w = 0; w < kWarps; ++w) {
#pragma unroll
      for (int i = 0; i < kNumStat; ++i) acc[i] += s_stat[w][i];
      acc[kNumStat + kRatioMax] = fmax(acc[kNumStat + kRatioMax], s_stat[w][kNumStat + kRatioMax]);
      acc[kNumStat + kNegWMin] = fmax(acc[kNumStat + kNegWMin], s_stat[w][kNumStat + kNegWMin]);
    }
#pragma unroll
    for (int i = 0; i < kNumStat; ++i) stat_part[(int64_t)blockIdx.x * kNumStat + i] = acc[i];
    max_part[(int64_t)blockIdx.x * kNumMax + kRatioMax] = acc[kNumStat + kRatioMax];
    max_part[(int64_t)blockIdx.x * kNumMax + kNegWMin] = acc[kNumStat + kNegWMin];
  }
}

template <int VPL, bool VEC>
__global__ void __launch_bounds__(kThreads)
token_logp_kernel(const float* __restrict__ mu, const int32_t* __restrict__ tokens, int64_t M,
                  int A, float* __restrict__ lp_out, double* __restrict__ bad_part) {
  using L = RowLayout<VPL, VEC>;
  __shared__ double s_bad[kWarps][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double bad_rows = 0.0, bad_tok = 0.0;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t stride = (int64_t)gridDim.x * kWarps * kRows;
  for (int64_t base = gw * kRows; base < M; base += stride) {
    float z[kRows][VPL];
#pragma unroll
    for (int r = 0; r < kRows; ++r)
      if (base + r < M) L::load(mu + (base + r) * A, lane, A, z[r]);
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int64_t row = base + r;
      if (row >= M) break;
      int tok = __ldg(tokens + row);
      const bool bt = tok < 0 || tok >= A;
      if (bt) tok = 0;
      const RowStats rs = row_stats<VPL, VEC>(z[r], lane, A, tok, false);
      if (lane == 0) lp_out[row] = rs.z_tok - rs.lse;
      bad_rows += rs.bad ? 1.0 : 0.0;
      bad_tok += bt ? 1.0 : 0.0;
    }
  }
  if (lane == 0) {
    s_bad[warp][0] = bad_rows;
    s_bad[warp][1] = bad_tok;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kWarps; ++w) {
      a += s_bad[w][0];
      b += s_bad[w][1];
    }
    bad_part[2 * (int64_t)blockIdx.x] = a;
    bad_part[2 * (int64_t)blockIdx.x + 1] = b;
  }
}

int grid_for_rows(int64_t M) {
  const int64_t warps_needed = ceil_div(M, kRows);
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps_needed, kWarps),
                                                     (int64_t)kNumSMs * 6));
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

template <int VPL, bool VEC>
struct LossLaunch {
  static int run(const float* logits, const float* bias, const int32_t* tokens,
                 const float* lp_old, const float* adv, int64_t M, int K, int A,
                 LossParams prm, const double* fix, float* dlogits, float* lp_new,
                 float* dbias_part, double* stat_part, double* max_part, int grid,
                 cudaStream_t s) {
    token_loss_kernel<VPL, VEC><<<grid, kThreads, 0, s>>>(logits, bias, tokens, lp_old, adv, M,
                                                          K, A, prm, fix, dlogits, lp_new,
                                                          dbias_part, stat_part, max_part);
    return post_launch("token_loss_kernel");
  }
};

template <int VPL, bool VEC>
struct LogpLaunch {
  static int run(const float* mu, const int32_t* tokens, int64_t M, int A, float* lp,
                 double* bad_part, int grid, cudaStream_t s) {
    token_logp_kernel<VPL, VEC><<<grid, kThreads, 0, s>>>(mu, tokens, M, A, lp, bad_part);
    return post_launch("token_logp_kernel");
  }
};

bool misaligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) & 15; }

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_token_grid(int64_t M) { return M > 0 ? grid_for_rows(M) : 1; }

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
