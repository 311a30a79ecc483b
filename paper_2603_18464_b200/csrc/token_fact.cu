// (b) Fused token loss with a factorized policy head: logits never exist in HBM.
//
// Reference: log_prob_chunk (models.py:219-223), policy_surrogate
// (trainer.py:183-239), entropy_bonus (trainer.py:242-251) and the dlogits
// assembly of train_step (trainer.py:425-435), with the head's logits
// (models.py:181-182) distributed over c = h2 + e_prev[prev] + e_pos:
//   logits[i, k] = H2W[frame_of[i]] + EPP[prev(i, k) * K + k]
//   H2W = h2 @ W_head^T (one row per frame)
//   EPP = e_prev @ W_head^T + e_pos @ W_head^T + b_head   ((A+1) * K rows, L2-resident)
// One warp owns a whole transition (K consecutive token rows).  Its H2W row is
// streamed once into a per-warp shared-memory ring by the bulk-copy (TMA)
// engine, kStages transitions in flight; the EPP row of the next token is
// prefetched into registers while the current token is processed.
//
// Per logit: 1 FADD (z), 1 FFMA + ex2 (p in the log2 domain, ftz), 1 FADD +
// 1 FFMA (partition sums), 1 FFMA + 1 FMUL (gradient), 1 FADD (G): the row
// max is one CREDUX, the chosen-token column is evaluated once per row and
// patched by a single lane, the float64 statistics are accumulated once per
// transition per lane.  Non-finite logits surface as a non-finite max, sum
// or sum(e*d) (0 * -inf = NaN), exactly where the reference's log_softmax
// raises.  Outputs:
//   dz      f32[M, A]  per-token dlogits (token-major) for the (prev, k)-grouped sums
//   g_frame f32[F, A]  G = sum_k dz[i, k] on the transition's frame row
#include "token_common.cuh"

namespace accel {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kGS = 2;  // H2W ring depth (transitions in flight per group) of the grouped kernel

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// epp[(prev * K + k) * A + a] = ep[prev * A + a] + pp[k * A + a] + bias[a]
__global__ void ep_plus_kernel(const float* __restrict__ ep, const float* __restrict__ pp,
                               const float* __restrict__ bias, int A, int K,
                               float* __restrict__ epp) {
  const int64_t total = (int64_t)(A + 1) * K * A;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e % A);
    const int64_t r = e / A;
    const int k = (int)(r % K);
    const int64_t prev = r / K;
    epp[e] = ep[prev * A + a] + pp[(int64_t)k * A + a] + bias[a];
  }
}

template <int VPL>
__device__ __forceinline__ void load_vec(const float* __restrict__ row, int lane, int A,
                                         float (&x)[VPL], bool full) {
#pragma unroll
  for (int q = 0; q < VPL / 4; ++q) {
    const int c = q * 128 + lane * 4;
    const float4 y = (full || c < A) ? __ldg(reinterpret_cast<const float4*>(row + c))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    x[4 * q] = y.x; x[4 * q + 1] = y.y; x[4 * q + 2] = y.z; x[4 * q + 3] = y.w;
  }
}

template <int VPL, bool FULL>
__global__ void __launch_bounds__(kThreads, 2)
token_loss_fact_kernel(const float* __restrict__ h2w, const float* __restrict__ epp,
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
  // smem: ring [kWarps][kStages][W] | s_oh [kWarps][W] | bars [kWarps][kStages]
  float* ring = reinterpret_cast<float*>(smem) + (size_t)warp * kStages * W;
  float* s_oh = reinterpret_cast<float*>(smem) + (size_t)kWarps * kStages * W + (size_t)warp * W;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(smem) +
                                               (size_t)kWarps * (kStages + 1) * W) +
                   warp * kStages;
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
  __syncwarp();
  const float ent2 = cx.ent_scale * kLn2;
  // per-lane statistics (lane k accumulates token k of every transition)
  double st_loss = 0.0, st_ent = 0.0, st_r = 0.0, st_w = 0.0;
  double st_rmax = -CUDART_INF, st_negw = -CUDART_INF;
  int st_out = 0, st_excl = 0, st_bad = 0, st_badtok = 0;

  // per-transition scalars prefetched one transition ahead
  int fi_n = 0, tok_n = 0;
  float lpo_n = 0.f, a_n = 0.f;
  if (gw < N) {
    fi_n = __ldg(frame_of + gw);
    tok_n = lane < K ? __ldg(tokens + gw * K + lane) : 0;
    lpo_n = lane < K ? __ldg(lp_old + gw * K + lane) : 0.f;
    a_n = __ldg(adv + gw);
  }
  int j = 0;
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
    // EPP row of token 0 (prev = chunk start A) and its chosen column
    const int tok0 = min(max(__shfl_sync(0xffffffffu, tok_l, 0), 0), A - 1);
    float epn[VPL];
    const float* er0 = epp + (int64_t)A * K * A;
    load_vec<VPL>(er0, lane, A, epn, FULL);
    float ep_tok = __ldg(er0 + tok0);
    mbar_wait(&bars[s], (unsigned)(j / kStages) & 1u);
    __syncwarp();  // reconverge: lanes may leave the spin-wait at different times
    float g[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] = 0.f;
    float my_coef = 0.f, my_H = 0.f;
    double my_term = 0.0, my_r = 1.0, my_w = 1.0;
    bool my_inc = false, my_bad = false, my_badtok = false, my_out = false;
    for (int k = 0; k < K; ++k) {
      const int tok_raw = __shfl_sync(0xffffffffu, tok_l, k);
      const float lpo = __shfl_sync(0xffffffffu, lpo_l, k);
      const bool bad_tok = tok_raw < 0 || tok_raw >= A;
      const int tok = bad_tok ? 0 : tok_raw;
      float z[VPL];
      L::load(hrow, lane, A, z, false);  // H2W row from the smem ring (re-read per token)
#pragma unroll
      for (int v = 0; v < VPL; ++v) z[v] += epn[v];
      const float z_tok = hrow[tok] + ep_tok;  // same arithmetic as z[] at column tok
      if (k + 1 < K) {  // prefetch the next token's EPP row (prev = this token) and column
        const int tn = min(max(__shfl_sync(0xffffffffu, tok_l, k + 1), 0), A - 1);
        const float* er = epp + ((int64_t)tok * K + k + 1) * A;
        load_vec<VPL>(er, lane, A, epn, FULL);
        ep_tok = __ldg(er + tn);
      }
      // row max (one CREDUX), partition sums in the log2 domain
      float mx = z[0];
#pragma unroll
      for (int v = 1; v < VPL; ++v) mx = fmaxf(mx, FULL || L::col(lane, v) < A ? z[v] : mx);
      mx = warp_max_nan(mx);
      const float nm2 = -mx * kLog2e;
      float e[VPL], sum = 0.f, sed = 0.f;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        z[v] = fmaf(z[v], kLog2e, nm2);  // d2 = (z - max) log2(e)
        e[v] = (FULL || L::col(lane, v) < A) ? ex2_ftz(z[v]) : 0.f;
        sum += e[v];
        sed = fmaf(e[v], z[v], sed);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        sed += __shfl_xor_sync(0xffffffffu, sed, o);
      }
      const bool bad = !isfinite(sum) || !isfinite(sed) || !isfinite(mx);
      const float inv_s = 1.f / sum;
      const float log_s = __logf(sum);
      const float sd2 = sed * inv_s;  // sum_a p_a d2_a
      const float H = log_s - sd2 * kLn2;
      const float d_tok = z_tok - mx;
      const float lpn = d_tok - log_s;
      const float dlt = lpn - lpo;
      const bool inc = !bad_tok && !bad && dlt <= 709.78271289f && dlt >= -745.13321910f;
      double term_d, r_d, w_d;
      bool outside;
      const float coef = token_coef(dlt, a, inc, cx, term_d, r_d, w_d, outside);
      // dz = p (ent (d - sum p d) - coef) = e * (Ac d2 + Cc)   (+coef at the token column)
      const float Ac = ent2 * inv_s;
      const float Cc = -(Ac * sd2) - coef * inv_s;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        e[v] *= fmaf(Ac, z[v], Cc);  // e[] now holds this row's dlogits
        g[v] += e[v];
      }
      const int64_t row = i * K + k;
      float* drow = dz + row * A;
      L::store(drow, lane, A, e);
      __syncwarp();
      if (lane == 0) {
        const float d2t = fmaf(z_tok, kLog2e, nm2);
        drow[tok] = fmaf(ex2_ftz(d2t), fmaf(Ac, d2t, Cc), coef);
        if (!cx.fixup) lp_new[row] = lpn;
      }
      // lane k keeps token k's scalars (predicated selects, no branch)
      const bool mine = lane == k;
      my_coef = mine ? coef : my_coef;
      my_H = mine ? H : my_H;
      my_term = mine ? term_d : my_term;
      my_r = mine ? r_d : my_r;
      my_w = mine ? w_d : my_w;
      my_inc = mine ? inc : my_inc;
      my_bad = mine ? bad : my_bad;
      my_badtok = mine ? bad_tok : my_badtok;
      my_out = mine ? outside : my_out;
    }
    // slot s is free: refill it with the transition kStages ahead
    // (no proxy fence: the slot's generic reads were consumed before this point;
    // a bulk copy issued after them cannot overtake them -- WAR, as in TMA pipelines)
    __syncwarp();
    if (lane == 0 && next < N) {
      mbar_expect_tx(&bars[s], row_bytes);
      bulk_g2s(ring + s * W, h2w + (int64_t)f_next * A, row_bytes, &bars[s]);
    }
    // one-hot part of G: sum_k coef_k [a == tok_k] (lane order: duplicates accumulate)
    for (int k = 0; k < K; ++k) {
      const int tk = __shfl_sync(0xffffffffu, tok_l, k);
      const float ck = __shfl_sync(0xffffffffu, my_coef, k);
      if (lane == 0 && tk >= 0 && tk < A) s_oh[tk] += ck;
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] += s_oh[L::col(lane, v)];
    L::store(g_frame + (int64_t)fi * A, lane, A, g);
    __syncwarp();
    if (lane < K && tok_l >= 0 && tok_l < A) s_oh[tok_l] = 0.f;
    __syncwarp();
    if (!cx.fixup && lane < K) {
      st_ent += (double)my_H;
      st_bad += my_bad;
      st_badtok += my_badtok;
      if (my_inc) {
        st_loss += my_term;
        st_r += my_r;
        st_w += my_w;
        st_out += my_out;
        st_rmax = fmax(st_rmax, my_r);
        st_negw = fmax(st_negw, -my_w);
      } else {
        ++st_excl;
      }
    }
  }
  if (cx.fixup) return;
  // warp reduction of the per-lane statistics (fixed xor order), then CTA
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st_loss += __shfl_xor_sync(0xffffffffu, st_loss, o);
    st_ent += __shfl_xor_sync(0xffffffffu, st_ent, o);
    st_r += __shfl_xor_sync(0xffffffffu, st_r, o);
    st_w += __shfl_xor_sync(0xffffffffu, st_w, o);
    st_rmax = fmax(st_rmax, __shfl_xor_sync(0xffffffffu, st_rmax, o));
    st_negw = fmax(st_negw, __shfl_xor_sync(0xffffffffu, st_negw, o));
  }
  st_out = __reduce_add_sync(0xffffffffu, st_out);
  st_excl = __reduce_add_sync(0xffffffffu, st_excl);
  st_bad = __reduce_add_sync(0xffffffffu, st_bad);
  st_badtok = __reduce_add_sync(0xffffffffu, st_badtok);
  LossAcc<1> acc;
  acc.init();
  acc.loss_num = st_loss;
  acc.ent_sum = st_ent;
  acc.ratio_sum = st_r;
  acc.w_sum = st_w;
  acc.rmax = st_rmax;
  acc.negwmin = st_negw;
  acc.n_out = st_out;
  acc.n_excl = st_excl;
  acc.n_bad = st_bad;
  acc.n_badtok = st_badtok;
  stats_epilogue<1>(acc, s_stat, stat_part, max_part);
}

// ---- grouped variant: LPT lanes per transition, TPW = 32 / LPT transitions per warp ----
// Full rows only (A == 4 * LPT * (VPL / 4)) and K <= LPT.  Every lane holds VPL
// logits of its group's current token, so the per-token scalar algebra (log-sum,
// ratio, trust weight, fix-up store) is issued once for TPW tokens.  Group-local
// reductions use xor shuffles below LPT and group-masked CREDUX.
// SC: write per-token scalars {nm2, Ac, Cc, coef} (tsc) instead of the dz rows;
// the grouped-sum pass recomputes dz from them (fact_group_sum_kernel)
template <int VPL, int LPT, bool SC>
__global__ void __launch_bounds__(kThreads, 2)
token_loss_fact_grp_kernel(const float* __restrict__ h2w, const float* __restrict__ epp,
                           const int32_t* __restrict__ frame_of,
                           const int32_t* __restrict__ tokens, const float* __restrict__ lp_old,
                           const float* __restrict__ adv, int64_t N, int K, int A,
                           LossParams prm, const double* __restrict__ fix_stats,
                           float* __restrict__ dz, float4* __restrict__ tsc, float* __restrict__ g_frame,
                           float* __restrict__ lp_new, double* __restrict__ stat_part,
                           double* __restrict__ max_part) {
  constexpr int TPW = 32 / LPT;
  constexpr int W = VPL * LPT;  // == A
  constexpr int Q = VPL / 4;    // float4 chunks per lane
  extern __shared__ __align__(128) unsigned char smem[];
  // per-token statistics, recorded by the group leader and folded into the
  // group's running sums once per transition (shared memory, not registers:
  // the k-loop's live set stays within the 128-register budget)
  constexpr int G = kWarps * TPW;
  __shared__ double s_td[G][LPT][3];  // term, r, w
  __shared__ float s_tf[G][LPT][2];   // coef, H
  __shared__ int s_ti[G][LPT];        // inc | bad << 1 | bad_tok << 2 | outside << 3
  __shared__ double s_gacc[G][6];     // loss, ent, r, w, rmax, -wmin
  __shared__ int s_gcnt[G][4];        // outside, excluded, bad rows, bad tokens
  RowCtx cx;
  if (!setup_ctx(prm, fix_stats, cx)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / LPT, gl = lane % LPT, gbase = grp * LPT;
  const int gidx = warp * TPW + grp;
  if (gl == 0) {
    s_gacc[gidx][0] = s_gacc[gidx][1] = s_gacc[gidx][2] = s_gacc[gidx][3] = 0.0;
    s_gacc[gidx][4] = s_gacc[gidx][5] = -CUDART_INF;
    s_gcnt[gidx][0] = s_gcnt[gidx][1] = s_gcnt[gidx][2] = s_gcnt[gidx][3] = 0;
  }
  // smem: ring [kWarps][kGS][TPW][W] | s_oh [kWarps][TPW][W] | bars [kWarps][kGS][TPW]
  float* ring = reinterpret_cast<float*>(smem) + ((size_t)warp * kGS * TPW + grp) * W;
  float* s_oh = reinterpret_cast<float*>(smem) + (size_t)kWarps * kGS * TPW * W +
                ((size_t)warp * TPW + grp) * W;
  // EPP rows: s_ep[2] = the chunk-start row (prev = A, k = 0), s_ep[0]/[1] a
  // double buffer for tokens k >= 1, each filled by a bulk copy one token ahead
  float* s_ep = reinterpret_cast<float*>(smem) + (size_t)kWarps * (kGS + 1) * TPW * W +
                ((size_t)warp * TPW + grp) * 3 * W;
  uint64_t* bar_base =
      reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(smem) + (size_t)kWarps * (kGS + 4) * TPW * W);
  uint64_t* bars = bar_base + ((size_t)warp * kGS) * TPW + grp;
  uint64_t* ebars = bar_base + (size_t)kWarps * kGS * TPW + ((size_t)warp * TPW + grp) * 2;
  for (int c = gl; c < W; c += LPT) {
    s_oh[c] = 0.f;
    s_ep[2 * W + c] = __ldg(epp + (int64_t)A * K * A + c);
  }
  const unsigned row_bytes = (unsigned)A * 4u;
  // transition of group `grp` at iteration j: i = gi0 + j * gstride
  const int64_t gi0 = ((int64_t)blockIdx.x * kWarps + warp) * TPW + grp;
  const int64_t gstride = (int64_t)gridDim.x * kWarps * TPW;
  unsigned eph = 0;  // ebars[0/1] phase bits
  if (gl == 0) {
    mbar_init(&ebars[0], 1);
    mbar_init(&ebars[1], 1);
#pragma unroll
    for (int s = 0; s < kGS; ++s) mbar_init(&bars[s * TPW], 1);
    fence_mbar_init();
#pragma unroll
    for (int s = 0; s < kGS; ++s) {
      const int64_t i = gi0 + s * gstride;
      if (i < N) {
        mbar_expect_tx(&bars[s * TPW], row_bytes);
        bulk_g2s(ring + (size_t)s * TPW * W, h2w + (int64_t)__ldg(frame_of + i) * A, row_bytes,
                 &bars[s * TPW]);
      }
    }
  }
  __syncwarp();
  const float ent2 = cx.ent_scale * kLn2;

  auto colof = [&](int q, int r) { return q * 4 * LPT + gl * 4 + r; };
  auto load_grp = [&](const float* __restrict__ row, float (&x)[VPL], bool global) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const float4* p = reinterpret_cast<const float4*>(row + q * 4 * LPT + gl * 4);
      const float4 y = global ? __ldg(p) : *p;
      x[4 * q] = y.x; x[4 * q + 1] = y.y; x[4 * q + 2] = y.z; x[4 * q + 3] = y.w;
    }
  };

  // per-transition scalars, prefetched one iteration ahead (lane gl < K: token gl)
  int fi_n = 0, tok_n = 0;
  float lpo_n = 0.f, a_n = 0.f;
  if (gi0 < N) {
    fi_n = __ldg(frame_of + gi0);
    tok_n = gl < K ? __ldg(tokens + gi0 * K + gl) : 0;
    lpo_n = gl < K ? __ldg(lp_old + gi0 * K + gl) : 0.f;
    a_n = __ldg(adv + gi0);
  }
  const int64_t n_iter = gi0 - grp < N ? ceil_div(N - (gi0 - grp), gstride) : 0;  // group 0's count
  for (int64_t j = 0; j < n_iter; ++j) {
    const int64_t i = gi0 + j * gstride;
    const bool act = i < N;
    const int s = (int)(j % kGS);
    const float* hrow = ring + (size_t)s * TPW * W;
    const int fi = fi_n, tok_l = tok_n;
    const float lpo_l = lpo_n, a = a_n;
    const int64_t next = i + kGS * gstride;
    const int f_next = (gl == 0 && next < N) ? __ldg(frame_of + next) : 0;
    if (i + gstride < N) {
      const int64_t i2 = i + gstride;
      fi_n = __ldg(frame_of + i2);
      tok_n = gl < K ? __ldg(tokens + i2 * K + gl) : 0;
      lpo_n = gl < K ? __ldg(lp_old + i2 * K + gl) : 0.f;
      a_n = __ldg(adv + i2);
    }
    // token 1's EPP row (prev = token 0) into slot 1; slot 1's last reader is done
    // (no proxy fence: the slot's generic reads were consumed before this point;
    // a bulk copy issued after them cannot overtake them -- WAR, as in TMA pipelines)
    __syncwarp();
    if (act && gl == 0 && K > 1) {
      const int t0 = min(max(tok_l, 0), A - 1);
      mbar_expect_tx(&ebars[1], row_bytes);
      bulk_g2s(s_ep + W, epp + ((int64_t)t0 * K + 1) * A, row_bytes, &ebars[1]);
    }
    if (act) mbar_wait(&bars[s * TPW], (unsigned)(j / kGS) & 1u);
    __syncwarp();  // reconverge both groups before the element loop
    // packed fp32x2 arithmetic (FFMA2/FADD2/FMUL2): half the elementwise instructions
    constexpr int P = VPL / 2;
    float2 g2[P];
#pragma unroll
    for (int p = 0; p < P; ++p) g2[p] = make_float2(0.f, 0.f);
    const int64_t row0 = i * K;  // this transition's first token row
    float* dz_i = SC ? nullptr : dz + row0 * A;
    for (int k = 0; k < K; ++k) {
      const int tok_raw = __shfl_sync(0xffffffffu, tok_l, gbase + k);
      const float lpo = __shfl_sync(0xffffffffu, lpo_l, gbase + k);
      const bool bad_tok = tok_raw < 0 || tok_raw >= A;
      const int tok = bad_tok ? 0 : tok_raw;
      const float* erow = s_ep + (k == 0 ? 2 : (k & 1)) * W;
      if (k > 0) {
        if (act) mbar_wait(&ebars[k & 1], (eph >> (k & 1)) & 1u);
        __syncwarp();
        eph ^= 1u << (k & 1);
        // token k+1's row goes into the slot token k-1 used (fully read by now)
        // (no proxy fence: the slot's generic reads were consumed before this point;
        // a bulk copy issued after them cannot overtake them -- WAR, as in TMA pipelines)
        __syncwarp();
        if (act && gl == 0 && k + 1 < K) {
          const int sl = (k + 1) & 1;
          mbar_expect_tx(&ebars[sl], row_bytes);
          bulk_g2s(s_ep + sl * W, epp + ((int64_t)tok * K + k + 1) * A, row_bytes, &ebars[sl]);
        }
      }
      float2 z2[P];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 h = *reinterpret_cast<const float4*>(hrow + colof(q, 0));
        const float4 ep = *reinterpret_cast<const float4*>(erow + colof(q, 0));
        z2[2 * q] = __fadd2_rn(make_float2(h.x, h.y), make_float2(ep.x, ep.y));
        z2[2 * q + 1] = __fadd2_rn(make_float2(h.z, h.w), make_float2(ep.z, ep.w));
      }
      const float z_tok = hrow[tok] + erow[tok];
      float mx = fmaxf(z2[0].x, z2[0].y);
#pragma unroll
      for (int p = 1; p < P; ++p) mx = fmaxf(mx, fmaxf(z2[p].x, z2[p].y));
      if (LPT == 32) {
        mx = warp_max_nan(mx);
      } else {
        // group max with full-warp xor shuffles: a group-masked CREDUX would split
        // the warp into its groups for the rest of the row (each ran the row alone)
        // (a NaN logit is dropped by FMNMX here but still poisons the partition
        // sum below, as +inf does through inf - inf and -inf through 0 * -inf)
#pragma unroll
        for (int o = LPT / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      const float nm2 = -mx * kLog2e;
      const float2 l2e = make_float2(kLog2e, kLog2e), n2 = make_float2(nm2, nm2);
      float2 e2[P], sum2 = make_float2(0.f, 0.f), sed2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        z2[p] = __ffma2_rn(z2[p], l2e, n2);  // d2 = (z - max) log2(e)
        e2[p] = make_float2(ex2_ftz(z2[p].x), ex2_ftz(z2[p].y));
        sum2 = __fadd2_rn(sum2, e2[p]);
        sed2 = __ffma2_rn(e2[p], z2[p], sed2);
      }
      float sum = sum2.x + sum2.y, sed = sed2.x + sed2.y;
#pragma unroll
      for (int o = LPT / 2; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        sed += __shfl_xor_sync(0xffffffffu, sed, o);
      }
      const bool bad = !isfinite(sum) || !isfinite(sed) || !isfinite(mx);
      const float inv_s = 1.f / sum;
      const float log_s = __logf(sum);
      const float sd2 = sed * inv_s;
      const float H = log_s - sd2 * kLn2;
      const float d_tok = z_tok - mx;
      const float lpn = d_tok - log_s;
      const float dlt = lpn - lpo;
      const bool inc = act && !bad_tok && !bad && dlt <= 709.78271289f && dlt >= -745.13321910f;
      double term_d, r_d, w_d;
      bool outside;
      const float coef = token_coef(dlt, a, inc, cx, term_d, r_d, w_d, outside);
      const float Ac = ent2 * inv_s;
      const float Cc = -(Ac * sd2) - coef * inv_s;
      const float2 A2 = make_float2(Ac, Ac), C2 = make_float2(Cc, Cc);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        e2[p] = __fmul2_rn(e2[p], __ffma2_rn(A2, z2[p], C2));
        g2[p] = __fadd2_rn(g2[p], e2[p]);
      }
      const int64_t row = row0 + k;
      if constexpr (SC) {
        if (act && gl == 0) {
          tsc[row] = make_float4(nm2, Ac, Cc, coef);
          if (!cx.fixup) lp_new[row] = lpn;
        }
      } else {
        float* drow = dz_i + k * A;
        if (act) {
#pragma unroll
          for (int q = 0; q < Q; ++q)
            __stcs(reinterpret_cast<float4*>(drow + colof(q, 0)),
                   make_float4(e2[2 * q].x, e2[2 * q].y, e2[2 * q + 1].x, e2[2 * q + 1].y));
        }
        __syncwarp();
        if (act && gl == 0) {
          const float d2t = fmaf(z_tok, kLog2e, nm2);
          drow[tok] = fmaf(ex2_ftz(d2t), fmaf(Ac, d2t, Cc), coef);
          if (!cx.fixup) lp_new[row] = lpn;
        }
      }
      if (gl == 0) {
        s_td[gidx][k][0] = term_d;
        s_td[gidx][k][1] = r_d;
        s_td[gidx][k][2] = w_d;
        s_tf[gidx][k][0] = coef;
        s_tf[gidx][k][1] = H;
        s_ti[gidx][k] = (int)inc | ((int)bad << 1) | ((int)bad_tok << 2) | ((int)outside << 3);
      }
    }
    // (no proxy fence: the slot's generic reads were consumed before this point;
    // a bulk copy issued after them cannot overtake them -- WAR, as in TMA pipelines)
    __syncwarp();
    if (gl == 0 && next < N) {
      mbar_expect_tx(&bars[s * TPW], row_bytes);
      bulk_g2s(ring + (size_t)s * TPW * W, h2w + (int64_t)f_next * A, row_bytes, &bars[s * TPW]);
    }
    // one-hot part of G (group leader, serial over k: duplicates accumulate)
    for (int k = 0; k < K; ++k) {
      const int tk = __shfl_sync(0xffffffffu, tok_l, gbase + k);
      if (gl == 0 && tk >= 0 && tk < A) s_oh[tk] += s_tf[gidx][k][0];
    }
    __syncwarp();
    if (act) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const float4 o = *reinterpret_cast<const float4*>(s_oh + colof(q, 0));
        __stcs(reinterpret_cast<float4*>(g_frame + (int64_t)fi * A + colof(q, 0)),
               make_float4(g2[2 * q].x + o.x, g2[2 * q].y + o.y, g2[2 * q + 1].x + o.z,
                           g2[2 * q + 1].y + o.w));
      }
    }
    __syncwarp();
    if (gl < K && tok_l >= 0 && tok_l < A) s_oh[tok_l] = 0.f;
    __syncwarp();
    if (!cx.fixup && act && gl == 0) {  // fold this transition's token statistics
      double loss = s_gacc[gidx][0], ent = s_gacc[gidx][1], rs = s_gacc[gidx][2];
      double ws = s_gacc[gidx][3], rmax = s_gacc[gidx][4], negw = s_gacc[gidx][5];
      int nout = 0, nex = 0, nbad = 0, nbt = 0;
      for (int k = 0; k < K; ++k) {
        const int fl = s_ti[gidx][k];
        ent += (double)s_tf[gidx][k][1];
        nbad += (fl >> 1) & 1;
        nbt += (fl >> 2) & 1;
        if (fl & 1) {
          const double r = s_td[gidx][k][1], w = s_td[gidx][k][2];
          loss += s_td[gidx][k][0];
          rs += r;
          ws += w;
          nout += (fl >> 3) & 1;
          rmax = fmax(rmax, r);
          negw = fmax(negw, -w);
        } else {
          ++nex;
        }
      }
      s_gacc[gidx][0] = loss; s_gacc[gidx][1] = ent; s_gacc[gidx][2] = rs;
      s_gacc[gidx][3] = ws; s_gacc[gidx][4] = rmax; s_gacc[gidx][5] = negw;
      s_gcnt[gidx][0] += nout; s_gcnt[gidx][1] += nex;
      s_gcnt[gidx][2] += nbad; s_gcnt[gidx][3] += nbt;
    }
    __syncwarp();
  }
  if (cx.fixup) return;
  __syncthreads();
  if (threadIdx.x == 0) {  // groups in fixed order: deterministic
    double sum[kNumStat];
#pragma unroll
    for (int q = 0; q < kNumStat; ++q) sum[q] = 0.0;
    double rmax = -CUDART_INF, negw = -CUDART_INF;
    for (int g = 0; g < G; ++g) {
      sum[kLossNum] += s_gacc[g][0];
      sum[kEntSum] += s_gacc[g][1];
      sum[kRatioSum] += s_gacc[g][2];
      sum[kWSum] += s_gacc[g][3];
      rmax = fmax(rmax, s_gacc[g][4]);
      negw = fmax(negw, s_gacc[g][5]);
      sum[kOutside] += s_gcnt[g][0];
      sum[kExcluded] += s_gcnt[g][1];
      sum[kBadRows] += s_gcnt[g][2];
      sum[kBadTok] += s_gcnt[g][3];
    }
#pragma unroll
    for (int q = 0; q < kNumStat; ++q) stat_part[(int64_t)blockIdx.x * kNumStat + q] = sum[q];
    max_part[(int64_t)blockIdx.x * kNumMax + kRatioMax] = rmax;
    max_part[(int64_t)blockIdx.x * kNumMax + kNegWMin] = negw;
  }
}

// ---- two-phase kernel: a warp per transition, lane k owns token k's scalars ----
// The per-token scalar chain (log-partition, ratio, trust weight / clip, the
// float64 statistics) was the issue bottleneck of the kernels above: it ran
// once per token on every lane.  Here a warp owns a transition (A = 32 VPL
// logits per token, VPL per lane):
//   phase A: for every token k: z = H2W[frame] + EPP[prev, k], exact row max
//            (one CREDUX), d2 = (z - max) log2(e), partition sums
//            sum_k = sum 2^d2 and sed_k = sum 2^d2 d2 -- K independent rows, so
//            the unrolled loop overlaps them; d2 of tokens k >= 1 is written
//            back over the token's EPP slot (each lane its own columns);
//   a transposed butterfly reduces all 2K partial sums in 2K - 1 + 5 - log2(2K)
//            shuffles and leaves token k's totals on lane k;
//   lane k runs token k's scalar algebra (all K tokens in one pass);
//   phase C: for every token: broadcast (Ac, Cc), reload d2 (token 0:
//            recompute from the resident chunk-start row), 2^d2 (SFU),
//            dz = 2^d2 (Ac d2 + Cc), G += dz, streaming stores; lane k then
//            patches dz[tok_k] (+coef) after one warp barrier.
// The transition's H2W row and EPP rows k >= 1 land in shared memory by bulk
// copy, double-buffered a whole transition ahead (one mbarrier per buffer);
// the chunk-start row EPP[A, 0] (every transition's token 0) is resident per CTA.
#ifndef ACCEL_F2_WARPS
#define ACCEL_F2_WARPS 7
#endif
constexpr int kF2MaxWarps = ACCEL_F2_WARPS;
constexpr int kF2Chunk = 32;  // transitions per dynamically claimed chunk (and statistics row)
static_assert(kF2Chunk == 1 << 5, "the compile-time chunk shift below is 5");
// small batches: shorter chunks so every warp of the persistent grid gets work
// (a chunk's transitions run serially in one warp); fixed by N, so the
// statistics rows -- and the pooled sums -- are still deterministic
inline int fact2_chunk(int64_t N) {
  int c = kF2Chunk;
  while (c > 4 && ceil_div(N, (int64_t)c) < (int64_t)kNumSMs * 2 * kF2MaxWarps) c >>= 1;
  return c;
}

// After the call lane l holds the warp total of value index l / (32 / NV).
template <int NV>
__device__ __forceinline__ float transpose_reduce(float (&x)[NV], int lane) {
#pragma unroll
  for (int lvl = 0; lvl < 5; ++lvl) {
    const int o = 16 >> lvl;
    const int n = NV >> lvl;
    if (n > 1) {
      const int half = n / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const float send = up ? x[j] : x[j + half];
        const float keep = up ? x[j + half] : x[j];
        x[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    } else {
      x[0] += __shfl_xor_sync(0xffffffffu, x[0], o);
    }
  }
  return x[0];
}

// shared memory floats per warp: 2 buffers x {H row, EPP rows 1..K-1} + one-hot row
__host__ __device__ constexpr int fact2_warp_floats(int K, int A) { return (2 * K + 1) * A; }

// KT > 0: K == KT at compile time (no per-token guards: the unrolled token loops
// interleave); KT == 0: runtime K <= KMAX.
// SC: write the per-token scalars {nm2, Ac, Cc, coef} (tsc) instead of the dz
// rows; the frame-blocked grouped sums recompute dz (fact_group_sum_kernel).
// CS >= 0: the chunk shift as a compile-time constant (the full-chunk case of
// large batches); CS < 0: chunk_shift at run time
template <int VPL, int KMAX, int KT, bool SC, int CS = -1>
__global__ void __launch_bounds__(kF2MaxWarps * 32, 2)
token_loss_fact2_kernel(const float* __restrict__ h2w, const float* __restrict__ epp,
                        const int32_t* __restrict__ frame_of, const int32_t* __restrict__ tokens,
                        const float* __restrict__ lp_old, const float* __restrict__ adv,
                        int64_t N, int K_rt, LossParams prm, const double* __restrict__ fix_stats,
                        float* __restrict__ dz, float* __restrict__ g_frame,
                        float* __restrict__ lp_new, double* __restrict__ stat_part,
                        double* __restrict__ max_part, unsigned* __restrict__ work_ctr,
                        float4* __restrict__ tsc, const int32_t* __restrict__ tsc_pos,
                        int chunk_shift_rt) {
  const int chunk_shift = CS >= 0 ? CS : chunk_shift_rt;
  constexpr int A = VPL * 32;
  constexpr int Q = VPL / 4;  // float4 chunks per lane (column q * 128 + lane * 4 + r)
  constexpr int P = VPL / 2;  // float2 pairs per lane
  constexpr int NV = 2 * KMAX;
  constexpr int kHold = 32 / NV;  // lane stride of the reduced values
  static_assert(NV <= 32 && VPL % 4 == 0 && KT <= KMAX, "layout");
  const int K = KT > 0 ? KT : K_rt;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(16) float s_e0[A];       // EPP[A, 0]: token 0 of every transition
  __shared__ float s_cf[kF2MaxWarps][32];       // per-lane coef (one-hot part of G)
  RowCtx cx;
  if (!setup_ctx(prm, fix_stats, cx)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int c = threadIdx.x; c < A; c += blockDim.x) s_e0[c] = __ldg(epp + (int64_t)A * K * A + c);
  // smem per warp: buf[2] = {H row [A], d2/EPP rows 1..K-1 [K-1][A]} | s_oh [A];
  // mbarriers after all warps
  const int per_warp = fact2_warp_floats(K, A);
  const int buf_floats = K * A;
  float* wbase = reinterpret_cast<float*>(smem) + (size_t)warp * per_warp;
  float* s_oh = wbase + 2 * buf_floats;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(smem) +
                                               (size_t)nwarps * per_warp) + 2 * warp;
  for (int c = lane; c < A; c += 32) s_oh[c] = 0.f;
  const unsigned row_bytes = (unsigned)A * 4u;
  if (lane == 0) {
    mbar_init(&bars[0], 32);
    mbar_init(&bars[1], 32);
    fence_mbar_init();
  }
  __syncthreads();  // s_e0 and the barriers

  // transition scalars: lane k < K holds token k / lp_old k; all lanes frame + advantage
  struct Sc { int tok, fi; float lpo, a; };
  auto load_sc = [&](int64_t i) {
    Sc s{0, 0, 0.f, 0.f};
    if (i < N) {
      s.fi = __ldg(frame_of + i);
      s.a = __ldg(adv + i);
      if (lane < K) {
        s.tok = __ldg(tokens + i * K + lane);
        s.lpo = __ldg(lp_old + i * K + lane);
      }
    }
    return s;
  };
  // 16-B cp.async copies of transition i's H2W row (slot 0) and EPP rows
  // 1..K-1 (token k's row is EPP[tok_{k-1}, k]) into buffer b.  Lane l copies
  // exactly the columns it later reads and overwrites (q * 128 + l * 4), so the
  // d2 write-back and the refill two transitions on are ordered by the lane's
  // own program order.  Every lane arrives (noinc) when its copies land.
  auto issue = [&](int b, const Sc& s) {
    float* hb = wbase + b * buf_floats;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (KT > 0 ? k < KT : k < K) {
        const float* src;
        if (k == 0) {
          src = h2w + (int64_t)s.fi * A;
        } else {
          const int prev = min(max(__shfl_sync(0xffffffffu, s.tok, k - 1), 0), A - 1);
          src = epp + ((int64_t)prev * K + k) * A;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           smem_u32(hb + k * A + q * 128 + lane * 4)),
                       "l"(src + q * 128 + lane * 4)
                       : "memory");
      }
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[b]))
                 : "memory");
  };
  // dynamic schedule: warps claim chunks of `chunk` consecutive transitions
  // from a device counter (zeroed by the host before the launch), one chunk
  // ahead, so SMs that run faster take more chunks; next(x) is the transition
  // after x in this warp's sequence (N = none)
  const int64_t cmask = ((int64_t)1 << chunk_shift) - 1;  // chunks are powers of two
  unsigned pend = 0;  // lane 0: the pre-claimed next chunk (resolved lazily)
  auto claim = [&]() -> unsigned { return lane == 0 ? atomicAdd(work_ctr, 1u) : 0u; };
  auto next_of = [&](int64_t x) -> int64_t {
    if (x >= N) return N;
    if (((x + 1) & cmask) != 0 && x + 1 < N) return x + 1;
    const int64_t y = (int64_t)__shfl_sync(0xffffffffu, pend, 0) << chunk_shift;
    pend = claim();
    return y < N ? y : N;
  };
  const float ent2 = cx.ent_scale * kLn2;
  const float2 l2e2 = make_float2(kLog2e, kLog2e);
  double st_loss = 0.0, st_ent = 0.0, st_r = 0.0, st_w = 0.0;
  double st_rmax = -CUDART_INF, st_negw = -CUDART_INF;
  int st_out = 0, st_excl = 0, st_bad = 0, st_badtok = 0;

  int64_t i = (int64_t)__shfl_sync(0xffffffffu, claim(), 0) << chunk_shift;
  i = i < N ? i : N;
  pend = claim();
  int64_t i1 = next_of(i);
  Sc cur = load_sc(i);
  Sc nxt = load_sc(i1);
  if (i < N) issue(0, cur);
  for (int64_t j = 0; i < N; ++j) {
    const int b = (int)(j & 1);
    // the other buffer was last read by transition j - 1: refill it with j + 1
    __syncwarp();
    if (i1 < N) issue(b ^ 1, nxt);
    const int64_t i2 = next_of(i1);
    const Sc nn = load_sc(i2);
    float* hrow = wbase + b * buf_floats;  // slot 0: H2W row; slots 1..K-1: EPP rows -> d2
    mbar_wait(&bars[b], (unsigned)(j >> 1) & 1u);
    __syncwarp();  // reconverge after the spin-wait

    const int kl = lane < K ? lane : 0;  // token owned by this lane
    const bool own = lane < K;
    const bool bad_tok = cur.tok < 0 || cur.tok >= A;
    const int tok = bad_tok ? 0 : cur.tok;
    // chosen-token logit, read before the EPP slots are overwritten with d2
    const float z_tok = hrow[tok] + (kl == 0 ? s_e0[tok] : hrow[kl * A + tok]);
    float2 h2[P];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const float4 h = *reinterpret_cast<const float4*>(hrow + q * 128 + lane * 4);
      h2[2 * q] = make_float2(h.x, h.y);
      h2[2 * q + 1] = make_float2(h.z, h.w);
    }
    __syncwarp();  // every lane has read z_tok before any d2 store
    // ---- phase A: row max and partition sums of every token ----
    float mx0 = 0.f, mx_l = 0.f, red[NV];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      red[k] = 0.f;
      red[KMAX + k] = 0.f;
      if (KT > 0 ? k < KT : k < K) {
        const float* er = k == 0 ? s_e0 : hrow + k * A;
        float2 z2[P];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const float4 ep = *reinterpret_cast<const float4*>(er + q * 128 + lane * 4);
          z2[2 * q] = __fadd2_rn(h2[2 * q], make_float2(ep.x, ep.y));
          z2[2 * q + 1] = __fadd2_rn(h2[2 * q + 1], make_float2(ep.z, ep.w));
        }
        float m2[P];  // max tree (short dependency chains)
#pragma unroll
        for (int p = 0; p < P; ++p) m2[p] = fmaxf(z2[p].x, z2[p].y);
#pragma unroll
        for (int w = 1; w < P; w *= 2)
#pragma unroll
          for (int p = 0; p + w < P; p += 2 * w) m2[p] = fmaxf(m2[p], m2[p + w]);
        const float mx = warp_max_nan(m2[0]);  // NaN logit -> NaN max; +inf -> NaN below
        if (k == 0) mx0 = mx;
        mx_l = kl == k ? mx : mx_l;
        const float2 n2 = make_float2(-mx * kLog2e, -mx * kLog2e);
        float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float2 sd2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int p = 0; p < P; ++p) {
          z2[p] = __ffma2_rn(z2[p], l2e2, n2);  // d2
          const float2 e2 = make_float2(ex2_ftz(z2[p].x), ex2_ftz(z2[p].y));
          s2[p & 1] = __fadd2_rn(s2[p & 1], e2);
          sd2[p & 1] = __ffma2_rn(e2, z2[p], sd2[p & 1]);  // 0 * (-inf) = NaN: -inf poisons it
        }
        if (k > 0) {
          float* dr = hrow + k * A;
#pragma unroll
          for (int q = 0; q < Q; ++q)
            *reinterpret_cast<float4*>(dr + q * 128 + lane * 4) =
                make_float4(z2[2 * q].x, z2[2 * q].y, z2[2 * q + 1].x, z2[2 * q + 1].y);
        }
        const float2 s = __fadd2_rn(s2[0], s2[1]), sd = __fadd2_rn(sd2[0], sd2[1]);
        red[k] = s.x + s.y;
        red[KMAX + k] = sd.x + sd.y;
      }
    }
    transpose_reduce<NV>(red, lane);
    const float sum = __shfl_sync(0xffffffffu, red[0], (kl * kHold) & 31);
    const float sed = __shfl_sync(0xffffffffu, red[0], ((KMAX + kl) * kHold) & 31);
    // ---- lane k: token k's scalar algebra ----
    const bool bad = !isfinite(sum) || !isfinite(sed) || !isfinite(mx_l);
    const float inv_s = 1.f / sum;
    const float log_s = __logf(sum);
    const float sdn = sed * inv_s;  // sum_a p_a d2_a
    const float Hk = log_s - sdn * kLn2;
    const float lpn = (z_tok - mx_l) - log_s;
    const float dlt = lpn - cur.lpo;
    const bool inc = own && !bad_tok && !bad && dlt <= 709.78271289f && dlt >= -745.13321910f;
    double term_d, r_d, w_d;
    bool outside;
    const float coef = token_coef(dlt, cur.a, inc, cx, term_d, r_d, w_d, outside);
    const float Ac = ent2 * inv_s;
    const float Cc = -(Ac * sdn) - coef * inv_s;
    const float d2t = fmaf(z_tok, kLog2e, -mx_l * kLog2e);  // == the row's d2 at column tok
    const float patch = fmaf(ex2_ftz(d2t), fmaf(Ac, d2t, Cc), coef);
    if (SC && own) {  // at the token's sorted position when the grouping provides it
      const int64_t t = i * K + lane;
      tsc[tsc_pos != nullptr ? (int64_t)__ldg(tsc_pos + t) : t] =
          make_float4(-mx_l * kLog2e, Ac, Cc, coef);
    }
    if (own && !cx.fixup) {
      lp_new[i * K + lane] = lpn;
      st_ent += (double)Hk;
      st_bad += bad;
      st_badtok += bad_tok;
      if (inc) {
        st_loss += term_d;
        st_r += r_d;
        st_w += w_d;
        st_out += outside;
        st_rmax = fmax(st_rmax, r_d);
        st_negw = fmax(st_negw, -w_d);
      } else {
        ++st_excl;
      }
    }
    // ---- phase C: dlogits rows, G accumulation ----
    float2 g2[P];
#pragma unroll
    for (int p = 0; p < P; ++p) g2[p] = make_float2(0.f, 0.f);
    float* dz_i = SC ? nullptr : dz + i * K * A;
    const float2 n20 = make_float2(-mx0 * kLog2e, -mx0 * kLog2e);
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (KT > 0 ? k < KT : k < K) {
        const float Ak = __shfl_sync(0xffffffffu, Ac, k);
        const float Ck = __shfl_sync(0xffffffffu, Cc, k);
        const float2 A2 = make_float2(Ak, Ak), C2 = make_float2(Ck, Ck);
        float2 d2[P];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          if (k == 0) {  // recompute from the resident chunk-start row
            const float4 ep = *reinterpret_cast<const float4*>(s_e0 + q * 128 + lane * 4);
            d2[2 * q] = __ffma2_rn(__fadd2_rn(h2[2 * q], make_float2(ep.x, ep.y)), l2e2, n20);
            d2[2 * q + 1] =
                __ffma2_rn(__fadd2_rn(h2[2 * q + 1], make_float2(ep.z, ep.w)), l2e2, n20);
          } else {
            const float4 v = *reinterpret_cast<const float4*>(hrow + k * A + q * 128 + lane * 4);
            d2[2 * q] = make_float2(v.x, v.y);
            d2[2 * q + 1] = make_float2(v.z, v.w);
          }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float2 e2 = make_float2(ex2_ftz(d2[p].x), ex2_ftz(d2[p].y));
          d2[p] = __fmul2_rn(e2, __ffma2_rn(A2, d2[p], C2));
          g2[p] = __fadd2_rn(g2[p], d2[p]);
        }
        if (!SC) {
          float* drow = dz_i + k * A;
#pragma unroll
          for (int q = 0; q < Q; ++q)
            __stcs(reinterpret_cast<float4*>(drow + q * 128 + lane * 4),
                   make_float4(d2[2 * q].x, d2[2 * q].y, d2[2 * q + 1].x, d2[2 * q + 1].y));
        }
      }
    }
    // one-hot part: dz[tok_k] += coef_k (after every lane's row stores) and
    // G[tok_k] += coef_k, duplicates summed in token order by their first lane
    s_cf[warp][lane] = coef;
    __syncwarp();
    if (!SC && own) dz_i[lane * A + tok] = patch;
    const unsigned same = __match_any_sync(0xffffffffu, own && !bad_tok ? tok : -1 - lane);
    if (own && !bad_tok && (same & ((1u << lane) - 1u)) == 0) {
      float acc = coef;
      for (unsigned m = same & (same - 1u); m; m &= m - 1u) acc += s_cf[warp][__ffs(m) - 1];
      s_oh[tok] = acc;
    }
    __syncwarp();
    float* grow = g_frame + (int64_t)cur.fi * A;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const float4 o = *reinterpret_cast<const float4*>(s_oh + q * 128 + lane * 4);
      __stcs(reinterpret_cast<float4*>(grow + q * 128 + lane * 4),
             make_float4(g2[2 * q].x + o.x, g2[2 * q].y + o.y, g2[2 * q + 1].x + o.z,
                         g2[2 * q + 1].y + o.w));
    }
    __syncwarp();
    if (own && !bad_tok) s_oh[tok] = 0.f;
    // a chunk of `chunk` transitions is done: its statistics go to the chunk's own
    // partial row (warp-reduced in a fixed order), so the pooled sums do not
    // depend on which warp the dynamic schedule handed the chunk to
    if (!cx.fixup && (((i + 1) & cmask) == 0 || i + 1 == N)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        st_loss += __shfl_xor_sync(0xffffffffu, st_loss, o);
        st_ent += __shfl_xor_sync(0xffffffffu, st_ent, o);
        st_r += __shfl_xor_sync(0xffffffffu, st_r, o);
        st_w += __shfl_xor_sync(0xffffffffu, st_w, o);
        st_rmax = fmax(st_rmax, __shfl_xor_sync(0xffffffffu, st_rmax, o));
        st_negw = fmax(st_negw, __shfl_xor_sync(0xffffffffu, st_negw, o));
      }
      st_out = __reduce_add_sync(0xffffffffu, st_out);
      st_excl = __reduce_add_sync(0xffffffffu, st_excl);
      st_bad = __reduce_add_sync(0xffffffffu, st_bad);
      st_badtok = __reduce_add_sync(0xffffffffu, st_badtok);
      if (lane == 0) {
        const int64_t c = i >> chunk_shift;
        double* st = stat_part + c * kNumStat;
        st[kLossNum] = st_loss;
        st[kEntSum] = st_ent;
        st[kRatioSum] = st_r;
        st[kWSum] = st_w;
        st[kOutside] = st_out;
        st[kExcluded] = st_excl;
        st[kBadRows] = st_bad;
        st[kBadTok] = st_badtok;
        max_part[c * kNumMax + kRatioMax] = st_rmax;
        max_part[c * kNumMax + kNegWMin] = st_negw;
      }
      st_loss = st_ent = st_r = st_w = 0.0;
      st_rmax = st_negw = -CUDART_INF;
      st_out = st_excl = st_bad = st_badtok = 0;
    }
    cur = nxt;
    nxt = nn;
    i = i1;
    i1 = i2;
  }
}

// Dprev[j] = sum_k Dpk[j, k], Dpos[k] = sum_j Dpk[j, k]  (Dpk f32[(A+1), K, A])
// Dprev: a thread per output (K terms).  Dpos: a block per (k, 32-column
// group): 8 warps each sum a fixed 1/8 of the nprev rows (eight loads in
// flight), the warp sums are added in warp order -- the long column sums run
// 8-way parallel instead of as one 257-load chain per thread.
__global__ void pk_marginals_kernel(const float* __restrict__ dpk, int K, int A, int nprev,
                                    int dprev_blocks, float* __restrict__ dprev,
                                    float* __restrict__ dpos) {
  if ((int)blockIdx.x < dprev_blocks) {
    const int64_t total = (int64_t)nprev * A;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)dprev_blocks * blockDim.x) {
      const int a = (int)(e % A);
      const int64_t r = e / A;
      float s = 0.f;
      for (int k = 0; k < K; ++k) s += __ldg(dpk + (r * K + k) * A + a);
      dprev[r * A + a] = s;
    }
    return;
  }
  __shared__ float s_part[8][32];
  const int groups = (A + 31) / 32;
  const int bid = (int)blockIdx.x - dprev_blocks;
  const int k = bid / groups, a = (bid % groups) * 32 + (threadIdx.x & 31);
  const int w = threadIdx.x >> 5;
  const int j0 = w * nprev / 8, j1 = (w + 1) * nprev / 8;
  float s = 0.f;
  if (a < A) {
    int jj = j0;
    for (; jj + 8 <= j1; jj += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(dpk + ((int64_t)(jj + u) * K + k) * A + a);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; jj < j1; ++jj) s += __ldg(dpk + ((int64_t)jj * K + k) * A + a);
  }
  s_part[w][threadIdx.x & 31] = s;
  __syncthreads();
  if (w == 0 && a < A) {
    float t = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) t += s_part[u][threadIdx.x];
    dpos[(int64_t)k * A + a] = t;
  }
}

// Grouped sums of dz over the (prev token, position) keys without dz in HBM:
// one CTA per piece (<= 256 tokens of one key, in the batch's stable key order)
// recomputes each token's dz row from its H2W row (gathered, 1 KB), the key's
// EPP row (shared memory) and the token scalars {nm2, Ac, Cc, coef} written by
// the SC loss pass -- the same float operations as the loss kernel:
//   d2 = (h + ep) log2(e) + nm2,  dz = 2^d2 (Ac d2 + Cc)  (+ coef at the token)
// Row-lanes of A/4 threads, 4 rows in flight per lane, fixed combine order.
constexpr int kGsThreads = 256;
constexpr int kGsRows = 256;  // piece rows (== the grouping's piece size)
__global__ void __launch_bounds__(kGsThreads)
fact_group_sum_kernel(const float* __restrict__ h2w, const float* __restrict__ epp,
                      const int32_t* __restrict__ frame_of, const int32_t* __restrict__ tokens,
                      const float4* __restrict__ tsc, const int32_t* __restrict__ perm,
                      const int64_t* __restrict__ seg_off, const int64_t* __restrict__ piece_off,
                      int nkeys, int key_mod, int K, int A, int piece_rows,
                      float* __restrict__ piece_out) {
  // smem: epp row [A] | partials [kGsThreads] float4 | per-token frame, token, scalars
  extern __shared__ __align__(16) float s_gs[];
  __shared__ int s_frame[kGsRows], s_tok[kGsRows];
  __shared__ float4 s_sc[kGsRows];
  const int64_t piece = blockIdx.x;
  if (piece >= piece_off[nkeys]) return;
  int lo = 0, hi = nkeys;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (piece_off[mid] <= piece) lo = mid; else hi = mid;
  }
  const int key = lo;
  const int64_t r0 = seg_off[key] + (piece - piece_off[key]) * piece_rows;
  const int nr = (int)min(seg_off[key + 1] - r0, (int64_t)piece_rows);
  float* s_ep = s_gs;
  float4* s_part = reinterpret_cast<float4*>(s_gs + A);
  // composite keys (frame-blocked grouping): the EPP row is key % key_mod
  const int64_t erow = key_mod > 0 ? key % key_mod : key;
  for (int c = threadIdx.x; c < A; c += kGsThreads) s_ep[c] = __ldg(epp + erow * A + c);
  // the piece's token metadata, gathered once (one token per thread)
  for (int r = threadIdx.x; r < nr; r += kGsThreads) {
    const int64_t t = __ldg(perm + r0 + r);
    s_frame[r] = __ldg(frame_of + t / K);
    s_tok[r] = __ldg(tokens + t);
    s_sc[r] = __ldg(tsc + t);
  }
  __syncthreads();
  const int A4 = A >> 2;
  const int span = A4 <= kGsThreads && kGsThreads % A4 == 0 ? A4 : kGsThreads;
  const int sub = kGsThreads / span;
  const int lr = threadIdx.x / span, lc = threadIdx.x % span;
  auto row = [&](int r, int c4, const float4& ep, float4& acc) {
    const float4 h = __ldg(reinterpret_cast<const float4*>(h2w + (int64_t)s_frame[r] * A) + c4);
    const float4 sc = s_sc[r];
    const int tok = s_tok[r];
    const float d[4] = {h.x + ep.x, h.y + ep.y, h.z + ep.z, h.w + ep.w};
    float o[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float d2 = fmaf(d[u], kLog2e, sc.x);
      o[u] = ex2_ftz(d2) * fmaf(sc.y, d2, sc.z);
    }
    if ((tok >> 2) == c4) o[tok & 3] += sc.w;
    acc.x += o[0]; acc.y += o[1]; acc.z += o[2]; acc.w += o[3];
  };
  for (int c0 = 0; c0 < A4; c0 += span) {
    const int c4 = c0 + lc;
    float4 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c4 < A4) {
      const float4 ep = reinterpret_cast<const float4*>(s_ep)[c4];
      int r = lr;
      for (; r + 3 * sub < nr; r += 4 * sub) {  // four independent row loads in flight
#pragma unroll
        for (int u = 0; u < 4; ++u) row(r + u * sub, c4, ep, acc[u]);
      }
      for (; r < nr; r += sub) row(r, c4, ep, acc[0]);
    }
    float4 t = acc[0];
#pragma unroll
    for (int u = 1; u < 4; ++u) { t.x += acc[u].x; t.y += acc[u].y; t.z += acc[u].z; t.w += acc[u].w; }
    s_part[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x < span && c0 + threadIdx.x < A4) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s2 = 0; s2 < sub; ++s2) {
        const float4 y = s_part[s2 * span + threadIdx.x];
        a.x += y.x; a.y += y.y; a.z += y.z; a.w += y.w;
      }
      reinterpret_cast<float4*>(piece_out + piece * A)[c0 + threadIdx.x] = a;
    }
    __syncthreads();
  }
}

// Recompute over a frame-blocked grouping with sorted metadata: one CTA per
// piece, pieces in (block, key) order so concurrently running CTAs gather H2W
// rows of one block of frames (L2-resident).  The piece's rows are contiguous
// in the sorted arrays row_frame / row_tok (fixed per batch) and tsc_sorted
// (written by the loss kernel at each token's sorted position), so the only
// dependent load before the sums is piece_key -> (seg_off, piece_off).  Eight
// row loads per lane are in flight; same float operations per element as the
// loss kernel.
constexpr int kGs2Threads = 256;
constexpr int kGs2Warps = kGs2Threads / 32;
// LPR = A / 8 lanes per row (8 columns per lane, packed fp32x2 math), 32 / LPR
// rows per warp, four rows in flight per lane.  The one-hot coef of a row is
// added by the single lane owning the token's column into that lane's private
// shared-memory slots (row order: deterministic), folded in at the end.
template <int LPR>
__global__ void __launch_bounds__(kGs2Threads)
fact_group_sum2_kernel(const float* __restrict__ h2w, const float* __restrict__ epp,
                       const int32_t* __restrict__ perm, const int32_t* __restrict__ frame_of,
                       const int32_t* __restrict__ tokens, int K,
                       const float4* __restrict__ tsc_sorted, const int64_t* __restrict__ seg_off,
                       const int64_t* __restrict__ piece_off, const int32_t* __restrict__ piece_key,
                       int nkeys, int key_mod, float* __restrict__ piece_out) {
  constexpr int A = LPR * 8;
  constexpr int RPW = 32 / LPR;             // rows per warp
  constexpr int RPC = RPW * kGs2Warps;      // rows in parallel per CTA
  __shared__ __align__(16) float s_ep[A];
  __shared__ int s_frame[kGsRows], s_tok[kGsRows];
  __shared__ float4 s_sc[kGsRows];
  __shared__ __align__(16) float s_patch[kGs2Threads][8];
  __shared__ __align__(16) float4 s_part[kGs2Threads][2];
  const int64_t p = blockIdx.x;
  if (p >= __ldg(piece_off + nkeys)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int key = __ldg(piece_key + p);
  const int64_t r0 = __ldg(seg_off + key) + (p - __ldg(piece_off + key)) * kGsRows;
  const int nr = (int)min(__ldg(seg_off + key + 1) - r0, (int64_t)kGsRows);
  const int64_t erow = key_mod > 0 ? key % key_mod : key;
  for (int c = tid; c < A; c += kGs2Threads) s_ep[c] = __ldg(epp + erow * A + c);
  if (tid < nr) {  // the piece's token rows through the permutation (L2-resident gathers)
    const int32_t t = __ldg(perm + r0 + tid);
    s_frame[tid] = __ldg(frame_of + t / K);
    s_tok[tid] = __ldg(tokens + t);
    s_sc[tid] = __ldg(tsc_sorted + r0 + tid);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) s_patch[tid][q] = 0.f;
  __syncthreads();
  const int lc = lane % LPR;               // this lane's 8 columns: 8 lc .. 8 lc + 7
  const int rw = warp * RPW + lane / LPR;  // first row of this lane
  float2 ep2[4];
  {
    const float4 e0 = reinterpret_cast<const float4*>(s_ep)[2 * lc];
    const float4 e1 = reinterpret_cast<const float4*>(s_ep)[2 * lc + 1];
    ep2[0] = make_float2(e0.x, e0.y); ep2[1] = make_float2(e0.z, e0.w);
    ep2[2] = make_float2(e1.x, e1.y); ep2[3] = make_float2(e1.z, e1.w);
  }
  const float2 l2e2 = make_float2(kLog2e, kLog2e);
  float2 acc[2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[u][q] = make_float2(0.f, 0.f);
  auto row = [&](int r, const float4& h0, const float4& h1, float2 (&a)[4]) {
    const float4 sc = s_sc[r];
    const float2 h[4] = {make_float2(h0.x, h0.y), make_float2(h0.z, h0.w),
                         make_float2(h1.x, h1.y), make_float2(h1.z, h1.w)};
    const float2 n2 = make_float2(sc.x, sc.x), A2 = make_float2(sc.y, sc.y),
                 C2 = make_float2(sc.z, sc.z);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 d2 = __ffma2_rn(__fadd2_rn(h[q], ep2[q]), l2e2, n2);
      const float2 e2 = make_float2(ex2_ftz(d2.x), ex2_ftz(d2.y));
      a[q] = __fadd2_rn(a[q], __fmul2_rn(e2, __ffma2_rn(A2, d2, C2)));
    }
    const int tok = s_tok[r];
    if ((tok >> 3) == lc) s_patch[tid][tok & 7] += sc.w;  // one lane per row
  };
  auto hrow = [&](int r, float4& h0, float4& h1) {
    const float4* hp = reinterpret_cast<const float4*>(h2w + (int64_t)s_frame[r] * A) + 2 * lc;
    h0 = __ldg(hp);
    h1 = __ldg(hp + 1);
  };
  int r = rw;
  for (; r + 3 * RPC < nr; r += 4 * RPC) {  // four rows in flight, no predicates
    float4 h[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) hrow(r + u * RPC, h[u][0], h[u][1]);
#pragma unroll
    for (int u = 0; u < 4; ++u) row(r + u * RPC, h[u][0], h[u][1], acc[u & 1]);
  }
  for (; r < nr; r += RPC) {
    float4 h0, h1;
    hrow(r, h0, h1);
    row(r, h0, h1, acc[0]);
  }
  // this lane's sums (+ its patch slots), then the RPC row-lanes of each column
  // group are combined in a fixed order
  {
    float pt[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pt[q] = s_patch[tid][q];
    float v[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[2 * q] = (acc[0][q].x + acc[1][q].x) + pt[2 * q];
      v[2 * q + 1] = (acc[0][q].y + acc[1][q].y) + pt[2 * q + 1];
    }
    s_part[tid][0] = make_float4(v[0], v[1], v[2], v[3]);
    s_part[tid][1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  __syncthreads();
  // thread t < 2 LPR: float4 column group t; sums the RPC row-lanes in order
  if (tid < 2 * LPR) {
    const int col = tid >> 1, half = tid & 1;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < RPC; ++j) {
      const int t = (j / RPW) * 32 + (j % RPW) * LPR + col;  // lane holding row-lane j, column col
      const float4 y = s_part[t][half];
      o.x += y.x; o.y += y.y; o.z += y.z; o.w += y.w;
    }
    reinterpret_cast<float4*>(piece_out + p * A)[tid] = o;
  }
}

// Sorted per-row metadata of a grouping (fixed per batch): row_frame[r] =
// frame_of[perm[r] / K], row_tok[r] = tokens[perm[r]], pos[perm[r]] = r.
__global__ void sorted_rows_kernel(const int32_t* __restrict__ perm,
                                   const int32_t* __restrict__ frame_of,
                                   const int32_t* __restrict__ tokens, int64_t R, int K,
                                   int32_t* __restrict__ row_frame, int32_t* __restrict__ row_tok,
                                   int32_t* __restrict__ pos) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    const int32_t t = __ldg(perm + r);
    row_frame[r] = __ldg(frame_of + t / K);
    row_tok[r] = __ldg(tokens + t);
    pos[t] = (int32_t)r;
  }
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_fact_group_sum(const float* h2w, const float* epp, const int32_t* frame_of,
                                    const int32_t* tokens, const void* tsc, const int32_t* perm,
                                    const int64_t* seg_off, const int64_t* piece_off, int nkeys,
                                    int key_mod, int K, int A, int piece_rows, int64_t n_pieces,
                                    float* piece_out, void* stream) {
  if (K < 1 || A < 4 || A % 4 || nkeys < 1 || piece_rows < 1 || piece_rows > kGsRows)
    return fail(kDimension, "fact_group_sum: bad sizes");
  if (n_pieces == 0) return kOk;
  if (!h2w || !epp || !frame_of || !tokens || !tsc || !perm || !seg_off || !piece_off || !piece_out)
    return fail(kDimension, "fact_group_sum: NULL buffer");
  if (misaligned16(h2w) || misaligned16(epp) || misaligned16(tsc) || misaligned16(piece_out))
    return fail(kDimension, "fact_group_sum: buffers must be 16B aligned");
  const size_t smem = (size_t)A * 4 + kGsThreads * sizeof(float4);
  fact_group_sum_kernel<<<(unsigned)n_pieces, kGsThreads, smem, as_stream(stream)>>>(
      h2w, epp, frame_of, tokens, static_cast<const float4*>(tsc), perm, seg_off, piece_off, nkeys,
      key_mod, K, A, piece_rows, piece_out);
  return post_launch("fact_group_sum_kernel");
}

// Recompute over a frame-blocked grouping with sorted metadata (see the kernel).
extern "C" int accel_fact_group_sum2(const float* h2w, const float* epp, const int32_t* perm,
                                     const int32_t* frame_of, const int32_t* tokens, int K,
                                     const void* tsc_sorted, const int64_t* seg_off,
                                     const int64_t* piece_off, const int32_t* piece_key, int nkeys,
                                     int key_mod, int A, int64_t n_pieces_max, float* piece_out,
                                     void* stream) {
  if (A < 4 || A % 4 || nkeys < 1 || K < 1) return fail(kDimension, "fact_group_sum2: bad sizes");
  if (n_pieces_max == 0) return kOk;
  if (!h2w || !epp || !perm || !frame_of || !tokens || !tsc_sorted || !seg_off || !piece_off ||
      !piece_key || !piece_out)
    return fail(kDimension, "fact_group_sum2: NULL buffer");
  if (misaligned16(h2w) || misaligned16(epp) || misaligned16(tsc_sorted) || misaligned16(piece_out))
    return fail(kDimension, "fact_group_sum2: buffers must be 16B aligned");
  if (A != 128 && A != 256) return fail(kDimension, "fact_group_sum2: A must be 128 or 256");
  auto go = [&](auto kernel) {
    kernel<<<(unsigned)n_pieces_max, kGs2Threads, 0, as_stream(stream)>>>(
        h2w, epp, perm, frame_of, tokens, K, static_cast<const float4*>(tsc_sorted), seg_off,
        piece_off, piece_key, nkeys, key_mod, piece_out);
    return post_launch("fact_group_sum2_kernel");
  };
  return A == 256 ? go(fact_group_sum2_kernel<32>) : go(fact_group_sum2_kernel<16>);
}

extern "C" int accel_sorted_rows(const int32_t* perm, const int32_t* frame_of,
                                 const int32_t* tokens, int64_t R, int K, int32_t* row_frame,
                                 int32_t* row_tok, int32_t* pos, void* stream) {
  if (R < 0 || K < 1) return fail(kDimension, "sorted_rows: bad sizes");
  if (R == 0) return kOk;
  if (!perm || !frame_of || !tokens || !row_frame || !row_tok || !pos)
    return fail(kDimension, "sorted_rows: NULL buffer");
  const int grid = (int)std::min<int64_t>(ceil_div(R, 256), (int64_t)kNumSMs * 8);
  sorted_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(perm, frame_of, tokens, R, K, row_frame,
                                                          row_tok, pos);
  return post_launch("sorted_rows_kernel");
}

// Rows of stat_part / max_part the loss kernel for (N, K, A, scalar output)
// writes: one per 32-transition chunk for the two-phase kernel (deterministic
// under its dynamic schedule), one per CTA (accel_fact_grid) otherwise.
extern "C" int64_t accel_fact_partials(int64_t N, int K, int A, int scalar_out) {
  (void)scalar_out;
  if (K <= 8 && (A == 128 || A == 256)) return std::max<int64_t>(1, ceil_div(N, (int64_t)fact2_chunk(N)));
  return accel_fact_grid(N);
}

extern "C" int accel_fact_grid(int64_t N) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(N, kWarps), (int64_t)kNumSMs * 2));
}

extern "C" int accel_ep_plus(const float* ep, const float* pp, const float* bias, int A, int K,
                             float* epp, void* stream) {
  if (A < 1 || K < 1 || !ep || !pp || !bias || !epp) return fail(kDimension, "ep_plus: bad args");
  const int64_t total = (int64_t)(A + 1) * K * A;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)kNumSMs * 4);
  ep_plus_kernel<<<grid, 256, 0, as_stream(stream)>>>(ep, pp, bias, A, K, epp);
  return post_launch("ep_plus_kernel");
}


extern "C" int accel_token_loss_fact2(const float* h2w, const float* epp, const int32_t* frame_of,
                                      const int32_t* tokens, const float* lp_old, const float* adv,
                                      int64_t N, int K, int A, int algo, double sigma,
                                      double clip_eps, double lambda_h, double m_global,
                                      const double* fix_stats, float* dz, void* tsc,
                                      const int32_t* tsc_pos, float* g_frame, float* lp_new,
                                      double* stat_part, double* max_part, unsigned* counters,
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
  if (!h2w || !epp || !frame_of || !tokens || !lp_old || !adv || (!dz && !tsc) || !g_frame ||
      (!fix_stats && (!lp_new || !stat_part || !max_part)))
    return fail(kDimension, "token_loss_fact: NULL buffer");
  if (misaligned16(h2w) || misaligned16(epp) || misaligned16(dz) || misaligned16(tsc) ||
      misaligned16(g_frame))
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
  // TPW == 0: per-warp kernel (ring kStages deep); TPW >= 1: grouped kernel
  // (ring kGS deep + s_oh + 3 EPP rows per group, 2 extra mbarriers per group)
  auto go = [&](auto kernel, int VPL, int TPW = 0) -> int {
    const size_t row_floats = (size_t)VPL * 32;  // floats per warp per stage
    const size_t smem =
        TPW == 0 ? (size_t)kWarps * (kStages + 1) * row_floats * 4 +
                       (size_t)kWarps * kStages * sizeof(uint64_t) + 16
                 : (size_t)kWarps * (kGS + 4) * row_floats * 4 +
                       (size_t)kWarps * (kGS + 2) * TPW * sizeof(uint64_t) + 16;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return fail(kCuda, "token_loss_fact smem: %s", cudaGetErrorString(e));
    }
    kernel<<<grid, kThreads, smem, s>>>(h2w, epp, frame_of, tokens, lp_old, adv, N, K, A, prm,
                                        fix_stats, dz, g_frame, lp_new, stat_part, max_part);
    return post_launch("token_loss_fact_kernel");
  };
  // grouped kernel in scalar mode or dz mode
  auto grp = [&](auto kernel_dz, auto kernel_sc, int VPL, int TPW) -> int {
    const size_t smem = (size_t)kWarps * (kGS + 4) * VPL * 32 * 4 +
                        (size_t)kWarps * (kGS + 2) * TPW * sizeof(uint64_t) + 16;
    auto launch = [&](auto kernel) -> int {
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(kCuda, "token_loss_fact smem: %s", cudaGetErrorString(e));
      }
      kernel<<<grid, kThreads, smem, s>>>(h2w, epp, frame_of, tokens, lp_old, adv, N, K, A, prm,
                                          fix_stats, dz, static_cast<float4*>(tsc), g_frame, lp_new,
                                          stat_part, max_part);
      return post_launch("token_loss_fact_grp_kernel");
    };
    return tsc ? launch(kernel_sc) : launch(kernel_dz);
  };
  // two-phase warp-per-transition kernel (dz output, K <= 8, A in {128, 256})
  auto two_phase = [&](auto kernel) -> int {
    // two CTAs per SM: 2 x (dynamic + ~5 KB static + 1 KB reserved) <= 228 KB
    const size_t per_warp = (size_t)fact2_warp_floats(K, A) * 4 + 2 * sizeof(uint64_t);
    const int nw = (int)std::max<size_t>(
        1, std::min<size_t>(kF2MaxWarps, (size_t)(107 * 1024) / per_warp));
    const size_t smem = (size_t)nw * per_warp + 16;
    if (smem > 48 * 1024) {
      cudaError_t e =
          cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return fail(kCuda, "token_loss_fact2 smem: %s", cudaGetErrorString(e));
    }
    // the work counter of this pass (a fix-up launch uses the second one, so a
    // skipped fix-up never races the next step's main pass)
    if (!counters) return fail(kDimension, "token_loss_fact2: NULL work counters");
    unsigned* ctr = counters + (fix_stats ? 1 : 0);
    if (cudaMemsetAsync(ctr, 0, sizeof(unsigned), s) != cudaSuccess)
      return fail(kCuda, "token_loss_fact2: counter reset");
    kernel<<<grid, nw * 32, smem, s>>>(h2w, epp, frame_of, tokens, lp_old, adv, N, K, prm,
                                       fix_stats, dz, g_frame, lp_new, stat_part, max_part, ctr,
                                       static_cast<float4*>(tsc), tsc_pos,
                                       __builtin_ctz((unsigned)fact2_chunk(N)));
    return post_launch("token_loss_fact2_kernel");
  };
  if (K == 7 && A == 256)
    return tsc ? (fact2_chunk(N) == kF2Chunk ? two_phase(token_loss_fact2_kernel<8, 8, 7, true, 5>)
                                             : two_phase(token_loss_fact2_kernel<8, 8, 7, true>))
               : two_phase(token_loss_fact2_kernel<8, 8, 7, false>);
  if (K <= 8 && A == 256)
    return tsc ? two_phase(token_loss_fact2_kernel<8, 8, 0, true>)
               : two_phase(token_loss_fact2_kernel<8, 8, 0, false>);
  if (K == 7 && A == 128)
    return tsc ? two_phase(token_loss_fact2_kernel<4, 8, 7, true>)
               : two_phase(token_loss_fact2_kernel<4, 8, 7, false>);
  if (K <= 8 && A == 128)
    return tsc ? two_phase(token_loss_fact2_kernel<4, 8, 0, true>)
               : two_phase(token_loss_fact2_kernel<4, 8, 0, false>);
  if (tsc_pos != nullptr)
    return fail(kDimension, "token_loss_fact: sorted scalar output needs K <= 8, A in {128, 256}");
  const bool full = A == 128 || A == 256 || A == 512 || A == 1024;
  // grouped kernel: 16 (32 at A = 1024) logits per lane, A / that lanes per transition
  if (A == 128 && K <= 8)
    return grp(token_loss_fact_grp_kernel<16, 8, false>, token_loss_fact_grp_kernel<16, 8, true>, 16, 4);
  if (A == 256 && K <= 16)
    return grp(token_loss_fact_grp_kernel<16, 16, false>, token_loss_fact_grp_kernel<16, 16, true>, 16, 2);
  if (A == 512 && K <= 32)
    return grp(token_loss_fact_grp_kernel<16, 32, false>, token_loss_fact_grp_kernel<16, 32, true>, 16, 1);
  if (A == 1024 && K <= 32)
    return grp(token_loss_fact_grp_kernel<32, 32, false>, token_loss_fact_grp_kernel<32, 32, true>, 32, 1);
  if (tsc) return fail(kDimension, "token_loss_fact: scalar output needs A in {128, 256, 512, 1024}");
  if (A <= 128)
    return full ? go(token_loss_fact_kernel<4, true>, 4) : go(token_loss_fact_kernel<4, false>, 4);
  if (A <= 256)
    return full ? go(token_loss_fact_kernel<8, true>, 8) : go(token_loss_fact_kernel<8, false>, 8);
  if (A <= 512)
    return full ? go(token_loss_fact_kernel<16, true>, 16)
                : go(token_loss_fact_kernel<16, false>, 16);
  return full ? go(token_loss_fact_kernel<32, true>, 32) : go(token_loss_fact_kernel<32, false>, 32);
}

extern "C" int accel_pk_marginals(const float* dpk, int K, int A, float* dprev, float* dpos,
                                  void* stream) {
  if (K < 1 || A < 1 || !dpk || !dprev || !dpos) return fail(kDimension, "pk_marginals: bad args");
  const int nprev = A + 1;
  const int dprev_blocks = (int)std::min<int64_t>(ceil_div((int64_t)nprev * A, 256), (int64_t)kNumSMs * 2);
  const int grid = dprev_blocks + K * ((A + 31) / 32);
  pk_marginals_kernel<<<grid, 256, 0, as_stream(stream)>>>(dpk, K, A, nprev, dprev_blocks, dprev,
                                                           dpos);
  return post_launch("pk_marginals_kernel");
}
