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
#include "token_common.cuh"

namespace accel {
namespace {

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
    __syncwarp();  // reconverge: lanes may leave the spin-wait at different times
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
    __syncwarp();  // reconverge: lanes may leave the spin-wait at different times
    float z[VPL], e[VPL];
    L::load(slot, lane, A, z, false);
    const bool bt = tok_raw < 0 || tok_raw >= A;
    const int tok = bt ? 0 : tok_raw;
    RowStats rs;
    if constexpr (FULL && VPL % 2 == 0) {
      rs = row_stats_logp<VPL>(z);
      rs.d_tok = slot[tok] - rs.d_tok;
    } else if (FULL) {
      rs = row_stats_full<VPL>(z, e, false);
      rs.d_tok = slot[tok] - rs.d_tok;
    } else {
      rs = row_stats<VPL, true>(z, e, lane, A, tok, false);
    }
    // (no proxy fence: the slot's reads were consumed by row_stats above; the bulk
    // copy refilling it is issued after them -- WAR ordering as in TMA pipelines)
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
