/*
 * accel.h — C ABI of libaccel.so, the sm_100a kernels behind the AcceRL
 * trainer hot path (paper_2603_18464_b200).
 *
 * The reference (`/root/reference/pkg/src/asyncrl`, pure Python + NumPy)
 * has no FFI; each entry point below replaces one NumPy block of the
 * reference trainer and names it (file:line, relative to
 * `pkg/src/asyncrl/`).  INTEGRATION.md shows the ctypes binding a
 * maintainer would add on the reference side.
 *
 * Conventions (all entry points):
 *   - plain device pointers + sizes; `stream` is a cudaStream_t passed as
 *     void*; every call is stream-ordered and asynchronous; no entry point
 *     allocates device memory (callers size workspaces with *_workspace_size);
 *   - return status: 0 ok, 1 invalid config/domain (DomainError),
 *     2 shape (DimensionError), 3 non-finite (NonFiniteError), 4 CUDA error;
 *   - accel_last_error() returns a thread-local message for the last
 *     non-zero status;
 *   - domain errors that depend on device data (e.g. a negative pooled
 *     variance) are reported through flag words in the output buffers that
 *     the caller reads at its next (already required) host sync;
 *   - no entry point allocates or keeps device-global scratch: work
 *     counters and multi-level partials live in caller buffers (e.g. the
 *     `counters` of accel_token_loss_fact2, the `scratch` of
 *     accel_reduce_f64), so calls on different streams are independent when
 *     their buffers are; host-side caches (grid sizes, SM counts) are per
 *     device.
 */
#ifndef ACCEL_H_
#define ACCEL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ---------------------------------------------------------- */
const char* accel_last_error(void);
/* number of kernels this library has launched in the process (for the
 * bench's gpu_launches claim) */
unsigned long long accel_launch_count(void);
/* Hash of the sources + flags this library was built from (build.py). */
const char* accel_build_id(void);
/* ABI version: 4 (3: row pitches on accel_tanh_grad_colsum, caller workspace on
 * accel_small_gemm, perm-based accel_fact_group_sum2, piece keys on
 * accel_grouped_rows_sum, accel_value_attn_backward; 4: heavy_key on
 * accel_fold_blocked_pieces). */
int accel_version(void);

/* One strided copy (cudaMemcpy2DAsync, any direction): `height` rows of
 * `width` bytes from src (row pitch spitch) to dst (row pitch dpitch).  Used to
 * upload frame rows into pitched device storage. */
int accel_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                  size_t height, void* stream);

/* ---- (a) advantages ---------------------------------------------------- */

/* Workspace bytes for accel_gae_segmented over n_traj trajectories holding
 * n_transitions steps (per-CTA float64 partials + an arrival counter; the
 * size does not depend on the batch). */
size_t accel_gae_workspace_size(int64_t n_traj, int64_t n_transitions);

/* Segmented reverse-scan GAE over a ragged CSR batch.
 * Replaces: the per-trajectory `compute_gae` loop (trainer.py:79-101) called
 * from `Trainer.build_train_batch` (trainer.py:365-381), plus the per-shard
 * (S, Q, N) sums of `shard_statistics` (trainer.py:128-132).
 *   rewards        f32[N]          transition rewards, trajectory-major
 *   values_frames  f32[N + n_traj] V(o_t) for t = 0..T of every trajectory
 *                                  (bootstrap frame last, trainer.py:369)
 *   traj_off       i64[n_traj + 1] transition offsets, traj_off[0] = 0,
 *                                  strictly increasing (T >= 1)
 *   done           u8[n_traj]      true termination (zeroes the bootstrap,
 *                                  trainer.py:92-93)
 *   adv_out, ret_out f32[N]        advantages and value targets (:100)
 *   frame_of_out   i32[N] or NULL  frame row of each transition (i + traj)
 *   sums_out       f64[4]          {sum A, sum A^2, N, #non-finite A/ret}
 */
int accel_gae_segmented(const float* rewards, const float* values_frames,
                        const int64_t* traj_off, const uint8_t* done,
                        int64_t n_traj, int64_t n_transitions,
                        double gamma, double lam,
                        float* adv_out, float* ret_out, int32_t* frame_of_out,
                        double* sums_out, void* workspace, size_t workspace_bytes,
                        void* stream);

/* Pooled mean/std from (possibly all-reduced) sums — trainer.py:135-150.
 *   sums   f64[3] {S, Q, N}
 *   stats_out f64[4] {mean, std, denom = std + eps, flags}
 *   flags bit0: N == 0 ("cannot normalize zero advantages", :143-144)
 *         bit1: pooled variance < -1e-12 (:147-148)                     */
int accel_normalize_finalize(const double* sums, double eps, double* stats_out,
                             void* stream);

/* adv_norm = (adv - mean) / denom — trainer.py:151. */
int accel_normalize_apply(const float* adv, int64_t n, const double* stats,
                          float* adv_norm_out, void* stream);

/* ---- (b) token loss --------------------------------------------------- */

/* CTA count used by the token kernels for M rows (sizes their partials). */
int accel_token_grid(int64_t M);

/* Behavior log-probs — replaces `behavior_log_probs` (trainer.py:289-293).
 *   mu f32[M, A] behavior logits, tokens i32[M] -> lp_out f32[M]
 *   bad_part f64[grid][2]: {rows with non-finite logits (the reference's
 *   log_softmax raises DomainError, numerics.py:138-139), tokens outside
 *   [0, A)} per CTA (grid = accel_token_grid(M)). */
int accel_token_logp(const float* mu, const int32_t* tokens, int64_t M, int A,
                     float* lp_out, double* bad_part, void* stream);

/* Fused token loss forward + backward over logit rows — replaces
 * `log_prob_chunk` (models.py:219-223), `policy_surrogate`
 * (trainer.py:183-239), `entropy_bonus` (:242-251) and the dlogits assembly
 * of `train_step` (:425-435).
 *   logits f32[M, A] (head GEMM output WITHOUT bias), bias f32[A] (b_head),
 *   tokens i32[M], lp_old f32[M], adv f32[M / K] (normalized, one per
 *   transition), algo 0 = "trust" (GIPO), 1 = "clip" (PPO),
 *   m_global = token count over all ranks (entropy mean denominator and the
 *   optimistic included count).
 *   fix_stats == NULL: main pass; writes dlogits f32[M, A], lp_new f32[M],
 *     dbias_part f32[grid][A], stat_part f64[grid][8] {sum w r a | sum min-surr,
 *     sum H, sum r, sum w, #outside clip band, #excluded, #non-finite rows,
 *     #bad tokens}, max_part f64[grid][2] {max r, -min w}.
 *   fix_stats != NULL (the reduced, all-rank stat vector): FIXUP pass; if
 *     0 < #excluded < m_global rewrites dlogits and dbias_part with the true
 *     included count, else returns immediately (device-side decision). */
int accel_token_loss(const float* logits, const float* bias, const int32_t* tokens,
                     const float* lp_old, const float* adv, int64_t M, int K, int A,
                     int algo, double sigma, double clip_eps, double lambda_h,
                     double m_global, const double* fix_stats, float* dlogits,
                     float* lp_new, float* dbias_part, double* stat_part,
                     double* max_part, void* stream);

/* Factorized-head variant (the production path for 128 <= A <= 1024,
 * A % 4 == 0, K <= 32): logits are never materialized.  logits[i,k] =
 * h2w[frame_of[i]] + epp[prev*K + k] with h2w = h2 W_head^T (f32[F, A]) and
 * epp = e_prev W_head^T + e_pos W_head^T + b_head (f32[(A+1)*K, A],
 * accel_ep_plus) — models.py:181-182 distributed over c = h2 + e_prev[prev]
 * + e_pos.  Writes either dz f32[N*K, A] (per-token dlogits) or, with dz =
 * NULL, tsc f32x4[N*K] = {nm2, Ac, Cc, coef} per token, from which
 * dz = 2^d2 (Ac d2 + Cc) (+ coef at the token), d2 = logit log2(e) + nm2 is
 * recomputed by accel_fact_group_sum (A in {128, 256, 512, 1024}); plus
 * g_frame f32[F, A] rows frame_of[i] = sum_k dz[i, k] (pre-zero the bootstrap
 * rows), lp_new, stat_part/max_part as accel_token_loss (grid =
 * accel_fact_grid(N)).  fix_stats: FIXUP pass as accel_token_loss. */
int accel_fact_grid(int64_t N);
/* Rows of stat_part / max_part accel_token_loss_fact2 writes for these sizes:
 * one per 32-transition chunk for the two-phase kernel (K <= 8, A in {128, 256};
 * fixed rows under its dynamic schedule, so the pooled statistics are bitwise
 * reproducible), accel_fact_grid(N) per-CTA rows otherwise. */
int64_t accel_fact_partials(int64_t N, int K, int A, int scalar_out);
/* epp[(prev*K+k)*A + a] = ep[prev*A + a] + pp[k*A + a] + bias[a] */
int accel_ep_plus(const float* ep, const float* pp, const float* bias, int A, int K,
                  float* epp, void* stream);
/* tsc_pos (nullable): token t's scalars go to tsc[tsc_pos[t]] (the sorted
 * position of a frame-blocked grouping).  counters: u32[2] caller workspace
 * (the dynamic schedule's work counters of the main / fix-up pass; reset on
 * the call's stream). */
int accel_token_loss_fact2(const float* h2w, const float* epp, const int32_t* frame_of,
                           const int32_t* tokens, const float* lp_old, const float* adv,
                           int64_t N, int K, int A, int algo, double sigma, double clip_eps,
                           double lambda_h, double m_global, const double* fix_stats, float* dz,
                           void* tsc, const int32_t* tsc_pos, float* g_frame, float* lp_new,
                           double* stat_part, double* max_part, unsigned* counters,
                           void* stream);
/* Grouped dz sums over the (prev, position) keys without dz in HBM: piece
 * partials f32[n_pieces, A] (then accel_grouped_rows_sum's key pass) of the dz
 * rows recomputed from h2w/epp and the tsc scalars, rows in the stable key
 * order of accel_group_by_key (perm/seg_off/piece_off; piece_rows = 256).
 * Reference: the np.add.at of models.py:195 (dc rows grouped by prev token). */
int accel_fact_group_sum(const float* h2w, const float* epp, const int32_t* frame_of,
                         const int32_t* tokens, const void* tsc, const int32_t* perm,
                         const int64_t* seg_off, const int64_t* piece_off, int nkeys,
                         int key_mod, int K, int A, int piece_rows, int64_t n_pieces,
                         float* piece_out, void* stream);
/* key_mod > 0: the grouping is frame-blocked (accel_group_by_key_blocked), its
 * composite key is block * key_mod + (prev * K + k) and the EPP row is
 * key % key_mod; consecutive pieces then gather H2W rows of one block of
 * frames, which stays L2-resident. */
/* Dprev f32[A+1, A] = sum_k dpk[j, k]; Dpos f32[K, A] = sum_j dpk[j, k]
 * from the (prev, k)-grouped dz sums dpk f32[(A+1)*K, A]. */
int accel_pk_marginals(const float* dpk, int K, int A, float* dprev, float* dpos,
                       void* stream);

/* ---- policy glue (models.py:165-209) ----------------------------------- */

/* z = tanh(z + b) in place, z f32[rows, cols] — models.py:176-177. */
int accel_bias_tanh(float* z, const float* b, int64_t rows, int cols, void* stream);

/* c[i*K+k] = h2[frame_of[i]] + e_prev[prev] + e_pos[k], prev = A for k = 0
 * else tokens[i*K+k-1] — models.py:178-181.  c_out f32[N*K, D]. */
int accel_build_c(const float* h2, const int32_t* frame_of, const int32_t* tokens,
                  const float* e_prev, const float* e_pos, int64_t N, int K, int A,
                  int D, float* c_out, void* stream);

/* Default CTA count for the column-reduction kernels over `rows` rows. */
int accel_rows_grid(int64_t rows);

/* From dc = dlogits @ W_head (f32[N*K, D]): dh2 = sum_k dc, dz2[frame] =
 * dh2 (1 - h2^2) (dz2 f32[F, D], bootstrap rows left untouched — pre-zero),
 * pos_part f32[grid][K][D] (de_pos), db1_part f32[grid][D] —
 * models.py:196-200.  K <= 16. */
int accel_dc_reduce(const float* dc, const float* h2, const int32_t* frame_of,
                    int64_t N, int K, int D, float* dz2, float* pos_part,
                    float* db1_part, int grid, void* stream);

/* g = g (1 - h^2) in place over f32[R, C] (row pitches ldg, ldh >= C);
 * col_part f32[grid][C] — models.py:202-204 (dz1 and db0). */
int accel_tanh_grad_colsum(float* g, int64_t ldg, const float* h, int64_t ldh, int64_t R, int C,
                           float* col_part, int grid, void* stream);

/* ---- deterministic scatter-add (np.add.at, models.py:195 and :305) ------ */

/* keys[i*K+k] = prev (with_pos = 0) or prev*K + k (with_pos = 1), prev = A
 * at k = 0 else tokens[i*K+k-1] (models.py:178-180). */
int accel_prev_keys(const int32_t* tokens, int64_t N, int K, int A, int with_pos,
                    int32_t* keys, void* stream);
/* keys[r] = steps[frame_of ? frame_of[r] : r]; bad_count += out-of-range
 * steps (the reference raises DimensionError, models.py:261-267). */
int accel_step_keys(const int32_t* steps, const int32_t* frame_of, int64_t R,
                    int n_steps, int32_t* keys, unsigned* bad_count, void* stream);
size_t accel_group_workspace_size(int64_t R, int nkeys);
int64_t accel_group_max_pieces(int64_t R, int nkeys);
/* Stable counting sort of R keys in [0, nkeys): perm i32[R], seg_off
 * i64[nkeys+1], piece_off i64[nkeys+1] (pieces of <= 256 rows per key). */
int accel_group_by_key(const int32_t* keys, int64_t R, int nkeys, int32_t* perm,
                       int64_t* seg_off, int64_t* piece_off, void* workspace,
                       size_t workspace_bytes, void* stream);
/* out f32[nkeys, D] = sum of vals rows per key, in perm order (bitwise
 * deterministic); piece_buf f32[accel_group_max_pieces(R, nkeys) * D].
 * vals = NULL: only the key pass (piece_buf already filled, e.g. by
 * accel_fact_group_sum). */
/* Frame-blocked variant: rows are cut into blocks of cpb 4096-row chunks
 * (cpb <= 0: one block) and sorted stably by (block, key); seg_off and
 * piece_off cover the blocks * nkeys composite keys (block-major). */
size_t accel_group_workspace_size_blocked(int64_t R, int nkeys, int64_t cpb);
int64_t accel_group_max_pieces_blocked(int64_t R, int nkeys, int64_t cpb);
int64_t accel_group_blocks(int64_t R, int64_t cpb);
int accel_group_by_key_blocked(const int32_t* keys, int64_t R, int nkeys, int64_t cpb,
                               int32_t* perm, int64_t* seg_off, int64_t* piece_off,
                               int32_t* piece_key, const int32_t* frame_of, const int32_t* tokens,
                               int K, int32_t* row_frame, int32_t* row_tok, int32_t* pos,
                               void* workspace, size_t workspace_bytes, void* stream);
/* pos != NULL: the scatter also writes the inverse permutation pos[perm[r]] = r
 * (coalesced); row_frame / row_tok != NULL (with frame_of, tokens, K): also the
 * sorted per-row metadata of a (prev, k) grouping, as accel_sorted_rows. */
/* piece_key (nullable) i32[accel_group_max_pieces_blocked]: owning composite key
 * of each piece. */
/* Sorted per-row metadata of a grouping (fixed per batch): row_frame[r] =
 * frame_of[perm[r] / K], row_tok[r] = tokens[perm[r]], pos[perm[r]] = r. */
int accel_sorted_rows(const int32_t* perm, const int32_t* frame_of, const int32_t* tokens,
                      int64_t R, int K, int32_t* row_frame, int32_t* row_tok, int32_t* pos,
                      void* stream);
/* accel_fact_group_sum over a blocked grouping: one CTA per piece (in (block,
 * key) order); a piece's token rows are perm[r] (frame frame_of[perm[r] / K],
 * token tokens[perm[r]]) and their scalars are contiguous in tsc_sorted (the
 * loss kernel's token scalars at their sorted positions, accel_token_loss_fact2
 * with tsc_pos = pos). */
int accel_fact_group_sum2(const float* h2w, const float* epp, const int32_t* perm,
                          const int32_t* frame_of, const int32_t* tokens, int K,
                          const void* tsc_sorted, const int64_t* seg_off,
                          const int64_t* piece_off, const int32_t* piece_key, int nkeys,
                          int key_mod, int A, int64_t n_pieces_max, float* piece_out,
                          void* stream);
/* out[nkeys, D] = sum over blocks (in order) of the pieces (in order) of the
 * composite keys b * nkeys + key: the key pass of a blocked grouping.
 * heavy_key (-1: none): a key holding a large share of the rows (the factorized
 * head's chunk-start key A * K), folded over more CTAs (a fixed partition:
 * deterministic). */
size_t accel_fold_workspace_size(int nkeys, int D);
int accel_fold_blocked_pieces(const float* piece_buf, const int64_t* piece_off, int nkeys,
                              int nblocks, int D, int heavy_key, float* out, void* workspace,
                              void* stream);
/* piece_key (nullable, from accel_group_by_key_blocked): the key of each piece
 * (else found by a binary search over piece_off per piece). */
int accel_grouped_rows_sum(const float* vals, int64_t R, int D, const int32_t* perm,
                           const int64_t* seg_off, const int64_t* piece_off,
                           const int32_t* piece_key, int nkeys, int64_t n_pieces,
                           float* piece_buf, float* out, void* stream);

/* ---- value head (models.py:273-314, trainer.py:438-443) ---------------- */

int accel_warp_grid(int64_t rows);
/* u = softmax_j(h_j . w_attn + b) pooled h + e_step[step]; U f32[R, D],
 * alpha f32[R, 2]; bad_part f64[grid][2] {non-finite scores, bad steps}. */
int accel_value_pool(const float* h1, const float* h2, const int32_t* row_frame,
                     const int32_t* steps, int64_t R, int D, int n_steps,
                     const float* w_attn, const float* b_attn, const float* e_step,
                     float* U, float* alpha, double* bad_part, int grid, void* stream);
/* zm f32[R, H] = u @ W0v^T (no bias); rows row_frame[r] (or r).  targets ==
 * NULL: forward only (values_out f32[R]).  Otherwise zm <- dzm, part
 * f32[grid][2H+1] {dw1v, db0v, db1v}, dpart f64[grid][2] {sum loss, non-finite
 * v}.  Loss: MSE (trainer.py:438-443), or with v_old f32[R] the PPO value-clip
 * loss max((v-R)^2, (v_old + clip(v - v_old, +-vclip) - R)^2) of the north star
 * (no reference counterpart; float64 checker oracle/trainer_ref.py). */
int accel_value_head(float* zm, const int32_t* row_frame, const float* b0v, const float* w1v,
                     const float* b1v, int64_t R, int H, const float* targets,
                     const float* v_old, double vclip, double lambda_v, double n_global,
                     float* values_out, float* part, double* dpart, int grid, void* stream);
/* de f32[R, 2] attention-score gradients, part f32[grid] (db_attn). */
int accel_value_attn_grad(const float* dU, const float* h1, const float* h2,
                          const int32_t* row_frame, const float* alpha, int64_t R, int D,
                          float* de, float* part, int grid, void* stream);
/* part f32[grid][D] (dw_attn). */
int accel_value_attn_wgrad(const float* de, const float* h1, const float* h2,
                           const int32_t* row_frame, int64_t R, int D, float* part,
                           int grid, void* stream);
/* Both of the above in one pass over (dU, h1, h2): bpart f32[grid] (db_attn),
 * wpart f32[grid][D] (dw_attn), de f32[R, 2] optional (NULL: not written;
 * required at widths other than D in {16, 32, 64, 128} with 16-B aligned rows). */
int accel_value_attn_backward(const float* dU, const float* h1, const float* h2,
                              const int32_t* row_frame, const float* alpha, int64_t R, int D,
                              float* de, float* bpart, float* wpart, int grid, void* stream);

/* ---- reductions, record, optimizer ------------------------------------- */

/* dst_i[j] = sum_p src_i[p * pitch_i + j] (fixed order), up to 16
 * segments; pitches == NULL means pitch_i = len_i. */
int accel_reduce_segments(const void* const* srcs, void* const* dsts,
                          const int64_t* parts, const int64_t* lens,
                          const int64_t* pitches, int nseg, void* stream);
/* out f64[nseg][3] = {sum, sum of squares, count} per segment of x —
 * shard_statistics (trainer.py:128-132). */
int accel_segment_moments(const float* x, const int64_t* off, int64_t nseg,
                          double* out, void* stream);
/* count += rows of x f32[*, C] (row pitch ld >= C; rows[r], or r when rows ==
 * NULL) holding a non-finite value — TrainBatch.check_finite on obs
 * (buffers.py:120-122). */
int accel_count_nonfinite_rows(const float* x, const int32_t* rows, int64_t R, int C,
                                int64_t ld, unsigned* count, void* stream);
/* out[c] = sum (mode 0) or max (mode 1) over p of part[p * width + c], in a
 * fixed order.  scratch: accel_reduce_f64_scratch_size(parts, width) bytes
 * (level-1 partials of the two-level path; NULL when that size is 0). */
size_t accel_reduce_f64_scratch_size(int64_t parts, int width);
int accel_reduce_f64(const double* part, int64_t parts, int width, int mode,
                     double* out, double* scratch, void* stream);
/* train_step record (trainer.py:417-464) -> record f64[17]:
 * {loss, policy_loss, value_loss, entropy, excluded_tokens, ratio_mean,
 *  ratio_max, trust_weight_mean, trust_weight_min, clipped_fraction,
 *  dropped, bad_logit_rows, bad_tokens, bad_attention, bad_grads,
 *  bad_steps, skip}; skip i32 gates accel_adam. */
int accel_step_finalize(const double* loss_sums, const double* loss_max,
                        const double* value_sums, const unsigned* bad_counts,
                        const double* attn_bad, int algo, double lambda_v,
                        double lambda_h, double n_tokens, double n_transitions,
                        double* record, int* skip, void* stream);
int accel_count_nonfinite(const float* x, int64_t n, unsigned* count, void* stream);
/* Adam (numerics.py:95-126) over a flat buffer: [0, n0) group0, [n0, n)
 * group1; group = HOST f64[6] {lr, beta1, beta2, eps, 1-beta1^t, 1-beta2^t}.
 * No-op when *skip; bad += non-finite new parameters. */
int accel_adam(const float* p_in, const float* g, const float* m_in, const float* v_in,
               float* p_out, float* m_out, float* v_out, int64_t n, int64_t n0,
               const double* group0, const double* group1, const int* skip,
               unsigned* bad, void* stream);
/* accel_adam with hyper f64[12] = {group 0, group 1} x {lr, beta1, beta2, eps,
 * 1 - beta1^t, 1 - beta2^t} in DEVICE memory, read at run time (CUDA-graph
 * replays of successive steps; the host refreshes hyper before each). */
int accel_adam_dev(const float* p_in, const float* g, const float* m_in, const float* v_in,
                   float* p_out, float* m_out, float* v_out, int64_t n, int64_t n0,
                   const double* hyper, const int* skip, unsigned* bad, void* stream);

/* Batched inference-service evaluation (inference.py:129-160, run_batch): one
 * warp per request, all of one kind; weights / dims as accel_imagine (unused
 * pointers of the other kinds may be dummies).  kind 0 policy: obs f64[n, O],
 * steps i32[n], uniforms f64[n, K] (the request's ticket substream) ->
 * tokens i32[n, K], logits f64[n, K, A], values f64[n]; kind 1 obs model:
 * chunks i32[n, K] -> next_obs f64[n, O]; kind 2 reward model -> probs f64[n]. */
int accel_serve(const void* const* weights, const int* dims, int kind, const double* obs,
                const int32_t* steps, const int32_t* chunks, const double* uniforms, int64_t n,
                int32_t* tokens_out, double* logits_out, double* values_out,
                double* next_obs_out, double* probs_out, void* stream);

/* ---- world-model training sub-steps (trainer.py:469-535), float64 ------- */

/* Workspace bytes of accel_wm_mlp2_grad for n rows, hidden dh, output dout. */
size_t accel_wm_workspace_size(int64_t n, int dh, int dout);
/* One forward + backward of a 2-layer tanh MLP (numerics.py:174-220):
 *   x f64[n, din], params f64 {w0 [dh, din], b0 [dh], w1 [dout, dh], b1 [dout]}
 *   kind 0: target f64[n, dout], loss = mean((out - target)^2)
 *           (train_obs_model_step, trainer.py:469-494)
 *   kind 1: target = labels f64[n], dout = 1, loss = mean(softplus(z) - y z)
 *           (train_reward_model_step, trainer.py:496-535)
 * grads f64 (same layout as params), loss_out f64[1], nonfinite u32[1] =
 * count of non-finite gradient entries (adam_step raises on them). */
int accel_wm_mlp2_grad(const double* x, const double* target, int64_t n, int din, int dh,
                       int dout, int kind, const double* params, double* grads,
                       double* loss_out, unsigned* nonfinite, void* workspace,
                       size_t workspace_bytes, void* stream);
/* Adam step t (>= 1) over a flat float64 buffer (numerics.py:95-126);
 * bad u32[1] = non-finite new parameters (ParamSet.check_finite). */
int accel_wm_adam(double* params, const double* grads, double* m, double* v, int64_t n,
                  double lr, double beta1, double beta2, double eps, int64_t t, unsigned* bad,
                  void* stream);

/* 3xTF32 operand split (x f32[n], n % 4 == 0): hi = x rounded to TF32, lo =
 * x - hi (diagnostics; the wide GEMMs below use accel_tf32_pairs). */
int accel_split_tf32(const float* x, int64_t n, float* hi, float* lo, void* stream);

/* Small products (<= a few hundred rows: e_prev / e_pos x W_head and their
 * gradients around the factorized head): C[M, N] = op(A) op(B)^T with A(m, k)
 * = a_trans ? A[k][m] : A[m][k], B(n, k) = b_trans ? B[k][n] : B[n][k]; fp32
 * FMA in a fixed k order. */
int accel_small_gemm(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                     int64_t lda, int64_t ldb, int64_t ldc, int a_trans, int b_trans,
                     float* ws, int64_t ws_floats, void* stream);
/* Workspace (floats) for split-K slices of accel_small_gemm: > 0 when the
 * product's output tiles leave SMs idle and k is long (e.g. e_pos [7, 4096] x
 * W_head^T at cfg4); the slices are summed in order (deterministic).  With a
 * smaller / NULL ws the product runs unsplit. */
int64_t accel_small_gemm_ws_floats(int64_t M, int64_t N, int64_t K);

/* ---- serving: per-ticket sampling uniforms (csrc/ticket_rng.cu) --------- */

/* out f64[n, K]: request i's uniforms as np.random.default_rng(SeedSequence(
 * [base_seed, tickets[i]])).random(K) (inference.py:146-159), one thread per
 * ticket; tickets >= 0.  The _host variant computes the same on the CPU. */
int accel_ticket_uniforms(uint64_t base_seed, const int64_t* tickets, int64_t n, int K,
                          double* out, void* stream);
int accel_ticket_uniforms_host(uint64_t base_seed, const int64_t* tickets, int64_t n, int K,
                               double* out);

/* ---- wide tensor-core GEMM (cfg4: O = D = 4096; csrc/tc_wide.cu) -------- */

/* bf16 "pair" operand of an fp32 matrix X [rows, cols] (pitch ld elements):
 * per 8-element group along K, [bf16(hi) x8 | bf16(lo) x8] ([lo | hi] when
 * lo_first), hi = trunc19(x) (the value a tf32 MMA reads from the raw word),
 * lo = x - hi.  row_pair = 0 (K = cols): out bf16[rows, 2*ceil8(cols)];
 * row_pair = 1 (K = rows): out bf16[2*ceil8(rows), cols]; pitch ldo elements,
 * ldo % 8 == 0, zero padding past K. */
int accel_tf32_pairs(const float* X, int64_t rows, int64_t cols, int64_t ld, void* out,
                     int64_t ldo, int row_pair, int lo_first, void* stream);
/* Tuning: k blocks (16 k) per fp32 accumulation chunk of accel_tc_gemm_wide
 * (0, the default: one chunk per work unit).  The tensor core's fp32
 * accumulate truncates; each chunk starts a fresh accumulator and the epilogue
 * adds chunks rounding to nearest through the output. */
void accel_tc_wide_set_chunk(int kblocks);
/* Tuning: 2 (default) = pairs of m tiles run as one 2-SM UMMA unit
 * (cta_group::2, clusters of 2, each CTA streaming half of the B tile);
 * 1 = 1-SM MMAs with the shared B tile multicast; 0 = one CTA per tile. */
void accel_tc_wide_set_multicast(int mode);
/* Work tiles (128 x BN, BN <= 256) of an M x N product (split-K sizing). */
int accel_tc_wide_tiles(int64_t M, int64_t N, int b_mn);
/* C = A . B^T with fp32-class accuracy from two tensor-core passes per 8-k
 * step: a tf32 MMA on the raw fp32 tiles (A_hi B_hi) plus a bf16 MMA on the
 * pair operands (A_hi B_lo + A_lo B_hi).  The dense products of the
 * OpenVLA-7B-shaped heads, forward and backward (models.py:176-209,
 * :283-314), where both dimensions exceed the resident-weight kernels.
 *   A: a_mn = 0 -> [M, K] (pitch lda), 1 -> stored [K, M];  Ap its pair array
 *      (accel_tf32_pairs with lo_first = 0, row_pair = a_mn), pitch ldap.
 *   B: b_mn = 0 -> [N, K], 1 -> stored [K, N];  Bp (lo_first = 1, row_pair =
 *      b_mn), pitch ldbp.
 *   epi 0: C[M, N] (ldc) = acc;  1: tanh(acc + bias[N]);  2: acc (1 - H^2)
 *      (H pitch ldh) and col_part f32[ceil(M/128)][N] = per-128-row-tile column
 *      sums of C (bias gradient, reduced in fixed order by the caller);
 *   3: split-K, C = f32[kslices][M][N] partial slices (caller reduces),
 *      kslices <= ceil(K / 16). */
int accel_tc_gemm_wide(const float* A, const void* Ap, const float* B, const void* Bp, float* C,
                       const float* bias, const float* H, float* col_part, int64_t M, int64_t N,
                       int64_t K, int64_t lda, int64_t ldap, int64_t ldb, int64_t ldbp,
                       int64_t ldc, int64_t ldh, int a_mn, int b_mn, int epi, int kslices,
                       void* stream);

/* ---- tensor-core GEMM (tcgen05, 3xTF32: fp32-accurate) ----------------- */

/* Streaming multiprocessors on the current device (persistent-grid size;
 * the weight-gradient mode takes kslices <= this). */
int accel_tc_sm_count(void);
/* Dense products of the policy/value heads (models.py:176-204, :283-314).
 *   a_trans = 0 (row transform): C[M, N] = act(A[M, K] . B^T + bias) (+ C if
 *     accumulate); B stored [N, K] (b_trans = 0) or [K, N] (b_trans = 1);
 *     kslices must be 1.  Persistent; B stays resident in shared memory.
 *   a_trans = b_trans = 1 (weight gradient, reduction over the K rows):
 *     A stored [K, M], B stored [K, N], M <= 256; C receives [2 * kslices][M][N]
 *     fp32 partials (two per persistent CTA, kslices <= accel_tc_sm_count())
 *     for a fixed-order reduction by the caller; no bias/act/accumulate.
 * fp32 in/out, N <= 256, any strides. */
/* accel_tc_gemm's row transform (a_trans = b_trans = 0) that also adds the
 * number of non-finite elements of A to *nonfinite (u32, device): the frame
 * finiteness check of build_train_batch (trainer.py:392-396) folded into the
 * first layer's read of the frames. */
int accel_tc_linear_checked(const float* A, const float* B, float* C, const float* bias,
                            int64_t M, int64_t K, int N, int64_t lda, int64_t ldb, int64_t ldc,
                            int act_tanh, unsigned* nonfinite, void* stream);
/* Persistent-grid size of the row-transform kernel for M rows. */
int accel_tc_rows_grid(int64_t M);
/* C[M, N] = (A[M, K] . B^T) * (1 - H[M, N]^2) -- a backward product fused with
 * the tanh derivative of the layer it feeds (models.py:197-200: dpre = dh (1 -
 * h^2)) -- and col_part f32[accel_tc_rows_grid(M)][N] = per-CTA column sums of C
 * (the bias gradient, reduced in fixed order by the caller).  B as in
 * accel_tc_gemm (b_trans); C and H need 16-byte aligned rows, N <= 256. */
int accel_tc_gemm_dtanh(const float* A, const float* B, float* C, const float* H,
                        float* col_part, int64_t M, int64_t K, int N, int64_t lda, int64_t ldb,
                        int64_t ldc, int64_t ldh, int b_trans, void* stream);
int accel_tc_gemm(const float* A, const float* B, float* C, const float* bias, int64_t M,
                  int64_t K, int N, int64_t lda, int64_t ldb, int64_t ldc, int a_trans,
                  int b_trans, int act_tanh, int accumulate, int kslices, void* stream);

/* ---- (c) world-model imagination (rollout.py:295-362) ------------------ */

/* Shared memory per 4-trajectory CTA (float64 activations). */
size_t accel_imagine_smem_bytes(int O, int D, int A, int HV, int HO, int HR);

/* H imagined steps for n trajectories in one launch, float64 throughout:
 * per step sample_chunk + state_value (models.py:135-150, :406-408),
 * ObsModel.predict (:349-355), snap_observation (env.py:259-283),
 * RewardModel.predict (models.py:375-377), r = p' - p, stop at p' >= threshold.
 *   weights  23 device pointers, f64, weight matrices TRANSPOSED ([in][out]):
 *            w0t b0 w1t b1 e_prev e_pos w_headt b_head | w_attn b_attn e_step
 *            w0vt b0v w1v b1v | ow0t ob0 ow1t ob1 | rw0t rb0 rw1 rb1
 *   dims     {O, D, K, A, n_steps, value_hidden, obs_hidden, reward_hidden,
 *             grid_h, grid_w, snap}
 *   uniforms f64[n, H+1, K] (request r of episode e uses uniforms[e, r]) or
 *            NULL for a Philox stream keyed by (seed, e)
 *   outputs  obs f64[n, H+1, O], steps i32[n, H+1], tokens i32[n, H, K],
 *            logits f64[n, H, K, A], values f64[n, H], rewards f64[n, H],
 *            boot f64[n], len i32[n], done u8[n], status i32[n]
 *            (0 ok, 1 non-finite obs prediction, 2 non-finite reward). */
int accel_imagine(const void* const* weights, const int* dims, int H, double threshold,
                  unsigned long long seed, const double* start_obs, const int32_t* start_step,
                  const double* uniforms, int64_t n, double* obs_out, int32_t* steps_out,
                  int32_t* tokens_out, double* logits_out, double* values_out,
                  double* rewards_out, double* boot_out, int32_t* len_out, uint8_t* done_out,
                  int32_t* status_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ACCEL_H_ */
