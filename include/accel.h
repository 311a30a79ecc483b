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
 *     the caller reads at its next (already required) host sync.
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
int accel_version(void);

/* ---- (a) advantages ---------------------------------------------------- */

/* Workspace bytes for accel_gae_segmented over n_transitions steps. */
size_t accel_gae_workspace_size(int64_t n_transitions);

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

#ifdef __cplusplus
}
#endif

#endif /* ACCEL_H_ */
