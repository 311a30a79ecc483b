/* TEST INFRASTRUCTURE — float64 C restatement of the reference GAE and
 * pooled-normalization statistics, for parity checks at full cfg2 sizes
 * where the Python loop of the reference (trainer.py:97-99) is too slow.
 *
 * oracle_gae_csr restates trainer.py:79-101 per trajectory of a CSR batch
 * (values hold T+1 frames per trajectory, bootstrap zeroed on done).
 * oracle_sums restates shard_statistics (trainer.py:128-132) for one shard.
 */
#include <stddef.h>
#include <stdint.h>

void oracle_gae_csr(const double* rewards, const double* values_frames,
                    const int64_t* off, const uint8_t* done, int64_t n_traj,
                    double gamma, double lam, double* adv, double* ret) {
  for (int64_t s = 0; s < n_traj; ++s) {
    const int64_t a = off[s], b = off[s + 1];
    const double* v = values_frames + a + s; /* T+1 values of trajectory s */
    const int64_t T = b - a;
    double carry = 0.0;
    for (int64_t t = T - 1; t >= 0; --t) {
      const double v_next = (t == T - 1 && done[s]) ? 0.0 : v[t + 1];
      const double delta = rewards[a + t] + gamma * v_next - v[t];
      carry = delta + gamma * lam * carry;
      adv[a + t] = carry;
      ret[a + t] = carry + v[t];
    }
  }
}

void oracle_sums(const double* x, int64_t n, double* s_out, double* q_out) {
  double s = 0.0, q = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    s += x[i];
    q += x[i] * x[i];
  }
  *s_out = s;
  *q_out = q;
}
