// Per-ticket uniforms for the serving path, computed on the device.
//
// Reference: inference.run_batch (inference.py:146-159) draws request i's
// sampling uniforms from np.random.default_rng(SeedSequence([base_seed,
// ticket])).random(K), so a request's tokens do not depend on which batch it
// was served in (tests/test_inference.py:148-170).  The host loop over
// tickets (one SeedSequence + PCG64 construction each, ~10 us) was the serving
// path's bottleneck; here one thread per ticket restates the same arithmetic
// and produces the identical doubles:
//   * SeedSequence (numpy/random/bit_generator.pyx): the entropy [base_seed,
//     ticket] as little-endian uint32 words (a zero int is one 0 word), hashed
//     into a 4-word pool (hashmix with INIT_A / MULT_A, cross-mixed with
//     MIX_MULT_L / MIX_MULT_R), then generate_state(4, uint64) with INIT_B /
//     MULT_B (uint32 words paired little-endian into uint64);
//   * PCG64 (XSL-RR 128/64): state 0, inc = (seq << 1) | 1, step, state +=
//     seed, step; each draw steps then outputs rotr64(hi ^ lo, state >> 122);
//   * random(): (next64 >> 11) * 2^-53.
// Integers up to 2^64 - 1 for base_seed and tickets (two entropy words each).
#include "common.cuh"

namespace accel {
namespace {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kShift = 16;

__host__ __device__ inline uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> kShift;
  return v;
}

__host__ __device__ inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kShift;
  return r;
}

// a non-negative integer as numpy's _int_to_uint32_array: little-endian words,
// zero -> one zero word
__host__ __device__ inline int int_words(uint64_t n, uint32_t* w) {
  if (n == 0) {
    w[0] = 0;
    return 1;
  }
  int c = 0;
  while (n > 0) {
    w[c++] = (uint32_t)(n & 0xFFFFFFFFull);
    n >>= 32;
  }
  return c;
}

__host__ __device__ inline uint64_t rotr64(uint64_t v, unsigned r) {
  return (v >> r) | (v << ((64u - r) & 63u));
}

__host__ __device__ inline void ticket_draws(uint64_t base_seed, uint64_t ticket, int K,
                                             double* out) {
  uint32_t ent[4];
  int ne = int_words(base_seed, ent);
  ne += int_words(ticket, ent + ne);
  // mix_entropy into a pool of 4 words
  uint32_t pool[4];
  uint32_t h = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u, h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], h));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s], h));
  // generate_state(4, uint64): 8 uint32 words cycling the pool
  uint32_t st[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> kShift;
    st[i] = v;
  }
  uint64_t w[4];
  for (int i = 0; i < 4; ++i) w[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
  // PCG64 seeding: seed = w0:w1 (high:low), seq = w2:w3
  using u128 = unsigned __int128;
  const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
  const u128 seed = ((u128)w[0] << 64) | (u128)w[1];
  const u128 seq = ((u128)w[2] << 64) | (u128)w[3];
  const u128 inc = (seq << 1) | (u128)1;
  u128 state = 0;
  state = state * mult + inc;
  state += seed;
  state = state * mult + inc;
  for (int k = 0; k < K; ++k) {
    state = state * mult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const uint64_t x = rotr64(hi ^ lo, (unsigned)(state >> 122));
    out[k] = (double)(x >> 11) * (1.0 / 9007199254740992.0);
  }
}

__global__ void ticket_uniforms_kernel(uint64_t base_seed, const int64_t* __restrict__ tickets,
                                       int64_t n, int K, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ticket_draws(base_seed, (uint64_t)__ldg(tickets + i), K, out + i * K);
}

}  // namespace
}  // namespace accel

using namespace accel;

extern "C" int accel_ticket_uniforms(uint64_t base_seed, const int64_t* tickets, int64_t n, int K,
                                     double* out, void* stream) {
  if (n < 0 || K < 0) return fail(kDimension, "ticket_uniforms: bad sizes");
  if (n == 0 || K == 0) return kOk;
  if (!tickets || !out) return fail(kDimension, "ticket_uniforms: NULL buffer");
  const int grid = (int)std::min<int64_t>(ceil_div(n, 128), (int64_t)kNumSMs * 4);
  ticket_uniforms_kernel<<<grid, 128, 0, as_stream(stream)>>>(base_seed, tickets, n, K, out);
  return post_launch("ticket_uniforms_kernel");
}

// The same arithmetic on the host (no device needed): the CPU tests pin it to
// numpy's draws.
extern "C" int accel_ticket_uniforms_host(uint64_t base_seed, const int64_t* tickets, int64_t n,
                                          int K, double* out) {
  if (n < 0 || K < 0) return fail(kDimension, "ticket_uniforms: bad sizes");
  if (n > 0 && K > 0 && (!tickets || !out)) return fail(kDimension, "ticket_uniforms: NULL buffer");
  for (int64_t i = 0; i < n; ++i) ticket_draws(base_seed, (uint64_t)tickets[i], K, out + i * K);
  return kOk;
}
