// host_rng.cu -- synthetic-data generator of the runtime (host side).
//
// The reference fixes its generator so weight draws and shuffles reproduce
// across platforms (rng.hpp:9-11): xoshiro256** seeded through splitmix64
// (rng.cpp:10-59).  The bench and the data feed use the same stream so the
// GPU run, the CPU baseline and the parity tests see identical inputs.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ck/ck.h"

namespace {
struct Rng {
  uint64_t s[4];
};
uint64_t splitmix64(uint64_t* st) {
  uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
inline uint64_t next(Rng* r) {
  uint64_t* s = r->s;
  uint64_t result = rotl(s[1] * 5, 7) * 9;
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}
inline double uniform(Rng* r) { return (double)(next(r) >> 11) * 0x1.0p-53; }
inline double normal(Rng* r) {
  double u1 = 1.0 - uniform(r);
  double u2 = uniform(r);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}
}  // namespace

extern "C" {
void* ck_rng_create(uint64_t seed) {
  Rng* r = new Rng;
  uint64_t sm = seed;
  for (int k = 0; k < 4; ++k) r->s[k] = splitmix64(&sm);
  return r;
}
void ck_rng_destroy(void* r) { delete static_cast<Rng*>(r); }
void ck_rng_uniform(void* r, float* out, int64_t n, float lo, float hi) {
  for (int64_t k = 0; k < n; ++k) out[k] = lo + (hi - lo) * (float)uniform(static_cast<Rng*>(r));
}
void ck_rng_normal(void* r, float* out, int64_t n, float scale) {
  for (int64_t k = 0; k < n; ++k) out[k] = (float)(scale * normal(static_cast<Rng*>(r)));
}
void ck_rng_labels(void* r, float* out, int64_t n, uint64_t classes) {
  for (int64_t k = 0; k < n; ++k)
    out[k] = (float)(1 + (classes ? next(static_cast<Rng*>(r)) % classes : 0));
}
// rng.cpp:51-59 Xoshiro256::permutation: Fisher-Yates with below(k + 1)
void ck_rng_permutation(void* r, int64_t n, int64_t* out) {
  Rng* g = static_cast<Rng*>(r);
  for (int64_t k = 0; k < n; ++k) out[k] = k;
  for (int64_t k = n - 1; k > 0; --k) {
    const uint64_t j = next(g) % (uint64_t)(k + 1);  // below(k + 1), rng.cpp:49
    const int64_t t = out[k];
    out[k] = out[j];
    out[j] = t;
  }
}
// rng.hpp:31-32 state() / set_state(): the generator state a checkpoint keeps
void ck_rng_get_state(const void* r, uint64_t state[4]) {
  for (int k = 0; k < 4; ++k) state[k] = static_cast<const Rng*>(r)->s[k];
}
void ck_rng_set_state(void* r, const uint64_t state[4]) {
  for (int k = 0; k < 4; ++k) static_cast<Rng*>(r)->s[k] = state[k];
}
}
