/* Counter-hash weight generator of synth.weight_bits, in C for full-size models (the bench's
 * CPU timing variant generates 7.9 G weights).  Same law, bit for bit (tests/test_oracle_model.py):
 *   h = splitmix64(seed ^ stream << 40 ^ i), k = (h >> 40) - 2^23,
 *   w = bf16_rne(f32(f32(k * 2^-23) * f32(0.02 * sqrt(3)))), returned as fp32.
 * Input generation only: no arithmetic of the method lives here.  */
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void synth_weight_values_f32(uint64_t seed, uint64_t stream, uint64_t start, uint64_t n, float amp, float *out) {
  const uint64_t base = seed ^ (stream << 40);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < (int64_t)n; ++j) {
    const uint64_t h = splitmix64(base ^ (start + (uint64_t)j));
    const int64_t k = (int64_t)(h >> 40) - (1 << 23);
    const volatile float v = (float)k * 0x1p-23f; /* exact */
    const volatile float w = v * amp;             /* one fp32 RNE product */
    uint32_t u;
    memcpy(&u, (const void *)&w, 4);
    u = ((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16) << 16;
    memcpy(&out[j], &u, 4);
  }
}
