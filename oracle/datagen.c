/* CPU restatement of the reference datagen (pkg/src/laspsim/datagen.py:22-57) —
 * TEST INFRASTRUCTURE ONLY, like the rest of oracle/: it fills the oracle's
 * inputs for bench.py's CPU arms at full size (numpy takes ~9 s per 2^28
 * values). Bit-exact with oracle/lasp_oracle.py::gen_data (tests/test_oracle.py).
 *
 *   h0 = mix64(seed ^ tag_word)                (tag_word: blake2b-8, computed in Python)
 *   h  = mix64(mix64(h0 ^ row) ^ col)
 *   x  = 2 * ((h >> 11) * 2^-53) - 1           (float64, then cast to the output dtype)
 */
#include <stdint.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline double value(uint64_t h0, int64_t r, int64_t c) {
  const uint64_t h = mix64(mix64(h0 ^ (uint64_t)r) ^ (uint64_t)c);
  return 2.0 * ((double)(h >> 11) * 0x1p-53) - 1.0;
}

void oracle_gen_data_f64(uint64_t h0, int64_t rows, int64_t cols, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = value(h0, r, c);
}

void oracle_gen_data_f32(uint64_t h0, int64_t rows, int64_t cols, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = (float)value(h0, r, c);
}
