/* mf_host.c -- host-side helpers: the config-4 signal generator and fold_checksum.
 *
 * Config-4 generator (BASELINE.json config 4):
 *
 * x_i = i/n + 0.01 * sqrt(-2 ln(1-u1)) * cos(2 pi u2), u1 then u2 two SplitMix64
 * (generators.hpp:16-29) uniforms (next>>11)*2^-53, evaluated left to right in double.
 * It depends on libm's log/cos and on floating-point contraction, so it is generated
 * on the host and built with -ffp-contract=off (SURVEY.md §8(c) pitfall); its
 * checksum is pinned by tests/golden/configs.json.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

static inline uint64_t sm64(uint64_t *s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void mf_generate_trend_f64_host(uint64_t seed, size_t n, double *out) {
  uint64_t s = seed;
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (size_t i = 0; i < n; ++i) {
    const double u1 = (double)(sm64(&s) >> 11) * 0x1.0p-53;
    const double u2 = (double)(sm64(&s) >> 11) * 0x1.0p-53;
    out[i] = (double)i / (double)n + 0.01 * sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
  }
}

/* fold_checksum (io.hpp:17-28): FNV-1a over the 8 little-endian bytes of every value,
 * 32-bit values sign-extended first.  Floats are folded over their signed totalOrder keys
 * (the key map of SURVEY.md §0.1), as the goldens are.  `state` chains folds: pass
 * MF_FOLD_INIT for a fresh fold, or the previous result to fold a continuation, so
 * fold(a ++ b) == fold(b, fold(a)) and per-shard outputs fold into the global checksum. */
uint64_t mf_fold_checksum(int dtype, const void *values, size_t n, uint64_t state) {
  uint64_t h = state;
  for (size_t i = 0; i < n; ++i) {
    int64_t v;
    if (dtype == 0) { /* MF_I32 */
      v = ((const int32_t *)values)[i];
    } else if (dtype == 1) { /* MF_I64 */
      v = ((const int64_t *)values)[i];
    } else if (dtype == 2) { /* MF_F32: key of the bits */
      const int32_t b = ((const int32_t *)values)[i];
      v = b >= 0 ? b : (b ^ 0x7FFFFFFF);
    } else { /* MF_F64 */
      const int64_t b = ((const int64_t *)values)[i];
      v = b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFll);
    }
    const uint64_t bits = (uint64_t)v;
    for (int byte = 0; byte < 8; ++byte) {
      h ^= (bits >> (8 * byte)) & 0xff;
      h *= 1099511628211ull;
    }
  }
  return h;
}
