// synthetic.cu -- host-side seeded generators of the reference core
// (synthetic.hpp:12-40, tensors.hpp:142-150, random.hpp:14-26), so callers of
// the library (the bench, the drop-in) get the reference's synthetic inputs
// without the reference: std::mt19937_64 raw draws (bit-specified by the C++
// standard), uniform(lo, hi) = lo + (hi - lo) * ((x >> 11) * 2^-53), evaluated
// as one fused multiply-add, the contraction the reference's -march=native
// build emits for that expression.
#include <cmath>
#include <cstdint>
#include <random>

#include "npcg_internal.cuh"

namespace {

struct Uniform {
  std::mt19937_64 g;
  explicit Uniform(uint64_t seed) : g(seed) {}
  double u01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double operator()(double lo, double hi) { return std::fma(hi - lo, u01(), lo); }
};

}  // namespace

extern "C" {

// synthetic.cpp:12-23 gen_uniform_cube: x, y, z in [0, extent), in that draw order
npcg_status npcg_gen_uniform_cube(int64_t n, double extent, uint64_t seed, double* xyz) {
  if (n < 0) return NPCG_ERR_SHAPE;
  if (!(extent > 0.0)) return NPCG_ERR_DOMAIN;
  if (n > 0 && !xyz) return NPCG_ERR_INVALID;
  Uniform u(seed);
  for (int64_t p = 0; p < 3 * n; ++p) xyz[p] = u(0.0, extent);
  return NPCG_OK;
}

// synthetic.hpp:33-40 gen_features: uniform in [-1, 1), cast to the feature type
npcg_status npcg_gen_features(int64_t n, int64_t groups, int64_t channels, uint64_t seed,
                              npcg_dtype dtype, void* out) {
  if (n < 0 || groups < 1 || channels < 1) return NPCG_ERR_SHAPE;
  const int64_t count = n * groups * channels;
  if (count > 0 && !out) return NPCG_ERR_INVALID;
  Uniform u(seed);
  if (dtype == NPCG_F32)
    for (int64_t p = 0; p < count; ++p) static_cast<float*>(out)[p] = static_cast<float>(u(-1.0, 1.0));
  else
    for (int64_t p = 0; p < count; ++p) static_cast<double*>(out)[p] = u(-1.0, 1.0);
  return NPCG_OK;
}

// tensors.hpp:142-150 make_weights: uniform in [-s, s), s = (G * C_in)^(-1/2)
npcg_status npcg_make_weights(int64_t t, int64_t groups, int64_t c_in, int64_t c_out,
                              uint64_t seed, npcg_dtype dtype, void* out) {
  if (t < 1 || t % 2 == 0 || groups < 1 || c_in < 1 || c_out < 1) return NPCG_ERR_SHAPE;
  if (!out) return NPCG_ERR_INVALID;
  const int64_t count = t * t * t * groups * c_in * c_out;
  const double s = 1.0 / std::sqrt(static_cast<double>(groups * c_in));
  Uniform u(seed);
  if (dtype == NPCG_F32)
    for (int64_t p = 0; p < count; ++p) static_cast<float*>(out)[p] = static_cast<float>(u(-s, s));
  else
    for (int64_t p = 0; p < count; ++p) static_cast<double*>(out)[p] = u(-s, s);
  return NPCG_OK;
}

}  // extern "C"
