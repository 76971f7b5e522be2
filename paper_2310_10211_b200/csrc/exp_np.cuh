// exp_np.cuh -- float64 exp bit-identical to the reference's np.exp.
//
// The reference evaluates `exponential` as np.exp (interpreter.py:106-108).
// numpy 2.3 on AVX-512 hosts dispatches float64 exp to Intel SVML
// `__svml_exp8_ha` (vendored in numpy).  This is that algorithm restated
// operation by operation (constants and the 16-entry 2^(j/16) table are the
// values SVML uses): round-toward-zero reduction x = (k + j/16) ln2 + r,
// degree-6 polynomial, T[j] * (1 + p(r)) + T_tail[j], vscalefpd by floor(k).
// Verified bit-exact against np.exp on 12M random inputs with |x| < 1021 ln2
// (tests/test_exp_model.py does the same check on the host model).  From
// |x| = 1021 ln2 (= 707.703..., located exactly by probing numpy) SVML takes
// a scalar "rare" path: exp_rare.h evaluates it in double-double, rounded
// once (subnormals included), which agrees with numpy except near rounding
// midpoints (match rates in tests/test_exp_model.py).
#pragma once
#include <stdint.h>
#define GEVO_HD __device__
#define GEVO_FMA __fma_rn
#include "exp_rare.h"
namespace gevo {

__device__ __constant__ uint64_t kExpTop[16] = {
    0x3ff0000000000000ULL, 0x3ff0b5586cf9890fULL,
    0x3ff172b83c7d517bULL, 0x3ff2387a6e756238ULL,
    0x3ff306fe0a31b715ULL, 0x3ff3dea64c123422ULL,
    0x3ff4bfdad5362a27ULL, 0x3ff5ab07dd485429ULL,
    0x3ff6a09e667f3bcdULL, 0x3ff7a11473eb0187ULL,
    0x3ff8ace5422aa0dbULL, 0x3ff9c49182a3f090ULL,
    0x3ffae89f995ad3adULL, 0x3ffc199bdd85529cULL,
    0x3ffd5818dcfba487ULL, 0x3ffea4afa2a490daULL};
__device__ __constant__ uint64_t kExpTail[16] = {
    0x0000000000000000ULL, 0x3c979aa65d837b6dULL,
    0xbc801b15eaa59348ULL, 0x3c968efde3a8a894ULL,
    0x3c834d754db0abb6ULL, 0x3c859f48a72a4c6dULL,
    0x3c7690cebb7aafb0ULL, 0x3c9063e1e21c5409ULL,
    0xbc93b3efbf5e2228ULL, 0xbc7b32dcb94da51dULL,
    0x3c8db72fc1f0eab4ULL, 0x3c71affc2b91ce27ULL,
    0x3c8c1a7792cb3387ULL, 0x3c736eae30af0cb3ULL,
    0x3c74a385a63d07a7ULL, 0xbc8ff7128fd391f0ULL};

__device__ __forceinline__ double u2d(uint64_t u) { return __longlong_as_double((long long)u); }

// a * 2^floor(kd) with a single rounding (vscalefpd)
__device__ __forceinline__ double scalef_floor(double a, double kd) {
  const int e = (int)floor(kd);
  if (e >= -1022 && e <= 1023) return __dmul_rn(a, u2d((uint64_t)(e + 1023) << 52));
  if (e < -1022) {
    const double t = __dmul_rn(a, u2d((uint64_t)(e + 200 + 1023) << 52));
    return __dmul_rn(t, u2d((uint64_t)(1023 - 200) << 52));
  }
  const double t = __dmul_rn(a, u2d((uint64_t)(e - 200 + 1023) << 52));
  return __dmul_rn(t, u2d((uint64_t)(200 + 1023) << 52));
}

__device__ __forceinline__ double exp_np(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return __longlong_as_double(0x7ff0000000000000LL);
  if (x < -745.1332191019412) return 0.0;
  if (fabs(x) >= 0x1.61da04cbafe44p+9) return gevo_exp_rare(x);   // |x| >= 1021 ln2
  const double t = __fma_rz(x, u2d(0x3ff71547652b82feULL), u2d(0x42f8000000003ff0ULL));
  const double kd = __dsub_rn(t, u2d(0x42f8000000003ff0ULL));
  const int j = (int)(__double_as_longlong(t) & 15);
  double r = fma(-kd, u2d(0x3fe62e42fefa39efULL), x);
  r = fma(-u2d(0x3c7abc9e3b39803fULL), kd, r);
  r = __longlong_as_double(__double_as_longlong(r) & (long long)0xbfffffffffffffffULL);
  const double r2 = __dmul_rn(r, r);
  double p = fma(u2d(0x3f57411836940c04ULL), r, u2d(0x3f81101cbbc265c0ULL));
  const double q = fma(u2d(0x3fa55557242d68feULL), r, u2d(0x3fc5555553939732ULL));
  const double s = fma(u2d(0x3fe000000000d008ULL), r, u2d(0x3fefffffffffff70ULL));
  p = fma(r2, p, q);
  p = fma(r2, p, s);
  const double top = u2d(kExpTop[j]);
  const double u = fma(p, r, u2d(kExpTail[j]));
  return scalef_floor(fma(top, u, top), kd);
}

}  // namespace gevo
