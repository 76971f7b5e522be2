// exec_core.cuh -- per-instruction semantics of the device executor.
//
// Each function mirrors one closure of the reference interpreter
// (pkg/src/evotir/interpreter.py:78-185) on 64-bit element words, and keeps
// numpy's floating-point evaluation order where the reference's result
// depends on it (summation order of reduce and dot, NaN propagation of
// maximum, x86 float->int64 conversion).  Compiled with -fmad=false: every
// fused multiply-add below is an explicit fma().
#pragma once
#include <stdint.h>
#include <math.h>
#include "gevo_plan.h"

namespace gevo {

// operand addressing modes chosen per instruction (aux2 of EW ops)
enum { AM_STRIDED = 0, AM_LINEAR = 1, AM_SCALAR = 2 };

__device__ __forceinline__ int64_t as_i64(double w) { return __double_as_longlong(w); }
__device__ __forceinline__ double as_w(int64_t v) { return __longlong_as_double(v); }

// C-order unravel of a linear output index over `rank` dims.
__device__ __forceinline__ void unravel(int i, int rank, const int32_t* shp, int* idx) {
#pragma unroll
  for (int d = GEVO_MAXR - 1; d >= 0; --d) {
    if (d < rank) {
      int e = shp[d];
      idx[d] = i % e;
      i /= e;
    } else {
      idx[d] = 0;
    }
  }
}

__device__ __forceinline__ int64_t addr(const gevo_operand& o, const int* idx, int rank) {
  int64_t a = o.off;
#pragma unroll
  for (int d = 0; d < GEVO_MAXR; ++d)
    if (d < rank) a += (int64_t)idx[d] * o.st[d];
  return a;
}

// numpy float64 maximum: NaN propagates, otherwise the first of equal values
// np.maximum on x86 (MAXPD): a when a > b or a is NaN, else b -- so the
// second operand on ties, which decides signed zeros: maximum(-0.0, 0.0) is
// 0.0 and maximum(0.0, -0.0) is -0.0 (tests/golden/edge_cases.json.gz,
// recorded from the reference).  np.max's running reduction keeps the same
// rule (the later element wins a tie: probed on numpy 2.3.5).
__device__ __forceinline__ double np_fmax(double a, double b) {
  return (a > b || a != a) ? a : b;
}

// numpy trunc(x).astype(int64) on x86: NaN/inf/out of range -> INT64_MIN
__device__ __forceinline__ int64_t x86_f2i(double x) {
  double t = trunc(x);
  if (!(t >= -9223372036854775808.0 && t < 9223372036854775808.0))
    return (int64_t)0x8000000000000000ULL;
  return (int64_t)t;
}

// reference _int_divide (interpreter.py:65-69): trunc(float(a)/float(b)), x/0 = 0
__device__ __forceinline__ int64_t np_idiv(int64_t a, int64_t b) {
  if (b == 0) return 0;
  double q = __ddiv_rn((double)a, (double)b);
  return x86_f2i(q);
}

__device__ __forceinline__ double exp_np(double x);   // exp_np.cuh

__device__ __forceinline__ double unary_f(int sub, double x) {
  switch (sub) {
    case GEVO_U_NEG: return -x;
    case GEVO_U_EXP: return exp_np(x);
    case GEVO_U_LOG: return log(x);
    default: return x;
  }
}

__device__ __forceinline__ double apply_unary(int sub, int kin, int kout, double w) {
  if (sub == GEVO_U_COPY) return w;
  if (sub == GEVO_U_CVT) {
    if (kout == GEVO_K_I1) {
      bool nz = (kin == GEVO_K_F64) ? (w != 0.0) : (as_i64(w) != 0);
      return as_w(nz ? 1 : 0);
    }
    if (kout == GEVO_K_I64) {
      if (kin == GEVO_K_F64) return as_w(x86_f2i(w));
      return w;  // i64 / i1 already integers
    }
    // -> f64
    if (kin == GEVO_K_F64) return w;
    return __ll2double_rn(as_i64(w));
  }
  if (kin == GEVO_K_F64) return unary_f(sub, w);
  // integer negate (wraps)
  return as_w((int64_t)(0ULL - (uint64_t)as_i64(w)));
}

__device__ __forceinline__ double apply_binary(int sub, int kin, double wa, double wb) {
  if (kin == GEVO_K_F64) {
    double a = wa, b = wb;
    switch (sub) {
      case GEVO_B_ADD: return __dadd_rn(a, b);
      case GEVO_B_SUB: return __dsub_rn(a, b);
      case GEVO_B_MUL: return __dmul_rn(a, b);
      case GEVO_B_DIV: return __ddiv_rn(a, b);
      case GEVO_B_MAX: return np_fmax(a, b);
      case GEVO_B_EQ: return as_w(a == b);
      case GEVO_B_NE: return as_w(a != b);
      case GEVO_B_LT: return as_w(a < b);
      case GEVO_B_LE: return as_w(a <= b);
      case GEVO_B_GT: return as_w(a > b);
      case GEVO_B_GE: return as_w(a >= b);
    }
    return 0.0;
  }
  int64_t a = as_i64(wa), b = as_i64(wb);
  switch (sub) {
    case GEVO_B_ADD: return as_w((int64_t)((uint64_t)a + (uint64_t)b));
    case GEVO_B_SUB: return as_w((int64_t)((uint64_t)a - (uint64_t)b));
    case GEVO_B_MUL: return as_w((int64_t)((uint64_t)a * (uint64_t)b));
    case GEVO_B_DIV: return as_w(np_idiv(a, b));
    case GEVO_B_MAX: return as_w(a >= b ? a : b);
    case GEVO_B_EQ: return as_w(a == b);
    case GEVO_B_NE: return as_w(a != b);
    case GEVO_B_LT: return as_w(a < b);
    case GEVO_B_LE: return as_w(a <= b);
    case GEVO_B_GT: return as_w(a > b);
    case GEVO_B_GE: return as_w(a >= b);
  }
  return 0.0;
}

// numpy DOUBLE_pairwise_sum (n elements at stride s): sequential below 8,
// 8 interleaved partial sums up to 128 with a fixed tree, recursive halving
// (split at a multiple of 8) above.
__device__ double pairwise_sum(const double* a, int n, int64_t s) {
  // explicit stack: at most log2(n/128)+1 levels for n < 2^31
  struct Frame { int64_t base; int n; int state; double left; };
  Frame st[24];
  int top = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.n <= 128) {
      double r;
      if (f.n < 8) {
        r = 0.0;
        for (int i = 0; i < f.n; ++i) r = __dadd_rn(r, a[(f.base + i) * s]);
      } else {
        double p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = a[(f.base + j) * s];
        int i = 8;
        int lim = f.n - (f.n % 8);
        for (; i < lim; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) p[j] = __dadd_rn(p[j], a[(f.base + i + j) * s]);
        }
        r = __dadd_rn(__dadd_rn(__dadd_rn(p[0], p[1]), __dadd_rn(p[2], p[3])),
                      __dadd_rn(__dadd_rn(p[4], p[5]), __dadd_rn(p[6], p[7])));
        for (; i < f.n; ++i) r = __dadd_rn(r, a[(f.base + i) * s]);
      }
      ret = r;
      --top;
      // deliver to parent
      while (top >= 0) {
        Frame& p = st[top];
        if (p.state == 1) {           // left done, run right
          p.left = ret;
          p.state = 2;
          int n2 = p.n / 2;
          n2 -= n2 % 8;
          st[++top] = {p.base + n2, p.n - n2, 0, 0.0};
          break;
        } else {                       // right done
          ret = __dadd_rn(p.left, ret);
          --top;
        }
      }
      continue;
    }
    // split
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    f.state = 1;
    st[++top] = {f.base, n2, 0, 0.0};
  }
  return ret;
}

}  // namespace gevo
