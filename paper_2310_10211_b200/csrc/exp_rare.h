/* exp_rare.h -- np.exp's rare range (|x| >= 707.7: results near overflow and
 * subnormal results), shared verbatim by the device (exp_np.cuh) and the
 * host model that checks it against numpy (tests/tools/exp_model.py).
 *
 * numpy 2.3's AVX-512 exp (SVML __svml_exp8_ha) leaves its vector path for
 * these inputs and evaluates them with a scalar routine accurate to about
 * 2^-8 ulp (measured: every mismatch against the correctly rounded value is
 * within 0.003 ulp of a rounding midpoint).  This is a double-double
 * evaluation rounded once, subnormals included: it agrees with numpy except
 * on those near-midpoint inputs (2 of 4 000 random rare-range inputs here,
 * tests/test_exp_model.py).  The vector-path restatement (exp_np.cuh) is
 * bit-exact elsewhere; before this, the rare range used it too and rounded
 * subnormal results twice (3 of the 16 full-size CNN mutants saw a 1-ulp
 * subnormal softmax probability).
 *
 * Plain C: only +, -, * and fma, each rounded to nearest (compile without
 * FMA contraction: nvcc -fmad=false, gcc -ffp-contract=off). */
#ifndef GEVO_EXP_RARE_H
#define GEVO_EXP_RARE_H
#ifndef GEVO_HD
#define GEVO_HD
#endif
#ifndef GEVO_FMA
#define GEVO_FMA fma
#endif

typedef struct { double h, l; } gevo_dd;

GEVO_HD static inline gevo_dd gevo_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  gevo_dd r = {s, (a - (s - bb)) + (b - bb)};
  return r;
}
GEVO_HD static inline gevo_dd gevo_dd_add(gevo_dd a, gevo_dd b) {
  gevo_dd s = gevo_two_sum(a.h, b.h);
  s.l = s.l + (a.l + b.l);
  return gevo_two_sum(s.h, s.l);
}
GEVO_HD static inline gevo_dd gevo_dd_mul(gevo_dd a, gevo_dd b) {
  const double p = a.h * b.h;
  double e = GEVO_FMA(a.h, b.h, -p);
  e = e + (a.h * b.l + a.l * b.h);
  return gevo_two_sum(p, e);
}

/* x in [-745.1332191019412, 709.782712893384], |x| >= 707.7 */
GEVO_HD static inline double gevo_exp_rare(double x) {
  /* 1/k!, k = 0..14, as double-doubles */
  const double fh[15] = {0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
                         0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
                         0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
                         0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33,
                         0x1.93974a8c07c9dp-37};
  const double fl[15] = {0.0, 0.0, 0.0, 0x1.5555555555555p-57, 0x1.5555555555555p-59,
                         0x1.1111111111111p-63, -0x1.f49f49f49f49fp-65, 0x1.a01a01a01a01ap-73,
                         0x1.a01a01a01a01ap-76, -0x1.c154f8ddc6c00p-73, 0x1.cbbc05b4fa99ap-76,
                         -0x1.c062e06d1f209p-80, -0x1.2aec959e14c06p-83, 0x1.f28e0cc748ebep-87,
                         0x1.05d6f8a2efd1fp-92};
  /* 2^(j/16), j = 0..15, as double-doubles */
  const double th[16] = {0x1p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
                         0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0,
                         0x1.5ab07dd485429p+0, 0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0,
                         0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0, 0x1.ae89f995ad3adp+0,
                         0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};
  const double tl[16] = {0.0, 0x1.8a62e4adc610bp-54, -0x1.19041b9d78a76p-55, 0x1.9b07eb6c70573p-54,
                         0x1.6f46ad23182e4p-55, 0x1.ada0911f09ebcp-55, 0x1.d4397afec42e2p-56,
                         0x1.6324c054647adp-54, -0x1.bdd3413b26456p-54, -0x1.41577ee04992fp-55,
                         0x1.6e9f156864b27p-54, 0x1.c7c46b071f2bep-56, 0x1.7a1cd345dcc81p-54,
                         0x1.11065895048ddp-55, 0x1.2ed02d75b3707p-55, -0x1.e9c23179c2893p-54};
  /* ln2/16 in three pieces: 38 + 38 + 53 bits */
  const double c1 = 0x1.62e42fefa0000p-5, c2 = 0x1.cf79abc9e0000p-44, c3 = 0x1.d9cc01f97b57ap-83;
  /* N = nearest(x * 16 / ln2): |N| < 2^14, so N*c1 and N*c2 are exact */
  const double big = 0x1.8p52;
  const double nd = (x * 0x1.71547652b82fep+4 + big) - big;
  const long long n = (long long)nd;
  const int j = (int)(n & 15);
  const long long m = (n - j) / 16;           /* floor(N / 16) */
  const double t1 = x - nd * c1;               /* exact (Sterbenz) */
  gevo_dd r = gevo_two_sum(t1, -(nd * c2));
  gevo_dd p3 = {-(nd * c3), 0.0};
  r = gevo_dd_add(r, p3);
  /* exp(r), |r| <= ln2/32: Taylor to degree 14 in double-double (Horner) */
  gevo_dd s = {fh[14], fl[14]};
  for (int k = 13; k >= 0; --k) {
    gevo_dd c = {fh[k], fl[k]};
    s = gevo_dd_add(gevo_dd_mul(s, r), c);
  }
  gevo_dd t = {th[j], tl[j]};
  s = gevo_dd_mul(s, t);                       /* 2^(j/16) exp(r), in [0.98, 1.95] */
  /* s.h is s rounded once; scale by 2^m */
  const long long e = m;
  if (e >= -1021) {                            /* normal result: exact scaling */
    double y = s.h;
    long long k = e;
    while (k > 1000) { y = y * 0x1p1000; k -= 1000; }
    union { unsigned long long u; double d; } sc;
    sc.u = (unsigned long long)(k + 1023) << 52;
    return y * sc.d;
  }
  /* subnormal (or smallest normal) result: round s * 2^e to a multiple of
     2^-1074 once.  H, L = s * 2^(e + 1074) (exact: normal range). */
  union { unsigned long long u; double d; } sc;
  sc.u = (unsigned long long)(e + 1074 + 1023) << 52;
  const double H = s.h * sc.d, L = s.l * sc.d;
  const double Hi = (H + big) - big;           /* nearest integer, ties even */
  const double g = (H - Hi) + L;               /* H - Hi exact */
  double q = Hi;
  if (g > 0.5) q = Hi + 1.0;
  else if (g < -0.5) q = Hi - 1.0;
  else if (g == 0.5 || g == -0.5) {            /* a tie of the double-double */
    const double up = g > 0 ? Hi + 1.0 : Hi - 1.0;
    const double half = up * 0.5;
    q = (half == (half + big) - big) ? up : Hi;
  }
  return q * 0x1p-1074;
}

#endif
