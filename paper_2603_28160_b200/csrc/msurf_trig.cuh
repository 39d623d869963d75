// Near-correctly-rounded fp64 sin/cos for the per-(time step, tooth) angle.
//
// The reference takes cos/sin of the tooth angle from glibc through NumPy
// (engine.py:252-255, kinematics.py:64-77). glibc's double sin/cos are not
// correctly rounded (max error ~0.51 ulp; measured here: 0.3 % of arguments in
// [-3000, 10] differ from the correctly rounded value by one ulp), and CUDA's
// built-in sin/cos carry up to 2 ulp. This routine evaluates both in
// double-double arithmetic and rounds once at the end, so its result is the
// correctly rounded value except with probability ~1e-7; any disagreement with
// glibc is then glibc's own rounding, a 1-ulp difference in c/s that moves
// workpiece coordinates by ~1e-15 mm.
//
// Algorithm (own restatement of textbook techniques):
//   1. k = rint(x * 2/pi); r = x - k*pi/2 in double-double with pi/2 split in
//      three doubles; k*P1 is formed exactly with an FMA two-product and the
//      leading subtraction is exact (Sterbenz).
//   2. r = j/128 + b with |b| <= 1/256; sin/cos(j/128) come from a
//      double-double table (tools/gen_trig_table.py, mpmath at 300 bits);
//      sin(b), cos(b) are short Taylor series, the O(1) terms in double-double.
//   3. angle-addition in double-double, quadrant swap, single final rounding.
//
// Host and device compile the same code: on the device every op is an explicit
// _rn intrinsic (never contracted); the host test build uses -ffp-contract=off
// and libm fma().
#pragma once

#if defined(__CUDACC__)
#define MSURF_HD __host__ __device__ __forceinline__
#else
#define MSURF_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define MSURF_TRIG_TABLE_QUAL static __device__ const
#define MS_FMA(a, b, c) __fma_rn((a), (b), (c))
#define MS_MUL(a, b) __dmul_rn((a), (b))
#define MS_ADD(a, b) __dadd_rn((a), (b))
#define MS_SUB(a, b) __dsub_rn((a), (b))
#define MS_RINT(a) rint(a)
#else
#include <math.h>
#define MSURF_TRIG_TABLE_QUAL static const
#define MS_FMA(a, b, c) fma((a), (b), (c))
#define MS_MUL(a, b) ((a) * (b))
#define MS_ADD(a, b) ((a) + (b))
#define MS_SUB(a, b) ((a) - (b))
#define MS_RINT(a) rint(a)
#endif

#include "msurf_trig_table.h"

typedef struct {
  double hi, lo;
} msurf_dd;

MSURF_HD msurf_dd ms_two_sum(double a, double b) {
  double s = MS_ADD(a, b);
  double bb = MS_SUB(s, a);
  double e = MS_ADD(MS_SUB(a, MS_SUB(s, bb)), MS_SUB(b, bb));
  msurf_dd r = {s, e};
  return r;
}

MSURF_HD msurf_dd ms_fast_two_sum(double a, double b) {
  double s = MS_ADD(a, b);
  double e = MS_SUB(b, MS_SUB(s, a));
  msurf_dd r = {s, e};
  return r;
}

MSURF_HD msurf_dd ms_two_prod(double a, double b) {
  double p = MS_MUL(a, b);
  double e = MS_FMA(a, b, -p);
  msurf_dd r = {p, e};
  return r;
}

MSURF_HD msurf_dd ms_dd_add(msurf_dd a, msurf_dd b) {
  msurf_dd s = ms_two_sum(a.hi, b.hi);
  msurf_dd t = ms_two_sum(a.lo, b.lo);
  s.lo = MS_ADD(s.lo, t.hi);
  s = ms_fast_two_sum(s.hi, s.lo);
  s.lo = MS_ADD(s.lo, t.lo);
  return ms_fast_two_sum(s.hi, s.lo);
}

MSURF_HD msurf_dd ms_dd_add_d(msurf_dd a, double b) {
  msurf_dd s = ms_two_sum(a.hi, b);
  s.lo = MS_ADD(s.lo, a.lo);
  return ms_fast_two_sum(s.hi, s.lo);
}

MSURF_HD msurf_dd ms_dd_mul(msurf_dd a, msurf_dd b) {
  msurf_dd p = ms_two_prod(a.hi, b.hi);
  double c = MS_ADD(MS_MUL(a.hi, b.lo), MS_MUL(a.lo, b.hi));
  p.lo = MS_ADD(p.lo, c);
  return ms_fast_two_sum(p.hi, p.lo);
}

MSURF_HD msurf_dd ms_dd_neg(msurf_dd a) {
  msurf_dd r = {-a.hi, -a.lo};
  return r;
}

// sin(x) and cos(x) for finite |x| < 2^40.
MSURF_HD void msurf_sincos(double x, double* s_out, double* c_out) {
  const double kd = MS_RINT(MS_MUL(x, MSURF_TWO_OVER_PI));
  // r = x - kd*(P1 + P2 + P3)
  const double p = MS_MUL(kd, MSURF_PIO2_1);
  const double pe = MS_FMA(kd, MSURF_PIO2_1, -p);
  const double s0 = MS_SUB(x, p);  // exact (Sterbenz) for kd != 0; exact for kd == 0
  msurf_dd r = ms_two_sum(s0, -pe);
  msurf_dd q2 = ms_two_prod(kd, MSURF_PIO2_2);
  r = ms_dd_add(r, ms_dd_neg(q2));
  r = ms_dd_add_d(r, -MS_MUL(kd, MSURF_PIO2_3));

  // r = a + b, a = j/128
  const double jd = MS_RINT(MS_MUL(r.hi, 128.0));
  const double bh = MS_SUB(r.hi, MS_MUL(jd, 0.0078125));  // exact
  const msurf_dd b = ms_two_sum(bh, r.lo);
  const double b2 = MS_MUL(b.hi, b.hi);

  // sin(b) = b + b^3 * (-1/6 + b^2/120 - b^4/5040 + b^6/362880)
  double ps = MS_ADD(-1.0 / 5040.0, MS_MUL(b2, 1.0 / 362880.0));
  ps = MS_ADD(1.0 / 120.0, MS_MUL(b2, ps));
  ps = MS_ADD(-1.0 / 6.0, MS_MUL(b2, ps));
  ps = MS_MUL(MS_MUL(b.hi, b2), ps);
  const msurf_dd sb = ms_dd_add_d(b, ps);

  // cos(b) = 1 - b^2/2 + b^4 * (1/24 - b^2/720 + b^4/40320)
  msurf_dd bb = ms_two_prod(b.hi, b.hi);
  bb.lo = MS_ADD(bb.lo, MS_MUL(MS_MUL(2.0, b.hi), b.lo));
  double pc = MS_ADD(-1.0 / 720.0, MS_MUL(b2, 1.0 / 40320.0));
  pc = MS_ADD(1.0 / 24.0, MS_MUL(b2, pc));
  pc = MS_MUL(MS_MUL(b2, b2), pc);
  msurf_dd cb = ms_two_sum(1.0, MS_MUL(-0.5, bb.hi));
  cb.lo = MS_ADD(cb.lo, MS_MUL(-0.5, bb.lo));
  cb = ms_fast_two_sum(cb.hi, cb.lo);
  cb = ms_dd_add_d(cb, pc);

  const int ji = (int)jd;
  const int ja = ji < 0 ? -ji : ji;
  msurf_dd sa = {msurf_trig_tab[4 * ja + 0], msurf_trig_tab[4 * ja + 1]};
  const msurf_dd ca = {msurf_trig_tab[4 * ja + 2], msurf_trig_tab[4 * ja + 3]};
  if (ji < 0) sa = ms_dd_neg(sa);

  // sin(a+b) = sa*cb + ca*sb ; cos(a+b) = ca*cb - sa*sb
  const msurf_dd sr = ms_dd_add(ms_dd_mul(sa, cb), ms_dd_mul(ca, sb));
  const msurf_dd cr = ms_dd_add(ms_dd_mul(ca, cb), ms_dd_neg(ms_dd_mul(sa, sb)));

  const long long quad = ((long long)kd) & 3;
  double sv, cv;
  if (quad == 0) {
    sv = sr.hi; cv = cr.hi;
  } else if (quad == 1) {
    sv = cr.hi; cv = -sr.hi;
  } else if (quad == 2) {
    sv = -sr.hi; cv = -cr.hi;
  } else {
    sv = -cr.hi; cv = sr.hi;
  }
  *s_out = sv;
  *c_out = cv;
}

MSURF_HD double msurf_sin(double x) {
  double s, c;
  msurf_sincos(x, &s, &c);
  return s;
}
