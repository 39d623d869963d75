/* Exactly rounded fused multiply-add over arrays for the extended CPU oracle
 * (TEST INFRASTRUCTURE ONLY): out[i] = fma(a[i], b[i], c[i]) with one
 * rounding, C99 fma() from libm (glibc: correctly rounded on every input).
 * NumPy has no fused multiply-add; the lead-tilt step of the extended model
 * is defined with three of them. */
#include <math.h>

void fma_arr(const double* a, const double* b, const double* c, double* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = fma(a[i], b[i], c[i]);
}
