// Host build of csrc/msurf_trig.cuh for CPU accuracy tests (tests/test_trig.py).
// Compiled by __graft_entry__.build() with -ffp-contract=off.
#include <stddef.h>
#include "../../paper_2603_28160_b200/csrc/msurf_trig.cuh"

void msurf_host_sincos_array(const double* x, double* s, double* c, size_t n) {
  for (size_t i = 0; i < n; ++i) msurf_sincos(x[i], &s[i], &c[i]);
}
