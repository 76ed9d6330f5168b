// Host build of csrc/psd_small.h for tests/test_psd_small.py (CPU only).
#include "../../paper_2509_00406_b200/csrc/psd_small.h"
extern "C" {
void host_project3(double* a, long n, double f) {
  for (long i = 0; i < n; ++i) mg::psd_small::project3(a + 6 * i, f);
}
void host_project2(double* a, long n, double f) {
  for (long i = 0; i < n; ++i) mg::psd_small::project2(a + 3 * i, f);
}
}
