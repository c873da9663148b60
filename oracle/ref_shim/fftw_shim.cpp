// SPDX-License-Identifier: Apache-2.0
// TEST INFRASTRUCTURE — the FFTW3 API subset of fftw3.h over the oracle's fp64
// rank-3 transforms (see fftw3.h for the semantics).
#include "fftw3.h"

#include <complex>

#include "../oracle.hpp"

struct vc_fftw_plan_s {
  bool r2c;
  int n0, n1, n2;
  double* real;
  fftw_complex* cplx;
};

extern "C" {

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out, unsigned) {
  return new vc_fftw_plan_s{true, n0, n1, n2, in, out};
}

fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out, unsigned) {
  return new vc_fftw_plan_s{false, n0, n1, n2, out, in};
}

void fftw_execute(const fftw_plan p) {
  auto* S = reinterpret_cast<std::complex<double>*>(p->cplx);  // fftw_complex is layout-compatible
  if (p->r2c)
    orc::rfft3(p->real, S, p->n2, p->n1, p->n0);
  else
    orc::irfft3(S, p->real, p->n2, p->n1, p->n0);
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
