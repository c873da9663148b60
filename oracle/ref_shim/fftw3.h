/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — NOT FFTW.
 *
 * The four FFTW3 entry points integrate.cpp uses (integrate.cpp:31-34,44,63,
 * 66-67), so the reference source compiles unmodified here (FFTW3 is absent,
 * SURVEY §8(c)).  Semantics are FFTW's for rank-3 r2c/c2r of double data
 * (FFTW 3.3 manual, "Multi-Dimensional DFTs of Real Data" and "What FFTW
 * Really Computes"):
 *   r2c_3d(n0,n1,n2): out[i0][i1][k2], k2 <= n2/2, = sum in * e^{-2 pi i (.)},
 *                     unnormalised, row-major with n2 contiguous;
 *   c2r_3d(n0,n1,n2): the inverse (e^{+}), unnormalised, of a half spectrum
 *                     that FFTW assumes Hermitian — its rdft2 solver for rank
 *                     >= 2 runs the complex transforms along n0, n1 first and
 *                     the c2r along n2 last, which reads only Re() of bins
 *                     k2 = 0 and n2/2 (halfcomplex storage has no slot for
 *                     their imaginary parts); the input is destroyed.
 * The transform itself is the oracle's fp64 FFT (orc::rfft3 / orc::irfft3 in
 * oracle_core.cpp), which tests/test_oracle_field.py pins to numpy's pocketfft
 * rfftn/irfftn to 1e-12 on non-Hermitian input.  Planning flags are ignored
 * (FFTW_ESTIMATE changes speed, not the transform). */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct vc_fftw_plan_s* fftw_plan;

#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
