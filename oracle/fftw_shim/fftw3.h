/* oracle/fftw_shim/fftw3.h — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * A CPU stand-in for the subset of the FFTW3 API the reference calls, so the reference
 * sources under /root/reference/proj/src compile unmodified for the parity oracle.
 * libfftw3 (unpinned in the reference: proj/src/CMakeLists.txt:1-3) is not installed in
 * this image. Call sites this header satisfies: proj/src/fft.cpp:24,26,27 (double) and
 * :36,38,39 (float); flags FFTW_FORWARD / FFTW_BACKWARD / FFTW_ESTIMATE at :55-60.
 *
 * Semantics (FFTW3 published contract): fftw_plan_dft_3d(n0,n1,n2,...) plans an
 * unnormalised complex 3-D DFT of a row-major n0 x n1 x n2 array (n2 fastest), sign -1
 * (forward, exp(-2 pi i k n / N)) or +1 (backward). execute_dft may be called on any
 * other array of the same size (in == out supported, which is the only mode used).
 */
#ifndef MMB_ORACLE_FFTW3_SHIM_H
#define MMB_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

typedef double fftw_complex[2];
typedef float fftwf_complex[2];

typedef struct mmb_shim_plan_d* fftw_plan;
typedef struct mmb_shim_plan_f* fftwf_plan;

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

fftwf_plan fftwf_plan_dft_3d(int n0, int n1, int n2, fftwf_complex* in, fftwf_complex* out,
                             int sign, unsigned flags);
void fftwf_execute_dft(const fftwf_plan p, fftwf_complex* in, fftwf_complex* out);
void fftwf_destroy_plan(fftwf_plan p);

#ifdef __cplusplus
}
#endif

#endif
