/* Minimal FFTW3 API stand-in (double precision, complex 2-D only).
 *
 * TEST INFRASTRUCTURE (oracle/): lets the unmodified reference source
 * proj/src/fft.cpp compile in this image, which has no FFTW.  Covers exactly
 * the calls the reference makes (fft.cpp:3,23-25,35,39).  The transform is
 * oracle/fft64.c; semantics follow FFTW's documented contract: sign
 * FFTW_FORWARD = -1 (exp(-2 pi i jk/n)), unnormalised both ways, n0 = rows
 * (slowest), n1 = columns (fastest), out-of-place allowed.
 */
#ifndef HOLO_SHIM_FFTW3_H
#define HOLO_SHIM_FFTW3_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct holo_shim_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
