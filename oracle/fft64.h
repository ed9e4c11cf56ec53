/* fft64 — double-precision mixed-radix Stockham FFT.
 *
 * TEST INFRASTRUCTURE (oracle/). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may use anything here.
 *
 * Stands in for FFTW3 (double, c2c), which the reference calls from
 * proj/src/fft.cpp:23-25,35,39 and which is absent from this image.  The
 * convention is FFTW's: sign -1 = forward exp(-2 pi i jk/n), sign +1 =
 * backward, both unnormalised; the 2-D transform is row-major [h][w] with w
 * fastest, matching fftw_plan_dft_2d(h, w, ...) at fft.cpp:23.
 *
 * Execution is single-threaded and reentrant: a plan is read-only after
 * creation, scratch is per call, so concurrent execution on distinct arrays
 * is safe (the reference parallelises over channels, propagation.cpp:98).
 */
#ifndef HOLO_ORACLE_FFT64_H
#define HOLO_ORACLE_FFT64_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fft64_plan fft64_plan;

fft64_plan* fft64_plan_new(int n);
void fft64_plan_free(fft64_plan* p);
int fft64_plan_size(const fft64_plan* p);

/* In-place 1-D transform of n interleaved complex doubles; work holds n
 * complex doubles of scratch. */
void fft64_exec(const fft64_plan* p, double* x, double* work, int sign);

/* In-place 2-D transform of a row-major h x w array (w fastest). */
void fft64_exec_2d(const fft64_plan* pw, const fft64_plan* ph, double* data, int w, int h, int sign);

#ifdef __cplusplus
}
#endif

#endif
