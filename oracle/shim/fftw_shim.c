/* FFTW3 stand-in implementation over oracle/fft64.c (see fftw3.h).
 * TEST INFRASTRUCTURE (oracle/). */
#include "fftw3.h"

#include <stdlib.h>
#include <string.h>

#include "../fft64.h"

struct holo_shim_fftw_plan_s {
    int n0, n1, sign;
    fft64_plan* rows;  /* length n1 transforms */
    fft64_plan* cols;  /* length n0 transforms */
    fftw_complex* in;
    fftw_complex* out;
};

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
    (void)flags;
    if (n0 < 1 || n1 < 1 || (sign != FFTW_FORWARD && sign != FFTW_BACKWARD)) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    if (!p) return NULL;
    p->n0 = n0;
    p->n1 = n1;
    p->sign = sign;
    p->rows = fft64_plan_new(n1);
    p->cols = fft64_plan_new(n0);
    p->in = in;
    p->out = out;
    if (!p->rows || !p->cols) {
        fftw_destroy_plan(p);
        return NULL;
    }
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const size_t n = (size_t)p->n0 * (size_t)p->n1;
    if (in != out) memcpy(out, in, sizeof(fftw_complex) * n);
    fft64_exec_2d(p->rows, p->cols, (double*)out, p->n1, p->n0, p->sign);
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    fft64_plan_free(p->rows);
    fft64_plan_free(p->cols);
    free(p);
}
