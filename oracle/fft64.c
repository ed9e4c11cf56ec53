/* fft64 — double-precision mixed-radix Stockham FFT (see fft64.h).
 *
 * TEST INFRASTRUCTURE (oracle/): the FFT behind both the FFTW3 stand-in used
 * to compile the reference (oracle/shim/fftw3.h) and the C restatement of the
 * hot path (oracle/holo_oracle.c).  Algorithm: self-sorting Stockham
 * decimation-in-time, radices 4, 2, 3, 5 plus a direct DFT for any other
 * prime factor, so every n >= 1 is supported (FFTW semantics, fft.cpp:23).
 */
#include "fft64.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FFT64_MAX_STAGES 64

struct fft64_plan {
    int n;
    int nstages;
    int radix[FFT64_MAX_STAGES];
    int ns[FFT64_MAX_STAGES];      /* product of the radices before this stage */
    double* tw[FFT64_MAX_STAGES];  /* forward twiddles, [k][r-1] complex, k < ns */
};

static void factorize(int n, int* radix, int* count) {
    int c = 0;
    while (n % 4 == 0) { radix[c++] = 4; n /= 4; }
    while (n % 2 == 0) { radix[c++] = 2; n /= 2; }
    while (n % 3 == 0) { radix[c++] = 3; n /= 3; }
    while (n % 5 == 0) { radix[c++] = 5; n /= 5; }
    for (int p = 7; n > 1; p += 2) {
        while (n % p == 0) { radix[c++] = p; n /= p; }
        if ((long long)p * p > n && n > 1) { radix[c++] = n; n = 1; }
    }
    *count = c;
}

fft64_plan* fft64_plan_new(int n) {
    if (n < 1) return NULL;
    fft64_plan* p = (fft64_plan*)calloc(1, sizeof(fft64_plan));
    if (!p) return NULL;
    p->n = n;
    factorize(n, p->radix, &p->nstages);
    const double two_pi = 6.283185307179586476925286766559;
    int ns = 1;
    for (int s = 0; s < p->nstages; ++s) {
        const int r = p->radix[s];
        p->ns[s] = ns;
        const int span = ns * r;
        p->tw[s] = (double*)malloc(sizeof(double) * 2 * (size_t)ns * (size_t)(r > 1 ? r - 1 : 1));
        for (int k = 0; k < ns; ++k) {
            for (int q = 1; q < r; ++q) {
                const long long e = ((long long)q * k) % span;
                const double ang = -two_pi * (double)e / (double)span;
                p->tw[s][2 * ((size_t)k * (r - 1) + (q - 1))] = cos(ang);
                p->tw[s][2 * ((size_t)k * (r - 1) + (q - 1)) + 1] = sin(ang);
            }
        }
        ns *= r;
    }
    return p;
}

void fft64_plan_free(fft64_plan* p) {
    if (!p) return;
    for (int s = 0; s < p->nstages; ++s) free(p->tw[s]);
    free(p);
}

int fft64_plan_size(const fft64_plan* p) { return p ? p->n : 0; }

/* One Stockham pass: x (n complex) -> y (n complex). */
static void stage(const double* x, double* y, int n, int r, int ns, const double* tw, int sign) {
    const int m = n / r;
    const int groups = m / ns;
    const double sg = (double)sign; /* -1 forward, +1 backward */
    double vr[64], vi[64];
    double* ar = vr;
    double* ai = vi;
    if (r > 64) {
        ar = (double*)malloc(sizeof(double) * (size_t)r);
        ai = (double*)malloc(sizeof(double) * (size_t)r);
    }
    for (int g = 0; g < groups; ++g) {
        for (int k = 0; k < ns; ++k) {
            const int j = g * ns + k;
            const double* w = tw + 2 * (size_t)k * (r - 1);
            ar[0] = x[2 * (size_t)j];
            ai[0] = x[2 * (size_t)j + 1];
            for (int q = 1; q < r; ++q) {
                const double xr = x[2 * ((size_t)j + (size_t)q * m)];
                const double xi = x[2 * ((size_t)j + (size_t)q * m) + 1];
                /* the table holds the forward twiddle exp(-i a); backward uses its conjugate */
                const double cr = w[2 * (q - 1)];
                const double ci = (sign < 0) ? w[2 * (q - 1) + 1] : -w[2 * (q - 1) + 1];
                ar[q] = xr * cr - xi * ci;
                ai[q] = xr * ci + xi * cr;
            }
            const size_t base = (size_t)g * ns * r + k;
            if (r == 2) {
                y[2 * base] = ar[0] + ar[1];
                y[2 * base + 1] = ai[0] + ai[1];
                y[2 * (base + ns)] = ar[0] - ar[1];
                y[2 * (base + ns) + 1] = ai[0] - ai[1];
            } else if (r == 4) {
                const double t0r = ar[0] + ar[2], t0i = ai[0] + ai[2];
                const double t1r = ar[0] - ar[2], t1i = ai[0] - ai[2];
                const double t2r = ar[1] + ar[3], t2i = ai[1] + ai[3];
                const double dr = ar[1] - ar[3], di = ai[1] - ai[3];
                /* t3 = (s i) * d */
                const double t3r = -sg * di, t3i = sg * dr;
                y[2 * base] = t0r + t2r;
                y[2 * base + 1] = t0i + t2i;
                y[2 * (base + ns)] = t1r + t3r;
                y[2 * (base + ns) + 1] = t1i + t3i;
                y[2 * (base + 2 * ns)] = t0r - t2r;
                y[2 * (base + 2 * ns) + 1] = t0i - t2i;
                y[2 * (base + 3 * ns)] = t1r - t3r;
                y[2 * (base + 3 * ns) + 1] = t1i - t3i;
            } else if (r == 3) {
                const double h = 0.86602540378443864676372317075294; /* sqrt(3)/2 */
                const double t1r = ar[1] + ar[2], t1i = ai[1] + ai[2];
                const double t2r = ar[1] - ar[2], t2i = ai[1] - ai[2];
                const double mr = ar[0] - 0.5 * t1r, mi = ai[0] - 0.5 * t1i;
                const double nr = -sg * h * t2i, ni = sg * h * t2r;
                y[2 * base] = ar[0] + t1r;
                y[2 * base + 1] = ai[0] + t1i;
                y[2 * (base + ns)] = mr + nr;
                y[2 * (base + ns) + 1] = mi + ni;
                y[2 * (base + 2 * ns)] = mr - nr;
                y[2 * (base + 2 * ns) + 1] = mi - ni;
            } else if (r == 5) {
                const double c1 = 0.30901699437494742410229341718282;  /* cos(2pi/5) */
                const double c2 = -0.80901699437494742410229341718282; /* cos(4pi/5) */
                const double s1 = 0.95105651629515357211643933337938;  /* sin(2pi/5) */
                const double s2 = 0.58778525229247312916870595463907;  /* sin(4pi/5) */
                const double t1r = ar[1] + ar[4], t1i = ai[1] + ai[4];
                const double t2r = ar[2] + ar[3], t2i = ai[2] + ai[3];
                const double t3r = ar[1] - ar[4], t3i = ai[1] - ai[4];
                const double t4r = ar[2] - ar[3], t4i = ai[2] - ai[3];
                const double b1r = ar[0] + c1 * t1r + c2 * t2r, b1i = ai[0] + c1 * t1i + c2 * t2i;
                const double b2r = ar[0] + c2 * t1r + c1 * t2r, b2i = ai[0] + c2 * t1i + c1 * t2i;
                const double e1r = s1 * t3r + s2 * t4r, e1i = s1 * t3i + s2 * t4i;
                const double e2r = s2 * t3r - s1 * t4r, e2i = s2 * t3i - s1 * t4i;
                /* d = (s i) * e */
                const double d1r = -sg * e1i, d1i = sg * e1r;
                const double d2r = -sg * e2i, d2i = sg * e2r;
                y[2 * base] = ar[0] + t1r + t2r;
                y[2 * base + 1] = ai[0] + t1i + t2i;
                y[2 * (base + ns)] = b1r + d1r;
                y[2 * (base + ns) + 1] = b1i + d1i;
                y[2 * (base + 4 * ns)] = b1r - d1r;
                y[2 * (base + 4 * ns) + 1] = b1i - d1i;
                y[2 * (base + 2 * ns)] = b2r + d2r;
                y[2 * (base + 2 * ns) + 1] = b2i + d2i;
                y[2 * (base + 3 * ns)] = b2r - d2r;
                y[2 * (base + 3 * ns) + 1] = b2i - d2i;
            } else {
                /* direct DFT for a generic prime radix */
                const double two_pi = 6.283185307179586476925286766559;
                for (int q = 0; q < r; ++q) {
                    double sr = 0.0, si = 0.0;
                    for (int t = 0; t < r; ++t) {
                        const long long e = ((long long)q * t) % r;
                        const double ang = sg * two_pi * (double)e / (double)r;
                        const double cr = cos(ang), ci = sin(ang);
                        sr += ar[t] * cr - ai[t] * ci;
                        si += ar[t] * ci + ai[t] * cr;
                    }
                    y[2 * (base + (size_t)q * ns)] = sr;
                    y[2 * (base + (size_t)q * ns) + 1] = si;
                }
            }
        }
    }
    if (r > 64) {
        free(ar);
        free(ai);
    }
}

void fft64_exec(const fft64_plan* p, double* x, double* work, int sign) {
    const int n = p->n;
    if (n == 1) return;
    double* src = x;
    double* dst = work;
    for (int s = 0; s < p->nstages; ++s) {
        stage(src, dst, n, p->radix[s], p->ns[s], p->tw[s], sign);
        double* t = src;
        src = dst;
        dst = t;
    }
    if (src != x) memcpy(x, src, sizeof(double) * 2 * (size_t)n);
}

void fft64_exec_2d(const fft64_plan* pw, const fft64_plan* ph, double* data, int w, int h, int sign) {
    const int cb = 8; /* columns per gathered block */
    const size_t maxn = (size_t)(w > h ? w : h);
    double* work = (double*)malloc(sizeof(double) * 2 * maxn);
    double* col = (double*)malloc(sizeof(double) * 2 * (size_t)h * cb);
    for (int y = 0; y < h; ++y) fft64_exec(pw, data + 2 * (size_t)y * w, work, sign);
    for (int x0 = 0; x0 < w; x0 += cb) {
        const int nc = (w - x0) < cb ? (w - x0) : cb;
        for (int y = 0; y < h; ++y) {
            const double* row = data + 2 * ((size_t)y * w + x0);
            for (int c = 0; c < nc; ++c) {
                col[2 * ((size_t)c * h + y)] = row[2 * c];
                col[2 * ((size_t)c * h + y) + 1] = row[2 * c + 1];
            }
        }
        for (int c = 0; c < nc; ++c) fft64_exec(ph, col + 2 * (size_t)c * h, work, sign);
        for (int y = 0; y < h; ++y) {
            double* row = data + 2 * ((size_t)y * w + x0);
            for (int c = 0; c < nc; ++c) {
                row[2 * c] = col[2 * ((size_t)c * h + y)];
                row[2 * c + 1] = col[2 * ((size_t)c * h + y) + 1];
            }
        }
    }
    free(col);
    free(work);
}
