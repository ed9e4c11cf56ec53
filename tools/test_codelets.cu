// Host-side check of the FFT codelets and the Stockham stage logic (fft.cuh):
// runs every stage of the plan on the CPU and compares with a direct DFT.
#include <complex>
#include <cstdio>
#include <random>
#include "fft.cuh"
using namespace holo_cuda;
template <int DIR, class T>
double run(int n) {
    FftPlan p;
    if (!make_plan(n, &p)) return -1;
    std::vector<cx<T>> a(n), b(n), tw(n);
    std::mt19937 g(n);
    std::normal_distribution<double> N;
    std::vector<std::complex<double>> x(n);
    for (int i = 0; i < n; ++i) { x[i] = {N(g), N(g)}; a[i] = mk<T>(x[i].real(), x[i].imag()); }
    for (int q = 0; q < n; ++q) { double ang = -2 * M_PI * q / n; tw[q] = mk<T>(std::cos(ang), std::sin(ang)); }
    cx<T>* src = a.data(); cx<T>* dst = b.data();
    int ns = 1;
    for (int s = 0; s < p.nstages; ++s) {
        int R = p.radix[s];
        for (int j = 0; j < n / R; ++j)
            butterfly_any<DIR, T>(R, j, n, ns, tw.data(), [&](int i) { return src[i]; }, [&](int i, cx<T> v) { dst[i] = v; });
        std::swap(src, dst); ns *= R;
    }
    double err = 0, nrm = 0;
    for (int k = 0; k < n; ++k) {
        std::complex<double> acc = 0;
        for (int t = 0; t < n; ++t) acc += x[t] * std::polar(1.0, DIR * 2 * M_PI * double((long long)t * k % n) / n);
        err += std::norm(acc - std::complex<double>(src[k].x, src[k].y)); nrm += std::norm(acc);
    }
    return std::sqrt(err / nrm);
}
int main() {
    int sizes[] = {2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,19,23,29,31,30,32,42,48,64,96,120,128,135,240,256,360,1080,1920,1024,2160};
    int bad = 0;
    for (int n : sizes) {
        FftPlan p; make_plan(n, &p);
        double e1 = run<-1, double>(n), e2 = run<+1, double>(n), e3 = run<-1, float>(n);
        printf("n=%5d plan=", n); for (int s = 0; s < p.nstages; ++s) printf("%d ", p.radix[s]);
        printf(" f64fwd=%.2e f64inv=%.2e f32fwd=%.2e\n", e1, e2, e3);
        if (e1 > 1e-12 || e2 > 1e-12 || e3 > 1e-5) ++bad;
    }
    printf("bad=%d\n", bad);
    return bad;
}
