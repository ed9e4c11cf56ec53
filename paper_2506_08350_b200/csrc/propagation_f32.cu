// fp32 instantiation of the propagation kernels (the render path) plus the
// precision-independent pieces: FFT planning, transfer-function constants and
// the render's row-IFFT epilogue kernel.
#define HOLO_PROPAGATION_COMMON
#include "propagation_impl.cuh"

namespace holo_cuda {
#define HC_INSTANTIATE(T)                                                                                        \
    template void rows_fft<T>(holo_ctx*, const cx<T>*, cx<T>*, int, long long, int, T);                           \
    template void cols_fft<T>(holo_ctx*, const cx<T>*, cx<T>*, int, int, int, int, T);                           \
    template void col_spectrum<T>(holo_ctx*, const cx<T>*, cx<T>*, int, int, int, int, const TfChan*, double,     \
                                  const ColOpts<T>&);                                                             \
    template void col_replay<T>(holo_ctx*, const cx<T>*, cx<T>*, int, int, int, int, const int*, const TfChan*,   \
                                double, const ColOpts<T>&);                                                       \
    template void pad_field<T>(holo_ctx*, const cx<T>*, cx<T>*, int, int, int);                                   \
    template void crop_field<T>(holo_ctx*, const cx<T>*, cx<T>*, int, int, int);                                  \
    template void accumulate<T>(holo_ctx*, const cx<T>*, cx<T>*, size_t, bool);                                   \
    template void intensity<T>(holo_ctx*, const cx<T>*, T*, size_t);                                              \
    template void transfer_function<T>(holo_ctx*, cx<T>*, int, int, int, const TfChan*, double);
HC_INSTANTIATE(float)
}  // namespace holo_cuda
