// Drop-in for proj/include/holo/fft.hpp: in-place 2-D c2c transforms on the GPU
// (f64), forward exp(-2 pi i f x) unnormalised, inverse with 1/(w h).
#pragma once

#include "holo/common.hpp"

namespace holo {

void fft2(c64* data, int w, int h);
void ifft2(c64* data, int w, int h);

}  // namespace holo
