// Device controls of the drop-in build (no counterpart in the reference):
// which GPU the calling thread's holo_ctx uses and the precision of the
// propagation operators (f64 matches the reference to ~1e-15; the render path
// is always fp32).
#pragma once

namespace holo::device {

void set_device(int device);                 // before the thread's first call
void set_operator_precision(bool use_f64);   // default true
bool operator_precision_f64();

}  // namespace holo::device
