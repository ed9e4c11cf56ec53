// Drop-in for proj/include/holo/field_io.hpp: HOLOFIELD container (16-byte magic
// "HOLOFIELD" zero padded, u32 W, H, C, then f64 (re, im) pairs, planar).
#pragma once

#include <string>

#include "holo/field.hpp"

namespace holo {

void write_field(const std::string& path, const ComplexField& f);
ComplexField read_field(const std::string& path, double pitch = 3.74e-6);

}  // namespace holo
