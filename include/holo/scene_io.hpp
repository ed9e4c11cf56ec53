// Drop-in for proj/include/holo/scene_io.hpp: the HOLOSCENE1 container
// (scene_io.cpp:29-95): 10-byte magic, u32 header length, JSON header {L, N,
// units}, then the seven f64 arrays of GaussianScene in declaration order.
#pragma once

#include <string>

#include "holo/scene.hpp"

namespace holo {

void write_scene(const std::string& path, const GaussianScene& s);
GaussianScene read_scene(const std::string& path);

}  // namespace holo
