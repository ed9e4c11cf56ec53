// Drop-in for the render-path part of proj/include/holo/scene.hpp (training-only
// members -- gradients, init, densification -- are out of scope for this build).
#pragma once

#include <Eigen/Dense>
#include <vector>

#include "holo/camera.hpp"
#include "holo/common.hpp"
#include "holo/wave_config.hpp"

namespace holo {

// Complex Gaussians, struct of arrays; 3 amplitude / phase channels.
struct GaussianScene {
    static constexpr int kChannels = 3;

    int num_planes = 1;
    std::vector<double> positions;       // N*3
    std::vector<double> rotations;       // N*4, (w, x, y, z)
    std::vector<double> log_scales;      // N*3
    std::vector<double> amplitudes;      // N*3
    std::vector<double> opacity_logits;  // N
    std::vector<double> phases;          // N*3
    std::vector<double> plane_logits;    // N*num_planes

    size_t size() const { return opacity_logits.size(); }
    void resize(size_t n);
    void validate() const;
    void renormalize();
};

// d(loss)/d(scene parameters), scene.hpp:40-46 of the reference
struct SceneGradients {
    std::vector<double> positions, rotations, log_scales, amplitudes, opacity_logits, phases, plane_logits;
    std::vector<double> mu_screen;  // N * 2, screen-space mean gradient (pixels)
    void resize_like(const GaussianScene& s);
    void clear();
};

// Sigma = R diag(e^s)^2 R^T for the normalised quaternion (scene.hpp:49)
Eigen::Matrix3d covariance_3d(const double* quat, const double* log_scales);

namespace detail {
Eigen::Matrix3d quat_to_rot(const double* q);  // scene.hpp:53
}

// argmax plane (ties -> lowest index); backward weights softmax(logits / tau)
struct SteAssign {
    int index = 0;
    std::vector<double> onehot;
    std::vector<double> backward_weights;
};
SteAssign ste_assign(const double* logits, int L, double tau);

}  // namespace holo
