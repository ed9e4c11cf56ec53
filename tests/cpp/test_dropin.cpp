// The drop-in C++ API (include/holo/*.hpp -> libholo.so -> libholo_cuda.so) on
// the GPU, written like the reference's own doctest suites
// (proj/tests/test_rasterizer.cpp, test_pipeline.cpp): KATs at fp32 tolerance
// for the rasteriser (the render path is fp32), reference tolerances for the
// f64 operators, shapes and error kinds.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>

#include "holo/device.hpp"
#include "holo/fft.hpp"
#include "holo/pipeline.hpp"

using namespace holo;

namespace {

WaveConfig desk(int n, int planes) {
    WaveConfig cfg;
    cfg.nx = n;
    cfg.ny = n;
    cfg.num_planes = planes;
    return cfg;
}

CameraView front(const WaveConfig& cfg, double f = 150.0) {
    CameraView cam;
    cam.focal_px = f;
    cam.width = cfg.nx;
    cam.height = cfg.ny;
    return cam;
}

GaussianScene centred(int n, const CameraView& cam) {
    GaussianScene s;
    s.num_planes = 1;
    s.resize(n);
    const double z = 0.3, off = 0.5 * z / cam.focal_px;
    for (int i = 0; i < n; ++i) {
        s.positions[3 * i] = off;
        s.positions[3 * i + 1] = off;
        s.positions[3 * i + 2] = z;
        for (int d = 0; d < 3; ++d) {
            s.log_scales[3 * i + d] = std::log(0.004);
            s.amplitudes[3 * i + d] = 1.0;
        }
    }
    return s;
}

}  // namespace

TEST_CASE("blending recurrence matches the hand-computed cases") {
    const WaveConfig cfg = desk(32, 1);
    const CameraView cam = front(cfg);
    GaussianScene s = centred(1, cam);
    s.opacity_logits = {logit(0.8)};
    RasterForward r = raster_forward(s, cam, cfg, RenderSettings{});
    CHECK(std::abs(r.layers[0].at(0, 16, 16) - c64(0.8, 0.0)) < 1e-6);
    CHECK(r.t_final[16 * 32 + 16] == doctest::Approx(0.2).epsilon(1e-6));
    CHECK(r.n_contrib[16 * 32 + 16] == 1);
    GaussianScene two = centred(2, cam);
    two.opacity_logits = {0.0, 0.0};
    for (int d = 0; d < 3; ++d) two.phases[3 + d] = kPi;
    r = raster_forward(two, cam, cfg, RenderSettings{});
    CHECK(std::abs(r.layers[0].at(0, 16, 16) - c64(0.25, 0.0)) < 1e-6);
    CHECK(r.entries.size() >= 2);
    CHECK(r.entries[0].gidx == 0);  // equal depth: index order
}

TEST_CASE("raster_backward: amplitude and phase gradients of a linear loss") {
    // L = Re sum_p <g, layer_p>: with g = 1 on channel 0, dL/d amp_0 = sum_p Re layer_p
    // (amp = 1, phase 0); with g = i, dL/d phase_0 is the same sum
    const WaveConfig cfg = desk(32, 1);
    const CameraView cam = front(cfg);
    GaussianScene s = centred(1, cam);
    s.opacity_logits = {logit(0.8)};
    const RasterForward r = raster_forward(s, cam, cfg, RenderSettings{});
    double sum_re = 0.0;
    for (int y = 0; y < 32; ++y)
        for (int x = 0; x < 32; ++x) sum_re += r.layers[0].at(0, y, x).real();
    std::vector<ComplexField> g(1, ComplexField(32, 32, 3, cfg.pitch));
    for (int y = 0; y < 32; ++y)
        for (int x = 0; x < 32; ++x) g[0].at(0, y, x) = c64(1.0, 0.0);
    SceneGradients gr = raster_backward(s, cam, cfg, RenderSettings{}, r, g);
    CHECK(gr.positions.size() == 3);
    CHECK(gr.plane_logits.size() == 1);
    CHECK(gr.amplitudes[0] == doctest::Approx(sum_re).epsilon(1e-5));
    CHECK(gr.amplitudes[1] == 0.0);
    for (int y = 0; y < 32; ++y)
        for (int x = 0; x < 32; ++x) g[0].at(0, y, x) = c64(0.0, 1.0);
    gr = raster_backward(s, cam, cfg, RenderSettings{}, r, g);
    CHECK(gr.phases[0] == doctest::Approx(sum_re).epsilon(1e-5));
    std::vector<ComplexField> wrong;
    CHECK_THROWS_AS(raster_backward(s, cam, cfg, RenderSettings{}, r, wrong), HoloError);
}

TEST_CASE("projection lands where the pinhole model says, f64 exact") {
    const WaveConfig cfg = desk(32, 1);
    const CameraView cam = front(cfg);
    GaussianScene s;
    s.num_planes = 1;
    s.resize(1);
    s.positions = {0.01, -0.005, 0.3};
    s.opacity_logits = {0.5};
    for (int d = 0; d < 3; ++d) {
        s.log_scales[d] = std::log(0.004);
        s.amplitudes[d] = 0.5;
    }
    const RasterForward r = raster_forward(s, cam, cfg, RenderSettings{});
    CHECK(r.projected[0].valid);
    CHECK(r.projected[0].mu_x == doctest::Approx(21.0).epsilon(1e-12));
    CHECK(r.projected[0].mu_y == doctest::Approx(13.5).epsilon(1e-12));
    CHECK(r.touched[0] == 1);
}

TEST_CASE("pipeline forward produces consistently shaped stages") {
    const WaveConfig cfg = desk(32, 2);
    const CameraView cam = front(cfg);
    GaussianScene s;
    s.num_planes = 2;
    s.resize(6);
    for (int i = 0; i < 6; ++i) {
        s.positions[3 * i] = 0.004 * (i - 3);
        s.positions[3 * i + 2] = 0.3 + 0.01 * i;
        s.opacity_logits[i] = 0.5;
        s.plane_logits[2 * i + (i % 2)] = 1.0;
        for (int d = 0; d < 3; ++d) {
            s.log_scales[3 * i + d] = std::log(0.006);
            s.amplitudes[3 * i + d] = 0.7;
            s.phases[3 * i + d] = 0.3 * d;
        }
    }
    const PipelineForward pf = pipeline_forward(s, cam, cfg, PipelineOptions{});
    CHECK(pf.hologram.w == 32);
    CHECK(pf.hologram.c == 3);
    REQUIRE(pf.replayed.size() == 2);
    REQUIRE(pf.intensities.size() == 2);
    double m = 0.0;
    for (size_t l = 0; l < 2; ++l) {
        const IntensityImage direct = intensity(pf.replayed[l]);
        for (size_t i = 0; i < direct.data.size(); ++i)
            m = std::max(m, std::abs(direct.data[i] - pf.intensities[l].data[i]) / (1e-3 + direct.data[i]));
    }
    CHECK(m < 1e-5);
    // the hologram's replay is the recorded layers' propagation chain
    const ComplexField rec = forward_record(pf.raster.layers, cfg);
    double num = 0, den = 0;
    for (size_t i = 0; i < rec.data.size(); ++i) {
        num += std::norm(rec.data[i] - pf.hologram.data[i]);
        den += std::norm(rec.data[i]);
    }
    CHECK(std::sqrt(num / den) < 1e-5);
}

TEST_CASE("make_target_from_scene masks follow the dominant rasterised plane") {
    // the device masks (holo_plane_masks) against pipeline.cpp:106-124 evaluated on
    // the host over the returned (widened) layers of the same scene
    const WaveConfig cfg = desk(48, 3);
    const CameraView cam = front(cfg);
    GaussianScene s;
    s.num_planes = 3;
    s.resize(40);
    for (int i = 0; i < 40; ++i) {
        s.positions[3 * i] = 0.0009 * ((i * 7) % 19 - 9);
        s.positions[3 * i + 1] = 0.0009 * ((i * 11) % 17 - 8);
        s.positions[3 * i + 2] = 0.3 + 0.002 * (i % 5);
        s.opacity_logits[i] = 0.2 * (i % 4);
        s.plane_logits[3 * i + (i % 3)] = 1.0;
        for (int d = 0; d < 3; ++d) {
            s.log_scales[3 * i + d] = std::log(0.002 + 0.0005 * (i % 3));
            s.amplitudes[3 * i + d] = 0.3 + 0.1 * ((i + d) % 5);
            s.phases[3 * i + d] = 0.4 * d + 0.1 * i;
        }
    }
    const PipelineOptions opt{};
    const FocalStackTarget t = make_target_from_scene(s, cam, cfg, opt);
    const PipelineForward f = pipeline_forward(s, cam, cfg, opt);
    REQUIRE(t.masks.size() == 3);
    int masked = 0;
    for (int y = 0; y < cfg.ny; ++y)
        for (int x = 0; x < cfg.nx; ++x) {
            int best = -1;
            double best_amp = 0.0;
            for (int l = 0; l < 3; ++l) {
                double amp = 0.0;
                for (int ch = 0; ch < f.raster.layers[l].c; ++ch) amp += std::abs(f.raster.layers[l].at(ch, y, x));
                if (amp > best_amp) {
                    best_amp = amp;
                    best = l;
                }
            }
            for (int l = 0; l < 3; ++l) CHECK(t.masks[l].at(0, y, x) == (l == best ? 1.0 : 0.0));
            masked += best >= 0;
        }
    CHECK(masked > 100);
    CHECK(masked < cfg.nx * cfg.ny);
}

TEST_CASE("f64 operators meet the reference tolerances") {
    WaveConfig cfg = desk(64, 1);
    ComplexField u(64, 64, 3, cfg.pitch);
    for (size_t i = 0; i < u.data.size(); ++i) u.data[i] = c64(std::sin(0.37 * i), std::cos(0.11 * i));
    const ComplexField rec = forward_record({u}, cfg);
    const ComplexField ref = propagate(u, cfg, cfg.distance);
    double m = 0;
    for (size_t i = 0; i < rec.data.size(); ++i) m = std::max(m, std::abs(rec.data[i] - ref.data[i]));
    CHECK(m == 0.0);  // test_propagation.cpp:117-123: identical code path
    ComplexField f = u;
    fft2(f.channel(0), 64, 64);
    ifft2(f.channel(0), 64, 64);
    m = 0;
    for (size_t i = 0; i < 64 * 64; ++i) m = std::max(m, std::abs(f.data[i] - u.data[i]));
    CHECK(m < 1e-12);
}

TEST_CASE("errors carry the reference kinds") {
    const WaveConfig cfg = desk(32, 2);
    GaussianScene s;
    s.num_planes = 1;
    s.resize(2);
    CHECK_THROWS_AS(raster_forward(s, front(cfg), cfg, RenderSettings{}), HoloError);
    CameraView bad = front(cfg);
    bad.width = 16;
    s.num_planes = 2;
    s.resize(2);
    CHECK_THROWS_AS(raster_forward(s, bad, cfg, RenderSettings{}), HoloError);
    try {
        propagate(ComplexField(32, 32, 1, cfg.pitch), cfg, 1e-3);
        CHECK(false);
    } catch (const HoloError& e) {
        CHECK(e.kind == "config");
    }
    RenderSettings st;
    st.tile = 12;
    try {
        raster_forward(s, front(cfg), cfg, st);
        CHECK(false);
    } catch (const HoloError& e) {
        CHECK(e.kind == "config");
    }
}
