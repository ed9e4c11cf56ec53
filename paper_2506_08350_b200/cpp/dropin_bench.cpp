// dropin_bench — wall time of holo::pipeline_forward through the drop-in C++ API
// (libholo.so), timed the way the reference times its own API (steady_clock
// around each call, holo_main.cpp:507-514).  Every call is the reference's value
// semantics end to end: the host scene goes in, the full PipelineForward (f64
// raster layers and lists, hologram, replayed fields, intensities) comes back.
//
//   dropin_bench SCENE.holoscene --nx W --ny H --planes L --wavelengths a,b,c
//                [--focal F] [--frames K] [--warmup W]
// prints one JSON line {frames_per_s, seconds_per_frame, ...}.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "holo/pipeline.hpp"
#include "holo/scene_io.hpp"

int main(int argc, char** argv) {
    try {
        if (argc < 2) {
            std::cerr << "usage: dropin_bench SCENE --nx W --ny H --planes L --wavelengths a,b,c [--focal F] "
                         "[--frames K] [--warmup W]\n";
            return 2;
        }
        const std::string path = argv[1];
        int nx = 0, ny = 0, planes = 0, frames = 5, warmup = 1;
        double focal = 0.0;
        std::vector<double> wl;
        for (int i = 2; i + 1 < argc; i += 2) {
            const std::string k = argv[i], v = argv[i + 1];
            if (k == "--nx") nx = std::atoi(v.c_str());
            else if (k == "--ny") ny = std::atoi(v.c_str());
            else if (k == "--planes") planes = std::atoi(v.c_str());
            else if (k == "--frames") frames = std::atoi(v.c_str());
            else if (k == "--warmup") warmup = std::atoi(v.c_str());
            else if (k == "--focal") focal = std::atof(v.c_str());
            else if (k == "--wavelengths") {
                std::stringstream ss(v);
                std::string t;
                while (std::getline(ss, t, ',')) wl.push_back(std::atof(t.c_str()));
            } else {
                std::cerr << "unknown option " << k << "\n";
                return 2;
            }
        }
        const holo::GaussianScene scene = holo::read_scene(path);
        holo::WaveConfig cfg;
        cfg.nx = nx;
        cfg.ny = ny;
        cfg.num_planes = planes;
        if (!wl.empty()) cfg.wavelengths = wl;
        holo::CameraView cam;
        cam.width = nx;
        cam.height = ny;
        cam.focal_px = focal > 0.0 ? focal : nx;
        holo::PipelineOptions opt;
        size_t entries = 0;
        for (int i = 0; i < warmup; ++i) entries = holo::pipeline_forward(scene, cam, cfg, opt).raster.entries.size();
        double total = 0.0;
        for (int i = 0; i < frames; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            const holo::PipelineForward f = holo::pipeline_forward(scene, cam, cfg, opt);
            const auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
            entries = f.raster.entries.size();
        }
        std::printf("{\"api\": \"holo::pipeline_forward (libholo.so)\", \"frames\": %d, \"seconds_per_frame\": %.6f, "
                    "\"frames_per_s\": %.4f, \"gaussians\": %zu, \"entries\": %zu}\n",
                    frames, total / frames, frames / total, scene.size(), entries);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dropin_bench: %s\n", e.what());
        return 1;
    }
}
