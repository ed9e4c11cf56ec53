// holo — command-line front end of the drop-in (the render / propagate / bench
// subcommands of proj/tools/holo_main.cpp) over libholo.so, so the GPU path is
// usable as a binary.  Same conventions as the reference: one JSON line on
// stdout per command, {"error": {"kind", "message"}} on stderr, exit code 2 for
// usage / config errors and 1 for the others (holo_main.cpp:695-724).
//
//   holo propagate --in F.hfld --out G.hfld --z-meters Z [--pixel-pitch P]
//                  [--wavelength L ...] [--pad2x] [--local-band-limit]
//   holo render --scene S.holoscene --out-dir DIR [--nx N --ny N] [--pixel-pitch P]
//               [--wavelength L ...] [--distance D] [--volume-depth V] [--focal-px F]
//               [--pose x y z rx ry rz]
//   holo bench [--grid N] [--n-list a,b,...] [--l-list a,b,...] [--out CSV]
//   holo phase-only --in F.hfld --out PHASE.png [--iters N] [--bits 8|10] [--lr R]
//                   [--lambda-ssim X] [--pixel-pitch P] [--wavelength L ...] [--no-pad]
//
// The reference's train / gradcheck / stats subcommands and its run
// configuration JSON are outside this repository's scope.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <zlib.h>

#include "holo/field_io.hpp"
#include "holo/phase_only.hpp"
#include "holo/pipeline.hpp"
#include "holo/propagation.hpp"
#include "holo/scene_io.hpp"

using namespace holo;

namespace {

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

std::string jnum(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

// --flag value [value ...] parser: values run until the next "--" token
struct Args {
    std::map<std::string, std::vector<std::string>> opt;
    explicit Args(int argc, char** argv, int first) {
        std::string cur;
        for (int i = first; i < argc; ++i) {
            const std::string a = argv[i];
            if (a.rfind("--", 0) == 0) {
                cur = a.substr(2);
                opt[cur];
            } else if (!cur.empty()) {
                opt[cur].push_back(a);
            } else {
                throw HoloError("usage", "unexpected argument: " + a);
            }
        }
    }
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k) const {
        auto it = opt.find(k);
        if (it == opt.end() || it->second.size() != 1) throw HoloError("usage", "--" + k + " needs one value");
        return it->second[0];
    }
    std::string str_or(const std::string& k, const std::string& d) const { return has(k) ? str(k) : d; }
    double num(const std::string& k, double d) const {
        if (!has(k)) return d;
        const std::string s = str(k);
        char* end = nullptr;
        const double v = std::strtod(s.c_str(), &end);
        if (end == s.c_str() || *end) throw HoloError("usage", "--" + k + ": not a number: " + s);
        return v;
    }
    std::vector<double> nums(const std::string& k) const {
        std::vector<double> out;
        auto it = opt.find(k);
        if (it == opt.end()) return out;
        for (const std::string& s0 : it->second) {
            std::stringstream ss(s0);
            std::string t;
            while (std::getline(ss, t, ',')) {
                char* end = nullptr;
                const double v = std::strtod(t.c_str(), &end);
                if (end == t.c_str() || *end) throw HoloError("usage", "--" + k + ": not a number: " + t);
                out.push_back(v);
            }
        }
        return out;
    }
    void require(const std::string& k) const {
        if (!has(k)) throw HoloError("usage", "--" + k + " is required");
    }
    void only(const std::vector<std::string>& allowed) const {
        for (const auto& kv : opt) {
            bool ok = false;
            for (const auto& a : allowed) ok = ok || a == kv.first;
            if (!ok) throw HoloError("usage", "unknown option --" + kv.first);
        }
    }
};

// holo_main.cpp:93-103
std::vector<double> wavelengths_for(const std::vector<double>& flags, int channels) {
    if (!flags.empty()) {
        if (static_cast<int>(flags.size()) != channels) throw HoloError("usage", "need one --wavelength per field channel");
        return flags;
    }
    const std::vector<double> stock = {639e-9, 532e-9, 473e-9};
    if (channels > static_cast<int>(stock.size()))
        throw HoloError("usage", "more than three channels need explicit --wavelength flags");
    return {stock.begin(), stock.begin() + channels};
}

// holo_main.cpp:314-341
int cmd_propagate(const Args& a) {
    a.only({"in", "out", "z-meters", "pixel-pitch", "wavelength", "pad2x", "local-band-limit"});
    a.require("in");
    a.require("out");
    a.require("z-meters");
    const double pitch = a.num("pixel-pitch", 3.74e-6);
    const ComplexField u = read_field(a.str("in"), pitch);
    WaveConfig cfg;
    cfg.nx = u.w;
    cfg.ny = u.h;
    cfg.pitch = pitch;
    cfg.wavelengths = wavelengths_for(a.nums("wavelength"), u.c);
    cfg.num_planes = 1;
    PropagationOptions opt;
    opt.pad2x = a.has("pad2x");
    opt.local_band_limit = a.has("local-band-limit");
    const double z = a.num("z-meters", 0.0);
    const ComplexField out = propagate(u, cfg, z, opt);
    write_field(a.str("out"), out);
    std::cout << "{\"command\":\"propagate\",\"in\":" << jstr(a.str("in")) << ",\"out\":" << jstr(a.str("out"))
              << ",\"z_meters\":" << jnum(z) << ",\"energy_in\":" << jnum(energy(u))
              << ",\"energy_out\":" << jnum(energy(out)) << "}\n";
    return 0;
}

// render a HOLOSCENE1 scene: hologram.hfld and replay_<l>.hfld in --out-dir
int cmd_render(const Args& a) {
    a.only({"scene", "out-dir", "nx", "ny", "pixel-pitch", "wavelength", "distance", "volume-depth", "focal-px",
            "pose"});
    a.require("scene");
    a.require("out-dir");
    const GaussianScene scene = read_scene(a.str("scene"));
    WaveConfig cfg;
    cfg.nx = static_cast<int>(a.num("nx", 1920));
    cfg.ny = static_cast<int>(a.num("ny", 1080));
    cfg.pitch = a.num("pixel-pitch", cfg.pitch);
    cfg.wavelengths = wavelengths_for(a.nums("wavelength"), GaussianScene::kChannels);
    cfg.distance = a.num("distance", cfg.distance);
    cfg.volume_depth = a.num("volume-depth", cfg.volume_depth);
    cfg.num_planes = scene.num_planes;
    CameraView cam;
    cam.width = cfg.nx;
    cam.height = cfg.ny;
    cam.focal_px = a.num("focal-px", cfg.nx);
    const std::vector<double> pose = a.nums("pose");
    if (!pose.empty()) {
        if (pose.size() != 6) throw HoloError("usage", "--pose needs x y z rx ry rz");
        for (int i = 0; i < 6; ++i) cam.pose[i] = pose[i];
    }
    const auto t0 = std::chrono::steady_clock::now();
    const PipelineForward f = pipeline_forward(scene, cam, cfg, PipelineOptions{});
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const std::string dir = a.str("out-dir");
    write_field(dir + "/hologram.hfld", f.hologram);
    for (size_t l = 0; l < f.replayed.size(); ++l) write_field(dir + "/replay_" + std::to_string(l) + ".hfld", f.replayed[l]);
    std::cout << "{\"command\":\"render\",\"scene\":" << jstr(a.str("scene")) << ",\"gaussians\":" << scene.size()
              << ",\"planes\":" << cfg.num_planes << ",\"entries\":" << f.raster.entries.size()
              << ",\"seconds\":" << jnum(secs) << ",\"hologram\":" << jstr(dir + "/hologram.hfld") << "}\n";
    return 0;
}

// holo_main.cpp:483-527: wall time of raster_forward and forward_record per (n, L)
int cmd_bench(const Args& a) {
    a.only({"grid", "n-list", "l-list", "out"});
    const int grid = static_cast<int>(a.num("grid", 256));
    std::vector<double> ns = a.nums("n-list"), ls = a.nums("l-list");
    if (ns.empty()) ns = {10000, 20000, 40000, 80000};
    if (ls.empty()) ls = {1, 2, 4, 8};
    std::string csv = "n,l,raster_seconds,record_seconds,total_seconds\n";
    for (double Ld : ls) {
        const int L = static_cast<int>(Ld);
        if (L < 1) throw HoloError("usage", "plane counts must be positive");
        WaveConfig cfg;
        cfg.nx = cfg.ny = grid;
        cfg.num_planes = L;
        CameraView cam;
        cam.width = cam.height = grid;
        cam.focal_px = grid;
        for (double nd : ns) {
            if (nd < 0) throw HoloError("usage", "gaussian counts must be non-negative");
            // a deterministic frustum-filling scene (splitmix64 counter RNG)
            const size_t n = static_cast<size_t>(nd);
            GaussianScene s;
            s.num_planes = L;
            s.resize(n);
            auto u = [](unsigned long long c) {
                unsigned long long z = c + 0x9E3779B97F4A7C15ull;
                z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
                z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
                z ^= z >> 31;
                return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);
            };
            for (size_t i = 0; i < n; ++i) {
                const unsigned long long k = (1234ull + L) * 0x100000000ull + 32ull * i;
                const double zc = 0.25 + 0.2 * u(k);
                s.positions[3 * i] = (u(k + 1) - 0.5) * grid * zc / grid;
                s.positions[3 * i + 1] = (u(k + 2) - 0.5) * grid * zc / grid;
                s.positions[3 * i + 2] = zc;
                s.rotations[4 * i] = 1.0;
                for (int d = 0; d < 3; ++d) {
                    s.log_scales[3 * i + d] = std::log((0.5 + 2.5 * u(k + 3 + d)) * 0.35 / grid);
                    s.amplitudes[3 * i + d] = 0.2 + 0.8 * u(k + 6 + d);
                    s.phases[3 * i + d] = 6.283185307179586 * u(k + 9 + d);
                }
                s.opacity_logits[i] = -2.0 + 4.0 * u(k + 12);
                for (int l = 0; l < L; ++l) s.plane_logits[i * L + l] = l == static_cast<int>(i % L) ? 2.0 : 0.1 * l;
            }
            const auto t0 = std::chrono::steady_clock::now();
            const RasterForward fwd = raster_forward(s, cam, cfg, RenderSettings{});
            const auto t1 = std::chrono::steady_clock::now();
            const ComplexField holo = forward_record(fwd.layers, cfg, PropagationOptions{});
            const auto t2 = std::chrono::steady_clock::now();
            (void)holo;
            const double rs = std::chrono::duration<double>(t1 - t0).count();
            const double ps = std::chrono::duration<double>(t2 - t1).count();
            char line[160];
            std::snprintf(line, sizeof line, "%zu,%d,%.6f,%.6f,%.6f\n", n, L, rs, ps, rs + ps);
            csv += line;
        }
    }
    if (a.has("out")) {
        std::ofstream o(a.str("out"), std::ios::binary);
        if (!o) throw HoloError("io", "cannot open for writing: " + a.str("out"));
        o << csv;
    } else {
        std::cout << csv;
    }
    return 0;
}

// ---- phase-only (holo_main.cpp:344-386) and its quantised phase PNGs (png_io.cpp:160-187)

void put_be32(std::string& s, unsigned v) {
    for (int k = 3; k >= 0; --k) s += static_cast<char>((v >> (8 * k)) & 0xff);
}

void png_chunk(std::string& out, const char* type, const std::string& data) {
    put_be32(out, static_cast<unsigned>(data.size()));
    const std::string td = std::string(type, 4) + data;
    out += td;
    put_be32(out, static_cast<unsigned>(crc32(0L, reinterpret_cast<const Bytef*>(td.data()), static_cast<uInt>(td.size()))));
}

// grayscale PNG, 8 or 16 bits per sample; `rows` holds the raw big-endian samples
void write_gray_png(const std::string& path, int w, int h, int depth, const std::string& raw) {
    std::string filtered;
    const size_t row_bytes = static_cast<size_t>(w) * (depth / 8);
    filtered.reserve((row_bytes + 1) * h);
    for (int y = 0; y < h; ++y) {
        filtered += '\0';  // filter type None
        filtered.append(raw, static_cast<size_t>(y) * row_bytes, row_bytes);
    }
    uLongf zlen = compressBound(static_cast<uLong>(filtered.size()));
    std::string z(zlen, '\0');
    if (compress2(reinterpret_cast<Bytef*>(z.data()), &zlen, reinterpret_cast<const Bytef*>(filtered.data()),
                  static_cast<uLong>(filtered.size()), 6) != Z_OK)
        throw HoloError("io", "png: compression failed");
    z.resize(zlen);
    std::string ihdr;
    put_be32(ihdr, static_cast<unsigned>(w));
    put_be32(ihdr, static_cast<unsigned>(h));
    ihdr += static_cast<char>(depth);
    ihdr += std::string("\0\0\0\0", 4);  // gray, deflate, no filter method, no interlace
    std::string png = "\x89PNG\r\n\x1a\n";
    png_chunk(png, "IHDR", ihdr);
    png_chunk(png, "IDAT", z);
    png_chunk(png, "IEND", "");
    std::ofstream o(path, std::ios::binary);
    if (!o) throw HoloError("io", "cannot open for writing: " + path);
    o.write(png.data(), static_cast<std::streamsize>(png.size()));
    if (!o) throw HoloError("io", "write failed: " + path);
}

// png_io.cpp:160-187: codes lround(wrap(phi) / step) mod 2^bits; 10-bit codes
// stored as 16-bit samples (code << 6 | code >> 4)
void write_phase_png(const std::string& path, const double* phase, int w, int h, int bits) {
    if (bits != 8 && bits != 10) throw HoloError("io", "png: phase bit depth must be 8 or 10");
    const int levels = 1 << bits;
    const double step = 2.0 * 3.14159265358979323846 / levels;
    const size_t n = static_cast<size_t>(w) * h;
    std::string raw;
    raw.reserve(n * (bits == 8 ? 1 : 2));
    for (size_t i = 0; i < n; ++i) {
        const unsigned code = static_cast<unsigned>(std::lround(wrap_phase(phase[i]) / step) % levels);
        if (bits == 8) {
            raw += static_cast<char>(code);
        } else {
            const unsigned v = (code << 6) | (code >> 4);
            raw += static_cast<char>((v >> 8) & 0xff);
            raw += static_cast<char>(v & 0xff);
        }
    }
    write_gray_png(path, w, h, bits == 8 ? 8 : 16, raw);
}

// png_io.cpp:217-226
std::string channel_path(const std::string& base, int ch, int channels) {
    if (channels == 1) return base;
    static const char* rgb[3] = {"_r", "_g", "_b"};
    const std::string suffix = channels == 3 ? rgb[ch] : "_c" + std::to_string(ch);
    const size_t dot = base.find_last_of('.');
    const size_t slash = base.find_last_of("/\\");
    if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) return base + suffix;
    return base.substr(0, dot) + suffix + base.substr(dot);
}

int cmd_phase_only(const Args& a) {
    a.only({"in", "out", "iters", "bits", "lr", "lambda-ssim", "pixel-pitch", "wavelength", "no-pad"});
    a.require("in");
    a.require("out");
    const int bits = static_cast<int>(a.num("bits", 8));
    if (bits != 8 && bits != 10) throw HoloError("usage", "--bits must be 8 or 10");
    const double pitch = a.num("pixel-pitch", 3.74e-6);
    const ComplexField P = read_field(a.str("in"), pitch);
    WaveConfig optics;  // the run configuration's default optics
    optics.nx = P.w;
    optics.ny = P.h;
    optics.pitch = pitch;
    optics.wavelengths = wavelengths_for(a.nums("wavelength"), P.c);
    PhaseOnlyOptions opt;
    opt.lambda_ssim = a.num("lambda-ssim", 1.0);
    if (a.has("no-pad")) opt.prop.pad2x = false;
    const int iters = static_cast<int>(a.num("iters", 1000));
    const PhaseOnlyResult res = convert_phase_only(P, optics, iters, a.num("lr", 0.02), opt);
    std::string files = "[";
    const std::string out = a.str("out");
    for (int ch = 0; ch < P.c; ++ch) {
        const std::string path = channel_path(out, ch, P.c);
        write_phase_png(path, res.hologram.phase.data() + static_cast<size_t>(ch) * P.h * P.w, P.w, P.h, bits);
        files += (ch ? "," : "") + jstr(path);
    }
    files += "]";
    const double init = res.trace.front();
    double best = init;
    for (double v : res.trace) best = std::min(best, v);
    std::cout << "{\"command\":\"phase-only\",\"iterations\":" << iters << ",\"bits\":" << bits
              << ",\"initial_loss\":" << jnum(init) << ",\"final_loss\":" << jnum(best)
              << ",\"ratio\":" << jnum(init > 0.0 ? best / init : 0.0) << ",\"files\":" << files << "}\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) throw HoloError("usage", "a subcommand is required: render | propagate | bench | phase-only");
        const std::string cmd = argv[1];
        const Args a(argc, argv, 2);
        if (cmd == "propagate") return cmd_propagate(a);
        if (cmd == "render") return cmd_render(a);
        if (cmd == "bench") return cmd_bench(a);
        if (cmd == "phase-only") return cmd_phase_only(a);
        throw HoloError("usage", "unknown subcommand: " + cmd);
    } catch (const HoloError& e) {
        std::cerr << "{\"error\":{\"kind\":" << jstr(e.kind) << ",\"message\":" << jstr(e.what()) << "}}\n";
        return (e.kind == "config" || e.kind == "usage") ? 2 : 1;
    } catch (const std::exception& e) {
        std::cerr << "{\"error\":{\"kind\":\"internal\",\"message\":" << jstr(e.what()) << "}}\n";
        return 1;
    }
}
