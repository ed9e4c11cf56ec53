"""The C++ drop-in (include/holo/*.hpp -> libholo.so -> libholo_cuda.so).

GPU: runs tests/cpp/test_dropin.cpp and -- compiled against the drop-in headers
by paper_2506_08350_b200/cpp/Makefile where /root/reference exists -- the
reference's OWN unit tests test_field.cpp, test_propagation.cpp,
test_losses.cpp, test_optimizer.cpp and test_phase_only.cpp, unmodified, at the
reference's tolerances (f64 operators, losses, optimizer and phase-only
conversion on the GPU), and test_pipeline.cpp / test_rasterizer.cpp with the
cases an fp32 render cannot meet allow-listed below, each with its reason.
CPU: libholo.so exports the reference API symbols."""
import os
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2506_08350_b200", "lib")


def test_libholo_exports_reference_api():
    so = os.path.join(LIB, "libholo.so")
    assert os.path.exists(so), "build with __graft_entry__.build()"
    syms = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True).stdout
    for name in ("holo::pipeline_forward(", "holo::raster_forward(", "holo::propagate(", "holo::forward_record(",
                 "holo::inverse_propagate(", "holo::transfer_function(", "holo::fft2(", "holo::ifft2(",
                 "holo::intensity(", "holo::plane_positions(", "holo::read_field(", "holo::write_field(",
                 "holo::total_loss(", "holo::loss_recon(", "holo::loss_ssim(", "holo::ssim_mean(", "holo::psnr(",
                 "holo::optimizer_step(", "holo::convert_phase_only(", "holo::phase_only_loss(",
                 "holo::make_target_from_scene(", "holo::brute_force_forward(", "holo::detail::project_gaussian("):
        assert name in syms, name


# test_pipeline.cpp's two finite-difference cases difference the loss with
# h = 1e-5 through the full render; the render computes in fp32 (the north star's
# precision), so the central difference is dominated by fp32 rounding of the loss
# and those two cases cannot pass.  Every other case of the
# file runs and must pass.
#
# test_rasterizer.cpp: four cases compare composited fp32 values with hand-derived
# f64 values at 1e-12 (1e-10 for t_final) -- below fp32's 6e-8 resolution -- and
# fail for the fp32 compositing the north star prescribes; the same KATs pass at
# fp32 tolerance in tests/test_gpu_render.py (blending, stacking, tie order, the
# pinhole centre).  The other seven, among them "tiled pass equals brute force
# bitwise when termination is off", "outputs are bitwise stable across thread
# counts", culling, plane routing and the clamp, pass unmodified.
EXPECTED_FAILURES = {
    "ref_test_pipeline": {"end-to-end gradients match finite differences",
                          "soft assignment exposes plane logit gradients to finite differences"},
    "ref_test_rasterizer": {"one gaussian lands where the pinhole model says",
                            "blending recurrence matches the hand-computed cases",
                            "stacked gaussians composite front to back",
                            "equal depths break ties by index"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("binary,cases", [("ref_test_pipeline", 11), ("ref_test_rasterizer", 11)])
def test_reference_suite_with_fp32_allowlist(binary, cases, tmp_path):
    path = os.path.join(LIB, binary)
    if not os.path.exists(path):
        pytest.skip(f"{binary} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, cwd=tmp_path, timeout=900)
    failed = {line.split("test case FAILED:", 1)[1].strip() for line in r.stdout.splitlines()
              if "test case FAILED:" in line}
    print(r.stdout[-6000:])
    assert failed <= EXPECTED_FAILURES[binary], failed
    assert f"test cases: {cases}" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("binary", ["test_dropin", "ref_test_field", "ref_test_propagation", "ref_test_losses",
                                    "ref_test_optimizer", "ref_test_phase_only"])
def test_cpp_suite(binary, tmp_path):
    path = os.path.join(LIB, binary)
    if not os.path.exists(path):
        pytest.skip(f"{binary} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, cwd=tmp_path, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "failed: 0;" in r.stdout
