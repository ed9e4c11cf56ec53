"""B200-native forward renderer for complex-valued holographic radiance fields
(arXiv 2506.08350): drop-in for the reference's render path
(proj/src/pipeline.cpp:20-29) on hand-written sm_100a kernels, with its
gradient (raster_backward, the adjoint propagation) and the training step
(total_loss, optimizer_step) around it.

The compute lives in ``lib/libholo_cuda.so`` (C-ABI: include/holo_cuda.h); this
package is the thin host side mirroring the reference API.
"""
from ._lib import HoloError  # noqa: F401
from .holotypes import (CameraView, GaussianScene, LossBreakdown, OptimizerConfig, PipelineForward,  # noqa: F401
                        PipelineOptions, PropagationOptions, RasterForward, RenderSettings, WaveConfig,
                        plane_positions)

__all__ = ["HoloError", "CameraView", "GaussianScene", "LossBreakdown", "OptimizerConfig", "PipelineForward",
           "PipelineOptions", "PropagationOptions", "RasterForward", "RenderSettings", "WaveConfig",
           "plane_positions"]
