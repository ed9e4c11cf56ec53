"""With a HOLO_COUNT build (EXTRA_NVFLAGS=-DHOLO_COUNT): print the compositing
kernel's hit statistics for one C3 frame -- warp-level hits walked, hits where some
lane accepts, and entries passing the accept-box test."""
import ctypes
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200 import _lib as L  # noqa: E402
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.scenes import CONFIGS, synthetic_scene  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
wave, cam = c.wave(), c.cameras()[0]
ctx = Context(0)
ctx.upload_scene(synthetic_scene(c.n, wave, c.seed))
ctx.render(cam, wave, outputs=L.OUT_HOLOGRAM)
ctx.synchronize()
ctypes.CDLL(None).fflush(None)
