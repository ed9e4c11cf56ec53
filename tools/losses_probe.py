"""One holo_losses call (with dL/dI) on C3-sized f64 stacks, for an ncu launch list."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2506_08350_b200.api import Context  # noqa: E402
from paper_2506_08350_b200.holotypes import PipelineOptions  # noqa: E402

L_, C_, H, W = 8, 3, 1080, 1920
g = torch.Generator(device="cuda").manual_seed(0)
I = torch.rand((L_, C_, H, W), dtype=torch.float64, device="cuda", generator=g)
G = torch.rand((L_, C_, H, W), dtype=torch.float64, device="cuda", generator=g)
M = (torch.rand((L_, H, W), dtype=torch.float64, device="cuda", generator=g) > 0.7).double()
ctx = Context(0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    b, _ = ctx.losses(I, G, M, PipelineOptions())
torch.cuda.synchronize()
print(b)
