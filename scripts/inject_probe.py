"""K3 with GroupNorm statistics (inject_gn) vs plain K3 at SDXL resnet-output shapes (ncu target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402
cl = torch.channels_last
for c, hw in [(640, 64), (1280, 32)]:
    sets = []
    for _ in range(16):
        h = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        sc = torch.randn_like(h)
        sets.append((h, sc, ops.groupnorm_workspace(h), torch.zeros(c, device="cuda")))
    for it in range(2):
        for h, sc, ws, b in sets:
            ops.residual_inject(h, [sc], [1.0], skip_bias=b, gn_workspace=ws)
        for h, sc, ws, b in sets:
            ops.residual_inject(h, [sc], [1.0], skip_bias=b)
    torch.cuda.synchronize()
