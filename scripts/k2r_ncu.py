"""Eager launches of K2's resident form (mode 4) for ncu (dev aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

n, c, h, w = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else (2, 320, 128, 128))]
x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
y = torch.empty_like(x)
gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
ws = ops.groupnorm_workspace(x)
for _ in range(3):
    with ops.groupnorm_mode(4):
        ops.groupnorm_silu(x, gm, bt, out=y, workspace=ws)
torch.cuda.synchronize()
