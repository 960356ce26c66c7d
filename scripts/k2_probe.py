"""K2 at the largest SDXL GN+SiLU site, inputs rotated over > 2x L2 (ncu target; development aid)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402

c, hw = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (320, 128)))
cl = torch.channels_last
g, b = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
sets = []
for _ in range(12):
    x = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
    sets.append((x, torch.empty_like(x), torch.zeros(2, c, device="cuda"), ops.groupnorm_workspace(x)))
for it in range(3):
    for x, y, add, ws in sets:
        ops.groupnorm_silu(x, g, b, out=y, add_nc=add, workspace=ws)
torch.cuda.synchronize()
