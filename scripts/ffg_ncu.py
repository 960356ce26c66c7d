"""One K5' launch at the SDXL 32x32-level shape for ncu (dev aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

m, k, f = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else (2048, 1280, 5120))]
x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
w = (torch.randn(2 * f, k, device="cuda") * 0.03).to(torch.bfloat16)
b = torch.randn(2 * f, device="cuda")
for _ in range(3):
    ops.ff_geglu(x, w, b)
torch.cuda.synchronize()
