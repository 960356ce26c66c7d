"""K6 at the SDXL shapes (ncu launch-list target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402
for m, c in [(2048, 1280), (8192, 640)]:
    sets = []
    for _ in range(16):
        x = torch.randn(m, c, device="cuda").to(torch.bfloat16)
        sets.append((x, torch.randn_like(x)))
    w = torch.ones(c, device="cuda", dtype=torch.bfloat16)
    b = torch.zeros(c, device="cuda", dtype=torch.bfloat16)
    for it in range(2):
        for x, d in sets:
            ops.add_layernorm(x, d, w, b)
    torch.cuda.synchronize()
