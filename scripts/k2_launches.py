"""K2 sites in a rotation, eager (ncu launch-list target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402
cl = torch.channels_last
for c, hw in [(320, 128), (1280, 32)]:
    g, b = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
    sets = []
    for _ in range(12 if hw == 128 else 48):
        x = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        sets.append((x, torch.empty_like(x), ops.groupnorm_workspace(x)))
    for it in range(2):
        for x, y, ws in sets:
            ops.groupnorm_silu(x, g, b, out=y, workspace=ws)
    torch.cuda.synchronize()
