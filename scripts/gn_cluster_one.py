"""One cluster-form GroupNorm launch per shape (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

for n, c, h in ((2, 1280, 32),):
    x = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    gamma = torch.rand(c, device="cuda") + 0.5
    beta = torch.randn(c, device="cuda")
    for _ in range(2):
        ops.groupnorm_silu(x, gamma, beta, 32, 1e-5, True)
    torch.cuda.synchronize()
