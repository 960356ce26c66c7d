"""K2 / K5 / K6 at their largest SDXL shapes, for ncu (development aid)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402


def main():
    cl = torch.channels_last
    x = torch.randn(2, 320, 128, 128, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
    g, b = torch.ones(320, device="cuda"), torch.zeros(320, device="cuda")
    add = torch.zeros(2, 320, device="cuda")
    ws = ops.groupnorm_workspace(x)
    y = torch.empty_like(x)
    tok = torch.randn(2, 4096, 640, device="cuda").to(torch.bfloat16)
    d = torch.randn_like(tok)
    lw, lb = torch.ones(640, device="cuda", dtype=torch.bfloat16), torch.zeros(640, device="cuda", dtype=torch.bfloat16)
    proj = torch.randn(2, 4096, 5120, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        ops.groupnorm_silu(x, g, b, out=y, add_nc=add, workspace=ws)
        ops.add_layernorm(tok, d, lw, lb)
        ops.geglu(proj)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
