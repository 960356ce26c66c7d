"""One eager launch of each K2 form at the given shapes for ncu (dev aid):
two-pass (gn_stats_kernel + gn_apply_kernel, mode 1) and the streamed
cluster form (gn_stream_kernel, mode 3), both with the temb add."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

for arg in sys.argv[1:] or ["2,320,128,128"]:
    n, c, h, w = [int(v) for v in arg.split(",")]
    x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    y = torch.empty_like(x)
    gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
    add = torch.randn(n, c, device="cuda")
    ws = ops.groupnorm_workspace(x)
    for mode in (1, 3):
        with ops.groupnorm_mode(mode):
            for _ in range(2):
                ops.groupnorm_silu(x, gm, bt, out=y, add_nc=add, workspace=ws)
    torch.cuda.synchronize()
