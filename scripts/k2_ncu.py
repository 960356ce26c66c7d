"""One eager launch of each K2 form at [2,320,128,128] for ncu (dev aid):
two-pass GN+SiLU (+temb): gn_stats_kernel + gn_apply_kernel; K3 with fused
statistics (inject_gn_kernel); the apply alone after it."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

cl = torch.channels_last
n, c, h, w = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else (2, 320, 128, 128))]
x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
y = torch.empty_like(x)
gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
add = torch.randn(n, c, device="cuda")
ws = ops.groupnorm_workspace(x)
rs = torch.randn_like(x)
out = torch.empty_like(x)
ws2 = ops.groupnorm_workspace(x)
for _ in range(2):
    with ops.groupnorm_mode(1):
        ops.groupnorm_silu(x, gm, bt, out=y, add_nc=add, workspace=ws)
    h0 = ops.residual_inject(x, [rs], [0.8], out=out, gn_workspace=ws2)
    ops.groupnorm_silu(h0, gm, bt, out=y)
torch.cuda.synchronize()
