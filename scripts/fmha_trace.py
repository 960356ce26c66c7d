"""Per-block timeline of CTA (0,0,0) of the K8 v2 kernel (SDB_FMHA_TRACE probe build): dev aid."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402
n, L, h = (2, 4096, 10) if len(sys.argv) < 2 else tuple(int(v) for v in sys.argv[1].split(","))
qkv = torch.randn(n, L, 3 * h * 64, device="cuda").to(torch.bfloat16)
for _ in range(3):
    o = ops.self_attention(qkv, h)
torch.cuda.synchronize()
t = o.view(-1).view(torch.int32)[1000000:1000000 + 6 * 64].cpu().tolist()
print("blk  S_ready  sm_done  P_full | S(j+1)_iss P(j)_seen PV(j)_iss   (clocks since CTA start)")
for j in range(min(64, L // int(os.environ.get("SDB_FMHA_BK", "64")))):
    e = t[6 * j:6 * j + 6]
    print(f"{j:3d} " + " ".join(f"{v:9d}" for v in e))
