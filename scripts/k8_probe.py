import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402
n, L, h = (2, 1024, 20) if len(sys.argv) < 2 else tuple(int(x) for x in sys.argv[1].split(","))
qkv = torch.randn(n, L, 3 * h * 64, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.self_attention(qkv, h)
torch.cuda.synchronize()
