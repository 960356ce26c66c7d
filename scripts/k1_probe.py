"""One K1 launch over all 794 SDXL matrices for ncu (development aid).

  ncu ... python scripts/k1_probe.py <ranks e.g. 64 or 8,32,64,128> <mode 0|1|2>
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402
from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.patcher import PatchSet, allocate_shadow, synthetic_lora  # noqa: E402

ranks = [int(r) for r in sys.argv[1].split(",")]
mode = int(sys.argv[2])
p = U.init_unet(U.SDXL, "cuda", torch.bfloat16, 0)
shadow = allocate_shadow(p)
ads = [(synthetic_lora(p, r, seed=i, adapter_id=f"a{i}"), 0.5) for i, r in enumerate(ranks)]
with ops.lora_kernel_mode(mode):
    ps = PatchSet(p, ads, shadow=shadow)
ps.launch()
torch.cuda.synchronize()
ps.launch()
torch.cuda.synchronize()
