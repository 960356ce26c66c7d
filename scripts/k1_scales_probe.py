"""K1 over all 794 SDXL matrices: equal vs distinct adapter scales (the
distinct case packs hi/lo K-blocks for the folded sources).  Prints ms and
algorithmic GB/s per launch (CUDA events, 10 back-to-back launches; W is
5.1 GB, far above L2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.patcher import PatchSet, allocate_shadow, synthetic_lora  # noqa: E402

p = U.init_unet(U.SDXL, "cuda", torch.bfloat16, 0)
shadow = allocate_shadow(p)
for ranks, scales in [((64, 64), (0.7, 0.7)), ((8, 32, 64, 128), (0.7,) * 4),
                      ((8, 32, 64, 128), (0.9, 0.55, 0.35, 1.3)), ((64, 64), (0.7, 0.5))]:
    ads = [(synthetic_lora(p, r, seed=i, adapter_id=f"a{i}"), s) for i, (r, s) in enumerate(zip(ranks, scales))]
    ps = PatchSet(p, ads, shadow=shadow)
    ps.launch()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        ps.launch()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"ranks={ranks} scales={scales}: {ms:.3f} ms  {ps.alg_bytes / ms / 1e6:.0f} GB/s  "
          f"kernel={ps.plan.kernel}", flush=True)
    del ps, ads
    torch.cuda.empty_cache()
