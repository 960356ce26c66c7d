"""One prepare() of the headline engine under the profiler (launch list)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.caas import LoopbackGroup  # noqa: E402
from paper_2407_02031_b200.pipeline import synthetic_batch  # noqa: E402

eng = LoopbackGroup(U.SDXL, 2, [0.8, 0.6], steps=30, dtype=torch.bfloat16, seed=0, concurrent=True)
eng.setup()
req = synthetic_batch(U.SDXL, 2, 1)
dev = dict(latent=torch.from_numpy(req.latent).cuda(), context=torch.from_numpy(req.context).cuda(),
           images=[torch.from_numpy(i).cuda() for i in req.images],
           pooled=torch.from_numpy(req.pooled).cuda(), time_ids=torch.from_numpy(req.time_ids).cuda())
eng.prepare(**dev)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.prepare(**dev)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
