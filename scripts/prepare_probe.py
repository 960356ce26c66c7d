"""Per-image time split on the headline engine (LoopbackGroup, SDXL, 2 CNs):
prepare() (hint embeddings, added-cond embeddings, K|V cache) vs the 30
denoising steps, device-timed."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.caas import LoopbackGroup  # noqa: E402
from paper_2407_02031_b200.patcher import synthetic_lora  # noqa: E402
from paper_2407_02031_b200.pipeline import synthetic_batch  # noqa: E402

cfg = U.SDXL
eng = LoopbackGroup(cfg, 2, [0.8, 0.6], steps=30, guidance=7.5, dtype=torch.bfloat16, seed=0, concurrent=True)
pipe = eng.base.pipe
eng.load_loras([(synthetic_lora(pipe.unet_p, 64, seed=10 + i), 0.7) for i in range(2)], host_resident=True)
eng.setup()
req = synthetic_batch(cfg, 2, 1)
dev = dict(latent=torch.from_numpy(req.latent).cuda(), context=torch.from_numpy(req.context).cuda(),
           images=[torch.from_numpy(i).cuda() for i in req.images],
           pooled=torch.from_numpy(req.pooled).cuda(), time_ids=torch.from_numpy(req.time_ids).cuda())
s = eng.main_stream
with torch.cuda.stream(s):
    eng.prepare(**dev)
    eng.denoise(patch=False)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for rep in range(3):
        ev[0].record(s)
        eng.prepare(**dev)
        ev[1].record(s)
        eng.denoise(patch=False)
        ev[2].record(s)
        ev[2].synchronize()
        print(f"prepare {ev[0].elapsed_time(ev[1]):.2f} ms, 30 steps {ev[1].elapsed_time(ev[2]):.1f} ms")
