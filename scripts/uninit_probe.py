"""Debug aid: does the fp32 SDXL engine read uninitialised memory?  Runs the
config-3 engine (2 steps) in a fresh allocator and again after the caching
allocator was filled with NaN; any difference means a buffer is consumed
before it is written."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.caas import LoopbackGroup  # noqa: E402
from paper_2407_02031_b200.patcher import synthetic_lora  # noqa: E402
from paper_2407_02031_b200.pipeline import AddonPipeline, synthetic_request  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
dtype = torch.float32 if len(sys.argv) < 2 else getattr(torch, sys.argv[1])
cfg = U.SDXL if len(sys.argv) < 3 else U.CONFIGS[sys.argv[2]]


def run(kind, patch):
    if kind in ("loop", "loopserial"):
        eng = LoopbackGroup(cfg, 2, [0.8, 0.6], steps=2, dtype=dtype, seed=0, concurrent=kind == "loop")
        unet_p = eng.base.pipe.unet_p
    else:
        eng = AddonPipeline(cfg, n_controlnets=2, cn_scales=[0.8, 0.6], steps=2, dtype=dtype, seed=0)
        unet_p = eng.unet_p
    if patch:
        eng.load_loras([(synthetic_lora(unet_p, 64, seed=10 + i), 0.7) for i in range(2)], host_resident=True)
    eng.setup()
    req = synthetic_request(cfg, 2, seed=0)
    dev = dict(latent=torch.from_numpy(req.latent).cuda(), context=torch.from_numpy(req.context).cuda(),
               images=[torch.from_numpy(i).cuda() for i in req.images])
    if req.pooled is not None:
        dev.update(pooled=torch.from_numpy(req.pooled).cuda(), time_ids=torch.from_numpy(req.time_ids).cuda())
    out = []
    eng.prepare(**dev)
    eng.denoise(patch=patch, boundary=1, on_step=lambda s, x: out.append(x.float().cpu().clone()))
    torch.cuda.synchronize()
    del eng
    torch.cuda.empty_cache()
    return out


kinds = sys.argv[3].split(",") if len(sys.argv) > 3 else ["loop", "pipe"]
for kind in kinds:
    for patch in (False, True):
        a = run(kind, patch)
        g = torch.full(((60 << 30) // 4,), float("nan"), device="cuda")
        del g                                   # the allocator keeps the NaN-filled blocks
        b = run(kind, patch)
        d = [float((x - y).abs().max()) for x, y in zip(a, b)]
        print(f"{kind} patch={patch} dtype={dtype}: fresh-vs-reused max|d| per step {d} "
              f"finite={[bool(torch.isfinite(y).all()) for y in b]}", flush=True)
        torch.cuda.empty_cache()
