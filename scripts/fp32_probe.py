"""Debug aid: fp32 SDXL engine (LoopbackGroup, concurrent) step-1 latent
under cuDNN's default algorithm choice, cudnn.deterministic, and cuDNN off,
against the CPU fp32 oracle's step 1 (one-step run of a 2-step schedule)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from oracle import pipeline_ref as R  # noqa: E402
from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.caas import LoopbackGroup  # noqa: E402
from paper_2407_02031_b200.pipeline import synthetic_request  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
cfg = U.SDXL
req = synthetic_request(cfg, 2, seed=0)


def run():
    eng = LoopbackGroup(cfg, 2, [0.8, 0.6], steps=2, dtype=torch.float32, seed=0, concurrent=True)
    eng.setup()
    dev = dict(latent=torch.from_numpy(req.latent).cuda(), context=torch.from_numpy(req.context).cuda(),
               images=[torch.from_numpy(i).cuda() for i in req.images],
               pooled=torch.from_numpy(req.pooled).cuda(), time_ids=torch.from_numpy(req.time_ids).cuda())
    out = []
    eng.prepare(**dev)
    eng.denoise(on_step=lambda s, x: out.append(x.float().cpu().clone()))
    torch.cuda.synchronize()
    up = R.to_cpu_params(eng.base.pipe.unet_p)
    del eng
    torch.cuda.empty_cache()
    return out[0], up


res = {}
for mode in ("default", "deterministic", "default_again"):
    torch.backends.cudnn.deterministic = mode == "deterministic"
    torch.backends.cudnn.enabled = mode != "nocudnn"
    res[mode], up = run()
    print(mode, "done", flush=True)
cps = [R.to_cpu_params(U.init_controlnet(cfg, "cuda", torch.float32, seed=1000 + i)) for i in range(2)]
ref = R.denoise(cfg, up, cps, req, [0.8, 0.6], 2, 7.5, max_steps=1)[0]
rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm())
for k, v in res.items():
    print(f"{k}: vs oracle {rel(v, ref):.3e}  vs default {rel(v, res['default']):.3e}", flush=True)
