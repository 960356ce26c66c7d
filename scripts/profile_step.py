"""Profiling driver for ncu (development aid).

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... \
      python scripts/profile_step.py [--steps 1] [--what step|patch|all]

Builds the bench workload (SDXL + 2 ControlNets + 2 LoRAs r64), warms up,
then opens the profiler range around: one K1 patch launch and N denoising
steps (eager, so every kernel is its own launch).
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.patcher import synthetic_lora  # noqa: E402
from paper_2407_02031_b200.pipeline import AddonPipeline, synthetic_request  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--what", default="all")
    ap.add_argument("--config", default="sdxl")
    ap.add_argument("--ranks", default="64,64")
    args = ap.parse_args()
    cfg = U.CONFIGS[args.config]
    pipe = AddonPipeline(cfg, n_controlnets=2, steps=30, dtype=torch.bfloat16, use_graphs=False)
    ranks = [int(r) for r in args.ranks.split(",")]
    pipe.load_loras([(synthetic_lora(pipe.unet_p, r, seed=10 + i), 0.7) for i, r in enumerate(ranks)])
    req = synthetic_request(cfg, 2)
    pipe.prepare(torch.from_numpy(req.latent), torch.from_numpy(req.context),
                 [torch.from_numpy(i) for i in req.images],
                 torch.from_numpy(req.pooled) if req.pooled is not None else None,
                 torch.from_numpy(req.time_ids) if req.time_ids is not None else None)
    pipe.step_once()
    pipe.patchset.launch()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    if args.what in ("patch", "all"):
        pipe.patchset.launch()
    if args.what in ("step", "all"):
        for _ in range(args.steps):
            pipe.step_once()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
