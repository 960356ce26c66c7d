"""Measured B200 stage times as a reference-format LatencyProfile.

The reference's latency model (addonsim/model.py:28-111 ``LatencyProfile``,
``PROFILES = {"paper-h800-sdxl": ...}`` :115-117) carries the paper's H800
stage constants.  This module measures the same stages on a B200 with the
real kernels — UNet encoder+mid, UNet decoder, one ControlNet, the residual
transfer, the K1 patch — using the ControlNet-as-a-service compute split
(caas.LoopbackGroup, whose graphs are exactly the per-stage graphs of the
multi-GPU path), and writes them as a ``LatencyProfile`` so the reference's
own policy arithmetic (serial vs parallel step latency, Gustafson bound,
patch planning) reports B200 numbers.

    python -m paper_2407_02031_b200.profile [--out profiles/b200_sdxl_profile.json]
"""

from __future__ import annotations

import argparse
import json
from dataclasses import asdict
from pathlib import Path

import torch

from .schedule import LatencyProfile

DEFAULT_PATH = Path(__file__).resolve().parent.parent / "profiles" / "b200_sdxl_profile.json"
# measured peer copy per direction on this pool's NVLink 5 (B200_PROFILING.md); the
# 1-GPU box cannot time a real transfer, so the link term uses this figure
NVLINK_GBPS = 770.0
NVLINK_LATENCY_MS = 0.02


def _time(fn, reps: int = 5) -> float:
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def measure(cfg_name: str = "sdxl", lora_ranks=(64, 64), steps_reference: int = 30) -> dict:
    from . import unet as U
    from .caas import LoopbackGroup
    from .patcher import synthetic_lora
    from .pipeline import synthetic_request

    cfg = U.CONFIGS[cfg_name]
    grp = LoopbackGroup(cfg, 1, [0.8], steps=steps_reference, dtype=torch.bfloat16, seed=0)
    grp.load_loras([(synthetic_lora(grp.base.pipe.unet_p, r, seed=10 + i), 0.7) for i, r in enumerate(lora_ranks)])
    grp.setup()
    req = synthetic_request(cfg, 1)
    grp.prepare(torch.from_numpy(req.latent), torch.from_numpy(req.context),
                [torch.from_numpy(i) for i in req.images],
                torch.from_numpy(req.pooled) if req.pooled is not None else None,
                torch.from_numpy(req.time_ids) if req.time_ids is not None else None)
    base, svc = grp.base, grp.services[0]
    enc = _time(lambda: base.base_encode("pristine"))
    dec = _time(lambda: base.base_decode("pristine"))
    cn = _time(svc.service_step)
    p = base.pipe
    patch = _time(lambda: p.patchset.launch(stream=torch.cuda.current_stream()), reps=3)
    payload_mib = base.flats[0].numel() * base.flats[0].element_size() / 2 ** 20
    step = enc + dec
    prof = LatencyProfile(
        unet_total_ms=step * steps_reference, steps_reference=steps_reference,
        encoder_mid_fraction=enc / step, controlnet_factor=cn / enc,
        comm_payload_mib=payload_mib, link_gibps=NVLINK_GBPS * 1e9 / 2 ** 30, link_latency_ms=NVLINK_LATENCY_MS,
        patch_inplace_ms=patch, unet_opt_multiplier=1.0,
    ).validate()
    return {"profile": asdict(prof),
            "measured_ms": {"unet_encoder_mid": enc, "unet_decoder": dec, "controlnet": cn, "lora_patch": patch},
            "config": {"model": cfg_name, "cfg_batch": 2, "latent": cfg.latent_hw, "lora_ranks": list(lora_ranks),
                       "link": f"assumed {NVLINK_GBPS} GB/s per direction (not measurable on a 1-GPU box)"}}


def load(path: Path = DEFAULT_PATH):
    """The committed measurement as a LatencyProfile (None if absent)."""
    if not Path(path).exists():
        return None
    d = json.loads(Path(path).read_text())["profile"]
    d["unet_opt_submultipliers"] = tuple(d["unet_opt_submultipliers"])
    return LatencyProfile(**d).validate()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(DEFAULT_PATH))
    ap.add_argument("--config", default="sdxl")
    args = ap.parse_args()
    res = measure(args.config)
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
