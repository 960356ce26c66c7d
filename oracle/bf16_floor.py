"""Where the bf16 latent-error floor comes from — TEST INFRASTRUCTURE ONLY.

The north_star asks for per-step latents within rel-L2 1e-3 of the fp32
oracle in bf16.  This module measures, on the builder-authored oracle itself
(oracle/pipeline_ref.py, config 1: toy UNet + 1 ControlNet, 20 DDIM steps,
CFG 7.5), how far the latents move when bf16 rounding is applied at chosen
sites only, every other op staying fp32:

* one site: the UNet's final GroupNorm+SiLU output (conv_norm_out), i.e. the
  single bf16 tensor the output convolution reads;
* all linear outputs / all conv outputs / all norm outputs;
* every site (the bf16 emulator tests/ compare the device against).

If rounding ONE activation tensor to bf16 already exceeds 1e-3, no
implementation that stores any activation in bf16 can meet the gate: CFG
multiplies (eps_c - eps_u) by 7.5 and the DDIM update at high noise levels
amplifies eps errors by 1/sqrt(alpha_t).  Used by tests/test_bf16_floor.py
and scripts/bf16_floor.py (profiles/r02_bf16_floor.txt)."""

from __future__ import annotations

import torch
import torch.nn.functional as F

from . import pipeline_ref as R


def _rnd(t):
    return t.bfloat16().float()


class _SiteNet:
    """Mixin: round only where ``self.site(kind, name)`` says so."""

    def lin(self, n, x):
        y = F.linear(x, self.p[n + ".weight"], self.p.get(n + ".bias"))
        return _rnd(y) if self.site("lin", n) else y

    def conv(self, n, x, stride=1):
        w = self.p[n + ".weight"]
        y = F.conv2d(x, w, self.p.get(n + ".bias"), stride=stride, padding=w.shape[-1] // 2)
        return _rnd(y) if self.site("conv", n) else y

    def gn(self, n, x, silu, eps=None):
        y = F.group_norm(x, self.cfg.groups, self.p[n + ".weight"], self.p[n + ".bias"],
                         self.cfg.gn_eps if eps is None else eps)
        y = F.silu(y) if silu else y
        return _rnd(y) if self.site("gn", n) else y


def denoise_rounded(cfg, unet_p, cn_ps, req, cn_scales, steps, guidance, site) -> list:
    """pipeline_ref.denoise with bf16 rounding at the sites ``site(kind,
    name) -> bool`` selects (both networks; the UNet's eps stays fp32)."""
    class U(_SiteNet, R.RefUNet):
        pass

    class C(_SiteNet, R.RefControlNet):
        pass
    U.site = C.site = staticmethod(site)
    saved = R.RefUNet, R.RefControlNet
    R.RefUNet, R.RefControlNet = U, C
    try:
        return R.denoise(cfg, unet_p, cn_ps, req, cn_scales, steps, guidance)
    finally:
        R.RefUNet, R.RefControlNet = saved


SITES = {
    "conv_norm_out only": lambda k, n: n == "conv_norm_out",
    "all linear outputs": lambda k, n: k == "lin",
    "all conv outputs": lambda k, n: k == "conv" and n != "conv_out",
    "all norm outputs": lambda k, n: k == "gn",
    "every site": lambda k, n: n != "conv_out",
}


def floor_table(cfg, unet_p, cn_ps, req, cn_scales=(0.8,), steps=20, guidance=7.5, which=None) -> dict:
    ref = R.denoise(cfg, unet_p, cn_ps, req, list(cn_scales), steps, guidance)
    out = {}
    for label, site in SITES.items():
        if which is not None and label not in which:
            continue
        got = denoise_rounded(cfg, unet_p, cn_ps, req, list(cn_scales), steps, guidance, site)
        out[label] = [float((a.double() - b.double()).norm() / b.double().norm()) for a, b in zip(got, ref)]
    return out


def toy_inputs(seed: int = 0):
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.pipeline import synthetic_request
    cfg = U.TOY
    up = R.to_cpu_params(U.init_unet(cfg, "cpu", torch.float32, seed))
    cp = R.to_cpu_params(U.init_controlnet(cfg, "cpu", torch.float32, 1000 + seed))
    return cfg, up, [cp], synthetic_request(cfg, 1, seed=seed)
