"""CPU baseline timing of the reference path — TEST/BENCH INFRASTRUCTURE ONLY.

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm.
The reference's own CPU arithmetic for this path is the numpy LoRA merge
(addonsim/lora.py:84-95), restated bit-exactly in oracle/lora_ref.py; the
denoising loop has no reference implementation, so its CPU cost is the
builder-authored fp32 torch oracle (oracle/pipeline_ref.py), kind "port".

One *sample* = one SDXL denoising step of UNet + n ControlNets at CFG batch 2
on the host cores, plus the reference LoRA merge of the matrices that fall in
a 1/steps slice of the SDXL inventory at the stacked rank — i.e. exactly
1/steps of one image's CPU work, so images/s = 1 / (steps * sample_s).
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import lora_ref
from . import pipeline_ref as R


class CpuWorkload:
    def __init__(self, cfg, n_cn: int, lora_rank: int, steps: int, seed: int = 0):
        torch.set_num_threads(os.cpu_count() or 1)
        self.cfg, self.n_cn, self.rank, self.steps = cfg, n_cn, lora_rank, steps
        from paper_2407_02031_b200 import unet as U  # layout only (meta device), no kernels
        meta_u = U.init_unet(cfg, device="meta", dtype=torch.float32)
        meta_c = U.init_controlnet(cfg, device="meta", dtype=torch.float32)
        self.matrices = [(n, tuple(meta_u.t[n + ".weight"].shape)) for n, _ in meta_u.matrices]
        self.unet = R.RefUNet(cfg, self._materialise(meta_u))
        cn_p = self._materialise(meta_c)  # ControlNets share values; timing does not depend on them
        self.cns = [R.RefControlNet(cfg, cn_p) for _ in range(n_cn)]
        h = cfg.latent_hw
        g = torch.Generator().manual_seed(seed)
        self.x = torch.randn(2, 4, h, h, generator=g)
        self.ctx = torch.randn(2, cfg.context_len, cfg.context_dim, generator=g)
        self.hint = torch.randn(2, cfg.block_channels[0], h, h, generator=g) * 0.1
        self.add = torch.randn(2, cfg.time_embed_dim, generator=g) * 0.1 if cfg.addition_embed else None
        rng = np.random.default_rng(seed)
        # the 1/steps slice of the inventory merged per sample
        order = rng.permutation(len(self.matrices))
        self.merge_slice = [self.matrices[i] for i in order[: max(1, len(order) // steps)]]
        self.merge_elems_total = sum(int(np.prod(s[:1])) * int(np.prod(s[1:])) for _, s in self.matrices)
        self.merge_elems_slice = sum(int(np.prod(s[:1])) * int(np.prod(s[1:])) for _, s in self.merge_slice)
        self.factors = [(rng.standard_normal((h1, lora_rank), dtype=np.float32),
                         rng.standard_normal((lora_rank, int(np.prod(rest))), dtype=np.float32))
                        for _, (h1, *rest) in self.merge_slice]

    @staticmethod
    def _materialise(meta) -> dict:
        out = {}
        for k, v in meta.t.items():
            t = torch.empty(v.shape, dtype=torch.float32)
            if k.endswith(".weight") and v.dim() >= 2:
                t.uniform_(-0.03, 0.03)
            elif "norm" in k and k.endswith(".weight"):
                t.fill_(1.0)
            else:
                t.zero_()
            out[k] = t
        return out

    def sample(self) -> dict:
        """Run one sample; returns its wall seconds split into parts."""
        t0 = time.perf_counter()
        with torch.inference_mode():
            res = [cn.forward(self.x, 500, self.ctx, self.hint, self.add) for cn in self.cns]
            self.unet.forward(self.x, 500, self.ctx, self.add, res, [0.8] * self.n_cn)
        t1 = time.perf_counter()
        for d, u in self.factors:
            w = np.zeros((d.shape[0], u.shape[1]), np.float32)
            lora_ref.accumulate(w, d, u, 1.0, 1.0)
        t2 = time.perf_counter()
        return {"step_s": t1 - t0, "merge_s": t2 - t1, "sample_s": t2 - t0}

    def describe(self) -> str:
        return (f"1 {self.cfg.name} denoising step (UNet + {self.n_cn} ControlNets, CFG batch 2, fp32 torch "
                f"oracle) + reference numpy LoRA merge (rank {self.rank}) of {len(self.merge_slice)}/"
                f"{len(self.matrices)} matrices; x{self.steps} = one image")
