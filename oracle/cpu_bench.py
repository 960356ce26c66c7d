"""CPU baseline timing of the reference path — TEST/BENCH INFRASTRUCTURE ONLY.

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm.
The reference's own CPU arithmetic for this path is the numpy LoRA merge
(addonsim/lora.py:84-104): when the unmodified reference is installed in
baseline/_ref (``pip install --target baseline/_ref``) its
``merge_in_place`` itself is timed, otherwise the bit-exact restatement
oracle/lora_ref.py.  The denoising loop has no reference implementation, so
its CPU cost is the builder-authored fp32 torch oracle (oracle/pipeline_ref.py),
kind "port".

One *sample* = one CFG half (batch 1: the uncond or the cond pass — the two
halves of a CFG batch-2 step cost the same) of one denoising step of UNet + n
ControlNets on the host cores, plus the reference LoRA merge of a
1/(2*steps) slice of the inventory at the stacked rank — exactly
1/(2*steps) of one image's CPU work, so images/s = 1 / (2 * steps * sample_s).
The merge slice is size-stratified (every k-th matrix of the inventory
sorted by size), so its cost scales to the whole inventory.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

from . import lora_ref
from . import pipeline_ref as R

_REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


def reference_lora():
    """The unmodified reference's lora module (baseline/_ref), or None."""
    if (_REF / "addonsim").exists() and str(_REF) not in sys.path:
        sys.path.insert(0, str(_REF))
    try:
        from addonsim import lora
        return lora
    except Exception:   # noqa: BLE001 — absent reference: the restatement is timed
        return None


def stratified(items: list, key, fraction_den: int, offset: int = 0) -> list:
    """Every fraction_den-th element of ``items`` sorted by ``key``."""
    order = sorted(items, key=key)
    return order[offset % fraction_den::fraction_den]


class MergeTimer:
    """Times the reference LoRA merge over a list of (h1, h2) shapes at rank r
    (weights and factors are synthetic uniform(-1, 1) like lora.bench_merge)."""

    def __init__(self, shapes, rank: int, seed: int = 0):
        self.shapes, self.rank = list(shapes), rank
        self.lora = reference_lora()
        self.kind = "reference" if self.lora is not None else "port"
        rng = np.random.default_rng(seed)
        self.data = []
        for h1, h2 in self.shapes:
            w = rng.uniform(-1, 1, (h1, h2)).astype(np.float32)
            d = rng.uniform(-1, 1, (h1, rank)).astype(np.float32)
            u = rng.uniform(-1, 1, (rank, h2)).astype(np.float32)
            self.data.append((w, d, u))

    @property
    def elements(self) -> int:
        return sum(h1 * h2 for h1, h2 in self.shapes)

    def run(self) -> float:
        t0 = time.perf_counter()
        for i, (w, d, u) in enumerate(self.data):
            if self.lora is not None:
                layer = self.lora.BaseLayer(w)
                adapter = self.lora.LowRankAdapter(f"a{i}", d, u, 1.0)
                self.lora.merge_in_place(layer, adapter)
            else:
                lora_ref.accumulate(w, d, u, 1.0, 1.0)
        return time.perf_counter() - t0


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
        self.x = torch.randn(1, 4, h, h, generator=g)
        self.ctx = torch.randn(1, cfg.context_len, cfg.context_dim, generator=g)
        self.hint = torch.randn(1, cfg.block_channels[0], h, h, generator=g) * 0.1
        self.add = torch.randn(1, cfg.time_embed_dim, generator=g) * 0.1 if cfg.addition_embed else None
        shapes = [(s[0], int(np.prod(s[1:]))) for _, s in self.matrices]
        self.merge_elems_total = sum(a * b for a, b in shapes)
        self.fraction = 2 * steps                       # a sample is 1/(2 steps) of an image
        self.merge = MergeTimer(stratified(shapes, lambda s: s[0] * s[1], self.fraction), lora_rank, seed)
        self._cursor = 0

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
        merge_s = self.merge.run() * self.merge_elems_total / (self.fraction * self.merge.elements)
        t2 = time.perf_counter()
        return {"step_half_s": t1 - t0, "merge_s": merge_s, "sample_s": (t1 - t0) + merge_s,
                "wall_s": t2 - t0}

    def images_per_s(self, sample_s: float) -> float:
        return 1.0 / (self.fraction * sample_s)

    def describe(self) -> str:
        return (f"1 CFG half (batch 1) of one {self.cfg.name} denoising step (UNet + {self.n_cn} ControlNets, "
                f"fp32 torch oracle, {torch.get_num_threads()} threads) + {self.merge.kind} numpy LoRA merge "
                f"(rank {self.rank}) of a size-stratified {len(self.merge.shapes)}/{len(self.matrices)}-matrix "
                f"slice scaled to 1/{self.fraction} of the inventory; x{self.fraction} = one image")
