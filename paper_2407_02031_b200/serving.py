"""Per-shape engine cache: the "decoupled CUDA graphs maintained in
standalone LRU caches, preventing out-of-memory errors" of the paper's
implementation.

A captured denoising step bakes in its shapes — CFG batch, latent resolution
— and pins its activation memory pool, so a server that sees several shapes
keeps one engine (static buffers + captured graphs) per shape and bounds how
many stay resident.  All engines share ONE weight set (and one LoRA shadow
copy): an engine costs only its activations and graphs, and evicting the
least recently used one returns that memory.  The reference has no graphs at
all (its 1.064 sub-multiplier, addonsim/model.py:70, stands for them).
"""

from __future__ import annotations

import dataclasses
from collections import OrderedDict
from typing import Callable, Optional, Sequence

import torch

from .pipeline import AddonPipeline, Request, SharedWeights
from .unet import UNetConfig, init_controlnet, init_unet


class LRUCache:
    """Key -> value with a capacity and an optional byte budget; values are
    built on a miss by ``factory(key)`` and released by ``release(value)``
    when evicted (least recently used first).  Host logic only."""

    def __init__(self, factory: Callable, capacity: int = 2, release: Optional[Callable] = None,
                 size_of: Optional[Callable] = None, budget_bytes: Optional[int] = None):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.factory, self.release, self.size_of = factory, release, size_of
        self.capacity, self.budget = capacity, budget_bytes
        self.items: "OrderedDict" = OrderedDict()
        self.hits = self.misses = self.evictions = 0

    def _bytes(self) -> int:
        return sum(self.size_of(v) for v in self.items.values()) if self.size_of else 0

    def get(self, key):
        if key in self.items:
            self.items.move_to_end(key)
            self.hits += 1
            return self.items[key]
        self.misses += 1
        # make room BEFORE building: the new engine's pool must not coexist with the victim's
        while len(self.items) >= self.capacity:
            self._evict()
        value = self.factory(key)
        self.items[key] = value
        while self.budget is not None and len(self.items) > 1 and self._bytes() > self.budget:
            self._evict()
        return value

    def _evict(self) -> None:
        _, victim = self.items.popitem(last=False)
        self.evictions += 1
        if self.release is not None:
            self.release(victim)

    def keys(self) -> list:
        return list(self.items)


class EngineCache:
    """AddonPipeline engines keyed by (batch, latent_hw) over one shared weight
    set, LRU-evicted; ``generate(req)`` picks (or captures) the engine of the
    request's shape.  The adapters of ``load_loras`` are re-applied to every
    engine built later, so a cached shape and a fresh one patch identically."""

    def __init__(self, cfg: UNetConfig, n_controlnets: int = 1, cn_scales: Optional[Sequence[float]] = None,
                 steps: int = 30, guidance: float = 7.5, device="cuda", dtype=torch.bfloat16, seed: int = 0,
                 capacity: int = 2, budget_bytes: Optional[int] = None):
        self.cfg, self.n_cn, self.cn_scales = cfg, n_controlnets, cn_scales
        self.steps, self.guidance, self.device, self.dtype = steps, guidance, torch.device(device), dtype
        self.weights = SharedWeights(init_unet(cfg, self.device, dtype, seed),
                                     [init_controlnet(cfg, self.device, dtype, seed=1000 + i)
                                      for i in range(n_controlnets)])
        self.adapters = None
        self.host_resident = False
        self.cache = LRUCache(self._build, capacity, release=self._release, size_of=self._footprint,
                              budget_bytes=budget_bytes)
        self.footprints: dict = {}

    def _build(self, key) -> AddonPipeline:
        batch, hw = key
        cfg = dataclasses.replace(self.cfg, latent_hw=hw) if hw != self.cfg.latent_hw else self.cfg
        before = torch.cuda.memory_allocated(self.device)
        eng = AddonPipeline(cfg, n_controlnets=self.n_cn, cn_scales=self.cn_scales, steps=self.steps,
                            guidance=self.guidance, device=self.device, dtype=self.dtype, batch=batch,
                            weights=self.weights)
        if self.adapters is not None:
            eng.load_loras(self.adapters, host_resident=self.host_resident)
        eng.setup()
        torch.cuda.synchronize(self.device)
        self.footprints[id(eng)] = torch.cuda.memory_allocated(self.device) - before
        return eng

    def _footprint(self, eng) -> int:
        return self.footprints.get(id(eng), 0)

    def _release(self, eng) -> None:
        torch.cuda.synchronize(self.device)
        self.footprints.pop(id(eng), None)
        eng.graphs.clear()
        eng.patch_graph = None
        eng.group_graphs = []
        eng.pool = None
        del eng
        torch.cuda.empty_cache()

    def load_loras(self, adapters, host_resident: bool = False) -> None:
        """Adapters for the next requests, applied to every resident engine
        (and to engines built later)."""
        self.adapters, self.host_resident = list(adapters), host_resident
        for eng in self.cache.items.values():
            eng.load_loras(self.adapters, host_resident=host_resident)

    def engine(self, batch: int, latent_hw: Optional[int] = None) -> AddonPipeline:
        return self.cache.get((batch, latent_hw or self.cfg.latent_hw))

    def generate(self, req: Request, patch: bool = False, boundary: Optional[int] = None,
                 pinned: Optional[dict] = None):
        lat = req.latent
        batch = 1 if lat.ndim == 3 else lat.shape[0]
        eng = self.engine(batch, lat.shape[-1])
        return eng.generate(req, patch=patch and self.adapters is not None, boundary=boundary, pinned=pinned)
