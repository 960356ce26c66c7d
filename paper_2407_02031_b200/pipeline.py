"""The per-step denoising loop with ControlNet residual injection, CFG and the
asynchronous LoRA patch — the path the north_star names, on one GPU.

What the reference models (addonsim/orchestrator.py, virtual clock) and where
it is real here:

* step = ControlNets then UNet encoder/decoder (serial mode,
  orchestrator.py:611-619 ``_run_plain_step``); ControlNet outputs are summed
  into the skips/mid by K3 with their conditioning scales; the
  decoder consumes them after every branch finished (orchestrator.py:652-653).
  The multi-GPU service mode (``_run_parallel_step`` :621-660) is caas.py.
* CFG: one batch of 2 ([uncond; cond]); K4 fuses guidance + DDIM update +
  re-batching of the next UNet input, and advances the device step counter,
  so each step replays as ONE CUDA graph with no host work in between.
* async LoRA (orchestrator.py:509-528, 698-719): the whole
  adapter set is patched by one K1 launch into shadow weights on a
  low-priority side stream while steps 1..k run; step k+1 onward replays the
  graph captured on the shadow weights after waiting on the patch event.
  k comes from ``schedule.plan_lora_patch`` with the measured patch time as
  the "load" (deterministic; parity tests force it).  Unpatch = switch back
  to the pristine graph (exact).

Latents are NHWC end to end (the fp32 master latent is [H, W, 4] flat).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import ops
from .patcher import AdapterBank, PatchSet, UNetLora, allocate_shadow, split_patch_groups
from .scheduler import ddim_tables
from .schedule import plan_lora_patch, plan_pipeline_patch
from .unet import ControlNet, UNet, UNetConfig, init_controlnet, init_unet


@dataclass
class Request:
    """Host-side inputs of one image — or of a serving batch of B images —
    with the CFG batch laid out [uncond x B; cond x B] (B = 1: [uncond; cond])."""

    latent: np.ndarray          # [4, H, W] (or [B, 4, H, W]) float32 initial noise
    context: np.ndarray         # [2B, ctx_len, ctx_dim] float32 text embeddings
    images: list                # per ControlNet: [2B, 3, 8H, 8W] float32 in [0, 1]
    pooled: Optional[np.ndarray] = None    # [2B, 1280] (SDXL)
    time_ids: Optional[np.ndarray] = None  # [2B, 6]    (SDXL)

    def nbytes(self) -> int:
        n = self.latent.nbytes + self.context.nbytes + sum(i.nbytes for i in self.images)
        n += self.pooled.nbytes if self.pooled is not None else 0
        n += self.time_ids.nbytes if self.time_ids is not None else 0
        return n


def synthetic_request(cfg: UNetConfig, n_controlnets: int, seed: int = 0) -> Request:
    """Seeds as SURVEY §8d: latents 1, control image 2, text 3 (offset by seed)."""
    h = cfg.latent_hw
    lat = np.random.default_rng(1 + seed).standard_normal((4, h, h)).astype(np.float32)
    ctx = np.random.default_rng(3 + seed).standard_normal((2, cfg.context_len, cfg.context_dim)).astype(np.float32)
    imgs = [np.random.default_rng(2 + seed + 17 * i).uniform(0, 1, (2, 3, 8 * h, 8 * h)).astype(np.float32)
            for i in range(n_controlnets)]
    pooled = time_ids = None
    if cfg.addition_embed:
        pooled = np.random.default_rng(4 + seed).standard_normal((2, cfg.pooled_dim)).astype(np.float32)
        px = 8 * h
        time_ids = np.array([[px, px, 0, 0, px, px]] * 2, dtype=np.float32)
    return Request(lat, ctx, imgs, pooled, time_ids)


def synthetic_batch(cfg: UNetConfig, n_controlnets: int, batch: int, seed: int = 0) -> Request:
    """B independent images (image i = synthetic_request(seed + 1000 i)) in
    the batched CFG layout [uncond_0 .. uncond_B-1, cond_0 .. cond_B-1]."""
    reqs = [synthetic_request(cfg, n_controlnets, seed + 1000 * i) for i in range(batch)]
    if batch == 1:
        return reqs[0]

    def cfg_cat(arrs):
        return np.concatenate([a[0:1] for a in arrs] + [a[1:2] for a in arrs], axis=0)
    return Request(np.stack([r.latent for r in reqs]), cfg_cat([r.context for r in reqs]),
                   [cfg_cat([r.images[i] for r in reqs]) for i in range(n_controlnets)],
                   cfg_cat([r.pooled for r in reqs]) if cfg.addition_embed else None,
                   cfg_cat([r.time_ids for r in reqs]) if cfg.addition_embed else None)


@dataclass
class SharedWeights:
    """One UNet + ControlNet weight set (and its LoRA shadow copy) shared by
    engines of different shapes (serving.EngineCache)."""
    unet_p: object
    cn_p: list
    shadow: Optional[dict] = None


class AddonPipeline:
    """SD-style UNet + N ControlNets + LoRA on one B200."""

    def __init__(self, cfg: UNetConfig, n_controlnets: int = 1, cn_scales: Optional[Sequence[float]] = None,
                 steps: int = 30, guidance: float = 7.5, device="cuda", dtype=torch.bfloat16,
                 seed: int = 0, use_graphs: bool = True, patch_max_ctas: int = 0, batch: int = 1,
                 weights: Optional["SharedWeights"] = None):
        ops.require_cuda(torch.empty(1, device=device))
        self.cfg, self.steps, self.guidance = cfg, steps, guidance
        self.device = torch.device(device)
        self.dtype = dtype
        self.weights = weights
        if weights is not None:   # engines of other shapes over the same weights (serving.EngineCache)
            if len(weights.cn_p) != n_controlnets:
                raise ValueError("shared weights hold a different number of ControlNets")
            self.unet_p, self.cn_p = weights.unet_p, weights.cn_p
        else:
            self.unet_p = init_unet(cfg, self.device, dtype, seed)
            self.cn_p = [init_controlnet(cfg, self.device, dtype, seed=1000 + i) for i in range(n_controlnets)]
        self.unet = UNet(cfg, self.unet_p)
        self.cns = [ControlNet(cfg, p) for p in self.cn_p]
        self.cn_scales = list(cn_scales) if cn_scales is not None else [0.8] * n_controlnets
        self.use_graphs = use_graphs
        self.patch_max_ctas = patch_max_ctas
        h = cfg.latent_hw
        dev = self.device
        # a serving batch of B images shares the step (and the LoRA set): the
        # CFG batch is [uncond x B; cond x B], the fp32 master latents [B, H, W, 4]
        self.batch = batch
        nb = 2 * batch
        self.L = batch * 4 * h * h
        self.x = torch.zeros(self.L, device=dev, dtype=torch.float32)
        self.unet_in = torch.zeros((nb, 4, h, h), device=dev, dtype=dtype).contiguous(memory_format=torch.channels_last)
        self.ctx = torch.zeros((nb, cfg.context_len, cfg.context_dim), device=dev, dtype=dtype)
        self.pooled = torch.zeros((nb, cfg.pooled_dim), device=dev, dtype=torch.float32)
        self.time_ids = torch.zeros((nb, cfg.time_ids), device=dev, dtype=torch.float32)
        self.images = [torch.zeros((nb, 3, 8 * h, 8 * h), device=dev, dtype=dtype) for _ in self.cns]
        self.hints = [torch.zeros((nb, cfg.block_channels[0], h, h), device=dev, dtype=dtype)
                      .contiguous(memory_format=torch.channels_last) for _ in self.cns]
        temb = cfg.time_embed_dim
        self.add_emb_unet = torch.zeros((nb, temb), device=dev, dtype=dtype) if cfg.addition_embed else None
        self.add_emb_cn = [torch.zeros((nb, temb), device=dev, dtype=dtype) if cfg.addition_embed else None
                           for _ in self.cns]
        # cross-attention K|V per request (pristine) and after the LoRA swap (patched)
        self.unet.enable_kv_cache(self.ctx, ("pristine", "patched"))
        for cn in self.cns:
            cn.enable_kv_cache(self.ctx, ("pristine",))
        tab = ddim_tables(steps, guidance)
        pad = 8  # capture warm-ups advance the step counter past the table end
        t_tab = np.concatenate([tab.timesteps.astype(np.float32), np.full(pad, tab.timesteps[-1], np.float32)])
        coef = np.concatenate([tab.coef, np.repeat(tab.coef[-1:], pad, axis=0)])
        self.timesteps = tab.timesteps
        self.t_table = torch.from_numpy(t_tab).to(dev)
        self.coef = torch.from_numpy(coef).to(dev)
        self.step_dev = torch.zeros(2, device=dev, dtype=torch.int32)
        self.main_stream = torch.cuda.Stream(device=dev, priority=-1)
        self.patch_stream = torch.cuda.Stream(device=dev, priority=0)
        self.copy_stream = torch.cuda.Stream(device=dev, priority=0)
        # this engine's own capture stream (library per-stream resources, e.g.
        # the cuBLAS workspace, must not be shared with graphs that another
        # engine may replay concurrently)
        self.capture_stream = torch.cuda.Stream(device=dev)
        self.bank = None
        self.patch_graph = None
        self.shadow = None
        self.patchset: Optional[PatchSet] = None
        self.graphs: dict = {}
        self.pool = None
        self.eps = None
        self.step_ms_est = None
        self.patch_ms_est = None
        self.last_first_patched_step = None
        self.patch_timing: Optional[list] = None   # bench: (start, K1 end) events of each patch launch
        self.last_patch_k1_event = None
        self.launches_per_step = 0
        # group-pipelined patching (orchestrator.py:244-278): M contiguous
        # matrix groups, each fetched / patched / swapped in on its own
        self.patch_groups: Optional[list] = None
        self.group_patchsets: list = []
        self.group_graphs: list = []
        self.group_loads_ms: Optional[list] = None
        self.last_group_boundaries: Optional[list] = None

    # ------------------------------------------------------------------
    def _weight_names(self) -> list:
        return [n for n, _ in self.unet_p.matrices] + list(self.unet_p.fused)

    def _variant_weights(self, which: str) -> dict:
        """{weight name: tensor} of a weight set: "pristine", "patched" (every
        LoRA group swapped in) or "pg<v>" (the first v patch groups swapped in,
        the rest pristine — group-pipelined patching)."""
        if which == "pristine":
            return self._pristine
        if which == "patched":
            return self.shadow
        if not which.startswith("pg") or self.patch_groups is None:
            raise ValueError(f"unknown weight set {which!r}")
        v = int(which[2:])
        swapped = set().union(*self.patch_groups[:v])
        for parent, members in self.unet_p.fused.items():
            if all(m in swapped for m in members):
                swapped.add(parent)
        return {n: (self.shadow[n] if n in swapped else self._pristine[n]) for n in self._weight_names()}

    def _use_weights(self, which: str) -> None:
        src = self._variant_weights(which)
        for name in self._weight_names():
            self.unet_p.t[name + ".weight"] = src[name]
        self.unet.kv_slot = which            # the matching cross-attention K|V slot
        for cn in self.cns:
            cn.kv_slot = "pristine"

    @property
    def _pristine(self) -> dict:
        if not hasattr(self, "_pristine_w"):
            self._pristine_w = {n: self.unet_p.t[n + ".weight"] for n in self._weight_names()}
        return self._pristine_w

    def step_once(self) -> None:
        """One denoising step, reading everything from static buffers."""
        t = self.t_table.index_select(0, self.step_dev[:1].long())
        residuals = [cn.forward(self.unet_in, t, self.ctx, self.hints[i], self.add_emb_cn[i])
                     for i, cn in enumerate(self.cns)]
        eps = self.unet.forward(self.unet_in, t, self.ctx, self.add_emb_unet,
                                residuals if residuals else None, self.cn_scales if residuals else None)
        ops.cfg_ddim_step(eps, self.x, self.coef, self.step_dev, unet_in=self.unet_in)
        self.eps = eps

    def _capture(self, which: str) -> None:
        _ = self._pristine
        self._use_weights(which)
        s = torch.cuda.current_stream(self.device)
        self.step_dev.zero_()
        side = self.capture_stream
        side.wait_stream(s)
        with torch.cuda.stream(side):
            for _ in range(2):
                self.step_once()
        s.wait_stream(side)
        self.step_dev.zero_()
        g = torch.cuda.CUDAGraph()
        c0 = ops.LAUNCHES["count"]
        with torch.cuda.graph(g, pool=self.pool, stream=side):
            self.step_once()
        self.launches_per_step = ops.LAUNCHES["count"] - c0   # our kernels per replay
        if self.pool is None:
            self.pool = g.pool()
        self.graphs[which] = g
        self._use_weights("pristine")
        torch.cuda.synchronize(self.device)

    # ------------------------------------------------------------------
    def load_loras(self, adapters: Sequence[tuple[UNetLora, float]], host_resident: bool = False,
                   groups: int = 1) -> PatchSet:
        """Stack the request's adapters into one planned K1 launch writing the
        shadow weights (allocated once).

        host_resident: the adapters live in pinned host memory (AdapterBank)
        and every patched request re-fetches them — the async LoRA fetch path
        (orchestrator.py:509-528): H2D on a copy stream,
        then ONE CUDA graph on the patch stream re-stacks/re-packs them and
        runs K1, all overlapped with the first denoising steps; the plan's
        "load" time is fetch + pack + patch.

        groups > 1: group-pipelined patching (orchestrator.py:244-278,
        PAPER.md:520-528) — the matrices split into ``groups`` contiguous runs
        (split_patch_groups); each group is fetched, packed and patched by its
        own K1 launch and swapped in at its own step boundary
        (plan_pipeline_patch), so the early groups need not wait for the whole
        adapter set.  One extra step graph per partial weight set."""
        if self.shadow is None:
            _ = self._pristine
            if self.weights is not None:      # one shadow copy per weight set, not per engine
                if self.weights.shadow is None:
                    self.weights.shadow = allocate_shadow(self.unet_p)
                self.shadow = self.weights.shadow
            else:
                self.shadow = allocate_shadow(self.unet_p)
        if groups > 1:
            return self._load_groups(adapters, host_resident, groups)
        self.patch_groups, self.group_patchsets, self.group_graphs = None, [], []
        self.bank = AdapterBank(self.unet_p, adapters, self.device) if host_resident else None
        if self.bank is not None:
            adapters = self.bank.adapters
            self.bank.fetch()
        self.patchset = PatchSet(self.unet_p, adapters, shadow=self.shadow)
        self.patchset.copy_unpatched()
        self.patch_graph = None
        if self.bank is not None:
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            self.patch_stream.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.graph(g, stream=self.patch_stream):
                self.patchset.refresh(self.patch_stream)
                self.patchset.launch(stream=self.patch_stream, max_ctas=self.patch_max_ctas)
            self.patch_graph = g
        if self.use_graphs and "patched" not in self.graphs:
            self._capture("patched")
        return self.patchset

    def _load_groups(self, adapters, host_resident: bool, n_groups: int) -> PatchSet:
        touched = {n for a, _ in adapters for n in a.factors}
        split = [g for g in split_patch_groups(self.unet_p, n_groups) if g & touched]
        self.patch_groups = split
        self.group_loads_ms = None
        self.bank = AdapterBank(self.unet_p, adapters, self.device, groups=split) if host_resident else None
        if self.bank is not None:
            adapters = self.bank.adapters
            self.bank.fetch()
        self.group_patchsets = [PatchSet(self.unet_p, adapters, shadow=self.shadow, only=g) for g in split]
        covered = set().union(*(ps.touched for ps in self.group_patchsets))
        for name, _ in self.unet_p.matrices:          # untouched shadow entries mirror pristine
            if name not in covered:
                self.shadow[name].copy_(self.unet_p.t[name + ".weight"])
        self.patchset = self.group_patchsets[-1]
        self.patch_graph = None
        self.group_graphs = []
        if self.bank is not None:
            torch.cuda.synchronize(self.device)
            self.patch_stream.wait_stream(torch.cuda.current_stream(self.device))
            for ps in self.group_patchsets:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.patch_stream):
                    ps.refresh(self.patch_stream)
                    ps.launch(stream=self.patch_stream, max_ctas=self.patch_max_ctas)
                self.group_graphs.append(g)
        key = tuple(frozenset(g) for g in split)
        if getattr(self, "_graph_split", None) != key:      # partial sets changed: recapture
            for k in [k for k in self.graphs if k.startswith("pg")]:
                del self.graphs[k]
            self._graph_split = key
        variants = [f"pg{v}" for v in range(1, len(split))] + ["patched"]
        for v in variants:
            self.unet.ensure_kv_slot(v)
            if self.use_graphs and v not in self.graphs:
                self._capture(v)
        return self.patchset

    def launch_patch_groups(self, timing: bool = False, fetch: bool = True):
        """Enqueue every group's fetch -> pack -> K1 -> K|V chain on the side
        streams (group m's fetch overlaps group m-1's patch); returns (start
        event, [ready event per group]).  Group m's ready event also covers
        the K|V slot of weight set m+1."""
        s = torch.cuda.current_stream(self.device)
        M = len(self.patch_groups)
        p0 = torch.cuda.Event(enable_timing=True) if timing else None
        self.copy_stream.wait_stream(s)
        self.copy_stream.wait_stream(self.patch_stream)       # previous request's packs done
        self.patch_stream.wait_stream(s)                      # shadow free once earlier steps finished
        if timing:
            p0.record(self.copy_stream if self.bank is not None else self.patch_stream)
            if self.bank is None:
                self.copy_stream.wait_event(p0)
        ready = []
        for m in range(M):
            if self.bank is not None:
                if fetch:
                    self.bank.fetch(self.copy_stream, group=m)
                fe = torch.cuda.Event()
                fe.record(self.copy_stream)
                self.patch_stream.wait_event(fe)
                with torch.cuda.stream(self.patch_stream):
                    self.group_graphs[m].replay()
            else:
                self.group_patchsets[m].launch(stream=self.patch_stream, max_ctas=self.patch_max_ctas)
            v = "patched" if m == M - 1 else f"pg{m + 1}"
            with torch.cuda.stream(self.patch_stream):
                self.unet.compute_kv(self.ctx, v, weights=self._variant_weights(v))
            ev = torch.cuda.Event(enable_timing=timing)
            ev.record(self.patch_stream)
            ready.append(ev)
        return p0, ready

    def calibrate_groups(self) -> list:
        """Measured ready time (ms after the request's start) of each patch
        group — plan_pipeline_patch's group_loads_ms."""
        if self.step_ms_est is None:
            return self.calibrate() and self.group_loads_ms
        torch.cuda.synchronize(self.device)
        with torch.cuda.stream(self.main_stream):
            p0, ready = self.launch_patch_groups(timing=True)
        ready[-1].synchronize()
        loads = [p0.elapsed_time(e) for e in ready]
        for i in range(1, len(loads)):      # events on one stream: guard float noise
            loads[i] = max(loads[i], loads[i - 1])
        self.group_loads_ms = loads
        return loads

    def denoise_pipelined(self, boundaries: Optional[Sequence[int]] = None, on_step=None,
                          fetch: bool = True) -> list:
        """Group-pipelined patching: group m is swapped in after step
        boundaries[m] (forced, non-decreasing) or at the boundary
        plan_pipeline_patch picks from the calibrated group ready times
        (per_group_patch_ms = 0: the patch runs on the side stream into the
        shadow weights).  Returns the boundary of each group (None = the group
        missed the request)."""
        if not self.patch_groups:
            raise RuntimeError("denoise_pipelined needs load_loras(groups > 1) first")
        M = len(self.patch_groups)
        if boundaries is None:
            if self.group_loads_ms is None:
                self.calibrate_groups()
            plan = plan_pipeline_patch(self.group_loads_ms, self.step_ms_est, 0.0, self.steps)
            bounds = [g.boundary_step for g in plan.groups] + [None] * (M - len(plan.groups))
        else:
            bounds = list(boundaries)
            if len(bounds) != M or any(b is not None and b < 0 for b in bounds):
                raise ValueError(f"need {M} non-negative boundaries")
            live = [b for b in bounds if b is not None]
            if any(b2 < b1 for b1, b2 in zip(live, live[1:])) or (None in bounds and
                                                                  any(b is not None for b in bounds[bounds.index(None):])):
                raise ValueError("group boundaries must be non-decreasing (None only as a suffix)")
        s = torch.cuda.current_stream(self.device)
        p0, ready = self.launch_patch_groups(timing=self.patch_timing is not None, fetch=fetch)
        waited = 0
        for step in range(1, self.steps + 1):
            v = sum(1 for b in bounds if b is not None and b + 1 <= step)
            while waited < v:
                s.wait_event(ready[waited])
                waited += 1
            which = "pristine" if v == 0 else ("patched" if v == M else f"pg{v}")
            self._replay(which)
            if on_step is not None:
                on_step(step, self.latent_nchw().clone())
        s.wait_event(ready[-1])              # never leave the side streams dangling
        self.last_group_boundaries = bounds
        live = [b for b in bounds if b is not None]
        self.last_first_patched_step = bounds[-1] + 1 if len(live) == M else self.steps + 1
        return bounds

    def launch_patch(self, timing: bool = False, fetch: bool = True):
        """Enqueue the request's patch on the side streams; returns (start, done)
        events (start is None unless timing; done = the patched weights AND the
        request's patched cross-attention K|V are ready).  Host-resident adapters: fetch on
        the copy stream (skipped with fetch=False: the staging already holds
        them), then the captured refresh+patch graph."""
        s = torch.cuda.current_stream(self.device)
        p0 = torch.cuda.Event(enable_timing=True) if timing else None
        if self.bank is not None and fetch:
            self.copy_stream.wait_stream(s)
            self.copy_stream.wait_stream(self.patch_stream)   # previous pack finished reading staging
            if timing:
                p0.record(self.copy_stream)
            self.bank.fetch(self.copy_stream)
            self.patch_stream.wait_stream(self.copy_stream)
            self.patch_stream.wait_stream(s)                  # shadow free once earlier steps finished
            with torch.cuda.stream(self.patch_stream):
                self.patch_graph.replay()                     # re-stack/re-pack + K1
        else:
            self.patch_stream.wait_stream(s)
            if timing:
                p0.record(self.patch_stream)
            self.patchset.launch(stream=self.patch_stream, max_ctas=self.patch_max_ctas)
        k1 = None
        if timing:   # end of the patch kernel itself (the bench's live K1 roofline)
            k1 = torch.cuda.Event(enable_timing=True)
            k1.record(self.patch_stream)
        with torch.cuda.stream(self.patch_stream):      # the request's K|V under the patched weights
            self.unet.compute_kv(self.ctx, "patched", weights=self.shadow)
        ev = torch.cuda.Event(enable_timing=timing)
        ev.record(self.patch_stream)
        self.last_patch_k1_event = k1
        return p0, ev

    def setup(self) -> None:
        if self.use_graphs and "pristine" not in self.graphs:
            self._capture("pristine")

    def calibrate(self, reps: int = 3) -> tuple[float, float]:
        """Measure one step and one patch launch (CUDA events) for the
        patch-boundary plan."""
        self.setup()
        torch.cuda.synchronize(self.device)
        s = self.main_stream
        with torch.cuda.stream(s):
            self.step_dev.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self._replay("pristine")
            e0.record(s)
            for _ in range(reps):
                self._replay("pristine")
            e1.record(s)
        e1.synchronize()
        self.step_ms_est = e0.elapsed_time(e1) / reps
        if self.patch_groups:
            self.patch_ms_est = self.calibrate_groups()[-1]
        elif self.patchset is not None:
            p0, p1 = self.launch_patch(timing=True)
            p1.synchronize()
            self.patch_ms_est = p0.elapsed_time(p1)   # the plan's "load": fetch + pack + patch
        return self.step_ms_est, self.patch_ms_est

    def _replay(self, which: str) -> None:
        if self.use_graphs:
            self.graphs[which].replay()
        else:
            self._use_weights(which)
            self.step_once()
            self._use_weights("pristine")

    # ------------------------------------------------------------------
    def prepare(self, latent: torch.Tensor, context: torch.Tensor, images: Sequence[torch.Tensor],
                pooled: Optional[torch.Tensor] = None, time_ids: Optional[torch.Tensor] = None) -> None:
        """Load one request's (device or pinned-host) inputs into the static
        buffers and compute the step-invariant pieces (hint embeddings, SDXL
        added-condition embeddings)."""
        h, B = self.cfg.latent_hw, self.batch
        nb = True
        lat = latent.to(self.device, non_blocking=nb)
        lat = lat.unsqueeze(0) if lat.dim() == 3 else lat
        self.x.view(B, h, h, 4).copy_(lat.permute(0, 2, 3, 1))
        xv = self.x.view(B, h, h, 4).permute(0, 3, 1, 2)
        self.unet_in[:B].copy_(xv)
        self.unet_in[B:].copy_(xv)
        self.ctx.copy_(context.to(self.device, non_blocking=nb))
        for buf, img in zip(self.images, images):
            buf.copy_(img.to(self.device, non_blocking=nb))
        if self.cfg.addition_embed:
            self.pooled.copy_(pooled.to(self.device, non_blocking=nb))
            self.time_ids.copy_(time_ids.to(self.device, non_blocking=nb))
            self.add_emb_unet.copy_(self.unet.add_embedding(self.pooled, self.time_ids))
        for i, cn in enumerate(self.cns):
            self.hints[i].copy_(cn.hint_embedding(self.images[i]))
            if self.cfg.addition_embed:
                self.add_emb_cn[i].copy_(cn.add_embedding(self.pooled, self.time_ids))
            cn.compute_kv(self.ctx, "pristine")
        self.unet.compute_kv(self.ctx, "pristine", weights=self._pristine)
        for net in [self.unet] + self.cns:
            if net.kv_slot is None:
                net.kv_slot = "pristine"
        self.step_dev.zero_()

    def denoise(self, patch: bool = False, boundary: Optional[int] = None, on_step=None,
                fetch: bool = True) -> int:
        """Run all steps on the current stream.  With ``patch`` the loaded
        PatchSet is launched on the side stream at the start and swapped in
        at boundary k (forced, or planned from the calibrated times).
        Returns first_patched_step (steps + 1 = never)."""
        s = torch.cuda.current_stream(self.device)
        first = self.steps + 1
        ev = None
        if patch:
            if self.patchset is None:
                raise RuntimeError("denoise(patch=True) needs load_loras() first")
            if boundary is None:
                if self.step_ms_est is None or self.patch_ms_est is None:
                    self.calibrate()
                plan = plan_lora_patch(self.patch_ms_est, self.step_ms_est, 0.0, self.steps)
                first = plan.first_patched_step
            else:
                first = boundary + 1
            p0, ev = self.launch_patch(timing=self.patch_timing is not None, fetch=fetch)
            if self.patch_timing is not None:
                self.patch_timing.append((p0, self.last_patch_k1_event))
        waited = False
        for step in range(1, self.steps + 1):
            use_patched = patch and step >= first
            if use_patched and not waited:
                s.wait_event(ev)
                waited = True
            self._replay("patched" if use_patched else "pristine")
            if on_step is not None:   # tests: per-step latent parity (syncs the host)
                on_step(step, self.latent_nchw().clone())
        if patch and not waited:
            s.wait_event(ev)  # never leave the side stream dangling past the request
        self.last_first_patched_step = first
        return first

    def latent_nchw(self) -> torch.Tensor:
        """[4, H, W] (B = 1) or [B, 4, H, W] view of the fp32 master latents."""
        h = self.cfg.latent_hw
        if self.batch == 1:
            return self.x.view(h, h, 4).permute(2, 0, 1)
        return self.x.view(self.batch, h, h, 4).permute(0, 3, 1, 2)

    # ------------------------------------------------------------------
    def generate(self, req: Request, patch: bool = False, boundary: Optional[int] = None,
                 pinned: Optional[dict] = None) -> np.ndarray:
        """The end-to-end call: host inputs in, host latent out (H2D + denoise
        + D2H on the current stream)."""
        def host(a, key):
            t = torch.from_numpy(a)
            if pinned is not None:
                buf = pinned.get(key)
                if buf is None or buf.shape != t.shape:
                    buf = torch.empty(t.shape, dtype=t.dtype).pin_memory()
                    pinned[key] = buf
                buf.copy_(t)
                return buf
            return t
        lat = host(req.latent, "latent")
        ctx = host(req.context, "ctx")
        imgs = [host(im, f"img{i}") for i, im in enumerate(req.images)]
        pooled = host(req.pooled, "pooled") if req.pooled is not None else None
        tids = host(req.time_ids, "tids") if req.time_ids is not None else None
        self.prepare(lat, ctx, imgs, pooled, tids)
        self.denoise(patch=patch, boundary=boundary)
        out = self.latent_nchw().contiguous().cpu()
        return out.numpy()

    def d2h_bytes(self) -> int:
        return self.L * 4
