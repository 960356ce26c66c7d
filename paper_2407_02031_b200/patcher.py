"""Whole-UNet LoRA patch sets: one batched K1 launch over every target matrix.

Reference semantics (addonsim/lora.py): a merge is W += s * down @ up per layer
(:98-104); several adapters merged together equal one merge of their stack
(:147-160, down' = [d_i * f32(s_i)], up' = [u_i], scale 1.0).  Here all
adapters of a request are stacked per matrix and ALL matrices of the UNet
(794 for SDXL) are patched by ONE launch of the K1 kernel — one W read and
one W write per element, regardless of how many adapters are stacked.

Two modes:
* shadow (serving): W_shadow = W_pristine + delta, written out of place on a
  low-priority side stream while the first denoising steps run on the
  pristine weights; the pipeline swaps to the patched CUDA graph at the
  boundary ``plan_lora_patch`` picks (schedule.py).  Unpatch is a pointer swap
  back to the pristine weights: exact, zero cost (SURVEY §7 hard part 3: a
  bf16 W + d - d round trip is not exact, so serving never subtracts).
* in place (the reference's merge/unmerge semantics): sign = -1 unmerges.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import ops
from .errors import ValidationError
from .unet import Params


@dataclass
class UNetLora:
    """One adapter over (a subset of) a UNet's matrices, reference factor
    convention: down (h1, r), up (r, h2) with h2 in LOGICAL (Cin, kh, kw) order."""

    adapter_id: str
    factors: dict            # name -> (down, up)
    scale: float = 1.0

    @property
    def rank(self) -> int:
        return max(d.shape[1] for d, _ in self.factors.values())

    @property
    def nbytes(self) -> int:
        return sum(d.numel() * d.element_size() + u.numel() * u.element_size() for d, u in self.factors.values())


def synthetic_lora(params: Params, rank: int, seed: int, adapter_id: str = "lora", scale: float = 1.0,
                   dtype=None, down_std: float = 0.1, up_std: float = 0.2,
                   targets: Optional[Sequence[str]] = None) -> UNetLora:
    """Random adapter on every matrix (or ``targets``): down ~ N(0,1)*down_std/sqrt(r),
    up ~ N(0,1)*up_std.  Defaults keep the delta ~ the weights' own scale."""
    dtype = dtype or params.dtype
    gen = torch.Generator(device=params.device).manual_seed(seed)
    names = [n for n, _ in params.matrices] if targets is None else list(targets)
    factors = {}
    for name in names:
        h1, h2 = logical_shape(params, name)
        d = torch.randn((h1, rank), generator=gen, device=params.device) * (down_std / rank ** 0.5)
        u = torch.randn((rank, h2), generator=gen, device=params.device) * up_std
        factors[name] = (d.to(dtype), u.to(dtype))
    return UNetLora(adapter_id, factors, scale)


def logical_shape(params: Params, name: str) -> tuple[int, int]:
    w = params.t[name + ".weight"]
    if w.dim() == 2:
        return tuple(w.shape)
    cout, cin, kh, kw = w.shape
    return cout, cin * kh * kw


def physical_up(params: Params, name: str, up: torch.Tensor) -> torch.Tensor:
    """Permute the columns of a LOGICAL-order ``up`` (r, Cin*kh*kw) into the
    physical channels_last column order (r, kh*kw*Cin) of the stored weight."""
    w = params.t[name + ".weight"]
    if w.dim() == 2:
        return up.contiguous()
    cout, cin, kh, kw = w.shape
    r = up.shape[0]
    return up.reshape(r, cin, kh, kw).permute(0, 2, 3, 1).reshape(r, kh * kw * cin).contiguous()


def allocate_shadow(params: Params) -> dict:
    """Patched copies of every matrix weight (same shape / memory format).
    Fused storages (e.g. attention q|k|v) get one shadow storage whose row
    blocks are the members' shadows, so the patched forward keeps its single
    GEMM; keys are matrix names plus the fused parents."""
    shadow = {}
    for parent, members in params.fused.items():
        ps = torch.empty_like(params.t[parent + ".weight"])
        shadow[parent] = ps
        rows = params.t[members[0] + ".weight"].shape[0]
        for i, m in enumerate(members):
            shadow[m] = ps[i * rows:(i + 1) * rows]
    for name, _ in params.matrices:
        if name not in shadow:
            shadow[name] = torch.empty_like(params.t[name + ".weight"])
    return shadow


class PatchSet:
    """The stacked adapters of one request over one UNet, planned as a single
    device-resident K1 job table."""

    def __init__(self, params: Params, adapters: Sequence[tuple[UNetLora, float]],
                 shadow: Optional[dict] = None, use_tma: bool = True, simt_max_rank: int = 0):
        if not adapters:
            raise ValidationError("PatchSet needs at least one adapter")
        self.params = params
        self.shadow = shadow
        names = [n for n, _ in params.matrices if any(n in a.factors for a, _ in adapters)]
        self.entries = []
        self.stacked = {}
        for name in names:
            downs, ups = [], []
            for a, s in adapters:
                if name not in a.factors:
                    continue
                d, u = a.factors[name]
                # lora.py:153 folds f32(s) into down; done in fp32, one rounding to the factor dtype
                downs.append((d.float() * np.float32(s)).to(d.dtype))
                ups.append(physical_up(params, name, u))
            down = torch.cat(downs, dim=1).contiguous()
            up = torch.cat(ups, dim=0).contiguous()
            self.stacked[name] = (down, up)
            w_in = params.matrix_view(name)
            w_out = None
            if shadow is not None:
                w_out = shadow[name].permute(0, 2, 3, 1).reshape(w_in.shape) if shadow[name].dim() == 4 \
                    else shadow[name]
            self.entries.append((w_in, w_out, down, up, 1.0))
        self.rank = max(d.shape[1] for d, _ in self.stacked.values())
        # bf16 matrices with 16-B aligned rows take the TMA / tcgen05 kernel (one
        # launch, factors packed here, once per adapter set); the rest (e.g.
        # SDXL conv_in, 320 x 36) the generic SIMT kernel.
        fast = [e for e in self.entries if use_tma and self.rank <= 256 and ops.tma_eligible(e[0])
                and e[2].dtype == torch.bfloat16]
        slow = [e for e in self.entries if not any(e is f for f in fast)]
        self.plans = []
        if fast:
            self.plans.append(ops.LoraTmaPlan(fast, simt_max_rank=simt_max_rank))
        if slow:
            self.plans.append(ops.LoraPatchPlan(slow))
        self.plan = self.plans[0]

    @property
    def alg_bytes(self) -> int:
        return sum(p.alg_bytes for p in self.plans)

    @property
    def alg_flops(self) -> int:
        return sum(p.alg_flops for p in self.plans)

    def launch(self, sign: float = 1.0, stream: Optional[torch.cuda.Stream] = None, max_ctas: int = 0):
        for p in self.plans:
            p.launch(sign=sign, stream=stream, max_ctas=max_ctas)

    def copy_unpatched(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Shadow entries not touched by any adapter must mirror the pristine
        weight (only needed when adapters cover a subset of matrices)."""
        if self.shadow is None:
            return
        touched = set(self.stacked)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for name, _ in self.params.matrices:
                if name not in touched:
                    self.shadow[name].copy_(self.params.t[name + ".weight"])


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
