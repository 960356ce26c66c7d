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

from dataclasses import dataclass
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
    up_physical: bool = False   # True: up columns already in the stored weight's order

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
                 shadow: Optional[dict] = None, use_tma: bool = True, simt_max_rank: int = 0,
                 only: Optional[set] = None, in_place_on_shadow: bool = False):
        """shadow: write W + delta there (out of place).  in_place_on_shadow:
        patch the shadow weights in place instead (W_shadow += sign * delta —
        the reference's merge / unmerge on a serving copy; micro-bench)."""
        if not adapters:
            raise ValidationError("PatchSet needs at least one adapter")
        self.params = params
        self.shadow = shadow
        self.adapters = list(adapters)
        names = [n for n, _ in params.matrices if any(n in a.factors for a, _ in adapters)
                 and (only is None or n in only)]
        if not names:
            raise ValidationError("PatchSet: no adapter touches the selected matrices")
        self.touched = set(names)
        ranks = {n: sum(a.factors[n][0].shape[1] for a, _ in adapters if n in a.factors) for n in names}
        self.rank = max(ranks.values())
        fast, slow = [], []
        self.stacked = {}    # name -> (down, up) for the generic-kernel matrices
        for name in names:
            present = [(a, s) for a, s in adapters if name in a.factors]
            w_in = params.matrix_view(name)
            w_out = None
            if shadow is not None:
                w_out = shadow[name].permute(0, 2, 3, 1).reshape(w_in.shape) if shadow[name].dim() == 4 \
                    else shadow[name]
                if in_place_on_shadow:
                    w_in, w_out = w_out, None
            ups = [a.factors[name][1] if a.up_physical else physical_up(params, name, a.factors[name][1])
                   for a, _ in present]
            if (use_tma and self.rank <= 256 and ops.tma_eligible(w_in)
                    and all(a.factors[name][0].dtype == torch.bfloat16 for a, _ in present)):
                # bf16, 16-B rows: the TMA / tcgen05 kernel; adapters stacked while packing
                srcs = [(a.factors[name][0], u, float(np.float32(s))) for (a, s), u in zip(present, ups)]
                fast.append((w_in, w_out, srcs, None, 1.0))
            else:
                # everything else (e.g. SDXL conv_in, 320 x 36): the generic kernel on a
                # stacked copy (lora.py:147-160; see _stack for how the scales stay exact)
                self.stacked[name] = self._stack(name, present, ups)
                down, up = self.stacked[name]
                slow.append((w_in, w_out, down, up, self._epi_scale(name, present)))
        self._slow_src = {n: [(a, s) for a, s in adapters if n in a.factors] for n in self.stacked}
        self.plans = []
        if fast:
            self.plans.append(ops.LoraTmaPlan(fast, simt_max_rank=simt_max_rank))
        if slow:
            self.plans.append(ops.LoraPatchPlan(slow))
        self.plan = self.plans[0]

    @staticmethod
    def _epi_scale(name, present) -> float:
        """The job scale of a stacked copy: 1.0 for fp32 factors (lora.py:153
        folds every f32(s) into down in fp32 — the reference's own rounding);
        for bf16 factors the nonzero scale carried by the largest share of the
        rank (first on ties), applied in the kernel's fp32 epilogue — the
        same choice sdb_lora_pack_multi makes."""
        if present[0][0].factors[name][0].dtype == torch.float32:
            return 1.0
        share = {}
        for a, s in present:
            s32 = float(np.float32(s))
            if s32 != 0.0:
                share[s32] = share.get(s32, 0) + a.factors[name][0].shape[1]
        best = 0.0
        for k, r in share.items():          # insertion order: first on ties
            if best == 0.0 or r > share[best]:
                best = k
        return best

    def _stack(self, name, present, ups=None, out=None):
        """(down', up') of lora.py:147-160.  fp32 factors: down' = [d_i * f32(s_i)]
        exactly as the reference.  bf16 factors: a bf16 rounding of s_i * d_i
        would add 2^-9 relative per element, so the sources at the epilogue
        scale s_e go in unscaled and every other one as x = d_i * f32(s_i / s_e)
        split into bf16 hi | lo columns (2^-17), with its up rows repeated."""
        if ups is None:
            ups = [a.factors[name][1] if a.up_physical else physical_up(self.params, name, a.factors[name][1])
                   for a, _ in present]
        dtype = present[0][0].factors[name][0].dtype
        downs, ups_out = [], []
        if dtype == torch.float32:
            downs = [a.factors[name][0].float() * np.float32(s) for a, s in present]
            ups_out = list(ups)
        else:
            se = np.float32(self._epi_scale(name, present))
            for (a, s), u in zip(present, ups):
                d = a.factors[name][0]
                fold = np.float32(1.0) if se == 0 else np.float32(np.float32(s) / se)
                if fold == 1.0:
                    downs.append(d)
                    ups_out.append(u)
                    continue
                x = d.float() * float(fold)
                hi = x.to(dtype)
                downs += [hi, (x - hi.float()).to(dtype)]
                ups_out += [u, u]
        if out is None:
            return torch.cat(downs, dim=1).contiguous(), torch.cat(ups_out, dim=0).contiguous()
        torch.cat(downs, dim=1, out=out[0])
        torch.cat(ups_out, dim=0, out=out[1])
        return out

    def refresh(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Re-stack / re-pack from the adapters' (refreshed) factor buffers,
        stream-ordered: the step between an async fetch and the patch."""
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for p in self.plans:
                if isinstance(p, ops.LoraTmaPlan):
                    p.repack(stream)
            for name, present in self._slow_src.items():
                self._stack(name, present, out=self.stacked[name])

    @property
    def alg_bytes(self) -> int:
        return sum(p.alg_bytes for p in self.plans)

    @property
    def alg_flops(self) -> int:
        return sum(p.alg_flops for p in self.plans)

    def launch(self, sign: float = 1.0, stream: Optional[torch.cuda.Stream] = None, max_ctas: int = 0):
        """One K1 launch for the tcgen05 plan; the few matrices the generic
        kernel takes (SDXL's 320 x 36 conv_in: a 5-CTA, ~30 us launch) run on
        a forked stream beside it instead of after it (graph-capturable
        fork / join)."""
        if len(self.plans) == 1:
            self.plans[0].launch(sign=sign, stream=stream, max_ctas=max_ctas)
            return
        main = stream if stream is not None else torch.cuda.current_stream()
        if getattr(self, "_side", None) is None or self._side.device != main.device:
            self._side = torch.cuda.Stream(device=main.device)
        self._side.wait_stream(main)
        for p in self.plans[1:]:
            p.launch(sign=sign, stream=self._side, max_ctas=max_ctas)
        self.plans[0].launch(sign=sign, stream=main, max_ctas=max_ctas)
        main.wait_stream(self._side)

    def copy_unpatched(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Shadow entries not touched by any adapter must mirror the pristine
        weight (only needed when adapters cover a subset of matrices)."""
        if self.shadow is None:
            return
        touched = self.touched
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for name, _ in self.params.matrices:
                if name not in touched:
                    self.shadow[name].copy_(self.params.t[name + ".weight"])


class AdapterBank:
    """Adapters resident in pinned HOST memory — the LoRA cache tier the paper
    fetches from (the reference's tiered fetch,
    addons.py:22-28) — each with a device staging twin.  ``fetch(stream)`` is
    one asynchronous H2D copy per adapter (copy engine, overlaps compute); the
    device views it fills are what a PatchSet packs from, so fetch -> repack ->
    patch is a stream-ordered chain that needs no host round trip."""

    def __init__(self, params: Params, adapters: Sequence[tuple[UNetLora, float]], device=None,
                 groups: Optional[Sequence[set]] = None):
        """groups: optional partition of the matrix names (patch groups, see
        ``split_patch_groups``): each adapter's factors are laid out group by
        group so ``fetch(stream, group=m)`` copies one group's slice."""
        device = torch.device(device) if device is not None else params.device
        self.host, self.dev, self.adapters = [], [], []
        self.nbytes = 0
        self.group_spans = []          # per adapter: [(begin, end)] element range of each group
        gidx = {}
        for m, g in enumerate(groups or []):
            for name in g:
                gidx[name] = m
        order = {n: i for i, (n, _) in enumerate(params.matrices)}
        for a, s in adapters:
            dtype = next(iter(a.factors.values()))[0].dtype
            items = []
            for name, (d, u) in sorted(a.factors.items(), key=lambda kv: (gidx.get(kv[0], 0), order.get(kv[0], 0))):
                up = u if a.up_physical else physical_up(params, name, u.to(params.device))
                items.append((name, d, up))
            total = sum(d.numel() + up.numel() for _, d, up in items)
            host = torch.empty(total, dtype=dtype).pin_memory()
            dev = torch.empty(total, dtype=dtype, device=device)
            views, off = {}, 0
            n_groups = max(1, len(groups or []))
            spans = [[None, None] for _ in range(n_groups)]
            for name, d, up in items:
                nd, nu = d.numel(), up.numel()
                host[off:off + nd].copy_(d.reshape(-1).cpu())
                host[off + nd:off + nd + nu].copy_(up.reshape(-1).cpu())
                views[name] = (dev[off:off + nd].view(d.shape), dev[off + nd:off + nd + nu].view(up.shape))
                m = gidx.get(name, 0)
                spans[m][0] = off if spans[m][0] is None else spans[m][0]
                spans[m][1] = off + nd + nu
                off += nd + nu
            self.group_spans.append([(b or 0, e or 0) for b, e in spans])
            self.host.append(host)
            self.dev.append(dev)
            self.nbytes += total * host.element_size()
            self.adapters.append((UNetLora(a.adapter_id, views, a.scale, up_physical=True), s))

    def fetch(self, stream: Optional[torch.cuda.Stream] = None, group: Optional[int] = None) -> None:
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for h, d, spans in zip(self.host, self.dev, self.group_spans):
                if group is None:
                    d.copy_(h, non_blocking=True)
                else:
                    b, e = spans[group]
                    if e > b:
                        d[b:e].copy_(h[b:e], non_blocking=True)


def split_patch_groups(params: Params, n_groups: int) -> list:
    """Partition the patchable matrices into n_groups contiguous runs of the
    UNet order with ~equal weight bytes (the pipelined loading of
    orchestrator.py:244-278 / PAPER.md:520-528: group m can be patched as soon
    as its own slice of the adapters has arrived).  Members of a fused storage
    (q|k|v, k|v) stay in one group: they are swapped together."""
    if n_groups < 1:
        raise ValidationError("n_groups must be >= 1")
    parent_of = {}
    for parent, members in params.fused.items():
        for m in members:
            parent_of[m] = parent
    names = [n for n, _ in params.matrices]
    sizes = {n: params.t[n + ".weight"].numel() for n in names}
    total = sum(sizes.values())
    groups, cur, acc = [], [], 0
    for i, n in enumerate(names):
        cur.append(n)
        acc += sizes[n]
        nxt = names[i + 1] if i + 1 < len(names) else None
        same_parent = nxt is not None and n in parent_of and parent_of.get(nxt) == parent_of[n]
        if (len(groups) < n_groups - 1 and acc >= total * (len(groups) + 1) / n_groups and not same_parent):
            groups.append(set(cur))
            cur = []
    groups.append(set(cur))
    return [g for g in groups if g]


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
