"""SD-style UNet and ControlNet on the B200 path (NHWC / channels_last, bf16).

The reference ships no network (its denoising loop is a latency
model, addonsim/orchestrator.py:586-719).  This module is the builder-authored
model the north_star names: SD1.5- and SDXL-shaped UNets plus a ControlNet
(encoder + mid copy with zero convs), laid out so that

* every GroupNorm(+SiLU) site runs K2 (``ops.groupnorm_silu``), with the ResNet
  time-embedding add fused into it (model.py:70 1.072);
* every skip connection is consumed by K3 (``ops.residual_inject``), which adds
  the ControlNet residuals while writing the up-block concat;
* every linear / conv weight is a row-major (h1, h2) matrix in the reference's
  LoRA layout (addonsim/lora.py:58-72: h1 = out, h2 = in*kh*kw), so one K1
  launch patches them all.  Conv weights are kept channels_last, i.e. the
  physical matrix is (Cout, kh*kw*Cin); LoRA ``up`` factors are permuted once
  at load time to that column order (patcher.py).

Convolutions, GEMMs, LayerNorm and attention (SDPA / flash) are library calls
(cuDNN / cuBLAS), as the north_star allows; GEGLU fusion and decoupled CUDA
graphs are the ranked "next" items.

Weights are synthetic random-init (N(0, 0.02), norms 1/0, zero-convs non-zero
N(0, 0.02) so residual parity is not vacuous, SURVEY §7 hard part 9).
"""

from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import os

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

from . import ops

# A/B switch for measurements: SDB_K3_GN_STATS=0 keeps the two-pass GroupNorm everywhere
_NO_K3_STATS = os.environ.get("SDB_K3_GN_STATS", "1") == "0"
# cuDNN's per-shape algorithm autotuning (torch.backends.cudnn.benchmark) for
# the 16-bit convolutions: the heuristic picks cost the SDXL step ~2% (945 vs
# 925 ms/image, bench.py A/B on one B200).  Each shape is tuned on its first
# (eager) call — the engines run every shape eagerly before capturing their
# CUDA graphs, and a capture then replays the tuned algorithm.  fp32 (the
# parity mode) keeps the heuristics.  SDB_CUDNN_BENCHMARK=0 turns it off.
_CUDNN_TUNE = os.environ.get("SDB_CUDNN_BENCHMARK", "1") != "0"


def _conv_tuning(x):
    if not _CUDNN_TUNE or x.dtype == torch.float32 or not x.is_cuda:
        return contextlib.nullcontext()
    cd = torch.backends.cudnn
    return cd.flags(enabled=cd.enabled, benchmark=True, deterministic=cd.deterministic, allow_tf32=cd.allow_tf32)


# K5' (the FF projection GEMM with GEGLU in its epilogue, tcgen05) replaces cuBLAS + K5
# for bf16 (scripts/ffg_probe.py: [8192,640]x5120 54.7 vs 66.9 us, [2048,1280]x10240 44.9
# vs 47.8 us); SDB_FF_FUSED=0 keeps the library GEMM + K5
_FF_FUSED = os.environ.get("SDB_FF_FUSED", "1") != "0"
# K8 (tcgen05 flash-style self-attention) is opt-in: SDB_SELF_ATTN=1 (round 1: slower than
# the library SDPA at SDXL's shapes, see csrc/self_attn.cu)
_SELF_ATTN = os.environ.get("SDB_SELF_ATTN", "0") == "1"


# --------------------------------------------------------------------------
# configurations
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class UNetConfig:
    name: str
    block_channels: tuple            # per resolution level
    layers_per_block: int
    attn_depth: tuple                # transformer depth per level (0 = no attention)
    mid_depth: int
    head_dim: Optional[int]          # SDXL: 64-dim heads
    num_heads: Optional[int]         # SD1.5: 8 heads
    context_dim: int
    addition_embed: bool             # SDXL text_time embedding
    addition_time_embed_dim: int = 256
    pooled_dim: int = 1280
    time_ids: int = 6
    latent_channels: int = 4
    groups: int = 32
    gn_eps: float = 1e-5
    tf_gn_eps: float = 1e-6
    hint_channels: tuple = (16, 32, 96, 256)  # ControlNet conditioning embedding
    latent_hw: int = 64
    context_len: int = 77

    @property
    def time_embed_dim(self) -> int:
        return self.block_channels[0] * 4

    def heads(self, c: int) -> int:
        return c // self.head_dim if self.head_dim else self.num_heads


SD15 = UNetConfig(name="sd15", block_channels=(320, 640, 1280, 1280), layers_per_block=2,
                  attn_depth=(1, 1, 1, 0), mid_depth=1, head_dim=None, num_heads=8,
                  context_dim=768, addition_embed=False, latent_hw=64)
SDXL = UNetConfig(name="sdxl", block_channels=(320, 640, 1280), layers_per_block=2,
                  attn_depth=(0, 2, 10), mid_depth=10, head_dim=64, num_heads=None,
                  context_dim=2048, addition_embed=True, latent_hw=128)
# config 1: toy CPU-oracle model
TOY = UNetConfig(name="toy", block_channels=(32, 64), layers_per_block=1, attn_depth=(1, 1),
                 mid_depth=1, head_dim=8, num_heads=None, context_dim=64, addition_embed=False,
                 hint_channels=(8, 16, 16, 32), latent_hw=64, context_len=8)

CONFIGS = {"sd15": SD15, "sdxl": SDXL, "toy": TOY}


# --------------------------------------------------------------------------
# parameters
# --------------------------------------------------------------------------
class Params:
    """Named parameter store.  ``matrices`` lists every LoRA-patchable weight
    as (name, 2-d row-major view of the physical storage, logical kind)."""

    def __init__(self, device, dtype, seed: int):
        self.device = torch.device(device)
        self.dtype = dtype
        # "meta" builds the layout only (inventory / planning without memory)
        self.gen = None if self.device.type == "meta" else torch.Generator(device=self.device).manual_seed(seed)
        self.t: dict[str, torch.Tensor] = {}
        self.matrices: list[tuple[str, str]] = []  # (name, "linear"|"conv")
        self.fused: dict[str, list] = {}           # parent -> member matrices (views of it)

    def _randn(self, shape, std):
        return (torch.randn(shape, generator=self.gen, device=self.device, dtype=torch.float32) * std)

    def linear(self, name, cin, cout, bias=True, std=0.02):
        self.t[name + ".weight"] = self._randn((cout, cin), std).to(self.dtype)
        if bias:
            self.t[name + ".bias"] = torch.zeros(cout, device=self.device, dtype=self.dtype)
        self.matrices.append((name, "linear"))

    def conv(self, name, cin, cout, k, bias=True, std=0.02):
        w = self._randn((cout, cin, k, k), std).to(self.dtype)
        self.t[name + ".weight"] = w.contiguous(memory_format=torch.channels_last)
        if bias:
            self.t[name + ".bias"] = torch.zeros(cout, device=self.device, dtype=self.dtype)
        self.matrices.append((name, "conv"))

    def norm(self, name, c):
        # GN affine in fp32 for K2; LayerNorm affine in the compute dtype
        self.t[name + ".weight"] = torch.ones(c, device=self.device, dtype=torch.float32)
        self.t[name + ".bias"] = torch.zeros(c, device=self.device, dtype=torch.float32)

    def lnorm(self, name, c):
        self.t[name + ".weight"] = torch.ones(c, device=self.device, dtype=self.dtype)
        self.t[name + ".bias"] = torch.zeros(c, device=self.device, dtype=self.dtype)

    def fused_linear(self, parent: str, members: list, cin: int, cout: int, std=0.02):
        """Bias-free linears sharing one (len(members)*cout, cin) storage: the
        forward runs ONE GEMM on ``parent``; LoRA targets each member (a row
        block, i.e. a contiguous row-major (cout, cin) view)."""
        w = self._randn((len(members) * cout, cin), std).to(self.dtype)
        self.t[parent + ".weight"] = w
        for i, m in enumerate(members):
            self.t[m + ".weight"] = w[i * cout:(i + 1) * cout]
            self.matrices.append((m, "linear"))
        self.fused[parent] = list(members)

    def matrix_view(self, name: str) -> torch.Tensor:
        """(h1, h2) row-major view of the weight's physical storage."""
        w = self.t[name + ".weight"]
        if w.dim() == 2:
            return w
        cout, cin, kh, kw = w.shape
        return w.permute(0, 2, 3, 1).reshape(cout, kh * kw * cin)  # a view: channels_last storage

    def numel(self) -> int:
        return sum(v.numel() for v in self.t.values())


def _resnet_params(p: Params, pre: str, cin: int, cout: int, temb: int):
    p.norm(pre + ".norm1", cin)
    p.conv(pre + ".conv1", cin, cout, 3)
    p.linear(pre + ".time_emb_proj", temb, cout)
    p.norm(pre + ".norm2", cout)
    p.conv(pre + ".conv2", cout, cout, 3)
    if cin != cout:
        p.conv(pre + ".conv_shortcut", cin, cout, 1)


def _transformer_params(p: Params, pre: str, c: int, depth: int, ctx: int):
    p.norm(pre + ".norm", c)
    p.linear(pre + ".proj_in", c, c)
    for d in range(depth):
        b = f"{pre}.blocks.{d}"
        p.lnorm(b + ".norm1", c)
        p.fused_linear(b + ".attn1.to_qkv", [b + ".attn1.to_q", b + ".attn1.to_k", b + ".attn1.to_v"], c, c)
        p.linear(b + ".attn1.to_out", c, c)
        p.lnorm(b + ".norm2", c)
        p.linear(b + ".attn2.to_q", c, c, bias=False)
        p.fused_linear(b + ".attn2.to_kv", [b + ".attn2.to_k", b + ".attn2.to_v"], ctx, c)
        p.linear(b + ".attn2.to_out", c, c)
        p.lnorm(b + ".norm3", c)
        p.linear(b + ".ff.proj", c, 8 * c)      # GEGLU: value and gate halves
        p.linear(b + ".ff.out", 4 * c, c)
    p.linear(pre + ".proj_out", c, c)


def _embedding_params(p: Params, cfg: UNetConfig):
    c0, temb = cfg.block_channels[0], cfg.time_embed_dim
    p.linear("time_embedding.linear_1", c0, temb)
    p.linear("time_embedding.linear_2", temb, temb)
    if cfg.addition_embed:
        p.linear("add_embedding.linear_1", cfg.time_ids * cfg.addition_time_embed_dim + cfg.pooled_dim, temb)
        p.linear("add_embedding.linear_2", temb, temb)
    p.conv("conv_in", cfg.latent_channels, c0, 3)


def _down_params(p: Params, cfg: UNetConfig):
    """Encoder; returns the channel count of every skip it produces."""
    temb = cfg.time_embed_dim
    skips = [cfg.block_channels[0]]
    cin = cfg.block_channels[0]
    n = len(cfg.block_channels)
    for i, c in enumerate(cfg.block_channels):
        for j in range(cfg.layers_per_block):
            _resnet_params(p, f"down.{i}.res.{j}", cin, c, temb)
            if cfg.attn_depth[i]:
                _transformer_params(p, f"down.{i}.attn.{j}", c, cfg.attn_depth[i], cfg.context_dim)
            cin = c
            skips.append(c)
        if i < n - 1:
            p.conv(f"down.{i}.downsample", c, c, 3)
            skips.append(c)
    cm = cfg.block_channels[-1]
    _resnet_params(p, "mid.res.0", cm, cm, temb)
    _transformer_params(p, "mid.attn.0", cm, cfg.mid_depth, cfg.context_dim)
    _resnet_params(p, "mid.res.1", cm, cm, temb)
    return skips


def init_unet(cfg: UNetConfig, device="cuda", dtype=torch.bfloat16, seed: int = 0) -> Params:
    p = Params(device, dtype, seed)
    _embedding_params(p, cfg)
    skips = _down_params(p, cfg)
    temb = cfg.time_embed_dim
    rev = list(reversed(cfg.block_channels))
    n = len(rev)
    cin = rev[0]
    for i, c in enumerate(rev):
        depth = cfg.attn_depth[n - 1 - i]
        for j in range(cfg.layers_per_block + 1):
            skip_c = skips.pop()
            _resnet_params(p, f"up.{i}.res.{j}", cin + skip_c, c, temb)
            if depth:
                _transformer_params(p, f"up.{i}.attn.{j}", c, depth, cfg.context_dim)
            cin = c
        if i < n - 1:
            p.conv(f"up.{i}.upsample", c, c, 3)
    p.norm("conv_norm_out", cfg.block_channels[0])
    p.conv("conv_out", cfg.block_channels[0], cfg.latent_channels, 3)
    return p


def init_controlnet(cfg: UNetConfig, device="cuda", dtype=torch.bfloat16, seed: int = 1) -> Params:
    p = Params(device, dtype, seed)
    _embedding_params(p, cfg)
    skips = _down_params(p, cfg)
    # conditioning embedding: 3 -> hint_channels..., stride-2 convs down to latent res, -> C0
    hc = cfg.hint_channels
    p.conv("cond_embedding.conv_in", 3, hc[0], 3)
    for i in range(len(hc) - 1):
        p.conv(f"cond_embedding.blocks.{2 * i}", hc[i], hc[i], 3)
        p.conv(f"cond_embedding.blocks.{2 * i + 1}", hc[i], hc[i + 1], 3)
    p.conv("cond_embedding.conv_out", hc[-1], cfg.block_channels[0], 3)
    for k, c in enumerate(skips):
        p.conv(f"zero_convs.{k}", c, c, 1)       # non-zero N(0, 0.02): parity is not vacuous
    p.conv("mid_zero_conv", cfg.block_channels[-1], cfg.block_channels[-1], 1)
    return p


def skip_channels(cfg: UNetConfig) -> list[int]:
    """Channel count of every down-path skip (= ControlNet down residual)."""
    skips = [cfg.block_channels[0]]
    for i, c in enumerate(cfg.block_channels):
        skips += [c] * cfg.layers_per_block
        if i < len(cfg.block_channels) - 1:
            skips.append(c)
    return skips


def skip_shapes(cfg: UNetConfig, batch: int) -> list[tuple]:
    """(N, C, H, W) of every down residual then the mid residual."""
    h = cfg.latent_hw
    shapes = [(batch, cfg.block_channels[0], h, h)]
    for i, c in enumerate(cfg.block_channels):
        shapes += [(batch, c, h, h)] * cfg.layers_per_block
        if i < len(cfg.block_channels) - 1:
            h //= 2
            shapes.append((batch, c, h, h))
    shapes.append((batch, cfg.block_channels[-1], h, h))
    return shapes


# --------------------------------------------------------------------------
# forward (device path: K2 / K3 kernels + library convs / GEMMs / SDPA)
# --------------------------------------------------------------------------
def timestep_embedding(t: torch.Tensor, dim: int, max_period: float = 10000.0) -> torch.Tensor:
    """Sinusoidal embedding, flip_sin_to_cos=True, shift 0 (diffusers SD config)."""
    half = dim // 2
    freqs = torch.exp(-math.log(max_period) * torch.arange(half, device=t.device, dtype=torch.float32) / half)
    args = t.float()[:, None] * freqs[None]
    return torch.cat([torch.cos(args), torch.sin(args)], dim=-1)


def _cl(x: torch.Tensor) -> torch.Tensor:
    return x.contiguous(memory_format=torch.channels_last)


class Net:
    """Shared forward machinery for the UNet and the ControlNet."""

    def __init__(self, cfg: UNetConfig, params: Params):
        self.cfg = cfg
        self.p = params
        self.t = params.t
        self._gn_ws: dict = {}
        self.kv: dict = {}          # slot -> {attn2 prefix: static K|V buffer}
        self.kv_slot: Optional[str] = None
        self.refresh_biases()

    # -- step-invariant cross-attention K|V ---------------------------------
    def kv_prefixes(self) -> list:
        return [k[: -len(".to_kv.weight")] for k in self.t if k.endswith(".attn2.to_kv.weight")]

    def enable_kv_cache(self, ctx: torch.Tensor, slots: Sequence[str] = ("pristine",)) -> None:
        """Static K|V buffers per cross-attention block and weight slot.  The
        text context is fixed for a request, so K|V = ctx @ W_kv^T is computed
        once per request (and once more after a LoRA swap changes W_kv) rather
        than by ~70 small GEMMs in every denoising step; graphs captured with
        ``kv_slot`` set read the slot's buffers."""
        n, l, _ = ctx.shape
        self.kv = {s: {pre: torch.zeros((n, l, self.t[pre + ".to_kv.weight"].shape[0]), device=ctx.device,
                                        dtype=self.p.dtype) for pre in self.kv_prefixes()} for s in slots}

    def ensure_kv_slot(self, slot: str) -> None:
        """Add one more static K|V slot (e.g. a partially patched weight set)."""
        if slot not in self.kv:
            ref = next(iter(self.kv.values()))
            self.kv[slot] = {pre: torch.zeros_like(buf) for pre, buf in ref.items()}

    def compute_kv(self, ctx: torch.Tensor, slot: str, weights: Optional[dict] = None) -> None:
        """Fill ``slot`` from ctx (stream-ordered on the current stream);
        weights: optional {"<prefix>.to_kv": tensor} override (e.g. the LoRA
        shadow weights)."""
        n, l, d = ctx.shape
        c2 = ctx.reshape(n * l, d)
        for pre, buf in self.kv[slot].items():
            w = weights.get(pre + ".to_kv") if weights is not None else None
            if w is None:
                w = self.t[pre + ".to_kv.weight"]
            torch.mm(c2, w.t(), out=buf.view(n * l, -1))

    def refresh_biases(self) -> None:
        """fp32 per-channel conv biases folded into the consumer kernels.

        cuDNN's channels_last bf16 convolutions add their bias in a separate
        broadcast pass (one full read + write of the output); instead each 3x3
        conv runs bias-free and its bias rides on the next kernel: the ResNet
        conv1 bias on the time-embedding projection (K2's per-(n, c) add), the
        conv2 + shortcut biases, the up/downsample and conv_in biases on K3.
        Call again whenever a bias tensor changes (CaaS scales the zero convs)."""
        t, fb = self.t, {}
        for k, v in t.items():
            if k.endswith(".bias") and t.get(k[:-5] + ".weight") is not None and t[k[:-5] + ".weight"].dim() == 4:
                fb[k[:-5]] = v.float().contiguous()
        for k in list(t):
            if k.endswith(".time_emb_proj.weight"):
                pre = k[: -len(".time_emb_proj.weight")]
                b = t.get(pre + ".time_emb_proj.bias")
                c1 = fb.get(pre + ".conv1")
                if b is not None or c1 is not None:
                    comb = (b.float() if b is not None else 0) + (c1 if c1 is not None else 0)
                    fb[pre + ".tproj_bias"] = comb.to(self.p.dtype).contiguous()
                    # the same sum in the param dtype, held in fp32: the bias of the fp32-output addmm
                    fb[pre + ".tproj_bias_f32"] = fb[pre + ".tproj_bias"].float()
                c2, sc = fb.get(pre + ".conv2"), fb.get(pre + ".conv_shortcut")
                if c2 is not None or sc is not None:
                    fb[pre + ".out_bias"] = ((c2 if c2 is not None else 0) + (sc if sc is not None else 0)).contiguous()
        for k, v in t.items():   # fp32 biases of the GEGLU projections (K5' adds them in its epilogue)
            if k.endswith(".ff.proj.bias"):
                fb[k[: -len(".bias")] + ".bias_f32"] = v.float().contiguous()
        self.fb = fb

    # -- primitives -------------------------------------------------------
    def lin(self, name, x):
        return F.linear(x, self.t[name + ".weight"], self.t.get(name + ".bias"))

    def ff_proj_geglu(self, name, x):
        """GEGLU(x W^T + b) of a transformer FF: K5' (one tcgen05 GEMM with the
        gating in its epilogue) for bf16, else the library GEMM then K5."""
        w = self.t[name + ".weight"]
        if _FF_FUSED and x.is_cuda and ops.ff_geglu_supported(x, w):
            return ops.ff_geglu(x, w, self.fb.get(name + ".bias_f32"))
        return ops.geglu(self.lin(name, x))   # K5

    def conv(self, name, x, stride=1, bias=True):
        """bias=False: the caller folds ``self.fb[name]`` into the next kernel.
        16-bit convolutions run with cuDNN's algorithm autotuning on (see
        _conv2d)."""
        with _conv_tuning(x):
            return self._conv(name, x, stride, bias)

    def _conv(self, name, x, stride=1, bias=True):
        w = self.t[name + ".weight"]
        pad = w.shape[-1] // 2
        if w.shape[1] % 8 != 0 and x.dtype != torch.float32:
            x, w = self._pad_cin(name, x, w)
        elif (tuple(w.shape[:2]) == (320, 256) and w.shape[-1] == 3 and x.shape[0] <= 4
              and x.dtype != torch.float32):
            # the hint embedding's conv_out: cuDNN's heuristic picks a TF32
            # fallback for 256 -> 320 (~410 us at 128x128, CFG batch 2; not at
            # batch 16); padded to 320 input channels it takes 54 us
            # (scripts/condout_probe.py)
            x, w = self._pad_cin(name, x, w, to=320)
        if (stride == 2 and w.shape[-1] == 3 and x.dim() == 4 and x.shape[-1] >= 128 and x.shape[1] >= 256
                and x.shape[0] <= 4 and x.dtype != torch.float32):
            # cuDNN has no good bf16 kernel for the 3x3 stride-2 downsample at
            # 128x128 (SDXL's first: 155 us, a TF32 fallback with conversions);
            # the stride-1 conv + subsample computes 4x the outputs and still
            # takes 59 us (scripts/convds_probe.py).  At CFG batch 16 cuDNN's
            # strided kernel is fine (104 us, scripts/conv_shapes_probe.py NB=16)
            y = F.conv2d(x, w, self.t.get(name + ".bias") if bias else None, stride=1, padding=pad)
            return y[:, :, ::2, ::2].contiguous(memory_format=torch.channels_last)
        return F.conv2d(x, w, self.t.get(name + ".bias") if bias else None, stride=stride, padding=pad)

    def _pad_cin(self, name, x, w, to=None):
        """conv_in's 4 latent channels (and the ControlNet hint's 3 image
        channels): cuDNN has no bf16 tensor-op kernel for C_in % 8 != 0 and
        falls back to convert -> TF32 conv -> convert (49 us per SDXL conv_in,
        3 per step; 152 us per hint conv).  Padded to 16 channels, incl. the
        copies: ~24 us and ~90 us (scripts/convin_probe.py; 16 beat 8, which
        still made cuDNN insert its own padding pass).  Zero-pad C_in to a multiple
        of 16 in persistent buffers (the padding channels stay zero; each call
        copies the live input and the live weight — the LoRA shadow or the
        pristine one, whichever the graph captured — into the first C_in)."""
        cin = w.shape[1]
        cp = to if to is not None else (cin + 15) // 16 * 16
        key = (name, tuple(x.shape), tuple(w.shape), x.dtype)
        bufs = getattr(self, "_cin_pad", None)
        if bufs is None:
            bufs = self._cin_pad = {}
        if key not in bufs:
            xp = torch.zeros((x.shape[0], cp) + tuple(x.shape[2:]), device=x.device, dtype=x.dtype)
            wp = torch.zeros((w.shape[0], cp) + tuple(w.shape[2:]), device=w.device, dtype=w.dtype)
            bufs[key] = (xp.contiguous(memory_format=torch.channels_last),
                         wp.contiguous(memory_format=torch.channels_last))
        xp, wp = bufs[key]
        xp[:, :cin].copy_(x)
        wp[:, :cin].copy_(w)
        return xp, wp

    def conv1x1(self, name, x, out=None):
        """A 1x1 convolution on NHWC storage is a GEMM over pixels: cuBLAS with
        the bias in its epilogue, optionally straight into ``out`` (an NHWC
        view, e.g. a slot of the CaaS residual buffer)."""
        w = self.t[name + ".weight"]
        n, c, hh, ww = x.shape
        cout = w.shape[0]
        x2 = x.permute(0, 2, 3, 1).reshape(n * hh * ww, c)
        w2 = w.reshape(cout, c)              # channels_last [Cout, 1, 1, Cin] memory == (Cout, Cin)
        b = self.t.get(name + ".bias")
        if out is None:
            y = F.linear(x2, w2, b)
        else:
            y = out.permute(0, 2, 3, 1).reshape(n * hh * ww, cout)
            assert y.data_ptr() == out.data_ptr(), "out must be an NHWC (channels_last) buffer"
            if b is None:
                torch.mm(x2, w2.t(), out=y)
            else:
                torch.addmm(b, x2, w2.t(), out=y)
        return y.view(n, hh, ww, cout).permute(0, 3, 1, 2)

    def conv_bias_inplace(self, name, x, stride=1):
        """3x3 conv whose bias has no fusable consumer: bias-free conv + K3's
        vectorised in-place per-channel add."""
        h = self.conv(name, x, stride=stride, bias=False)
        return ops.residual_inject(h, [], [], skip_bias=self.fb.get(name), gn_workspace=self.k3ws(name, h),
                                   groups=self.cfg.groups)

    def k3ws(self, key, x, channels: Optional[int] = None):
        """GroupNorm-statistics workspace of one K3 call site whose output is
        the next GroupNorm's input (the K3 pass publishes its statistics).
        Sized for the K3 OUTPUT: x's batch and pixels with ``channels``
        channels (the concat's hidden + skip) when given."""
        if _NO_K3_STATS:
            return None
        k = ("k3", key, tuple(x.shape), channels)
        ws = self._gn_ws.get(k)
        if ws is None:
            ws = self._gn_ws[k] = ops.groupnorm_workspace(x, self.cfg.groups, channels)
        return ws

    def gn(self, name, x, silu, eps=None, add_nc=None):
        # one K2 workspace per (site, shape) of THIS network: graphs of different
        # networks (UNet, ControlNets) may replay concurrently on other streams
        key = (name, tuple(x.shape))
        ws = self._gn_ws.get(key)
        if ws is None:
            ws = self._gn_ws[key] = ops.groupnorm_workspace(x, self.cfg.groups)
        return ops.groupnorm_silu(x, self.t[name + ".weight"], self.t[name + ".bias"],
                                  groups=self.cfg.groups, eps=self.cfg.gn_eps if eps is None else eps,
                                  silu=silu, add_nc=add_nc, workspace=ws)

    # -- blocks -----------------------------------------------------------
    def resnet(self, pre, x, temb_act, gn_next: bool = True):
        """gn_next: the block's output is the input of a GroupNorm (the next
        ResNet's norm1 or a transformer's norm): only then does the closing K3
        pass also publish that GroupNorm's statistics."""
        h = self.conv(pre + ".conv1", self.gn(pre + ".norm1", x, True), bias=False)
        # conv1's bias rides on the time-embedding projection (tproj_bias = b_temb + b_conv1)
        wt, tb = self.t[pre + ".time_emb_proj.weight"], self.fb.get(pre + ".tproj_bias")
        if temb_act.dtype == torch.float32:
            tproj = F.linear(temb_act, wt, tb).contiguous()
        elif tb is not None:   # fp32 accumulate-and-store in cuBLAS (torch still broadcasts the bias first)
            tproj = torch.addmm(self.fb[pre + ".tproj_bias_f32"], temb_act, wt.t(), out_dtype=torch.float32)
        else:
            tproj = torch.mm(temb_act, wt.t(), out_dtype=torch.float32)
        h = self.gn(pre + ".norm2", h, True, add_nc=tproj)       # fused temb add + GN + SiLU
        h = self.conv(pre + ".conv2", h, bias=False)
        if (pre + ".conv_shortcut.weight") in self.t:
            w = self.t[pre + ".conv_shortcut.weight"]
            sc = self.conv1x1(pre + ".conv_shortcut", x) if w.shape[-1] == 1 else \
                self.conv(pre + ".conv_shortcut", x, bias=False)
            bias = self.fb.get(pre + ".conv2") if w.shape[-1] == 1 else self.fb.get(pre + ".out_bias")
        else:
            sc, bias = x, self.fb.get(pre + ".conv2")
        # K3 in-place add (NHWC, vectorised) with conv2's (+ shortcut's) bias folded,
        # accumulating the next GroupNorm's statistics of the block output
        return ops.residual_inject(h, [sc], [1.0], skip_bias=bias,
                                   gn_workspace=self.k3ws(pre, h) if gn_next else None, groups=self.cfg.groups)

    def attention(self, pre, x, ctx, heads):
        n, l, c = x.shape
        if ctx is None:   # self-attention: one GEMM for q, k, v (fused weight storage)
            qkv = F.linear(x, self.t[pre + ".to_qkv.weight"])
            if _SELF_ATTN and qkv.is_cuda and ops.self_attention_supported(qkv, heads):
                # K8: flash-style tcgen05 attention straight off the fused projection
                return self.lin(pre + ".to_out", ops.self_attention(qkv, heads))
            q, k, v = qkv.split(c, dim=-1)
        else:             # cross-attention: q from x, one GEMM for k, v from the context
            q = self.lin(pre + ".to_q", x)
            kv = self.kv[self.kv_slot][pre] if self.kv_slot is not None else F.linear(ctx, self.t[pre + ".to_kv.weight"])
            if q.is_cuda and ops.cross_attention_supported(q, kv, heads):
                # K7: 77-token context staged in smem, exact softmax, one pass over q
                return self.lin(pre + ".to_out", ops.cross_attention(q, kv, heads))
            k, v = kv.split(c, dim=-1)
        d = c // heads
        q = q.view(n, l, heads, d).transpose(1, 2)
        k = k.view(n, -1, heads, d).transpose(1, 2)
        v = v.view(n, -1, heads, d).transpose(1, 2)
        if ctx is not None and q.is_cuda and q.dtype != torch.float32:
            # 77-token cross-attention: the flash kernel beats cuDNN's pick
            # (scripts/attn_probe.py on B200: 15.6 vs 18.7 us at 32x32)
            with sdpa_kernel([SDPBackend.FLASH_ATTENTION, SDPBackend.CUDNN_ATTENTION]):
                o = F.scaled_dot_product_attention(q, k, v)
        else:
            o = F.scaled_dot_product_attention(q, k, v)
        o = o.transpose(1, 2).reshape(n, l, c)
        return self.lin(pre + ".to_out", o)

    def transformer(self, pre, x, ctx, depth, gn_next: bool = True):
        n, c, h, w = x.shape
        res = x
        hs = self.gn(pre + ".norm", x, False, eps=self.cfg.tf_gn_eps)
        tok = hs.permute(0, 2, 3, 1).reshape(n, h * w, c)       # NHWC storage: a free view
        tok = self.lin(pre + ".proj_in", tok)
        heads = self.cfg.heads(c)
        delta = None   # pending residual: fused into the next block's add + LayerNorm (K6)
        for d in range(depth):
            b = f"{pre}.blocks.{d}"
            ln = lambda k, dl: ops.add_layernorm(tok, dl, self.t[f"{b}.{k}.weight"], self.t[f"{b}.{k}.bias"])
            y = ln("norm1", delta)
            y = ln("norm2", self.attention(b + ".attn1", y, None, heads))
            y = ln("norm3", self.attention(b + ".attn2", y, ctx, heads))
            delta = self.lin(b + ".ff.out", self.ff_proj_geglu(b + ".ff.proj", y))
        tok = ops.residual_inject(tok, [delta], [1.0])
        tok = self.lin(pre + ".proj_out", tok)
        out = tok.view(n, h, w, c).permute(0, 3, 1, 2)            # channels_last view
        return ops.residual_inject(out, [res], [1.0], gn_workspace=self.k3ws(pre, out) if gn_next else None,
                                   groups=self.cfg.groups)

    # -- embeddings ---------------------------------------------------------
    def add_embedding(self, pooled: torch.Tensor, time_ids: torch.Tensor) -> torch.Tensor:
        """SDXL text_time embedding — step-invariant, computed once per request."""
        cfg = self.cfg
        n = pooled.shape[0]
        tid = timestep_embedding(time_ids.reshape(-1), cfg.addition_time_embed_dim).reshape(n, -1)
        a = torch.cat([pooled.float(), tid], dim=-1).to(self.p.dtype)
        return self.lin("add_embedding.linear_2", F.silu(self.lin("add_embedding.linear_1", a)))

    def time_embedding(self, t: torch.Tensor, batch: int, add_emb: Optional[torch.Tensor]):
        te = timestep_embedding(t.reshape(-1)[:1].expand(batch), self.cfg.block_channels[0]).to(self.p.dtype)
        emb = self.lin("time_embedding.linear_2", F.silu(self.lin("time_embedding.linear_1", te)))
        if add_emb is not None:
            emb = emb + add_emb
        return F.silu(emb)   # every consumer (time_emb_proj) applies SiLU first

    # -- encoder ------------------------------------------------------------
    def encode(self, x, temb_act, ctx, hint=None, on_skip=None):
        """conv_in + down blocks + mid; returns (mid, [skips]).  on_skip(k, h)
        is called as soon as skip k exists (the ControlNet's zero convs and
        per-level pushes hang off it)."""
        cfg = self.cfg
        if hint is not None:   # conv_in + bias + the ControlNet hint in one K3 pass
            h = self.conv("conv_in", x, bias=False)
            h = ops.residual_inject(h, [hint], [1.0], skip_bias=self.fb.get("conv_in"),
                                    gn_workspace=self.k3ws("conv_in", h), groups=self.cfg.groups)
        else:
            h = self.conv_bias_inplace("conv_in", x)
        skips = []

        def skip(h):
            skips.append(h)
            if on_skip is not None:
                on_skip(len(skips) - 1, h)
        skip(h)
        n = len(cfg.block_channels)
        for i in range(n):
            for j in range(cfg.layers_per_block):
                # a GroupNorm reads this output next unless a downsample conv does
                nxt_gn = j < cfg.layers_per_block - 1 or i == n - 1
                h = self.resnet(f"down.{i}.res.{j}", h, temb_act, gn_next=nxt_gn or bool(cfg.attn_depth[i]))
                if cfg.attn_depth[i]:
                    h = self.transformer(f"down.{i}.attn.{j}", h, ctx, cfg.attn_depth[i], gn_next=nxt_gn)
                skip(h)
            if i < n - 1:
                h = self.conv_bias_inplace(f"down.{i}.downsample", h, stride=2)
                skip(h)
        h = self.resnet("mid.res.0", h, temb_act)
        h = self.transformer("mid.attn.0", h, ctx, cfg.mid_depth)
        # the UNet decoder adds the mid residuals / the ControlNet's zero conv reads it: no GroupNorm
        h = self.resnet("mid.res.1", h, temb_act, gn_next=False)
        return h, skips


class UNet(Net):
    def decode(self, h, skips, temb_act, ctx, residuals=None, res_scales=None):
        """Up path.  ``residuals``: per ControlNet, a list of down residuals
        (same order as skips) + a mid residual, scaled by ``res_scales``; they
        are injected by K3 while the skip concat is written."""
        cfg = self.cfg
        nres = 0 if residuals is None else len(residuals)
        if nres:
            ops.residual_inject(h, [r[-1] for r in residuals], res_scales)       # mid (in place)
        rev = list(reversed(cfg.block_channels))
        n = len(rev)
        k = len(skips)
        hb = None   # pending bias of the upsample conv that produced h (folded into K3's hidden part)
        for i, c in enumerate(rev):
            depth = cfg.attn_depth[n - 1 - i]
            for j in range(cfg.layers_per_block + 1):
                k -= 1
                res_k = [r[k] for r in residuals] if nres else []
                h = ops.residual_inject(skips[k], res_k, res_scales if nres else [], hidden=h, hidden_bias=hb,
                                        gn_workspace=self.k3ws(f"up.{i}.cat.{j}", skips[k],
                                                               h.shape[1] + skips[k].shape[1]),
                                        groups=self.cfg.groups)
                hb = None
                # next: the transformer's norm, the next concat (K3, computes its own
                # statistics), the upsample conv, or conv_norm_out after the last block
                last = i == n - 1 and j == cfg.layers_per_block
                h = self.resnet(f"up.{i}.res.{j}", h, temb_act, gn_next=bool(depth) or last)
                if depth:
                    h = self.transformer(f"up.{i}.attn.{j}", h, ctx, depth, gn_next=last)
            if i < n - 1:
                h = ops.upsample2x(_cl(h))                      # K10 (nearest 2x, NHWC)
                h = self.conv(f"up.{i}.upsample", h, bias=False)
                hb = self.fb.get(f"up.{i}.upsample")
        h = self.gn("conv_norm_out", h, True)
        # eps leaves the UNet in fp32: CFG amplifies (eps_c - eps_u) by the
        # guidance scale, so a bf16 rounding here would dominate the latent error
        w = self.t["conv_out.weight"]
        b = self.t.get("conv_out.bias")
        if ops.conv_out_supported(h, w):
            return ops.conv_out(h, w, self.fb.get("conv_out"))       # K9, fp32 accumulate
        return F.conv2d(h.float(), w.float(), None if b is None else b.float(), padding=w.shape[-1] // 2)

    def forward(self, x, t, ctx, add_emb=None, residuals=None, res_scales=None):
        temb_act = self.time_embedding(t, x.shape[0], add_emb)
        h, skips = self.encode(x, temb_act, ctx)
        return self.decode(h, skips, temb_act, ctx, residuals, res_scales)


class ControlNet(Net):
    def hint_embedding(self, image: torch.Tensor) -> torch.Tensor:
        """Conditioning image (N, 3, 8H, 8W) -> (N, C0, H, W).  Step-invariant:
        computed once per request (SURVEY App. B pitfall 8)."""
        hc = self.cfg.hint_channels
        h = F.silu(self._conv_bias("cond_embedding.conv_in", _cl(image)), inplace=True)
        for i in range(len(hc) - 1):
            h = F.silu(self._conv_bias(f"cond_embedding.blocks.{2 * i}", h), inplace=True)
            h = F.silu(self._conv_bias(f"cond_embedding.blocks.{2 * i + 1}", h, stride=2), inplace=True)
        return self._conv_bias("cond_embedding.conv_out", h)

    def _conv_bias(self, name, x, stride=1):
        """Bias-free cuDNN conv + K3's vectorised in-place per-channel bias add
        (cuDNN's own channels_last bias pass is a non-vectorised broadcast add:
        ~70 us per 1024x1024 hint map)."""
        h = self.conv(name, x, stride=stride, bias=False)
        b = self.fb.get(name)
        if b is None or h.shape[1] % 8 != 0:
            return h if b is None else h.add_(self.t[name + ".bias"].view(1, -1, 1, 1))
        return ops.residual_inject(h, [], [], skip_bias=b, out=h)

    def forward(self, x, t, ctx, hint, add_emb=None, outs=None, on_level=None):
        """Returns [down residuals..., mid residual] (unscaled; the
        conditioning scale is applied by K3 on the consumer side).  The zero
        convs are 1x1: cuBLAS GEMMs (bias in the epilogue), written straight
        into ``outs`` (NHWC views, e.g. the CaaS send buffer) when given.
        Each level's zero conv runs as soon as its skip exists, and
        on_level(k, out_k) lets the caller push it to the base right away —
        shallow levels (the largest) first, overlapped with the deeper levels'
        compute (SURVEY App. B pitfall 7)."""
        temb_act = self.time_embedding(t, x.shape[0], add_emb)
        res = []

        def level(k, s, name):
            r = self.zero_conv(name, s, None if outs is None else outs[k])
            res.append(r)
            if on_level is not None:
                on_level(k, r)
        h, skips = self.encode(x, temb_act, ctx, hint=hint, on_skip=lambda k, s: level(k, s, f"zero_convs.{k}"))
        level(len(skips), h, "mid_zero_conv")
        return res

    def zero_conv(self, name, x, out=None):
        if self.t[name + ".weight"].shape[-1] == 1:
            return self.conv1x1(name, x, out)
        y = self.conv(name, x)
        if out is not None:
            out.copy_(y)
            return out
        return y


def patchable_matrices(params: Params) -> list[tuple[str, torch.Tensor]]:
    """Every LoRA target of a UNet as (name, (h1, h2) matrix view)."""
    return [(name, params.matrix_view(name)) for name, _ in params.matrices]
