"""CPU fp32 oracle of the denoising loop — TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED at the latent level: the reference (addonsim) has no UNet,
ControlNet, CFG or scheduler arithmetic, so this is a
builder-authored restatement of the same architecture in plain eager torch
(CPU, fp32, NCHW) over the SAME parameter values as the device model, written
independently of paper_2407_02031_b200/unet.py's kernels:

* GroupNorm/SiLU: F.group_norm + F.silu          (device: K2, NHWC, fused temb add)
* skip concat + ControlNet residuals: torch.cat of skip + sum s_i r_i
                                                  (device: K3)
* CFG + DDIM: float64 formulas                    (device: K4)
* LoRA: oracle.lora_ref.accumulate (the pinned restatement of
  addonsim/lora.py:84-95) on the LOGICAL (Cout, Cin*kh*kw) matrices at a
  FORCED boundary k: steps 1..k unpatched, k+1.. patched
  (addonsim/orchestrator.py:227-241 first_patched_step = k + 1)
* ControlNet outputs summed into skips and mid, decoder after
  every branch (orchestrator.py:652-653)
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from . import lora_ref


def to_cpu_params(params, dtype=torch.float32) -> dict:
    """Device Params -> {name: CPU NCHW-contiguous tensor} (fp32; fp64 for the
    rounding-floor measurements)."""
    return {k: v.detach().cpu().to(dtype).contiguous() for k, v in params.t.items()}


def ddim_coefs(steps: int, guidance: float):
    betas = np.linspace(0.00085 ** 0.5, 0.012 ** 0.5, 1000, dtype=np.float64) ** 2
    ac = np.cumprod(1.0 - betas)
    ratio = 1000 // steps
    ts = (np.arange(steps) * ratio)[::-1] + 1
    return [(int(t), ac[t], ac[t - ratio] if t - ratio >= 0 else ac[0]) for t in ts]


class RefNet:
    """bf16_acts=True rounds every linear / conv / norm output to bf16 (fp32
    math in between; the UNet's eps stays fp32 as on the device) and the
    merged LoRA weights to bf16: the error floor of a bf16-activation
    implementation, used to bound the device bf16 path
    (tests/test_pipeline_gpu.py, tests/test_sdxl_engine_gpu.py)."""

    def __init__(self, cfg, p: dict, bf16_acts: bool = False):
        self.cfg, self.p = cfg, p
        self.dt = next(iter(p.values())).dtype      # fp32 (fp64: the truth the fp32 floor is measured against)
        self.rnd = (lambda t: t.bfloat16().float()) if bf16_acts else (lambda t: t)

    def lin(self, n, x):
        return self.rnd(F.linear(x, self.p[n + ".weight"], self.p.get(n + ".bias")))

    def conv(self, n, x, stride=1):
        w = self.p[n + ".weight"]
        return self.rnd(F.conv2d(x, w, self.p.get(n + ".bias"), stride=stride, padding=w.shape[-1] // 2))

    def gn(self, n, x, silu, eps=None):
        y = F.group_norm(x, self.cfg.groups, self.p[n + ".weight"], self.p[n + ".bias"],
                         self.cfg.gn_eps if eps is None else eps)
        return self.rnd(F.silu(y) if silu else y)

    def temb(self, t, n, add_emb):
        half = self.cfg.block_channels[0] // 2
        freqs = torch.exp(-math.log(10000.0) * torch.arange(half, dtype=self.dt) / half)
        a = float(t) * freqs
        te = torch.cat([torch.cos(a), torch.sin(a)])[None].expand(n, -1)
        e = self.lin("time_embedding.linear_2", F.silu(self.lin("time_embedding.linear_1", te)))
        if add_emb is not None:
            e = e + add_emb
        return F.silu(e)

    def add_embedding(self, pooled, time_ids):
        d = self.cfg.addition_time_embed_dim
        half = d // 2
        freqs = torch.exp(-math.log(10000.0) * torch.arange(half, dtype=self.dt) / half)
        a = time_ids.reshape(-1, 1).to(self.dt) * freqs[None]
        tid = torch.cat([torch.cos(a), torch.sin(a)], -1).reshape(pooled.shape[0], -1)
        x = torch.cat([pooled.to(self.dt), tid], -1)
        return self.lin("add_embedding.linear_2", F.silu(self.lin("add_embedding.linear_1", x)))

    def resnet(self, pre, x, temb):
        h = self.conv(pre + ".conv1", self.gn(pre + ".norm1", x, True))
        h = h + self.lin(pre + ".time_emb_proj", temb)[:, :, None, None]
        h = self.conv(pre + ".conv2", self.gn(pre + ".norm2", h, True))
        sc = self.conv(pre + ".conv_shortcut", x) if pre + ".conv_shortcut.weight" in self.p else x
        return self.rnd(h + sc)

    def attn(self, pre, x, ctx, heads):
        n, l, c = x.shape
        src = x if ctx is None else ctx
        q, k, v = self.lin(pre + ".to_q", x), self.lin(pre + ".to_k", src), self.lin(pre + ".to_v", src)
        d = c // heads
        q = q.view(n, l, heads, d).transpose(1, 2)
        k = k.view(n, -1, heads, d).transpose(1, 2)
        v = v.view(n, -1, heads, d).transpose(1, 2)
        o = self.rnd(F.scaled_dot_product_attention(q, k, v))  # CPU: softmax(q k^T / sqrt(d)) v
        return self.lin(pre + ".to_out", o.transpose(1, 2).reshape(n, l, c))

    def transformer(self, pre, x, ctx, depth):
        n, c, h, w = x.shape
        tok = self.gn(pre + ".norm", x, False, self.cfg.tf_gn_eps).permute(0, 2, 3, 1).reshape(n, h * w, c)
        tok = self.lin(pre + ".proj_in", tok)
        heads = self.cfg.heads(c)
        for d in range(depth):
            b = f"{pre}.blocks.{d}"
            ln = lambda k, t: self.rnd(F.layer_norm(t, (c,), self.p[f"{b}.{k}.weight"], self.p[f"{b}.{k}.bias"]))
            tok = self.rnd(tok + self.attn(b + ".attn1", ln("norm1", tok), None, heads))
            tok = self.rnd(tok + self.attn(b + ".attn2", ln("norm2", tok), ctx, heads))
            hv, gate = self.lin(b + ".ff.proj", ln("norm3", tok)).chunk(2, -1)
            tok = self.rnd(tok + self.lin(b + ".ff.out", self.rnd(hv * F.gelu(gate))))
        tok = self.lin(pre + ".proj_out", tok)
        return self.rnd(tok.view(n, h, w, c).permute(0, 3, 1, 2) + x)

    def encode(self, x, temb, ctx, hint=None):
        cfg = self.cfg
        h = self.conv("conv_in", x)
        if hint is not None:
            h = h + hint
        skips = [h]
        for i in range(len(cfg.block_channels)):
            for j in range(cfg.layers_per_block):
                h = self.resnet(f"down.{i}.res.{j}", h, temb)
                if cfg.attn_depth[i]:
                    h = self.transformer(f"down.{i}.attn.{j}", h, ctx, cfg.attn_depth[i])
                skips.append(h)
            if i < len(cfg.block_channels) - 1:
                h = self.conv(f"down.{i}.downsample", h, 2)
                skips.append(h)
        h = self.resnet("mid.res.0", h, temb)
        h = self.transformer("mid.attn.0", h, ctx, cfg.mid_depth)
        return self.resnet("mid.res.1", h, temb), skips


class RefUNet(RefNet):
    def forward(self, x, t, ctx, add_emb, residuals, scales):
        cfg = self.cfg
        temb = self.temb(t, x.shape[0], add_emb)
        h, skips = self.encode(x, temb, ctx)
        for r, s in zip(residuals, scales):
            skips = [sk + s * rr for sk, rr in zip(skips, r[:-1])]
            h = h + s * r[-1]
        skips = [self.rnd(sk) for sk in skips]
        h = self.rnd(h)
        rev = list(reversed(cfg.block_channels))
        for i, _ in enumerate(rev):
            depth = cfg.attn_depth[len(rev) - 1 - i]
            for j in range(cfg.layers_per_block + 1):
                h = torch.cat([h, skips.pop()], dim=1)
                h = self.resnet(f"up.{i}.res.{j}", h, temb)
                if depth:
                    h = self.transformer(f"up.{i}.attn.{j}", h, ctx, depth)
            if i < len(rev) - 1:
                h = self.conv(f"up.{i}.upsample", F.interpolate(h, scale_factor=2.0, mode="nearest"))
        # eps leaves the device UNet in fp32 (K9): no bf16 rounding of conv_out
        w = self.p["conv_out.weight"]
        return F.conv2d(self.gn("conv_norm_out", h, True), w, self.p.get("conv_out.bias"), padding=w.shape[-1] // 2)


class RefControlNet(RefNet):
    def hint(self, image):
        hc = self.cfg.hint_channels
        h = F.silu(self.conv("cond_embedding.conv_in", image))
        for i in range(len(hc) - 1):
            h = F.silu(self.conv(f"cond_embedding.blocks.{2 * i}", h))
            h = F.silu(self.conv(f"cond_embedding.blocks.{2 * i + 1}", h, 2))
        return self.conv("cond_embedding.conv_out", h)

    def forward(self, x, t, ctx, hint, add_emb):
        temb = self.temb(t, x.shape[0], add_emb)
        h, skips = self.encode(x, temb, ctx, hint)
        return [self.conv(f"zero_convs.{k}", s) for k, s in enumerate(skips)] + [self.conv("mid_zero_conv", h)]


def merge_loras(p: dict, adapters, matrices, round_bf16: bool = False) -> dict:
    """Patched copy of the UNet params: for every target, W_logical (Cout,
    Cin*kh*kw) += stacked adapters via the pinned lora_ref (fp64 accumulate).
    adapters: [(factors{name: (down, up)} with LOGICAL up, scale)].
    round_bf16: store the merged weights rounded to bf16 (a bf16 weight
    store's single rounding, lora_ref.accumulate_bf16's contract)."""
    out = dict(p)
    for name, _ in matrices:
        present = [(f[name], s) for f, s in adapters if name in f]
        if not present:
            continue
        w = p[name + ".weight"]
        wl = w.reshape(w.shape[0], -1).float().numpy().copy()   # the reference merges fp32 weights
        down, up = lora_ref.stack([(d.float().cpu().numpy(), u.float().cpu().numpy(), s) for (d, u), s in present])
        lora_ref.accumulate(wl, down, up, 1.0, 1.0)
        merged = torch.from_numpy(wl).reshape(w.shape).to(w.dtype)
        out[name + ".weight"] = merged.bfloat16().float() if round_bf16 else merged
    return out


def denoise(cfg, unet_p: dict, cn_ps: list, req, cn_scales, steps: int, guidance: float,
            adapters=None, matrices=None, boundary=None, bf16_acts: bool = False,
            groups=None, group_boundaries=None, max_steps=None) -> list:
    """Returns the fp32 [4, H, W] latent after every step (the first
    ``max_steps`` steps of the ``steps``-step schedule when given).

    groups / group_boundaries: group-pipelined patching
    (addonsim/orchestrator.py:244-278) — matrix group m (a set of names) is
    patched after step group_boundaries[m] (None = never); the steps in
    between run a UNet with only the groups patched so far merged."""
    unet = RefUNet(cfg, unet_p, bf16_acts)
    if groups is not None and adapters:
        nets, firsts = [unet], []
        for v in range(1, len(groups) + 1):
            names = set().union(*groups[:v])
            nets.append(RefUNet(cfg, merge_loras(unet_p, adapters, [m for m in matrices if m[0] in names],
                                                 bf16_acts), bf16_acts))
            b = group_boundaries[v - 1]
            firsts.append(steps + 1 if b is None else b + 1)

        def pick(s):
            return nets[sum(1 for f in firsts if s >= f)]
    else:
        patched = RefUNet(cfg, merge_loras(unet_p, adapters, matrices, bf16_acts), bf16_acts) if adapters else None
        first = (boundary + 1) if (adapters and boundary is not None) else steps + 1

        def pick(s):
            return patched if (patched is not None and s >= first) else unet
    cns = [RefControlNet(cfg, p, bf16_acts) for p in cn_ps]
    dt = unet.dt
    ctx = torch.from_numpy(req.context).to(dt)
    add_u = add_c = None
    if cfg.addition_embed:
        pooled, tids = torch.from_numpy(req.pooled), torch.from_numpy(req.time_ids)
        add_u = unet.add_embedding(pooled, tids)
        add_c = [cn.add_embedding(pooled, tids) for cn in cns]
    hints = [cn.hint(torch.from_numpy(im).to(dt)) for cn, im in zip(cns, req.images)]
    x = torch.from_numpy(req.latent).double()
    out = []
    for s, (t, a_t, a_p) in enumerate(ddim_coefs(steps, guidance), start=1):
        if max_steps is not None and s > max_steps:
            break
        inp = x.to(dt)[None].expand(2, -1, -1, -1)
        res = [cn.forward(inp, t, ctx, hints[i], add_c[i] if add_c else None) for i, cn in enumerate(cns)]
        net = pick(s)
        eps = net.forward(inp, t, ctx, add_u, res, cn_scales).double()
        e = eps[0] + guidance * (eps[1] - eps[0])
        x0 = (x - math.sqrt(1 - a_t) * e) / math.sqrt(a_t)
        x = math.sqrt(a_p) * x0 + math.sqrt(1 - a_p) * e
        out.append(x.float().clone())
    return out
