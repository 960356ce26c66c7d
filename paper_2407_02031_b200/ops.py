"""Torch-facing wrappers over the C-ABI kernels (device tensors in, no copies).

PyTorch supplies device memory and streams; every arithmetic op on this path
is a hand-written sm_100a kernel in libsdb.so.  Inputs must already be CUDA
tensors — there is deliberately no CPU branch (a CPU tensor raises).
"""

from __future__ import annotations

import contextlib
import ctypes
from typing import Optional, Sequence

import torch

from . import _lib
from .errors import DeviceError, ValidationError

_DTYPES = {torch.float32: _lib.SDB_F32, torch.bfloat16: _lib.SDB_BF16, torch.float16: _lib.SDB_F16}
_checked_devices: set[int] = set()

#: kernels issued by this process through the C-ABI (a CUDA-graph capture
#: counts the launches its replays will issue).  bench.py reports it.
LAUNCHES = {"count": 0}


def _count(n: int) -> None:
    LAUNCHES["count"] += n


def sdb_dtype(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise ValidationError(f"unsupported dtype {t.dtype}") from None


def require_cuda(*tensors: torch.Tensor) -> None:
    """Fail loudly unless every tensor lives on an sm_100 CUDA device."""
    for t in tensors:
        if t is None:
            continue
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise DeviceError("paper_2407_02031_b200 kernels need CUDA tensors on a B200 "
                              "(sm_100); there is no CPU fallback")
        dev = t.device.index if t.device.index is not None else torch.cuda.current_device()
        if dev not in _checked_devices:
            if not _lib.lib().sdb_device_ok(dev):
                raise DeviceError(f"cuda:{dev} is not an sm_100 (Blackwell B200) device")
            _checked_devices.add(dev)


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# --------------------------------------------------------------------------
# K1 — LoRA patch
# --------------------------------------------------------------------------
def _row_stride(t: torch.Tensor, what: str) -> int:
    if t.dim() != 2:
        raise ValidationError(f"{what} must be 2-d, got shape {tuple(t.shape)}")
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise ValidationError(f"{what} must have unit column stride")
    return max(t.stride(0), t.shape[1])


def lora_patch_one(w_in: torch.Tensor, down: torch.Tensor, up: torch.Tensor, scale: float,
                   sign: float = 1.0, w_out: Optional[torch.Tensor] = None,
                   stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """W_out = W_in + sign*scale*down@up on one matrix (in place if w_out is None)."""
    require_cuda(w_in, down, up, w_out)
    out = w_in if w_out is None else w_out
    if out.shape != w_in.shape or out.stride() != w_in.stride() or out.dtype != w_in.dtype:
        raise ValidationError("w_out must match w_in in shape, stride and dtype")
    if down.dtype != up.dtype:
        raise ValidationError("down and up must share a dtype")
    h1, h2 = w_in.shape
    if down.shape[0] != h1 or up.shape[1] != h2 or down.shape[1] != up.shape[0]:
        raise ValidationError(f"factor shapes {tuple(down.shape)} x {tuple(up.shape)} do not match "
                              f"weight ({h1}, {h2})")
    _count(1)
    _lib.check("sdb_lora_patch_one", _lib.lib().sdb_lora_patch_one(
        w_in.data_ptr(), out.data_ptr(), h1, h2, _row_stride(w_in, "weight"),
        down.data_ptr(), _row_stride(down, "down"), up.data_ptr(), _row_stride(up, "up"),
        int(down.shape[1]), float(scale), float(sign), sdb_dtype(w_in), sdb_dtype(down),
        _stream_ptr(stream)))
    return out


class LoraPatchPlan:
    """A planned, device-resident job table for one batched K1 launch.

    entries: sequence of (w_in, w_out or None, down, up, scale).  All weights
    share one dtype and all factors another.  The table (a packed array of
    ``sdb_lora_job``) is uploaded once; ``launch`` is then a single kernel
    launch, capturable in a CUDA graph and cheap enough to run on a side
    stream at every patch event.
    """

    def __init__(self, entries: Sequence[tuple], device: Optional[torch.device] = None):
        if not entries:
            raise ValidationError("LoraPatchPlan needs at least one job")
        jobs = (_lib.LoraJob * len(entries))()
        w_dt = f_dt = None
        self._keep = []  # keep tensors alive as long as the plan
        self.alg_bytes = 0
        self.alg_flops = 0
        for i, (w_in, w_out, down, up, scale) in enumerate(entries):
            out = w_in if w_out is None else w_out
            require_cuda(w_in, out, down, up)
            if w_dt is None:
                w_dt, f_dt = sdb_dtype(w_in), sdb_dtype(down)
            if sdb_dtype(w_in) != w_dt or sdb_dtype(out) != w_dt or sdb_dtype(down) != f_dt \
                    or sdb_dtype(up) != f_dt:
                raise ValidationError("all jobs of a plan must share weight and factor dtypes")
            h1, h2 = w_in.shape
            r = down.shape[1]
            if down.shape[0] != h1 or up.shape[1] != h2 or up.shape[0] != r:
                raise ValidationError(f"job {i}: factor shapes {tuple(down.shape)} x {tuple(up.shape)} "
                                      f"do not match weight ({h1}, {h2})")
            if out.stride() != w_in.stride():
                raise ValidationError(f"job {i}: w_out stride differs from w_in")
            j = jobs[i]
            j.w_in, j.w_out = w_in.data_ptr(), out.data_ptr()
            j.down, j.up = down.data_ptr(), up.data_ptr()
            j.h1, j.h2 = h1, h2
            j.ldw = _row_stride(w_in, "weight")
            j.ldd = _row_stride(down, "down")
            j.ldu = _row_stride(up, "up")
            j.rank = r
            j.scale = float(scale)
            self._keep += [w_in, out, down, up]
            ws, fs = w_in.element_size(), down.element_size()
            self.alg_bytes += 2 * h1 * h2 * ws + (h1 + h2) * r * fs
            self.alg_flops += 2 * h1 * h2 * r
        total = ctypes.c_int64(0)
        path = ctypes.c_int(0)
        _lib.check("sdb_lora_plan", _lib.lib().sdb_lora_plan(
            jobs, len(entries), w_dt, f_dt, ctypes.byref(total), ctypes.byref(path)))
        raw = bytes(jobs)
        dev = device if device is not None else entries[0][0].device
        self.table = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
        self.n_jobs = len(entries)
        self.total_tiles = total.value
        self.path = path.value
        self.w_dtype, self.f_dtype = w_dt, f_dt

    def launch(self, sign: float = 1.0, stream: Optional[torch.cuda.Stream] = None,
               max_ctas: int = 0) -> None:
        _count(1)
        _lib.check("sdb_lora_patch", _lib.lib().sdb_lora_patch(
            self.table.data_ptr(), self.n_jobs, self.total_tiles, self.w_dtype, self.f_dtype,
            self.path, float(sign), int(max_ctas), _stream_ptr(stream)))


def tma_eligible(w: torch.Tensor) -> bool:
    """bf16 matrix whose rows are 16-B aligned: the TMA / tcgen05 K1 path applies."""
    return (w.dtype == torch.bfloat16 and w.dim() == 2 and w.stride(1) == 1
            and _row_stride(w, "weight") % 8 == 0 and w.data_ptr() % 16 == 0)


@contextlib.contextmanager
def lora_kernel_mode(mode: int):
    """Force the K1 kernel for LoraTmaPlans built inside the block: 0 auto
    (= CTA pair), 1 single CTA, 2 CTA pair (cta_group::2, the B panel split
    across the two SMs of a TPC).  A plan keeps the kernel it was built with."""
    lib = _lib.lib()
    prev = lib.sdb_lora_tc_set_mode(int(mode))
    if prev < 0:
        _lib.check("sdb_lora_tc_set_mode", prev)
    try:
        yield
    finally:
        lib.sdb_lora_tc_set_mode(prev)


class LoraTmaPlan:
    """K1 fast path for bf16 weights: factors packed once (UMMA K-major
    SWIZZLE_128B tiles), W streamed through a TMA ring, rank contraction on
    tcgen05 at every rank (ranks padded to 16 for the MMA K step; an FFMA
    variant measured 3x slower even at R = 8).  One launch covers every job.

    entries: (w_in, w_out or None, down (h1, R) bf16, up (R, h2) bf16, scale)
    or (w_in, w_out or None, [(down_i, up_i, s_i), ...], None, scale) — the
    adapters of a stack given separately: they are stacked (lora.py:147-160)
    while packing, straight from their own buffers, with the scales kept
    exact (epilogue scale + hi/lo split of the others, sdb_lora_pack_multi).  Every
    w_in must satisfy ``tma_eligible``.  ``repack(stream)`` re-runs the
    packing from the same factor buffers (after they were refreshed, e.g. by
    an async host-to-device fetch)."""

    def __init__(self, entries: Sequence[tuple], simt_max_rank: int = 0, stream=None):
        if not entries:
            raise ValidationError("LoraTmaPlan needs at least one job")
        lib = _lib.lib()
        dev = entries[0][0].device
        sizes = []
        self.alg_bytes = 0
        self.alg_flops = 0
        self.max_rank = 0
        self._srcs = []      # per job: (ctypes sdb_lora_src array, n, h1, h2, a, b)
        self._keep = []
        norm = []
        for i, (w_in, w_out, down, up, scale) in enumerate(entries):
            out = w_in if w_out is None else w_out
            srcs = list(down) if isinstance(down, (list, tuple)) else [(down, up, 1.0)]
            if not (tma_eligible(w_in) and tma_eligible(out)):
                raise ValidationError(f"job {i}: weight is not TMA-eligible (bf16, ldw % 8 == 0)")
            h1, h2 = w_in.shape
            r = 0
            arr = (_lib.LoraSrc * len(srcs))()
            for k, (d, u, s) in enumerate(srcs):
                require_cuda(w_in, out, d, u)
                if d.dtype != torch.bfloat16 or u.dtype != torch.bfloat16:
                    raise ValidationError(f"job {i}: factors must be bf16 on the TMA path")
                if d.shape[0] != h1 or u.shape != (d.shape[1], h2):
                    raise ValidationError(f"job {i}: factor shapes do not match weight ({h1}, {h2})")
                r += d.shape[1]
                arr[k].down, arr[k].ldd = d.data_ptr(), _row_stride(d, "down")
                arr[k].up, arr[k].ldu = u.data_ptr(), _row_stride(u, "up")
                arr[k].rank, arr[k].scale = d.shape[1], float(s)
                self._keep += [d, u]
            # packed sizes, the epilogue scale and the hi/lo K blocks of this stack
            a_b, b_b = ctypes.c_size_t(0), ctypes.c_size_t(0)
            epi, lo = ctypes.c_float(0), ctypes.c_int32(0)
            _lib.check("sdb_lora_pack_multi_layout", lib.sdb_lora_pack_multi_layout(
                arr, len(srcs), h1, h2, ctypes.byref(a_b), ctypes.byref(b_b), ctypes.byref(epi), ctypes.byref(lo)))
            sizes.append((a_b.value, b_b.value))
            self.alg_bytes += 2 * h1 * h2 * 2 + (h1 + h2) * r * 2
            self.alg_flops += 2 * h1 * h2 * r
            self.max_rank = max(self.max_rank, r)
            norm.append((w_in, out, arr, len(srcs), r, float(scale) * epi.value, lo.value))
        # one arena, every packed block 1024-B aligned
        offs, total = [], 0
        for a_b, b_b in sizes:
            offs.append((total, total + a_b))
            total += a_b + b_b
        self.arena = torch.empty(total + 1024, dtype=torch.uint8, device=dev)
        base = (self.arena.data_ptr() + 1023) // 1024 * 1024
        jobs = (_lib.LoraTcJob * len(entries))()
        for i, (w_in, out, arr, n_src, r, scale, lo_mask) in enumerate(norm):
            h1, h2 = w_in.shape
            a_ptr, b_ptr = base + offs[i][0], base + offs[i][1]
            self._srcs.append((arr, n_src, h1, h2, a_ptr, b_ptr))
            j = jobs[i]
            j.w_in, j.w_out = w_in.data_ptr(), out.data_ptr()
            j.h1, j.h2, j.ldw = h1, h2, _row_stride(w_in, "weight")
            j.a_packed, j.b_packed = a_ptr, b_ptr
            j.rank, j.scale, j.lo_mask = r, scale, lo_mask
            self._keep += [w_in, out]
        self.repack(stream)
        need, n_units, kb_max = ctypes.c_size_t(0), ctypes.c_int(0), ctypes.c_int(0)
        _lib.check("sdb_lora_tc_plan", lib.sdb_lora_tc_plan(jobs, len(entries), None, 0, ctypes.byref(need),
                                                            ctypes.byref(n_units), ctypes.byref(kb_max)))
        host = (ctypes.c_uint8 * need.value)()
        _lib.check("sdb_lora_tc_plan", lib.sdb_lora_tc_plan(jobs, len(entries), host, need.value,
                                                            ctypes.byref(need), ctypes.byref(n_units),
                                                            ctypes.byref(kb_max)))
        self.blob = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
        self.n_jobs = len(entries)
        self.n_units = n_units.value
        self.kb_max = kb_max.value                 # opaque: kb | kernel << 8 | A K-blocks << 12
        self.kernel = "pair" if ((self.kb_max >> 8) & 0xF) == 2 else "single"
        self.simt_rank = 0   # reserved in the ABI: tcgen05 at every rank
        self.path = 1   # 1 = TMA + tcgen05 (0 = the generic SIMT kernel of LoraPatchPlan)

    def repack(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """(Re-)stack and pack every job's factors into the arena (2 kernels per job)."""
        lib, sp = _lib.lib(), _stream_ptr(stream)
        for arr, n, h1, h2, a_ptr, b_ptr in self._srcs:
            _count(2)
            _lib.check("sdb_lora_pack_multi", lib.sdb_lora_pack_multi(arr, n, h1, h2, a_ptr, b_ptr, sp))

    def launch(self, sign: float = 1.0, stream: Optional[torch.cuda.Stream] = None,
               max_ctas: int = 0) -> None:
        _count(1)
        _lib.check("sdb_lora_tc_patch", _lib.lib().sdb_lora_tc_patch(
            self.blob.data_ptr(), self.n_jobs, self.n_units, self.kb_max, self.simt_rank, float(sign),
            int(max_ctas), _stream_ptr(stream)))


class BatchedCopy:
    """dst_i <- src_i for a fixed list of equally shaped device tensor pairs in
    ONE launch (``sdb_batched_copy``): the restore-from-pristine unpatch of a
    whole UNet.  Tensors must be contiguous in memory (any memory format), 16-B
    aligned, with a size that is a multiple of 16 bytes."""

    def __init__(self, srcs: Sequence[torch.Tensor], dsts: Sequence[torch.Tensor]):
        if len(srcs) != len(dsts) or not srcs:
            raise ValidationError("BatchedCopy needs matching, non-empty source / destination lists")
        dev = srcs[0].device
        nvec, ps, pd = [], [], []
        for a, b in zip(srcs, dsts):
            require_cuda(a, b)
            nb = a.numel() * a.element_size()
            if b.numel() * b.element_size() != nb or a.dtype != b.dtype:
                raise ValidationError("BatchedCopy: source and destination differ in size or dtype")
            if a.data_ptr() % 16 or b.data_ptr() % 16 or nb % 16:
                raise ValidationError("BatchedCopy: 16-B aligned tensors of a multiple of 16 bytes only")
            if not (a.is_contiguous() or a.is_contiguous(memory_format=torch.channels_last)) or \
                    a.stride() != b.stride():
                raise ValidationError("BatchedCopy: dense tensors with identical strides only")
            nvec.append(nb // 16)
            ps.append(a.data_ptr())
            pd.append(b.data_ptr())
        chunk = int(_lib.lib().sdb_batched_copy_chunk_vectors())
        prefix = [0]
        for v in nvec:
            prefix.append(prefix[-1] + (v + chunk - 1) // chunk)
        self.n, self.chunks = len(nvec), prefix[-1]
        self.nbytes = 16 * sum(nvec)
        tab = torch.tensor(ps + pd + nvec + prefix, dtype=torch.int64)
        self._tab = tab.to(dev)
        self._keep = (list(srcs), list(dsts))

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        n, base = self.n, self._tab.data_ptr()
        _count(1)
        _lib.check("sdb_batched_copy", _lib.lib().sdb_batched_copy(
            base, base + 8 * n, base + 16 * n, base + 24 * n, n, self.chunks, _stream_ptr(stream)))


# --------------------------------------------------------------------------
# K2 — GroupNorm (+SiLU), NHWC
# --------------------------------------------------------------------------
_ws_cache: dict = {}


def _workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)  # K2 counters start at 0
        _ws_cache[key] = buf
    return buf


def nhwc_view(x: torch.Tensor) -> tuple[int, int, int]:
    """(N, HW, C) of a 4-d channels_last tensor (or a 3-d [N, L, C] tensor)."""
    if x.dim() == 4:
        n, c, h, w = x.shape
        if not x.is_contiguous(memory_format=torch.channels_last):
            raise ValidationError("feature maps must be channels_last (NHWC) contiguous")
        return n, h * w, c
    if x.dim() == 3:
        if not x.is_contiguous():
            raise ValidationError("[N, L, C] tensors must be contiguous")
        n, l, c = x.shape
        return n, l, c
    raise ValidationError(f"expected a 3-d or 4-d tensor, got {x.dim()}-d")


@contextlib.contextmanager
def groupnorm_mode(mode: int):
    """K2 form for calls inside the block: 0 = single-pass cluster form where
    eligible (default), 1 = two-pass form (tests / probes)."""
    _lib.lib().sdb_groupnorm_set_mode(int(mode))
    try:
        yield
    finally:
        _lib.lib().sdb_groupnorm_set_mode(0)


def groupnorm_workspace(x: torch.Tensor, groups: int = 32, channels: Optional[int] = None) -> torch.Tensor:
    """A zeroed K2 workspace sized for x — or for x's batch and pixels with
    ``channels`` channels (a K3 concat's output) — (its arrival counters must
    start at zero; every launch leaves them at zero)."""
    n, hw, c = nhwc_view(x)
    c = c if channels is None else int(channels)
    return torch.zeros(max(_lib.lib().sdb_groupnorm_workspace(n, hw, c, groups), 256), dtype=torch.uint8,
                       device=x.device)


def groupnorm_silu(x: torch.Tensor, gamma: Optional[torch.Tensor], beta: Optional[torch.Tensor],
                   groups: int = 32, eps: float = 1e-5, silu: bool = True,
                   out: Optional[torch.Tensor] = None,
                   add_nc: Optional[torch.Tensor] = None,
                   workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """act(GroupNorm(x + add_nc[:, :, None, None])) in one NHWC pass pair.

    add_nc: optional fp32 [N, C] bias added before normalisation (the ResNet
    time-embedding projection).  workspace: a buffer from
    ``groupnorm_workspace`` owned by the call site (required when calls may run
    concurrently on different streams, e.g. inside concurrently replayed CUDA
    graphs); default: one shared per stream."""
    require_cuda(x, gamma, beta, out, add_nc)
    n, hw, c = nhwc_view(x)
    if out is None:
        out = torch.empty_like(x)
    for t in (gamma, beta, add_nc):
        if t is not None and (t.dtype != torch.float32 or not t.is_contiguous()):
            raise ValidationError("gamma / beta / add_nc must be contiguous fp32")
    if add_nc is not None and add_nc.numel() != n * c:
        raise ValidationError(f"add_nc must hold N*C = {n * c} values")
    pending = getattr(x, "_sdb_gn", None)
    if pending is not None and pending[1] == groups and pending[2] == x.data_ptr() and add_nc is None:
        # x's statistics were accumulated by the K3 pass that wrote it: apply only
        # (not with add_nc: GroupNorm(x + add_nc) needs the statistics of the sum)
        _count(1)
        _lib.check("sdb_groupnorm_apply", _lib.lib().sdb_groupnorm_apply(
            x.data_ptr(), out.data_ptr(), gamma.data_ptr() if gamma is not None else None,
            beta.data_ptr() if beta is not None else None,
            add_nc.data_ptr() if add_nc is not None else None, n, hw, c, groups, float(eps), int(silu),
            sdb_dtype(x), pending[0].data_ptr(), _stream_ptr(None)))
        return out
    ws_bytes = _lib.lib().sdb_groupnorm_workspace(n, hw, c, groups)
    if workspace is not None:
        if workspace.numel() < ws_bytes:
            raise ValidationError("groupnorm workspace too small for this input")
        ws = workspace
    else:
        ws = _workspace(ws_bytes, x.device)
    _count(_lib.lib().sdb_groupnorm_launches(n, hw, c, groups, sdb_dtype(x)))
    _lib.check("sdb_groupnorm_silu", _lib.lib().sdb_groupnorm_silu(
        x.data_ptr(), out.data_ptr(), gamma.data_ptr() if gamma is not None else None,
        beta.data_ptr() if beta is not None else None,
        add_nc.data_ptr() if add_nc is not None else None, n, hw, c, groups, float(eps), int(silu),
        sdb_dtype(x), ws.data_ptr(), _stream_ptr(None)))
    return out


# --------------------------------------------------------------------------
# K3 — residual injection fused with the skip concat
# --------------------------------------------------------------------------
def residual_inject(skip: torch.Tensor, residuals: Sequence[torch.Tensor], scales: Sequence[float],
                    hidden: Optional[torch.Tensor] = None,
                    out: Optional[torch.Tensor] = None,
                    skip_bias: Optional[torch.Tensor] = None,
                    hidden_bias: Optional[torch.Tensor] = None,
                    gn_workspace: Optional[torch.Tensor] = None, groups: int = 32) -> torch.Tensor:
    """hidden is None: returns skip + sum s_i r_i (in place into ``out`` or skip).
    otherwise: returns cat([hidden, skip + sum s_i r_i], dim=C) in channels_last.
    skip_bias / hidden_bias: optional contiguous fp32 per-channel vectors added
    to the skip / hidden part (the producing convolution's bias, folded).
    gn_workspace: a ``groupnorm_workspace`` buffer — the same pass also
    accumulates the GroupNorm(groups) statistics of the output, and the next
    ``groupnorm_silu`` of the returned tensor runs its apply half only."""
    require_cuda(skip, hidden, out, skip_bias, hidden_bias, *residuals)
    if len(residuals) != len(scales):
        raise ValidationError("one scale per residual")
    n, hw, cs = nhwc_view(skip)
    for r in residuals:
        if r.shape != skip.shape or r.dtype != skip.dtype:
            raise ValidationError(f"residual shape {tuple(r.shape)} != skip {tuple(skip.shape)}")
        nhwc_view(r)
    ch = 0
    if hidden is not None:
        hn, hhw, ch = nhwc_view(hidden)
        if (hn, hhw) != (n, hw) or hidden.dtype != skip.dtype:
            raise ValidationError("hidden and skip must agree on N, H, W and dtype")
        if out is None:
            if skip.dim() == 4:
                out = torch.empty((n, ch + cs, skip.shape[2], skip.shape[3]), dtype=skip.dtype,
                                  device=skip.device, memory_format=torch.channels_last)
            else:
                out = torch.empty((n, hw, ch + cs), dtype=skip.dtype, device=skip.device)
    elif out is None:
        out = skip
    for b, cnt, what in ((skip_bias, cs, "skip_bias"), (hidden_bias, ch, "hidden_bias")):
        if b is not None and (b.dtype != torch.float32 or not b.is_contiguous() or b.numel() != cnt):
            raise ValidationError(f"{what} must be a contiguous fp32 vector of {cnt} channels")
    if hidden_bias is not None and hidden is None:
        raise ValidationError("hidden_bias given without hidden")
    k = len(residuals)
    ptrs = (ctypes.c_void_p * max(k, 1))(*[r.data_ptr() for r in residuals])
    sc = (ctypes.c_float * max(k, 1))(*[float(s) for s in scales])
    _count(1)
    if gn_workspace is not None and skip.dim() == 4 and k <= 4 and skip.dtype in (torch.bfloat16, torch.float16) \
            and (ch + cs) % groups == 0:
        need = _lib.lib().sdb_groupnorm_workspace(n, hw, ch + cs, groups)
        if gn_workspace.numel() < need:       # sized for the OUTPUT (hidden | skip) map
            raise ValidationError(f"gn_workspace holds {gn_workspace.numel()} B, the {ch + cs}-channel output "
                                  f"needs {need} B (groupnorm_workspace of the output shape)")
        _lib.check("sdb_residual_inject_gn", _lib.lib().sdb_residual_inject_gn(
            out.data_ptr(), hidden.data_ptr() if hidden is not None else None, skip.data_ptr(), ptrs, sc, k,
            n, hw, ch, cs, hidden_bias.data_ptr() if hidden_bias is not None else None,
            skip_bias.data_ptr() if skip_bias is not None else None, groups, gn_workspace.data_ptr(),
            sdb_dtype(skip), _stream_ptr(None)))
        out._sdb_gn = (gn_workspace, groups, out.data_ptr())
        return out
    if hasattr(out, "_sdb_gn"):
        del out._sdb_gn      # rewritten without statistics
    if skip_bias is None and hidden_bias is None:
        _lib.check("sdb_residual_inject", _lib.lib().sdb_residual_inject(
            out.data_ptr(), hidden.data_ptr() if hidden is not None else None, skip.data_ptr(),
            ptrs, sc, k, n * hw, ch, cs, sdb_dtype(skip), _stream_ptr(None)))
    else:
        _lib.check("sdb_residual_inject_bias", _lib.lib().sdb_residual_inject_bias(
            out.data_ptr(), hidden.data_ptr() if hidden is not None else None, skip.data_ptr(),
            ptrs, sc, k, n * hw, ch, cs, hidden_bias.data_ptr() if hidden_bias is not None else None,
            skip_bias.data_ptr() if skip_bias is not None else None, sdb_dtype(skip), _stream_ptr(None)))
    return out


# --------------------------------------------------------------------------
# K5 / K6 — GEGLU and residual-add + LayerNorm of the transformer blocks
# --------------------------------------------------------------------------
def ff_geglu_supported(x: torch.Tensor, w: torch.Tensor) -> bool:
    return (x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16 and x.shape[-1] % 64 == 0
            and w.dim() == 2 and w.shape[0] % 256 == 0 and w.shape[1] == x.shape[-1])


def ff_geglu(x: torch.Tensor, w: torch.Tensor, bias: Optional[torch.Tensor] = None) -> torch.Tensor:
    """GEGLU(x W^T + bias) in one tcgen05 GEMM (K5'): W = [W_value; W_gate]
    ([2F, K] bf16, the GEGLU proj weight as stored), bias fp32 [2F] or None;
    returns [..., F]."""
    require_cuda(x, w, bias)
    k = x.shape[-1]
    if not ff_geglu_supported(x, w):
        raise ValidationError("ff_geglu: bf16, K % 64 == 0, W [2F, K] with F % 128 == 0")
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != w.shape[0] or not bias.is_contiguous()):
        raise ValidationError("ff_geglu: bias must be a contiguous fp32 vector of 2F values")
    x2 = x.reshape(-1, k)
    if not x2.is_contiguous() or not w.is_contiguous():
        raise ValidationError("ff_geglu: x rows and W must be contiguous")
    f = w.shape[0] // 2
    out = torch.empty((*x.shape[:-1], f), dtype=x.dtype, device=x.device)
    _count(1)
    _lib.check("sdb_ff_geglu", _lib.lib().sdb_ff_geglu(
        x2.data_ptr(), w.data_ptr(), bias.data_ptr() if bias is not None else None, out.data_ptr(),
        x2.shape[0], k, f, _stream_ptr(None)))
    return out


def geglu(proj: torch.Tensor) -> torch.Tensor:
    """proj [..., 2F] contiguous -> [..., F] = proj[..., :F] * gelu(proj[..., F:])."""
    require_cuda(proj)
    if not proj.is_contiguous():
        raise ValidationError("geglu input must be contiguous")
    f2 = proj.shape[-1]
    out = torch.empty(proj.shape[:-1] + (f2 // 2,), dtype=proj.dtype, device=proj.device)
    _count(1)
    _lib.check("sdb_geglu", _lib.lib().sdb_geglu(proj.data_ptr(), out.data_ptr(), proj.numel() // f2, f2 // 2,
                                                 sdb_dtype(proj), _stream_ptr(None)))
    return out


def upsample2x(x: torch.Tensor) -> torch.Tensor:
    """K10: nearest 2x upsample of a channels_last [N, C, H, W] map."""
    require_cuda(x)
    n, c, h, w = x.shape
    if not x.is_contiguous(memory_format=torch.channels_last) or (c * x.element_size()) % 16:
        raise ValidationError("upsample2x: channels_last input with C * element size a multiple of 16")
    y = torch.empty((n, c, 2 * h, 2 * w), device=x.device, dtype=x.dtype, memory_format=torch.channels_last)
    _count(1)
    _lib.check("sdb_upsample2x", _lib.lib().sdb_upsample2x(x.data_ptr(), y.data_ptr(), n, h, w, c,
                                                           x.element_size(), _stream_ptr(None)))
    return y


def add_layernorm(x: torch.Tensor, d: Optional[torch.Tensor], gamma: torch.Tensor, beta: torch.Tensor,
                  eps: float = 1e-5) -> torch.Tensor:
    """x += d (in place, d may be None); returns LayerNorm(x) * gamma + beta."""
    require_cuda(x, d, gamma, beta)
    if not x.is_contiguous() or (d is not None and (not d.is_contiguous() or d.shape != x.shape)):
        raise ValidationError("add_layernorm: x and d must be contiguous and of equal shape")
    c = x.shape[-1]
    y = torch.empty_like(x)
    _count(1)
    _lib.check("sdb_add_layernorm", _lib.lib().sdb_add_layernorm(
        x.data_ptr(), d.data_ptr() if d is not None else None, y.data_ptr(), gamma.data_ptr(), beta.data_ptr(),
        x.numel() // c, c, float(eps), sdb_dtype(x), _stream_ptr(None)))
    return y


# --------------------------------------------------------------------------
# K7 — cross-attention against the short text context
# --------------------------------------------------------------------------
def cross_attention_supported(q: torch.Tensor, kv: torch.Tensor, heads: int) -> bool:
    c = q.shape[-1]
    d = c // heads
    return (q.dtype == torch.bfloat16 and kv.dtype == torch.bfloat16 and q.dim() == 3 and kv.dim() == 3
            and 1 <= kv.shape[1] <= 128 and 8 <= d <= 160 and d % 8 == 0 and c % heads == 0)


def cross_attention(q: torch.Tensor, kv: torch.Tensor, heads: int, scale: Optional[float] = None,
                    out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """softmax(scale * Q K^T) V per head.  q [N, Lq, C] (last dim contiguous),
    kv [N, Lk, 2C] holding K | V (Lk <= 128), bf16; returns [N, Lq, C]."""
    require_cuda(q, kv, out)
    n, lq, c = q.shape
    if kv.shape[0] != n or kv.shape[2] < 2 * c:
        raise ValidationError(f"kv must be [N, Lk, 2C] (got {tuple(kv.shape)} for C = {c})")
    if q.stride(2) != 1 or kv.stride(2) != 1 or q.stride(0) != lq * q.stride(1) or kv.stride(0) != kv.shape[1] * kv.stride(1):
        raise ValidationError("cross_attention: rows must be contiguous and batch-packed")
    d = c // heads
    if out is None:
        out = torch.empty((n, lq, c), dtype=q.dtype, device=q.device)
    _count(1)
    _lib.check("sdb_cross_attention", _lib.lib().sdb_cross_attention(
        q.data_ptr(), q.stride(1), kv.data_ptr(), kv.stride(1), c, out.data_ptr(), out.stride(1), n, lq,
        kv.shape[1], heads, d, float(scale if scale is not None else d ** -0.5), sdb_dtype(q), _stream_ptr(None)))
    return out


# --------------------------------------------------------------------------
# K8 — self-attention (head dim 64) on tcgen05
# --------------------------------------------------------------------------
def self_attention_supported(qkv: torch.Tensor, heads: int) -> bool:
    n, l, c3 = qkv.shape
    return (qkv.dtype == torch.bfloat16 and c3 % 3 == 0 and (c3 // 3) == heads * 64 and l % 128 == 0
            and qkv.stride(2) == 1 and qkv.stride(1) % 8 == 0 and qkv.stride(0) == l * qkv.stride(1))


def self_attention(qkv: torch.Tensor, heads: int, scale: Optional[float] = None,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """softmax(scale * Q K^T) V per head from the fused q|k|v projection
    [N, L, 3C] (C = heads * 64, L % 128 == 0), bf16; returns [N, L, C]."""
    require_cuda(qkv, out)
    n, l, c3 = qkv.shape
    c = c3 // 3
    if out is None:
        out = torch.empty((n, l, c), dtype=qkv.dtype, device=qkv.device)
    _count(1)
    _lib.check("sdb_self_attention", _lib.lib().sdb_self_attention(
        qkv.data_ptr(), qkv.stride(1), out.data_ptr(), out.stride(1), n, l, heads, 64,
        float(scale if scale is not None else 64 ** -0.5), sdb_dtype(qkv), _stream_ptr(None)))
    return out


# --------------------------------------------------------------------------
# K4 — CFG combine + DDIM step (+ CFG re-batch of the next UNet input)
# --------------------------------------------------------------------------
def conv_out_supported(x: torch.Tensor, w: torch.Tensor) -> bool:
    return (x.dim() == 4 and w.dim() == 4 and w.shape[0] == 4 and tuple(w.shape[2:]) == (3, 3)
            and x.dtype in (torch.bfloat16, torch.float32) and w.dtype == x.dtype
            and x.shape[3] % 16 == 0 and x.shape[1] % 2 == 0 and x.shape[1] <= 1280
            and x.is_contiguous(memory_format=torch.channels_last))


def conv_out(x: torch.Tensor, w: torch.Tensor, bias: Optional[torch.Tensor] = None,
             out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K9: 3x3 pad-1 convolution C -> 4 with an fp32 result (the UNet's
    conv_out), x channels_last bf16/fp32, fp32 accumulation.  Returns an fp32
    channels_last [N, 4, H, W] tensor."""
    require_cuda(x, w, bias, out)
    n, c, h, wd = x.shape
    if not conv_out_supported(x, w) or w.shape[1] != c:
        raise ValidationError("conv_out: needs channels_last x [N, C, H, W] (W % 16 == 0, C even <= 1280) "
                              "and a same-dtype [4, C, 3, 3] weight")
    wp = w.permute(0, 2, 3, 1)
    if not wp.is_contiguous():
        wp = wp.contiguous()
    b = None
    if bias is not None:
        b = bias if bias.dtype == torch.float32 and bias.is_contiguous() else bias.float().contiguous()
    if out is None:
        out = torch.empty((n, 4, h, wd), device=x.device, dtype=torch.float32,
                          memory_format=torch.channels_last)
    elif out.dtype != torch.float32 or not out.is_contiguous(memory_format=torch.channels_last) \
            or tuple(out.shape) != (n, 4, h, wd):
        raise ValidationError("conv_out: out must be fp32 channels_last [N, 4, H, W]")
    _count(1)
    _lib.check("sdb_conv_out", _lib.lib().sdb_conv_out(
        x.data_ptr(), wp.data_ptr(), b.data_ptr() if b is not None else None, out.data_ptr(),
        n, h, wd, c, 4, sdb_dtype(x), _stream_ptr(None)))
    return out


def cfg_ddim_step(eps: torch.Tensor, x: torch.Tensor, coef: torch.Tensor, step_dev: torch.Tensor,
                  x_out: Optional[torch.Tensor] = None,
                  unet_in: Optional[torch.Tensor] = None) -> torch.Tensor:
    require_cuda(eps, x, coef, step_dev, x_out, unet_in)
    if x.dtype != torch.float32 or coef.dtype != torch.float32 or step_dev.dtype != torch.int32:
        raise ValidationError("x / coef must be fp32 and step_dev int32")
    L = x.numel()
    if eps.numel() != 2 * L:
        raise ValidationError("eps must hold the [uncond; cond] batch of 2 latents")
    if unet_in is not None and unet_in.numel() != 2 * L:
        raise ValidationError("unet_in must hold 2 latents")
    # the master latent is NHWC-flat: eps / unet_in must be stored NHWC too
    for name, t in (("eps", eps), ("unet_in", unet_in)):
        if t is not None and t.dim() == 4 and not t.is_contiguous(memory_format=torch.channels_last):
            raise ValidationError(f"{name} must be channels_last (NHWC) like the latent")
    out = x if x_out is None else x_out
    _count(1)
    _lib.check("sdb_cfg_ddim_step", _lib.lib().sdb_cfg_ddim_step(
        eps.data_ptr(), sdb_dtype(eps), x.data_ptr(), out.data_ptr(),
        unet_in.data_ptr() if unet_in is not None else None,
        sdb_dtype(unet_in) if unet_in is not None else _lib.SDB_F32, L, coef.data_ptr(),
        step_dev.data_ptr(), _stream_ptr(None)))
    return out
