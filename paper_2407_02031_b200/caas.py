"""ControlNet-as-a-service across GPUs — the multi-GPU form of the denoising loop.

Reference semantics (addonsim/orchestrator.py:181-188 ``parallel_step_latency``,
:621-660 ``_run_parallel_step``): each ControlNet runs on its
own service GPU concurrently with the base UNet's encoder; its outputs are
shipped to the base GPU and the decoder starts once the encoder AND every
branch are done (orchestrator.py:652-653).  Here that is a real exchange:

* one process per GPU (torch.distributed, NCCL over NVLink/NVSwitch);
  ``caas_layout`` splits the ranks into groups of 1 base + up to n_cn service
  GPUs; leftover ranks serve whole images alone (``solo``, the serial
  orchestrator.py:611-619 step).
* per request: the base broadcasts the conditioning inputs (text embeddings,
  control images, SDXL added conditions) to its services once; hint and
  added-condition embeddings are then computed locally (step-invariant).
* per step (``CaaSPeerProtocol``, the default whenever the group's GPUs can
  map each other's memory): the base raises each service's "message ready"
  flag (a GPU-side ``cuStreamWriteValue32`` into the service's memory) once
  the 4xHxW fp32 latent + timestep (256 KiB for SDXL, the paper's "send
  latent" C0) is written; each service's stream waits on it, pulls the
  message over NVLink (CUDA-IPC mapping), runs its ControlNet(s) — scales
  folded into the zero convolutions — and pushes each residual level into
  its own receive buffer on the base as soon as it exists (shallow, largest
  levels first: the paper's 108 MiB "feature map" transfer C1, overlapped
  with the deeper levels and the base's encoder), then raises the base's
  "residuals ready" flag.  The base's decoder waits on every service's flag
  and K3 sums the per-service buffers into the skip concat.  No collective
  and no host round trip on the per-step data path.
* ``SDB_CAAS_TRANSPORT=nccl`` selects ``CaaSProtocol`` instead: NCCL
  broadcast of the message + send/recv of each service's flat buffer (gloo
  with host staging on CPU-only process groups, which the CPU tests use).

The transport (``CaaSProtocol``) is separated from the compute so the same
protocol code runs under gloo on CPU in the tests with a stand-in compute.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Group:
    base: int
    services: tuple          # ranks
    cn_of_service: tuple     # per service rank: tuple of ControlNet indices it runs

    @property
    def ranks(self) -> tuple:
        return (self.base,) + self.services


@dataclass(frozen=True)
class CaaSLayout:
    world: int
    n_cn: int
    groups: tuple            # Group, including size-1 "solo" groups

    def group_of(self, rank: int) -> Group:
        for g in self.groups:
            if rank in g.ranks:
                return g
        raise ValueError(f"rank {rank} not in layout")

    def role(self, rank: int) -> str:
        g = self.group_of(rank)
        if not g.services:
            return "solo"
        return "base" if rank == g.base else "service"


def caas_layout(world: int, n_cn: int) -> CaaSLayout:
    """Groups of min(world, 1 + n_cn) ranks (base first); ControlNet i runs on
    service i % n_services; leftover ranks are solo replicas."""
    if world < 1 or n_cn < 0:
        raise ValueError("world must be >= 1 and n_cn >= 0")
    gs = max(1, min(world, 1 + n_cn))
    groups = []
    n_groups = world // gs
    for k in range(n_groups):
        base = k * gs
        services = tuple(range(base + 1, base + gs))
        cn_of = tuple(tuple(i for i in range(n_cn) if services and i % len(services) == j)
                      for j in range(len(services)))
        groups.append(Group(base, services, cn_of))
    for r in range(n_groups * gs, world):
        groups.append(Group(r, (), ()))
    return CaaSLayout(world, n_cn, tuple(groups))


def make_groups(layout: CaaSLayout, rank: int):
    """Create every multi-rank group's communicator — collectively: EVERY rank
    (solo ones included) must call this, in the same order.  Returns this
    rank's group (None for a solo rank)."""
    mine = None
    for g in layout.groups:
        if g.services:
            pg = dist.new_group(list(g.ranks))
            if rank in g.ranks:
                mine = pg
    return mine


class CaaSProtocol:
    """The per-request / per-step exchange of one group (NCCL on GPU, gloo on CPU).

    msg    float32 [L + 1]: the fp32 latent (NHWC order) and the timestep.
    flats  residual buffers: on a service, its own one (the conditioning-scaled
           sum of its ControlNets' down + mid residuals, NHWC, concatenated);
           on the base, one receive buffer per service (K3 sums them while it
           writes the skip concat, so the base never zeroes or reduces).

    Ordering: the broadcast and the point-to-point transfers of a group share
    one communicator (one NCCL stream), so a service's next-step receive
    completes only after its previous send — the service may then overwrite
    its buffer without an extra fence."""

    def __init__(self, layout: CaaSLayout, rank: int, msg: torch.Tensor, flats: Sequence[torch.Tensor], pg=None):
        self.layout = layout
        self.rank = rank
        self.group = layout.group_of(rank)
        self.role = layout.role(rank)
        self.msg = msg
        self.flats = list(flats)
        self.pg = pg if pg is not None else make_groups(layout, rank)
        # gloo carries host tensors only: device buffers are staged through host
        # copies (used to run the multi-process path on ONE GPU in the tests)
        self.staged = msg.is_cuda and dist.get_backend(self.pg) == "gloo"
        if self.staged:
            self._msg_h = torch.empty(msg.shape, dtype=msg.dtype)
            self._flats_h = [torch.empty(f.shape, dtype=f.dtype) for f in self.flats]
        self._pending = []

    # -- per request --------------------------------------------------------
    def share_request(self, tensors: Sequence[torch.Tensor]) -> None:
        """Broadcast the request's conditioning tensors from the base (in place)."""
        for t in tensors:
            if self.staged:
                h = t.cpu()
                dist.broadcast(h, src=self.group.base, group=self.pg)
                t.copy_(h)
            else:
                dist.broadcast(t, src=self.group.base, group=self.pg)

    # -- per step -------------------------------------------------------------
    def base_step_begin(self) -> list:
        """Base: ship (latent, t) and post one receive per service; returns the
        handles to wait on before the decoder.  Everything is stream-ordered
        after the work already queued (the previous step's K4)."""
        if self.staged:
            self._msg_h.copy_(self.msg)
            dist.broadcast(self._msg_h, src=self.group.base, group=self.pg)
            ops = [dist.P2POp(dist.irecv, h, peer=s, group=self.pg)
                   for h, s in zip(self._flats_h, self.group.services)]
            return [_StagedWork(dist.batch_isend_irecv(ops), list(zip(self._flats_h, self.flats)))]
        dist.broadcast(self.msg, src=self.group.base, group=self.pg, async_op=True)
        ops = [dist.P2POp(dist.irecv, f, peer=s, group=self.pg) for f, s in zip(self.flats, self.group.services)]
        return dist.batch_isend_irecv(ops)

    def service_receive(self) -> None:
        if self.staged:
            for w in self._pending:     # previous send done before the buffer is reused
                w.wait()
            self._pending = []
            dist.broadcast(self._msg_h, src=self.group.base, group=self.pg)
            self.msg.copy_(self._msg_h)
            return
        work = dist.broadcast(self.msg, src=self.group.base, group=self.pg, async_op=True)
        work.wait()

    def service_send(self):
        if self.staged:
            self._flats_h[0].copy_(self.flats[0])
            self._pending = dist.batch_isend_irecv([dist.P2POp(dist.isend, self._flats_h[0], peer=self.group.base,
                                                               group=self.pg)])
            return self._pending
        return dist.batch_isend_irecv([dist.P2POp(dist.isend, self.flats[0], peer=self.group.base, group=self.pg)])


class CaaSPeerProtocol(CaaSProtocol):
    """The per-step exchange with no collective on the data path: GPU-to-GPU
    copies through CUDA IPC mappings (NVLink peer copies across GPUs) ordered
    by GPU-side sequence flags (``sdb_stream_write_value32`` /
    ``sdb_stream_wait_value32``, stream memory operations — no NCCL call and
    no host round trip per step).

    base     owns msg, one receive buffer per service and one int32 "residuals
             ready" flag per service; writes each service's "message ready"
             flag (step k) once the previous decoder + K4 wrote msg, and makes
             its decoder stream wait for every service's flag >= k.
    service  waits for its flag >= k, copies the base's msg (256 KiB), runs its
             ControlNets into its local buffer, copies that buffer into its
             receive buffer on the base (107.5 MB for SDXL) and writes the
             base's flag = k (the write is fenced after the copy).
    A service writes step k+1's residuals only after its k+1 message flag,
    which the base raises after decoder k consumed step k's — no extra fence.
    Setup (IPC handle exchange) and the per-request conditioning broadcast use
    the group's communicator (NCCL or gloo)."""

    def __init__(self, layout: CaaSLayout, rank: int, msg: torch.Tensor, flats: Sequence[torch.Tensor], pg=None):
        super().__init__(layout, rank, msg, flats, pg)
        from torch.multiprocessing.reductions import reduce_tensor
        dev = msg.device
        self.step = 0
        services = list(self.group.services)
        if self.role == "base":
            self.res_flags = torch.zeros(len(services), dtype=torch.int32, device=dev)
            export = {"msg": reduce_tensor(msg), "flats": [reduce_tensor(f) for f in self.flats],
                      "flags": reduce_tensor(self.res_flags)}
        else:
            self.msg_flag = torch.zeros(1, dtype=torch.int32, device=dev)
            export = {"flag": reduce_tensor(self.msg_flag)}
        objs = [None] * len(self.group.ranks)
        dist.all_gather_object(objs, export, group=self.pg)

        def rebuild(x):
            fn, args = x
            return fn(*args)
        if self.role == "base":
            self.peer_msg_flags = [rebuild(objs[1 + i]["flag"]) for i in range(len(services))]
        else:
            k = services.index(rank)
            b = objs[0]
            self.peer_msg = rebuild(b["msg"])
            self.peer_flat = rebuild(b["flats"][k])
            self.peer_res_flag = rebuild(b["flags"])[k:k + 1]
        self._export = export     # keep the exported tensors' IPC records alive
        self._push_stream = None
        self._pushed = False

    def _lib(self):
        from . import _lib
        return _lib

    def _write(self, flag: torch.Tensor, value: int) -> None:
        _lib = self._lib()
        _lib.check("sdb_stream_write_value32", _lib.lib().sdb_stream_write_value32(
            torch.cuda.current_stream().cuda_stream, flag.data_ptr(), value & 0xFFFFFFFF))

    def _copy(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        _lib = self._lib()
        _lib.check("sdb_memcpy_async", _lib.lib().sdb_memcpy_async(
            dst.data_ptr(), src.data_ptr(), src.numel() * src.element_size(), torch.cuda.current_stream().cuda_stream))

    def _wait(self, flag: torch.Tensor, value: int) -> None:
        _lib = self._lib()
        _lib.check("sdb_stream_wait_value32", _lib.lib().sdb_stream_wait_value32(
            torch.cuda.current_stream().cuda_stream, flag.data_ptr(), value & 0xFFFFFFFF))

    def base_step_begin(self) -> list:
        self.step += 1
        for f in self.peer_msg_flags:          # msg (latent, t) of this step is written
            self._write(f, self.step)
        return [_FlagWait(self, i, self.step) for i in range(len(self.peer_msg_flags))]

    def service_receive(self) -> None:
        self.step += 1
        self._wait(self.msg_flag, self.step)
        self._copy(self.msg, self.peer_msg)

    def push_level(self, k: int, out: torch.Tensor) -> None:
        """Inside the service graph: copy residual level k (just written by
        its zero conv into the local buffer) into the base's buffer on a side
        stream, overlapping the deeper levels' compute."""
        if self._push_stream is None:
            self._push_stream = torch.cuda.Stream(device=out.device)
            self._levels = None
        cur = torch.cuda.current_stream()
        self._push_stream.wait_stream(cur)
        off = out.data_ptr() - self.flats[0].data_ptr()
        nbytes = out.numel() * out.element_size()
        _lib = self._lib()
        _lib.check("sdb_memcpy_async", _lib.lib().sdb_memcpy_async(
            self.peer_flat.data_ptr() + off, out.data_ptr(), nbytes, self._push_stream.cuda_stream))
        self._pushed = True

    def join_pushes(self) -> None:
        if self._push_stream is not None:
            torch.cuda.current_stream().wait_stream(self._push_stream)

    def service_send(self):
        if not self._pushed:      # the graph did not push per level: one copy of the whole buffer
            self._copy(self.peer_flat, self.flats[0])
        self._write(self.peer_res_flag, self.step)
        return []


    _TEST = 0x5DB0_0001    # flag / marker value of the setup self-test (never a step number)

    def self_test(self) -> bool:
        """Exercise each peer operation the per-step protocol uses once, with
        host-side checks only (no device-side wait that could hang): the base
        raises every service's message flag and writes a marker into its
        message; each service checks its flag, pulls the message over the
        mapping and checks the marker, then raises the base's residual flag
        and writes a marker into its slice of the base's receive buffer; the
        base checks both.  Flags are reset to 0 afterwards.  Returns this
        rank's verdict (``make_protocol`` takes the group's AND).  Run once at
        setup, so a GPU pair whose NVLink mapping, stream memory operations or
        peer copies misbehave falls back to the NCCL transport instead of
        failing inside a captured step graph."""
        ok = True
        t = self._TEST
        msg_i32 = self.msg.view(-1).view(torch.uint8)[:16].view(torch.int32)
        try:
            if self.role == "base":
                msg_i32.fill_(t)
                for f in self.peer_msg_flags:
                    self._write(f, t)
                torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.pg)
            if self.role != "base":
                ok &= int(self.msg_flag.item()) == t
                pulled = torch.empty_like(self.msg)
                self._copy(pulled, self.peer_msg)
                torch.cuda.current_stream().synchronize()
                ok &= bool((pulled.view(-1).view(torch.uint8)[:16].view(torch.int32) == t).all().item())
                mark = torch.full((4,), self.rank + 1, dtype=torch.int32, device=self.msg.device)
                _lib = self._lib()
                _lib.check("sdb_memcpy_async", _lib.lib().sdb_memcpy_async(
                    self.peer_flat.data_ptr(), mark.data_ptr(), 16, torch.cuda.current_stream().cuda_stream))
                self._write(self.peer_res_flag, t)
                torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.pg)
            if self.role == "base":
                ok &= bool((self.res_flags == t).all().item())
                for i, s in enumerate(self.group.services):
                    got = self.flats[i].view(-1).view(torch.uint8)[:16].view(torch.int32)
                    ok &= bool((got == s + 1).all().item())
        except Exception:   # noqa: BLE001 — any failure of the peer path selects the NCCL transport
            ok = False
        import os
        if os.environ.get("SDB_CAAS_P2P_SELFTEST") == f"fail{self.rank}":   # fault injection (tests)
            ok = False
        # reset this rank's own flags (and the test markers) before any step runs
        if self.role == "base":
            self.res_flags.zero_()
            msg_i32.zero_()
            for f in self.flats:
                f.view(-1).view(torch.uint8)[:16].zero_()
        else:
            self.msg_flag.zero_()
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.pg)
        return ok


class _FlagWait:
    """Base side: the current stream waits for service i's residuals of a step."""

    def __init__(self, proto: CaaSPeerProtocol, i: int, step: int):
        self.proto, self.i, self.step = proto, i, step

    def wait(self):
        self.proto._wait(self.proto.res_flags[self.i:self.i + 1], self.step)


def make_protocol(layout: CaaSLayout, rank: int, msg: torch.Tensor, flats: Sequence[torch.Tensor], pg,
                  transport: Optional[str] = None):
    """The group's transport: ``p2p`` (CaaSPeerProtocol; default when every
    GPU of the group can map its peers' memory) or ``nccl`` (CaaSProtocol:
    broadcast + send/recv; gloo-staged on CPU-only process groups)."""
    import os
    transport = transport or os.environ.get("SDB_CAAS_TRANSPORT", "auto")
    if transport == "auto":
        dev = torch.tensor([msg.device.index if msg.is_cuda else -1])
        devs = [None] * len(layout.group_of(rank).ranks)
        dist.all_gather_object(devs, int(dev.item()), group=pg)
        ok = all(d >= 0 for d in devs) and all(
            a == b or torch.cuda.can_device_access_peer(a, b) for a in devs for b in devs)
        transport = "p2p" if ok else "nccl"
    if transport == "p2p":
        try:
            proto = CaaSPeerProtocol(layout, rank, msg, flats, pg)
            ok = proto.self_test()
        except Exception:   # noqa: BLE001 — e.g. an IPC mapping the driver refuses
            proto, ok = None, False
        verdicts = [None] * len(layout.group_of(rank).ranks)
        dist.all_gather_object(verdicts, bool(ok), group=pg)
        if all(verdicts):
            return proto
        transport = "nccl"      # every rank of the group falls back together
    if transport == "nccl":
        return CaaSProtocol(layout, rank, msg, flats, pg)
    raise ValueError(f"unknown CaaS transport {transport!r} (p2p | nccl | auto)")


class _StagedWork:
    """gloo receive into host buffers, then the device copy the decoder reads."""

    def __init__(self, works, pairs):
        self.works, self.pairs = works, pairs

    def wait(self):
        for w in self.works:
            w.wait()
        for h, d in self.pairs:
            d.copy_(h, non_blocking=False)


def residual_layout(shapes: Sequence[tuple]) -> tuple[list, int]:
    """Offsets of each (N, C, H, W) residual inside the flat buffer."""
    offs, total = [], 0
    for s in shapes:
        offs.append(total)
        total += int(np.prod(s))
    return offs, total


def flat_views(flat: torch.Tensor, shapes: Sequence[tuple]) -> list:
    """channels_last 4-d views of the flat residual buffer (NHWC memory)."""
    offs, _ = residual_layout(shapes)
    out = []
    for o, (n, c, h, w) in zip(offs, shapes):
        out.append(flat[o:o + n * c * h * w].view(n, h, w, c).permute(0, 3, 1, 2))
    return out


# ---------------------------------------------------------------------------
# the real node: graph-captured compute on B200 around the protocol
# ---------------------------------------------------------------------------
class PatchSchedule:
    """Which base weight set each step runs — "pristine", "pg<v>" (the first
    v patch groups swapped in) or "patched" — given each group's boundary
    (None = the group missed this request) and its ready event; the stream
    waits for a group's event before the first step that uses it."""

    def __init__(self, bounds: Sequence[Optional[int]], ready: Sequence, steps: int):
        self.bounds, self.ready, self.M = list(bounds), list(ready), len(bounds)
        self.waited = 0
        live = [b for b in self.bounds if b is not None]
        self.first_full = (self.bounds[-1] + 1) if self.M and len(live) == self.M else steps + 1

    def weights_at(self, step: int, stream) -> str:
        v = sum(1 for b in self.bounds if b is not None and b + 1 <= step)
        while self.waited < v:
            stream.wait_event(self.ready[self.waited])
            self.waited += 1
        if v == 0:
            return "pristine"
        return "patched" if v == self.M else f"pg{v}"

    def finish(self, stream) -> None:
        """Never leave the side streams dangling past the request."""
        if self.ready:
            stream.wait_event(self.ready[-1])
        self.waited = self.M


class CaaSNode:
    """One rank of the ControlNet-as-a-service deployment.

    base:    UNet + K4; encoder graph || (service ControlNets + reduce); decoder graph
    service: the ControlNets assigned to this rank; one graph per step
    solo:    the single-GPU AddonPipeline (ControlNets inline)
    """

    def __init__(self, cfg, layout: CaaSLayout, rank: int, cn_scales: Sequence[float], steps: int = 30,
                 guidance: float = 7.5, dtype=torch.bfloat16, seed: int = 0, device=None, batch: int = 1):
        from . import ops
        from .pipeline import AddonPipeline
        from .unet import ControlNet, init_controlnet, skip_shapes
        self.cfg, self.layout, self.rank = cfg, layout, rank
        self.role = layout.role(rank)
        self.group = layout.group_of(rank)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.steps = steps
        n_cn = layout.n_cn
        self.ops = ops
        h = cfg.latent_hw
        self.batch = batch                   # serving batch of B images: CFG batch 2B
        nb = 2 * batch
        self.L = batch * 4 * h * h
        # communicators are created collectively by every rank, solo ones included
        self.pg = make_groups(layout, rank) if dist.is_initialized() else None
        if self.role == "solo":
            self.pipe = AddonPipeline(cfg, n_controlnets=n_cn, cn_scales=cn_scales, steps=steps, guidance=guidance,
                                      device=self.device, dtype=dtype, seed=seed, batch=batch)
            return
        self.shapes = skip_shapes(cfg, nb)
        _, total = residual_layout(self.shapes)
        self.msg = torch.zeros(self.L + 1, device=self.device, dtype=torch.float32)
        n_flat = len(self.group.services) if self.role == "base" else 1
        self.flats = [torch.zeros(total, device=self.device, dtype=dtype) for _ in range(n_flat)]
        self.views = [flat_views(f, self.shapes) for f in self.flats]
        if self.role == "base":
            # UNet only (no ControlNet weights on the base GPU)
            self.pipe = AddonPipeline(cfg, n_controlnets=0, steps=steps, guidance=guidance, device=self.device,
                                      dtype=dtype, seed=seed, use_graphs=False, batch=batch)   # own graphs
            self.pipe.x = self.msg[: self.L]            # K4 writes the latent straight into the message
        else:
            mine = self.group.cn_of_service[self.group.services.index(rank)]
            self.cn_idx = mine
            self.cn_p = [init_controlnet(cfg, self.device, dtype, seed=1000 + i) for i in mine]
            for p, i in zip(self.cn_p, mine):       # fold the conditioning scale into the zero convs
                for k in list(p.t):
                    if k.startswith("zero_convs.") or k.startswith("mid_zero_conv."):
                        p.t[k] = (p.t[k].float() * float(cn_scales[i])).to(p.t[k].dtype)
            self.cns = [ControlNet(cfg, p) for p in self.cn_p]
            temb = cfg.time_embed_dim
            self.unet_in = torch.zeros((nb, 4, h, h), device=self.device, dtype=dtype).contiguous(
                memory_format=torch.channels_last)
            self.ctx = torch.zeros((nb, cfg.context_len, cfg.context_dim), device=self.device, dtype=dtype)
            self.hints = [torch.zeros((nb, cfg.block_channels[0], h, h), device=self.device, dtype=dtype)
                          .contiguous(memory_format=torch.channels_last) for _ in mine]
            self.add_emb = [torch.zeros((nb, temb), device=self.device, dtype=dtype) if cfg.addition_embed else None
                            for _ in mine]
            for cn in self.cns:                      # per-request cross-attention K|V (finish_prepare)
                cn.enable_kv_cache(self.ctx, ("pristine",))
                cn.kv_slot = "pristine"
        # loopback (all roles in one process, see LoopbackGroup) and solo ranks run without a transport
        self.proto = (make_protocol(layout, rank, self.msg, self.flats, self.pg)
                      if dist.is_initialized() and self.role != "solo" else None)
        self.graphs = {}
        self.graph_launches = {}
        # every node captures on its OWN stream: library calls inside a capture
        # bake in per-stream resources (cuBLAS keys its workspace by stream),
        # and the services' graphs replay concurrently with the base's encoder
        # graph (LoopbackGroup(concurrent=True)) — one shared capture stream
        # would make them race on one cuBLAS workspace
        self.capture_stream = torch.cuda.Stream(device=self.device)

    # -- capture --------------------------------------------------------------
    def _service_step(self):
        h, B = self.cfg.latent_hw, self.batch
        lat = self.msg[: self.L].view(B, h, h, 4).permute(0, 3, 1, 2)
        self.unet_in[:B].copy_(lat)
        self.unet_in[B:].copy_(lat)
        t = self.msg[self.L:self.L + 1]
        # the first ControlNet's zero convs write straight into the send buffer;
        # further ControlNets on this GPU are summed into it in place (K3).
        # With the peer transport and one ControlNet per service, each level
        # is pushed to the base over NVLink the moment its zero conv is done
        # (a copy on a side stream, inside this graph), shallow levels first.
        push = getattr(self.proto, "push_level", None) if len(self.cns) == 1 else None
        outs = [cn.forward(self.unet_in, t, self.ctx, self.hints[i], self.add_emb[i],
                           outs=self.views[0] if i == 0 else None, on_level=push if i == 0 else None)
                for i, cn in enumerate(self.cns)]
        if push is not None:
            self.proto.join_pushes()
        if len(outs) > 1:
            for j, v in enumerate(self.views[0]):
                self.ops.residual_inject(v, [o[j] for o in outs[1:]], [1.0] * (len(outs) - 1), out=v)

    def _base_encode(self):
        p = self.pipe
        t = p.t_table.index_select(0, p.step_dev[:1].long())
        temb = p.unet.time_embedding(t, 2 * self.batch, p.add_emb_unet)
        h, skips = p.unet.encode(p.unet_in, temb, p.ctx)
        self._enc = (temb, h, skips)

    def _base_decode(self):
        p = self.pipe
        temb, h, skips = self._enc
        eps = p.unet.decode(h, skips, temb, p.ctx, self.views, [1.0] * len(self.views))
        self.ops.cfg_ddim_step(eps, p.x, p.coef, p.step_dev, unet_in=p.unet_in)
        # timestep of the NEXT step rides in the message
        self.msg[self.L:self.L + 1].copy_(p.t_table.index_select(0, p.step_dev[:1].long()))

    def _capture(self, name, fn, pool=None):
        s = torch.cuda.current_stream(self.device)
        side = self.capture_stream
        side.wait_stream(s)
        with torch.cuda.stream(side):
            fn()                                  # warm-up on the capture stream
        s.wait_stream(side)
        g = torch.cuda.CUDAGraph()
        c0 = self.ops.LAUNCHES["count"]
        with torch.cuda.graph(g, pool=pool, stream=side):
            fn()
        self.graph_launches[name] = self.ops.LAUNCHES["count"] - c0   # our kernels per replay
        self.graphs[name] = g
        return g

    @property
    def launches_per_step(self) -> int:
        """This repo's kernels issued per denoising step by this node's graphs."""
        if self.role == "solo":
            return self.pipe.launches_per_step
        g = self.graph_launches
        if self.role == "base":
            return g.get("enc_pristine", 0) + g.get("dec_pristine", 0)
        if self.role == "service":
            return g.get("svc", 0)
        return self.pipe.launches_per_step

    def load_loras(self, adapters, host_resident: bool = False, groups: int = 1) -> None:
        """LoRA lives on the base UNet only (ControlNets are not patched).
        groups > 1: group-pipelined patching (AddonPipeline.load_loras)."""
        if self.role in ("base", "solo"):
            self.pipe.load_loras(adapters, host_resident=host_resident, groups=groups)

    def setup(self) -> None:
        if self.role == "solo":
            self.pipe.setup()
            return
        if self.role == "base":
            p = self.pipe
            _ = p._pristine
            variants = ["pristine"] + (["patched"] if p.patchset is not None else [])
            if p.patch_groups:           # partially patched weight sets of the grouped patch
                variants += [f"pg{v}" for v in range(1, len(p.patch_groups))]
            for which in variants:
                # one memory pool per (encoder, decoder) pair: the pair hands its
                # activations over inside the pool, pairs never share one
                p._use_weights(which)
                p.step_dev.zero_()
                g = self._capture("enc_" + which, self._base_encode)
                self._capture("dec_" + which, self._base_decode, pool=g.pool())
                p._use_weights("pristine")
            p.step_dev.zero_()
        else:
            self._capture("svc", self._service_step)
        torch.cuda.synchronize(self.device)

    # -- per request -------------------------------------------------------------
    def request_tensors(self, context=None, images=None, pooled=None, time_ids=None) -> list:
        """The conditioning tensors shipped base -> services once per request
        (filled on the base, receive buffers elsewhere)."""
        cfg, dev, h, nb = self.cfg, self.device, self.cfg.latent_hw, 2 * self.batch
        ctx = torch.empty((nb, cfg.context_len, cfg.context_dim), device=dev, dtype=torch.float32)
        imgs = [torch.empty((nb, 3, 8 * h, 8 * h), device=dev, dtype=torch.float32) for _ in range(self.layout.n_cn)]
        extra = [torch.empty((nb, cfg.pooled_dim), device=dev), torch.empty((nb, cfg.time_ids), device=dev)] \
            if cfg.addition_embed else []
        if self.role == "base":
            ctx.copy_(context.to(dev, non_blocking=True))
            for b, im in zip(imgs, images):
                b.copy_(im.to(dev, non_blocking=True))
            if cfg.addition_embed:
                extra[0].copy_(pooled.to(dev, non_blocking=True))
                extra[1].copy_(time_ids.to(dev, non_blocking=True))
        return [ctx] + imgs + extra

    def finish_prepare(self, shared: list, latent=None) -> None:
        """Step-invariant per-request work once the conditioning is local."""
        cfg = self.cfg
        ctx, imgs = shared[0], shared[1:1 + self.layout.n_cn]
        extra = shared[1 + self.layout.n_cn:]
        if self.role == "base":
            self.pipe.prepare(latent, ctx, [], extra[0] if extra else None, extra[1] if extra else None)
            self.msg[self.L:self.L + 1].copy_(self.pipe.t_table[:1])
            return
        self.ctx.copy_(ctx)
        for k, (i, cn) in enumerate(zip(self.cn_idx, self.cns)):
            self.hints[k].copy_(cn.hint_embedding(imgs[i].to(self.ctx.dtype)))
            if cfg.addition_embed:
                self.add_emb[k].copy_(cn.add_embedding(extra[0], extra[1]))
            cn.compute_kv(self.ctx, "pristine")

    def prepare(self, latent=None, context=None, images=None, pooled=None, time_ids=None) -> None:
        """Base passes the request; services receive it (their args are ignored)."""
        if self.role == "solo":
            self.pipe.prepare(latent, context, images, pooled, time_ids)
            return
        shared = self.request_tensors(context, images, pooled, time_ids)
        self.proto.share_request(shared)
        self.finish_prepare(shared, latent)

    def base_encode(self, which: str = "pristine") -> None:
        self.graphs["enc_" + which].replay()

    def base_decode(self, which: str = "pristine") -> None:
        self.graphs["dec_" + which].replay()

    def service_step(self) -> None:
        self.graphs["svc"].replay()

    def start_patch(self, boundary: Optional[int] = None, fetch: bool = True):
        """Base: launch the request's LoRA patch (shadow weights, low-priority
        side stream) and return (first_patched_step, event) — same semantics as
        AddonPipeline.denoise (schedule.plan_lora_patch)."""
        from .schedule import plan_lora_patch
        p = self.pipe
        if boundary is None:
            if p.step_ms_est is None or p.patch_ms_est is None:
                raise RuntimeError("calibrate the base (step_ms_est / patch_ms_est) or pass a boundary")
            first = plan_lora_patch(p.patch_ms_est, p.step_ms_est, 0.0, self.steps).first_patched_step
        else:
            first = boundary + 1
        timing = p.patch_timing is not None
        p0, ev = p.launch_patch(timing=timing, fetch=fetch)
        if timing:
            p.patch_timing.append((p0, p.last_patch_k1_event))
        p.last_first_patched_step = first
        return first, ev

    def start_patch_schedule(self, patch: bool, boundary: Optional[int] = None, fetch: bool = True,
                             boundaries: Optional[Sequence[int]] = None) -> "PatchSchedule":
        """Base: launch the request's patch — one K1 launch, or with grouped
        adapters every group's fetch -> pack -> K1 chain — and return the
        per-step weight-set schedule (forced boundary / boundaries, or planned
        by plan_lora_patch / plan_pipeline_patch from the calibrated times)."""
        p = self.pipe
        if not patch:
            return PatchSchedule([], [], self.steps)
        if not p.patch_groups:
            first, ev = self.start_patch(boundary, fetch=fetch)
            return PatchSchedule([first - 1 if first <= self.steps else None], [ev], self.steps)
        from .schedule import plan_pipeline_patch
        M = len(p.patch_groups)
        if boundaries is not None:
            bounds = list(boundaries)
        elif boundary is not None:
            bounds = [boundary] * M
        else:
            if p.step_ms_est is None or p.group_loads_ms is None:
                raise RuntimeError("calibrate the base (step_ms_est / calibrate_groups) or pass boundaries")
            plan = plan_pipeline_patch(p.group_loads_ms, p.step_ms_est, 0.0, self.steps)
            bounds = [g.boundary_step for g in plan.groups] + [None] * (M - len(plan.groups))
        if len(bounds) != M:
            raise ValueError(f"need {M} group boundaries")
        _, ready = p.launch_patch_groups(timing=False, fetch=fetch)
        p.last_group_boundaries = bounds
        sched = PatchSchedule(bounds, ready, self.steps)
        p.last_first_patched_step = sched.first_full
        return sched

    def denoise(self, patch: bool = False, boundary: Optional[int] = None, fetch: bool = True,
                boundaries: Optional[Sequence[int]] = None, timeline: Optional["StepTimeline"] = None) -> None:
        """timeline: per-step events — on the base the encoder end, decoder
        start / end (the decoder start is when every service's residuals were
        in); on a service the ControlNet compute (message arrival -> residuals
        pushed).  A solo rank records nothing."""
        if self.role == "solo":
            if self.pipe.patch_groups and patch:
                self.pipe.denoise_pipelined(boundaries or ([boundary] * len(self.pipe.patch_groups)
                                                           if boundary is not None else None), fetch=fetch)
            else:
                self.pipe.denoise(patch=patch, boundary=boundary, fetch=fetch)
            return
        sched = (self.start_patch_schedule(patch, boundary, fetch, boundaries) if self.role == "base"
                 else PatchSchedule([], [], self.steps))
        s = torch.cuda.current_stream(self.device)
        for step in range(1, self.steps + 1):
            if self.role == "base":
                which = sched.weights_at(step, s)
                rec = timeline.begin(s) if timeline is not None else None
                works = self.proto.base_step_begin()
                self.base_encode(which)               # overlaps the services' ControlNets
                if rec is not None:
                    rec["enc_end"].record(s)
                for w in works:
                    w.wait()                          # decoder after the encoder AND every branch
                if rec is not None:
                    rec["dec_start"].record(s)
                self.base_decode(which)
                if rec is not None:
                    rec["dec_end"].record(s)
            else:
                self.proto.service_receive()
                rec = timeline.begin(s) if timeline is not None else None
                self.service_step()
                self.proto.service_send()
                if rec is not None:                   # a service's step: its compute (+ push)
                    for k in ("enc_end", "dec_start", "dec_end"):
                        rec[k].record(s)
        sched.finish(s)

    def latent_nchw(self) -> Optional[torch.Tensor]:
        if self.role == "service":
            return None
        return self.pipe.latent_nchw()


class StepTimeline:
    """Per-step CUDA events of the CaaS step (orchestrator.py:621-660) and the
    reference's split of the decoder's wait (``_attribute_stall``
    :662-678): the gap between the encoder's end and the decoder's start is
    charged, back to front along the critical (last-ready) branch, to the
    transfer tail (comm), the branch's ControlNet compute, a weight fetch
    (none here: the ControlNets stay resident) and, for what remains,
    queueing.  Times come from events on the streams that did the work."""

    def __init__(self):
        self.steps = []     # per step: dict of events

    @staticmethod
    def _ev():
        return torch.cuda.Event(enable_timing=True)

    def begin(self, stream) -> dict:
        rec = {"start": self._ev(), "branches": [], "enc_end": self._ev(), "dec_start": self._ev(),
               "dec_end": self._ev()}
        rec["start"].record(stream)
        self.steps.append(rec)
        return rec

    def summary(self, comm_ms: float = 0.0, branch_ms: Optional[float] = None) -> dict:
        """Mean per-step ms: encoder, each branch (ControlNet compute, from the
        step start), decoder, the decoder's wait and its comm / compute /
        fetch / queue split (reference accounting).  branch_ms: the critical
        branch's per-step time measured elsewhere (multi-GPU: on the service
        ranks, compute + push) when this timeline has no branch events."""
        n = len(self.steps)
        if n == 0:
            return {}
        acc = {"encoder_ms": 0.0, "decoder_ms": 0.0, "decoder_wait_ms": 0.0, "comm_ms": 0.0,
               "controlnet_wait_ms": 0.0, "cache_fetch_ms": 0.0, "queue_ms": 0.0, "step_ms": 0.0}
        branch = None
        for r in self.steps:
            enc = r["start"].elapsed_time(r["enc_end"])
            br = [r["start"].elapsed_time(e) for e in r["branches"]]
            gap = max(0.0, r["enc_end"].elapsed_time(r["dec_start"]))
            acc["encoder_ms"] += enc
            acc["decoder_ms"] += r["dec_start"].elapsed_time(r["dec_end"])
            acc["step_ms"] += r["start"].elapsed_time(r["dec_end"])
            acc["decoder_wait_ms"] += gap
            branch = [a + b for a, b in zip(branch, br)] if branch is not None else br
            crit = max(br) if br else branch_ms
            if gap > 0 and crit is not None:
                comm = min(gap, comm_ms)
                rest = gap - comm
                compute = min(rest, crit)             # the critical branch's compute
                rest -= compute
                acc["comm_ms"] += comm
                acc["controlnet_wait_ms"] += compute
                acc["queue_ms"] += rest               # fetch: 0 (resident weights)
        out = {k: v / n for k, v in acc.items()}
        out["branch_ms"] = [b / n for b in (branch or [])]
        out["steps"] = n
        return out


class LoopbackGroup:
    """One CaaS group with every role in ONE process on ONE GPU.

    The services read the base's message buffer and write straight into the
    base's per-service residual buffers (aliased, no transfer).  Exercises
    exactly the split compute of the multi-GPU path — encoder and decoder
    graphs, scale-folded service ControlNets, per-service residual buffers
    summed by K3 — so its parity with the single-GPU pipeline is testable on
    one B200.  With ``concurrent=True`` each service's ControlNet graph runs on
    its own stream alongside the base's encoder graph (the paper's branch
    parallelism inside one GPU: the 32x32-level GEMMs of SDXL at CFG batch 2
    fill barely half of the 148 SMs, the branches fill the rest); the decoder
    waits for every branch (orchestrator.py:652-653)."""

    def __init__(self, cfg, n_cn: int, cn_scales: Sequence[float], steps: int = 30, guidance: float = 7.5,
                 dtype=torch.bfloat16, seed: int = 0, n_services: Optional[int] = None,
                 concurrent: bool = False, batch: int = 1):
        world = 1 + (n_cn if n_services is None else n_services)
        self.layout = caas_layout(world, n_cn)
        self.nodes = [CaaSNode(cfg, self.layout, r, cn_scales, steps, guidance, dtype, seed, batch=batch)
                      for r in range(world)]
        self.base, self.services = self.nodes[0], self.nodes[1:]
        for k, svc in enumerate(self.services):   # alias before any graph is captured
            svc.msg = self.base.msg
            svc.flats = [self.base.flats[k]]
            svc.views = [self.base.views[k]]
        self.steps = steps
        self.concurrent = concurrent
        dev = self.base.device
        self.streams = [torch.cuda.Stream(device=dev) for _ in self.services] if concurrent else []
        self.main_stream = torch.cuda.Stream(device=dev, priority=-1)

    def setup(self) -> None:
        for n in self.nodes:
            n.setup()

    def prepare(self, latent, context, images, pooled=None, time_ids=None) -> None:
        shared = self.base.request_tensors(context, images, pooled, time_ids)
        self.base.finish_prepare(shared, latent)
        for s in self.services:
            s.finish_prepare([t.clone() for t in shared])

    def denoise(self, patch: bool = False, boundary: Optional[int] = None, on_step=None,
                fetch: bool = True, boundaries: Optional[Sequence[int]] = None,
                timeline: Optional[StepTimeline] = None) -> None:
        sched = self.base.start_patch_schedule(patch, boundary, fetch, boundaries)
        s = torch.cuda.current_stream()
        for step in range(1, self.steps + 1):
            which = sched.weights_at(step, s)
            rec = timeline.begin(s) if timeline is not None else None
            if self.concurrent:
                done = []
                for svc, st in zip(self.services, self.streams):
                    st.wait_stream(s)              # message of this step is written
                    with torch.cuda.stream(st):
                        svc.service_step()
                    e = torch.cuda.Event(enable_timing=rec is not None)
                    e.record(st)
                    done.append(e)
                self.base.base_encode(which)
                if rec is not None:
                    rec["enc_end"].record(s)
                    rec["branches"] = done
                for e in done:
                    s.wait_event(e)
            else:
                for svc in self.services:
                    svc.service_step()
                    if rec is not None:
                        e = StepTimeline._ev()
                        e.record(s)
                        rec["branches"].append(e)
                self.base.base_encode(which)
                if rec is not None:
                    rec["enc_end"].record(s)
            if rec is not None:
                rec["dec_start"].record(s)
            self.base.base_decode(which)
            if rec is not None:
                rec["dec_end"].record(s)
            if on_step is not None:
                on_step(step, self.latent_nchw().clone())
        sched.finish(s)

    def load_loras(self, adapters, host_resident: bool = False, groups: int = 1) -> None:
        self.base.load_loras(adapters, host_resident=host_resident, groups=groups)

    def latent_nchw(self) -> torch.Tensor:
        return self.base.latent_nchw()
