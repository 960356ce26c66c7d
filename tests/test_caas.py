"""ControlNet-as-a-service host logic on CPU (gloo, world sizes 2 and 3): the
layout planner and the per-request / per-step exchange protocol of caas.py,
driven by a stand-in compute, checked against the serial schedule
(reference: addonsim/orchestrator.py:181-188, 621-660 — the decoder consumes
every branch's output; outputs are summed)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_02031_b200.caas import CaaSProtocol, caas_layout, flat_views, make_groups, residual_layout

L = 16
SHAPES = [(2, 8, 4, 4), (2, 8, 2, 2), (2, 16, 2, 2)]   # two "down" levels + mid
STEPS = 3
SCALES = [0.8, 0.5]


def test_layouts():
    lay = caas_layout(1, 2)
    assert lay.role(0) == "solo"
    lay = caas_layout(2, 2)
    assert lay.groups[0].services == (1,) and lay.groups[0].cn_of_service == ((0, 1),)
    assert lay.role(0) == "base" and lay.role(1) == "service"
    lay = caas_layout(3, 2)
    assert lay.groups[0].cn_of_service == ((0,), (1,))
    lay = caas_layout(4, 2)
    assert [g.ranks for g in lay.groups] == [(0, 1, 2), (3,)] and lay.role(3) == "solo"
    lay = caas_layout(8, 3)
    assert [g.ranks for g in lay.groups] == [(0, 1, 2, 3), (4, 5, 6, 7)]
    assert all(len(c) == 1 for g in lay.groups for c in g.cn_of_service)
    lay = caas_layout(8, 2)
    assert [g.ranks for g in lay.groups] == [(0, 1, 2), (3, 4, 5), (6,), (7,)]


def test_flat_views_are_channels_last_windows():
    offs, total = residual_layout(SHAPES)
    flat = torch.arange(total, dtype=torch.float32)
    views = flat_views(flat, SHAPES)
    for o, v, s in zip(offs, views, SHAPES):
        assert v.shape == s and v.is_contiguous(memory_format=torch.channels_last)
        assert v.data_ptr() == flat[o:].data_ptr()


def fake_branch(msg, cn):
    """Stand-in ControlNet: residual level j = scale * (sum(latent) * (cn + 1) + t + j)."""
    s = float(msg[:L].sum()) * (cn + 1) + float(msg[L])
    return [torch.full(sh, SCALES[cn] * (s + j)) for j, sh in enumerate(SHAPES)]


def serial_reference():
    msg = torch.zeros(L + 1)
    msg[:L] = torch.linspace(-1, 1, L)
    msg[L] = 999.0
    for _ in range(STEPS):
        res = [fake_branch(msg, cn) for cn in range(2)]
        total = sum(float(r.sum()) for rr in res for r in rr)
        msg[:L] = msg[:L] * 0.5 + total / 1e4
        msg[L] -= 50.0
    return msg


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lay = caas_layout(world, 2)
    role = lay.role(rank)
    g = lay.group_of(rank)
    if role == "solo":          # still takes part in creating every group's communicator
        assert make_groups(lay, rank) is None
        dist.barrier()
        dist.destroy_process_group()
        return
    _, total = residual_layout(SHAPES)
    msg = torch.zeros(L + 1)
    nflat = len(g.services) if role == "base" else 1
    flats = [torch.zeros(total) for _ in range(nflat)]
    proto = CaaSProtocol(lay, rank, msg, flats)
    # per request: the base's conditioning reaches every service
    cond = torch.arange(6, dtype=torch.float32) if role == "base" else torch.zeros(6)
    proto.share_request([cond])
    assert torch.equal(cond, torch.arange(6, dtype=torch.float32))
    if role == "base":
        msg[:L] = torch.linspace(-1, 1, L)
        msg[L] = 999.0
    mine = g.cn_of_service[g.services.index(rank)] if role == "service" else ()
    for _ in range(STEPS):
        if role == "base":
            works = proto.base_step_begin()
            for w in works:
                w.wait()
            total_sum = sum(float(f.sum()) for f in flats)
            msg[:L] = msg[:L] * 0.5 + total_sum / 1e4
            msg[L] -= 50.0
        else:
            proto.service_receive()
            views = flat_views(flats[0], SHAPES)
            parts = [fake_branch(msg, cn) for cn in mine]
            for j, v in enumerate(views):
                v.copy_(sum(p[j] for p in parts))
            for w in proto.service_send():
                w.wait()
    if role == "base":
        out[0] = msg.clone()
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3, 4])
def test_protocol_matches_serial_schedule(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = out[0]
    ref = serial_reference()
    assert torch.allclose(got, ref, rtol=1e-5, atol=1e-4), (got, ref)
