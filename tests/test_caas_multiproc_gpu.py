"""The multi-PROCESS ControlNet-as-a-service path end to end on one B200:
world-size 2 and 3 process groups (gloo, device buffers staged through host
memory — NCCL refuses two ranks on one GPU) running caas.CaaSNode exactly as
bench.py does under torchrun: per-request conditioning broadcast, per-step
latent broadcast + residual sends, encoder/decoder graphs on the base, LoRA
patched asynchronously on the base.  The base's latent must equal the
single-GPU pipeline's (fp32, TF32 off)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
STEPS = 4
SCALES = [0.8, 0.6]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, transport):
    import torch.distributed as dist
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.caas import CaaSNode, caas_layout
    from paper_2407_02031_b200.patcher import synthetic_lora
    from paper_2407_02031_b200.pipeline import synthetic_request
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SDB_CAAS_TRANSPORT=transport.split("-")[0])
    if transport.endswith("-fail1"):       # rank 1's peer self-test fails: the group must fall back together
        os.environ["SDB_CAAS_P2P_SELFTEST"] = "fail1"
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    node = CaaSNode(U.TOY, caas_layout(world, 2), rank, SCALES, steps=STEPS, dtype=torch.float32, seed=0)
    if node.role == "base":
        node.load_loras([(synthetic_lora(node.pipe.unet_p, 8, seed=7), 0.75)])
    node.setup()
    req = synthetic_request(U.TOY, 2)
    if node.role in ("base", "solo"):
        if node.role == "solo":
            node.load_loras([(synthetic_lora(node.pipe.unet_p, 8, seed=7), 0.75)])
            node.setup()
        node.prepare(torch.from_numpy(req.latent), torch.from_numpy(req.context),
                     [torch.from_numpy(i) for i in req.images])
        node.denoise(patch=True, boundary=1)
        torch.cuda.synchronize()
        out["latent" if node.role == "base" else f"solo{rank}"] = node.latent_nchw().cpu().clone()
        if node.role == "base":
            out["transport"] = type(node.proto).__name__
    else:
        node.prepare()
        node.denoise()
        torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def single_gpu():
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.patcher import synthetic_lora
    from paper_2407_02031_b200.pipeline import AddonPipeline, synthetic_request
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    pipe = AddonPipeline(U.TOY, n_controlnets=2, cn_scales=SCALES, steps=STEPS, dtype=torch.float32, seed=0)
    pipe.load_loras([(synthetic_lora(pipe.unet_p, 8, seed=7), 0.75)])
    pipe.setup()
    req = synthetic_request(U.TOY, 2)
    pipe.prepare(torch.from_numpy(req.latent), torch.from_numpy(req.context), [torch.from_numpy(i) for i in req.images])
    pipe.denoise(patch=True, boundary=1)
    torch.cuda.synchronize()
    return pipe.latent_nchw().cpu().clone()


@pytest.mark.parametrize("world,transport", [(2, "p2p"), (3, "p2p"), (4, "p2p"), (3, "nccl"), (3, "p2p-fail1")])
def test_multiprocess_caas_matches_single_gpu(world, transport):
    """transport p2p: CaaSPeerProtocol (IPC mappings + GPU-side step flags; on
    one GPU the 'peer' copies are same-device copies); nccl: CaaSProtocol
    (here gloo, device buffers staged through the host).  world 4 adds a solo
    rank (serves whole images alone, no transport); p2p-fail1: rank 1's setup
    self-test of the peer path fails, so the whole group takes the NCCL
    transport (caas.make_protocol)."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out, transport)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    got = out["latent"]
    assert out["transport"] == ("CaaSPeerProtocol" if transport == "p2p" else "CaaSProtocol")   # p2p-fail1: fallback
    ref = single_gpu()
    rel = float((got.double() - ref.double()).norm() / ref.double().norm())
    print(f"world {world}: multi-process CaaS vs single GPU rel-L2 {rel:.2e}")
    assert rel <= 1e-5
    for k in out.keys():
        if k.startswith("solo"):    # a solo rank runs the whole pipeline itself
            r2 = float((out[k].double() - ref.double()).norm() / ref.double().norm())
            assert r2 <= 1e-5, (k, r2)
