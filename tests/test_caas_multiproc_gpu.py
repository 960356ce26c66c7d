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


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.caas import CaaSNode, caas_layout
    from paper_2407_02031_b200.patcher import synthetic_lora
    from paper_2407_02031_b200.pipeline import synthetic_request
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    node = CaaSNode(U.TOY, caas_layout(world, 2), rank, SCALES, steps=STEPS, dtype=torch.float32, seed=0)
    if node.role == "base":
        node.load_loras([(synthetic_lora(node.pipe.unet_p, 8, seed=7), 0.75)])
    node.setup()
    req = synthetic_request(U.TOY, 2)
    if node.role == "base":
        node.prepare(torch.from_numpy(req.latent), torch.from_numpy(req.context),
                     [torch.from_numpy(i) for i in req.images])
        node.denoise(patch=True, boundary=1)
        torch.cuda.synchronize()
        out["latent"] = node.latent_nchw().cpu().clone()
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


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_caas_matches_single_gpu(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    got = out["latent"]
    ref = single_gpu()
    rel = float((got.double() - ref.double()).norm() / ref.double().norm())
    print(f"world {world}: multi-process CaaS vs single GPU rel-L2 {rel:.2e}")
    assert rel <= 1e-5
