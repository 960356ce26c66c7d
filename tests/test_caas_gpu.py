"""The multi-GPU ControlNet-as-a-service compute split, exercised on ONE B200
through the loopback group (caas.LoopbackGroup): encoder / decoder graphs on
the base, scale-folded ControlNets on the services, per-service residual
buffers summed by K3.  It must reproduce the single-GPU pipeline (which runs
the ControlNets inline, addonsim/orchestrator.py:611-619) — the reference's
claim that CaaS changes latency, not results."""

import pytest
import torch

from paper_2407_02031_b200 import unet as U
from paper_2407_02031_b200.caas import LoopbackGroup
from paper_2407_02031_b200.patcher import synthetic_lora
from paper_2407_02031_b200.pipeline import AddonPipeline, synthetic_request

pytestmark = pytest.mark.gpu
STEPS = 6
SCALES = [0.8, 0.6]


def rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm())


@pytest.fixture(scope="module")
def fp32_mode():
    old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old


def inputs(req):
    return [torch.from_numpy(req.latent), torch.from_numpy(req.context), [torch.from_numpy(i) for i in req.images]]


def single_gpu(dtype, patch):
    pipe = AddonPipeline(U.TOY, n_controlnets=2, cn_scales=SCALES, steps=STEPS, dtype=dtype, seed=0)
    if patch:
        pipe.load_loras([(synthetic_lora(pipe.unet_p, 8, seed=7), 0.75)])
    pipe.setup()
    req = synthetic_request(U.TOY, 2)
    pipe.prepare(*inputs(req))
    lat = []
    pipe.denoise(patch=patch, boundary=2, on_step=lambda s, x: lat.append(x.float().cpu()))
    return lat


def loopback(dtype, patch, n_services, concurrent=False):
    grp = LoopbackGroup(U.TOY, 2, SCALES, steps=STEPS, dtype=dtype, seed=0, n_services=n_services,
                        concurrent=concurrent)
    if patch:
        grp.load_loras([(synthetic_lora(grp.base.pipe.unet_p, 8, seed=7), 0.75)])
    grp.setup()
    req = synthetic_request(U.TOY, 2)
    grp.prepare(*inputs(req))
    lat = []
    grp.denoise(patch=patch, boundary=2, on_step=lambda s, x: lat.append(x.float().cpu()))
    return lat


@pytest.mark.parametrize("n_services", [1, 2])
def test_caas_split_matches_single_gpu_fp32(fp32_mode, n_services):
    ref = single_gpu(torch.float32, patch=True)
    got = loopback(torch.float32, patch=True, n_services=n_services)
    errs = [rel(a, b) for a, b in zip(got, ref)]
    print("caas vs single (fp32):", ["%.1e" % e for e in errs])
    assert max(errs) <= 1e-5


def test_concurrent_branches_are_bitwise_serial():
    """ControlNet graphs on their own streams beside the encoder graph: same
    kernels, same inputs -> bitwise the serial loopback (no shared workspace)."""
    a = loopback(torch.bfloat16, patch=True, n_services=2, concurrent=True)
    b = loopback(torch.bfloat16, patch=True, n_services=2, concurrent=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_caas_split_bf16_within_the_bf16_floor(fp32_mode):
    """bf16 CaaS differs from bf16 single-GPU only by rounding placement (scales
    folded into the zero convs, per-service sums); both must sit inside the
    bf16 error band around the fp32 result (tests/test_pipeline_gpu.py)."""
    ref32 = single_gpu(torch.float32, patch=True)
    single = single_gpu(torch.bfloat16, patch=True)
    got = loopback(torch.bfloat16, patch=True, n_services=2)
    e_single = [rel(a, b) for a, b in zip(single, ref32)]
    e_caas = [rel(a, b) for a, b in zip(got, ref32)]
    print("bf16 single vs fp32:", ["%.1e" % e for e in e_single])
    print("bf16 caas   vs fp32:", ["%.1e" % e for e in e_caas])
    assert max(e_caas) <= 2e-2 and max(e_single) <= 2e-2


def test_caas_group_pipelined_patch_matches_single_gpu(fp32_mode):
    """Group-pipelined patching on the CaaS base (encoder/decoder graphs per
    partial weight set) == the single-GPU pipeline's denoise_pipelined at the
    same group boundaries."""
    bounds = [1, 2, 4]
    lora_of = lambda p: [(synthetic_lora(p.unet_p, 8, seed=7), 0.75)]   # noqa: E731
    pipe = AddonPipeline(U.TOY, n_controlnets=2, cn_scales=SCALES, steps=STEPS, dtype=torch.float32, seed=0)
    pipe.load_loras(lora_of(pipe), host_resident=True, groups=3)
    pipe.setup()
    req = synthetic_request(U.TOY, 2)
    pipe.prepare(*inputs(req))
    ref = []
    pipe.denoise_pipelined(bounds, on_step=lambda s, x: ref.append(x.float().cpu()))
    grp = LoopbackGroup(U.TOY, 2, SCALES, steps=STEPS, dtype=torch.float32, seed=0, concurrent=True)
    grp.load_loras(lora_of(grp.base.pipe), host_resident=True, groups=3)
    grp.setup()
    grp.prepare(*inputs(req))
    got = []
    grp.denoise(patch=True, boundaries=bounds, on_step=lambda s, x: got.append(x.float().cpu()))
    assert grp.base.pipe.last_group_boundaries == bounds
    errs = [rel(a, b) for a, b in zip(got, ref)]
    print("caas grouped vs single grouped (fp32):", ["%.1e" % e for e in errs])
    assert max(errs) <= 1e-5
    # and the partial sets really differ from an all-at-once patch at the last boundary
    once = loopback(torch.float32, patch=True, n_services=2)
    assert rel(got[2], once[2]) > 1e-6 or rel(got[3], once[3]) > 1e-6
