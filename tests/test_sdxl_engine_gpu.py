"""The benchmarked engine itself against the CPU oracle, at the headline
config (BASELINE config 3) and at config 2 (SD1.5 512^2 + 1 ControlNet + 1
LoRA r16, same engine).  Config 3: SDXL-shaped UNet at 128x128 latent + 2
ControlNets (scales 0.8 / 0.6) on their own streams beside the UNet encoder
(``caas.LoopbackGroup(concurrent=True)``, exactly what ``bench.py`` times) +
2 LoRAs r64 at 0.7, host-resident (``AdapterBank`` -> H2D -> ``pack_multi``
-> K1) and swapped in after step 1 (boundary 1), CFG 7.5, DDIM.

Two steps of a 2-step schedule (step 1 on the pristine weights, step 2 on
the patched ones), compared per step with oracle/pipeline_ref.denoise on the
same parameter values (parity unpinned by the reference, see its header):

* fp32 engine (TF32 off) against the fp32 oracle AND the same oracle in
  fp64 (the exact result): the north_star's 1e-5 is below the fp32 floor
  at SDXL / SD1.5 depth (the fp32 oracle is itself 7.8e-6 / 1.9e-5 from
  fp64), so the gate is "as accurate as the fp32 oracle" — see the test.
  The LoRA runs through the SIMT K1 (fp32 weights).
* bf16 engine (the benchmarked precision; tcgen05 K1 pair kernel, K7
  tcgen05 form at head dim 64, gn_cluster, conv_in / hint padding,
  stride-1 downsample + subsample): against the bf16-emulated oracle
  (every linear / conv / norm output and the merged weights rounded to
  bf16) and the fp32 oracle.  Gates: device-vs-fp32 <= 1.25x the
  emulator's own distance to fp32 (+1e-4) — the device adds no error beyond
  the rounding floor of bf16 activations — and device-vs-emulator <= 1.5x
  that floor (independent roundings of equal size differ by ~sqrt(2)x).
  DESIGN.md §4 shows why 1e-3 vs fp32 is below that floor.

Per-step numbers are printed (``-s``) and kept in profiles/r02_sdxl_parity.txt.
The CPU oracle runs one SDXL step of UNet + 2 ControlNets in ~15 s on the GPU
box's host cores, plus the reference-restated fp64 LoRA merge of all 794
matrices."""

import pytest
import torch

from oracle import pipeline_ref as R
from paper_2407_02031_b200 import unet as U
from paper_2407_02031_b200.caas import LoopbackGroup
from paper_2407_02031_b200.patcher import synthetic_lora
from paper_2407_02031_b200.pipeline import synthetic_request

pytestmark = pytest.mark.gpu

STEPS, BOUNDARY, GUIDANCE = 2, 1, 7.5
LORA_SCALE = 0.7
# BASELINE config 3 (the headline) and config 2 (SD1.5 + 1 ControlNet + 1 LoRA r16)
ENGINES = {"sdxl": (U.SDXL, [0.8, 0.6], (64, 64)), "sd15": (U.SD15, [0.8], (16,))}


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm())


def run_engine(dtype, name="sdxl"):
    cfg, scales, ranks = ENGINES[name]
    n_cn = len(scales)
    grp = LoopbackGroup(cfg, n_cn, scales, steps=STEPS, guidance=GUIDANCE, dtype=dtype, seed=0, concurrent=True)
    pipe = grp.base.pipe
    loras = [synthetic_lora(pipe.unet_p, r, seed=10 + i, adapter_id=f"lora{i}", scale=LORA_SCALE)
             for i, r in enumerate(ranks)]
    grp.load_loras([(lo, LORA_SCALE) for lo in loras], host_resident=True)
    grp.setup()
    req = synthetic_request(cfg, n_cn, seed=0)
    dev = dict(latent=torch.from_numpy(req.latent).cuda(), context=torch.from_numpy(req.context).cuda(),
               images=[torch.from_numpy(i).cuda() for i in req.images])
    if req.pooled is not None:
        dev.update(pooled=torch.from_numpy(req.pooled).cuda(), time_ids=torch.from_numpy(req.time_ids).cuda())
    per_step = []
    with torch.cuda.stream(grp.main_stream):
        grp.prepare(**dev)
        grp.denoise(patch=True, boundary=BOUNDARY, on_step=lambda s, x: per_step.append(x.float().cpu()))
    torch.cuda.synchronize()
    # oracle inputs: the same parameter values; the services fold the
    # conditioning scale into their zero convs, so the oracle takes the
    # unscaled ControlNets (same seeds) and applies the scales itself
    up = R.to_cpu_params(pipe.unet_p)
    cps = [R.to_cpu_params(U.init_controlnet(cfg, "cuda", dtype, seed=1000 + i)) for i in range(n_cn)]
    factors = [(lo.factors, LORA_SCALE) for lo in loras]
    return per_step, up, cps, factors, pipe.unet_p.matrices, req


def oracle(up, cps, factors, matrices, req, bf16_acts, name="sdxl", max_steps=None):
    cfg, scales, _ = ENGINES[name]
    return R.denoise(cfg, up, cps, req, scales, STEPS, GUIDANCE, adapters=factors, matrices=matrices,
                     boundary=BOUNDARY, bf16_acts=bf16_acts, max_steps=max_steps)


@pytest.fixture
def fp32_mode():
    old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old


@pytest.mark.parametrize("name", ["sdxl", "sd15"])
def test_engine_fp32_per_step(fp32_mode, name):
    dev, up, cps, factors, matrices, req = run_engine(torch.float32, name)
    torch.cuda.empty_cache()
    ref = oracle(up, cps, factors, matrices, req, False, name)
    errs = [rel(a, b) for a, b in zip(dev, ref)]
    # the same oracle in fp64 (step 1, before the patch lands): how far fp32
    # arithmetic itself (device or CPU) sits from the exact result at SDXL depth
    up64 = {k: v.double() for k, v in up.items()}
    cps64 = [{k: v.double() for k, v in c.items()} for c in cps]
    del up, cps
    truth = oracle(up64, cps64, None, matrices, req, False, name, max_steps=1)   # step 1: pristine weights
    d_truth = [rel(a, b) for a, b in zip(dev, truth)]
    o_truth = [rel(a, b) for a, b in zip(ref, truth)]
    print(f"{name} engine fp32 per-step rel-L2: device-vs-oracle", ["%.2e" % e for e in errs],
          "device-vs-fp64", ["%.2e" % e for e in d_truth], "oracle(fp32)-vs-fp64", ["%.2e" % e for e in o_truth])
    assert len(errs) == STEPS
    # The north_star's 1e-5 sits AT the fp32 arithmetic floor of these
    # networks: the fp32 CPU oracle itself is 7.8e-6 (SDXL) / 1.9e-5 (SD1.5)
    # from the fp64 truth, so two correct fp32 evaluations differ by about
    # that much (measured: profiles/r02_sdxl_parity.txt).  Gate: the device
    # is as accurate as the fp32 oracle (vs the fp64 truth, within 2x), and
    # device-vs-oracle <= 1e-5 or, where the oracle's own floor exceeds it,
    # <= 2x that floor.
    for d, o in zip(d_truth, o_truth):
        assert d <= 2.0 * o
    assert max(errs) <= max(1e-5, 2.0 * max(o_truth))


@pytest.mark.parametrize("name", ["sdxl", "sd15"])
def test_engine_bf16_per_step(name):
    dev, up, cps, factors, matrices, req = run_engine(torch.bfloat16, name)
    torch.cuda.empty_cache()
    ref = oracle(up, cps, factors, matrices, req, False, name)
    emu = oracle(up, cps, factors, matrices, req, True, name)
    d_ref = [rel(a, b) for a, b in zip(dev, ref)]
    d_emu = [rel(a, b) for a, b in zip(dev, emu)]
    floor = [rel(a, b) for a, b in zip(emu, ref)]
    print(f"{name} engine bf16 per-step rel-L2: device-vs-fp32", ["%.2e" % e for e in d_ref],
          "device-vs-bf16-emulator", ["%.2e" % e for e in d_emu], "emulator-vs-fp32", ["%.2e" % e for e in floor])
    for a, e, f in zip(d_ref, d_emu, floor):
        # two bf16 implementations with independent rounding sit ~sqrt(2) x
        # the floor apart; the device adds nothing beyond the floor itself
        assert e <= 1.5 * f
        assert a <= 1.25 * f + 1e-4
