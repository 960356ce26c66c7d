"""bench.py — BASELINE.json's headline: SDXL + 2 ControlNets + 2 LoRAs (rank
64), 30 DDIM steps, CFG, 1024x1024 (128x128 latent), on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config sdxl|sd15|serve|lora]

--config selects the BASELINE config the line is measured on (default sdxl =
configs[2], the metric's own config; sd15 = configs[1]; serve = configs[4]
folded onto the GPUs given; lora = configs[3], the K1 patch/unpatch
micro-bench).  The default run also carries the config-4 micro-bench, the
patch-overhead arm and the CaaS stall accounting as extra keys, so the
driver's line shows them.

A bench *step* is one image: the full 30-step denoising loop of UNet + the
ControlNets at CFG batch 2, with the request's LoRAs patched by one K1
launch into shadow weights on a low-priority side stream and swapped in at
the planned boundary (async LoRA, schedule.plan_lora_patch).  Weights are
synthetic random-init of the SDXL architecture; inputs are synthetic.

value   images/s over the whole job, inputs already resident in HBM
e2e     the same through the public API (AddonPipeline.generate): pinned host
        inputs -> H2D -> denoise -> D2H of the final latent, every image
roofline K1 (the LoRA patch kernel, north_star's >=70%-of-HBM target): algorithmic
        bytes per launch / its CUDA-event duration on the patch stream inside
        the timed region (it runs concurrently with the UNet there); the
        isolated launch is reported beside it
N > 1   one process per GPU (torchrun, NCCL): ControlNet-as-a-service groups
        (1 base + 1 GPU per ControlNet, caas.py); leftover ranks serve whole
        images alone; scaling is weak; timing is the max over ranks of
        CUDA-event time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "p50 s/image & images/s, SDXL+2 ControlNet+2 LoRA, 1/2/4/8 B200 vs CPU ref"
DENOISE_STEPS = 30
LORA_SCALE = 0.7

# BASELINE.json configs as bench workloads
CONFIGS = {
    "sdxl": dict(cfg="sdxl", n_cn=2, cn_scales=(0.8, 0.6), lora_ranks=(64, 64), batch=1, metric=METRIC,
                 workload="SDXL 1024^2 (128x128 latent) + 2 ControlNets + 2 LoRAs r64 (stacked R=128), "
                          "30 DDIM steps, CFG batch 2, async LoRA patch",
                 model="sdxl-shaped UNet (2.57B) + 2 ControlNets (1.25B each), random init"),
    "sd15": dict(cfg="sd15", n_cn=1, cn_scales=(0.8,), lora_ranks=(16,), batch=1,
                 metric="p50 s/image & images/s, SD1.5 512^2 + 1 ControlNet + 1 LoRA r16, 1 B200 (config 2)",
                 workload="SD1.5 512^2 (64x64 latent) + 1 ControlNet + 1 LoRA r16, 30 DDIM steps, CFG batch 2, "
                          "async LoRA patch",
                 model="sd1.5-shaped UNet (0.86B) + 1 ControlNet, random init"),
    "serve": dict(cfg="sdxl", n_cn=3, cn_scales=(0.8, 0.6, 0.5), lora_ranks=(64, 64), batch=8,
                  metric="images/s & p50/p99 s/batch, SDXL serving batch 8 + 3 ControlNets + 2 LoRAs (config 5)",
                  workload="SDXL 1024^2 serving batch of 8 images per step (CFG batch 16, one shared LoRA set) + "
                           "3 ControlNets + 2 LoRAs r64, 30 DDIM steps",
                  model="sdxl-shaped UNet (2.57B) + 3 ControlNets (1.25B each), random init"),
}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if os.environ.get("SDB_SHARE_ONE_GPU") == "1":
            # test harness only: every rank on cuda:0 over gloo (device buffers
            # staged through host memory by caas.CaaSProtocol) — exercises the
            # multi-GPU control path on a 1-GPU box; numbers are meaningless
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier_sync(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _red_device() -> str:
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else "cuda"


# ---------------------------------------------------------------------------
def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"), default=0)
    except Exception:  # noqa: BLE001
        return 0


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """The reference CPU path on the host cores (oracle/cpu_bench.py: the
    builder's fp32 torch restatement of the denoising step — the reference
    has none — plus the reference's own numpy LoRA merge, addonsim from
    baseline/_ref when installed).  Every bench step is one bounded sample =
    1/(2 * 30) of an image; warm-up samples as asked; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.cpu_bench import CpuWorkload
    from paper_2407_02031_b200 import unet as U
    c = CONFIGS.get(args.config, CONFIGS["sdxl"])
    wl = CpuWorkload(U.CONFIGS[c["cfg"]], c["n_cn"], sum(c["lora_ranks"]), DENOISE_STEPS)
    for _ in range(args.warmup):
        wl.sample()
    t0 = time.perf_counter()
    samples = [wl.sample() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    sample_s = [x["sample_s"] for x in samples]
    ms_per_step = 1000.0 * wall / args.steps
    value = wl.images_per_s(wall / args.steps)          # whole-run throughput: units / time
    cores = torch_threads()
    line = {
        "impl": "reference", "metric": c["metric"], "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "p50_s_per_image": wl.fraction * statistics.median(sample_s),
        "config": {"workload": c["workload"] + " — CPU, one bounded sample per step (see cpu_baseline.sample)",
                   "model": c["model"], "global_batch": 1, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "merge_kind": wl.merge.kind, "blas_threads": blas_threads(), "cpu_model": cpu_model(),
                         "sample": wl.describe()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "samples_s": [round(x, 3) for x in sample_s],
        "merge_s": [round(x["merge_s"], 3) for x in samples],
    }
    print(json.dumps(line), flush=True)


def torch_threads():
    import torch
    return torch.get_num_threads()


def cpu_baseline_leg(c: dict) -> dict:
    """Bounded CPU sample on rank 0 at N=1 (two samples, ~15 s)."""
    from oracle.cpu_bench import CpuWorkload
    from paper_2407_02031_b200 import unet as U
    wl = CpuWorkload(U.CONFIGS[c["cfg"]], c["n_cn"], sum(c["lora_ranks"]), DENOISE_STEPS)
    wl.sample()                                  # warm-up (allocator, thread pool)
    x = wl.sample()
    return {"value": wl.images_per_s(x["sample_s"]), "unit": "images/s", "cores": torch_threads(), "kind": "port",
            "merge_kind": wl.merge.kind, "blas_threads": blas_threads(), "cpu_model": cpu_model(),
            "sample": wl.describe(), "sample_s": round(x["sample_s"], 2),
            "s_per_image_est": round(wl.fraction * x["sample_s"], 1)}


# ---------------------------------------------------------------------------
def _inputs(req):
    import torch
    dev = dict(latent=torch.from_numpy(req.latent).cuda(), context=torch.from_numpy(req.context).cuda(),
               images=[torch.from_numpy(i).cuda() for i in req.images])
    if req.pooled is not None:
        dev["pooled"] = torch.from_numpy(req.pooled).cuda()
        dev["time_ids"] = torch.from_numpy(req.time_ids).cuda()
    pinned = {k: (v.cpu().pin_memory() if not isinstance(v, list) else [x.cpu().pin_memory() for x in v])
              for k, v in dev.items()}
    return dev, pinned


def gpu_minute_accounting(images: int, wall_ms: float, busy_ms: float, n_gpus: int) -> dict:
    """orchestrator.py:768-782 ``throughput``: images over the GPU time
    consumed, in minutes — busy time of every GPU, service GPUs included —
    beside the allocation form (every GPU charged for the whole run)."""
    return {"images_per_gpu_minute": images / (busy_ms / 60_000.0) if busy_ms > 0 else None,
            "images_per_gpu_minute_allocated": images / (n_gpus * wall_ms / 60_000.0),
            "gpu_busy_ms": busy_ms, "wall_ms": wall_ms, "n_gpus": n_gpus}


def run_caas(args, world, rank, local):
    """N > 1: ControlNet-as-a-service groups (caas.py) — base GPU + one GPU per
    ControlNet; leftover ranks serve whole images alone."""
    import torch
    import torch.distributed as dist
    from paper_2407_02031_b200 import ops
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.caas import CaaSNode, StepTimeline, caas_layout
    from paper_2407_02031_b200.patcher import synthetic_lora
    from paper_2407_02031_b200.pipeline import synthetic_batch

    c = CONFIGS[args.config]
    cfg, n_cn = U.CONFIGS[c["cfg"]], c["n_cn"]
    B = args.batch or c["batch"]
    layout = caas_layout(world, n_cn)
    node = CaaSNode(cfg, layout, rank, list(c["cn_scales"]), steps=DENOISE_STEPS, guidance=7.5,
                    dtype=torch.bfloat16, seed=0, batch=B)
    role = node.role
    if role in ("base", "solo"):
        node.load_loras([(synthetic_lora(node.pipe.unet_p, r, seed=10 + i, adapter_id=f"lora{i}"), LORA_SCALE)
                         for i, r in enumerate(c["lora_ranks"])])
    node.setup()
    req = synthetic_batch(cfg, n_cn, B, seed=rank)
    dev_in, pinned = _inputs(req)
    producer = role in ("base", "solo")
    p = node.pipe if producer else None

    def image(inputs, patch=True, timeline=None):
        if producer:
            node.prepare(**inputs)
        else:
            node.prepare()
        if producer:
            node.denoise(patch=patch, timeline=timeline)
        else:
            node.denoise(timeline=timeline)

    s = torch.cuda.current_stream()
    # calibrate the patch plan on the base: one unpatched image, one isolated patch
    if producer:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
    image(dev_in, patch=False)
    if producer:
        b.record()
        b.synchronize()
        p.step_ms_est = a.elapsed_time(b) / DENOISE_STEPS
        c0_, d0_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0_.record(p.patch_stream)
        p.patchset.launch(stream=p.patch_stream)
        d0_.record(p.patch_stream)
        d0_.synchronize()
        p.patch_ms_est = c0_.elapsed_time(d0_)
    for _ in range(args.warmup):
        image(dev_in)
    barrier_sync(world)
    clocks = ClockSampler(local)
    clocks.start()
    c0 = ops.LAUNCHES["count"]
    evs = []
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(s)
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        image(dev_in)
        b.record(s)
        evs.append((a, b))
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record(s)
    barrier_sync(world)
    host_launches = ops.LAUNCHES["count"] - c0
    total_ms = max_over_ranks(t0.elapsed_time(t1), world)
    per_image = [a.elapsed_time(b) / 1000.0 for a, b in evs] if producer else []
    # e2e: pinned host inputs -> H2D -> denoise -> D2H of the latent, every image
    barrier_sync(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.steps):
        image(pinned)
        if producer:
            node.latent_nchw().contiguous().cpu()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(s)
    barrier_sync(world)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    clk = clocks.stop()
    # per-step accounting (one more image, events on every rank): the base's
    # decoder wait split like orchestrator.py:662-678, service compute per step
    tl = StepTimeline()
    barrier_sync(world)
    image(dev_in, timeline=tl)
    barrier_sync(world)
    mine_tl = tl.summary()
    red = torch.tensor([mine_tl.get("step_ms", 0.0) if role == "service" else 0.0,
                        1.0 if role == "service" else 0.0], device=_red_device(), dtype=torch.float64)
    dist.all_reduce(red, op=dist.ReduceOp.SUM)
    svc_ms = float(red[0].item() / red[1].item()) if red[1].item() > 0 else 0.0
    # the base's decoder wait, split with the services' measured step (compute + push)
    summ = tl.summary(branch_ms=svc_ms) if role == "base" else mine_tl
    producers = len(layout.groups)
    images = args.steps * producers * B
    lat = torch.tensor([statistics.median(per_image) if (role == "base" or (role == "solo" and
                        all(not g.services for g in layout.groups))) else 0.0], device=_red_device(),
                       dtype=torch.float64)
    dist.all_reduce(lat, op=dist.ReduceOp.MAX)
    # this repo's kernels launched in the timed region, summed over ranks:
    # host-issued launches + every graph replay's captured launches
    mine = host_launches + node.launches_per_step * DENOISE_STEPS * args.steps
    tot = torch.tensor([float(mine)], device=_red_device(), dtype=torch.float64)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    hbm, _, src = peaks()
    line = None
    if rank == 0:
        alg = p.patchset.alg_bytes
        n_svc_gpus = sum(len(g.services) for g in layout.groups)
        busy = total_ms * producers + svc_ms * DENOISE_STEPS * args.steps * n_svc_gpus
        line = {
            "metric": c["metric"], "value": images / (total_ms / 1000.0), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "p50_s_per_image": float(lat.item()),
            "config": {"workload": c["workload"], "model": c["model"],
                       "global_batch": producers * B, "seq_len": None,
                       "parallelism": "ControlNet-as-a-service groups " +
                                      "; ".join(str(g.ranks) for g in layout.groups),
                       "l2": "inputs larger than L2 (weights re-read every step)"},
            "e2e": {"value": images / (e2e_ms / 1000.0), "unit": "images/s",
                    "h2d_bytes_per_step": req.nbytes(), "d2h_bytes_per_step": 4 * node.L},
            "gpu_launches": int(tot.item()),
            "roofline": {"kernel": f"sdb lora_patch (K1, stacked R={sum(c['lora_ranks'])}, all UNet matrices)",
                         "bound": "hbm", "achieved": alg / (p.patch_ms_est * 1e-3) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": alg / (p.patch_ms_est * 1e-3) / 1e9 / hbm, "traffic": k1_traffic(),
                         "alg_bytes_per_launch": alg, "launch_ms_isolated": p.patch_ms_est,
                         "peak_source": src},
            "clocks": clk,
            "caas_accounting": {"base": summ, "service_step_ms": svc_ms,
                                **gpu_minute_accounting(images, total_ms, busy, world)},
            "detail": {"layout": [list(g.ranks) for g in layout.groups],
                       "first_patched_step": p.last_first_patched_step, "step_ms_est": p.step_ms_est},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def k1_traffic():
    """DRAM bytes (read + write) of one K1 launch of this workload, from the
    committed `ncu --set full` capture (profiles/k1_traffic.json)."""
    p = ROOT / "profiles" / "k1_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d["dram_bytes_read"] + d["dram_bytes_write"]


def other_kernels_roofline(hbm: float) -> list:
    """The step's HBM-bound kernels at their largest SDXL shapes (CFG batch 2).

    Each kernel is captured REPS times into one CUDA graph, every launch on
    its own copy of the inputs (ROT copies, > 126 MB in total, so each launch
    finds its inputs outside L2 — what the UNet's freshly evicted activations
    look like), and timed as graph replays with CUDA events: device time per
    launch without host launch overhead.  Algorithmic bytes: one read of every
    input + one write of every output (K2's second read of x, served from L2,
    is not counted)."""
    import torch
    from paper_2407_02031_b200 import ops
    dev = "cuda"
    cl = torch.channels_last
    L2 = 126 << 20

    def timed(make, nbytes_in, reps=24):
        rot = max(2, -(-2 * L2 // max(nbytes_in, 1)))           # copies spanning > 2x L2
        rot = min(rot, reps)
        bufs = [make() for _ in range(rot)]                      # each: a zero-arg launch closure
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for f in bufs:
                f()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps):
                bufs[i % rot]()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            g.replay()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / (3 * reps)
        del g, bufs
        torch.cuda.empty_cache()
        return ms

    out = []
    g, bta = torch.ones(320, device=dev), torch.zeros(320, device=dev)

    def mk_gn(mode):
        def make():
            x = torch.randn(2, 320, 128, 128, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
            add = torch.zeros(2, 320, device=dev)
            ws = ops.groupnorm_workspace(x)
            y = torch.empty_like(x)

            def f():
                with ops.groupnorm_mode(mode):
                    ops.groupnorm_silu(x, g, bta, out=y, add_nc=add, workspace=ws)
            return f
        return make
    n_gn = 2 * 320 * 128 * 128
    out.append(("K2 groupnorm+silu (+temb) [2,320,128,128] bf16, resident form (the shipped choice: one cooperative "
                "launch, tiles resident in shared memory, one grid barrier; the 9 two-pass sites at 128x128 per "
                "SDXL step incl. ControlNets)", 2 * n_gn * 2, timed(mk_gn(0), n_gn * 2)))
    out.append(("K2 groupnorm+silu (+temb) [2,320,128,128] bf16, two-pass form (stats + apply; round 1's choice)",
                2 * n_gn * 2, timed(mk_gn(1), n_gn * 2)))

    g6, b6 = torch.ones(640, device=dev), torch.zeros(640, device=dev)

    def mk_gn64(mode):
        def make():
            x = torch.randn(2, 640, 64, 64, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
            add = torch.zeros(2, 640, device=dev)
            ws = ops.groupnorm_workspace(x)
            y = torch.empty_like(x)

            def f():
                with ops.groupnorm_mode(mode):
                    ops.groupnorm_silu(x, g6, b6, out=y, add_nc=add, workspace=ws)
            return f
        return make
    n_64 = 2 * 640 * 64 * 64
    out.append(("K2 groupnorm+silu (+temb) [2,640,64,64] bf16, resident form (the shipped choice at the 9 two-pass "
                "sites at 64x64 per SDXL step)", 2 * n_64 * 2, timed(mk_gn64(0), n_64 * 2)))
    out.append(("K2 groupnorm+silu (+temb) [2,640,64,64] bf16, streamed cluster form (one launch, one read, "
                "one write; the choice before the resident form)", 2 * n_64 * 2, timed(mk_gn64(3), n_64 * 2)))
    out.append(("K2 groupnorm+silu (+temb) [2,640,64,64] bf16, two-pass form (round 1's choice at this site)",
                2 * n_64 * 2, timed(mk_gn64(1), n_64 * 2)))

    def mk_gn_apply(c):
        def make():
            x = torch.randn(2, c, 128, 128, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
            ws = ops.groupnorm_workspace(x)
            h0 = ops.residual_inject(x, [], [], out=x, gn_workspace=ws)    # K3 publishes the statistics
            y = torch.empty_like(x)
            gg, bb = torch.ones(c, device=dev), torch.zeros(c, device=dev)

            def f():
                h0._sdb_gn = (ws, 32, h0.data_ptr())
                ops.groupnorm_silu(h0, gg, bb, out=y)
            return f
        return make
    for c_ in (320, 640):
        n_c = 2 * c_ * 128 * 128
        out.append((f"K2 groupnorm+silu [2,{c_},128,128] bf16, apply-only (statistics from the producing K3: "
                    f"29 of 46 SDXL sites)", 2 * n_c * 2, timed(mk_gn_apply(c_), n_c * 2)))
    lw, lb = torch.ones(640, device=dev, dtype=torch.bfloat16), torch.zeros(640, device=dev, dtype=torch.bfloat16)

    def mk_ln():
        tok = torch.randn(2, 4096, 640, device=dev).to(torch.bfloat16)
        d = torch.randn_like(tok)
        return lambda: ops.add_layernorm(tok, d, lw, lb)
    n_ln = 2 * 4096 * 640
    out.append(("K6 add+layernorm [2,4096,640] bf16", 4 * n_ln * 2, timed(mk_ln, 2 * n_ln * 2)))

    def mk_geglu():
        proj = torch.randn(2, 4096, 5120, device=dev).to(torch.bfloat16)
        return lambda: ops.geglu(proj)
    n_pj = 2 * 4096 * 5120
    out.append(("K5 geglu [2,4096,5120]->[...,2560] bf16", n_pj * 2 * 3 // 2, timed(mk_geglu, n_pj * 2)))

    def mk_inject():
        hid = torch.randn(2, 640, 128, 128, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        skip = torch.randn(2, 320, 128, 128, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        res = [torch.randn_like(skip) for _ in range(2)]
        outb = torch.empty((2, 960, 128, 128), device=dev, dtype=torch.bfloat16, memory_format=cl)
        return lambda: ops.residual_inject(skip, res, [0.8, 0.6], hidden=hid, out=outb)
    nh, ns = 2 * 640 * 128 * 128, 2 * 320 * 128 * 128
    out.append(("K3 inject 2 residuals + concat [2,640|320,128,128] bf16", (nh + 3 * ns + nh + ns) * 2,
                timed(mk_inject, (nh + 3 * ns) * 2)))

    def mk_xattn():
        q = torch.randn(2, 4096, 640, device=dev).to(torch.bfloat16)
        kv = torch.randn(2, 77, 1280, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        return lambda: ops.cross_attention(q, kv, 10, out=o)
    nq = 2 * 4096 * 640
    out.append(("K7 cross-attention [2,4096,640] x 77 tokens, 10 heads bf16 (mma.sync form)", 2 * nq * 2,
                timed(mk_xattn, nq * 2)))

    def mk_xattn_tc():
        q = torch.randn(2, 1024, 1280, device=dev).to(torch.bfloat16)
        kv = torch.randn(2, 77, 2560, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        return lambda: ops.cross_attention(q, kv, 20, out=o)
    nq = 2 * 1024 * 1280
    out.append(("K7 cross-attention [2,1024,1280] x 77 tokens, 20 heads bf16 (tcgen05 form)", 2 * nq * 2,
                timed(mk_xattn_tc, nq * 2)))

    def mk_xattn_srv():
        q = torch.randn(16, 1024, 1280, device=dev).to(torch.bfloat16)
        kv = torch.randn(16, 77, 2560, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        return lambda: ops.cross_attention(q, kv, 20, out=o)
    nq = 16 * 1024 * 1280
    out.append(("K7 cross-attention [16,1024,1280] x 77 tokens, 20 heads bf16 (config 5's CFG batch 16: persistent "
                "tcgen05 form)", 2 * nq * 2 + 16 * 77 * 2560 * 2, timed(mk_xattn_srv, nq * 2)))
    res = [{"kernel": k, "bound": "hbm", "achieved": b / (m * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": b / (m * 1e-3) / 1e9 / hbm, "alg_bytes": b, "launch_ms": m,
            "method": "CUDA-graph replay, inputs rotated over > 2x L2"} for k, b, m in out]

    # K5': the FF projection GEMM with GEGLU in its tcgen05 epilogue — tensor-bound
    tpk = _tensor_peak_burst()
    for m_, k_, f_ in ((8192, 640, 2560), (2048, 1280, 5120)):
        wf = (torch.randn(2 * f_, k_, device=dev) * 0.03).to(torch.bfloat16)
        bff = torch.randn(2 * f_, device=dev)

        def mk_ff(m_=m_, k_=k_, wf=wf, bff=bff):
            xf = torch.randn(m_, k_, device=dev).to(torch.bfloat16)
            return lambda: ops.ff_geglu(xf, wf, bff)
        ms = timed(mk_ff, m_ * 2 * f_ * 2)
        flops = 2 * m_ * k_ * 2 * f_
        res.append({"kernel": f"K5' FF GEMM + GEGLU epilogue [{m_},{k_}]x{2 * f_} bf16 (tcgen05, CTA pairs)",
                    "bound": "tensor", "achieved": flops / (ms * 1e-3) / 1e12, "peak": tpk, "unit": "TFLOP/s",
                    "frac": flops / (ms * 1e-3) / 1e12 / tpk, "alg_flops": flops, "launch_ms": ms,
                    "method": "CUDA-graph replay, activations rotated over > 2x L2; peak = measured bf16 burst"})
    return res


def _tensor_peak_burst() -> float:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["bf16_tflops"])
    return 1637.0


def blocking_preamble(pipe) -> dict:
    """The Diffusers-style baseline the async path replaces
    (orchestrator.py:555-571 `_blocking_lora_preamble`; lora.py:132-144
    create-and-replace): fetch every LoRA, build new weight copies and merge
    into them, all before step 1 — measured on this GPU (device events per
    stage, host wall for the whole, untimed by the headline)."""
    import torch
    from paper_2407_02031_b200.patcher import PatchSet
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(s)
    pipe.bank.fetch(s)                                                      # every LoRA, H2D
    ev[1].record(s)
    copy = {n: pipe.unet_p.t[n + ".weight"].clone() for n, _ in pipe.unet_p.matrices}   # create
    ev[2].record(s)
    ps = PatchSet(pipe.unet_p, pipe.bank.adapters, shadow=copy)             # replace: merge into the copy
    ps.launch(stream=s)
    ev[3].record(s)
    ev[3].synchronize()
    wall = (time.perf_counter() - t0) * 1000.0
    out = {"h2d_fetch_ms": ev[0].elapsed_time(ev[1]), "copy_weights_ms": ev[1].elapsed_time(ev[2]),
           "plan_and_patch_ms": ev[2].elapsed_time(ev[3]), "total_wall_ms": wall,
           "note": "blocking preamble (fetch + create-and-replace before step 1); the headline hides its "
                   "async equivalent behind step 1"}
    del copy, ps
    torch.cuda.empty_cache()
    return out


def lora_microbench(unet_p, shadow, hbm: float, cpu_full: bool = False, reps: int = 5) -> dict:
    """BASELINE config 4: K1 over every patchable SDXL matrix with 4 LoRAs at
    ranks 8/32/64/128 (stacked R = 232) and four distinct scales, bf16 weights.
    Extends the reference's ``bench_merge`` keys (lora.py:163-199): patch
    (out of place into the serving copy, and in place = merge_in_place),
    unpatch (sign -1 in place = unmerge_in_place; restore from pristine; the
    serving path's pointer swap), each as the median of ``reps`` CUDA-event
    timed launches, with algorithmic GB/s and the fraction of the measured
    HBM peak.  Beside it, the reference's own numpy ``merge_in_place`` (or
    its restatement) on the host cores, BLAS at 1 thread and at all threads."""
    import torch
    from paper_2407_02031_b200.patcher import PatchSet, synthetic_lora
    ranks, scales = (8, 32, 64, 128), (0.9, 0.55, 0.35, 1.3)
    ads = [(synthetic_lora(unet_p, r, seed=40 + i, adapter_id=f"cfg4_{i}"), sc)
           for i, (r, sc) in enumerate(zip(ranks, scales))]
    out_of_place = PatchSet(unet_p, ads, shadow=shadow)
    in_place = PatchSet(unet_p, ads, shadow=shadow, in_place_on_shadow=True)
    from paper_2407_02031_b200.ops import BatchedCopy
    names = [n for n, _ in unet_p.matrices if n not in unet_p.fused]
    # fused storages (q|k|v, k|v) are restored as one block each
    parents = list(unet_p.fused)
    members = {m for ms in unet_p.fused.values() for m in ms}
    names = [n for n in names if n not in members] + parents
    pristine = [unet_p.t[n + ".weight"] for n in names]
    dst = [shadow[n] for n in names]
    restore = BatchedCopy(pristine, dst)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    alg = out_of_place.alg_bytes
    w_bytes = restore.nbytes
    res = {}
    res["patch_out_of_place_ms"] = timed(lambda: out_of_place.launch())
    restore.launch()
    res["merge_in_place_ms"] = timed(lambda: in_place.launch(sign=1.0))
    res["unmerge_in_place_ms"] = timed(lambda: in_place.launch(sign=-1.0))
    res["restore_from_pristine_ms"] = timed(lambda: restore.launch())     # sdb_batched_copy, one launch
    res["pointer_swap_ms"] = 0.0
    out = {"layers": len(unet_p.matrices), "restore_tensors": len(names), "ranks": list(ranks),
           "scales": list(scales), "stacked_rank": sum(ranks),
           "kernel": out_of_place.plan.kernel, "alg_bytes_patch": alg, "alg_bytes_restore": 2 * w_bytes,
           "in_place_nbytes": w_bytes, "create_and_replace_nbytes": 2 * w_bytes + sum(
               a.nbytes for a, _ in ads), **{k: round(v, 4) for k, v in res.items()}}
    for k in ("patch_out_of_place", "merge_in_place", "unmerge_in_place"):
        gbs = alg / (res[k + "_ms"] * 1e-3) / 1e9
        out[k + "_gbs"], out[k + "_frac"] = round(gbs, 1), round(gbs / hbm, 4)
    gbs = 2 * w_bytes / (res["restore_from_pristine_ms"] * 1e-3) / 1e9
    out["restore_from_pristine_gbs"], out["restore_from_pristine_frac"] = round(gbs, 1), round(gbs / hbm, 4)
    out["peak_gbs"] = hbm
    del out_of_place, in_place, ads
    torch.cuda.empty_cache()
    mats = [unet_p.matrix_view(n) for n, _ in unet_p.matrices]
    out["cpu_reference"] = cpu_merge_leg([tuple(m.shape) for m in mats], sum(ranks), full=cpu_full)
    return out


def cpu_merge_leg(shapes, rank: int, full: bool) -> dict:
    """The reference numpy merge on the host cores (addonsim.lora.merge_in_place
    from baseline/_ref, else the bit-exact restatement), fp32 weights, over the
    whole inventory (full) or a size-stratified 1/10 slice scaled up."""
    from oracle.cpu_bench import MergeTimer, stratified
    den = 1 if full else 10
    sl = stratified(shapes, lambda s: s[0] * s[1], den)
    total = sum(a * b for a, b in shapes)
    mt = MergeTimer(sl, rank)
    out = {"kind": mt.kind, "rank": rank, "matrices_timed": len(sl), "matrices_total": len(shapes),
           "cpu_model": cpu_model(), "cores": os.cpu_count()}
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # noqa: BLE001
        threadpool_limits = None
    for label, n in (("blas_1_thread", 1), ("blas_all_threads", os.cpu_count())):
        if threadpool_limits is not None:
            with threadpool_limits(limits=n, user_api="blas"):
                t = mt.run()
        else:
            t = mt.run()
        s_full = t * total / mt.elements
        out[label] = {"s_inventory": round(s_full, 2), "gbs_fp32": round(8 * total / s_full / 1e9, 3),
                      "threads": n}
    return out


def parity_leg(eng, c: dict, dev_in: dict, req) -> dict:
    """The benchmarked engine's step-1 latent (bf16, one more image with the
    patch forced at boundary 1, so step 1 runs the pristine weights) against
    the CPU fp32 oracle's step 1 on the same parameter values and inputs
    (oracle/pipeline_ref.py, the checker).  The bf16 floor — the oracle with
    bf16 activations vs fp32 — is measured by tests/test_sdxl_engine_gpu.py."""
    import torch
    from oracle import pipeline_ref as R
    from paper_2407_02031_b200 import unet as U
    cfg = U.CONFIGS[c["cfg"]]
    got = []
    eng.prepare(**dev_in)
    eng.denoise(patch=True, boundary=1, on_step=lambda k, x: got.append(x.float().cpu()) if k == 1 else None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe = eng.base.pipe
    up = R.to_cpu_params(pipe.unet_p)
    cps = []
    for i in range(c["n_cn"]):
        p = U.init_controlnet(cfg, "cuda", torch.bfloat16, seed=1000 + i)   # unscaled (services fold the scale)
        cps.append(R.to_cpu_params(p))
        del p
    torch.cuda.empty_cache()
    ref = R.denoise(cfg, up, cps, req, list(c["cn_scales"]), DENOISE_STEPS, 7.5, max_steps=1)[0]
    rel = float((got[0].double() - ref.double()).norm() / ref.double().norm())
    return {"step": 1, "rel_l2_vs_fp32_oracle": rel, "dtype": "bf16", "oracle": "oracle/pipeline_ref.py fp32 CPU",
            "oracle_s": round(time.perf_counter() - t0, 1),
            "note": "bf16-activation floor at this config: tests/test_sdxl_engine_gpu.py "
                    "(profiles/r02_sdxl_parity.txt)"}


def run_ours(args):
    import torch
    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if args.config == "lora":
        return run_lora(args)
    if world > 1:
        return run_caas(args, world, rank, local)
    from paper_2407_02031_b200 import ops
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.caas import LoopbackGroup, StepTimeline
    from paper_2407_02031_b200.patcher import synthetic_lora
    from paper_2407_02031_b200.pipeline import AddonPipeline, synthetic_batch

    c = CONFIGS[args.config]
    cfg, n_cn, scales = U.CONFIGS[c["cfg"]], c["n_cn"], list(c["cn_scales"])
    B = args.batch or c["batch"]
    req = synthetic_batch(cfg, n_cn, B, seed=rank)
    dev_in, pinned = _inputs(req)
    if args.mode == "serial":
        # ControlNets inline (orchestrator.py:611-619), one CUDA graph per step
        eng = AddonPipeline(cfg, n_controlnets=n_cn, cn_scales=scales, steps=DENOISE_STEPS, guidance=7.5,
                            dtype=torch.bfloat16, seed=0, patch_max_ctas=args.patch_ctas, batch=B)
        pipe = eng
    else:
        # ControlNet branches on their own streams beside the UNet encoder (CaaS split on one GPU)
        eng = LoopbackGroup(cfg, n_cn, scales, steps=DENOISE_STEPS, guidance=7.5, dtype=torch.bfloat16,
                            seed=0, concurrent=True, batch=B)
        pipe = eng.base.pipe
        pipe.patch_max_ctas = args.patch_ctas
    loras = [(synthetic_lora(pipe.unet_p, r, seed=10 + i, adapter_id=f"lora{i}"), LORA_SCALE) for i, r in
             enumerate(c["lora_ranks"])]
    # the LoRAs live in pinned host memory (the LoRA cache tier); the e2e loop
    # re-fetches them every image (H2D on the copy stream, re-pack, patch), the
    # resident loop finds them in HBM and only patches
    eng.load_loras(loras, host_resident=True)
    eng.setup()
    if args.mode == "serial":
        step_ms, patch_ms = pipe.calibrate(reps=3)
        s = pipe.main_stream
    else:
        s = eng.main_stream
        with torch.cuda.stream(s):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            eng.prepare(**dev_in)
            a.record(s)
            eng.denoise(patch=False)
            b.record(s)
            b.synchronize()
            pipe.step_ms_est = step_ms = a.elapsed_time(b) / DENOISE_STEPS
            c0_, d0_ = pipe.launch_patch(timing=True, fetch=True)   # the plan's load: fetch + pack + patch
            d0_.synchronize()
            pipe.patch_ms_est = patch_ms = c0_.elapsed_time(d0_)
    lora_h2d = pipe.bank.nbytes

    def image_resident(patch=True):
        eng.prepare(**dev_in)
        eng.denoise(patch=patch, fetch=False)

    def image_e2e():
        # the public call: pinned host inputs (+ the LoRAs) -> H2D -> denoise -> D2H of the final latent
        eng.prepare(**pinned)
        eng.denoise(patch=True, fetch=True)
        eng.latent_nchw().contiguous().cpu()

    with torch.cuda.stream(s):
        for _ in range(args.warmup):
            image_resident()
        image_e2e()
    barrier_sync(world)

    def timed_images(fn, n):
        evs = []
        with torch.cuda.stream(s):
            t_a = torch.cuda.Event(enable_timing=True)
            t_a.record(s)
            for _ in range(n):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                fn()
                b.record(s)
                evs.append((a, b))
            t_b = torch.cuda.Event(enable_timing=True)
            t_b.record(s)
        barrier_sync(world)
        return t_a.elapsed_time(t_b), [a.elapsed_time(b) / 1000.0 for a, b in evs]

    # ---- timed: device-resident inputs ------------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    pipe.patch_timing = []
    c0 = ops.LAUNCHES["count"]
    barrier_sync(world)
    total_ms, per_image = timed_images(image_resident, args.steps)
    host_launches = ops.LAUNCHES["count"] - c0
    total_ms = max_over_ranks(total_ms, world)
    patch_ms_live = [p0.elapsed_time(p1) for p0, p1 in pipe.patch_timing]
    pipe.patch_timing = None

    # ---- timed: end to end through the public API (host buffers) ----------
    barrier_sync(world)
    e2e_ms, _ = timed_images(image_e2e, args.steps)
    e2e_ms = max_over_ranks(e2e_ms, world)
    clk = clocks.stop()

    # ---- the same loop without the LoRA: is the patch hidden? ------------
    plain_ms, per_plain = timed_images(lambda: image_resident(patch=False), args.steps)
    overhead = {"patched_mean_s": statistics.mean(per_image), "unpatched_mean_s": statistics.mean(per_plain),
                "patched_p50_s": statistics.median(per_image), "unpatched_p50_s": statistics.median(per_plain),
                "patch_overhead_ms_per_image": 1000.0 * (statistics.mean(per_image) - statistics.mean(per_plain)),
                "note": "identical image loops (resident inputs) with and without the async LoRA patch, "
                        "back to back in this run (PAPER.md:519-521; orchestrator.py:698-719)"}
    overhead["patch_overhead_pct"] = 100.0 * overhead["patch_overhead_ms_per_image"] / (
        1000.0 * overhead["unpatched_mean_s"])

    # ---- CaaS per-step accounting (orchestrator.py:621-678, 768-782) ------
    accounting = None
    if args.mode == "branch":
        tl = StepTimeline()
        with torch.cuda.stream(s):
            eng.prepare(**dev_in)
            eng.denoise(patch=True, fetch=False, timeline=tl)
        torch.cuda.synchronize()
        accounting = {"per_step": tl.summary(comm_ms=0.0),
                      "note": "1 GPU: ControlNet branches on side streams beside the encoder, residual buffers "
                              "aliased (no transfer, comm 0); decoder wait split comm -> ControlNet compute -> "
                              "fetch -> queue as orchestrator.py:662-678",
                      **gpu_minute_accounting(args.steps * B, total_ms, total_ms, 1)}

    # ---- K1 isolated (for the roofline's context) --------------------------
    iso = []
    with torch.cuda.stream(pipe.patch_stream):
        for _ in range(3):
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(pipe.patch_stream)
            pipe.patchset.launch(stream=pipe.patch_stream)
            p1.record(pipe.patch_stream)
            p1.synchronize()
            iso.append(p0.elapsed_time(p1))
    torch.cuda.synchronize()

    # kernels issued in the timed region: graph replays issue what the capture counted
    graph_launches_per_step = pipe.launches_per_step if args.mode == "serial" else \
        sum(n.launches_per_step for n in eng.nodes)
    gpu_launches = host_launches + graph_launches_per_step * DENOISE_STEPS * args.steps

    hbm, tflops, src = peaks()
    alg = pipe.patchset.alg_bytes
    live = statistics.mean(patch_ms_live) if patch_ms_live else None
    achieved = alg / (live * 1e-3) / 1e9 if live else None
    images = args.steps * world * B
    value = images / (total_ms / 1000.0)
    R = sum(c["lora_ranks"])
    line = {
        "metric": c["metric"], "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "p50_s_per_image": statistics.median(per_image),
        "config": {"workload": c["workload"] + (f"; serving batch of {B} images per step (CFG batch {2 * B}, "
                                                f"one LoRA set)" if B > 1 else ""),
                   "model": c["model"], "global_batch": world * B, "seq_len": None,
                   "parallelism": ("1 GPU, ControlNet branches on side streams concurrent with the UNet encoder"
                                   if args.mode == "branch" else "1 GPU, ControlNets inline"),
                   "l2": "inputs larger than L2 (UNet + ControlNet weights, GBs, re-read every step)"},
        "e2e": {"value": images / (e2e_ms / 1000.0), "unit": "images/s",
                "h2d_bytes_per_step": req.nbytes() + lora_h2d, "d2h_bytes_per_step": pipe.d2h_bytes(),
                "note": "inputs + the LoRAs fetched from pinned host memory every image"},
        "gpu_launches": int(gpu_launches),
        "roofline": {"kernel": f"sdb lora_patch (K1, stacked R={R}, all {len(pipe.unet_p.matrices)} UNet matrices)",
                     "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm if achieved else None,
                     "traffic": k1_traffic() if args.config == "sdxl" else None,
                     "alg_bytes_per_launch": alg, "launch_ms_live": live,
                     "launch_ms_isolated": statistics.median(iso),
                     "frac_isolated": alg / (statistics.median(iso) * 1e-3) / 1e9 / hbm,
                     "peak_source": f"{src} MEASURED_PEAKS.json hbm_gbs" if src == "measured" else src},
        "clocks": clk,
        "detail": {"step_ms_calibrated": step_ms, "first_patched_step": pipe.last_first_patched_step,
                   "patch_path": pipe.patchset.plan.path, "per_image_s": [round(x, 4) for x in per_image],
                   "patch_overhead": overhead,
                   "programmatic_dependent_launch": os.environ.get("SDB_PDL", "1") != "0"},
    }
    if accounting is not None:
        line["caas_accounting"] = accounting
    if B > 1:   # every image of a batch completes with the batch: its latency is the batch time
        line["p50_s_per_batch"] = statistics.median(per_image)
        line["p99_s_per_batch"] = sorted(per_image)[min(len(per_image) - 1, int(0.99 * len(per_image)))]
        line["detail"]["per_batch_s"] = line["detail"].pop("per_image_s")
    line["roofline_other_kernels"] = other_kernels_roofline(hbm)
    if args.config == "sdxl" and args.mode == "branch":
        try:   # BASELINE config 4 (K1 patch / unpatch micro-bench) on the engine's own weights
            line["lora_microbench"] = lora_microbench(pipe.unet_p, pipe.shadow, hbm)
        except Exception as e:  # noqa: BLE001 — a side measurement must not sink the bench line
            line["lora_microbench"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    try:
        line["detail"]["blocking_lora_preamble"] = blocking_preamble(pipe)
    except Exception as e:  # noqa: BLE001
        line["detail"]["blocking_lora_preamble"] = {"error": f"{type(e).__name__}: {e}"[:200]}
    if rank == 0 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline_leg(c)
        except Exception as exc:  # reported, never silently dropped
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
        if args.mode == "branch" and B == 1:
            try:
                with torch.cuda.stream(s):
                    line["parity"] = parity_leg(eng, c, dev_in, req)
            except Exception as exc:  # noqa: BLE001
                line["parity"] = {"error": repr(exc)[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_lora(args):
    """--config lora: BASELINE config 4 alone — the K1 patch / unpatch
    micro-bench over every SDXL matrix (R = 232, four scales), timed K times
    after W warm-ups; the reference numpy merge over the FULL inventory."""
    import torch
    from paper_2407_02031_b200 import ops
    from paper_2407_02031_b200 import unet as U
    from paper_2407_02031_b200.patcher import allocate_shadow
    hbm, _, src = peaks()
    p = U.init_unet(U.SDXL, "cuda", torch.bfloat16, 0)
    shadow = allocate_shadow(p)
    clocks = ClockSampler(0)
    clocks.start()
    c0 = ops.LAUNCHES["count"]
    mb = lora_microbench(p, shadow, hbm, cpu_full=True, reps=max(args.steps, 1))
    clk = clocks.stop()
    n_launch = ops.LAUNCHES["count"] - c0
    ms = mb["patch_out_of_place_ms"]
    line = {
        "metric": "K1 LoRA patch GB/s, all 794 SDXL matrices, 4 LoRAs r8-128 (R=232), bf16 (config 4)",
        "value": mb["patch_out_of_place_gbs"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "K1 over all 794 SDXL UNet matrices (2.57 G elements), 4 LoRAs r 8/32/64/128 at "
                               "scales 0.9/0.55/0.35/1.3, stacked R=232; patch out of place + merge/unmerge in "
                               "place + restore", "model": "sdxl-shaped UNet weights, random init",
                   "global_batch": 1, "parallelism": "1 GPU",
                   "l2": "inputs larger than L2 (5.1 GB of weights per launch)"},
        "e2e": {"value": mb["patch_out_of_place_gbs"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0, "note": "factors resident (the fetch path is in the headline's e2e)"},
        "gpu_launches": int(n_launch),
        "roofline": {"kernel": "sdb lora_patch (K1, R=232)", "bound": "hbm", "achieved": mb["patch_out_of_place_gbs"],
                     "peak": hbm, "unit": "GB/s", "frac": mb["patch_out_of_place_frac"], "traffic": None,
                     "peak_source": src},
        "clocks": clk, "lora_microbench": mb,
        "cpu_baseline": {"value": 8 * 2.566e9 / mb["cpu_reference"]["blas_all_threads"]["s_inventory"] / 1e9,
                         "unit": "GB/s (fp32 weights)", "cores": os.cpu_count(),
                         "kind": mb["cpu_reference"]["kind"],
                         "sample": "the reference numpy merge_in_place over all 794 SDXL matrices, R=232"},
    }
    print(json.dumps(line), flush=True)


def main():
    # a run that outlives ~6 minutes (a normal default run takes ~100 s) dumps
    # every thread's Python stack to stderr, every 6 minutes: a hang leaves a
    # trace of where it sits instead of an empty log
    import faulthandler
    faulthandler.dump_traceback_later(360, repeat=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS) + ["lora"], default="sdxl",
                    help="BASELINE config: sdxl (configs[2], default), sd15 (configs[1]), serve (configs[4]), "
                         "lora (configs[3] micro-bench)")
    ap.add_argument("--patch-ctas", type=int, default=0, help="cap the K1 grid (0 = one CTA per tile)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--batch", type=int, default=0,
                    help="images per denoising batch sharing one LoRA set (0 = the config's: 1, serve 8)")
    ap.add_argument("--mode", choices=["branch", "serial"], default="branch",
                    help="1 GPU: ControlNet branches concurrent with the encoder (branch) or inline (serial)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
