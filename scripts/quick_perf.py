"""Quick B200 timing probe (development aid; the contract numbers come from bench.py).

  python scripts/quick_perf.py lora      # SDXL all-matrix K1 patch at several stacked ranks
  python scripts/quick_perf.py step      # SDXL + 2 CN step time (graph replay)
"""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2407_02031_b200 import unet as U  # noqa: E402
from paper_2407_02031_b200.patcher import PatchSet, allocate_shadow, synthetic_lora  # noqa: E402

PEAK = 6458.1


def time_launch(fn, reps=10):
    for _ in range(2):
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
    ts.sort()
    return ts[len(ts) // 2]


def lora():
    cfg = U.SDXL
    p = U.init_unet(cfg, "cuda", torch.bfloat16, 0)
    shadow = allocate_shadow(p)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = []
    from paper_2407_02031_b200 import ops
    modes = [int(m) for m in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2"])]
    for (ranks, simt), mode in [(x, m) for x in (([8], 0), ([16], 0), ([64], 0), ([64, 64], 0),
                                                 ([8, 32, 64, 128], 0)) for m in modes]:
        ads = [(synthetic_lora(p, r, seed=i, adapter_id=f"a{i}"), 0.5) for i, r in enumerate(ranks)]
        with ops.lora_kernel_mode(mode):
            ps = PatchSet(p, ads, shadow=shadow, simt_max_rank=simt)

        def run():
            flush.zero_()
            ps.launch()
        flush_ms = time_launch(lambda: flush.zero_())
        ms = time_launch(run) - flush_ms
        gbps = ps.alg_bytes / (ms * 1e-3) / 1e9
        out.append({"ranks": ranks, "R": ps.rank, "mode": mode, "path": [pl.path for pl in ps.plans],
                    "ms": round(ms, 3), "alg_GB": round(ps.alg_bytes / 1e9, 3), "GBps": round(gbps, 1),
                    "frac": round(gbps / PEAK, 3)})
        print(json.dumps(out[-1]), flush=True)
        del ps, ads
        torch.cuda.empty_cache()


def step():
    from paper_2407_02031_b200.pipeline import AddonPipeline, synthetic_request
    t0 = time.time()
    pipe = AddonPipeline(U.SDXL, n_controlnets=2, steps=30, dtype=torch.bfloat16)
    ads = [(synthetic_lora(pipe.unet_p, 64, seed=i, adapter_id=f"l{i}"), 0.7) for i in range(2)]
    pipe.load_loras(ads)
    pipe.setup()
    print("setup s", round(time.time() - t0, 1), flush=True)
    step_ms, patch_ms = pipe.calibrate(reps=5)
    print(json.dumps({"step_ms": step_ms, "patch_ms": patch_ms}), flush=True)
    req = synthetic_request(U.SDXL, 2)
    pin = {}
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.time()
        pipe.generate(req, patch=True, pinned=pin)
        torch.cuda.synchronize()
        print("image s", round(time.time() - t, 3), "first_patched", pipe.last_first_patched_step, flush=True)


if __name__ == "__main__":
    {"lora": lora, "step": step}[sys.argv[1]]()
