"""K7 cross-attention forms at the SDXL shapes (dev aid): persistent tcgen05
(mode 2), per-tile tcgen05 / mma.sync (mode 1), mma.sync (mode 0); device
time per launch from CUDA-graph replays (24 launches, inputs rotated over
> 2x L2, as bench.py's roofline_other_kernels), algorithmic bytes = q read +
o write + K/V read."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

L2 = 126 << 20
peaks = ROOT / "MEASURED_PEAKS.json"
hbm = json.loads(peaks.read_text())["hbm_gbs"] if peaks.exists() else 6548.8
lib = ops._lib.lib()


def timed(make, nbytes_in, reps=24):
    rot = min(reps, max(2, -(-2 * L2 // max(nbytes_in, 1))))
    fns = [make() for _ in range(rot)]
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fns[i % rot]()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (5 * reps)


for n, lq, c, h in [(2, 4096, 640, 10), (2, 1024, 1280, 20), (16, 4096, 640, 10), (16, 1024, 1280, 20)]:
    nbytes = 2 * n * lq * c * 2 + n * 77 * 2 * c * 2
    line = f"[{n},{lq},{c}] x 77, {h} heads, {nbytes / 1e6:.1f} MB:"
    ref = None
    for mode in (2, 1, 0):
        prev = lib.sdb_cross_attention_set_mode(mode)
        try:
            q = torch.randn(n, lq, c, device="cuda").to(torch.bfloat16)
            kv = torch.randn(n, 77, 2 * c, device="cuda").to(torch.bfloat16)
            o = ops.cross_attention(q, kv, h)
            if ref is None:
                ref = o
            diff = (o.float() - ref.float()).abs().max().item()

            def mk():
                qq = torch.randn(n, lq, c, device="cuda").to(torch.bfloat16)
                kk = torch.randn(n, 77, 2 * c, device="cuda").to(torch.bfloat16)
                oo = torch.empty_like(qq)
                return lambda: ops.cross_attention(qq, kk, h, out=oo)
            t = timed(mk, nbytes)
        finally:
            lib.sdb_cross_attention_set_mode(prev)
        gbs = nbytes / t / 1e6
        line += f" | mode {mode}: {t * 1e3:6.2f} us {gbs:5.0f} GB/s ({gbs / hbm:4.0%}) max|d vs mode 2| {diff:.1e}"
    print(line, flush=True)
