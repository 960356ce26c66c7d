"""K3 residual inject with / without the fused GroupNorm statistics (dev aid):
device time per launch from CUDA-graph replays (24 launches, inputs rotated
over > 2x L2).  Algorithmic bytes: read skip + residuals, write out."""
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
cl = torch.channels_last


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


tag = sys.argv[1] if len(sys.argv) > 1 else ""
line = tag
for n, c, h, w, nr in [(2, 320, 128, 128, 1), (2, 640, 64, 64, 1), (2, 1280, 32, 32, 1), (2, 320, 128, 128, 0)]:
    numel = n * c * h * w
    for stats in (False, True):
        def mk():
            sk = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
            rs = [torch.randn_like(sk) for _ in range(nr)]
            out = torch.empty_like(sk)
            ws = ops.groupnorm_workspace(sk) if stats else None
            sb = torch.randn(c, device="cuda")
            return lambda: ops.residual_inject(sk, rs, [0.8] * nr, out=out, skip_bias=sb, gn_workspace=ws)
        nb = (2 + nr) * numel * 2
        t = timed(mk, (1 + nr) * numel * 2)
        line += f" | [{n},{c},{h},{w}]+{nr} {'stats' if stats else 'plain'} {t * 1e3:6.2f} us ({nb / t / 1e6 / hbm:4.0%})"
print(line, flush=True)
