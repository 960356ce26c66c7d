"""K6 add+LayerNorm at the SDXL shapes (dev aid): device time per launch
from CUDA-graph replays (24 launches, inputs rotated over > 2x L2);
algorithmic bytes = read x, d + write x, y."""
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


line = sys.argv[1] if len(sys.argv) > 1 else ""
for n, l, c in [(2, 4096, 640), (2, 1024, 1280), (16, 4096, 640), (16, 1024, 1280), (2, 4096, 320)]:
    w, b = torch.ones(c, device="cuda", dtype=torch.bfloat16), torch.zeros(c, device="cuda", dtype=torch.bfloat16)

    def mk():
        x = torch.randn(n, l, c, device="cuda").to(torch.bfloat16)
        d = torch.randn_like(x)
        y = torch.empty_like(x)
        return lambda: ops.add_layernorm(x, d, w, b)
    nb = 4 * n * l * c * 2
    t = timed(mk, 2 * n * l * c * 2)
    gbs = nb / t / 1e6
    line += f" | [{n},{l},{c}] {t * 1e3:6.2f} us ({gbs / hbm:4.0%})"
print(line, flush=True)
