"""to_out GEMM + residual add + LayerNorm (dev aid): (A) d = o W^T + b, then
K6 (x += d, LN) vs (B) x += o W^T inside cuBLAS (beta = 1, in place), then
the LayerNorm pass alone.  CUDA-graph replays, inputs rotated over > 2x L2."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

L2 = 126 << 20


def gt(fns, reps=24):
    for f in fns:
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fns[i % len(fns)]()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (5 * reps) * 1000


for m, c, kin in [(2048, 1280, 1280), (8192, 640, 640), (2048, 1280, 5120), (8192, 640, 2560)]:
    rot = max(2, -(-2 * L2 // (m * c * 2 * 3)))
    w = torch.randn(c, kin, device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.randn(c, device="cuda", dtype=torch.bfloat16)
    g_, be = torch.ones(c, device="cuda", dtype=torch.bfloat16), torch.zeros(c, device="cuda", dtype=torch.bfloat16)
    os_ = [torch.randn(m, kin, device="cuda", dtype=torch.bfloat16) for _ in range(rot)]
    xs = [torch.randn(m, c, device="cuda", dtype=torch.bfloat16) for _ in range(rot)]

    def a_(i):
        d = F.linear(os_[i], w, b)
        ops.add_layernorm(xs[i], d, g_, be)

    def b_(i):
        xs[i].addmm_(os_[i], w.t())
        ops.add_layernorm(xs[i], None, g_, be)
    ta = gt([lambda i=i: a_(i) for i in range(rot)])
    tb = gt([lambda i=i: b_(i) for i in range(rot)])
    tg1 = gt([lambda i=i: F.linear(os_[i], w, b) for i in range(rot)])
    tg2 = gt([lambda i=i: xs[i].addmm_(os_[i], w.t()) for i in range(rot)])
    print(f"[{m},{kin}]->{c}: A gemm+bias -> K6(x,d) {ta:.1f} us (gemm {tg1:.1f}) | B addmm_ -> LN {tb:.1f} us "
          f"(gemm {tg2:.1f}) | saves {ta - tb:.1f} us", flush=True)
