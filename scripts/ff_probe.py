"""FF1 GEMM -> K5 GEGLU back to back (dev aid): is K5's input still in L2
when it follows the GEMM that wrote it?  CUDA-graph replays, each pair on its
own rotated inputs (> 2x L2), vs the GEMM alone and K5 alone (cold)."""
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


for m, k, f2 in [(8192, 640, 5120), (2048, 1280, 10240), (16384, 1280, 10240)]:
    rot = max(2, -(-2 * L2 // (m * f2 * 2)))
    w = torch.randn(f2, k, device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.zeros(f2, device="cuda", dtype=torch.bfloat16)
    xs = [torch.randn(m, k, device="cuda", dtype=torch.bfloat16) for _ in range(rot)]
    ps = [torch.empty(m, f2, device="cuda", dtype=torch.bfloat16) for _ in range(rot)]
    outs = [torch.empty(m, f2 // 2, device="cuda", dtype=torch.bfloat16) for _ in range(rot)]
    t_gemm = gt([lambda i=i: torch.addmm(b, xs[i], w.t(), out=ps[i]) for i in range(rot)])
    t_k5 = gt([lambda i=i: ops.geglu(ps[i]) for i in range(rot)])

    def pair(i):
        torch.addmm(b, xs[i], w.t(), out=ps[i])
        ops.geglu(ps[i])
    t_pair = gt([lambda i=i: pair(i) for i in range(rot)])
    print(f"[{m},{k}]x{f2}: gemm {t_gemm:.1f} us, geglu cold {t_k5:.1f} us, gemm->geglu {t_pair:.1f} us "
          f"(geglu in situ ~{t_pair - t_gemm:.1f} us)", flush=True)
