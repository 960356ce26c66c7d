"""K5' (FF GEMM + GEGLU epilogue, tcgen05) vs cuBLAS + K5 at the SDXL shapes
(dev aid): parity vs an fp32 reference and CUDA-graph timing with inputs
rotated over > 2x L2."""
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


for m, k, f in [(8192, 640, 2560), (2048, 1280, 5120), (300, 128, 256), (16384, 1280, 5120)]:
    w = (torch.randn(2 * f, k, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.randn(2 * f, device="cuda").to(torch.bfloat16)
    bf = b.float()
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = ops.ff_geglu(x, w, bf)
    p = x.float() @ w.float().t() + bf
    ref = p[:, :f] * F.gelu(p[:, f:])
    lib = ops.geglu(F.linear(x, w, b))
    err = (y.float() - ref).abs().max().item()
    lerr = (lib.float() - ref).abs().max().item()
    rel = ((y.float() - ref).norm() / ref.norm()).item()
    rot = max(2, -(-2 * L2 // (m * 2 * f * 2)))
    xs = [torch.randn(m, k, device="cuda").to(torch.bfloat16) for _ in range(rot)]
    t_f = gt([lambda i=i: ops.ff_geglu(xs[i], w, bf) for i in range(rot)])
    t_l = gt([lambda i=i: ops.geglu(F.linear(xs[i], w, b)) for i in range(rot)])
    t_g = gt([lambda i=i: F.linear(xs[i], w, b) for i in range(rot)])
    tf = 2 * m * k * 2 * f / (t_f * 1e-6) / 1e12
    print(f"[{m},{k}]x{2 * f}: fused {t_f:.1f} us ({tf:.0f} TFLOP/s) | cuBLAS+K5 {t_l:.1f} us (GEMM {t_g:.1f}) | "
          f"max|err| {err:.2e} (library {lerr:.2e}) rel-L2 {rel:.1e}", flush=True)
