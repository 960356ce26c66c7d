"""K2 single-pass cluster form vs the two-pass form at the SDXL GN sites
(CUDA-graph replays of 16 launches, inputs rotated over > 2x L2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def graph_time(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(2):
            fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (3 * reps) * 1000


for n, c, h in ((2, 320, 128), (2, 640, 64), (2, 1280, 32), (2, 960, 64), (2, 2560, 32), (16, 320, 128)):
    nbytes = n * c * h * h * 2
    R = max(2, int(300e6 // nbytes) + 1)
    xs = [cl(torch.randn(n, c, h, h, device="cuda").bfloat16()) for _ in range(R)]
    ys = [torch.empty_like(x) for x in xs]
    gamma = torch.rand(c, device="cuda") + 0.5
    beta = torch.randn(c, device="cuda")
    add = torch.randn(n, c, device="cuda")
    ws = ops.groupnorm_workspace(xs[0], 32)
    res = {}
    for mode in (0, 1):
        with ops.groupnorm_mode(mode):
            res[mode] = graph_time(lambda i: ops.groupnorm_silu(xs[i % R], gamma, beta, 32, 1e-5, True,
                                                                out=ys[i % R], add_nc=add, workspace=ws), 16)
    print(f"[{n},{c},{h},{h}] {nbytes / 1e6:.1f} MB: cluster {res[0]:.2f} us "
          f"({2 * nbytes / res[0] / 1e3:.0f} GB/s) | two-pass {res[1]:.2f} us ({2 * nbytes / res[1] / 1e3:.0f} GB/s)")
