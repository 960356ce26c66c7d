"""K9 vs the cast + cuDNN (TF32) route, SDXL conv_out [2, 320, 128, 128] -> 4 fp32.
Times CUDA-graph replays of each (inputs rotated over > L2)."""
import torch
import torch.nn.functional as F

from paper_2407_02031_b200 import ops


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def bench(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000


for n in (2, 16):
    R = 8
    xs = [cl(torch.randn(n, 320, 128, 128, device="cuda").bfloat16()) for _ in range(R)]
    w = cl((torch.randn(4, 320, 3, 3, device="cuda") / 54).bfloat16())
    b = torch.randn(4, device="cuda")
    out = cl(torch.empty(n, 4, 128, 128, device="cuda"))
    t_k9 = bench(lambda i: ops.conv_out(xs[i % R], w, b, out=out))
    t_ref = bench(lambda i: F.conv2d(xs[i % R].float(), w.float(), b, padding=1))
    hbm = n * 320 * 128 * 128 * 2 / (t_k9 * 1e-6) / 1e9
    print(f"N={n}: K9 {t_k9:.1f} us ({hbm:.0f} GB/s of the activation read)  cast+cuDNN {t_ref:.1f} us")
    y = ops.conv_out(xs[0], w, b)
    ref = F.conv2d(xs[0].double(), w.double(), b.double(), padding=1)
    print("  max abs err vs fp64:", (y.double() - ref).abs().max().item())
