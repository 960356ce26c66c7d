"""The ControlNet hint embedding's conv_out ([2,256,128,128] -> 320, 3x3): cuDNN
picks a TF32 fallback; variants (CUDA-graph replays)."""
import torch
import torch.nn.functional as F


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def gt(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000


x = cl(torch.randn(2, 256, 128, 128, device="cuda").bfloat16())
w = cl(torch.randn(320, 256, 3, 3, device="cuda").bfloat16() * 0.02)
xp = cl(torch.zeros(2, 320, 128, 128, device="cuda").bfloat16())
wp = cl(torch.zeros(320, 320, 3, 3, device="cuda").bfloat16())
xp[:, :256].copy_(x)
wp[:, :256].copy_(w)
print("native", gt(lambda: F.conv2d(x, w, padding=1)))
print("cin padded to 320", gt(lambda: F.conv2d(xp, wp, padding=1)))
print("contiguous (NCHW)", gt(lambda: F.conv2d(x.contiguous(), w.contiguous(), padding=1)))
w2 = cl(torch.randn(256, 256, 3, 3, device="cuda").bfloat16() * 0.02)
print("256 -> 256", gt(lambda: F.conv2d(x, w2, padding=1)))
