"""cuDNN 3x3 conv efficiency at every distinct SDXL UNet conv shape (bf16,
channels_last, CFG batch 2; CUDA-graph replays): finds shapes where cuDNN
falls off its tensor-op kernels."""
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


shapes = [(4, 320, 128, 1), (320, 320, 128, 2), (256, 320, 128, 1), (320, 320, 128, 1), (640, 320, 128, 1), (960, 320, 128, 1), (640, 640, 128, 1),
          (320, 640, 64, 1), (640, 640, 64, 1), (640, 640, 64, 2), (1280, 640, 64, 1), (1920, 640, 64, 1),
          (960, 640, 64, 1), (1280, 1280, 64, 1),
          (640, 1280, 32, 1), (1280, 1280, 32, 1), (2560, 1280, 32, 1), (1920, 1280, 32, 1)]
import os
NB = int(os.environ.get("NB", "2"))
for cin, cout, hw, st in shapes:
    x = cl(torch.randn(NB, cin, hw, hw, device="cuda").bfloat16())
    w = cl(torch.randn(cout, cin, 3, 3, device="cuda").bfloat16() * 0.02)
    t = gt(lambda: F.conv2d(x, w, stride=st, padding=1))
    ho = hw // st
    fl = 2 * NB * ho * ho * cout * cin * 9
    print(f"[{NB},{cin},{hw},{hw}] -> {cout} s{st}: {t:7.1f} us {fl / t / 1e6:6.0f} TF/s")
