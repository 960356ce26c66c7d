"""conv_in (4 -> 320, 3x3) at SDXL's [2, 4, 128, 128]: cuDNN on the 4-channel
input vs zero-padded to 8 channels (+ the two copies), CUDA-graph replays."""
import torch
import torch.nn.functional as F


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def gt(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
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


for cin, cout, n, hw in ((4, 320, 2, 128), (3, 16, 2, 1024), (4, 320, 16, 128)):
    x = cl(torch.randn(n, cin, hw, hw, device="cuda").bfloat16())
    w = cl(torch.randn(cout, cin, 3, 3, device="cuda").bfloat16())
    xp = cl(torch.zeros(n, 8, hw, hw, device="cuda").bfloat16())
    wp = cl(torch.zeros(cout, 8, 3, 3, device="cuda").bfloat16())
    xp16 = cl(torch.zeros(n, 16, hw, hw, device="cuda").bfloat16())
    wp16 = cl(torch.zeros(cout, 16, 3, 3, device="cuda").bfloat16())

    def pad():
        xp[:, :cin].copy_(x)
        wp[:, :cin].copy_(w)
        return F.conv2d(xp, wp, padding=1)

    def pad_conv_only():
        return F.conv2d(xp, wp, padding=1)

    t0 = gt(lambda: F.conv2d(x, w, padding=1))
    t1 = gt(pad)
    t2 = gt(pad_conv_only)
    t3 = gt(lambda: F.conv2d(xp16, wp16, padding=1))
    print(f"[{n},{cin},{hw},{hw}] -> {cout}: cin={cin} {t0:.1f} us | padded to 8 incl. copies {t1:.1f} us "
          f"(conv alone {t2:.1f} us; 16 channels {t3:.1f} us)")
