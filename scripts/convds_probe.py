"""The downsample convs (3x3 stride 2) at SDXL shapes: cuDNN heuristics vs
cudnn.benchmark autotuning (CUDA-graph replays)."""
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


for bench in (False, True):
    torch.backends.cudnn.benchmark = bench
    for c, hw, stride in ((320, 128, 2), (640, 64, 2), (320, 128, 1), (640, 64, 1), (1280, 32, 1)):
        x = cl(torch.randn(2, c, hw, hw, device="cuda").bfloat16())
        w = cl(torch.randn(c, c, 3, 3, device="cuda").bfloat16() * 0.02)
        t = gt(lambda: F.conv2d(x, w, stride=stride, padding=1))
        print(f"benchmark={bench} [2,{c},{hw},{hw}] 3x3 s{stride}: {t:.1f} us")

torch.backends.cudnn.benchmark = False
for c, hw in ((320, 128), (640, 64)):
    x = cl(torch.randn(2, c, hw, hw, device="cuda").bfloat16())
    w = cl(torch.randn(c, c, 3, 3, device="cuda").bfloat16() * 0.02)
    t_sub = gt(lambda: cl(F.conv2d(x, w, padding=1)[:, :, ::2, ::2]))
    ref = F.conv2d(x, w, stride=2, padding=1)
    sub = cl(F.conv2d(x, w, padding=1)[:, :, ::2, ::2])
    print(f"[2,{c},{hw},{hw}] s1 conv + subsample: {t_sub:.1f} us  max|diff| vs s2 {(ref.float() - sub.float()).abs().max().item():.3e}")
