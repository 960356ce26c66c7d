"""cuBLAS (torch) bf16 GEMM efficiency at the SDXL step's linear shapes
(CUDA-graph replays; TFLOP/s vs the measured dense peak)."""
import json
import torch
import torch.nn.functional as F

peak = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {}


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


shapes = [  # (M tokens, K in, N out, bias, what)
    (2048, 1280, 1280, True, "L2 attn out / proj"), (2048, 1280, 3840, False, "L2 qkv"),
    (2048, 1280, 10240, True, "L2 ff.proj"), (2048, 5120, 1280, True, "L2 ff.out"),
    (8192, 640, 640, True, "L1 attn out / proj"), (8192, 640, 1920, False, "L1 qkv"),
    (8192, 640, 5120, True, "L1 ff.proj"), (8192, 2560, 640, True, "L1 ff.out"),
]
for m, k, n, bias, what in shapes:
    x = torch.randn(m, k, device="cuda").bfloat16()
    w = torch.randn(n, k, device="cuda").bfloat16()
    b = torch.randn(n, device="cuda").bfloat16() if bias else None
    t = gt(lambda: F.linear(x, w, b))
    tf = 2 * m * n * k / t / 1e6
    print(f"{what:22s} [{m}x{k}] x [{k}x{n}]: {t:7.1f} us {tf:6.0f} TF/s")
print("peaks:", {k: v for k, v in peak.items() if "bf16" in k.lower() or "tflop" in k.lower()})
