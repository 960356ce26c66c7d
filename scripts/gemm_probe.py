"""cuBLAS efficiency on the SDXL step's GEMM shapes (development aid)."""

import torch
import torch.nn.functional as F

PEAK = 1652.1  # TF/s burst, MEASURED_PEAKS.json


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    shapes = {  # (M tokens, K in, N out) for CFG batch 2
        "l1 qkv": (8192, 640, 1920), "l1 out": (8192, 640, 640), "l1 ff.proj": (8192, 640, 5120),
        "l1 ff.out": (8192, 2560, 640), "l2 qkv": (2048, 1280, 3840), "l2 out": (2048, 1280, 1280),
        "l2 ff.proj": (2048, 1280, 10240), "l2 ff.out": (2048, 5120, 1280), "l2 q(cross)": (2048, 1280, 1280),
        "kv ctx 1280": (154, 2048, 2560), "temb proj": (2, 1280, 1280),
    }
    for name, (m, k, n) in shapes.items():
        x = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
        ms = t(lambda: F.linear(x, w))
        tf = 2 * m * n * k / (ms * 1e-3) / 1e12
        print(f"{name:14s} M={m:5d} K={k:5d} N={n:5d}: {ms * 1000:8.1f} us  {tf:7.1f} TF/s  {100 * tf / PEAK:5.1f}% of peak",
              flush=True)
    for name, (c, h) in {"conv 320@128": (320, 128), "conv 640@64": (640, 64), "conv 1280@32": (1280, 32)}.items():
        x = torch.randn(2, c, h, h, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
        w = torch.randn(c, c, 3, 3, device="cuda", dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
        ms = t(lambda: F.conv2d(x, w, padding=1))
        tf = 2 * 2 * h * h * c * c * 9 / (ms * 1e-3) / 1e12
        print(f"{name:14s}: {ms * 1000:8.1f} us  {tf:7.1f} TF/s  {100 * tf / PEAK:5.1f}% of peak", flush=True)


if __name__ == "__main__":
    main()
