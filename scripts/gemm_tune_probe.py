"""SDXL linear shapes: default cuBLAS pick vs PyTorch TunableOp (cuBLASLt solutions tuned per shape).
Timed as CUDA-graph replays (no host overhead)."""
import json
import os
import sys

import torch
import torch.nn.functional as F


def gtime(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (5 * reps) * 1000


SHAPES = [  # (M tokens, K in, N out, bias)
    (2048, 1280, 1280, True), (2048, 1280, 3840, False), (2048, 1280, 10240, True), (2048, 5120, 1280, True),
    (8192, 640, 640, True), (8192, 640, 1920, False), (8192, 640, 5120, True), (8192, 2560, 640, True),
    (154, 2048, 2560, False),
]


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "default"
    if mode == "tunable":
        import torch.cuda.tunable as tun
        tun.enable(True)
        tun.tuning_enable(True)
        tun.set_filename(os.environ.get("TUNE_FILE", "/tmp/tunableop_results.csv"))
    out = []
    for m, k, n, bias in SHAPES:
        x = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        w = torch.randn(n, k, device="cuda", dtype=torch.bfloat16) * 0.02
        b = torch.zeros(n, device="cuda", dtype=torch.bfloat16) if bias else None
        if mode == "tunable":
            F.linear(x, w, b)   # tunes this shape (outside graph capture)
        us = gtime(lambda: F.linear(x, w, b))
        tf = 2 * m * k * n / (us * 1e-6) / 1e12
        out.append({"mode": mode, "m": m, "k": k, "n": n, "bias": bias, "us": round(us, 2), "TFLOPs": round(tf, 1)})
        print(json.dumps(out[-1]), flush=True)
    if mode == "tunable":
        import torch.cuda.tunable as tun
        tun.write_file()


if __name__ == "__main__":
    main()
