"""Self-attention library options at SDXL's shapes (hd 64): torch SDPA (cuDNN)
vs the CuTe-DSL FA4 kernel shipped with vllm (vllm.vllm_flash_attn.cute),
incl. its JIT compile time and CUDA-graph capture."""
import time

import torch
import torch.nn.functional as F


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1000


t0 = time.time()
from vllm.vllm_flash_attn.cute.interface import flash_attn_func  # noqa: E402
print(f"import {time.time() - t0:.1f}s")
for n, L, H in ((2, 4096, 10), (2, 1024, 20), (16, 4096, 10), (16, 1024, 20)):
    C = H * 64
    qkv = torch.randn(n, L, 3 * C, device="cuda", dtype=torch.bfloat16)
    q = qkv[..., :C].view(n, L, H, 64)
    k = qkv[..., C:2 * C].view(n, L, H, 64)
    v = qkv[..., 2 * C:].view(n, L, H, 64)
    flops = 4 * n * H * L * L * 64

    def sdpa():
        return F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2))

    t0 = time.time()
    try:
        o4 = flash_attn_func(q, k, v)
        o4 = o4[0] if isinstance(o4, tuple) else o4
        torch.cuda.synchronize()
        tc = time.time() - t0
        err = (o4.float() - sdpa().transpose(1, 2).float()).abs().max().item()
        t4 = timeit(lambda: flash_attn_func(q, k, v))
        # graph capture
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            flash_attn_func(q, k, v)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            flash_attn_func(q, k, v)
        g.replay()
        torch.cuda.synchronize()
        tg = timeit(lambda: g.replay())
        fa4 = f"FA4 {t4:.1f} us ({flops / t4 / 1e6:.0f} TF/s), graph {tg:.1f} us, compile {tc:.1f}s, max|err| {err:.2e}"
    except Exception as e:  # noqa: BLE001
        fa4 = f"FA4 failed: {type(e).__name__}: {str(e)[:300]}"
    ts = timeit(sdpa)
    print(f"n={n} L={L} H={H}: sdpa {ts:.1f} us ({flops / ts / 1e6:.0f} TF/s) | {fa4}")
