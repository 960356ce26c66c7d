"""Self-attention at SDXL's shapes: cuDNN SDPA (the current library path) vs
flashinfer's trtllm-gen Blackwell FMHA (paged-KV context kernel, non-causal),
reading q / k / v straight out of the fused q|k|v projection.  Development aid."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (3 * reps) * 1000.0


t0 = time.time()
import flashinfer  # noqa: E402
from flashinfer.prefill import trtllm_batch_context_with_kv_cache  # noqa: E402
print("flashinfer", flashinfer.__version__, "import", round(time.time() - t0, 1), "s", flush=True)

for n, L, heads in [(2, 4096, 10), (2, 1024, 20), (16, 4096, 10), (16, 1024, 20)]:
    d = 64
    C = heads * d
    qkv = torch.randn(n, L, 3 * C, device="cuda", dtype=torch.bfloat16)
    q, k, v = qkv.split(C, dim=-1)
    qh = q.view(n, L, heads, d).transpose(1, 2)
    kh = k.view(n, L, heads, d).transpose(1, 2)
    vh = v.view(n, L, heads, d).transpose(1, 2)

    def sdpa():
        return F.scaled_dot_product_attention(qh, kh, vh)
    t_sdpa = timed(sdpa)
    ref = sdpa().transpose(1, 2).reshape(n * L, C).float()
    # trtllm-gen: paged KV with page_size P tokens, NHD view straight into q|k|v
    res = {}
    for P in (16, 32, 64):
        try:
            pages = L // P
            kc = k.reshape(n * pages, P, heads, d)        # strided views (token stride 3C)
            vc = v.reshape(n * pages, P, heads, d)
            qq = q.reshape(n * L, heads, d)
            block_tables = torch.arange(n * pages, device="cuda", dtype=torch.int32).view(n, pages)
            seq_lens = torch.full((n,), L, device="cuda", dtype=torch.int32)
            cum = torch.arange(0, (n + 1) * L, L, device="cuda", dtype=torch.int32)
            ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
            out = torch.empty(n * L, heads, d, device="cuda", dtype=torch.bfloat16)

            def fmha():
                return trtllm_batch_context_with_kv_cache(
                    qq, (kc, vc), ws, block_tables, seq_lens, L, L, d ** -0.5, 1.0, n, cum, cum,
                    out=out, kv_layout="NHD", causal=False)
            t = timed(fmha)
            err = float((fmha().reshape(n * L, C).float() - ref).abs().max())
            res[P] = (round(t, 1), f"{err:.1e}")
        except Exception as e:  # noqa: BLE001
            res[P] = f"{type(e).__name__}: {str(e)[:160]}"
    print(f"[{n},{L},{heads}x{d}] cuDNN SDPA {t_sdpa:.1f} us | trtllm-gen {res}", flush=True)
