"""K8 self-attention vs the library (cuDNN SDPA) at SDXL's shapes: error vs
fp32 and device time per call (CUDA-graph replays).  SDB_FMHA=1 selects round
1's single-tile kernel (one process per setting).  Development aid."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402


def graph_time(fn, reps=20):
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


shapes = [(2, 4096, 10), (2, 1024, 20)] if len(sys.argv) < 2 else [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for n, L, h in shapes:
    c = h * 64
    qkv = torch.randn(n, L, 3 * c, device="cuda").to(torch.bfloat16)
    q, k, v = (t.reshape(n, L, h, 64).transpose(1, 2) for t in qkv.split(c, dim=-1))
    ref = F.scaled_dot_product_attention(q.float(), k.float(), v.float()).transpose(1, 2).reshape(n, L, c)
    o = ops.self_attention(qkv, h)
    err = (o.float() - ref).abs().max().item()
    lib = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(n, L, c)
    lerr = (lib.float() - ref).abs().max().item()
    t_ours = graph_time(lambda: ops.self_attention(qkv, h))
    t_lib = graph_time(lambda: F.scaled_dot_product_attention(q, k, v))
    flops = 4 * n * h * L * L * 64
    print(f"[{n},{L},{h}] ours {t_ours:7.2f} us ({flops / t_ours / 1e6:6.0f} TF/s) err {err:.2e} | "
          f"cuDNN {t_lib:7.2f} us ({flops / t_lib / 1e6:6.0f} TF/s) err {lerr:.2e}", flush=True)
