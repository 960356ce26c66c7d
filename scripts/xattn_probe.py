"""K7 cross-attention vs the library SDPA kernels at the SDXL shapes (development aid).
L2 is flushed before every launch (inputs << L2 otherwise)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")   # 256 MB, READ to evict L2 (no dirty lines)
sink = torch.empty(64 << 20 >> 20, device="cuda")[:0]


def t(fn, reps=50, cold=True):
    """cold: L2 evicted (read sweep) before each launch, per-launch events;
    warm: reps back-to-back launches between two events (launch latency hidden)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if not cold:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps * 1000
    tot = 0.0
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1000


for name, (n, lq, c, h) in {"cross64": (2, 4096, 640, 10), "cross32": (2, 1024, 1280, 20)}.items():
    q = torch.randn(n, lq, c, device="cuda", dtype=torch.bfloat16)
    kv = torch.randn(n, 77, 2 * c, device="cuda", dtype=torch.bfloat16)
    d = c // h
    qs = q.view(n, lq, h, d).transpose(1, 2)
    ks = kv[..., :c].reshape(n, 77, h, d).transpose(1, 2)
    vs = kv[..., c:].reshape(n, 77, h, d).transpose(1, 2)
    res = {}
    import os
    if os.environ.get("WARM_ONLY"):
        res["k7_warm"] = t(lambda: ops.cross_attention(q, kv, h), cold=False)
        print(name, os.environ.get("SDB_XATTN_TPW"), res, flush=True)
        continue
    for cold in (True, False):
        sfx = "" if cold else "_warm"
        res["k7" + sfx] = t(lambda: ops.cross_attention(q, kv, h), cold=cold)
        with sdpa_kernel([SDPBackend.FLASH_ATTENTION]):
            res["flash" + sfx] = t(lambda: F.scaled_dot_product_attention(qs, ks, vs), cold=cold)
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            res["cudnn" + sfx] = t(lambda: F.scaled_dot_product_attention(qs, ks, vs), cold=cold)
    gb = 2 * q.numel() * 2 / 1e9
    print(name, {k: round(v, 2) for k, v in res.items()}, "us; k7 GB/s", round(gb / (res["k7"] * 1e-6), 1), flush=True)
