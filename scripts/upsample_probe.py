"""Nearest 2x upsample of NHWC bf16 maps (SDXL decoder): F.interpolate vs an
expand + copy (CUDA-graph replays)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402


def cl(t):
    return t.contiguous(memory_format=torch.channels_last)


def gt(fn, reps=20):
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


def up_expand(x):
    n, c, h, w = x.shape
    v = x.permute(0, 2, 3, 1)[:, :, None, :, None, :].expand(n, h, 2, w, 2, c).reshape(n, 2 * h, 2 * w, c)
    return v.permute(0, 3, 1, 2)


for c, hw in ((1280, 32), (640, 64)):
    x = cl(torch.randn(2, c, hw, hw, device="cuda").bfloat16())
    t0 = gt(lambda: F.interpolate(x, scale_factor=2.0, mode="nearest"))
    t1 = gt(lambda: up_expand(x))
    t2 = gt(lambda: ops.upsample2x(x))
    a = F.interpolate(x, scale_factor=2.0, mode="nearest")
    b = up_expand(x)
    print(f"[2,{c},{hw},{hw}]: interpolate {t0:.1f} us, expand+copy {t1:.1f} us, K10 {t2:.1f} us, equal={torch.equal(a, b)}, "
          f"cl={b.is_contiguous(memory_format=torch.channels_last)} / {a.is_contiguous(memory_format=torch.channels_last)}")
