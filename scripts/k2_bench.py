"""K2 timing + parity at the SDXL GroupNorm sites (development aid).

Each form is captured REPS times in one CUDA graph, every launch on its own
copy of the inputs (copies spanning > 2x L2), and timed as graph replays:
device time per launch.  Forms: two-pass GN+SiLU with the temb add (stats +
apply), the K3 pass with fused statistics, and the apply alone after it.
Algorithmic bytes: one read + one write of the map (K3: its inputs + output)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

L2 = 126 << 20
hbm = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6548.8
cl = torch.channels_last


def timed(make, nbytes_in, reps=24):
    rot = min(reps, max(2, -(-2 * L2 // max(nbytes_in, 1))))
    fns = [make() for _ in range(rot)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fns[i % rot]()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (5 * reps)


shapes = [(2, 320, 128, 128), (2, 640, 128, 128), (2, 960, 128, 128), (2, 640, 64, 64), (2, 1280, 64, 64),
          (2, 1920, 64, 64), (2, 2560, 32, 32)]
for n, c, h, w in shapes:
    numel = n * c * h * w
    gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
    add = torch.randn(n, c, device="cuda")
    # parity of the two-pass form (+temb) vs fp32 torch
    x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
    with ops.groupnorm_mode(1):
        y = ops.groupnorm_silu(x, gm, bt, add_nc=add)
    ref = F.silu(F.group_norm(x.float() + add[:, :, None, None], 32, gm, bt, 1e-5))
    err = float((y.float() - ref).abs().max())

    def mk_two():
        xx = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        yy = torch.empty_like(xx)
        ws = ops.groupnorm_workspace(xx)

        def f():
            with ops.groupnorm_mode(1):
                ops.groupnorm_silu(xx, gm, bt, out=yy, add_nc=add, workspace=ws)
        return f
    t2 = timed(mk_two, numel * 2)

    def mk_inj():
        sk = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        rs = torch.randn_like(sk)
        out = torch.empty_like(sk)
        ws = ops.groupnorm_workspace(sk)
        return lambda: ops.residual_inject(sk, [rs], [0.8], out=out, gn_workspace=ws)
    t3 = timed(mk_inj, numel * 4)

    def mk_apply():
        sk = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        out = torch.empty_like(sk)
        ws = ops.groupnorm_workspace(sk)
        h0 = ops.residual_inject(sk, [], [], out=sk, gn_workspace=ws)     # publishes the statistics
        torch.cuda.synchronize()

        def f():
            h0._sdb_gn = (ws, 32, h0.data_ptr())
            ops.groupnorm_silu(h0, gm, bt, out=out)
        return f
    ta = timed(mk_apply, numel * 2)
    b2 = 2 * numel * 2
    print(f"[{n},{c},{h},{w}] {numel * 2 / 1e6:.1f} MB  two-pass(+temb) {t2 * 1e3:.1f} us "
          f"{b2 / t2 / 1e6:.0f} GB/s ({b2 / t2 / 1e6 / hbm:.2f})  | K3+stats {t3 * 1e3:.1f} us "
          f"{3 * numel * 2 / t3 / 1e6:.0f} GB/s | apply-only {ta * 1e3:.1f} us {b2 / ta / 1e6:.0f} GB/s "
          f"({b2 / ta / 1e6 / hbm:.2f}) | max|dy| {err:.2e}", flush=True)
