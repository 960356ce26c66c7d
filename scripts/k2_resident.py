"""K2 forms at SDXL's two-pass GroupNorm sites (development aid): two-pass
(mode 1), streamed cluster (mode 3), resident cooperative form (mode 4), auto
(mode 0) — device time per launch from CUDA-graph replays with inputs rotated
over > 2x L2 (scripts/k2_bench.py's harness), parity vs fp32 torch, rerun
determinism, and concurrent launches on three streams (eager and as parallel
graph branches) against the sequential results."""
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

L2 = 126 << 20
peaks = ROOT / "MEASURED_PEAKS.json"
hbm = json.loads(peaks.read_text())["hbm_gbs"] if peaks.exists() else 6548.8
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


lib = ops._lib.lib()
shapes = [(2, 320, 128, 128), (2, 640, 64, 64), (2, 960, 64, 64), (2, 1280, 32, 32), (2, 320, 64, 64),
          (1, 320, 128, 128), (2, 640, 32, 32), (2, 1920, 32, 32)]
for n, c, h, w in shapes:
    numel = n * c * h * w
    gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
    add = torch.randn(n, c, device="cuda")
    plan = (ctypes.c_int * 4)()
    ok = lib.sdb_groupnorm_resident_plan(n, h * w, c, 32, plan)
    x = torch.randn(n, c, h, w, device="cuda").mul(2).add(0.7).to(torch.bfloat16).contiguous(memory_format=cl)
    ref = F.silu(F.group_norm(x.float() + add[:, :, None, None], 32, gm, bt, 1e-5))
    line = f"[{n},{c},{h},{w}] {numel * 2 / 1e6:5.1f} MB plan {list(plan) if ok else None}"
    for mode, name in ((1, "two-pass"), (3, "stream"), (4, "resident"), (0, "auto")):
        with ops.groupnorm_mode(mode):
            launches = lib.sdb_groupnorm_launches(n, h * w, c, 32, ops.sdb_dtype(x))
            if mode == 4 and not ok:
                line += f" | {name}: n/a"
                continue
            y = ops.groupnorm_silu(x, gm, bt, add_nc=add)
            y2 = ops.groupnorm_silu(x, gm, bt, add_nc=add)
        err = float(((y.float() - ref).abs() / (ref.abs() * 2 ** -8 + 2e-3)).max())

        def mk():
            xx = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
            yy = torch.empty_like(xx)
            ws = ops.groupnorm_workspace(xx)

            def f():
                with ops.groupnorm_mode(mode):
                    ops.groupnorm_silu(xx, gm, bt, out=yy, add_nc=add, workspace=ws)
            return f
        t = timed(mk, numel * 2)
        gbs = 2 * numel * 2 / t / 1e6
        line += (f" | {name}[{launches}]: {t * 1e3:6.2f} us {gbs:5.0f} GB/s ({gbs / hbm:4.0%}) "
                 f"err/bound {err:.2f} det {torch.equal(y, y2)}")
    print(line, flush=True)

# concurrency: three streams (separate workspaces, as separate networks have)
n, c, h, w = 2, 320, 128, 128
xs = [torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl) for _ in range(3)]
wss = [ops.groupnorm_workspace(x) for x in xs]
gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
with ops.groupnorm_mode(4):
    seq = [ops.groupnorm_silu(x, gm, bt, workspace=ws) for x, ws in zip(xs, wss)]
    outs = [torch.empty_like(x) for x in xs]
    streams = [torch.cuda.Stream() for _ in range(3)]
    torch.cuda.synchronize()
    for rep in range(50):
        for x, ws, o, s in zip(xs, wss, outs, streams):
            with torch.cuda.stream(s):
                ops.groupnorm_silu(x, gm, bt, out=o, workspace=ws)
    torch.cuda.synchronize()
    eager_ok = all(torch.equal(a, b) for a, b in zip(seq, outs))
    for o in outs:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cap):
        for rep in range(10):
            for x, ws, o, s in zip(xs, wss, outs, streams):
                s.wait_stream(cap)
                with torch.cuda.stream(s):
                    ops.groupnorm_silu(x, gm, bt, out=o, workspace=ws)
        for s in streams:
            cap.wait_stream(s)
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    graph_ok = all(torch.equal(a, b) for a, b in zip(seq, outs))
print(f"concurrent resident launches on 3 streams: eager bitwise {eager_ok}, graph branches bitwise {graph_ok}")
