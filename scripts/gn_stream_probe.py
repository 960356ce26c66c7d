"""K2 forms side by side at the SDXL / SD1.5 GroupNorm sites: the two-pass
form (mode 1), round 1's cluster form (mode 2) and the streamed cluster form
(mode 3): parity vs fp32 torch and device time per launch (CUDA-graph
replays, inputs rotated over > 2x L2).  SDB_GN_SLAB="S,cs" pins the streamed
form's slab / cluster size (one process per setting).  Development aid."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2407_02031_b200 import _lib, ops  # noqa: E402

L2 = 126 << 20
HBM = 6548.8


def graph_time(fns, reps=16):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fns[:2]:
            f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fns[i % len(fns)]()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (5 * reps) * 1000


shapes = [(2, 320, 128, 128), (2, 640, 64, 64), (2, 1280, 32, 32), (2, 640, 128, 128), (2, 960, 64, 64),
          (2, 320, 64, 64), (2, 640, 32, 32), (16, 320, 128, 128), (16, 640, 64, 64)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
lib = _lib.lib()
for n, c, h, w in shapes:
    nbytes = n * c * h * w * 2
    rot = max(2, -(-2 * L2 // nbytes))
    xs = [torch.randn(n, c, h, w, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last) * 3 + 1
          for _ in range(rot)]
    ys = [torch.empty_like(x) for x in xs]
    gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
    add = torch.randn(n, c, device="cuda")
    ws = ops.groupnorm_workspace(xs[0], 32)
    plan = (ctypes.c_int * 7)()
    ok = lib.sdb_groupnorm_stream_plan(n, h * w, c, 32, plan)
    ref = F.silu(F.group_norm(xs[0].float() + add[:, :, None, None], 32, gm, bt, 1e-5))
    line = [f"[{n},{c},{h},{w}] {nbytes / 1e6:5.1f} MB plan {list(plan) if ok else None}"]
    for mode, name in ((1, "two-pass"), (2, "v1"), (3, "stream")):
        with ops.groupnorm_mode(mode):
            launches = lib.sdb_groupnorm_launches(n, h * w, c, 32, _lib.SDB_BF16)
            if mode != 1 and launches != 1:
                line.append(f"{name}: n/a")
                continue
            y = ops.groupnorm_silu(xs[0], gm, bt, 32, 1e-5, True, out=ys[0], add_nc=add, workspace=ws)
            err = float((y.float() - ref).abs().max())
            y2 = ops.groupnorm_silu(xs[0], gm, bt, 32, 1e-5, True, add_nc=add, workspace=ws)
            det = bool(torch.equal(y, y2))
            us = graph_time([(lambda i=i: ops.groupnorm_silu(xs[i], gm, bt, 32, 1e-5, True, out=ys[i], add_nc=add,
                                                              workspace=ws)) for i in range(rot)])
        line.append(f"{name}: {us:6.2f} us {2 * nbytes / us / 1e3:5.0f} GB/s ({2 * nbytes / us / 1e3 / HBM:4.0%}) "
                    f"err {err:.1e} det {det}")
    print(" | ".join(line), flush=True)
