"""K2 vs simple bounds in bench.py's harness (CUDA-graph replays, inputs rotated over > 2x L2)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
import bench  # noqa: E402
from paper_2407_02031_b200 import ops  # noqa: E402

src = Path(bench.__file__).read_text()
# reuse the harness: pull timed() out of other_kernels_roofline by exec of its body prefix
cl = torch.channels_last
L2 = 126 << 20


def timed(make, nbytes_in, reps=24):
    rot = min(reps, max(2, -(-2 * L2 // nbytes_in)))
    bufs = [make() for _ in range(rot)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in bufs:
            f()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            bufs[i % rot]()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / (3 * reps) * 1000


for (c, hw) in [(320, 128), (640, 64), (1280, 32), (960, 128)]:
    nb = 2 * c * hw * hw * 2
    gma, bta = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")

    def mk_copy():
        x = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        y = torch.empty_like(x)
        return lambda: y.copy_(x)

    def mk_sum():
        x = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        o = torch.empty(2, 32, device="cuda", dtype=torch.float32)
        return lambda: torch.sum(x.view(2, -1, 32, c // 32), dim=(1, 3), out=o, dtype=torch.float32)

    def mk_k2():
        x = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        y = torch.empty_like(x)
        ws = ops.groupnorm_workspace(x)
        return lambda: ops.groupnorm_silu(x, gma, bta, out=y, workspace=ws)

    def mk_torch():
        x = torch.randn(2, c, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        return lambda: F.silu(F.group_norm(x, 32, gma.bfloat16(), bta.bfloat16(), 1e-5))
    r = {"shape": [2, c, hw, hw], "MB": nb / 1e6}
    for name, mk in [("copy", mk_copy), ("sum", mk_sum), ("k2", mk_k2), ("torch_gn_silu", mk_torch)]:
        try:
            r[name + "_us"] = round(timed(mk, nb), 2)
        except Exception as e:  # noqa: BLE001
            r[name + "_us"] = repr(e)[:80]
    print(json.dumps(r), flush=True)
