"""Per-CTA phase timeline of K2's resident form (dev aid; needs the probe
build: make -C paper_2407_02031_b200/csrc NVFLAGS+=-DSDB_RS_TRACE).
Phases (globaltimer, ns from the first CTA's entry): 0 entry, 1 after the PDL
wait, 2 statistics of the landed tile done, 3 partials published (arrive),
4 grid barrier passed, 5 apply + stores issued."""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

lib = ops._lib.lib()
for shape in sys.argv[1:] or ["2,320,128,128", "2,640,32,32"]:
    n, c, h, w = [int(v) for v in shape.split(",")]
    x = torch.randn(n, c, h, w, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    y = torch.empty_like(x)
    gm, bt = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda")
    ws = ops.groupnorm_workspace(x)
    plan = (ctypes.c_int * 4)()
    lib.sdb_groupnorm_resident_plan(n, h * w, c, 32, plan)
    ctas = plan[3]
    buf = (ctypes.c_ulonglong * (ctas * 16))()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for it in range(6):
        if os.environ.get("NOFLUSH") != "1":
            flush.zero_()
        torch.cuda.synchronize()
        with ops.groupnorm_mode(4):
            for _ in range(int(os.environ.get("BACK2BACK", "1"))):   # the last launch is traced
                ops.groupnorm_silu(x, gm, bt, out=y, workspace=ws, silu=os.environ.get("SILU", "1") == "1")
        torch.cuda.synchronize()
        lib.sdb_debug_rs_trace(buf, ctas)
        t = np.frombuffer(buf, dtype=np.uint64).reshape(ctas, 16).astype(np.int64)
        if it >= 2:
            rows.append(t)
    print(f"[{shape}] plan {list(plan)}")
    for t in rows:
        base = t[:, 0].min()
        rel = (t[:, :7] - base) / 1000.0
        q = lambda k: f"{np.min(rel[:, k]):6.2f}/{np.median(rel[:, k]):6.2f}/{np.max(rel[:, k]):6.2f}"
        print("  entry " + q(0) + " | pdl " + q(1) + " | stats " + q(2) + " | fold " + q(6) + " | arrive " + q(3) + " | passed " + q(4) +
              " | done " + q(5) + f" | sms {len(set(t[:, 15].tolist()))}")
