"""Per-CTA phase timeline of K7's persistent form (dev aid; probe build
-DSDB_XA_TRACE).  Slots: 0 entry, 1 TMEM allocated / barrier, 2 S_0 issued
(thread 0 waited K/V + Q_0), then per tile i: 3+4i S_i ready, 4+4i P_i
written, 5+4i epilogue of tile i-1 done; 15 last epilogue done (us from the
first CTA's entry)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_02031_b200 import ops  # noqa: E402

lib = ops._lib.lib()
names = ["entry", "alloc", "S0iss"] + [f"{p}{i}" for i in range(3) for p in ("S", "P", "ep", "-")]
names = names[:15] + ["end"]
for n, lq, c, h in [(2, 4096, 640, 10), (2, 1024, 1280, 20)]:
    q = torch.randn(n, lq, c, device="cuda").to(torch.bfloat16)
    kv = torch.randn(n, 77, 2 * c, device="cuda").to(torch.bfloat16)
    qt = (lq + 127) // 128
    total = qt * h * n
    ctas = min(total, 296)
    buf = (ctypes.c_ulonglong * (ctas * 16))()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for it in range(4):
        flush.zero_()
        torch.cuda.synchronize()
        ctypes.memset(buf, 0, ctypes.sizeof(buf))
        lib.sdb_debug_xa_trace(buf, ctas)   # clear: copy back zeros is not possible; mark with zeros below
        ops.cross_attention(q, kv, h)
        torch.cuda.synchronize()
        lib.sdb_debug_xa_trace(buf, ctas)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(ctas, 16).astype(np.int64)
    base = t[:, 0].min()
    line = f"[{n},{lq},{c}] ctas {ctas} tiles {total}:"
    for k, nm in enumerate(names):
        col = t[:, k]
        ok = col >= base
        if ok.sum() == 0:
            continue
        rel = (col[ok] - base) / 1000.0
        line += f" | {nm} {np.median(rel):.2f}/{rel.max():.2f}"
    print(line)
