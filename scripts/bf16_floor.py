"""Writes profiles/r02_bf16_floor.txt: the latent error of bf16 rounding at
chosen sites of the toy oracle (oracle/bf16_floor.py), CPU only."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import bf16_floor as B  # noqa: E402

cfg, up, cps, req = B.toy_inputs()
tab = B.floor_table(cfg, up, cps, req)
lines = ["# bf16 rounding sites vs the fp32 oracle — toy config 1 (20 DDIM steps, CFG 7.5, 1 ControlNet)",
         "# per-step latent rel-L2 (steps 1, 5, 10, 15, 20); every other op fp32; eps stays fp32", ""]
for label, errs in tab.items():
    lines.append(f"{label:24s} " + "  ".join(f"{errs[i]:.2e}" for i in (0, 4, 9, 14, 19)) +
                 f"   max {max(errs):.2e}")
text = "\n".join(lines) + "\n"
print(text)
(ROOT / "profiles" / "r02_bf16_floor.txt").write_text(text)
