"""Print bench.py's per-kernel roofline rows alone (development aid)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
hbm, _, _ = bench.peaks()
for r in bench.other_kernels_roofline(hbm):
    print(json.dumps(r))
