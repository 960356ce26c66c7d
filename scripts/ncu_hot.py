"""Top stall lines of an ncu --set full capture (source page): dev aid.
usage: python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[i_s]) for r in data) or 1
print("total samples", tot)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {}
for r in data:
    for h in reasons:
        v = r[hdr.index(h)]
        if v.isdigit():
            agg[h] = agg.get(h, 0) + int(v)
print("stall totals:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for r in sorted(data, key=lambda r: -int(r[i_s]))[:top_n]:
    rs = sorted(((int(r[hdr.index(h)]) if r[hdr.index(h)].isdigit() else 0, h[6:]) for h in reasons), reverse=True)[:2]
    print(r[0][-5:], r[1].strip()[:60].ljust(60), f"{int(r[i_s]) / tot:6.1%}", rs)
