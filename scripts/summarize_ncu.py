"""Summarise ncu outputs into profiles/ (development aid).

  python scripts/summarize_ncu.py launches <launches.csv> > profiles/<name>.md
  python scripts/summarize_ncu.py full <report.ncu-rep> > profiles/<name>.md
"""

import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "dram__bytes_write.sum.per_second", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        key = r[ki].split("(")[0][:100]
        tot[key] += v
        cnt[key] += 1
    T = sum(tot.values())
    ours = sum(v for k, v in tot.items() if "sdb::" in k)
    print(f"Source: `{path}` — every launch, `ncu --metrics gpu__time_duration.sum --clock-control none` "
          f"(serialised one launch at a time: compare SHARES, not the step time).\n")
    print(f"Total {T:.3f} ms over {sum(cnt.values())} launches; this repo's kernels (sdb::) "
          f"{ours:.3f} ms = {100 * ours / T:.1f}%.\n")
    print("| ms | share | launches | kernel |\n|---:|---:|---:|---|")
    for k, v in tot.most_common(30):
        print(f"| {v:.3f} | {100 * v / T:.1f}% | {cnt[k]} | `{k}` |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2:]
    print(f"Source: `{path}` — `ncu --set full --clock-control none --import-source on`.\n")
    for v in vals:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"### `{name[:120]}`\n\n| metric | value | unit |\n|---|---:|---|")
        for i, k in enumerate(h):
            if k in FULL_METRICS:
                print(f"| {k} | {v[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
