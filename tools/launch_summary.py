"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel launches, mean and total device time, share.  The bench step
(buffered decode + flush) share is reported separately.

    python tools/launch_summary.py launches.csv > summary.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi and r[vi]:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print("kernel,launches,mean_us,total_us,share_of_all_pct")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"\"{k}\",{len(v)},{sum(v) / len(v):.2f},{sum(v):.1f},{100 * sum(v) / tot:.1f}")
dec = [v for k, v in agg.items() if k.startswith("void chunk_cta_kernel<__nv_bfloat16, float, 2, 1, 1, 1")]
fl = [v for k, v in agg.items() if "fold_kernel<__nv_bfloat16, float" in k]
if dec and fl:
    d, f = sum(dec[0]) / len(dec[0]), sum(fl[0]) / len(fl[0])
    print(f"# bench step (16 decode launches + 1 flush per layer): decode share {100 * 16 * d / (16 * d + f):.1f}%, "
          f"flush share {100 * f / (16 * d + f):.1f}% (ncu: cold-cache, serialised)")
