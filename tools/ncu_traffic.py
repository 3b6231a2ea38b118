"""Write profiles/ncu_traffic.json (DRAM bytes per launch of each hot-path
kernel) and a per-kernel summary CSV from `ncu --set full` reports.

    python tools/ncu_traffic.py OUT_DIR decode=rep1.ncu-rep flush=rep2.ncu-rep ...

bench.py reads ncu_traffic.json for the roofline "traffic" field.  Each
report holds 1-2 launches of one kernel; the per-launch mean is recorded.
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    return [dict(zip(h, x)) for x in r[2:]], dict(zip(h, units))


def num(v, unit):
    return float(v.replace(",", "")) * SCALE.get(unit, 1.0)


def main():
    out_dir = sys.argv[1]
    traffic, summary = {}, []
    for arg in sys.argv[2:]:
        key, rep = arg.split("=", 1)
        launches, units = rows(rep)
        if not launches:
            continue
        rd = [num(l["dram__bytes_read.sum"], units["dram__bytes_read.sum"]) for l in launches]
        wr = [num(l["dram__bytes_write.sum"], units["dram__bytes_write.sum"]) for l in launches]
        us = [num(l["gpu__time_duration.sum"], units["gpu__time_duration.sum"]) for l in launches]
        traffic[key] = {"dram_bytes": sum(rd) / len(rd) + sum(wr) / len(wr),
                        "dram_read_bytes": sum(rd) / len(rd), "dram_write_bytes": sum(wr) / len(wr),
                        "ncu_us": sum(us) / len(us), "kernel": launches[0].get("Kernel Name", "")[:160],
                        "report": os.path.basename(rep)}
        for l in launches:
            summary.append([key, l.get("Kernel Name", "")[:100]] + [f"{l.get(k, '')} {units.get(k, '')}".strip() for k in KEYS])
    with open(os.path.join(out_dir, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    with open(os.path.join(out_dir, "ncu_summary.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["key", "kernel"] + KEYS)
        w.writerows(summary)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
