"""Summarise an ncu report: key metrics + SASS hotspots (stall samples).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--sass N]
"""
import csv
import io
import subprocess
import sys
import collections

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_misc_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        out.append(d)
    return h, rows[1], out


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 25
    h, units, kernels = raw(rep)
    u = dict(zip(h, units))
    for d in kernels:
        print("==", d.get("Kernel Name", "")[:120])
        for k in KEYS:
            if k in d:
                print(f"   {k:80s} {d[k]:>14s} {u.get(k, '')}")
    if nsass <= 0:
        return
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    hh = rows[hi]
    si, ns, ie = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    data = []
    for r in rows[hi + 1:]:
        if len(r) <= ie:
            continue
        try:
            data.append((r[0], float(r[ns] or 0), float(r[ie] or 0), r[si]))
        except ValueError:
            continue
    ts = sum(d[1] for d in data) or 1
    te = sum(d[2] for d in data) or 1
    print(f"-- SASS: {len(data)} instructions, {te:.0f} executed, {ts:.0f} stall samples")
    op = collections.Counter()
    ops = collections.Counter()
    for a, s, e, src in data:
        toks = src.split()
        o = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        o = o.split(".")[0]
        op[o] += e
        ops[o] += s
    for o, e in op.most_common(15):
        print(f"   {o:12s} {100 * e / te:5.1f}% inst {100 * ops[o] / ts:5.1f}% stall")
    print("-- hottest instructions by stall samples")
    for i, d in enumerate(sorted(data, key=lambda x: -x[1])[:nsass]):
        idx = data.index(d)
        print(f"   #{idx:5d} {100 * d[1] / ts:5.1f}% {d[2]:10.0f}  {d[3][:100]}")


if __name__ == "__main__":
    main()
