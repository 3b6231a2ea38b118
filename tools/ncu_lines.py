"""Per-source-line warp-stall samples of an ncu report (needs -lineinfo and
--import-source on):  python tools/ncu_lines.py x.ncu-rep [top N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
lines, tot = [], 0
for r in rows[rows.index(hdr) + 1:]:
    if r and r[0] and r[0] != "Line No":
        try:
            v = int(r[iS])
        except (ValueError, IndexError):
            continue
        tot += v
        ins = r[iI] if iI is not None and iI < len(r) else ""
        lines.append((v, r[0], r[1].strip()[:100], ins))
lines.sort(reverse=True)
print(f"total stall samples {tot}")
for v, ln, src, ins in lines[:top]:
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}%  inst {ins:>10s}  L{ln}: {src}")
