"""Phase timeline of the mode-ii kernel (CTA 0, warps 0 and 6, first 8 units or CTAs 0..7)
from a -DLABUF_UT_PROF build (LABUF_LIB=ab/liblabuf_prof.so)."""
import ctypes, os, subprocess, sys
sys.argv = [sys.argv[0]]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "time_raw_flush.py")).read())
from paper_2605_19049_b200 import labuf as L
lib = ctypes.CDLL(os.environ["LABUF_LIB"])
buf = (ctypes.c_longlong * (2 * 8 * 12))()
print("rc", lib.la_debug_ut_prof(buf))
names = ["start", "loaded", "gram", "inv", "ktvt", "S", "ugemm", "fold", "end", "-"]
for w in range(2):
    for k in range(8):
        row = [buf[(w * 8 + k) * 12 + i] for i in range(10)]
        base = row[0]
        print("warp", 6 * w, "unit", k, " ".join(f"{n}={(x - base):6d}" for n, x in zip(names, row)))
