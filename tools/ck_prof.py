"""Per-CTA timeline of one config-2 decode launch (batch 64, C = 16, bf16,
occupancy j after warm-up), or of one config-3 verify launch (batch 256,
N drafts, empty buffers) from a -DLABUF_CK_PROF build:
    LABUF_LIB=ab/liblabuf_ckprof.so python tools/ck_prof.py [j | verify N]
Prints the launch span, per-phase latency percentiles and the CTAs resident
per SM over time."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

C, Hk, Hv = 16, 16, 32
reader = "la_debug_ck_prof"
if len(sys.argv) > 2 and sys.argv[1] == "direct":   # config 4: batch 1024, context L0 -> L0 + 1
    L0 = int(sys.argv[2])
    B, reader = 1024, "la_debug_ck_prof_direct"
    b4 = L.LaBuf(L.make_config(B, Hk, Hv, chunk=16, short_cap=128, u_dtype="f16"), device="cuda")
    b4.reset(mode=L.LA_MODE_DIRECT, zero_state=False)
    pre = sd.tokens(30, B, L0, Hk, Hv)
    po = torch.empty(B, L0, Hv, 128, device="cuda")
    b4.direct_short(0, pre["q"], pre["k"], pre["v"], pre["alpha"], pre["beta"], po)
    x = sd.tokens(40, B, 1, Hk, Hv)
    o = torch.empty(B, 1, Hv, 128, device="cuda")
    b4.direct_short(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
elif len(sys.argv) > 2 and sys.argv[1] == "verify":
    N = int(sys.argv[2])
    B, j = 256, 0
    bufs = [L.LaBuf(L.make_config(B, Hk, Hv, chunk=C, max_drafts=N), device="cuda") for _ in range(2)]
    for i, b in enumerate(bufs):
        b.reset(zero_state=False)
        b.state.copy_(sd.state0(i, B, Hv))
    x = sd.tokens(10, B, N, Hk, Hv)
    o = torch.empty(B, N, Hv, 128, device="cuda")
    na = torch.zeros(B, dtype=torch.int32, device="cuda")
    for rep in range(3):
        for b in bufs:
            b.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
            if rep < 2:
                b.commit_accepted(0, na)
else:
    B = 64
    j = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    bufs = [L.LaBuf(L.make_config(B, Hk, Hv, chunk=C), device="cuda") for _ in range(4)]
    for i, b in enumerate(bufs):
        b.reset(zero_state=False)
        b.state.copy_(sd.state0(i, B, Hv))
    xs = [sd.tokens(10 + t, B, 1, Hk, Hv, squeeze=True) for t in range(C)]
    o = torch.empty(B, Hv, 128, device="cuda")
    for t in range(j + 1):   # the last launch runs at occupancy j (4 handles rotated: L2 holds none of the state)
        for b in bufs:
            b.decode_step(0, xs[t]["q"], xs[t]["k"], xs[t]["v"], xs[t]["alpha"], xs[t]["beta"], o)
torch.cuda.synchronize()
if "LABUF_LIB" not in os.environ:   # (driver for an ncu capture of the same launches)
    sys.exit(0)
lib = ctypes.CDLL(os.environ["LABUF_LIB"])
raw = (ctypes.c_ulonglong * (8192 * 9))()
assert getattr(lib, reader)(raw) == 0
a = np.frombuffer(raw, dtype=np.uint64).reshape(8192, 9).astype(np.int64)
a = a[a[:, 0] > 0]
a = a[a[:, 0] >= a[:, 0].max() - 10**6]   # the last launch
t0 = a[:, 0].min()
st, land, recs, end, sm = a[:, 0] - t0, a[:, 1] - t0, a[:, 2] - t0, a[:, 3] - t0, a[:, 8]
sland, spass, presub, postsub = a[:, 4] - t0, a[:, 5] - t0, a[:, 6] - t0, a[:, 7] - t0
print(f"{' '.join(sys.argv[1:])}: {len(a)} CTAs, span {end.max() / 1e3:.2f} us (first start 0, last start {st.max() / 1e3:.2f})")
for name, x in (("load (state+tokens)", land - st), ("records after state", recs - land), ("compute after records", end - recs),
                ("CTA life", end - st)) + ((("state landed (MMA)", sland - st), ("state pass", spass - sland),
                ("to substitution", presub - spass), ("substitution", postsub - presub), ("stores + exit", end - postsub))
                if a[:, 4].min() > 0 else ()):
    p = np.percentile(x, [5, 50, 95]) / 1e3
    print(f"  {name:24s} p5 {p[0]:.2f}  p50 {p[1]:.2f}  p95 {p[2]:.2f} us")
# resident CTAs per SM, sampled every 0.5 us
grid = np.arange(0, end.max(), 500)
res = [(np.sum((st <= g) & (end > g)) / len(np.unique(sm))) for g in grid]
print("  resident CTAs per SM every 0.5 us:", " ".join(f"{x:.1f}" for x in res))
loading = [(np.sum((st <= g) & (land > g)) / len(np.unique(sm))) for g in grid]
print("  CTAs waiting for the state per SM:  ", " ".join(f"{x:.1f}" for x in loading))
