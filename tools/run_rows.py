"""Profiling driver for the config-3 / config-4 kernels:
  python tools/run_rows.py verify   -- batch 256, 4 drafts: verify + commit, x reps
  python tools/run_rows.py direct   -- batch 1024, context 64: direct decode steps
  python tools/run_rows.py rverify  -- batch 256, 4 drafts: recurrent verify + copy commit
(for `ncu -k regex:chunk_cta` / `regex:fold`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

what = sys.argv[1] if len(sys.argv) > 1 else "verify"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
Hk, Hv = 16, 32
if what == "verify":
    B, N = 256, 4
    buf = L.LaBuf(L.make_config(B, Hk, Hv, chunk=16, max_drafts=N), device="cuda")
    buf.reset(zero_state=False)
    buf.state.copy_(sd.state0(1, B, Hv))
    x = sd.tokens(5, B, N, Hk, Hv)
    o = torch.empty(B, N, Hv, 128, device="cuda")
    na = sd.n_accepted(6, B, N)
    for _ in range(reps):
        buf.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
        buf.commit_accepted(0, na)
elif what == "rverify":
    B, N = 256, 4
    buf = L.LaBuf(L.make_config(B, Hk, Hv, chunk=16, max_drafts=N), device="cuda")
    buf.reset(zero_state=False)
    buf.state.copy_(sd.state0(1, B, Hv))
    x = sd.tokens(5, B, N, Hk, Hv)
    o = torch.empty(B, N, Hv, 128, device="cuda")
    temp = torch.empty(B, N, Hv, 128, 128, device="cuda")
    na = sd.n_accepted(6, B, N)
    for _ in range(reps):
        buf.recurrent_verify(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], temp, o)
        buf.recurrent_commit(0, na, temp)
else:
    B, L0 = 1024, 64
    buf = L.LaBuf(L.make_config(B, Hk, Hv, chunk=16, short_cap=128, u_dtype="f16"), device="cuda")
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=False)
    pre = sd.tokens(5, B, L0, Hk, Hv)
    o = torch.empty(B, L0, Hv, 128, device="cuda")
    buf.direct_short(0, pre["q"], pre["k"], pre["v"], pre["alpha"], pre["beta"], o)
    o1 = torch.empty(B, 1, Hv, 128, device="cuda")
    for t in range(reps):
        x = sd.tokens(10 + t, B, 1, Hk, Hv)
        buf.direct_short(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o1)
torch.cuda.synchronize()
print("ok")
