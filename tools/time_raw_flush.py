"""Time flush mode ii (LA_FLUSH_RAW) at config 2 (batch 64, C = 16, keep_raw),
4 layer instances rotated: CUDA events around each flush, after warm-up.
Prints us per flush launch (median) and the algorithmic GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

B, C, Hk, Hv, NL = 64, 16, 16, 32, 4
kind = L.LA_FLUSH_FULL | (0 if "--mode-i" in sys.argv else L.LA_FLUSH_RAW)
bufs = [L.LaBuf(L.make_config(B, Hk, Hv, chunk=C, keep_raw=True), device="cuda") for _ in range(NL)]
for i, b in enumerate(bufs):
    b.reset(zero_state=False)
    b.state.copy_(sd.state0(i, B, Hv))
xs = [sd.tokens(10 + t, B, 1, Hk, Hv, squeeze=True) for t in range(C)]
o = torch.empty(B, Hv, 128, device="cuda")
ts = []
for rep in range(8):
    for b in bufs:
        for x in xs:
            b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
    for b in bufs:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.flush(0, B, kind)
        e1.record()
        if rep >= 2:
            ts.append((e0, e1))
torch.cuda.synchronize()
us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)[len(ts) // 2]
byt = B * Hv * (2 * 128 * 128 * 4) + B * C * (Hk * 128 * 2 + Hv * 128 * 2 + 8 * Hv)
print(f"flush {'mode i' if '--mode-i' in sys.argv else 'mode ii'}: {us:.1f} us, {byt / us / 1e3:.0f} GB/s")
