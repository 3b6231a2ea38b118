"""Profiling driver: config-2 batch (64 slots, C = 16, keep_raw) -- one decode
cycle then one LA_FLUSH_RAW (mode ii) flush, repeated; the only fold kernels
launched are mode-ii ones (for `ncu -k regex:fold_kernel`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

B, C, Hk, Hv = 64, 16, 16, 32
buf = L.LaBuf(L.make_config(B, Hk, Hv, chunk=C, keep_raw=True), device="cuda")
buf.reset(zero_state=False)
buf.state.copy_(sd.state0(1, B, Hv))
xs = [sd.tokens(10 + t, B, 1, Hk, Hv, squeeze=True) for t in range(C)]
o = torch.empty(B, Hv, 128, device="cuda")
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    for x in xs:
        buf.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
    buf.flush(0, B, L.LA_FLUSH_FULL | L.LA_FLUSH_RAW)
torch.cuda.synchronize()
print("ok")
