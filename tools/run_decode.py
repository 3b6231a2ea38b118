"""Profiling driver, config-2 shapes (batch 64, C = 16, bf16 q/k/v, fp32
state): `reps` buffer cycles (16 buffered decode launches + the FULL flush)
followed by 16 recurrent steps; for `ncu -k regex:chunk_cta|fold|recurrent_step`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

B, C, Hk, Hv = 64, 16, 16, 32
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
fused = len(sys.argv) > 2 and sys.argv[2] == "fused"
buf = L.LaBuf(L.make_config(B, Hk, Hv, chunk=C), device="cuda")
buf.set_auto_flush(fused)
buf.reset(zero_state=False)
buf.state.copy_(sd.state0(1, B, Hv))
xs = [sd.tokens(10 + t, B, 1, Hk, Hv, squeeze=True) for t in range(C)]
o = torch.empty(B, Hv, 128, device="cuda")
for _ in range(reps):
    for x in xs:
        buf.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
    buf.flush(0, B, L.LA_FLUSH_FULL)
for x in xs:
    buf.recurrent_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
torch.cuda.synchronize()
print("ok")
