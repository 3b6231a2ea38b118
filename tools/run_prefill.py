"""Profiling driver: chunked prefill of 256-token prompts at batch 64 (one
Qwen3-Next GDN layer, 64-token chunks): for `ncu -k regex:chunk_cta|fold`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

B, T = 64, 256
b = L.LaBuf(L.make_config(B, 16, 32, chunk=16, short_cap=64), device="cuda")
b.reset(zero_state=False)
b.state.copy_(sd.state0(1, B, 32))
x = sd.tokens(2, B, T, 16, 32)
o = torch.empty(B, T, 32, 128, device="cuda")
b.prefill(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
torch.cuda.synchronize()
print("ok")
