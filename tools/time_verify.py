"""Time verify (kernel 3) at batch 256 for N drafts in {2, 4, 8} (CUDA events,
2 layer instances rotated, after warm-up).  LABUF_TC=0/1 selects the CUDA-core
or tensor-core state pass.  Prints: N, us per verify launch, algorithmic GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import cost
from paper_2605_19049_b200 import labuf as L

B, Hk, Hv, NL = 256, 16, 32, 2
lb = cost.LayerBytes.make(Hk, Hv, 128, 2, 4)
for N in (2, 4, 8):
    bufs = [L.LaBuf(L.make_config(B, Hk, Hv, chunk=16, max_drafts=N), device="cuda") for _ in range(NL)]
    for i, b in enumerate(bufs):
        b.reset(zero_state=False)
        b.state.copy_(sd.state0(i, B, Hv))
    torch.cuda.synchronize()
    xs = [sd.tokens(5 + i, B, N, Hk, Hv) for i in range(NL)]
    o = torch.empty(B, N, Hv, 128, device="cuda")
    res = []
    for nacc in (0, N):
        na = torch.full((B,), nacc, dtype=torch.int32, device="cuda")
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(10 * NL)]
        def rnd(k0):
            for i, (b, x) in enumerate(zip(bufs, xs)):
                e = ev[k0 + i]
                e[0].record()
                b.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
                e[1].record()
                b.commit_accepted(0, na)
                e[2].record()
        for _ in range(3):
            rnd(0)
        torch.cuda.synchronize()
        for k in range(10):
            rnd(k * NL)
        torch.cuda.synchronize()
        tv = sorted(e[0].elapsed_time(e[1]) for e in ev)[len(ev) // 2] * 1e3
        tc = sorted(e[1].elapsed_time(e[2]) for e in ev)[len(ev) // 2] * 1e3
        res += [round(tv, 1), round(tc, 1)]
    print("N", N, "verify_us", res[0], "commit0_us", res[1], "| verify_us", res[2], f"commit{N}_us", res[3], flush=True)
    del bufs
    torch.cuda.empty_cache()
