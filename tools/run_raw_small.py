"""Small mode-ii (LA_FLUSH_RAW) driver for compute-sanitizer: 2 slots, the
config-2 head shape, bf16 and fp32 records; a C = 22 cycle folded by the UT
kernel (two chunks), and a 40-token direct slot compressed by FORCE | RAW
(S0 = 0, three chunks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

R, C, Hk, Hv = 2, 22, 16, 32
for dt in ("bf16", "f32"):
    buf = L.LaBuf(L.make_config(R, Hk, Hv, chunk=C, keep_raw=True, in_dtype=dt, short_cap=64), device="cuda")
    buf.reset(zero_state=False)
    buf.state.copy_(sd.state0(1, R, Hv))
    xs = sd.tokens(10, R, C, Hk, Hv, in_dtype=dt)
    o = torch.empty(R, Hv, 128, device="cuda")
    for t in range(C):
        buf.decode_step(0, xs["q"][:, t].contiguous(), xs["k"][:, t].contiguous(), xs["v"][:, t].contiguous(),
                        xs["alpha"][:, t].contiguous(), xs["beta"][:, t].contiguous(), o)
    buf.flush(0, R, L.LA_FLUSH_FULL | L.LA_FLUSH_RAW)
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=False)
    p = sd.tokens(20, R, 40, Hk, Hv, in_dtype=dt)
    po = torch.empty(R, 40, Hv, 128, device="cuda")
    buf.direct_short(0, p["q"], p["k"], p["v"], p["alpha"], p["beta"], po)
    buf.flush(0, R, L.LA_FLUSH_FORCE | L.LA_FLUSH_RAW)
    torch.cuda.synchronize()
    assert torch.isfinite(buf.state).all()
print("ok")
