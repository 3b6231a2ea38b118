"""Config-5 driver for a launch list: the 36-layer mixed stack (MixedStack,
one paged handle per layer) on this GPU, warm-up, then `steps` timed stack
steps (CUDA events) -- python tools/run_config5.py [steps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth.device as sd
from paper_2605_19049_b200.stack import MixedStack, StackSpec, short_groups

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda")
spec = StackSpec(n_layers=36, n_long=1536, n_short=512)
Hk, Hv = spec.n_qk_heads, spec.n_v_heads
st = MixedStack.create(spec, dev, state_headroom=max(1, spec.n_short // len(spec.short_l0)))
st.reset(lambda l, view: sd.fill_state0(view, 7 + l))
for b in st.layers:
    b.set_overlap(True)
xs4 = [sd.tokens(100 + l, 2048, 1, Hk, Hv, squeeze=True) for l in range(4)]
xin = [xs4[l % 4] for l in range(36)]
o1 = torch.empty(2048, Hv, 128, device=dev)
pre = {}


def short_tok(l, g):
    f, m, l0 = short_groups(spec)[g]
    if (m, l0) not in pre:
        pre[(m, l0)] = sd.tokens(300 + l0, m, l0, Hk, Hv)
    return pre[(m, l0)]


st.warmup(lambda l, t: {k: v[:spec.n_long] for k, v in xin[l].items()}, short_tok)
pre.clear()
st.step(xin, [o1] * 36)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    st.step(xin, [o1] * 36)
e1.record()
torch.cuda.synchronize()
print(f"config5: {e0.elapsed_time(e1) / steps:.2f} ms per stack step")
