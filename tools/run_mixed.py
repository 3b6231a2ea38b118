"""A small paged, state-pooled handle driven through la_decode_mixed
(chunkwise decode + eager flush, KV-only decode, compression at short_cap),
verify + append commit, and a state fork: for compute-sanitizer and ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth.device as sd
from paper_2605_19049_b200 import labuf as L

Hk, Hv, R = 16, 32, 8
cfg = L.make_config(R, Hk, Hv, chunk=8, max_drafts=4, short_cap=16, block_tokens=8, n_blocks=R * 2 + 4,
                    state_slots=8, validate=True)
b = L.LaBuf(cfg, device="cuda")
b.set_overlap(True)
b.reset(0, 4, mode=L.LA_MODE_CHUNKWISE, zero_state=True)
b.reset(4, 4, mode=L.LA_MODE_DIRECT, zero_state=False)
for step in range(20):
    x = sd.tokens(100 + step, R, 1, Hk, Hv, squeeze=True)
    o = torch.empty(R, Hv, 128, device="cuda")
    b.decode_mixed(np.random.default_rng(step).permutation(R), x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
torch.cuda.synchronize()
b.flush(0, R, L.LA_FLUSH_FORCE)
x = sd.tokens(7, 4, 4, Hk, Hv)
o = torch.empty(4, 4, Hv, 128, device="cuda")
b.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
b.commit_append(0, sd.n_accepted(8, 4, 4))
b.flush(0, 4, L.LA_FLUSH_FORCE)
flags, _ = b.device_status()
print("ok, status", flags, b.pool_info())
