"""Config 5 (BASELINE.json configs[4]) at full batch: a stack of Qwen3-Next
GDN layers serving 2048 mixed requests -- 1536 long-context slots (buffered
decode, C = 16, occupancies staggered over 0..15 so flushes spread over the
cycle) and 512 short ones (KV-only decode, no state, L0 in {16, 40, 64, 96}).
Two layers here (the layer count changes nothing per layer; bench/tools run
the 36-layer stack); 17 decode steps so every long group folds at least once.
Sampled slots of every group are recomputed by the fp64 oracle one by one and
compared in full (all heads, every output, the long slots' final states);
every output of the whole batch is checked finite."""
import numpy as np
import pytest
import torch

import synth.device as sd
from harness import TOL, Oracle, assert_close
from paper_2605_19049_b200 import labuf as L
from paper_2605_19049_b200.stack import GdnStack, StackSpec, long_groups, short_groups

pytestmark = pytest.mark.gpu

HK, HV = 16, 32
N_STEPS = 17


def _seed(kind, l, t):
    return 50000 + 1000 * l + (0 if kind == "long" else 500) + t


def test_config5_mixed_batch_stack(cuda_device):
    spec = StackSpec(n_layers=2)
    st = GdnStack.create(spec, cuda_device)
    lg, sg = long_groups(spec), short_groups(spec)
    occ0 = np.concatenate([[occ] * m for _, m, occ in lg])
    # sampled slots: first and last of every long group, one per short group + the ends
    long_sample = sorted({f for f, m, _ in lg} | {f + m - 1 for f, m, _ in lg})
    short_sample = sorted({f + m // 2 for f, m, _ in sg} | {0, spec.n_short - 1})
    S0 = [sd.state0(40000 + l, spec.n_long, HV, device=cuda_device) for l in range(spec.n_layers)]
    st.reset(S0)
    orc_long = [Oracle(S0[l][long_sample].double().cpu().numpy()) for l in range(spec.n_layers)]
    orc_short = [Oracle(np.zeros((len(short_sample), HV, 128, 128))) for _ in range(spec.n_layers)]
    tol = TOL["bf16"]

    def long_tok(l, t):
        return sd.tokens(_seed("long", l, t), spec.n_long, 1, HK, HV, device=cuda_device, squeeze=True)

    short_pre = {}

    def short_tok(l, g):
        f, m, l0 = sg[g]
        short_pre[(l, g)] = sd.tokens(_seed("short", l, 100 + g), m, l0, HK, HV, device=cuda_device)
        return short_pre[(l, g)]

    warm_long = {(l, t): long_tok(l, t) for l in range(spec.n_layers) for t in range(spec.chunk - 1)}
    outs = st.warmup(lambda l, t: warm_long[(l, t)], short_tok)
    torch.cuda.synchronize()
    # warm-up outputs of the sampled slots
    for l in range(spec.n_layers):
        for t in range(spec.chunk - 1):
            first, o = outs[("long", l, t)]
            idx = [i for i, s in enumerate(long_sample) if occ0[s] > t]
            if not idx:
                continue
            sl = [long_sample[i] for i in idx]
            tok = sd.host_tokens({k: v.unsqueeze(1) for k, v in warm_long[(l, t)].items()}, sl)
            ref = orc_long[l].run(idx, tok)
            assert_close(o[[s - first for s in sl]].cpu().numpy(), ref[:, 0], tol, f"layer {l} warm-up {t}")
        for g, (f, m, l0) in enumerate(sg):
            first, o = outs[("short", l, g)]
            idx = [i for i, s in enumerate(short_sample) if f <= s < f + m]
            if idx:
                sl = [short_sample[i] - f for i in idx]
                ref = orc_short[l].run(idx, sd.host_tokens(short_pre[(l, g)], sl))
                assert_close(o[sl].cpu().numpy(), ref, tol, f"layer {l} short prefill group {g}")
    for l in range(spec.n_layers):
        info = [st.layers[l].long.slot_info(s).occ for s in range(spec.n_long)]
        assert info == occ0.tolist()

    long_out = [torch.empty(spec.n_long, HV, 128, dtype=torch.float32, device=cuda_device) for _ in range(spec.n_layers)]
    short_out = [torch.empty(spec.n_short, 1, HV, 128, dtype=torch.float32, device=cuda_device) for _ in range(spec.n_layers)]
    for t in range(N_STEPS):
        li = [long_tok(l, 100 + t) for l in range(spec.n_layers)]
        si = [sd.tokens(_seed("short", l, t), spec.n_short, 1, HK, HV, device=cuda_device) for l in range(spec.n_layers)]
        st.step(li, si, long_out, short_out)
        torch.cuda.synchronize()
        for l in range(spec.n_layers):
            assert torch.isfinite(long_out[l]).all() and torch.isfinite(short_out[l]).all()
            tok = sd.host_tokens({k: v.unsqueeze(1) for k, v in li[l].items()}, long_sample)
            ref = orc_long[l].run(np.arange(len(long_sample)), tok)
            assert_close(long_out[l][long_sample].cpu().numpy(), ref[:, 0], tol, f"layer {l} step {t} long")
            ref = orc_short[l].run(np.arange(len(short_sample)), sd.host_tokens(si[l], short_sample))
            assert_close(short_out[l][short_sample].cpu().numpy(), ref, tol, f"layer {l} step {t} short")
    for l in range(spec.n_layers):
        lay = st.layers[l]
        assert [lay.long.slot_info(s).occ for s in range(spec.n_long)] == ((occ0 + N_STEPS) % spec.chunk).tolist()
        assert [lay.short.slot_info(s).len for s in range(spec.n_short)] == \
            [l0 + N_STEPS for f, m, l0 in sg for _ in range(m)]
        lay.long.flush(0, spec.n_long, L.LA_FLUSH_FORCE)
        for i, s in enumerate(long_sample):
            assert_close(lay.long.state[s].cpu().numpy(), orc_long[l].S[i], tol, f"layer {l} slot {s} final state")
        flags, _ = lay.long.device_status()
        assert flags == 0
