"""GPU parity at the BASELINE.json sizes, in the launch configuration bench.py
times (whole batch per call, decode cycle captured as a CUDA graph), checked
on sampled slots that the fp64 oracle recomputes one by one (DESIGN.md
"Parity").  Inputs come from the seeded device generator (synth.device); the
oracle gets the sampled slots' stored values.  Tolerance: the north-star
max-abs 2e-3 (bf16 q/k/v, fp32 state)."""
import numpy as np
import pytest
import torch

import synth.device as sd
from harness import TOL, Oracle, assert_close, make_buf
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV = 16, 32


def _capture(fn, stream):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def test_config2_full_batch_graph_cycle(cuda_device):
    """Config 2: Qwen3-Next GDN layer, batch 64, C = 16, synthetic 32K-context
    states; one captured cycle (16 decode steps + FULL flush) replayed twice,
    every output and the post-flush state of ALL 64 slots vs the oracle."""
    B, C = 64, 16
    sample = list(range(B))
    buf = make_buf(B, HK, HV, C=C, validate=False)
    buf.reset(zero_state=False)
    S0 = sd.state0(2002, B, HV, device=cuda_device)
    buf.state.copy_(S0)
    orc = Oracle(S0[sample].double().cpu().numpy())
    toks = [sd.tokens(3000 + t, B, 1, HK, HV, device=cuda_device, squeeze=True) for t in range(2 * C)]
    outs = [torch.empty(B, HV, 128, dtype=torch.float32, device=cuda_device) for _ in range(2 * C)]
    stream = torch.cuda.Stream(device=cuda_device)
    torch.cuda.synchronize()

    def cycle(c):
        def fn():
            for t in range(C):
                x = toks[c * C + t]
                buf.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], outs[c * C + t])
            buf.flush(0, B, L.LA_FLUSH_FULL)
        return fn

    graphs = [_capture(cycle(c), stream) for c in range(2)]
    for c in range(2):
        graphs[c].replay()
        torch.cuda.synchronize()
        for t in range(C):
            ref = orc.run(np.arange(len(sample)), sd.host_tokens(toks[c * C + t], sample))
            assert_close(outs[c * C + t][sample].cpu().numpy(), ref[:, 0], TOL["bf16"], f"cycle {c} step {t}")
        for i, s in enumerate(sample):
            assert_close(buf.state[s].cpu().numpy(), orc.S[i], TOL["bf16"], f"cycle {c} slot {s} state")
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [0] * B


@pytest.mark.parametrize("N", [4, 8])
def test_config3_full_batch_verify_commit(cuda_device, N):
    """Config 3: batch 256, 4 drafts (8: the tensor-core state pass), parallel
    verify + accepted-prefix commit with p_accept = 0.7, three rounds after a
    3-token decode prefix; sampled slots cover every n_acc value."""
    B, C = 256, 16
    buf = make_buf(B, HK, HV, C=C, N=N, validate=False)
    buf.reset(zero_state=False)
    S0 = sd.state0(2003, B, HV, device=cuda_device)
    buf.state.copy_(S0)
    o1 = torch.empty(B, HV, 128, dtype=torch.float32, device=cuda_device)
    pre = [sd.tokens(4000 + t, B, 1, HK, HV, device=cuda_device, squeeze=True) for t in range(3)]
    rounds = [sd.tokens(5000 + r, B, N, HK, HV, device=cuda_device) for r in range(3)]
    naccs = [sd.n_accepted(6000 + r, B, N, device=cuda_device) for r in range(3)]
    na0 = naccs[0].cpu().numpy()
    sample = sorted({int(np.flatnonzero(na0 == v)[0]) for v in range(N + 1) if (na0 == v).any()} | {0, B - 1})
    orc = Oracle(S0[sample].double().cpu().numpy())
    idx = np.arange(len(sample))
    for t in range(3):
        x = pre[t]
        buf.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o1)
        ref = orc.run(idx, sd.host_tokens(x, sample))
        assert_close(o1[sample].cpu().numpy(), ref[:, 0], TOL["bf16"], f"prefix decode {t}")
    o = torch.empty(B, N, HV, 128, dtype=torch.float32, device=cuda_device)
    for rnd in range(3):
        x = rounds[rnd]
        na = naccs[rnd]
        buf.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
        buf.commit_accepted(0, na)
        torch.cuda.synchronize()
        ref = orc.run(idx, sd.host_tokens(x, sample), n_acc=na.cpu().numpy()[sample])
        assert_close(o[sample].cpu().numpy(), ref, TOL["bf16"], f"round {rnd} drafts")
        for i, s in enumerate(sample):
            assert_close(buf.state[s].cpu().numpy(), orc.S[i], TOL["bf16"], f"round {rnd} slot {s} committed")
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [0] * B


def test_config4_full_batch_direct(cuda_device):
    """Config 4: batch 1024 short contexts, direct KV-only decoding with no
    state: ragged prefills (8 groups of 128 slots, L0 = 16..72) then 8 decode
    steps of the whole batch; one sampled slot per group plus the ends."""
    B, G = 1024, 8
    per = B // G
    L0s = [16 + 8 * i for i in range(G)]
    buf = make_buf(B, HK, HV, C=16, short_cap=128, u_dtype="f16", validate=False)
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=False)
    sample = sorted({gi * per + 5 for gi in range(G)} | {0, B - 1})
    orc = Oracle(np.zeros((len(sample), HV, 128, 128)))
    for gi, L0 in enumerate(L0s):
        x = sd.tokens(7000 + gi, per, L0, HK, HV, device=cuda_device)
        o = torch.empty(per, L0, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.direct_short(gi * per, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
        torch.cuda.synchronize()
        mine = [(i, s - gi * per) for i, s in enumerate(sample) if gi * per <= s < (gi + 1) * per]
        for i, loc in mine:
            ref = orc.run([i], sd.host_tokens(x, [loc]))
            assert_close(o[loc].cpu().numpy(), ref[0], TOL["bf16"], f"prefill group {gi} slot {loc}")
    o1 = torch.empty(B, 1, HV, 128, dtype=torch.float32, device=cuda_device)
    for t in range(8):
        x = sd.tokens(8000 + t, B, 1, HK, HV, device=cuda_device)
        buf.direct_short(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o1)
        torch.cuda.synchronize()
        ref = orc.run(np.arange(len(sample)), sd.host_tokens(x, sample))
        assert_close(o1[sample].cpu().numpy(), ref, TOL["bf16"], f"direct decode {t}")
    flags, (_, ln, mode) = buf.device_status()
    assert flags == 0 and mode == [1] * B
    assert ln == [L0s[s // per] + 8 for s in range(B)]
