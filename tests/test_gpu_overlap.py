"""Launch overlap (la_set_overlap: programmatic dependent launch with the
state tiles requested before griddepcontrol.wait when the overlapped kernel
cannot have written them).  It must change nothing but timing: every call
sequence below -- interleaved layers, same-handle decode -> flush -> decode,
verify -> commit -> verify, prefill chunks, recurrent steps on one handle,
eager and captured in a CUDA graph -- gives outputs and states bit-identical
to the same sequence without overlap, and within tolerance of the oracle."""
import numpy as np
import pytest
import torch

import synth
import synth.device as sd
from harness import TOL, Oracle, assert_close, make_buf, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV = 16, 32


def _run(overlap, dev, graph=False):
    B, C, N, NL = 8, 4, 3, 3
    bufs = [make_buf(B, HK, HV, C=C, N=N) for _ in range(NL)]
    for l, b in enumerate(bufs):
        b.reset(zero_state=False)
        b.state.copy_(sd.state0(600 + l, B, HV, device=dev))
        b.set_overlap(overlap)
    torch.cuda.synchronize()   # the state copies are foreign kernels (la_set_overlap contract)
    toks = [[sd.tokens(700 + 10 * l + t, B, 1, HK, HV, device=dev, squeeze=True) for t in range(2 * C + 1)]
            for l in range(NL)]
    drafts = [sd.tokens(800 + l, B, N, HK, HV, device=dev) for l in range(NL)]
    nacc = sd.n_accepted(900, B, N, device=dev)
    outs = []

    def seq():
        # interleaved layers, a flush of one layer directly before its own next decode
        for t in range(2 * C):
            for l, b in enumerate(bufs):
                x = toks[l][t]
                o = torch.empty(B, HV, 128, dtype=torch.float32, device=dev)
                b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
                b.flush(0, B, L.LA_FLUSH_FULL)
                outs.append(o)
        # verify -> commit -> decode on the same handle, then recurrent steps back to back
        for l, b in enumerate(bufs):
            x = drafts[l]
            o = torch.empty(B, N, HV, 128, dtype=torch.float32, device=dev)
            b.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
            b.commit_accepted(0, nacc)
            outs.append(o)
            y = toks[l][2 * C]
            o2 = torch.empty(B, HV, 128, dtype=torch.float32, device=dev)
            b.recurrent_step(0, y["q"], y["k"], y["v"], y["alpha"], y["beta"], o2)
            o3 = torch.empty(B, HV, 128, dtype=torch.float32, device=dev)
            b.recurrent_step(0, y["q"], y["k"], y["v"], y["alpha"], y["beta"], o3)
            outs.extend([o2, o3])

    if graph:
        s = torch.cuda.Stream(device=dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            seq()
        g.replay()
    else:
        seq()
    torch.cuda.synchronize()
    return [o.cpu() for o in outs], [b.state.cpu() for b in bufs]


@pytest.mark.parametrize("graph", [False, True])
def test_overlap_is_bit_identical(cuda_device, graph):
    o0, s0 = _run(False, cuda_device, graph)
    o1, s1 = _run(True, cuda_device, graph)
    assert len(o0) == len(o1)
    for i, (a, b) in enumerate(zip(o0, o1)):
        assert torch.equal(a, b), f"output {i}"
    for l, (a, b) in enumerate(zip(s0, s1)):
        assert torch.equal(a, b), f"state {l}"


def test_overlap_prefill_decode_matches_oracle(cuda_device):
    """Config-1-like stream with overlap on: prefill (chunk kernel -> fold ->
    chunk kernel -> fold on one handle), then decode cycles with flushes."""
    rc = synth.Recipe(seed=1201, dist="stress", in_dtype="f32")
    buf = make_buf(2, 2, 4, C=8, in_dtype="f32")
    buf.reset(zero_state=True)
    buf.set_overlap(True)
    slots = np.arange(2)
    orc = Oracle(np.zeros((2, 4, 128, 128)))
    tok = synth.tokens(rc, slots, np.arange(40), 2, 4, 128)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, "f32", cuda_device)
    o = torch.empty(2, 40, 4, 128, dtype=torch.float32, device=cuda_device)
    buf.prefill(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), ref, TOL["f32"], "prefill")
    for t in range(20):
        tk = synth.tokens(rc, slots, [40 + t], 2, 4, 128)
        r1 = orc.run(slots, tk)
        dd = upload_tokens(tk, "f32", cuda_device, squeeze_t=True)
        o1 = torch.empty(2, 4, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_step(0, dd["q"], dd["k"], dd["v"], dd["alpha"], dd["beta"], o1)
        buf.flush(0, 2, L.LA_FLUSH_FULL)
        assert_close(o1.cpu().numpy(), r1[:, 0], TOL["f32"], f"decode {t}")
    buf.flush(0, 2, L.LA_FLUSH_FORCE)
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], TOL["f32"], f"slot {s}")
