"""Fused flush (la_set_auto_flush): the decode step that fills a
slot's buffer folds the C records into the state in the same kernel.  Every
output and every state after a fold must match the fp64 oracle (and the
unfused path within the same tolerance); occupancies must follow the host
mirror exactly (the filling step leaves occ = 0)."""
import numpy as np
import pytest
import torch

import synth
import synth.device as sd
from harness import TOL, Oracle, assert_close, make_buf, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C,in_dtype", [(8, "bf16"), (16, "bf16"), (22, "f32"), (32, "bf16"), (16, "f32")])
def test_auto_flush_matches_oracle(cuda_device, C, in_dtype):
    rc = synth.Recipe(seed=1301, dist="stress" if in_dtype == "f32" else "qwen", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    R = 4
    slots = np.arange(R)
    buf = make_buf(R, 16, 32, C=C, in_dtype=in_dtype)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    buf.set_auto_flush(True)
    orc = Oracle(S0)
    # stagger: slot r starts with r buffered tokens (so the filling step differs per slot)
    for r in range(R):
        for t in range(r):
            tok = synth.tokens(rc, [r], [900 + t], 16, 32, 128)
            orc.run([r], tok)
            d = upload_tokens(tok, in_dtype, cuda_device, squeeze_t=True)
            o = torch.empty(1, 32, 128, dtype=torch.float32, device=cuda_device)
            buf.decode_step(r, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    occ = [r for r in range(R)]
    for t in range(2 * C + 3):
        tok = synth.tokens(rc, slots, [t], 16, 32, 128)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, in_dtype, cuda_device, squeeze_t=True)
        o = torch.empty(R, 32, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"C={C} step {t}")
        occ = [(x + 1) % C for x in occ]
        assert [buf.slot_info(r).occ for r in range(R)] == occ
        for r in range(R):
            if occ[r] == 0:   # just folded inside the decode kernel
                assert_close(buf.state_get(r).cpu().numpy(), orc.S[r], tol, f"C={C} step {t} slot {r} state")
    flags, (docc, _, _) = buf.device_status()
    assert flags == 0 and docc == occ
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    for r in range(R):
        assert_close(buf.state_get(r).cpu().numpy(), orc.S[r], tol, f"C={C} final slot {r}")


def test_auto_flush_graph_with_overlap(cuda_device):
    """Config-2 shape, batch 64, C = 16, two layers interleaved, overlap on,
    one cycle captured as a CUDA graph and replayed twice; sampled slots vs
    the oracle after each cycle."""
    B, C = 64, 16
    sample = [0, 17, 63]
    bufs, orcs, toks = [], [], []
    for l in range(2):
        b = make_buf(B, 16, 32, C=C, validate=False)
        b.reset(zero_state=False)
        S0 = sd.state0(4100 + l, B, 32, device=cuda_device)
        b.state.copy_(S0)
        orcs.append(Oracle(S0[sample].double().cpu().numpy()))
        bufs.append(b)
        toks.append([sd.tokens(4200 + 50 * l + t, B, 1, 16, 32, device=cuda_device, squeeze=True) for t in range(C)])
    torch.cuda.synchronize()
    for b in bufs:
        b.set_overlap(True)
        b.set_auto_flush(True)
    outs = [[torch.empty(B, 32, 128, dtype=torch.float32, device=cuda_device) for _ in range(C)] for _ in range(2)]
    s = torch.cuda.Stream(device=cuda_device)

    def cycle():
        for t in range(C):
            for l, b in enumerate(bufs):
                x = toks[l][t]
                b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], outs[l][t])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cycle()
    for rep in range(2):
        g.replay()
        torch.cuda.synchronize()
        for l in range(2):
            for t in range(C):
                ref = orcs[l].run(np.arange(len(sample)),
                                  sd.host_tokens({k: v.unsqueeze(1) for k, v in toks[l][t].items()}, sample))
                assert_close(outs[l][t][sample].cpu().numpy(), ref[:, 0], TOL["bf16"], f"rep {rep} layer {l} step {t}")
            for i, sl in enumerate(sample):
                assert_close(bufs[l].state[sl].cpu().numpy(), orcs[l].S[i], TOL["bf16"], f"rep {rep} layer {l} slot {sl}")
        flags, (docc, _, _) = bufs[0].device_status()
        assert docc == [0] * B
