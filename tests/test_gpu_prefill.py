"""Chunked prefill at scale (chunkwise matrix form
P:390-399): prompts of hundreds of tokens folded in chunks of up to 64
tokens (ragged last chunk), every prompt output and the final state against
the fp64 oracle, then decoding continues from the prefilled state."""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV = 16, 32


@pytest.mark.parametrize("in_dtype,n_tok,short_cap,drafts,pc", [
    ("bf16", 300, 64, 0, 64), ("f32", 150, 64, 0, 64), ("bf16", 77, 0, 4, 0), ("bf16", 129, 128, 0, 48),
    ("bf16", 200, 64, 0, 0), ("f32", 70, 0, 0, 0)])
def test_long_prompt_prefill(cuda_device, in_dtype, n_tok, short_cap, drafts, pc):
    rc = synth.Recipe(seed=3601 + n_tok, dist="stress", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    R = 3
    cfg = L.make_config(R, HK, HV, chunk=16, max_drafts=drafts, short_cap=short_cap, in_dtype=in_dtype,
                        validate=True)
    buf = L.LaBuf(cfg, device=cuda_device)
    buf.set_prefill_chunk(pc)                       # 0: the handle's chunk (16)
    slots = np.arange(R)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    tok = synth.tokens(rc, slots, np.arange(n_tok), HK, HV, 128)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, in_dtype, cuda_device)
    o = torch.empty(R, n_tok, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.prefill(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), ref, tol, f"prefill outputs ({n_tok} tokens)")
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"state after prefill, slot {s}")
    # decode continues from the prefilled state
    nxt = synth.tokens(rc, slots, [n_tok], HK, HV, 128)
    r1 = orc.run(slots, nxt)
    d1 = upload_tokens(nxt, in_dtype, cuda_device, squeeze_t=True)
    o1 = torch.empty(R, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.decode_step(0, d1["q"], d1["k"], d1["v"], d1["alpha"], d1["beta"], o1)
    assert_close(o1.cpu().numpy(), r1[:, 0], tol, "decode after prefill")
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [1] * R


def test_prefill_without_outputs_matches(cuda_device):
    """o = NULL folds the prompt without writing outputs: the same state."""
    rc = synth.Recipe(seed=3610, dist="qwen", in_dtype="bf16")
    R, n_tok = 2, 100
    cfg = L.make_config(R, HK, HV, chunk=16, short_cap=64, validate=True)
    bufs = [L.LaBuf(cfg, device=cuda_device) for _ in range(2)]
    tok = synth.tokens(rc, np.arange(R), np.arange(n_tok), HK, HV, 128)
    d = upload_tokens(tok, "bf16", cuda_device)
    o = torch.empty(R, n_tok, HV, 128, dtype=torch.float32, device=cuda_device)
    for b, out in zip(bufs, (o, None)):
        b.reset(zero_state=True)
        b.prefill(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], out)
    torch.cuda.synchronize()
    assert torch.equal(bufs[0].state, bufs[1].state)
