"""Linear-attention variants (Table 1):
vanilla LA (S_t = S_{t-1} + v_t k_t^T) and scalar-gated LA
(S_t = alpha_t S_{t-1} + v_t k_t^T) through the same buffered kernels --
decode with flush, verify + commit, direct + compression, recurrent step --
against the fp64 oracle run with erase coefficient 0 and write coefficient
1 (and alpha = 1 for vanilla), the oracle's reading Z7."""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV = 16, 32


def _buf(variant, R, C=8, N=4, short_cap=32, in_dtype="bf16", u_dtype="f32", device="cuda"):
    cfg = L.make_config(R, HK, HV, chunk=C, max_drafts=N, short_cap=short_cap, in_dtype=in_dtype,
                        u_dtype=u_dtype, validate=True, variant=variant)
    return L.LaBuf(cfg, device=device)


@pytest.mark.parametrize("in_dtype", ["bf16", "f32"])
@pytest.mark.parametrize("variant", ["vanilla", "gated"])
def test_variant_decode_verify_commit(cuda_device, variant, in_dtype):
    rc = synth.Recipe(seed=3401, dist="qwen", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    R, C, N = 3, 8, 4
    buf = _buf(variant, R, C=C, N=N, in_dtype=in_dtype)
    slots = np.arange(R)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0, variant)
    for t in range(C + 3):
        tok = synth.tokens(rc, slots, [t], HK, HV, 128)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, in_dtype, cuda_device, squeeze_t=True)
        o = torch.empty(R, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        buf.flush(0, R, L.LA_FLUSH_FULL)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"{variant} decode {t}")
    for rnd in range(2):
        tok = synth.tokens(rc, slots, np.arange(50 + 10 * rnd, 50 + 10 * rnd + N), HK, HV, 128)
        n_acc = synth.n_accepted(rc, slots, N, round_idx=rnd)
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, in_dtype, cuda_device)
        o = torch.empty(R, N, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        buf.commit_accepted(0, torch.from_numpy(n_acc).to(cuda_device))
        assert_close(o.cpu().numpy(), ref, tol, f"{variant} verify {rnd}")
        for s in slots:
            assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"{variant} commit {rnd} slot {s}")
    # the recurrent baseline honours the variant too
    for t in range(3):
        tok = synth.tokens(rc, slots, [200 + t], HK, HV, 128)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, in_dtype, cuda_device, squeeze_t=True)
        o = torch.empty(R, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.recurrent_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"{variant} recurrent {t}")
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"{variant} recurrent state {s}")
    flags, _ = buf.device_status()
    assert flags == 0


@pytest.mark.parametrize("variant", ["vanilla", "gated"])
def test_variant_direct_then_compress(cuda_device, variant):
    rc = synth.Recipe(seed=3402, dist="stress", in_dtype="bf16")
    tol = TOL["bf16"]
    R = 2
    buf = _buf(variant, R, short_cap=32, u_dtype="f16")
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=True)
    orc = Oracle(np.zeros((R, HV, 128, 128)), variant)
    slots = np.arange(R)
    tok = synth.tokens(rc, slots, np.arange(20), HK, HV, 128)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, "bf16", cuda_device)
    o = torch.empty(R, 20, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.direct_short(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), ref, tol, f"{variant} direct prefill")
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"{variant} compressed {s}")


def test_vanilla_equals_brute_force_attention(cuda_device):
    """Vanilla LA from a zero state is softmax-free causal attention
    o_t = sum_{i<=t} (q_t . k_i) v_i: the GPU direct path against
    that brute-force formula (not the recurrence) on the stored inputs."""
    rc = synth.Recipe(seed=3403, dist="qwen", in_dtype="f32")
    buf = _buf("vanilla", 1, short_cap=64, in_dtype="f32")
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=True)
    tok = synth.tokens(rc, [0], np.arange(40), HK, HV, 128)
    d = upload_tokens(tok, "f32", cuda_device)
    o = torch.empty(1, 40, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.direct_short(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    q = synth.expand_qk_to_v_heads(tok["q"], HV)[0].astype(np.float64)   # [T, Hv, d]
    k = synth.expand_qk_to_v_heads(tok["k"], HV)[0].astype(np.float64)
    v = tok["v"][0].astype(np.float64)
    scores = np.einsum("thd,shd->hts", q, k) * np.tril(np.ones((40, 40)))[None]
    ref = np.einsum("hts,shd->thd", scores, v)
    assert_close(o.cpu().numpy()[0], ref, TOL["f32"], "vanilla vs (QK^T (.) M) V")
