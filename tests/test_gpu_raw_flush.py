"""GPU parity of flush mode ii (LA_FLUSH_RAW): the delta values are
recomputed inside the flush kernel from the raw records (k, v, beta, G) and
S0 by the UT transform (P:392-399 with K~ corrected per reading Z4) -- the
C x C forward substitution in shared memory -- and then folded on the tensor
cores.  Checked against the fp64 recurrence (the oracle) and against mode i
on the same stream."""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, make_buf, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

RAW_FULL = L.LA_FLUSH_FULL | L.LA_FLUSH_RAW
RAW_FORCE = L.LA_FLUSH_FORCE | L.LA_FLUSH_RAW


def _decode(bufs, orc, rc, slots, pos, Hk, Hv, tol, label, flush_kind=None):
    dev = bufs[0].device
    tok = synth.tokens(rc, slots, [pos], Hk, Hv, 128)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, rc.in_dtype, dev, squeeze_t=True)
    outs = []
    for b, kind in zip(bufs, flush_kind or [None] * len(bufs)):
        o = torch.empty(len(slots), Hv, 128, dtype=torch.float32, device=dev)
        b.decode_step(int(slots[0]), d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        if kind is not None:
            b.flush(int(slots[0]), len(slots), kind)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"{label} output")
        outs.append(o)
    return outs


@pytest.mark.parametrize("in_dtype,C", [("bf16", 16), ("bf16", 32), ("bf16", 64), ("f32", 16), ("f32", 22)])
def test_raw_flush_matches_oracle(cuda_device, in_dtype, C):
    """Config-2 shape (16 QK / 32 V heads): two full cycles folded by mode ii
    plus a ragged tail folded by FORCE|RAW; every output and every state after
    a fold against the oracle."""
    rc = synth.Recipe(seed=1102, dist="stress" if in_dtype == "f32" else "qwen", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    R = 3
    slots = np.arange(R)
    buf = make_buf(R, 16, 32, C=C, in_dtype=in_dtype, keep_raw=True)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    pos = 0
    for cyc in range(2):
        for t in range(C):
            _decode([buf], orc, rc, slots, pos, 16, 32, tol, f"C={C} cycle {cyc} step {t}", [RAW_FULL])
            pos += 1
        assert [buf.slot_info(r).occ for r in range(R)] == [0] * R
        for s in slots:
            assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"C={C} cycle {cyc} slot {s}")
    tail = max(1, C // 3)
    for t in range(tail):
        _decode([buf], orc, rc, slots, pos, 16, 32, tol, f"C={C} tail {t}", [RAW_FULL])
        pos += 1
    assert [buf.slot_info(r).occ for r in range(R)] == [tail % C] * R
    buf.flush(0, R, RAW_FORCE)
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"C={C} tail fold slot {s}")
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [0] * R


def test_raw_and_u_given_flush_agree(cuda_device):
    """Mode i (buffered u) and mode ii (u recomputed by the UT transform) fold
    the same records into states that agree within the fp32 bar, on a
    staggered batch (slots at different occupancies)."""
    rc = synth.Recipe(seed=1103, dist="stress", in_dtype="f32")
    R, C = 4, 16
    slots = np.arange(R)
    bi = make_buf(R, 16, 32, C=C, in_dtype="f32", keep_raw=True)
    bii = make_buf(R, 16, 32, C=C, in_dtype="f32", keep_raw=True)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    for b in (bi, bii):
        b.reset(zero_state=False)
        set_states(b, S0, slots)
    orc = Oracle(S0)
    for r in range(R):           # stagger: slot r starts with 3r buffered tokens
        for t in range(3 * r):
            tok = synth.tokens(rc, [r], [5000 + t], 16, 32, 128)
            orc.run([r], tok)
            d = upload_tokens(tok, "f32", cuda_device, squeeze_t=True)
            for b in (bi, bii):
                o = torch.empty(1, 32, 128, dtype=torch.float32, device=cuda_device)
                b.decode_step(r, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    for t in range(7):
        _decode([bi, bii], orc, rc, slots, t, 16, 32, TOL["f32"], f"step {t}", [L.LA_FLUSH_FULL, RAW_FULL])
    bi.flush(0, R, L.LA_FLUSH_FORCE)
    bii.flush(0, R, RAW_FORCE)
    for s in slots:
        a = bi.state_get(int(s)).cpu().numpy()
        b = bii.state_get(int(s)).cpu().numpy()
        assert_close(a, orc.S[s], TOL["f32"], f"mode i slot {s}")
        assert_close(b, orc.S[s], TOL["f32"], f"mode ii slot {s}")
        assert_close(a, b, TOL["f32"], f"mode i vs ii slot {s}")


@pytest.mark.parametrize("L0", [16, 64, 128])
def test_raw_compress_direct_slot(cuda_device, L0):
    """A DIRECT slot (no state) compressed by FORCE|RAW: S0 = 0, so the UT
    transform alone produces u from the raw records of the whole context
     -- up to d = 128 tokens in one forward substitution."""
    rc = synth.Recipe(seed=1104, dist="qwen", in_dtype="bf16")
    R = 2
    slots = np.arange(R)
    buf = make_buf(R, 16, 32, C=16, short_cap=128, keep_raw=True)
    buf.reset(mode=L.LA_MODE_DIRECT)
    orc = Oracle(np.zeros((R, 32, 128, 128)))
    tok = synth.tokens(rc, slots, np.arange(L0), 16, 32, 128)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, "bf16", cuda_device)
    done = 0
    while done < L0:
        m = min(16, L0 - done)
        sub = {k: v[:, done:done + m].contiguous() for k, v in d.items()}
        o = torch.empty(R, m, 32, 128, dtype=torch.float32, device=cuda_device)
        buf.direct_short(0, sub["q"], sub["k"], sub["v"], sub["alpha"], sub["beta"], o)
        assert_close(o.cpu().numpy(), ref[:, done:done + m], TOL["bf16"], f"direct tokens {done}..")
        done += m
    buf.flush(0, R, RAW_FORCE)
    info = buf.slot_info(0)
    assert info.mode == L.LA_MODE_CHUNKWISE and info.len == 0 and info.occ == 0
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], TOL["bf16"], f"compressed slot {s}")
    # and decoding continues from the compressed state
    _decode([buf], orc, rc, slots, L0, 16, 32, TOL["bf16"], "after compression")


def test_raw_flush_needs_keep_raw(cuda_device):
    buf = make_buf(1, 16, 32, C=4, keep_raw=False)
    buf.reset(zero_state=True)
    with pytest.raises(L.LaError) as e:
        buf.flush(0, 1, RAW_FORCE)
    assert e.value.status == L.LA_ERR_INVALID
