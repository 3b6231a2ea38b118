"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
the same seeded inputs.  Tolerances are the north-star ones: max-abs 2e-3
for bf16 q/k/v with an fp32 state, 1e-5 all-fp32 (tests/harness.TOL)."""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, make_buf, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

QWEN = dict(Hk=16, Hv=32)


def _tok(rc, slots, pos, Hk, Hv):
    return synth.tokens(rc, slots, pos, Hk, Hv, 128)


def _decode_steps(buf, orc, rc, slots, pos0, n_steps, Hk, Hv, tol, flush_each=True, label=""):
    dev = buf.device
    first, n = int(slots[0]), len(slots)
    errs = []
    for t in range(n_steps):
        tok = _tok(rc, slots, [pos0 + t], Hk, Hv)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, rc.in_dtype, dev, squeeze_t=True)
        o = torch.empty(n, Hv, 128, dtype=torch.float32, device=dev)
        buf.decode_step(first, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        if flush_each:
            buf.flush(first, n, L.LA_FLUSH_FULL)
        errs.append(assert_close(o.cpu().numpy(), ref[:, 0], tol, f"{label} step {t} output"))
    return max(errs) if errs else 0.0


def _check_states(buf, orc, slots, tol, what):
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"{what} slot {s} state")


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("in_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("dist", ["stress", "qwen"])
def test_config1_prefill_then_decode(cuda_device, in_dtype, dist):
    """Config 1: 1 request, 1 GDN head, d = 128, 64-token prefill + 64 decode
    steps, C = 16, against the recurrent oracle; every output and the state
    after every flush."""
    rc = synth.Recipe(seed=1001, dist=dist, in_dtype=in_dtype)
    tol = TOL[in_dtype]
    buf = make_buf(1, 1, 1, C=16, in_dtype=in_dtype)
    buf.reset(zero_state=True)
    orc = Oracle(np.zeros((1, 1, 128, 128)))
    slots = np.array([0])
    tok = _tok(rc, slots, np.arange(64), 1, 1)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, in_dtype, cuda_device)
    o = torch.empty(1, 64, 1, 128, dtype=torch.float32, device=cuda_device)
    buf.prefill(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), ref, tol, "prefill outputs")
    _check_states(buf, orc, slots, tol, "after prefill")
    assert buf.slot_info(0).occ == 0
    for cyc in range(4):
        _decode_steps(buf, orc, rc, slots, 64 + 16 * cyc, 16, 1, 1, tol, label=f"cycle {cyc}")
        assert buf.slot_info(0).occ == 0
        _check_states(buf, orc, slots, tol, f"after flush {cyc}")
    flags, (occ, ln, mode) = buf.device_status()
    assert flags == 0 and occ == [0]


@pytest.mark.parametrize("in_dtype", ["f32", "bf16"])
def test_config1_recurrent_baseline(cuda_device, in_dtype):
    """Kernel (5a) on config 1: 128 recurrent steps against the oracle."""
    rc = synth.Recipe(seed=1001, dist="stress", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    buf = make_buf(1, 1, 1, C=16, in_dtype=in_dtype)
    buf.reset(zero_state=True)
    orc = Oracle(np.zeros((1, 1, 128, 128)))
    slots = np.array([0])
    for t in range(128):
        tok = _tok(rc, slots, [t], 1, 1)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, in_dtype, cuda_device, squeeze_t=True)
        o = torch.empty(1, 1, 128, dtype=torch.float32, device=cuda_device)
        buf.recurrent_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"recurrent step {t}")
    _check_states(buf, orc, slots, tol, "recurrent final")


# ------------------------------------------------------------------ config 2 (reduced batch)
@pytest.mark.parametrize("C", [1, 8, 16, 22, 32])
def test_qwen_decode_chunk_sweep(cuda_device, C):
    """Config 2 shape (16 QK / 32 V heads, d = 128, bf16 in, fp32 state) with
    synthetic long-context states, C swept; 40 steps cross several flushes
    and end on a ragged partial buffer that a FORCE flush folds."""
    rc = synth.Recipe(seed=1002, dist="qwen", in_dtype="bf16")
    R = 4
    slots = np.arange(R)
    buf = make_buf(R, **QWEN, C=C)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    _decode_steps(buf, orc, rc, slots, 0, 40, 16, 32, TOL["bf16"], label=f"C={C}")
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    _check_states(buf, orc, slots, TOL["bf16"], f"C={C} final")
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [0] * R


def test_qwen_decode_staggered_fp32(cuda_device):
    """Staggered occupancies (occ_r = r mod C at the start) in one batch,
    all-fp32 inputs at the 1e-5 bar."""
    rc = synth.Recipe(seed=1012, dist="stress", in_dtype="f32")
    R, C = 6, 8
    slots = np.arange(R)
    buf = make_buf(R, **QWEN, C=C, in_dtype="f32")
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    # stagger: slot r first decodes r tokens alone
    for r in range(R):
        for t in range(r):
            tok = _tok(rc, [r], [1000 + t], 16, 32)
            ref = orc.run([r], tok)
            d = upload_tokens(tok, "f32", cuda_device, squeeze_t=True)
            o = torch.empty(1, 32, 128, dtype=torch.float32, device=cuda_device)
            buf.decode_step(r, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
            buf.flush(r, 1, L.LA_FLUSH_FULL)
            assert_close(o.cpu().numpy(), ref[:, 0], TOL["f32"], "stagger warmup")
    assert [buf.slot_info(r).occ for r in range(R)] == [r % C for r in range(R)]
    _decode_steps(buf, orc, rc, slots, 0, 20, 16, 32, TOL["f32"], label="staggered")
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    _check_states(buf, orc, slots, TOL["f32"], "staggered final")


def test_qwen_recurrent_step(cuda_device):
    rc = synth.Recipe(seed=1002, dist="qwen", in_dtype="bf16")
    R = 3
    slots = np.arange(R)
    buf = make_buf(R, **QWEN)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    for t in range(6):
        tok = _tok(rc, slots, [t], 16, 32)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, "bf16", cuda_device, squeeze_t=True)
        o = torch.empty(R, 32, 128, dtype=torch.float32, device=cuda_device)
        buf.recurrent_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref[:, 0], TOL["bf16"], f"recurrent {t}")
    _check_states(buf, orc, slots, TOL["bf16"], "recurrent final")


# ------------------------------------------------------------------ config 3
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_verify_commit_every_nacc(cuda_device, N):
    """Parallel verification of N drafts and accepted-prefix commit: for every
    n_acc in [0, N] (slot r gets n_acc = r mod (N+1)), outputs of all drafts and
    the committed state match the oracle; n_acc = 0 leaves the state
    bit-identical.  Rounds start with a non-empty decode buffer (reading Z17)."""
    rc = synth.Recipe(seed=1003, dist="qwen", in_dtype="bf16")
    R = N + 1
    slots = np.arange(R)
    buf = make_buf(R, **QWEN, C=16, N=N)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    pos = 0
    for rnd in range(3):
        _decode_steps(buf, orc, rc, slots, pos, rnd + 1, 16, 32, TOL["bf16"], label=f"round {rnd} decode")
        pos += rnd + 1
        tok = _tok(rc, slots, np.arange(pos, pos + N), 16, 32)
        n_acc = np.array([(r + rnd) % (N + 1) for r in range(R)], dtype=np.int32)
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, "bf16", cuda_device)
        o = torch.empty(R, N, 32, 128, dtype=torch.float32, device=cuda_device)
        buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, TOL["bf16"], f"round {rnd} draft outputs")
        buf.commit_accepted(0, torch.from_numpy(n_acc).to(cuda_device))
        pos += N
        for i, s in enumerate(slots):
            after = buf.state_get(int(s))
            assert_close(after.cpu().numpy(), orc.S[s], TOL["bf16"], f"round {rnd} slot {s} committed")
        assert all(buf.slot_info(int(s)).occ == 0 for s in slots)
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [0] * R


def test_commit_zero_accepted_is_bit_identical(cuda_device):
    rc = synth.Recipe(seed=1013, dist="qwen", in_dtype="bf16")
    R, N = 2, 4
    buf = make_buf(R, **QWEN, C=16, N=N)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, np.arange(R), 32, 128, 128)
    set_states(buf, S0, np.arange(R))
    before = buf.state.clone()
    tok = _tok(rc, np.arange(R), np.arange(N), 16, 32)
    d = upload_tokens(tok, "bf16", cuda_device)
    o = torch.empty(R, N, 32, 128, dtype=torch.float32, device=cuda_device)
    buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    buf.commit_accepted(0, torch.zeros(R, dtype=torch.int32, device=cuda_device))
    torch.cuda.synchronize()
    assert torch.equal(before, buf.state)


def test_verify_causality_bit_identical(cuda_device):
    """Draft t's output is bit-identical whatever drafts t+1.. contain."""
    rc = synth.Recipe(seed=1014, dist="stress", in_dtype="bf16")
    R, N = 2, 8
    buf = make_buf(R, **QWEN, C=16, N=N)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, np.arange(R), 32, 128, 128)
    set_states(buf, S0, np.arange(R))
    tok = _tok(rc, np.arange(R), np.arange(N), 16, 32)
    d = upload_tokens(tok, "bf16", cuda_device)
    o1 = torch.empty(R, N, 32, 128, dtype=torch.float32, device=cuda_device)
    buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o1)
    buf.commit_accepted(0, torch.zeros(R, dtype=torch.int32, device=cuda_device))
    d2 = {k: v.clone() for k, v in d.items()}
    d2["v"][:, 5:] = -d2["v"][:, 5:]
    d2["k"][:, 6:] = d2["k"][:, 6:].flip(-1)
    o2 = torch.empty_like(o1)
    buf.verify_drafts(0, d2["q"], d2["k"], d2["v"], d2["alpha"], d2["beta"], o2)
    buf.commit_accepted(0, torch.zeros(R, dtype=torch.int32, device=cuda_device))
    torch.cuda.synchronize()
    assert torch.equal(o1[:, :5], o2[:, :5])
    assert not torch.equal(o1[:, 5:], o2[:, 5:])


def test_recurrent_verify_commit(cuda_device):
    """Kernel (5b) + baseline commit (state <- temporary state n_acc - 1)."""
    rc = synth.Recipe(seed=1003, dist="qwen", in_dtype="bf16")
    N = 4
    R = N + 1
    slots = np.arange(R)
    buf = make_buf(R, **QWEN, C=16, N=N)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, 32, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    for rnd in range(2):
        tok = _tok(rc, slots, np.arange(rnd * N, rnd * N + N), 16, 32)
        n_acc = np.array([(r + rnd) % (N + 1) for r in range(R)], dtype=np.int32)
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, "bf16", cuda_device)
        o = torch.empty(R, N, 32, 128, dtype=torch.float32, device=cuda_device)
        temp = torch.empty(R, N, 32, 128, 128, dtype=torch.float32, device=cuda_device)
        buf.recurrent_verify(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], temp, o)
        assert_close(o.cpu().numpy(), ref, TOL["bf16"], "recurrent verify outputs")
        buf.recurrent_commit(0, torch.from_numpy(n_acc).to(cuda_device), temp)
        _check_states(buf, orc, slots, TOL["bf16"], f"recurrent commit round {rnd}")


# ------------------------------------------------------------------ config 4
@pytest.mark.parametrize("u_dtype", ["f16", "f32"])
def test_direct_short_then_compress(cuda_device, u_dtype):
    """Direct (KV-only) decoding with no state: short prefills of ragged
    lengths, decode steps, then compression of the buffer into a state
    (FORCE flush) and chunkwise decode from it."""
    rc = synth.Recipe(seed=1004, dist="qwen", in_dtype="bf16")
    R = 4
    slots = np.arange(R)
    L0 = [1, 17, 40, 64]
    buf = make_buf(R, **QWEN, C=16, short_cap=128, u_dtype=u_dtype)
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=True)
    orc = Oracle(np.zeros((R, 32, 128, 128)))
    tol = TOL["bf16"]
    for r in range(R):
        tok = _tok(rc, [r], np.arange(L0[r]), 16, 32)
        ref = orc.run([r], tok)
        d = upload_tokens(tok, "bf16", cuda_device)
        o = torch.empty(1, L0[r], 32, 128, dtype=torch.float32, device=cuda_device)
        buf.direct_short(r, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, tol, f"direct prefill slot {r} L0={L0[r]}")
    for t in range(24):
        tok = synth.tokens(rc, slots, [200 + t], 16, 32, 128)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, "bf16", cuda_device)
        o = torch.empty(R, 1, 32, 128, dtype=torch.float32, device=cuda_device)
        buf.direct_short(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, tol, f"direct decode {t}")
    assert [buf.slot_info(r).len for r in range(R)] == [l + 24 for l in L0]
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    assert all(buf.slot_info(r).mode == L.LA_MODE_CHUNKWISE for r in range(R))
    _check_states(buf, orc, slots, tol, "compressed")
    _decode_steps(buf, orc, rc, slots, 500, 5, 16, 32, tol, label="post-compress")
    flags, (occ, ln, mode) = buf.device_status()
    assert flags == 0 and mode == [0] * R and ln == [0] * R and occ == [5] * R


# ------------------------------------------------------------------ harness properties
def test_determinism_run_to_run(cuda_device):
    rc = synth.Recipe(seed=1015, dist="qwen", in_dtype="bf16")
    R, C = 4, 8
    outs = []
    for rep in range(2):
        buf = make_buf(R, **QWEN, C=C)
        buf.reset(zero_state=False)
        set_states(buf, synth.state0(rc, np.arange(R), 32, 128, 128), np.arange(R))
        os = []
        for t in range(10):
            tok = _tok(rc, np.arange(R), [t], 16, 32)
            d = upload_tokens(tok, "bf16", cuda_device, squeeze_t=True)
            o = torch.empty(R, 32, 128, dtype=torch.float32, device=cuda_device)
            buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
            buf.flush(0, R, L.LA_FLUSH_FULL)
            os.append(o)
        outs.append((torch.stack(os), buf.state.clone()))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_sharded_equals_unsharded(cuda_device):
    """Data-parallel sharding: running slot ranges separately gives bit-identical
    results to one batch (kernels are per (slot, head) independent)."""
    rc = synth.Recipe(seed=1016, dist="qwen", in_dtype="bf16")
    R, C = 6, 4
    S0 = synth.state0(rc, np.arange(R), 32, 128, 128)
    res = []
    for split in ([(0, R)], [(0, 2), (2, 3), (5, 1)]):
        buf = make_buf(R, **QWEN, C=C)
        buf.reset(zero_state=False)
        set_states(buf, S0, np.arange(R))
        os = []
        for t in range(6):
            tok = _tok(rc, np.arange(R), [t], 16, 32)
            d = upload_tokens(tok, "bf16", cuda_device, squeeze_t=True)
            o = torch.empty(R, 32, 128, dtype=torch.float32, device=cuda_device)
            for f, n in split:
                buf.decode_step(f, d["q"][f:f + n], d["k"][f:f + n], d["v"][f:f + n],
                                d["alpha"][f:f + n], d["beta"][f:f + n], o[f:f + n])
                buf.flush(f, n, L.LA_FLUSH_FULL)
            os.append(o)
        res.append((torch.stack(os), buf.state.clone()))
    torch.cuda.synchronize()
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])


def test_error_paths_all_or_nothing(cuda_device):
    buf = make_buf(2, **QWEN, C=2, N=2, short_cap=8)
    buf.reset(zero_state=True)
    rc = synth.Recipe(seed=5)
    d = upload_tokens(_tok(rc, [0, 1], [0], 16, 32), "bf16", cuda_device, squeeze_t=True)
    o = torch.empty(2, 32, 128, dtype=torch.float32, device=cuda_device)
    for _ in range(2):
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    n0 = buf.kernel_launches()
    with pytest.raises(L.LaError) as e:
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert e.value.status == L.LA_ERR_CAPACITY and buf.kernel_launches() == n0
    assert buf.slot_info(0).occ == 2
    with pytest.raises(L.LaError) as e:
        buf.commit_accepted(0, torch.zeros(2, dtype=torch.int32, device=cuda_device))
    assert e.value.status == L.LA_ERR_MODE
    with pytest.raises(L.LaError) as e:
        buf.direct_short(0, d["q"][:, None], d["k"][:, None], d["v"][:, None],
                         d["alpha"][:, None], d["beta"][:, None], o[:, None])
    assert e.value.status == L.LA_ERR_MODE
    buf.flush(0, 2, L.LA_FLUSH_FULL)
    assert buf.slot_info(0).occ == 0 and buf.kernel_launches() == n0 + 1
    buf.flush(0, 2, L.LA_FLUSH_FULL)          # empty flush: no-op, not an error
    assert buf.kernel_launches() == n0 + 1
    dq = {k: v[:, None].expand(-1, 3, *v.shape[1:]).contiguous() for k, v in d.items()}
    o3 = torch.empty(2, 3, 32, 128, dtype=torch.float32, device=cuda_device)
    with pytest.raises(L.LaError) as e:
        buf.verify_drafts(0, dq["q"], dq["k"], dq["v"], dq["alpha"], dq["beta"], o3)
    assert e.value.status == L.LA_ERR_INVALID   # 3 > max_drafts


def test_validate_status_bits(cuda_device):
    buf = make_buf(1, 1, 1, C=4, validate=True)
    buf.reset(zero_state=True)
    rc = synth.Recipe(seed=6)
    d = upload_tokens(_tok(rc, [0], [0], 1, 1), "bf16", cuda_device, squeeze_t=True)
    d["alpha"].fill_(1.5)
    o = torch.empty(1, 1, 128, dtype=torch.float32, device=cuda_device)
    buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    flags, _ = buf.device_status()
    assert flags & L.STATUS_BITS["bad_alpha"]


def test_fault_injection_is_detected():
    """Harness self-test (SPEC run_equiv_suite fault mode): a 1e-3 perturbation
    of one output must fail the bf16/fp32 comparisons it would hide in."""
    ref = np.random.default_rng(0).standard_normal((4, 32, 128))
    bad = ref.copy()
    bad[2, 7, 99] += 1e-3
    with pytest.raises(AssertionError):
        assert_close(bad, ref, TOL["f32"], "fault")
    bad[2, 7, 99] += 3e-3
    with pytest.raises(AssertionError):
        assert_close(bad, ref, TOL["bf16"], "fault")
