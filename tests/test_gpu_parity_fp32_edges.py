"""GPU parity, part 2: the all-fp32 regime at the north-star 1e-5 bar for every
multi-token path (verify, commit, direct, recurrent verify), drafts above 8,
and the method's decay / gate edge cases:

  * alpha ~ U(0.5, 1]  -- strong decay: gamma underflow, the log-domain G path
                          over 128 direct tokens (gamma reaches ~1e-18);
  * alpha == 1         -- no decay: the largest error growth;
  * beta in {0, 1}     -- no write / full delta-rule overwrite.

Every output and every committed / flushed / compressed state is compared
element by element with the fp64 oracle (the recurrence P:362-365) on the same
stored inputs.  Tolerances are tests/harness.TOL (north star), never loosened.
"""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, make_buf, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV, D = 16, 32, 128

EDGES = {
    "alpha_strong": dict(alpha_lo=0.5, alpha_hi=1.0),
    "alpha_one": dict(alpha_lo=1.0, alpha_hi=1.0),
    "beta01": dict(),
}


def _recipe(seed, in_dtype, edge=None, dist="stress"):
    kw = EDGES.get(edge, {}) if edge else {}
    return synth.Recipe(seed=seed, dist=dist, in_dtype=in_dtype, **kw)


def _tok(rc, slots, pos, edge=None):
    tok = synth.tokens(rc, slots, pos, HK, HV, D)
    if edge == "beta01":
        # beta in {0, 1}: a seeded coin per (slot, token, head); stored values
        # are exact, both sides consume them unchanged
        key = int(rc.seed) * 7919 + int(np.asarray(pos).ravel()[0])
        coin = np.random.default_rng(key).random(tok["beta"].shape) < 0.5
        tok["beta"] = np.where(coin, 1.0, 0.0).astype(np.float32)
    return tok


def _decode(buf, orc, rc, slots, pos0, n_steps, tol, edge=None, label=""):
    dev = buf.device
    n = len(slots)
    for t in range(n_steps):
        tok = _tok(rc, slots, [pos0 + t], edge)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, rc.in_dtype, dev, squeeze_t=True)
        o = torch.empty(n, HV, D, dtype=torch.float32, device=dev)
        buf.decode_step(int(slots[0]), d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        buf.flush(int(slots[0]), n, L.LA_FLUSH_FULL)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"{label} decode {t}")


def _states(buf, orc, slots, tol, what):
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"{what} slot {s} state")


def _verify_rounds(dev, in_dtype, N, edge=None, seed=2101, rounds=3, C=16):
    """Rounds of (rnd decode steps, verify N drafts, commit n_acc = (r + rnd)
    mod (N + 1)): every n_acc value in [0, N] in every round; round 0 starts
    on an empty buffer, so its n_acc = 0 slot must stay bit-identical."""
    rc = _recipe(seed, in_dtype, edge)
    tol = TOL[in_dtype]
    R = N + 1
    slots = np.arange(R)
    buf = make_buf(R, HK, HV, C=C, N=N, in_dtype=in_dtype, device=dev)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, D, D)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    pos = 0
    for rnd in range(rounds):
        _decode(buf, orc, rc, slots, pos, rnd, tol, edge, label=f"N={N} round {rnd}")
        pos += rnd
        occ_before = [buf.slot_info(int(s)).occ for s in slots]
        tok = _tok(rc, slots, np.arange(pos, pos + N), edge)
        n_acc = np.array([(r + rnd) % (N + 1) for r in range(R)], dtype=np.int32)
        before = buf.state.clone()
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, in_dtype, dev)
        o = torch.empty(R, N, HV, D, dtype=torch.float32, device=dev)
        buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, tol, f"N={N} round {rnd} draft outputs")
        buf.commit_accepted(0, torch.from_numpy(n_acc).to(dev))
        pos += N
        torch.cuda.synchronize()
        for i, s in enumerate(slots):
            if n_acc[i] == 0 and occ_before[i] == 0:
                # nothing to fold: the state is not written at all
                assert torch.equal(buf.state[s], before[s]), f"N={N} round {rnd} slot {s}: n_acc=0 not bit-identical"
            assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"N={N} round {rnd} slot {s} committed")
        assert all(buf.slot_info(int(s)).occ == 0 for s in slots)
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ == [0] * R


# ------------------------------------------------------------------ fp32 regime, 1e-5
@pytest.mark.parametrize("N", [1, 2, 3, 4, 8, 9, 12, 16])
def test_verify_commit_fp32_every_nacc(cuda_device, N):
    """All-fp32 verify (CUDA-core state pass for N < 8, split-TF32 tcgen05 pass
    with the third fp32 remainder pass for N >= 8) and commit of every
    accepted prefix, at 1e-5."""
    _verify_rounds(cuda_device, "f32", N)


@pytest.mark.parametrize("N", [9, 12, 16])
def test_verify_commit_bf16_large_drafts(cuda_device, N):
    """Drafts above 8 (max_drafts allows 16) with bf16 inputs, at 2e-3."""
    _verify_rounds(cuda_device, "bf16", N, seed=2102)


def test_recurrent_verify_commit_fp32(cuda_device):
    """Kernel (5b) + baseline commit in the all-fp32 regime, at 1e-5."""
    rc = _recipe(2103, "f32")
    N = 4
    R = N + 1
    slots = np.arange(R)
    buf = make_buf(R, HK, HV, C=16, N=N, in_dtype="f32", device=cuda_device)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, D, D)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    for rnd in range(2):
        tok = _tok(rc, slots, np.arange(rnd * N, rnd * N + N))
        n_acc = np.array([(r + rnd) % (N + 1) for r in range(R)], dtype=np.int32)
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, "f32", cuda_device)
        o = torch.empty(R, N, HV, D, dtype=torch.float32, device=cuda_device)
        temp = torch.empty(R, N, HV, D, D, dtype=torch.float32, device=cuda_device)
        buf.recurrent_verify(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], temp, o)
        assert_close(o.cpu().numpy(), ref, TOL["f32"], "fp32 recurrent verify outputs")
        buf.recurrent_commit(0, torch.from_numpy(n_acc).to(cuda_device), temp)
        _states(buf, orc, slots, TOL["f32"], f"fp32 recurrent commit round {rnd}")


def _direct_to_cap(dev, in_dtype, u_dtype, edge=None, seed=2104, L0=(1, 40, 64, 100), cap=128):
    """Direct (KV-only) slots with ragged prefills, decoded together until the
    longest reaches short_cap = d = 128, then compressed into a state (FORCE
    flush of up to 128 records) and decoded chunkwise from it."""
    rc = _recipe(seed, in_dtype, edge)
    tol = TOL[in_dtype]
    R = len(L0)
    slots = np.arange(R)
    buf = make_buf(R, HK, HV, C=16, short_cap=cap, in_dtype=in_dtype, u_dtype=u_dtype, device=dev)
    buf.reset(mode=L.LA_MODE_DIRECT, zero_state=True)
    orc = Oracle(np.zeros((R, HV, D, D)))
    for r in range(R):
        tok = _tok(rc, [r], np.arange(L0[r]), edge)
        ref = orc.run([r], tok)
        d = upload_tokens(tok, in_dtype, dev)
        o = torch.empty(1, L0[r], HV, D, dtype=torch.float32, device=dev)
        buf.direct_short(r, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, tol, f"{edge} direct prefill slot {r} L0={L0[r]}")
    steps = cap - max(L0)
    for t in range(steps):
        tok = _tok(rc, slots, [300 + t], edge)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, in_dtype, dev)
        o = torch.empty(R, 1, HV, D, dtype=torch.float32, device=dev)
        buf.direct_short(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, tol, f"{edge} direct decode {t}")
    assert [buf.slot_info(r).len for r in range(R)] == [l + steps for l in L0]
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    _states(buf, orc, slots, tol, f"{edge} compressed")
    _decode(buf, orc, rc, slots, 900, 3, tol, edge, label=f"{edge} post-compress")
    flags, (occ, ln, mode) = buf.device_status()
    assert flags == 0 and mode == [0] * R and ln == [0] * R and occ == [3] * R


def test_direct_fp32_to_128(cuda_device):
    """All-fp32 direct decoding up to L = d = 128 and compression, at 1e-5."""
    _direct_to_cap(cuda_device, "f32", "f32")


def test_direct_bf16_u32_to_128(cuda_device):
    _direct_to_cap(cuda_device, "bf16", "f32", seed=2105)


# ------------------------------------------------------------------ decay / gate edge cases
@pytest.mark.parametrize("in_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("edge", sorted(EDGES))
def test_edge_decode_cycles(cuda_device, edge, in_dtype):
    """Buffered decode + tcgen05 flush over 3 cycles of C = 16 and a ragged
    tail (FORCE flush) under the edge distributions; also flush mode ii."""
    rc = _recipe(2110, in_dtype, edge)
    tol = TOL[in_dtype]
    R = 3
    slots = np.arange(R)
    buf = make_buf(R, HK, HV, C=16, in_dtype=in_dtype, device=cuda_device)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, D, D)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    _decode(buf, orc, rc, slots, 0, 53, tol, edge, label=edge)
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    _states(buf, orc, slots, tol, f"{edge} final")


@pytest.mark.parametrize("in_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("edge", sorted(EDGES))
def test_edge_raw_flush(cuda_device, edge, in_dtype):
    """Flush mode ii (UT transform from raw records) under the edge cases."""
    rc = _recipe(2111, in_dtype, edge)
    tol = TOL[in_dtype]
    R = 2
    slots = np.arange(R)
    buf = make_buf(R, HK, HV, C=16, in_dtype=in_dtype, keep_raw=True, device=cuda_device)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, D, D)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    for cyc in range(2):
        for t in range(16):
            tok = _tok(rc, slots, [16 * cyc + t], edge)
            ref = orc.run(slots, tok)
            d = upload_tokens(tok, in_dtype, cuda_device, squeeze_t=True)
            o = torch.empty(R, HV, D, dtype=torch.float32, device=cuda_device)
            buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
            assert_close(o.cpu().numpy(), ref[:, 0], tol, f"{edge} raw cycle {cyc} step {t}")
        buf.flush(0, R, L.LA_FLUSH_FULL | L.LA_FLUSH_RAW)
        _states(buf, orc, slots, tol, f"{edge} raw flush {cyc}")


@pytest.mark.parametrize("in_dtype", ["f32", "bf16"])
@pytest.mark.parametrize("edge", sorted(EDGES))
def test_edge_verify_commit(cuda_device, edge, in_dtype):
    for N in (4, 8):
        _verify_rounds(cuda_device, in_dtype, N, edge=edge, seed=2112, rounds=2)


@pytest.mark.parametrize("edge", sorted(EDGES))
def test_edge_direct_128(cuda_device, edge):
    """128-token direct contexts under strong / no decay and 0/1 gates
    (fp32, 1e-5): the log-domain decay path with gamma down to ~1e-18."""
    _direct_to_cap(cuda_device, "f32", "f32", edge=edge, seed=2113, L0=(2, 77, 100))


@pytest.mark.parametrize("edge", sorted(EDGES))
def test_edge_prefill(cuda_device, edge):
    """Chunkwise prefill (UT transform per chunk + tensor-core fold) of 80
    tokens, fp32, 1e-5, outputs and state."""
    rc = _recipe(2114, "f32", edge)
    R = 2
    slots = np.arange(R)
    buf = make_buf(R, HK, HV, C=16, in_dtype="f32", device=cuda_device)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, D, D)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    tok = _tok(rc, slots, np.arange(80), edge)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, "f32", cuda_device)
    o = torch.empty(R, 80, HV, D, dtype=torch.float32, device=cuda_device)
    buf.prefill(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), ref, TOL["f32"], f"{edge} prefill outputs")
    _states(buf, orc, slots, TOL["f32"], f"{edge} prefill")


def test_recurrent_step_edges(cuda_device):
    """Kernel (5a) under every edge distribution, fp32, 1e-5."""
    for edge in sorted(EDGES):
        rc = _recipe(2115, "f32", edge)
        R = 2
        slots = np.arange(R)
        buf = make_buf(R, HK, HV, C=16, in_dtype="f32", device=cuda_device)
        buf.reset(zero_state=False)
        S0 = synth.state0(rc, slots, HV, D, D)
        set_states(buf, S0, slots)
        orc = Oracle(S0)
        for t in range(40):
            tok = _tok(rc, slots, [t], edge)
            ref = orc.run(slots, tok)
            d = upload_tokens(tok, "f32", cuda_device, squeeze_t=True)
            o = torch.empty(R, HV, D, dtype=torch.float32, device=cuda_device)
            buf.recurrent_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
            assert_close(o.cpu().numpy(), ref[:, 0], TOL["f32"], f"{edge} recurrent {t}")
        _states(buf, orc, slots, TOL["f32"], f"{edge} recurrent")
