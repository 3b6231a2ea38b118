"""Paged KV-buffer pool, state pool and mixed-form index-array batches
("allocates the KV buffer for a request from a pool
of memory shared system-wide ... a block, which can store 8 or 16 KVs",
P:205 dynamic blocks for KV-only contexts, P:207 compression once L >= d,
P:323-325 interleaving decoding forms in one batch).

Every output and every exported state is compared with the fp64 oracle at
the north-star tolerance; the pool counters obey the SPEC invariants
(conservation, exclusive ownership, all-or-nothing on exhaustion)."""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV = 16, 32


def _paged(R, C, N=0, short_cap=0, bt=8, n_blocks=None, states=None, u_dtype="f32", in_dtype="bf16",
           device="cuda"):
    T = (max(C + N, short_cap) + 3) // 4 * 4
    n_blocks = R * ((T + bt - 1) // bt) if n_blocks is None else n_blocks
    cfg = L.make_config(R, HK, HV, chunk=C, max_drafts=N, short_cap=short_cap, in_dtype=in_dtype,
                        u_dtype=u_dtype, validate=True, block_tokens=bt, n_blocks=n_blocks,
                        state_slots=R if states is None else states)
    return L.LaBuf(cfg, device=device)


def _held(buf, R):
    info = [buf.pool_info(r) for r in range(R)]
    return sum(i["slot_blocks"] for i in info), [i["slot_state"] for i in info]


def _invariants(buf, R):
    p = buf.pool_info()
    held, states = _held(buf, R)
    assert p["free_blocks"] + held == p["total_blocks"]
    live = [s for s in states if s >= 0]
    assert len(live) == len(set(live))                       # a state belongs to one slot
    assert p["free_states"] + len(live) == p["total_states"]


def test_paged_decode_verify_commit(cuda_device):
    """Chunkwise decode cycles, parallel verify + commit on a paged handle
    (blocks of 8 records, a state pool): outputs and states vs the oracle."""
    rc = synth.Recipe(seed=3101, dist="qwen", in_dtype="bf16")
    R, C, N = 5, 16, 4
    tol = TOL["bf16"]
    buf = _paged(R, C, N=N, bt=8)
    slots = np.arange(R)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    _invariants(buf, R)
    for t in range(C + 5):
        tok = synth.tokens(rc, slots, [t], HK, HV, 128)
        ref = orc.run(slots, tok)
        d = upload_tokens(tok, "bf16", cuda_device, squeeze_t=True)
        o = torch.empty(R, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        buf.flush(0, R, L.LA_FLUSH_FULL)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"paged decode {t}")
        _invariants(buf, R)
    # (5 records stay buffered; the first commit folds them with the accepted drafts)
    # verify 4 drafts on top of 5 buffered records (positions 5..8 cross a block edge), commit
    for rnd in range(3):
        tok = synth.tokens(rc, slots, np.arange(100 + 10 * rnd, 100 + 10 * rnd + N), HK, HV, 128)
        n_acc = synth.n_accepted(rc, slots, N, round_idx=rnd)
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, "bf16", cuda_device)
        o = torch.empty(R, N, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        buf.commit_accepted(0, torch.from_numpy(n_acc).to(cuda_device))
        assert_close(o.cpu().numpy(), ref, tol, f"paged verify round {rnd}")
        for s in slots:
            assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"paged commit {rnd} slot {s}")
        _invariants(buf, R)
    flags, _ = buf.device_status()
    assert flags == 0


@pytest.mark.parametrize("u_dtype", ["f16", "f32"])
def test_mixed_batches_route_and_compress(cuda_device, u_dtype):
    """la_decode_mixed over index-array batches in shuffled order with slots
    dropping in and out: chunkwise slots decode from their state (eager flush
    when a buffer fills), KV-only slots from their records only, and a KV-only
    slot whose context reaches short_cap is compressed into a state from the
    pool and continues chunkwise -- all against the oracle."""
    rc = synth.Recipe(seed=3202, dist="stress", in_dtype="bf16")
    R, C, cap = 8, 8, 32
    tol = TOL["bf16"]
    buf = _paged(R, C, short_cap=cap, bt=8, states=6, u_dtype=u_dtype)
    long_s, short_s = np.arange(4), np.arange(4, 8)
    buf.reset(0, 4, mode=L.LA_MODE_CHUNKWISE, zero_state=False)
    buf.reset(4, 4, mode=L.LA_MODE_DIRECT, zero_state=False)
    S0 = np.zeros((R, HV, 128, 128))
    S0[long_s] = synth.state0(rc, long_s, HV, 128, 128)
    set_states(buf, S0[long_s], long_s)
    orc = Oracle(S0)
    _invariants(buf, R)
    assert buf.pool_info()["free_states"] == 2
    # KV-only prefills of ragged lengths
    L0 = {4: 1, 5: 9, 6: 24, 7: 31}
    for r, l0 in L0.items():
        tok = synth.tokens(rc, [r], np.arange(l0), HK, HV, 128)
        ref = orc.run([r], tok)
        d = upload_tokens(tok, "bf16", cuda_device)
        o = torch.empty(1, l0, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.direct_short(r, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref, tol, f"kv-only prefill {r}")
    _invariants(buf, R)
    rng = np.random.default_rng(5)
    pos = {r: 1000 for r in range(R)}
    for step in range(14):
        batch = rng.permutation(R)
        if step % 3 == 1:                      # a slot sits this step out
            batch = batch[1:]
        tok = synth.tokens(rc, batch, [0], HK, HV, 128)
        # each slot's own token position (the generator keys on (slot, position))
        for i, r in enumerate(batch):
            one = synth.tokens(rc, [r], [pos[r]], HK, HV, 128)
            for k_ in tok:
                tok[k_][i] = one[k_][0]
            pos[r] += 1
        ref = orc.run(batch, tok)
        d = upload_tokens(tok, "bf16", cuda_device, squeeze_t=True)
        o = torch.empty(len(batch), HV, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_mixed(batch, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        assert_close(o.cpu().numpy(), ref[:, 0], tol, f"mixed step {step}")
        _invariants(buf, R)
    # slots 6 and 7 reached short_cap and were compressed; all states vs the oracle
    modes = [buf.slot_info(r).mode for r in range(R)]
    assert modes[6] == L.LA_MODE_CHUNKWISE and modes[7] == L.LA_MODE_CHUNKWISE, modes
    assert modes[4] == L.LA_MODE_DIRECT and modes[5] == L.LA_MODE_DIRECT
    assert buf.pool_info()["free_states"] == 0
    chunk = [r for r in range(R) if modes[r] == L.LA_MODE_CHUNKWISE]
    for r in chunk:
        buf.flush(r, 1, L.LA_FLUSH_FORCE)
        assert_close(buf.state_get(r).cpu().numpy(), orc.S[r], tol, f"state after mixed steps, slot {r}")
    flags, (occ, ln, mode) = buf.device_status()
    assert flags == 0
    assert mode == modes and ln == [buf.slot_info(r).len for r in range(R)]
    # release returns everything
    buf.release(0, R)
    p = buf.pool_info()
    assert p["free_blocks"] == p["total_blocks"] and p["free_states"] == p["total_states"]


def test_pool_exhaustion_is_all_or_nothing(cuda_device):
    """A call that needs more blocks (or states) than the pool has fails with
    LA_ERR_CAPACITY before enqueueing anything: counters, pools and device
    state unchanged; after a release the same call succeeds."""
    rc = synth.Recipe(seed=3303, dist="qwen", in_dtype="bf16")
    R, C = 4, 8
    buf = _paged(R, C, short_cap=16, bt=4, n_blocks=6, states=1)
    buf.reset(0, R, mode=L.LA_MODE_DIRECT, zero_state=False)
    slots = np.arange(R)
    tok = synth.tokens(rc, slots, np.arange(5), HK, HV, 128)      # 5 records = 2 blocks per slot: 8 > 6
    d = upload_tokens(tok, "bf16", cuda_device)
    o = torch.empty(R, 5, HV, 128, dtype=torch.float32, device=cuda_device)
    before = (buf.pool_info(), [buf.slot_info(r) for r in slots])
    with pytest.raises(L.LaError) as ei:
        buf.direct_short(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert ei.value.status == L.LA_ERR_CAPACITY
    assert (buf.pool_info(), [buf.slot_info(r) for r in slots]) == before
    # only one state: two slots cannot both become CHUNKWISE
    with pytest.raises(L.LaError) as ei:
        buf.reset(0, 2, mode=L.LA_MODE_CHUNKWISE)
    assert ei.value.status == L.LA_ERR_CAPACITY
    assert buf.pool_info() == before[0]
    # three slots fit (6 blocks); the fourth then fails; release one and it fits
    orc = Oracle(np.zeros((R, HV, 128, 128)))
    ref = orc.run(slots[:3], {k_: v_[:3] for k_, v_ in tok.items()})
    o3 = torch.empty(3, 5, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.direct_short(0, *(d[k_][:3].contiguous() for k_ in ("q", "k", "v", "alpha", "beta")), o3)
    assert_close(o3.cpu().numpy(), ref, TOL["bf16"], "3 slots")
    assert buf.pool_info()["free_blocks"] == 0
    one = {k_: d[k_][3:].contiguous() for k_ in d}
    o1 = torch.empty(1, 5, HV, 128, dtype=torch.float32, device=cuda_device)
    with pytest.raises(L.LaError):
        buf.direct_short(3, one["q"], one["k"], one["v"], one["alpha"], one["beta"], o1)
    buf.release(0, 1)
    buf.direct_short(3, one["q"], one["k"], one["v"], one["alpha"], one["beta"], o1)
    ref1 = Oracle(np.zeros((1, HV, 128, 128))).run([0], {k_: v_[3:] for k_, v_ in tok.items()})
    assert_close(o1.cpu().numpy(), ref1, TOL["bf16"], "slot 3 after release")


def test_block_and_state_ids_are_deterministic(cuda_device):
    """The same call sequence gives the same state ids (LIFO over ascending
    initial order, SPEC buffer_manager design decision)."""
    ids = []
    for rep in range(2):
        buf = _paged(6, 8, short_cap=16, bt=8, states=4)
        buf.reset(0, 6, mode=L.LA_MODE_DIRECT, zero_state=False)
        buf.reset(1, 1, mode=L.LA_MODE_CHUNKWISE)
        buf.reset(3, 2, mode=L.LA_MODE_CHUNKWISE)
        buf.release(3, 1)
        buf.reset(5, 1, mode=L.LA_MODE_CHUNKWISE)
        ids.append([buf.pool_info(r)["slot_state"] for r in range(6)])
    assert ids[0] == ids[1] == [-1, 0, -1, -1, 2, 1]


@pytest.mark.parametrize("in_dtype,bt", [("bf16", 16), ("f32", 8)])
def test_paged_prefill_self_fold(cuda_device, in_dtype, bt):
    """Prefill on a paged handle with a state pool whose slot -> state map is
    not the identity: 16-token chunks fold their own records into the pooled
    state (TMA stores through the state index) and a ragged tail; outputs,
    states and the next decode step vs the oracle."""
    rc = synth.Recipe(seed=3150 + bt, dist="stress", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    R, C, n_tok = 4, 16, 77
    buf = _paged(R, C, bt=bt, in_dtype=in_dtype, states=R + 2)
    # states handed out in reverse slot order: slot r -> state R - 1 - r (+ the spares stay free)
    for r in reversed(range(R)):
        buf.reset(r, 1, zero_state=False)
    assert [buf.pool_info(r)["slot_state"] for r in range(R)] == list(reversed(range(R)))
    allslots = np.arange(R)
    S0 = synth.state0(rc, allslots, HV, 128, 128)
    set_states(buf, S0, allslots)
    orc = Oracle(S0)
    slots = np.arange(1, R)                       # a range that does not start at slot 0
    tok = synth.tokens(rc, slots, np.arange(n_tok), HK, HV, 128)
    ref = orc.run(slots, tok)
    d = upload_tokens(tok, in_dtype, cuda_device)
    o = torch.empty(len(slots), n_tok, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.prefill(1, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), ref, tol, "paged prefill outputs")
    for s in allslots:   # (slot 0 untouched)
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"paged prefill state, slot {s}")
    nxt = synth.tokens(rc, slots, [n_tok], HK, HV, 128)
    r1 = orc.run(slots, nxt)
    d1 = upload_tokens(nxt, in_dtype, cuda_device, squeeze_t=True)
    o1 = torch.empty(len(slots), HV, 128, dtype=torch.float32, device=cuda_device)
    buf.decode_step(1, d1["q"], d1["k"], d1["v"], d1["alpha"], d1["beta"], o1)
    assert_close(o1.cpu().numpy(), r1[:, 0], tol, "decode after paged prefill")
    _invariants(buf, R)
    flags, (occ, _, _) = buf.device_status()
    assert flags == 0 and occ[1:] == [1] * (R - 1)
