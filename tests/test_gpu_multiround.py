"""Multi-round buffered speculation and state fork.

* la_commit_append: the accepted prefix stays buffered (its records are the
  recurrence's records), the state is folded only when the buffer
  could not take another round -- every round's draft outputs and the states
  after the folds against the oracle; the host keeps an occupancy bound and
  refuses calls that need the exact count.
* la_state_fork: the state after the first n buffered records of one slot
  becomes another slot's state -- from a CHUNKWISE slot (S0 + prefix) and
  from a KV-only slot (the state rebuilt from cached KVs alone, the
  prefix-caching design of P:330-331)."""
import numpy as np
import pytest
import torch

import synth
from harness import TOL, Oracle, assert_close, set_states, upload_tokens
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV = 16, 32


@pytest.mark.parametrize("in_dtype", ["bf16", "f32"])
def test_append_commit_rounds(cuda_device, in_dtype):
    rc = synth.Recipe(seed=3501, dist="qwen", in_dtype=in_dtype)
    tol = TOL[in_dtype]
    R, C, N = 4, 16, 4
    cfg = L.make_config(R, HK, HV, chunk=C, max_drafts=N, in_dtype=in_dtype, validate=True)
    buf = L.LaBuf(cfg, device=cuda_device)
    slots = np.arange(R)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    occ_true = np.zeros(R, dtype=int)
    folds = 0
    for rnd in range(9):
        tok = synth.tokens(rc, slots, np.arange(10 * rnd, 10 * rnd + N), HK, HV, 128)
        n_acc = synth.n_accepted(rc, slots, N, round_idx=rnd)
        ref = orc.run(slots, tok, n_acc=n_acc)
        d = upload_tokens(tok, in_dtype, cuda_device)
        o = torch.empty(R, N, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.verify_drafts(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
        before = buf.kernel_launches()
        buf.commit_append(0, torch.from_numpy(n_acc).to(cuda_device))
        assert_close(o.cpu().numpy(), ref, tol, f"append round {rnd}")
        info = buf.slot_info(0)
        if info.occ == 0:          # this commit folded: the states are comparable
            folds += 1
            occ_true[:] = 0
            for s in slots:
                assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"fold after round {rnd}, slot {s}")
        else:
            occ_true += n_acc
            assert buf.kernel_launches() == before + 1          # one tiny counter kernel, no fold
            _, (occ, _, _) = buf.device_status()
            assert occ == list(occ_true)                         # device counters: exact
            with pytest.raises(L.LaError) as ei:                 # host: only a bound
                buf.flush(0, R, L.LA_FLUSH_FULL)
            assert ei.value.status == L.LA_ERR_MODE
    assert folds >= 1
    buf.flush(0, R, L.LA_FLUSH_FORCE)
    for s in slots:
        assert_close(buf.state_get(int(s)).cpu().numpy(), orc.S[s], tol, f"final state slot {s}")


def test_state_fork_from_prefix_and_from_kvs(cuda_device):
    rc = synth.Recipe(seed=3502, dist="stress", in_dtype="bf16")
    tol = TOL["bf16"]
    R, C = 4, 16
    cfg = L.make_config(R, HK, HV, chunk=C, short_cap=32, validate=True)
    buf = L.LaBuf(cfg, device=cuda_device)
    buf.reset(0, 2, mode=L.LA_MODE_CHUNKWISE, zero_state=False)
    buf.reset(2, 2, mode=L.LA_MODE_DIRECT, zero_state=False)
    S0 = synth.state0(rc, [0], HV, 128, 128)
    set_states(buf, S0, [0])
    # slot 0: 10 buffered decode records on top of S0
    tok = synth.tokens(rc, [0], np.arange(10), HK, HV, 128)
    for t in range(10):
        d = upload_tokens({k_: v_[:, t:t + 1] for k_, v_ in tok.items()}, "bf16", cuda_device, squeeze_t=True)
        o = torch.empty(1, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    # fork the state after 6 of them into slot 1
    buf.reset(1, 1, mode=L.LA_MODE_CHUNKWISE, zero_state=True)
    buf.state_fork(0, 1, 6)
    ref = Oracle(S0)
    ref.run([0], {k_: v_[:, :6] for k_, v_ in tok.items()}, want_o=False)
    assert_close(buf.state_get(1).cpu().numpy(), ref.S[0], tol, "fork of a 6-record prefix")
    assert buf.slot_info(0).occ == 10                     # the source is untouched
    # slot 2: 20 KV-only tokens; rebuild the state of its first 13 into slot 3
    kv = synth.tokens(rc, [2], np.arange(20), HK, HV, 128)
    d = upload_tokens(kv, "bf16", cuda_device)
    o = torch.empty(1, 20, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.direct_short(2, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    buf.reset(3, 1, mode=L.LA_MODE_CHUNKWISE, zero_state=True)
    buf.state_fork(2, 3, 13)
    ref3 = Oracle(np.zeros((1, HV, 128, 128)))
    ref3.run([0], {k_: v_[:, :13] for k_, v_ in kv.items()}, want_o=False)
    assert_close(buf.state_get(3).cpu().numpy(), ref3.S[0], tol, "state rebuilt from 13 cached KVs")
    # the rebuilt slot decodes on from there
    nxt = synth.tokens(rc, [3], [100], HK, HV, 128)
    r_o = ref3.run([0], nxt)
    d = upload_tokens(nxt, "bf16", cuda_device, squeeze_t=True)
    o = torch.empty(1, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.decode_step(3, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    assert_close(o.cpu().numpy(), r_o[:, 0], tol, "decode after the rebuild")
    with pytest.raises(L.LaError):
        buf.state_fork(2, 3, 21)                           # more records than the source holds


@pytest.mark.parametrize("n_branch,n_draft", [(3, 4), (4, 2), (2, 8)])
def test_branch_verify_and_commit(cuda_device, n_branch, n_draft):
    """Beam/branch candidates: n_branch branches of n_draft tokens
    from the same prefix (state + 3 buffered records) verified in one launch,
    each branch's outputs equal to the recurrence over that branch alone; the
    accepted branch's prefix is folded, the others never touch the state."""
    rc = synth.Recipe(seed=3503 + n_branch, dist="stress", in_dtype="bf16")
    tol = TOL["bf16"]
    R, C = 3, 16
    tot = n_branch * n_draft
    cfg = L.make_config(R, HK, HV, chunk=C, max_drafts=16, validate=True)
    buf = L.LaBuf(cfg, device=cuda_device)
    slots = np.arange(R)
    buf.reset(zero_state=False)
    S0 = synth.state0(rc, slots, HV, 128, 128)
    set_states(buf, S0, slots)
    orc = Oracle(S0)
    pre = synth.tokens(rc, slots, np.arange(3), HK, HV, 128)        # 3 buffered records
    orc.run(slots, pre, want_o=False)
    for t in range(3):
        d = upload_tokens({k_: v_[:, t:t + 1] for k_, v_ in pre.items()}, "bf16", cuda_device, squeeze_t=True)
        o = torch.empty(R, HV, 128, dtype=torch.float32, device=cuda_device)
        buf.decode_step(0, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    tok = synth.tokens(rc, slots, np.arange(100, 100 + tot), HK, HV, 128)   # branch-major
    d = upload_tokens(tok, "bf16", cuda_device)
    o = torch.empty(R, tot, HV, 128, dtype=torch.float32, device=cuda_device)
    buf.verify_branches(0, n_branch, d["q"], d["k"], d["v"], d["alpha"], d["beta"], o)
    got = o.cpu().numpy()
    for bb in range(n_branch):
        sub = {k_: v_[:, bb * n_draft:(bb + 1) * n_draft] for k_, v_ in tok.items()}
        ref = Oracle(orc.S.copy()).run(slots, sub)
        assert_close(got[:, bb * n_draft:(bb + 1) * n_draft], ref, tol, f"branch {bb} outputs")
    branch = np.array([r % n_branch for r in range(R)], dtype=np.int32)
    n_acc = synth.n_accepted(rc, slots, n_draft, round_idx=9)
    buf.commit_branch(0, torch.from_numpy(branch).to(cuda_device), torch.from_numpy(n_acc).to(cuda_device))
    for i, s in enumerate(slots):
        bb = branch[i]
        sub = {k_: v_[i:i + 1, bb * n_draft:bb * n_draft + n_acc[i]] for k_, v_ in tok.items()}
        ref = Oracle(orc.S[[s]].copy())
        if n_acc[i]:
            ref.run([0], sub, want_o=False)
        assert_close(buf.state_get(int(s)).cpu().numpy(), ref.S[0], tol, f"slot {s}: branch {bb}, {n_acc[i]} accepted")
    assert buf.slot_info(0).occ == 0 and buf.slot_info(0).pending == 0
    flags, _ = buf.device_status()
    assert flags == 0
