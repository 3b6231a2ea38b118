"""Pins for the fp64 oracle (CPU only).

The oracle (oracle/gdn_oracle.c) is the GDN recurrence of PAPER.md:362-365.
Each test below checks it against something other than itself: a closed form,
brute force, exact rational arithmetic in the paper's own row convention, or
an independently written alternative form from the paper (oracle/forms.py),
chosen so that a dropped term, a wrong sign or index, a transposed operand or
a wrong decay order fails at least one of them.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import forms

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def rand_seq(rng, n, d, alpha=(0.5, 1.0), beta=(0.0, 1.0), S0=True, unit=True):
    Q = rng.standard_normal((n, d))
    K = rng.standard_normal((n, d))
    if unit:
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
        K /= np.linalg.norm(K, axis=1, keepdims=True)
    V = rng.standard_normal((n, d))
    a = rng.uniform(alpha[0], alpha[1], n)
    b = rng.uniform(beta[0], beta[1], n)
    S = rng.standard_normal((d, d)) / np.sqrt(4 * d) if S0 else np.zeros((d, d))
    return S, Q, K, V, a, b


def run1(S, Q, K, V, a, b, bw=None):
    o, Se = oracle.gdn_run(S[None], Q[None], K[None], V[None], a[None], b[None],
                           None if bw is None else bw[None])
    return o[0], Se[0]


# ---------------------------------------------------------------- P1
def test_orthonormal_keys_closed_form():
    """P1 (north star): from S0 = 0 with orthonormal keys, S_{i-1} k_i = 0, so
    u_i = beta_i v_i and S_n = sum_i (prod_{l>i} alpha_l) beta_i v_i k_i^T."""
    rng = np.random.default_rng(11)
    d, n = 16, 12
    Kq, _ = np.linalg.qr(rng.standard_normal((d, d)))
    K = Kq[:, :n].T.copy()
    Q = rng.standard_normal((n, d))
    V = rng.standard_normal((n, d))
    a = rng.uniform(0.5, 1.0, n)
    b = rng.uniform(0.0, 1.0, n)
    o, S = run1(np.zeros((d, d)), Q, K, V, a, b)
    for t in range(n):
        St = np.zeros((d, d))
        for i in range(t + 1):
            St += np.prod(a[i + 1:t + 1]) * b[i] * np.outer(V[i], K[i])
        np.testing.assert_allclose(o[t], St @ Q[t], atol=1e-13, rtol=0)
    np.testing.assert_allclose(S, St, atol=1e-14, rtol=0)


# ---------------------------------------------------------------- P2
def test_vanilla_linear_attention_bruteforce():
    """P2 (reading Z7): alpha = 1, erase 0, write 1 is vanilla LA; its outputs
    equal the brute-force parallel form o_t = sum_{i<=t} (q_t k_i^T) v_i
    (Eq. 2) and ((Q K^T) o M) V (Eq. 1)."""
    rng = np.random.default_rng(12)
    d, n = 8, 20
    Q, K, V = (rng.standard_normal((n, d)) for _ in range(3))
    ones, zeros = np.ones(n), np.zeros(n)
    o, S = run1(np.zeros((d, d)), Q, K, V, ones, zeros, bw=ones)
    brute = np.zeros((n, d))
    for t in range(n):
        for i in range(t + 1):
            brute[t] += (Q[t] @ K[i]) * V[i]
    np.testing.assert_allclose(o, brute, atol=1e-12, rtol=0)
    np.testing.assert_allclose(o, forms.vanilla_parallel(Q, K, V), atol=1e-12, rtol=0)
    np.testing.assert_allclose(S, V.T @ K, atol=1e-12, rtol=0)  # S_t = sum v_i k_i^T


# ---------------------------------------------------------------- P3
def test_beta_zero_is_pure_decay():
    """P3 (reading Z7, literal): beta = 0 -> S_t = (prod alpha) S0, o_t = S_t q_t;
    with alpha = 1 as well the state is frozen."""
    rng = np.random.default_rng(13)
    S0, Q, K, V, a, _ = rand_seq(rng, 9, 8)
    o, S = run1(S0, Q, K, V, a, np.zeros(9))
    for t in range(9):
        np.testing.assert_allclose(o[t], np.prod(a[:t + 1]) * S0 @ Q[t], atol=1e-15, rtol=0)
    np.testing.assert_allclose(S, np.prod(a) * S0, atol=1e-15, rtol=0)
    o1, S1 = run1(S0, Q, K, V, np.ones(9), np.zeros(9))
    assert np.array_equal(S1, S0)


# ---------------------------------------------------------------- P4
def test_unit_key_overwrite():
    """P4 (SPEC gdn_recurrent_step example): alpha = beta = 1, the same unit key
    written with v1 then v2 from S = 0 retrieves exactly v2 (the delta rule
    replaces, (I - k^T k) k^T = 0)."""
    rng = np.random.default_rng(14)
    d = 8
    k = rng.standard_normal(d); k /= np.linalg.norm(k)
    v1, v2 = rng.standard_normal(d), rng.standard_normal(d)
    K = np.stack([k, k]); V = np.stack([v1, v2]); Q = np.stack([k, k])
    o, S = run1(np.zeros((d, d)), Q, K, V, np.ones(2), np.ones(2))
    np.testing.assert_allclose(S @ k, v2, atol=1e-14, rtol=0)
    np.testing.assert_allclose(o[0], v1, atol=1e-14, rtol=0)
    np.testing.assert_allclose(o[1], v2, atol=1e-14, rtol=0)


# ---------------------------------------------------------------- Z1 exact
def _paper_row_form_exact(Sp, qs, ks, vs, alphas, betas):
    """Paper convention, exact rationals: S~ = alpha S; S = (I - beta k^T k) S~
    + beta k^T v; o = q S, S_p is d_k x d_v."""
    d = len(ks[0])
    outs = []
    for q, k, v, al, be in zip(qs, ks, vs, alphas, betas):
        St = [[al * Sp[r][c] for c in range(d)] for r in range(d)]
        # (I - beta k^T k) St
        kS = [sum(k[r] * St[r][c] for r in range(d)) for c in range(d)]   # k S~ (1 x d_v)
        Sp = [[St[r][c] - be * k[r] * kS[c] + be * k[r] * v[c] for c in range(d)]
              for r in range(d)]
        outs.append([sum(q[r] * Sp[r][c] for r in range(d)) for c in range(d)])
    return outs, Sp


def test_exact_rational_tiny_paper_convention():
    """Reading Z1: the oracle's transposed (north-star) convention equals the
    paper's row-vector recurrence evaluated in exact rational arithmetic on
    dyadic inputs (so fp64 widening is exact)."""
    rng = np.random.default_rng(15)
    d, n = 3, 4
    def dy(x):  # dyadic rational with 8 fractional bits
        return Fraction(int(round(x * 256)), 256)
    Sp0 = [[dy(rng.uniform(-1, 1)) for _ in range(d)] for _ in range(d)]
    qs = [[dy(rng.uniform(-1, 1)) for _ in range(d)] for _ in range(n)]
    ks = [[dy(rng.uniform(-.7, .7)) for _ in range(d)] for _ in range(n)]
    vs = [[dy(rng.uniform(-1, 1)) for _ in range(d)] for _ in range(n)]
    al = [dy(rng.uniform(0.5, 1)) for _ in range(n)]
    be = [dy(rng.uniform(0, 1)) for _ in range(n)]
    outs, Sp = _paper_row_form_exact(Sp0, qs, ks, vs, al, be)
    f = lambda m: np.array([[float(x) for x in r] for r in m])
    o, S = run1(f(Sp0).T, f(qs), f(ks), f(vs), np.array([float(x) for x in al]),
                np.array([float(x) for x in be]))
    np.testing.assert_allclose(o, f(outs), atol=1e-14, rtol=0)
    np.testing.assert_allclose(S, f(Sp).T, atol=1e-14, rtol=0)


# ---------------------------------------------------------------- P5
def test_chunk_of_one_equals_one_step():
    """P5 (reading Z2): a chunk of one token, P:405-407 with j = 0:
    u = beta (v - alpha k S0), S1 = alpha S0 + k^T u, o = alpha q S0 + (q k^T) u
    equals one recurrent step; chunkwise decode with C = 1 equals recurrence."""
    rng = np.random.default_rng(16)
    S0, Q, K, V, a, b = rand_seq(rng, 1, 8)
    u = b[0] * (V[0] - a[0] * S0 @ K[0])
    S1 = a[0] * S0 + np.outer(u, K[0])
    o1 = a[0] * S0 @ Q[0] + (Q[0] @ K[0]) * u
    o, S = run1(S0, Q, K, V, a, b)
    np.testing.assert_allclose(S, S1, atol=1e-15, rtol=0)
    np.testing.assert_allclose(o[0], o1, atol=1e-15, rtol=0)
    S0, Q, K, V, a, b = rand_seq(rng, 13, 8)
    O, Se, _ = forms.chunkwise_decode(S0, Q, K, V, a, b, C=1)
    o, S = run1(S0, Q, K, V, a, b)
    np.testing.assert_allclose(O, o, atol=1e-13, rtol=0)
    np.testing.assert_allclose(Se, S, atol=1e-13, rtol=0)


# ---------------------------------------------------------------- P6
@pytest.mark.parametrize("seed", range(5))
def test_matrix_chunk_form_corrected_equals_recurrence(seed):
    """P6 (readings Z4, Z5): the chunkwise matrix form of P:392-399 with the
    corrected K~ = A Diag(beta) Diag(gamma) K and Gram K K^T equals the
    recurrence, outputs and state."""
    rng = np.random.default_rng(100 + seed)
    S0, Q, K, V, a, b = rand_seq(rng, 6 + seed, 8)
    res = forms.chunk_matrix_form(S0, Q, K, V, a, b)
    o, S = run1(S0, Q, K, V, a, b)
    np.testing.assert_allclose(res["O"], o, atol=1e-13, rtol=0)
    np.testing.assert_allclose(res["S"], S, atol=1e-13, rtol=0)


def test_matrix_chunk_form_printed_order_is_wrong():
    """Regression for reading Z4: K~ = Diag(gamma) A Diag(beta) K as printed
    at P:396 does NOT reproduce the recurrence when alpha varies."""
    rng = np.random.default_rng(17)
    S0, Q, K, V, a, b = rand_seq(rng, 6, 8)
    res = forms.chunk_matrix_form(S0, Q, K, V, a, b, printed_order=True)
    o, _ = run1(S0, Q, K, V, a, b)
    assert np.max(np.abs(res["O"] - o)) > 1e-3


# ---------------------------------------------------------------- P7
@pytest.mark.parametrize("n", [1, 5, 24])
def test_parallel_form_equals_recurrence(n):
    """P7: the parallel form from a zero state equals the
    recurrence (direct short-context decoding)."""
    rng = np.random.default_rng(200 + n)
    _, Q, K, V, a, b = rand_seq(rng, n, 8, S0=False)
    o, _ = run1(np.zeros((8, 8)), Q, K, V, a, b)
    np.testing.assert_allclose(forms.parallel_form(Q, K, V, a, b), o, atol=1e-13, rtol=0)


def test_parallel_all_beta_zero_is_zero():
    rng = np.random.default_rng(18)
    _, Q, K, V, a, _ = rand_seq(rng, 7, 8, S0=False)
    o, _ = run1(np.zeros((8, 8)), Q, K, V, a, np.zeros(7))
    assert np.all(o == 0.0)
    assert np.all(forms.parallel_form(Q, K, V, a, np.zeros(7)) == 0.0)


# ---------------------------------------------------------------- P8
@pytest.mark.parametrize("C", [1, 2, 4, 7, 16])
def test_incremental_chunkwise_decode_equals_recurrence(C):
    """P8 (reading Z3): single-token chunkwise decoding with a deferred state
    and folds every C tokens equals the recurrence, including the
    state after each fold and a ragged final partial chunk."""
    rng = np.random.default_rng(300 + C)
    n = 37
    S0, Q, K, V, a, b = rand_seq(rng, n, 16)
    O, Se, folds = forms.chunkwise_decode(S0, Q, K, V, a, b, C=C)
    o, S = run1(S0, Q, K, V, a, b)
    np.testing.assert_allclose(O, o, atol=1e-12, rtol=0)
    np.testing.assert_allclose(Se, S, atol=1e-12, rtol=0)
    for f_i, Sf in enumerate(folds[:-1] if n % C else folds):
        t = (f_i + 1) * C
        _, Sref = run1(S0, Q[:t], K[:t], V[:t], a[:t], b[:t])
        np.testing.assert_allclose(Sf, Sref, atol=1e-12, rtol=0)


# ---------------------------------------------------------------- P9
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_verify_then_commit_every_nacc(N):
    """P9: parallel verification outputs of all N drafts equal the recurrence;
    committing the accepted prefix of every length n_acc in [0, N] gives the
    recurrence's state after exactly n_acc drafts; n_acc = 0 is bit-identical."""
    rng = np.random.default_rng(400 + N)
    S0, Q, K, V, a, b = rand_seq(rng, N, 16)
    o_all, _ = run1(S0, Q, K, V, a, b)
    for n_acc in range(N + 1):
        O, Sc = forms.verify_then_commit(S0, Q, K, V, a, b, n_acc)
        np.testing.assert_allclose(O, o_all, atol=1e-13, rtol=0)
        _, Sref = run1(S0, Q[:n_acc], K[:n_acc], V[:n_acc], a[:n_acc], b[:n_acc])
        if n_acc == 0:
            assert np.array_equal(Sc, S0) and np.array_equal(Sref, S0)
        np.testing.assert_allclose(Sc, Sref, atol=1e-13, rtol=0)


def test_verify_outputs_causal():
    """Draft t's output does not depend on drafts after t (causality)."""
    rng = np.random.default_rng(19)
    S0, Q, K, V, a, b = rand_seq(rng, 6, 8)
    O1 = forms.chunk_matrix_form(S0, Q, K, V, a, b)["O"]
    V2 = V.copy(); V2[4:] += 1.0
    K2 = K.copy(); K2[5] = -K2[5]
    O2 = forms.chunk_matrix_form(S0, Q, K2, V2, a, b)["O"]
    np.testing.assert_allclose(O1[:4], O2[:4], atol=1e-14, rtol=0)


# ---------------------------------------------------------------- P10
def test_A_residual_and_gamma_monotone_and_chunk_boundaries():
    """P10 (SPEC gdn_core invariants): (I + L) A = I to 1e-10; chunk-local
    gamma non-increasing for alpha in (0, 1]; splitting a sequence into chunks
    at arbitrary boundaries gives the same final state."""
    rng = np.random.default_rng(20)
    S0, Q, K, V, a, b = rand_seq(rng, 32, 16)
    res = forms.chunk_matrix_form(S0, Q, K, V, a, b)
    n = 32
    assert np.max(np.abs((np.eye(n) + res["L"]) @ res["A"] - np.eye(n))) <= 1e-10
    assert np.all(np.diff(res["gamma"]) <= 0)
    _, Sref = run1(S0, Q, K, V, a, b)
    for cuts in ([0, 5, 6, 19, 32], [0, 32], [0, 1, 2, 3, 31, 32]):
        S = S0
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            S = forms.chunk_matrix_form(S, Q[lo:hi], K[lo:hi], V[lo:hi], a[lo:hi], b[lo:hi])["S"]
        np.testing.assert_allclose(S, Sref, atol=1e-12, rtol=0)


# ---------------------------------------------------------------- harness
def test_zero_tokens_and_threads_invariance():
    rng = np.random.default_rng(21)
    S0, Q, K, V, a, b = rand_seq(rng, 5, 8)
    S0s = np.stack([S0] * 7); Qs = np.stack([Q] * 7); Ks = np.stack([K] * 7)
    Vs = np.stack([V] * 7); As = np.stack([a] * 7); Bs = np.stack([b] * 7)
    o1, S1 = oracle.gdn_run(S0s, Qs, Ks, Vs, As, Bs, n_threads=1)
    o4, S4 = oracle.gdn_run(S0s, Qs, Ks, Vs, As, Bs, n_threads=4)
    assert np.array_equal(o1, o4) and np.array_equal(S1, S4)
    o0, S0e = oracle.gdn_run(S0s, Qs[:, :0], Ks[:, :0], Vs[:, :0], As[:, :0], Bs[:, :0])
    assert o0.shape == (7, 0, 8) and np.array_equal(S0e, S0s)


def test_qwen_shape_d128_forms():
    """The equivalences hold at the real head dimension d = 128."""
    rng = np.random.default_rng(22)
    S0, Q, K, V, a, b = rand_seq(rng, 20, 128, alpha=(0.9, 1.0))
    O, Se, _ = forms.chunkwise_decode(S0, Q, K, V, a, b, C=16)
    o, S = run1(S0, Q, K, V, a, b)
    np.testing.assert_allclose(O, o, atol=1e-12, rtol=0)
    np.testing.assert_allclose(Se, S, atol=1e-12, rtol=0)
