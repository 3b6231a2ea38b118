"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Independent fp64 implementations of the paper's alternative computation forms
of Gated DeltaNet, written in the paper's own row-vector convention
(q, k, v in R^{1 x d}, state S_p in R^{d_k x d_v}) and
converted to the north-star convention S = S_p^T only at the boundary
(reading Z1).  They exist to prove, in tests/test_oracle.py, that the
buffered forms the GPU path implements reach exactly (up to rounding) the
result of the recurrence in oracle/gdn_oracle.c.  The GPU path is never
compared against these.

Every function handles ONE sequence (one request slot x one V head).
Decay products are formed as the paper writes them, gamma_t = prod alpha
(P:374), with ratios gamma_t / gamma_i.
"""
from __future__ import annotations

import numpy as np


def _as64(*arrs):
    return [np.asarray(a, dtype=np.float64) for a in arrs]


def forward_substitution_inverse(Lstrict: np.ndarray) -> np.ndarray:
    """A = (I + L)^{-1} for strictly lower-triangular L by forward substitution
    (P:376/P:395 write A as this inverse; unit diagonal because L is strict).
    Solves (I + L) A = I column by column, row by row, ascending."""
    n = Lstrict.shape[0]
    A = np.zeros((n, n), dtype=np.float64)
    for c in range(n):
        for r in range(n):
            acc = 1.0 if r == c else 0.0
            for i in range(r):
                acc -= Lstrict[r, i] * A[i, c]
            A[r, c] = acc
    return A


def chunk_matrix_form(S0, Q, K, V, alpha, beta, printed_order=False):
    """Chunkwise matrix form of GDN, P:392-399 (eq:chunkwise_gdn_spec_verify),
    plus the chunk state update of P:407 in matrix form.

    gamma_t = prod_{i<=t} alpha_i        (chunk-local, Par(t) within the chunk)
    Gamma_ij = gamma_i / gamma_j, i >= j  (else 0)
    A  = [I + strictLower(Diag(beta)(Gamma o K K^T))]^{-1}   (Gram K K^T, reading Z5)
    K~ = A Diag(beta) Diag(gamma) K       (corrected order, reading Z4)
         Diag(gamma) A Diag(beta) K       (as printed at P:396, printed_order=True)
    V~ = A Diag(beta) V
    U  = V~ - K~ S_p
    O  = Diag(gamma) Q S_p + (Q K^T o Gamma) U
    S_p' = gamma_n S_p + sum_i (gamma_n / gamma_i) k_i^T u_i

    S0 is north-star [d_v, d_k]; returns dict with O [n, d_v], S [d_v, d_k]
    (north-star), U, A and the strict-lower matrix L.
    """
    S0, Q, K, V, alpha, beta = _as64(S0, Q, K, V, alpha, beta)
    Sp = S0.T
    n = Q.shape[0]
    gamma = np.cumprod(alpha)
    Gamma = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            Gamma[i, j] = gamma[i] / gamma[j]
    KK = K @ K.T
    L = np.tril(np.diag(beta) @ (Gamma * KK), k=-1)
    A = forward_substitution_inverse(L)
    if printed_order:
        Kt = np.diag(gamma) @ A @ np.diag(beta) @ K
    else:
        Kt = A @ np.diag(beta) @ np.diag(gamma) @ K
    Vt = A @ np.diag(beta) @ V
    U = Vt - Kt @ Sp
    O = np.diag(gamma) @ Q @ Sp + ((Q @ K.T) * Gamma) @ U
    if n:
        Sp_new = gamma[-1] * Sp + K.T @ (np.diag(gamma[-1] / gamma) @ U)
    else:
        Sp_new = Sp.copy()
    return {"O": O, "S": Sp_new.T.copy(), "U": U, "A": A, "L": L, "gamma": gamma}


def parallel_form(Q, K, V, alpha, beta):
    """GDN parallel form from a zero state, P:374-378 (eq:parallel_gdn_decoding):
    gamma over the whole prefix Par(t); O = (Q K^T o Gamma) A Diag(beta) V."""
    Q, K, V, alpha, beta = _as64(Q, K, V, alpha, beta)
    n = Q.shape[0]
    gamma = np.cumprod(alpha)
    Gamma = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            Gamma[i, j] = gamma[i] / gamma[j]
    L = np.tril(np.diag(beta) @ (Gamma * (K @ K.T)), k=-1)
    A = forward_substitution_inverse(L)
    Vt = A @ np.diag(beta) @ V
    return ((Q @ K.T) * Gamma) @ Vt


def chunkwise_decode(S0, Q, K, V, alpha, beta, C, flush_at_end=True):
    """Single-token chunkwise decoding against a deferred state, P:401-407
    (eq:chunkwise_gdn_decoding) with the subscripts read as in DESIGN.md Z2/Z3:
    gamma_t is the product of alpha from the first token after the last fold
    through t inclusive, and gamma_t/gamma_i pairs with k_i and u_i of the same
    buffered token i.  The buffer is folded into the state right after
    the step that fills it to C tokens (reading Z15).

      u_t = beta_t v_t - beta_t (gamma_t k_t S + sum_i (gamma_t/gamma_i)(k_t k_i^T) u_i)
      o_t = gamma_t q_t S + sum_{i<=t} (gamma_t/gamma_i)(q_t k_i^T) u_i
      S  <- gamma_t S + sum_i (gamma_t/gamma_i) k_i^T u_i     (at a fold)

    Returns (O [n, d_v], S_end north-star [d_v, d_k], fold_states list).
    """
    S0, Q, K, V, alpha, beta = _as64(S0, Q, K, V, alpha, beta)
    Sp = S0.T.copy()
    n = Q.shape[0]
    O = np.zeros((n, V.shape[1]))
    buf_k, buf_u, buf_g = [], [], []
    folds = []

    def fold():
        nonlocal Sp, buf_k, buf_u, buf_g
        if buf_k:
            g_last = buf_g[-1]
            new = g_last * Sp
            for ki, ui, gi in zip(buf_k, buf_u, buf_g):
                new = new + (g_last / gi) * np.outer(ki, ui)
            Sp = new
        buf_k, buf_u, buf_g = [], [], []
        folds.append(Sp.T.copy())

    for t in range(n):
        g_t = (buf_g[-1] if buf_g else 1.0) * alpha[t]
        k_t, q_t = K[t], Q[t]
        corr = g_t * (k_t @ Sp)
        for ki, ui, gi in zip(buf_k, buf_u, buf_g):
            corr = corr + (g_t / gi) * (k_t @ ki) * ui
        u_t = beta[t] * V[t] - beta[t] * corr
        o_t = g_t * (q_t @ Sp)
        for ki, ui, gi in zip(buf_k, buf_u, buf_g):
            o_t = o_t + (g_t / gi) * (q_t @ ki) * ui
        o_t = o_t + (q_t @ k_t) * u_t
        O[t] = o_t
        buf_k.append(k_t); buf_u.append(u_t); buf_g.append(g_t)
        if len(buf_k) == C:
            fold()
    if flush_at_end and buf_k:
        fold()
    return O, Sp.T.copy(), folds


def verify_then_commit(S0, Q, K, V, alpha, beta, n_acc):
    """Parallel draft verification and accepted-prefix commit, GDN version of
    P:173-177 (Eq. 7/8) via the chunkwise matrix form P:392-399 (reading Z18):
    outputs of all N drafts from the chunk form; the state is then updated once
    with the delta values of only the first n_acc drafts (P:407 restricted to
    the accepted prefix).  n_acc = 0 leaves the state untouched.
    Returns (O [N, d_v], S_commit north-star)."""
    res = chunk_matrix_form(S0, Q, K, V, alpha, beta)
    S0 = np.asarray(S0, dtype=np.float64)
    if n_acc == 0:
        return res["O"], S0.copy()
    Kp = np.asarray(K, dtype=np.float64)[:n_acc]
    U = res["U"][:n_acc]
    gamma = np.cumprod(np.asarray(alpha, dtype=np.float64)[:n_acc])
    Sp = S0.T
    Sp_new = gamma[-1] * Sp + Kp.T @ (np.diag(gamma[-1] / gamma) @ U)
    return res["O"], Sp_new.T.copy()


def vanilla_parallel(Q, K, V):
    """Vanilla linear attention parallel form, Eq. 1: O = ((Q K^T) o M) V
    with the causal mask M_ij = 1 for j <= i.  Brute force."""
    Q, K, V = _as64(Q, K, V)
    n = Q.shape[0]
    M = np.tril(np.ones((n, n)))
    return ((Q @ K.T) * M) @ V
