"""Shared test harness: runs the same seeded inputs through the CUDA library
(via the C ABI binding) and through the fp64 oracle, and compares.

The oracle side only ever sees the stored input values produced by synth/;
nothing computed by the CUDA path is fed to it.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth
from paper_2605_19049_b200 import labuf as L

TOL = {"bf16": 2e-3, "f32": 1e-5}   # north-star max-abs tolerances


def to_dev(x, dtype, device):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device, dtype=dtype)


class Oracle:
    """fp64 reference states for slots x V heads (north-star [d_v, d_k])."""

    def __init__(self, S0: np.ndarray, variant: str = "gdn"):   # [R, Hv, d, d]
        """variant: 'gdn' (the recurrence P:362-365), 'gated' (alpha S + v k^T:
        erase coefficient 0, write 1) or 'vanilla' (S + v k^T: alpha 1,
        erase 0, write 1) -- the oracle's separate erase / write coefficients."""
        self.S = np.array(S0, dtype=np.float64, copy=True)
        self.variant = variant

    def run(self, slots, tok, n_acc=None, want_o=True):
        """Advance `slots` by the tokens in tok (arrays [n, T, ...] from
        synth.tokens).  Returns outputs [n, T, Hv, d] (fp64).  If n_acc is
        given (array [n]), outputs cover all T tokens but each slot's state
        advances by only n_acc[i] of them (verify-then-commit semantics)."""
        slots = np.asarray(slots)
        n, T, Hv = tok["v"].shape[:3]
        d = tok["v"].shape[3]
        qv = synth.expand_qk_to_v_heads(tok["q"], Hv)       # [n,T,Hv,d]
        kv = synth.expand_qk_to_v_heads(tok["k"], Hv)
        def seq(x):   # [n,T,Hv,...] -> [n*Hv, T, ...]
            return np.ascontiguousarray(np.swapaxes(x, 1, 2).reshape((n * Hv, T) + x.shape[3:]))
        S = self.S[slots].reshape(n * Hv, d, d)
        alpha, beta_e, beta_w = seq(tok["alpha"]), seq(tok["beta"]), None
        if self.variant != "gdn":
            beta_e, beta_w = np.zeros_like(beta_e), np.ones_like(beta_e)
            if self.variant == "vanilla":
                alpha = np.ones_like(alpha)
        o, S_end = oracle.gdn_run(S, seq(qv), seq(kv), seq(tok["v"]), alpha, beta_e, beta_w=beta_w,
                                  want_o=want_o)
        out = None if o is None else np.swapaxes(o.reshape(n, Hv, T, d), 1, 2)
        if n_acc is None:
            self.S[slots] = S_end.reshape(n, Hv, d, d)
        else:
            for i, s in enumerate(slots):
                m = int(n_acc[i])
                if m == 0:
                    continue
                sub = {k_: v_[i:i + 1, :m] for k_, v_ in tok.items()}
                saved = self.S[[s]].copy()
                o2 = Oracle(saved, self.variant)
                o2.run([0], sub, want_o=False)
                self.S[s] = o2.S[0]
        return out


def max_abs(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise AssertionError(f"shape mismatch {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    d = np.abs(a - b)
    if not np.all(np.isfinite(a)):
        return float("inf")
    return float(d.max())


def assert_close(gpu, ref, tol, what=""):
    err = max_abs(gpu, ref)
    assert err <= tol, f"{what}: max-abs error {err:.3e} > {tol:.1e}"
    return err


def make_buf(R, Hk, Hv, C=16, N=0, short_cap=0, in_dtype="bf16", u_dtype="f32", keep_raw=False,
             validate=True, device="cuda"):
    cfg = L.make_config(R, Hk, Hv, chunk=C, max_drafts=N, short_cap=short_cap,
                        in_dtype=in_dtype, u_dtype=u_dtype, keep_raw=keep_raw, validate=validate)
    return L.LaBuf(cfg, device=device)


def upload_tokens(tok, in_dtype, device, squeeze_t=False):
    tdt = torch.bfloat16 if in_dtype == "bf16" else torch.float32
    out = {}
    for name in ("q", "k", "v"):
        out[name] = to_dev(tok[name], tdt, device)
    for name in ("alpha", "beta"):
        out[name] = to_dev(tok[name], torch.float32, device)
    if squeeze_t:
        out = {k: v[:, 0].contiguous() for k, v in out.items()}
    return out


def set_states(buf, S0, slots):
    """Write fp32 start states [n, Hv, d, d] into the given slots."""
    for i, s in enumerate(slots):
        buf.state_set(int(s), to_dev(S0[i], torch.float32, buf.device))
