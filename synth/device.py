"""Seeded synthetic inputs drawn on the GPU, for full-size (BASELINE) runs.

Same distributions as :mod:`synth`: q, k ~ N(0,1)
L2-normalised per head (q additionally scaled by d^-1/2 for 'qwen'), v ~ N(0,1),
alpha ~ U(alpha_lo, 1], beta = sigmoid(N(0,1)), S0 ~ N(0, 1/(4 d_k)); values
rounded to the stored dtype.  Drawn with torch's seeded device generator, so a
64-slot or 1024-slot batch takes milliseconds instead of the counter-based
generator's minutes.  Like :mod:`synth` it holds none of the method's
arithmetic: it only produces stored input values, which the CUDA path and the
oracle (tests copy the sampled slots to the host) then both consume
unchanged.
"""
from __future__ import annotations

import torch

D = 128


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def tokens(seed, n_slots, n_tok, n_qk_heads, n_v_heads, d=D, in_dtype="bf16", device="cuda",
           dist="qwen", alpha_lo=0.9, squeeze=False):
    """q, k [n, T, Hk, d], v [n, T, Hv, d] in in_dtype; alpha, beta [n, T, Hv] fp32.
    squeeze=True drops the token axis (T must be 1)."""
    g = _gen(seed, device)
    tdt = torch.bfloat16 if in_dtype == "bf16" else torch.float32
    q = torch.randn(n_slots, n_tok, n_qk_heads, d, generator=g, device=device, dtype=torch.float64)
    k = torch.randn(n_slots, n_tok, n_qk_heads, d, generator=g, device=device, dtype=torch.float64)
    q = q / q.norm(dim=-1, keepdim=True)
    if dist == "qwen":
        q = q / d ** 0.5
    k = k / k.norm(dim=-1, keepdim=True)
    v = torch.randn(n_slots, n_tok, n_v_heads, d, generator=g, device=device, dtype=torch.float64)
    ua = torch.rand(n_slots, n_tok, n_v_heads, generator=g, device=device, dtype=torch.float64)
    a = 1.0 - (1.0 - alpha_lo) * ua                       # in (alpha_lo, 1]
    b = torch.sigmoid(torch.randn(n_slots, n_tok, n_v_heads, generator=g, device=device,
                                  dtype=torch.float64))
    out = {"q": q.float().to(tdt), "k": k.float().to(tdt), "v": v.float().to(tdt),
           "alpha": a.float(), "beta": b.float()}
    if squeeze:
        out = {n: x[:, 0].contiguous() for n, x in out.items()}
    return {n: x.contiguous() for n, x in out.items()}


def state0(seed, n_slots, n_v_heads, d=D, device="cuda"):
    """Synthetic long-context start states [n, Hv, d_v, d_k] fp32 ~ N(0, 1/(4 d_k))."""
    g = _gen(seed, device)
    return (torch.randn(n_slots, n_v_heads, d, d, generator=g, device=device) * (1.0 / (4 * d)) ** 0.5).contiguous()


def fill_state0(out, seed):
    """state0 written in place into `out` ([n, Hv, d, d] fp32 on the device):
    the same distribution, no temporaries (large pools)."""
    g = _gen(seed, out.device)
    torch.randn(out.shape, generator=g, device=out.device, dtype=out.dtype, out=out)
    out.mul_((1.0 / (4 * out.shape[-1])) ** 0.5)
    return out


def n_accepted(seed, n_slots, n_draft, p_accept=0.7, device="cuda"):
    """Accepted-prefix length per slot: first failed Bernoulli(p) trial among n_draft."""
    g = _gen(seed, device)
    ok = torch.rand(n_slots, n_draft, generator=g, device=device) <= p_accept
    fail = ~ok
    first = torch.where(fail.any(dim=1), fail.int().argmax(dim=1), torch.full((n_slots,), n_draft, device=device))
    return first.to(torch.int32).contiguous()


def host_tokens(tok, slots):
    """The stored values of the given slots as float32 numpy arrays, in the
    layout tests/harness.Oracle expects ([n, T, H, d] / [n, T, Hv])."""
    idx = torch.as_tensor(slots, device=tok["q"].device, dtype=torch.long)
    out = {}
    for name, x in tok.items():
        y = x.index_select(0, idx)
        if y.dim() == (3 if name in ("alpha", "beta") else 4) - 1:   # squeezed token axis
            y = y.unsqueeze(1)
        out[name] = y.float().cpu().numpy()
    return out
