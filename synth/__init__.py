"""Seeded synthetic inputs shared by the oracle side and the GPU side.

This module holds NONE of the method's arithmetic: it only draws random
numbers and rounds them to the stored dtypes.  Both the oracle (tests,
cpu_baseline) and the CUDA path (tests, bench, smoke) consume exactly the
stored values it returns, so "the same inputs" is true bit for bit.

Recipe:
  * counter-based generator: splitmix64 finaliser over a 64-bit counter built
    from (tag, layer, slot, token position, head, element) and the seed, so any
    (layer, slot, head) subset can be regenerated independently;
  * normals by Box-Muller in fp64;
  * q, k ~ N(0, 1) per head, L2-normalised (Qwen3-Next normalises q and k
    before the GDN step; reading Z9), q additionally scaled by d^-1/2 in the
    'qwen' distribution ('stress' leaves q unit-norm);
  * v ~ N(0, 1);
  * alpha ~ U(alpha_lo, alpha_hi] fp32 (default (0.9, 1]); beta = sigmoid(N(0,1)) fp32;
  * long-context start state S0 ~ N(0, 1/(4 d_k)) fp32 per (slot, V head);
  * rounding: fp64 -> fp32 (RNE) -> bf16 (RNE) when the input dtype is bf16
    (reading Z12);
  * draft acceptance: n_acc = index of the first failed Bernoulli(p) trial
    among N, keyed by (seed, layer, round, slot) (reading Z23).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)

TAG_Q, TAG_K, TAG_V, TAG_ALPHA, TAG_BETA, TAG_S0, TAG_ACC = 1, 2, 3, 4, 5, 6, 7


def _mix(z):
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _seed_base(seed: int) -> np.uint64:
    return _mix(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64) * _GOLD)[0]


def _counters(tag, layer, slot, pos, head, elem):
    """Pack indices into a 64-bit counter: tag 4b | layer 8b | slot 16b |
    pos 16b | head 8b | elem 12b  (= 64 bits)."""
    u = np.uint64
    c = (u(tag) << u(60)) | (u(layer) << u(52))
    c = c | (np.asarray(slot, dtype=np.uint64) << u(36))
    c = c | (np.asarray(pos, dtype=np.uint64) << u(20))
    c = c | (np.asarray(head, dtype=np.uint64) << u(12))
    c = c | np.asarray(elem, dtype=np.uint64)
    return c


def _uniform01(seed, counters):
    """Uniform in (0, 1] from a splitmix64 draw (53 mantissa bits)."""
    with np.errstate(over="ignore"):
        x = _mix(counters * _GOLD + _seed_base(seed))
    return ((x >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)


def _normal(seed, tag, layer, slot, pos, head, elem):
    """Box-Muller normal; element e uses counters 2e and 2e+1."""
    e2 = np.asarray(elem, dtype=np.uint64) * np.uint64(2)
    u1 = _uniform01(seed, _counters(tag, layer, slot, pos, head, e2))
    u2 = _uniform01(seed, _counters(tag, layer, slot, pos, head, e2 + np.uint64(1)))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def round_f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def round_bf16(x32):
    """fp32 -> bf16 with round-to-nearest-even, returned as fp32 values."""
    b = np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32)
    lsb = (b >> np.uint32(16)) & np.uint32(1)
    with np.errstate(over="ignore"):
        r = (b + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def round_in(x, in_dtype):
    x32 = round_f32(x)
    return round_bf16(x32) if in_dtype == "bf16" else x32


@dataclass(frozen=True)
class Recipe:
    seed: int = 1002
    dist: str = "qwen"          # 'qwen' | 'stress'
    in_dtype: str = "bf16"      # 'bf16' | 'f32'
    alpha_lo: float = 0.9
    alpha_hi: float = 1.0
    p_accept: float = 0.7


def _grid(slots, positions, heads, d):
    s = np.asarray(slots, dtype=np.uint64)[:, None, None, None]
    p = np.asarray(positions, dtype=np.uint64)[None, :, None, None]
    h = np.arange(heads, dtype=np.uint64)[None, None, :, None]
    e = np.arange(d, dtype=np.uint64)[None, None, None, :]
    return s, p, h, e


def tokens(rc: Recipe, slots, positions, n_qk_heads, n_v_heads, d, layer=0):
    """Per-token GDN inputs for the given slot ids and token positions.

    Returns float32 arrays (values exactly representable in rc.in_dtype):
      q, k  [S, T, Hk, d]; v [S, T, Hv, d]; alpha, beta [S, T, Hv] (fp32)
    """
    slots = np.atleast_1d(np.asarray(slots))
    positions = np.atleast_1d(np.asarray(positions))
    s, p, h, e = _grid(slots, positions, n_qk_heads, d)
    out = {}
    for name, tag in (("q", TAG_Q), ("k", TAG_K)):
        x = _normal(rc.seed, tag, layer, s, p, h, e)
        x = x / np.sqrt(np.sum(x * x, axis=-1, keepdims=True))
        if name == "q" and rc.dist == "qwen":
            x = x / np.sqrt(float(d))
        out[name] = round_in(x, rc.in_dtype)
    s, p, h, e = _grid(slots, positions, n_v_heads, d)
    out["v"] = round_in(_normal(rc.seed, TAG_V, layer, s, p, h, e), rc.in_dtype)
    s3, p3, h3 = s[..., 0], p[..., 0], h[..., 0]
    ua = _uniform01(rc.seed, _counters(TAG_ALPHA, layer, s3, p3, h3, 0))
    a = rc.alpha_hi - (rc.alpha_hi - rc.alpha_lo) * (1.0 - ua)   # in (lo, hi]
    out["alpha"] = round_f32(a)
    nb = _normal(rc.seed, TAG_BETA, layer, s3, p3, h3, 0)
    out["beta"] = round_f32(1.0 / (1.0 + np.exp(-nb)))
    return out


def state0(rc: Recipe, slots, n_v_heads, d_v, d_k, layer=0):
    """Synthetic long-context start state S0 ~ N(0, 1/(4 d_k)), fp32,
    shape [S, Hv, d_v, d_k] (north-star orientation, d_k contiguous)."""
    slots = np.atleast_1d(np.asarray(slots))
    s = np.asarray(slots, dtype=np.uint64)[:, None, None, None]
    h = np.arange(n_v_heads, dtype=np.uint64)[None, :, None, None]
    j = np.arange(d_v, dtype=np.uint64)[None, None, :, None]
    c = np.arange(d_k, dtype=np.uint64)[None, None, None, :]
    # 'pos' field carries the row index j, 'elem' the column.
    z = _normal(rc.seed, TAG_S0, layer, s, j, h, c)
    return round_f32(z * np.sqrt(1.0 / (4.0 * d_k)))


def n_accepted(rc: Recipe, slots, n_draft, round_idx, layer=0):
    """Accepted-prefix length per slot: index of the first failed
    Bernoulli(p_accept) trial among n_draft trials (so in [0, n_draft])."""
    slots = np.atleast_1d(np.asarray(slots, dtype=np.uint64))
    trials = np.arange(n_draft, dtype=np.uint64)
    u = _uniform01(rc.seed, _counters(TAG_ACC, layer, slots[:, None],
                                      np.uint64(round_idx), 0, trials[None, :]))
    ok = u <= rc.p_accept
    fail = ~ok
    first_fail = np.where(fail.any(axis=1), fail.argmax(axis=1), n_draft)
    return first_fail.astype(np.int32)


def expand_qk_to_v_heads(x, n_v_heads):
    """[.., Hk, d] -> [.., Hv, d]: V head h reads QK head floor(h * Hk / Hv)
    (GQA grouping, Qwen3-Next repeat_interleave)."""
    hk = x.shape[-2]
    g = n_v_heads // hk
    return np.repeat(x, g, axis=-2)
