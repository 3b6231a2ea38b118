"""Config 5 driver: a stack of GDN layers serving a mixed batch (SURVEY §8d
config 5, BASELINE.json configs[4]).

Per layer two handles of the C ABI: a CHUNKWISE handle for the long-context
requests (buffered decode + flush, u fp32) and a DIRECT handle for the short
ones (KV-only decode, u fp16, no state is ever created for them, P:35,
P:200-213).  Every slot of a handle sits in one contiguous range, so one call
per handle per layer serves the whole batch.  Host logic only: argument
marshalling and call ordering; every arithmetic step runs in the library's
kernels.

Ragged starting points use contiguous groups so each call still covers one
range: long slots are staggered over occupancies 0..C-1 (group g holds occ =
g, so flushes spread over the C steps of a cycle), short slots start at
group-wise context lengths L0 (a KV-only prefill per group).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import labuf as L


@dataclass
class StackSpec:
    n_layers: int = 36
    n_long: int = 1536
    n_short: int = 512
    n_qk_heads: int = 16
    n_v_heads: int = 32
    chunk: int = 16
    short_cap: int = 128
    short_l0: tuple = (16, 40, 64, 96)     # context length per short group (U{16..96} in 4 groups)
    in_dtype: str = "bf16"


def long_groups(spec: StackSpec):
    """[(first, n, occupancy)] of the staggered long slots (n_long split into C groups)."""
    C, n = spec.chunk, spec.n_long
    base, extra = divmod(n, C)
    out, first = [], 0
    for g in range(C):
        m = base + (1 if g < extra else 0)
        out.append((first, m, g))
        first += m
    return out


def short_groups(spec: StackSpec):
    """[(first, n, L0)] of the short slots."""
    G, n = len(spec.short_l0), spec.n_short
    base, extra = divmod(n, G)
    out, first = [], 0
    for g, l0 in enumerate(spec.short_l0):
        m = base + (1 if g < extra else 0)
        out.append((first, m, l0))
        first += m
    return out


def _configs(spec: StackSpec):
    """The per-layer handle configurations: long (chunkwise) [, short (direct)]."""
    out = [L.make_config(spec.n_long, spec.n_qk_heads, spec.n_v_heads, chunk=spec.chunk,
                         in_dtype=spec.in_dtype, u_dtype="f32", validate=False)]
    if spec.n_short:
        out.append(L.make_config(spec.n_short, spec.n_qk_heads, spec.n_v_heads, chunk=spec.chunk,
                                 short_cap=spec.short_cap, in_dtype=spec.in_dtype,
                                 u_dtype="f16" if spec.in_dtype == "bf16" else "f32", validate=False))
    return out


@dataclass
class Layer:
    long: L.LaBuf
    short: L.LaBuf | None


@dataclass
class GdnStack:
    spec: StackSpec
    device: torch.device
    layers: list = field(default_factory=list)

    @classmethod
    def create(cls, spec: StackSpec, device):
        st = cls(spec, torch.device(device))
        cfgs = _configs(spec)
        for _ in range(spec.n_layers):
            sb = L.LaBuf(cfgs[1], device=st.device) if len(cfgs) > 1 else None
            st.layers.append(Layer(L.LaBuf(cfgs[0], device=st.device), sb))
        return st

    def reset(self, states):
        """states[l]: fp32 [n_long, Hv, d, d] start states of layer l's long slots."""
        for lay, S0 in zip(self.layers, states):
            lay.long.reset(zero_state=False)
            lay.long.state.copy_(S0)
            if lay.short is not None:
                lay.short.reset(mode=L.LA_MODE_DIRECT, zero_state=False)

    def warmup(self, long_tok, short_tok):
        """Bring the slots to their ragged starting points.

        long_tok(l, t)  -> decode inputs of token t for ALL long slots of layer l
                           (dict q,k,v,alpha,beta [n_long, ...], token axis squeezed)
        short_tok(l, g) -> prefill inputs of short group g ([n_g, L0_g, ...])
        Outputs of the warm-up are written to scratch and returned per call
        for tests: {("long", l, t): o, ("short", l, g): o}."""
        outs = {}
        spec = self.spec
        Hv, d = spec.n_v_heads, 128
        for l, lay in enumerate(self.layers):
            groups = long_groups(spec)
            for t in range(spec.chunk - 1):
                # groups with occupancy > t decode token t (a suffix of the range)
                first = next((f for f, m, occ in groups if occ > t), None)
                if first is None:
                    break
                x = long_tok(l, t)
                n = spec.n_long - first
                o = torch.empty(n, Hv, d, dtype=torch.float32, device=self.device)
                lay.long.decode_step(first, *(x[k][first:] for k in ("q", "k", "v", "alpha", "beta")), o)
                outs[("long", l, t)] = (first, o)
            if lay.short is not None:
                for g, (first, m, l0) in enumerate(short_groups(spec)):
                    x = short_tok(l, g)
                    o = torch.empty(m, l0, Hv, d, dtype=torch.float32, device=self.device)
                    lay.short.direct_short(first, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
                    outs[("short", l, g)] = (first, o)
        return outs

    def step(self, long_in, short_in, long_out, short_out):
        """One decode step of the whole stack: per layer, one buffered decode
        call over all long slots (+ the FULL flush of the slots it filled) and
        one KV-only call over all short slots.  *_in[l] / *_out[l] are the
        layer's device tensors (short ones with a token axis of 1)."""
        for l, lay in enumerate(self.layers):
            x = long_in[l]
            lay.long.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], long_out[l])
            lay.long.flush(0, self.spec.n_long, L.LA_FLUSH_FULL)
            if lay.short is not None:
                y = short_in[l]
                lay.short.direct_short(0, y["q"], y["k"], y["v"], y["alpha"], y["beta"], short_out[l])

    @staticmethod
    def footprint_of(spec: StackSpec) -> int:
        """Device bytes the stack would allocate (la_buf_query), before creating it."""
        tot = 0
        for cfg in _configs(spec):
            sz = L.query(cfg)
            tot += sz.state_bytes + sz.buffer_bytes + sz.meta_bytes
        return tot * spec.n_layers

    def footprint_bytes(self):
        tot = 0
        for lay in self.layers:
            for b in (lay.long, lay.short):
                if b is not None:
                    tot += b.sizes.state_bytes + b.sizes.buffer_bytes + b.sizes.meta_bytes
        return tot


@dataclass
class MixedStack:
    """Config 5 on ONE handle per layer: a paged record pool
    (blocks of 16 tokens) and a state pool sized for the
    long-context requests plus headroom for compressions, serving the mixed
    batch with one la_decode_mixed call per layer per step -- long slots
    decode chunkwise (eager flush), short slots KV-only, and a short slot
    whose context reaches short_cap is compressed into a pool state.
    Short requests hold no state at all, so the stack fits one B200 (the two-
    handle layout above reserves a state per short slot too)."""
    spec: StackSpec
    device: torch.device
    layers: list = field(default_factory=list)
    state_headroom: int = 64
    block_tokens: int = 16

    def config(self):
        s = self.spec
        n = s.n_long + s.n_short
        bt = self.block_tokens
        blocks = s.n_long * -(-s.chunk // bt) + s.n_short * -(-s.short_cap // bt)
        return L.make_config(n, s.n_qk_heads, s.n_v_heads, chunk=s.chunk, short_cap=s.short_cap,
                             in_dtype=s.in_dtype, u_dtype="f16" if s.in_dtype == "bf16" else "f32",
                             validate=False, block_tokens=bt, n_blocks=blocks,
                             state_slots=s.n_long + self.state_headroom)

    @classmethod
    def create(cls, spec: StackSpec, device, state_headroom=64):
        st = cls(spec, torch.device(device), state_headroom=state_headroom)
        cfg = st.config()
        st.layers = [L.LaBuf(cfg, device=st.device) for _ in range(spec.n_layers)]
        return st

    @staticmethod
    def footprint_of(spec: StackSpec, state_headroom=64) -> int:
        sz = L.query(MixedStack(spec, torch.device("cpu"), state_headroom=state_headroom).config())
        return (sz.state_bytes + sz.buffer_bytes + sz.meta_bytes) * spec.n_layers

    def footprint_bytes(self):
        return sum(b.sizes.state_bytes + b.sizes.buffer_bytes + b.sizes.meta_bytes for b in self.layers)

    def reset(self, fill):
        """Long slots 0..n_long-1 CHUNKWISE (a fresh pool hands them states
        0..n_long-1 in order), short slots DIRECT; fill(l, view) writes layer
        l's start states into the fp32 [n_long, Hv, d, d] view in place."""
        s = self.spec
        for l, b in enumerate(self.layers):
            b.reset(0, s.n_long, mode=L.LA_MODE_CHUNKWISE, zero_state=False)
            if s.n_short:
                b.reset(s.n_long, s.n_short, mode=L.LA_MODE_DIRECT, zero_state=False)
            assert b.pool_info(s.n_long - 1)["slot_state"] == s.n_long - 1
            fill(l, b.state[:s.n_long])

    def warmup(self, long_tok, short_tok):
        """Ragged starting points as in GdnStack.warmup (long occupancies
        staggered over 0..C-1, short contexts L0 per group); returns the
        warm-up outputs for tests."""
        outs = {}
        s = self.spec
        Hv, d = s.n_v_heads, 128
        groups = long_groups(s)
        for l, b in enumerate(self.layers):
            for t in range(s.chunk - 1):
                first = next((f for f, m, occ in groups if occ > t), None)
                if first is None:
                    break
                x = long_tok(l, t)
                idx = list(range(first, s.n_long))
                o = torch.empty(len(idx), Hv, d, dtype=torch.float32, device=self.device)
                b.decode_mixed(idx, *(x[k][first:].contiguous() for k in ("q", "k", "v", "alpha", "beta")), o)
                outs[("long", l, t)] = (first, o)
            for g, (first, m, l0) in enumerate(short_groups(s)):
                x = short_tok(l, g)
                o = torch.empty(m, l0, Hv, d, dtype=torch.float32, device=self.device)
                b.direct_short(s.n_long + first, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
                outs[("short", l, g)] = (first, o)
        return outs

    def step(self, inputs, outputs, slots=None):
        """One decode step of the stack: per layer ONE la_decode_mixed over the
        batch (`slots`, default all, in slot order); inputs[l] / outputs[l]
        are the layer's [n, ...] tensors by batch row."""
        s = self.spec
        if slots is None:
            if getattr(self, "_all_slots", None) is None:
                import numpy as np
                self._all_slots = np.arange(s.n_long + s.n_short, dtype=np.int32)
            slots = self._all_slots
        for b, x, o in zip(self.layers, inputs, outputs):
            b.decode_mixed(slots, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o)
