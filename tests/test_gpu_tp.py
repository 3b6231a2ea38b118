"""Tensor parallelism over heads on one GPU.

A rank of a G-way TP group owns QK heads [g Hk/G, (g+1) Hk/G) and the V heads
that read them (dp.head_range), with its own handle of Hk/G, Hv/G heads.
Because no kernel reads another head's data, the per-rank handles run on the
head slices of the same inputs must reproduce the unsharded handle's outputs
and states BIT FOR BIT; gathering the head-major outputs [Hv][B][d] of the
ranks then gives the full layer output.  The NCCL all-gather itself
(la_tp_allgather) runs here as a world-1 communicator (one GPU per box)."""
import numpy as np
import pytest
import torch

import synth.device as sd
from harness import make_buf
from paper_2605_19049_b200 import dp
from paper_2605_19049_b200 import labuf as L

pytestmark = pytest.mark.gpu

HK, HV, B, C = 16, 32, 8, 8


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tp_head_shards_bit_identical(cuda_device, world):
    full = make_buf(B, HK, HV, C=C)
    full.reset(zero_state=False)
    S0 = sd.state0(777, B, HV, device=cuda_device)
    full.state.copy_(S0)
    ranks = []
    for g in range(world):
        q0, nq, v0, nv = dp.head_range(HK, HV, g, world)
        b = make_buf(B, nq, nv, C=C)
        b.reset(zero_state=False)
        b.state.copy_(S0[:, v0:v0 + nv])
        ranks.append((b, q0, nq, v0, nv))
    for t in range(C + 3):
        x = sd.tokens(900 + t, B, 1, HK, HV, device=cuda_device, squeeze=True)
        o_full = torch.empty(B, HV, 128, dtype=torch.float32, device=cuda_device)
        full.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o_full)
        full.flush(0, B, L.LA_FLUSH_FULL)
        # head-major gather target [Hv][B][d]: rank g's slice is contiguous
        gathered = torch.empty(HV, B, 128, dtype=torch.float32, device=cuda_device)
        for b, q0, nq, v0, nv in ranks:
            o = torch.empty(B, nv, 128, dtype=torch.float32, device=cuda_device)
            b.decode_step(0, x["q"][:, q0:q0 + nq].contiguous(), x["k"][:, q0:q0 + nq].contiguous(),
                          x["v"][:, v0:v0 + nv].contiguous(), x["alpha"][:, v0:v0 + nv].contiguous(),
                          x["beta"][:, v0:v0 + nv].contiguous(), o)
            b.flush(0, B, L.LA_FLUSH_FULL)
            gathered[v0:v0 + nv] = o.transpose(0, 1)
        assert torch.equal(gathered.transpose(0, 1), o_full), f"step {t}"
    full.flush(0, B, L.LA_FLUSH_FORCE)
    for b, q0, nq, v0, nv in ranks:
        b.flush(0, B, L.LA_FLUSH_FORCE)
        assert torch.equal(b.state, full.state[:, v0:v0 + nv])


def test_tp_allgather_world1(cuda_device):
    """la_tp_init / la_tp_allgather / la_tp_destroy through the C ABI."""
    uid = L.tp_unique_id()
    assert len(uid) == 128
    comm = L.TPComm(uid, 0, 1, cuda_device.index if cuda_device.index is not None else 0)
    try:
        send = torch.arange(HV * B * 128, dtype=torch.float32, device=cuda_device).reshape(HV, B, 128)
        recv = torch.zeros_like(send)
        comm.allgather(send, recv)
        torch.cuda.synchronize()
        assert torch.equal(recv, send)
        with pytest.raises(ValueError):
            comm.allgather(send, torch.zeros(7, dtype=torch.float32, device=cuda_device))
    finally:
        comm.destroy()
