"""Multi-process (world size 2, gloo, CPU) checks of the N > 1 host logic:
data-parallel slot shards partition the batch, the max-over-ranks timing
reduction, the tensor-parallel head partition keeps GQA groups together, and
running the (oracle) recurrence on each rank's shard and gathering equals the
unsharded run — the "no exchange step" claim of DESIGN.md §8."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19049_b200 import dp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        B, Hk, Hv, d, T = 6, 2, 4, 16, 5
        first, n = dp.shard_range(B, rank, world)
        rc = synth.Recipe(seed=77, in_dtype="f32")
        slots = np.arange(first, first + n)
        S0 = synth.state0(rc, slots, Hv, d, d).astype(np.float64)
        tok = synth.tokens(rc, slots, np.arange(T), Hk, Hv, d)
        qv = synth.expand_qk_to_v_heads(tok["q"], Hv)
        kv = synth.expand_qk_to_v_heads(tok["k"], Hv)
        seq = lambda x: np.ascontiguousarray(np.swapaxes(x, 1, 2).reshape((n * Hv, T) + x.shape[3:]))
        o, S = oracle.gdn_run(S0.reshape(n * Hv, d, d), seq(qv), seq(kv), seq(tok["v"]), seq(tok["alpha"]),
                              seq(tok["beta"]), n_threads=1)
        np.save(os.path.join(out_dir, f"o{rank}.npy"), o)
        np.save(os.path.join(out_dir, f"S{rank}.npy"), S)
        # timing reduction: max over ranks
        m = dp.max_over_ranks(1.5 + rank)
        tot = dp.sum_over_ranks(n)
        np.save(os.path.join(out_dir, f"red{rank}.npy"), np.array([m, tot]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_dp_shards_equal_unsharded_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import oracle
    import synth
    B, Hk, Hv, d, T = 6, 2, 4, 16, 5
    rc = synth.Recipe(seed=77, in_dtype="f32")
    slots = np.arange(B)
    S0 = synth.state0(rc, slots, Hv, d, d).astype(np.float64)
    tok = synth.tokens(rc, slots, np.arange(T), Hk, Hv, d)
    qv = synth.expand_qk_to_v_heads(tok["q"], Hv)
    kv = synth.expand_qk_to_v_heads(tok["k"], Hv)
    seq = lambda x: np.ascontiguousarray(np.swapaxes(x, 1, 2).reshape((B * Hv, T) + x.shape[3:]))
    o_ref, S_ref = oracle.gdn_run(S0.reshape(B * Hv, d, d), seq(qv), seq(kv), seq(tok["v"]),
                                  seq(tok["alpha"]), seq(tok["beta"]), n_threads=1)
    o = np.concatenate([np.load(tmp_path / f"o{r}.npy") for r in range(world)])
    S = np.concatenate([np.load(tmp_path / f"S{r}.npy") for r in range(world)])
    assert np.array_equal(o, o_ref) and np.array_equal(S, S_ref)   # bit-identical: no exchange step
    for r in range(world):
        m, tot = np.load(tmp_path / f"red{r}.npy")
        assert m == 2.5 and tot == B


@pytest.mark.parametrize("B,world", [(64, 1), (64, 2), (64, 8), (2048, 8), (7, 3), (1, 2)])
def test_shard_range_partitions(B, world):
    ranges = [dp.shard_range(B, r, world) for r in range(world)]
    covered = [s for f, n in ranges for s in range(f, f + n)]
    assert covered == list(range(B))
    sizes = [n for _, n in ranges]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_head_range_keeps_gqa_groups(world):
    Hk, Hv = 16, 32
    qs, vs = [], []
    for r in range(world):
        q0, nq, v0, nv = dp.head_range(Hk, Hv, r, world)
        qs += list(range(q0, q0 + nq))
        vs += list(range(v0, v0 + nv))
        for h in range(v0, v0 + nv):
            assert q0 <= h // (Hv // Hk) < q0 + nq      # V head h reads QK head h // g on the same rank
    assert qs == list(range(Hk)) and vs == list(range(Hv))


def test_mixed_assignment_same_mix():
    n_long, n_short, world = 1536, 512, 8
    shards = [dp.mixed_assignment(n_long, n_short, r, world) for r in range(world)]
    assert sorted(i for s in shards for i in s.long_ids + s.short_ids) == list(range(n_long + n_short))
    assert {len(s.long_ids) for s in shards} == {n_long // world}
    assert {len(s.short_ids) for s in shards} == {n_short // world}
