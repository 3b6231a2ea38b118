"""bench.py's multi-rank logic on CPU (world size 2, gloo): the self-relaunch
under torchrun when `--gpus N` is given without a launcher, the world-size
check, per-rank seeds, the max-over-ranks timing reduction and the whole-job
value (DP sums the ranks' batches, TP serves one batch), and an end-to-end
`--gpus 2` run of the reference arm through the relaunch path (rank 0 prints
exactly one JSON line, rank 1 exits without work)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_spawn_command_only_without_launcher():
    args = bench.parse_args(["--gpus", "4", "--steps", "3"])
    cmd = bench.spawn_command(args, ["--gpus", "4", "--steps", "3"], {})
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"][-3:] and cmd[-5].endswith("bench.py")
    assert bench.spawn_command(args, [], {"WORLD_SIZE": "4"}) is None          # already under torchrun
    assert bench.spawn_command(bench.parse_args([]), [], {}) is None           # one GPU: no relaunch


def test_check_world_rejects_mismatch():
    with pytest.raises(SystemExit):
        bench.check_world(bench.parse_args(["--gpus", "8"]), 1)
    bench.check_world(bench.parse_args(["--gpus", "2"]), 2)


def test_whole_job_value():
    # DP: every rank serves its own batch; TP: the ranks share one batch
    assert bench.whole_job_value(4, 64, 30.0, "dp") == pytest.approx(4 * 64 / 30e-6)
    assert bench.whole_job_value(4, 64, 30.0, "tp") == pytest.approx(64 / 30e-6)


def _worker(rank, world, port, out):
    env = {"WORLD_SIZE": str(world), "RANK": str(rank), "LOCAL_RANK": str(rank)}
    os.environ.update(env, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_19049_b200 import dp
        w, r, lr = bench.rank_env()
        args = bench.parse_args(["--gpus", str(world)])
        bench.check_world(args, w)
        seed = bench.rank_seed(args, r)
        seeds = [None] * world
        dist.all_gather_object(seeds, seed)
        step_ms = dp.max_over_ranks(3.0 + r)          # the bench's timing reduction
        out[r] = (w, r, lr, tuple(seeds), step_ms, dp.shard_range(2048, r, w))
    finally:
        dist.destroy_process_group()


def test_rank_logic_world2_gloo():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        w, rr, lr, seeds, step_ms, (first, n) = res[r]
        assert (w, rr, lr) == (world, r, r)
        assert len(set(seeds)) == world                 # each rank draws its own shard
        assert step_ms == 3.0 + world - 1               # max over ranks, on every rank
        assert (first, n) == (r * 1024, 1024)


def test_reference_arm_relaunches_under_torchrun():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--batch", "2"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
