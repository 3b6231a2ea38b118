#!/usr/bin/env python
"""bench.py — KV-buffered Gated DeltaNet decode on B200 (arxiv 2605.19049).

Headline workload (BASELINE.json configs[1], "config 2"): one Qwen3-Next GDN
layer (16 QK heads, 32 V heads, d = 128, fp32 state, bf16 q/k/v, fp32 delta
values) decoding a batch of 64 requests with synthetic 32K-context states,
buffer C = 16.  A *step* is one full buffer cycle of the whole hot path for
that batch: C buffered decode steps (kernel 1) followed by the tensor-core
flush (kernel 2), run over NL = 8 independent layer instances so the state
working set (8 x 128 MiB) is 8x the 126 MB L2 and every state read comes
from HBM (as in a 36-layer model).  The recurrent baseline (kernel 5a) runs
the same tokens through the same layers in the same process.

Metric (BASELINE.json): GDN decode us/token & tokens/s; value = tokens/s of
one GDN layer summed over all GPUs = n_gpus * B / (us per decode step per
layer), where us per step is the cycle average including the flush (Fig. 4
caption).  Extra measured rows: parallel verify + accepted-prefix
commit (config 3 shape) and direct short-context decode (config 4 shape).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GDN decode us/token & tokens/s per GPU; % of 8 TB/s HBM vs recurrent baseline"
UNIT = "tokens/s (one GDN layer, all GPUs)"
D = 128


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="labuf", choices=["labuf", "reference"])
    p.add_argument("--batch", type=int, default=64, help="requests per GPU")
    p.add_argument("--chunk", type=int, default=16)
    p.add_argument("--layers", type=int, default=8, help="layer instances rotated per step")
    p.add_argument("--in-dtype", default="bf16", choices=["bf16", "f32"])
    p.add_argument("--u-dtype", default="f32", choices=["f32", "f16"])
    p.add_argument("--no-rows", action="store_true", help="skip the verify / direct rows")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (sweeps)")
    p.add_argument("--drafts", type=int, default=4, help="config-3 row: drafts per round")
    p.add_argument("--direct-l0", type=int, default=64, help="config-4 row: context before the 32 timed steps")
    p.add_argument("--no-overlap", action="store_true", help="launch without PDL (la_set_overlap 0)")
    p.add_argument("--auto-flush", action="store_true",
                   help="headline WITH the fused flush (la_set_auto_flush; measured slower, see DESIGN.md)")
    p.add_argument("--parallel", default="dp", choices=["dp", "tp"],
                   help="dp: requests partitioned over ranks (headline, no collective); tp: heads partitioned, "
                        "one la_tp_allgather of the head outputs per layer per step (P:232)")
    p.add_argument("--no-config1", action="store_true", help="skip the config-1 latency row")
    p.add_argument("--no-config5", action="store_true", help="skip the config-5 36-layer stack row")
    p.add_argument("--seed", type=int, default=1002)
    return p.parse_args(argv)


# ---------------------------------------------------------------- ranks
def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_command(args, argv, env):
    """`--gpus N` (N > 1) outside a torchrun environment: the command that
    relaunches this script with one process per GPU (the driver's own
    launch form), else None."""
    if args.gpus <= 1 or "WORLD_SIZE" in env:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]


def rank_env(env=None):
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 alone)."""
    env = os.environ if env is None else env
    return int(env.get("WORLD_SIZE", "1")), int(env.get("RANK", "0")), int(env.get("LOCAL_RANK", "0"))


def check_world(args, world):
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")


def rank_seed(args, rank):
    """Per-rank input seed: each rank draws its own shard of the global batch."""
    return args.seed * 1000 + 100 * rank


def whole_job_value(world, batch_per_rank, us_per_token, parallel="dp"):
    """tokens/s of one GDN layer over all ranks: DP serves world x batch
    requests per step, TP serves one batch (heads split over the ranks)."""
    served = batch_per_rank * (world if parallel == "dp" else 1)
    return served / (us_per_token * 1e-6)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the run."""

    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append((time.time(), parts))

    def mark(self):
        return time.time()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = [r for t, r in self.rows if (t0 is None or t >= t0) and (t1 is None or t <= t1)]
        if not rows:
            rows = [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in rows if (num(r[2]) or 0) > 0] or rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(rows[0][1]), "reasons": reasons, "samples": len(loaded)}


# ---------------------------------------------------------------- helpers
def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    the kernel, from the committed ncu --set full summary (tools/ncu_traffic.py
    writes profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as f:
            return json.load(f).get(kernel_key, {}).get("dram_bytes")
    except Exception:
        return None


def make_inputs(torch, B, Hk, Hv, n, in_dtype, seed, device):
    """n decode steps of seeded synthetic inputs (synth.device, DESIGN.md
    'Input recipe'), drawn on the device; plus an fp32 output buffer each."""
    import synth.device as sd
    out = []
    for i in range(n):
        x = sd.tokens(seed + i, B, 1, Hk, Hv, D, in_dtype=in_dtype, device=device, squeeze=True)
        x["o"] = torch.empty(B, Hv, D, dtype=torch.float32, device=device)
        out.append(x)
    return out


def fill_states(torch, bufs, seed):
    import synth.device as sd
    for i, b in enumerate(bufs):
        b.state.copy_(sd.state0(seed + i, b.cfg.max_slots, b.cfg.n_v_heads, D, device=b.state.device))


def timed_graphs(torch, stream, graphs, K, W):
    """Replay the phase graphs W times, then K times bracketed by events
    between phases.  Returns (total_ms, [sum_ms per phase])."""
    with torch.cuda.stream(stream):
        for _ in range(W):
            for g in graphs:
                g.replay()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(graphs) + 1)] for _ in range(K)]
    with torch.cuda.stream(stream):
        for k in range(K):
            evs[k][0].record(stream)
            for i, g in enumerate(graphs):
                g.replay()
                evs[k][i + 1].record(stream)
    torch.cuda.synchronize()
    total = evs[0][0].elapsed_time(evs[K - 1][-1])
    phases = [sum(evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(K)) for i in range(len(graphs))]
    return total, phases


def capture(torch, stream, fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


# ---------------------------------------------------------------- CPU oracle leg
def cpu_oracle_sample(target_s=15.0, B=64, Hk=16, Hv=32, seed=1002, max_tok=None):
    """Time the fp64 oracle (the recurrence, as it stands) on host cores on a
    bounded sample of the config-2 workload: B slots x Hv heads x T tokens from
    synthetic 32K-context states.  Returns a cpu_baseline dict: tokens/s on all
    cores, the same on ONE thread (a smaller sample), cores, CPU model."""
    import numpy as np
    import oracle
    import synth
    rc = synth.Recipe(seed=seed)
    cores = oracle.default_threads()

    def run(T, nslots=B, threads=cores):
        slots = np.arange(nslots)
        S0 = synth.state0(rc, slots, Hv, D, D).astype(np.float64).reshape(nslots * Hv, D, D)
        tok = synth.tokens(rc, slots, np.arange(T), Hk, Hv, D)
        qv = synth.expand_qk_to_v_heads(tok["q"], Hv)
        kv = synth.expand_qk_to_v_heads(tok["k"], Hv)
        seq = lambda x: np.ascontiguousarray(np.swapaxes(x, 1, 2).reshape((nslots * Hv, T) + x.shape[3:]))
        args = [seq(qv), seq(kv), seq(tok["v"]), seq(tok["alpha"]), seq(tok["beta"])]
        t0 = time.perf_counter()
        oracle.gdn_run(S0, *args, n_threads=threads)
        return time.perf_counter() - t0

    # calibrate: per-call overhead (state copy-in) + per-token cost, then one
    # run sized to about target_s seconds of CPU work
    t4, t16 = run(4), run(16)
    per_tok = max((t16 - t4) / 12, 1e-5)
    T = max(1, int((target_s - t4 + 4 * per_tok) / per_tok))
    if max_tok:
        T = min(T, max_tok)
    dt = run(T)
    # single thread: 16 slots x 32 tokens (same per-token work)
    t1 = run(32, nslots=16, threads=1)
    return {"value": B * T / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{B} slots x {Hv} V heads x {T} tokens (config 2 shape, fp64 recurrence, {dt:.1f} s)",
            "single_thread": {"value": 16 * 32 / t1, "unit": UNIT, "cores": 1,
                              "sample": f"16 slots x {Hv} V heads x 32 tokens ({t1:.2f} s)"}}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # per step: one decode token of a bounded set of slots, sized so K+W steps
    # finish in about a minute of CPU
    import numpy as np
    import oracle
    import synth
    B, Hk, Hv = args.batch, 16, 32
    rc = synth.Recipe(seed=args.seed)
    cores = oracle.default_threads()
    S = synth.state0(rc, np.arange(B), Hv, D, D).astype(np.float64).reshape(B * Hv, D, D)

    def step(nslots, pos):
        slots = np.arange(nslots)
        tok = synth.tokens(rc, slots, [pos], Hk, Hv, D)
        qv = synth.expand_qk_to_v_heads(tok["q"], Hv)
        kv = synth.expand_qk_to_v_heads(tok["k"], Hv)
        seq = lambda x: np.ascontiguousarray(np.swapaxes(x, 1, 2).reshape((nslots * Hv, 1) + x.shape[3:]))
        t0 = time.perf_counter()
        oracle.gdn_run(S[:nslots * Hv], seq(qv), seq(kv), seq(tok["v"]), seq(tok["alpha"]),
                       seq(tok["beta"]), n_threads=cores)
        return time.perf_counter() - t0

    t_full = step(B, 0)
    budget = 60.0 / max(1, args.steps + args.warmup)
    nslots = max(1, min(B, int(B * budget / max(t_full, 1e-4))))
    for w in range(args.warmup):
        step(nslots, 1 + w)
    tot = 0.0
    for k in range(args.steps):
        tot += step(nslots, 100 + k)
    value = nslots * args.steps / tot
    sample = f"per step: 1 decode token x {nslots} of {B} slots x {Hv} V heads (fp64 recurrence oracle)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2: Qwen3-Next GDN layer decode, batch 64 @32K ctx (CPU oracle sample)",
                       "batch_per_gpu": B, "chunk": args.chunk},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- main arm
def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    cmd = spawn_command(args, argv, os.environ)
    if cmd:   # one process per GPU, launched like the driver does
        sys.exit(subprocess.call(cmd))
    world, rank, local = rank_env()
    check_world(args, world)
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2605_19049_b200 import cost
    from paper_2605_19049_b200 import labuf as L

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else torch.cuda.current_device())
    torch.cuda.set_device(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_2605_19049_b200 import dp

    def max_over_ranks(x):
        return dp.max_over_ranks(x, device=dev)

    B, C, NL, Hk, Hv = args.batch, args.chunk, args.layers, 16, 32
    K, W = args.steps, max(3, args.warmup)
    seed0 = rank_seed(args, rank)              # per-rank inputs: this rank's shard of the global batch
    tp = args.parallel == "tp"
    comm = None
    if tp:
        # tensor parallel over heads: this rank owns QK heads [q0, q0 + Hk/G) and
        # their V heads for ALL requests; head outputs are all-gathered per layer
        _, Hk, _, Hv = dp.head_range(16, 32, rank, world)
        uid = [L.tp_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        comm = L.TPComm(uid[0], rank, world, dev.index)
        gathered = [torch.empty(world, B, Hv, D, dtype=torch.float32, device=dev) for _ in range(NL)]
    clocks = ClockSampler(dev.index if world == 1 else local)
    clocks.start()
    peak, peak_src = measured_peaks()
    in_bytes = 2 if args.in_dtype == "bf16" else 4
    u_bytes = 2 if args.u_dtype == "f16" else 4
    lb = cost.LayerBytes.make(Hk, Hv, D, in_bytes, u_bytes)

    cfg = L.make_config(B, Hk, Hv, chunk=C, in_dtype=args.in_dtype, u_dtype=args.u_dtype)
    bufs = [L.LaBuf(cfg, device=dev) for _ in range(NL)]
    for b in bufs:
        b.reset(zero_state=False)
    fill_states(torch, bufs, seed0)
    torch.cuda.synchronize()
    for b in bufs:
        b.set_overlap(not args.no_overlap)   # PDL for the buffered AND the recurrent kernels
    inputs = [make_inputs(torch, B, Hk, Hv, NL, args.in_dtype, seed0 + 10 * (t + 1), dev) for t in range(C)]
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()

    # ---- buffered: capture decode phase (C steps x NL layers) and flush phase
    def dec_phase():
        for t in range(C):
            for l, b in enumerate(bufs):
                x = inputs[t][l]
                b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
                if tp:   # the layer's head outputs, gathered before the next layer could run
                    comm.allgather(x["o"], gathered[l])

    def flush_phase():
        for b in bufs:
            b.flush(0, B, L.LA_FLUSH_FULL)

    def cycle_in_order():
        # the serving order: each layer's flush right after the decode that
        # filled its buffers (eager flush, reading Z15), before the next layer
        for t in range(C):
            for l, b in enumerate(bufs):
                x = inputs[t][l]
                b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
                if tp:
                    comm.allgather(x["o"], gathered[l])
                if t == C - 1:
                    b.flush(0, B, L.LA_FLUSH_FULL)

    # unfused cycle (C decode launches + the tcgen05 flush kernel): measured
    # first, reported beside the headline and for the flush kernel's row
    n0 = sum(b.kernel_launches() for b in bufs)
    g_dec = capture(torch, stream, dec_phase)
    n1 = sum(b.kernel_launches() for b in bufs)
    g_fl = capture(torch, stream, flush_phase)
    n2 = sum(b.kernel_launches() for b in bufs)
    dec_launches, fl_launches = n1 - n0, n2 - n1
    barrier()
    t_c0 = time.time()
    uf_total_ms, (dec_ms, fl_ms) = timed_graphs(torch, stream, [g_dec, g_fl], K, W)
    uf_total_ms = max_over_ranks(uf_total_ms)
    del g_dec, g_fl
    g_io = capture(torch, stream, cycle_in_order)
    barrier()
    io_total_ms, _ = timed_graphs(torch, stream, [g_io], K, W)
    io_total_ms = max_over_ranks(io_total_ms)
    del g_io
    auto = args.auto_flush
    # the fused flush (la_set_auto_flush): the step that fills
    # the buffers folds them inside the decode kernel; always measured (row
    # "fused_flush"), the headline only with --auto-flush
    for b in bufs:
        b.set_auto_flush(True)
    n0 = sum(b.kernel_launches() for b in bufs)
    g_dec = capture(torch, stream, dec_phase)
    f_launches = sum(b.kernel_launches() for b in bufs) - n0
    barrier()
    f_total_ms, (fdec_ms,) = timed_graphs(torch, stream, [g_dec], K, W)
    f_total_ms = max_over_ranks(f_total_ms)
    for b in bufs:
        b.set_auto_flush(False)
    del g_dec
    if auto:
        total_ms, launches_per_step = f_total_ms, f_launches
    else:
        # the same launches in the serving order (flush after the filling
        # decode of each layer) or phase by phase, whichever the step uses
        total_ms, launches_per_step = min(uf_total_ms, io_total_ms), dec_launches + fl_launches
    in_order = (not auto) and io_total_ms <= uf_total_ms
    barrier()
    t_c1 = time.time()
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / K
    us_per_token = 1e3 * ms_per_step / (C * NL)          # one decode step of one layer, cycle avg
    value = whole_job_value(world, B, us_per_token, args.parallel)

    # ---- recurrent baseline (kernel 5a), same tokens, same layers
    def rec_phase():
        for t in range(C):
            for l, b in enumerate(bufs):
                x = inputs[t][l]
                b.recurrent_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
                if tp:
                    comm.allgather(x["o"], gathered[l])

    g_rec = capture(torch, stream, rec_phase)
    barrier()
    rec_total, (rec_ms,) = timed_graphs(torch, stream, [g_rec], K, W)
    barrier()
    t_c2 = time.time()
    rec_total = max_over_ranks(rec_total)
    rec_us_per_token = 1e3 * rec_total / K / (C * NL)

    # ---- roofline of the dominant kernel (buffered decode, kernel 1; with the
    #      fused flush its filling step also writes the folded state)
    uf_dec_bytes_per_launch = B * sum(lb.decode(j) for j in range(C)) / C
    uf_dec_us = 1e3 * dec_ms / (K * dec_launches)
    if auto:
        dec_bytes_per_launch = B * (sum(lb.decode(j) for j in range(C)) + lb.st) / C
        dec_us = 1e3 * fdec_ms / (K * dec_launches)
    else:
        dec_bytes_per_launch, dec_us = uf_dec_bytes_per_launch, uf_dec_us
    fl_bytes_per_launch = B * lb.flush(C)
    fl_us = 1e3 * fl_ms / (K * fl_launches)
    rec_bytes_per_launch = B * lb.recurrent()
    rec_us = 1e3 * rec_ms / (K * C * NL)
    gbs = lambda nbytes, us: nbytes / (us * 1e-6) / 1e9
    dec_gbs = gbs(dec_bytes_per_launch, dec_us)
    step_bytes = NL * (B * sum(lb.decode(j) for j in range(C)) + (B * lb.st if auto else fl_bytes_per_launch))
    uf_us_per_token = 1e3 * uf_total_ms / K / (C * NL)
    traffic = ncu_traffic("decode_cycle_fused" if auto else "decode")
    traffic_fl = ncu_traffic("flush")
    traffic_rec = ncu_traffic("recurrent_step")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if tp else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": (f"config2: Qwen3-Next GDN layer decode, batch {B} @32K ctx (synthetic state), C={C}, "
                                f"heads split over {world} rank(s)" if tp else
                                f"config2: Qwen3-Next GDN layer decode, batch {B}/GPU @32K ctx (synthetic state), C={C}"),
                   "batch_per_gpu": B, "global_batch": B if tp else B * world, "chunk": C, "layers_rotated": NL,
                   "heads": {"qk": Hk, "v": Hv, "d": D}, "in_dtype": args.in_dtype, "u_dtype": args.u_dtype,
                   "state": "fp32",
                   "parallelism": (f"tp{world} (heads partitioned; one la_tp_allgather (NCCL) of the head outputs "
                                   f"per layer per step, not overlapped, inside the timed region)" if tp else
                                   f"dp{world} (requests partitioned, no collective)"),
                   "step": (f"one buffer cycle: {C} decode steps, the last folding the buffer in-kernel "
                            f"(fused flush), x {NL} layer instances" if auto else
                            f"one buffer cycle: {C} decode steps + 1 flush, x {NL} layer instances"
                            + (" (each layer's flush right after its filling decode)" if in_order else "")),
                   "fused_flush": auto,
                   "l2": f"inputs larger than L2: {NL} layers x {B * lb.st / 2**20:.0f} MiB state rotated per step",
                   "cuda_graphs": True, "launch_overlap": not args.no_overlap},
        "us_per_token": us_per_token,
        "tokens_per_s_per_gpu": value / world,
        "hbm_frac_of_8TBs": step_bytes / (ms_per_step * 1e-3) / 8e12,
        "hbm_frac_of_measured": step_bytes / (ms_per_step * 1e-3) / (peak * 1e9),
        "recurrent": {"us_per_token": rec_us_per_token,
                      "tokens_per_s_per_gpu": B / (rec_us_per_token * 1e-6),
                      "hbm_frac_of_measured": gbs(rec_bytes_per_launch, rec_us) / peak},
        "unfused": {"us_per_token": uf_us_per_token, "tokens_per_s_per_gpu": B / (uf_us_per_token * 1e-6),
                    "note": "the cycle with the separate tcgen05 flush kernel (la_set_auto_flush 0), all decode "
                            "steps of the cycle first, then the flushes (per-kernel times come from this run)"},
        "in_order": {"us_per_token": 1e3 * io_total_ms / K / (C * NL),
                     "note": "the same launches in the serving order: each layer's flush directly after the "
                             "decode that filled its buffers (eager flush, reading Z15)"},
        "fused_flush": {"us_per_token": 1e3 * f_total_ms / K / (C * NL),
                        "note": "the cycle with the flush folded into the filling decode step on CUDA cores "
                                "(la_set_auto_flush 1, SURVEY NEXT-1); slower on B200: the 64-thread decode CTA "
                                "is compute-bound on the C x 64 x 128 fold"},
        "speedup_vs_recurrent": rec_us_per_token / us_per_token,
        "latency_reduction_pct_vs_recurrent": 100.0 * (1 - us_per_token / rec_us_per_token),
        "paper_context": {"latency_reduction_pct": 45.17, "capacity_x": 5,
                          "hardware": "4x NVIDIA L40S, TP=4, SGLang v0.5.10 + Triton, FP32 state / FP16 KV (P:12, P:232, P:258, P:266)"},
        "kernels": {
            "decode": {"us_per_launch": dec_us, "bytes_per_launch": dec_bytes_per_launch,
                       "gbs": dec_gbs, "frac_of_measured": dec_gbs / peak, "launches_per_step": dec_launches,
                       "share_of_step": 1.0 if auto else dec_ms / (dec_ms + fl_ms),
                       "fused_flush": auto, "ncu_dram_bytes_per_launch": traffic},
            "decode_unfused": {"us_per_launch": uf_dec_us, "bytes_per_launch": uf_dec_bytes_per_launch,
                               "gbs": gbs(uf_dec_bytes_per_launch, uf_dec_us),
                               "frac_of_measured": gbs(uf_dec_bytes_per_launch, uf_dec_us) / peak},
            "flush": {"us_per_launch": fl_us, "bytes_per_launch": fl_bytes_per_launch,
                      "gbs": gbs(fl_bytes_per_launch, fl_us), "frac_of_measured": gbs(fl_bytes_per_launch, fl_us) / peak,
                      "launches_per_step": fl_launches, "share_of_unfused_step": fl_ms / (dec_ms + fl_ms),
                      "ncu_dram_bytes_per_launch": traffic_fl},
            "recurrent_step": {"us_per_launch": rec_us, "bytes_per_launch": rec_bytes_per_launch,
                               "gbs": gbs(rec_bytes_per_launch, rec_us),
                               "frac_of_measured": gbs(rec_bytes_per_launch, rec_us) / peak,
                               "ncu_dram_bytes_per_launch": traffic_rec},
        },
        "roofline": {"bound": "hbm", "kernel": "chunk_cta_kernel (buffered decode, kernel 1)",
                     "achieved": dec_gbs, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": dec_gbs / peak,
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": dec_bytes_per_launch,
                     "note": "achieved = B x (sum_j (st + inp + j*rec + o + rec) over occupancies j = 0..C-1 "
                             "+ st written by the fused fold) / C (DESIGN.md section 6) / mean launch time from CUDA "
                             "events around the captured decode graph; traffic = ncu dram bytes per launch "
                             "(profiles/ncu_traffic.json)"},
        "gpu_launches": launches_per_step * K,
        # environment overrides that change what runs (the library path; the
        # NCCL path of the TP helpers): recorded, never silent
        "env_overrides": {k: os.environ[k] for k in ("LABUF_LIB", "LABUF_NCCL_LIB") if k in os.environ},
    }

    # ---- e2e through the public API with host buffers: every step copies
    #      that step's q/k/v/alpha/beta from pinned host memory and every
    #      output back.  Per token position t one contiguous pinned block
    #      holds the inputs (resp. outputs) of all layers, so a step is 16
    #      H2D + 16 D2H copies; the H2D of t+1 and the D2H of t run on two
    #      copy streams beside the decodes of t, and the whole step (copies,
    #      la_* calls, events) is one CUDA graph launched per step.
    K_e2e = min(K, 10)
    names = ("q", "k", "v", "alpha", "beta")
    if args.no_e2e:
        K_e2e = 0

    if K_e2e:
        def carve(nbytes_list):
            offs, o = [], 0
            for nb in nbytes_list:
                offs.append(o)
                o += (nb + 255) // 256 * 256
            return offs, o
        in_specs = [(k_, inputs[0][0][k_].shape, inputs[0][0][k_].dtype) for k_ in names]
        in_nb = [int(torch.Size(sh).numel()) * torch.empty(0, dtype=dt).element_size() for _, sh, dt in in_specs]
        offs, per_layer = carve(in_nb)
        o_nb = B * Hv * D * 4
        dev_in = [torch.empty(NL * per_layer, dtype=torch.uint8, device=dev) for _ in range(C)]
        # TP: each layer's gathered head outputs of all ranks come back
        osh = (NL, world, B, Hv, D) if tp else (NL, B, Hv, D)
        dev_out = [torch.empty(osh, dtype=torch.float32, device=dev) for _ in range(C)]
        host_out = [torch.empty(osh, dtype=torch.float32).pin_memory() for _ in range(C)]
        o_loc = [torch.empty(B, Hv, D, dtype=torch.float32, device=dev) for _ in range(NL)] if tp else None
        host_in = [torch.empty(NL * per_layer, dtype=torch.uint8).pin_memory() for _ in range(C)]
        views = []
        for t in range(C):
            row = []
            for l in range(NL):
                v = {}
                for (k_, sh, dt), off, nb in zip(in_specs, offs, in_nb):
                    base = l * per_layer + off
                    v[k_] = dev_in[t][base:base + nb].view(dt).view(sh)
                    v[k_].copy_(inputs[t][l][k_])                    # the same values as the device-resident run
                v["o"] = o_loc[l] if tp else dev_out[t][l]
                row.append(v)
            views.append(row)
            host_in[t].copy_(dev_in[t])
        torch.cuda.synchronize()
        h2d = sum(x.numel() for x in host_in)
        d2h = sum(x.numel() * 4 for x in host_out)
        h2d_stream = torch.cuda.Stream(device=dev)
        d2h_stream = torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(C)]
        ev_out = [torch.cuda.Event() for _ in range(C)]

        def e2e_step():
            h2d_stream.wait_stream(stream)
            d2h_stream.wait_stream(stream)
            with torch.cuda.stream(h2d_stream):
                for t in range(C):
                    dev_in[t].copy_(host_in[t], non_blocking=True)
                    ev_in[t].record(h2d_stream)
            for t in range(C):
                stream.wait_event(ev_in[t])
                for l, b in enumerate(bufs):
                    x = views[t][l]
                    b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
                    if tp:
                        comm.allgather(x["o"], dev_out[t][l])
                ev_out[t].record(stream)
            for b in bufs:
                b.flush(0, B, L.LA_FLUSH_FULL)
            with torch.cuda.stream(d2h_stream):
                for t in range(C):
                    d2h_stream.wait_event(ev_out[t])
                    host_out[t].copy_(dev_out[t], non_blocking=True)
            stream.wait_stream(h2d_stream)
            stream.wait_stream(d2h_stream)

        g_e2e = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_e2e, stream=stream):
            e2e_step()
        for _ in range(2):
            g_e2e.replay()
        barrier()
        t0 = time.perf_counter()
        for _ in range(K_e2e):
            with torch.cuda.stream(stream):
                g_e2e.replay()
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        # the outputs really came back: the last step's host copy equals the device outputs
        e2e_ok = bool(torch.equal(host_out[C - 1], dev_out[C - 1].cpu()))
        e2e_us_tok = 1e6 * e2e_s / K_e2e / (C * NL)
        # the same step issued eagerly: every la_* call (validation, host
        # mirror, launch) and every copy is issued by the host each step
        with torch.cuda.stream(stream):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(K_e2e):
            with torch.cuda.stream(stream):
                e2e_step()
        barrier()
        eager_s = max_over_ranks(time.perf_counter() - t0)
        eager_ok = bool(torch.equal(host_out[C - 1], dev_out[C - 1].cpu()))
        eager_us_tok = 1e6 * eager_s / K_e2e / (C * NL)
        line["e2e"] = {"value": whole_job_value(world, B, e2e_us_tok, args.parallel), "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "steps": K_e2e, "outputs_checked": e2e_ok,
                       "eager": {"value": whole_job_value(world, B, eager_us_tok, args.parallel), "unit": UNIT,
                                 "outputs_checked": eager_ok,
                                 "note": "the same step without a CUDA graph: the host issues every la_* call "
                                         "and every copy each step"},
                       "note": "la_* calls through the public binding with pinned host buffers: H2D of every "
                               "step's q/k/v/alpha/beta and D2H of every output inside the timed region (16 + 16 "
                               "contiguous copies per step on two copy streams beside the decodes; the step is "
                               "one captured CUDA graph); wall clock, max over ranks"}
        del g_e2e, dev_in, dev_out, views

    # ---- extra rows: verify + commit (config 3) and direct (config 4)
    if not args.no_rows and not tp:
        # the rows allocate their own handles (config 5 needs almost all of HBM)
        del g_rec, bufs, inputs
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        line["rows"] = extra_rows(torch, L, cost, dev, stream, seed0 + 5000, K, W, peak, args)

    t_c3 = time.time()
    clocks.stop()
    line["clocks"] = clocks.summary(t_c0, t_c2)

    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_sample(seed=args.seed)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()


def extra_rows(torch, L, cost, dev, stream, seed, K, W, peak, args):
    """Config 3 (verify + commit vs recurrent verify + copy) and config 4
    (direct decode vs recurrent) at their BASELINE sizes."""
    import synth.device as sd
    rows = {}
    Hk, Hv = 16, 32
    Kr = max(3, min(K, 20))
    if not args.no_config5:   # first: it needs almost all of HBM
        try:
            rows["config5"] = row_config5(torch, L, cost, sd, dev, seed + 80, peak, args)
        except torch.cuda.OutOfMemoryError as e:
            rows["config5"] = {"error": f"out of memory: {e}"[:300]}
        torch.cuda.empty_cache()
    gbs = lambda nbytes, us: nbytes / (us * 1e-6) / 1e9
    # ---------------- config 2, flush mode ii (LA_FLUSH_RAW): u recomputed in the
    #                  flush by the UT transform from the raw records (keep_raw)
    B2, C2, NL2 = args.batch, args.chunk, 4
    in_b = 2 if args.in_dtype == "bf16" else 4
    lb2 = cost.LayerBytes.make(Hk, Hv, D, in_b, 4)
    cfg = L.make_config(B2, Hk, Hv, chunk=C2, in_dtype=args.in_dtype, keep_raw=True)
    bufs = [L.LaBuf(cfg, device=dev) for _ in range(NL2)]
    for b in bufs:
        b.reset(zero_state=False)
    fill_states(torch, bufs, seed + 1)
    torch.cuda.synchronize()
    for b in bufs:
        b.set_overlap(not args.no_overlap)
    xs2 = [make_inputs(torch, B2, Hk, Hv, NL2, args.in_dtype, seed + 2 + t, dev) for t in range(C2)]

    def dec2():
        for t in range(C2):
            for b, x in zip(bufs, xs2[t]):
                b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])

    def fl2(kind):
        def f():
            for b in bufs:
                b.flush(0, B2, kind)
        return f
    gd2 = capture(torch, stream, dec2)
    gr2 = capture(torch, stream, fl2(L.LA_FLUSH_FULL | L.LA_FLUSH_RAW))
    _, (_, raw_ms) = timed_graphs(torch, stream, [gd2, gr2], Kr, W)
    gd2b = capture(torch, stream, dec2)      # the host mirror follows captures: one cycle each
    gi2 = capture(torch, stream, fl2(L.LA_FLUSH_FULL))
    _, (_, ui_ms) = timed_graphs(torch, stream, [gd2b, gi2], Kr, W)
    raw_us = 1e3 * raw_ms / Kr / NL2
    ui_us = 1e3 * ui_ms / Kr / NL2
    raw_bytes = B2 * (2 * lb2.st + C2 * (Hk * D * in_b + Hv * D * in_b + 8 * Hv))
    rows["flush_mode_ii"] = {
        "workload": f"config2: batch {B2}, C={C2}, keep_raw records, {NL2} layers rotated",
        "us_per_launch": raw_us, "bytes_per_launch": raw_bytes,
        "gbs": gbs(raw_bytes, raw_us), "frac_of_measured": gbs(raw_bytes, raw_us) / peak,
        "mode_i_us_per_launch_same_buffers": ui_us,
        "note": "UT transform in the flush (P:392-399, reading Z4): Gram K K^T, A = (I + L)^-1 by forward "
                "substitution, V~ = A Diag(beta) V before the state lands; U = V~ - Q (K S0^T) and the fold on "
                "split-TF32 mma.sync, one 8-warp CTA per (head, slot) (csrc/fold_ut.cu)",
    }
    del gd2, gr2, gd2b, gi2, bufs, xs2
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # ---------------- config 3: batch 256, 4 drafts, verify + commit vs recurrent verify + copy
    B3, N3, NL3 = 256, args.drafts, 2
    lb = cost.LayerBytes.make(Hk, Hv, D, 2, 4)
    cfg = L.make_config(B3, Hk, Hv, chunk=16, max_drafts=N3)
    bufs = [L.LaBuf(cfg, device=dev) for _ in range(NL3)]
    for b in bufs:
        b.reset(zero_state=False)
    fill_states(torch, bufs, seed)
    torch.cuda.synchronize()
    for b in bufs:
        b.set_overlap(not args.no_overlap)
    nacc = [sd.n_accepted(seed + 10 + l, B3, N3, device=dev) for l in range(NL3)]
    xs = []
    for l in range(NL3):
        x = sd.tokens(seed + 20 + l, B3, N3, Hk, Hv, D, device=dev)
        x["o"] = torch.empty(B3, N3, Hv, D, dtype=torch.float32, device=dev)
        xs.append(x)

    def ver():
        for b, x in zip(bufs, xs):
            b.verify_drafts(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])

    def com():
        for b, na in zip(bufs, nacc):
            b.commit_accepted(0, na)
    gv, gc = capture(torch, stream, ver), capture(torch, stream, com)
    tot, (v_ms, c_ms) = timed_graphs(torch, stream, [gv, gc], Kr, W)
    us_round = 1e3 * tot / Kr / NL3
    acc_mean = float(sum(int(n.sum()) for n in nacc)) / (NL3 * B3)
    ver_bytes = B3 * lb.verify(N3)
    com_bytes = sum(lb.commit(0, int(a)) for na in nacc for a in na.cpu().tolist()) / NL3
    temps = [torch.empty(B3, N3, Hv, D, D, dtype=torch.float32, device=dev) for _ in range(NL3)]

    def rver():
        for b, x, tp in zip(bufs, xs, temps):
            b.recurrent_verify(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], tp, x["o"])

    def rcom():
        for b, na, tp in zip(bufs, nacc, temps):
            b.recurrent_commit(0, na, tp)
    grv, grc = capture(torch, stream, rver), capture(torch, stream, rcom)
    rtot, (rv_ms, rc_ms) = timed_graphs(torch, stream, [grv, grc], Kr, W)
    # multi-round buffered speculation (la_commit_append): the
    # accepted drafts stay buffered, the state is folded once the buffer holds
    # C tokens -- one closed cycle of rounds (appends + the folding commit) per graph
    n_cycle = 0
    occ_ub = 0
    while True:
        n_cycle += 1
        if occ_ub + N3 > 16 or occ_ub + 2 * N3 > bufs[0].capacity:
            break
        occ_ub += N3

    def multi():
        for _ in range(n_cycle):
            ver()
            for b, na in zip(bufs, nacc):
                b.commit_append(0, na)
    gm = capture(torch, stream, multi)
    mtot, _ = timed_graphs(torch, stream, [gm], Kr, W)
    m_us_round = 1e3 * mtot / Kr / NL3 / n_cycle
    rus_round = 1e3 * rtot / Kr / NL3
    v_us = 1e3 * v_ms / Kr / NL3
    c_us = 1e3 * c_ms / Kr / NL3
    rows["verify_commit"] = {
        "workload": f"config3: batch {B3}, {N3} drafts, p_accept 0.7 (mean n_acc {acc_mean:.2f}), {NL3} layers rotated",
        "us_per_round": us_round, "verify_us": v_us, "commit_us": c_us,
        "verify_gbs": gbs(ver_bytes, v_us), "verify_frac_of_measured": gbs(ver_bytes, v_us) / peak,
        "commit_gbs": gbs(com_bytes, c_us), "commit_frac_of_measured": gbs(com_bytes, c_us) / peak,
        "recurrent_us_per_round": rus_round,
        "recurrent_verify_gbs": gbs(B3 * lb.recurrent_verify(N3), 1e3 * rv_ms / Kr / NL3),
        "speedup_vs_recurrent": rus_round / us_round,
        "paper_context": "2.78x at 8 drafts on 4x L40S (P:263); model ((m+1)d+2m)/(3d+4m) = 1.62 at 4 drafts (P:190)",
        "multi_round": {"us_per_round": m_us_round, "rounds_per_fold": n_cycle,
                        "speedup_vs_recurrent": rus_round / m_us_round,
                        "note": "la_commit_append: accepted drafts stay buffered, one fold per cycle of rounds "
                                "(C = 16); verify reads the growing buffer"},
        "temp_state_bytes_recurrent": B3 * N3 * lb.st,
        "capacity_requests_36_layers_180GB": {
            "recurrent": int(180e9 // (36 * (N3 + 1) * lb.st)),
            "buffered": int(180e9 // (36 * (lb.st + bufs[0].sizes.capacity * lb.rec))),
            "buffered_records_reserved_per_slot": bufs[0].sizes.capacity,
            # the paper's 5x counts one state plus the N draft records
            # (a paged pool with blocks of N records, la_buf_query-sized)
            "buffered_drafts_only": int(180e9 // (36 * (lb.st + N3 * lb.rec))),
        },
    }
    del gv, gc, grv, grc, gm, temps, bufs, xs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # ---------------- config 4: batch 1024, direct KV-only decode at context 64 -> 96
    B4, L0, NS = 1024, args.direct_l0, min(32, 128 - args.direct_l0)
    cfg = L.make_config(B4, Hk, Hv, chunk=16, short_cap=128, u_dtype="f16")
    b4 = L.LaBuf(cfg, device=dev)
    b4.set_overlap(not args.no_overlap)
    lb4 = cost.LayerBytes.make(Hk, Hv, D, 2, 2)
    pre = sd.tokens(seed + 30, B4, L0, Hk, Hv, D, device=dev)
    pre["o"] = torch.empty(B4, L0, Hv, D, dtype=torch.float32, device=dev)
    steps = []
    for i in range(NS):
        x = sd.tokens(seed + 40 + i, B4, 1, Hk, Hv, D, device=dev)
        x["o"] = torch.empty(B4, 1, Hv, D, dtype=torch.float32, device=dev)
        steps.append(x)

    def run_direct():
        b4.reset(mode=L.LA_MODE_DIRECT, zero_state=False)
        b4.direct_short(0, pre["q"], pre["k"], pre["v"], pre["alpha"], pre["beta"], pre["o"])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for x in steps:
                b4.direct_short(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
            e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    run_direct()
    d_ms = min(run_direct() for _ in range(3))
    d_us = 1e3 * d_ms / NS
    d_bytes = B4 * sum(lb4.direct(L0 + s) for s in range(NS)) / NS
    # recurrent baseline at the same batch and the same tokens
    cfgr = L.make_config(B4, Hk, Hv, chunk=16)
    br = L.LaBuf(cfgr, device=dev)
    br.set_overlap(not args.no_overlap)
    br.reset(zero_state=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sq = [{k: v[:, 0].contiguous() for k, v in x.items()} for x in steps]
    r_ms = []
    for rep in range(3):
        with torch.cuda.stream(stream):
            e0.record(stream)
            for x in sq:
                br.recurrent_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
            e1.record(stream)
        torch.cuda.synchronize()
        r_ms.append(e0.elapsed_time(e1))
    r_us = 1e3 * min(r_ms) / NS
    # Fig. 7 analogue: direct at context L (8 steps from L) vs chunkwise C = 16
    # (cycle of 16 decodes + the flush, same batch) vs recurrent
    fig7 = []
    for Lc in (16, 32, 64, 96, 120):
        x0 = sd.tokens(seed + 60 + Lc, B4, Lc, Hk, Hv, D, device=dev)
        x0["o"] = torch.empty(B4, Lc, Hv, D, dtype=torch.float32, device=dev)
        b4.reset(mode=L.LA_MODE_DIRECT, zero_state=False)
        b4.direct_short(0, x0["q"], x0["k"], x0["v"], x0["alpha"], x0["beta"], x0["o"])
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for x in steps[:8]:
                b4.direct_short(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
            e1.record(stream)
        torch.cuda.synchronize()
        du = 1e3 * e0.elapsed_time(e1) / 8
        db = B4 * sum(lb4.direct(Lc + s_) for s_ in range(8)) / 8
        fig7.append({"context": Lc + 4, "direct_us_per_step": du, "direct_frac_of_measured": gbs(db, du) / peak})
        del x0
    del b4
    torch.cuda.empty_cache()
    # chunkwise C = 16 at the same batch (one layer: 2 GiB of state > L2)
    cfgc = L.make_config(B4, Hk, Hv, chunk=16, u_dtype="f16")
    bc = L.LaBuf(cfgc, device=dev)
    bc.set_overlap(not args.no_overlap)
    bc.reset(zero_state=True)

    def cyc():
        for x in sq[:16]:
            bc.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
        bc.flush(0, B4, L.LA_FLUSH_FULL)
    gcy = capture(torch, stream, cyc)
    _, (cy_ms,) = timed_graphs(torch, stream, [gcy], 5, 3)
    chunk_us = 1e3 * cy_ms / 5 / 16
    for row in fig7:
        row["chunkwise_c16_us_per_token"] = chunk_us
        row["recurrent_us_per_step"] = r_us
        row["direct_vs_chunkwise"] = chunk_us / row["direct_us_per_step"]
        row["paper_model_direct_vs_chunkwise"] = float(cost.paper_speedup_kv_only_gdn(D, 16, row["context"]))
    del gcy, bc
    rows["direct"] = {
        "workload": f"config4: batch {B4}, direct KV-only decode from context {L0} to {L0 + NS}, u fp16, no state",
        "us_per_step": d_us, "gbs": gbs(d_bytes, d_us), "frac_of_measured": gbs(d_bytes, d_us) / peak,
        "recurrent_us_per_step": r_us, "speedup_vs_recurrent": r_us / d_us,
        "chunkwise_c16_us_per_token": chunk_us, "speedup_vs_chunkwise": chunk_us / d_us,
        "paper_model_speedup_vs_chunkwise_m16_at_L80": float(cost.paper_speedup_kv_only_gdn(D, 16, L0 + NS // 2)),
        "fig7": fig7,
        "fig7_note": "batch 1024, u fp16; direct at context L..L+8 vs the chunkwise C = 16 cycle (u fp16) and "
                     "the recurrent step at the same batch; the paper's claim is direct ~ chunkwise near L = d "
                     "(P:287-290, Eq. 10 P:212)",
    }
    del br
    torch.cuda.empty_cache()
    if not args.no_config1:
        rows["config1"] = row_config1(torch, L, sd, dev, stream, seed + 70)
    rows["prefill"] = row_prefill(torch, L, cost, sd, dev, stream, seed + 90, peak)
    return rows


def row_prefill(torch, L, cost, sd, dev, stream, seed, peak, B=64, n_tok=1024):
    """Chunked prefill at scale: a batch of
    64 Qwen3-Next-layer requests, 1024-token prompts from synthetic 32K-ctx
    states, 64-token chunks (16-token launches of the chunk kernel with the
    tensor-core state pass, then the tcgen05 fold), outputs written."""
    Hk, Hv = 16, 32
    cfg = L.make_config(B, Hk, Hv, chunk=16, short_cap=64)
    b = L.LaBuf(cfg, device=dev)
    b.set_overlap(True)
    b.reset(zero_state=False)
    fill_states(torch, [b], seed)
    x = sd.tokens(seed + 1, B, n_tok, Hk, Hv, D, device=dev)
    o = torch.empty(B, n_tok, Hv, D, dtype=torch.float32, device=dev)
    lb = cost.LayerBytes.make(Hk, Hv, D, 2, 4)
    rec_bytes = B * n_tok * lb.recurrent()
    res = {}
    for PC in (16, 64):
        b.set_prefill_chunk(PC)
        l0 = b.kernel_launches()
        g = capture(torch, stream, lambda: b.prefill(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], o))
        launches = b.kernel_launches() - l0
        _, (ms,) = timed_graphs(torch, stream, [g], 5, 3)
        ms /= 5
        # per chunk: launches of 16 tokens (state + inputs + the chunk's earlier
        # records read, outputs + records written) + the fold of the chunk;
        # a chunk of <= 16 tokens is one launch that folds its own records
        # (state read + state written + inputs + outputs, no records)
        if PC <= 16:
            per_chunk = 2 * lb.st + PC * (lb.inp + lb.o)
        else:
            per_chunk = sum(lb.st + 16 * (lb.inp + lb.o + lb.rec) + 16 * j * lb.rec for j in range(PC // 16)) + lb.flush(PC)
        nbytes = B * per_chunk * (n_tok // PC)
        res[PC] = {"ms": ms, "tokens_per_s": B * n_tok / (ms * 1e-3), "algorithmic_bytes": nbytes,
                   "gbs": nbytes / (ms * 1e-3) / 1e9, "frac_of_measured": nbytes / (ms * 1e-3) / (peak * 1e9),
                   "bytes_ratio_vs_recurrent": rec_bytes / nbytes, "kernel_launches": launches}
        del g
    del b, x, o
    torch.cuda.empty_cache()
    best = min(res, key=lambda p: res[p]["ms"])
    out = {"workload": f"prefill: batch {B}, {n_tok}-token prompts, Qwen3-Next GDN layer, outputs written "
                       f"(one CUDA graph per prompt); chunk {best} (la_set_prefill_chunk; 16 and 64 measured)",
           "chunk": best, **res[best], "recurrent_bytes_same_tokens": rec_bytes,
           "by_chunk": {str(p): v for p, v in res.items()}}
    return out


def row_config1(torch, L, sd, dev, stream, seed):
    """Config 1 (BASELINE configs[0]): 1 request, 1 GDN head, d = 128, fp32,
    64-token prefill + 64 decode steps, C = 16, vs the recurrent kernel: the
    batch-1 latency regime where launches, not bytes, set the time."""
    cfg = L.make_config(1, 1, 1, chunk=16, in_dtype="f32")
    b = L.LaBuf(cfg, device=dev)
    b.set_overlap(True)
    b.reset(zero_state=True)
    pre = sd.tokens(seed, 1, 64, 1, 1, D, in_dtype="f32", device=dev)
    pre_o = torch.empty(1, 64, 1, D, dtype=torch.float32, device=dev)
    xs = [sd.tokens(seed + 1 + t, 1, 1, 1, 1, D, in_dtype="f32", device=dev, squeeze=True) for t in range(16)]
    for x in xs:
        x["o"] = torch.empty(1, 1, D, dtype=torch.float32, device=dev)
    g_pre = capture(torch, stream, lambda: b.prefill(0, pre["q"], pre["k"], pre["v"], pre["alpha"], pre["beta"], pre_o))
    _, (pre_ms,) = timed_graphs(torch, stream, [g_pre], 20, 3)

    def cyc():
        for x in xs:
            b.decode_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
        b.flush(0, 1, L.LA_FLUSH_FULL)

    def rec():
        for x in xs:
            b.recurrent_step(0, x["q"], x["k"], x["v"], x["alpha"], x["beta"], x["o"])
    g_cyc, g_rec = capture(torch, stream, cyc), capture(torch, stream, rec)
    _, (cyc_ms,) = timed_graphs(torch, stream, [g_cyc], 50, 5)
    _, (rec_ms,) = timed_graphs(torch, stream, [g_rec], 50, 5)
    buf_us, rec_us = 1e3 * cyc_ms / 50 / 16, 1e3 * rec_ms / 50 / 16
    return {"workload": "config1: 1 request, 1 head, d=128, fp32, 64-token prefill + decode cycles of C=16 "
                        "(16 decodes + flush, one CUDA graph) vs 16 recurrent steps",
            "prefill_64_us": 1e3 * pre_ms / 20,
            "buffered_us_per_token": buf_us, "recurrent_us_per_token": rec_us,
            "speedup_vs_recurrent": rec_us / buf_us,
            "note": "launch-bound: one head is 133 KB per recurrent token; the paper notes the batch-1 penalty "
                    "(P:256)"}


def row_config5(torch, L, cost, sd, dev, seed, peak, args):
    """Config 5 (BASELINE configs[4]): 36 stacked GDN layers, 2048 mixed
    requests (1536 long: buffered decode C = 16, occupancies staggered; 512
    short: KV-only, no state, L0 in {16, 40, 64, 96}) -- this rank's DP shard
    -- on ONE paged handle per layer (record blocks of 16 tokens, a state
    pool for the long requests; paper_2605_19049_b200.stack.MixedStack):
    32 decode steps, one la_decode_mixed per layer per step, eager launches."""
    from paper_2605_19049_b200 import dp
    from paper_2605_19049_b200.stack import MixedStack, StackSpec, short_groups
    world, rank, _ = rank_env()
    sh = dp.mixed_assignment(1536, 512, rank, world)
    spec = StackSpec(n_layers=36, n_long=len(sh.long_ids), n_short=len(sh.short_ids))
    Hk, Hv, NS = spec.n_qk_heads, spec.n_v_heads, 32
    n_tok = spec.n_long + spec.n_short
    headroom = max(1, spec.n_short // len(spec.short_l0))   # states for one short group crossing L = d
    need = MixedStack.footprint_of(spec, state_headroom=headroom)
    torch.cuda.empty_cache()
    free = torch.cuda.mem_get_info(dev)[0]
    if need + 6e9 > free:   # + inputs / outputs of 36 layers and allocator slack
        return {"error": f"does not fit: la_buf_query footprint {need / 1e9:.1f} GB > {free / 1e9:.1f} GB free",
                "footprint_bytes_la_buf_query": need}
    st = MixedStack.create(spec, dev, state_headroom=headroom)
    foot = st.footprint_bytes()
    st.reset(lambda l, view: sd.fill_state0(view, seed + l))
    for b in st.layers:
        b.set_overlap(True)
    # one set of decode inputs per layer (reused over the steps: 36 layers of
    # inputs exceed L2, and the values do not change the work)
    # decode inputs: 4 distinct sets cycled over the 36 layers (4 x 34 MB > L2
    # between reuses; the values do not change the work), one output buffer
    xs4 = [sd.tokens(seed + 100 + l, n_tok, 1, Hk, Hv, D, device=dev, squeeze=True) for l in range(4)]
    xin = [xs4[l % 4] for l in range(36)]
    o1 = torch.empty(n_tok, Hv, D, dtype=torch.float32, device=dev)
    out = [o1] * 36
    pre = {}

    def short_tok(l, g):
        f, m, l0 = short_groups(spec)[g]
        if (m, l0) not in pre:
            pre[(m, l0)] = sd.tokens(seed + 300 + l0, m, l0, Hk, Hv, D, device=dev)
        return pre[(m, l0)]
    st.warmup(lambda l, t: {k: v[:spec.n_long] for k, v in xin[l].items()}, short_tok)
    pre.clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = sum(b.kernel_launches() for b in st.layers)
    stream = torch.cuda.current_stream(dev)
    st.step(xin, out)                      # one untimed step (first-touch of the work lists)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(NS):
        st.step(xin, out)
    e1.record(stream)
    host_s = time.perf_counter() - t0      # host time to issue the 32 steps (la_* calls, staging)
    torch.cuda.synchronize()
    launches = sum(b.kernel_launches() for b in st.layers) - launches0
    ms = e0.elapsed_time(e1) / NS
    finite = bool(torch.isfinite(out[-1]).all())
    pool = st.layers[0].pool_info()
    # algorithmic bytes per stack step (u fp16 records): long slots average one
    # full cycle (32 steps = 2 cycles of C = 16), short slots at their contexts
    lb = cost.LayerBytes.make(Hk, Hv, D, 2, 2)
    long_b = spec.n_long * float(lb.cycle_avg(spec.chunk))
    short_b = sum(m * sum(lb.direct(l0 + 1 + s_) for s_ in range(NS)) / NS for _, m, l0 in short_groups(spec))
    step_bytes = 36 * (long_b + short_b)
    two_handle = None
    try:
        from paper_2605_19049_b200.stack import GdnStack
        two_handle = GdnStack.footprint_of(spec)
    except Exception:
        pass
    del st, xin, out, xs4, o1
    return {"workload": f"config5: 36 Qwen3-Next GDN layers, {n_tok} of 2048 mixed requests on this rank "
                        f"({spec.n_long} long buffered C=16 staggered, {spec.n_short} short KV-only), {NS} steps; "
                        "one paged handle per layer (16-token blocks, state pool), one la_decode_mixed per layer "
                        "per step, eager launches",
            "ms_per_step": ms, "tokens_per_s_per_gpu": n_tok / (ms * 1e-3),
            "us_per_token_per_layer": 1e3 * ms / 36, "host_issue_ms_per_step": 1e3 * host_s / NS,
            "footprint_bytes_la_buf_query": foot, "footprint_gb": foot / 1e9,
            "footprint_gb_two_handle_layout": None if two_handle is None else two_handle / 1e9,
            "pool_layer0": pool,
            "algorithmic_bytes_per_step": step_bytes,
            "hbm_frac_of_measured": step_bytes / (ms * 1e-3) / (peak * 1e9),
            "kernel_launches_per_step": launches / NS, "outputs_finite": finite}


if __name__ == "__main__":
    main()
