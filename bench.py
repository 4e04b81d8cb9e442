#!/usr/bin/env python
"""Benchmark of the CompactFusion residual-compression path on B200.

Metric (BASELINE.json): activation GB/s compressed + reconstructed per GPU, and
exposed communication µs/layer, at 1/2/4/8 B200.

One *step* = one FLUX.1 denoising step of the patch-parallel exchange over
`--layers` (57) independent layer channels of a [4096, 3072] bf16 activation:
per layer, every rank compresses its row shard with the fused residual /
error-feedback 2-bit kernel (K1), all-gathers the packed bodies over NCCL, and
rebuilds every peer's rows into its cached base (K2).  With one GPU the step is
BASELINE config 1 (sender + loopback receiver, world_size=1).  Inputs are
synthetic FLUX-like activations (per-token x per-channel log-normal scales,
small step-to-step drift) resident in HBM; the per-step working set (57 layers
x ~150 MB of state) is far larger than the 126 MB L2, so nothing is L2-warm
between a layer's consecutive steps.

value   = whole-job activation GB/s = sum over ranks of the activation bytes each
          rank reconstructs (the full 2*4096*3072 B per layer) / step time
          (max over ranks); per_gpu_gbs = value / N.  Every rank rebuilds the
          full activation whatever N is, so per-GPU work is fixed ("weak").
e2e     = same metric through the public API with pinned HOST inputs: per layer
          H2D of the bf16 shard, exchange, D2H of the packed body + StepRecord
roofline: K1 (encode_step: residual -> scales -> quantize/pack -> state update)
          achieved = algorithmic bytes (18 + b/8 B per own element + scales)
          / K1 duration, measured with CUDA events recorded INSIDE the replayed
          CUDA graph around every K1 (the headline's launch mode)
cpu_baseline: the reference's own pipeline.encode_step + decode_step
          (oracle/_ref, the unmodified reference package; the numpy port in
          oracle/cc_oracle.py when it is absent) on the host cores, one process
          per core, per-GPU-equivalent work (own-shard encode + (N-1) decodes).

`--gpus N` without a torchrun environment relaunches itself under
torch.distributed.run with N ranks.  `--impl reference` times that same CPU path
as the reference arm (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ROWS, COLS = 4096, 3072
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(ROOT, "profiles", "k1_traffic.json")
BITS = {"sign1bit": 1, "quant2bit": 2, "quant4bit": 4}
METRIC = "activation GB/s compressed+reconstructed per GPU and exposed comm us/layer"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--codec", default="quant2bit", choices=sorted(BITS))
    ap.add_argument("--layers", type=int, default=57)
    ap.add_argument("--topology", default="allgather", choices=["allgather", "ring"],
                    help="patch-parallel all-gather (default) or ring-attention style P-1 hop forwarding")
    ap.add_argument("--rows", type=int, default=ROWS)
    ap.add_argument("--cols", type=int, default=COLS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sim", action="store_true", help="skip the single-GPU per-rank simulations of "
                    "the 2/4/8-GPU patch-parallel and 8-GPU Ulysses configs (`per_rank_sim`)")
    ap.add_argument("--no-overlap", action="store_true", help="K2 on the compute stream (default: its own "
                    "decode stream, so layer l's decode overlaps layer l+1's K1: +3 %% at N=1, measured)")
    ap.add_argument("--pdl", type=int, default=None, help="programmatic dependent launch for K1/K2 "
                    "(1 on, 0 off; default: the library default)")
    ap.add_argument("--overlap", action="store_true", help="(default) K2 on its own decode stream")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel from Python instead of "
                                                             "replaying a captured CUDA graph per step")
    ap.add_argument("--cpu-procs", type=int, default=None, help="host processes for the CPU path "
                    "(default: min(cpu_count, 16) for cpu_baseline, cpu_count for --impl reference)")
    return ap.parse_args(argv)


def bench_config(a, world):
    """The workload both arms run (identical dict in both JSON lines)."""
    n_own = a.rows // world
    return {"workload": (f"FLUX.1 [{a.rows}x{a.cols}] {a.codec} residual+EF patch-parallel exchange, "
                         f"{a.layers} layer channels per step, world_size={world}: per rank-layer encode_step(own "
                         f"[{n_own},{a.cols}] shard) + {'(N-1) peer decode_steps' if world > 1 else 'loopback receiver decode_step (BASELINE config 1)'}"),
            "codec": a.codec, "layers": a.layers, "rows": a.rows, "cols": a.cols, "shard_rows": n_own,
            "parallelism": f"patch{world}", "topology": a.topology, "input_dtype": "bf16", "state_dtype": "f32",
            "l2": "per-step working set >> 126 MB L2 (no flush needed)"}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(a):
    """`--gpus N` outside torchrun: re-exec this script as N torchrun ranks."""
    import torch

    have = torch.cuda.device_count()
    if have < a.gpus:
        print(f"bench: --gpus {a.gpus} needs {a.gpus} GPUs, this node has {have}", file=sys.stderr, flush=True)
        return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local if world > 1 else 0)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank


def max_over_ranks(v, world):
    import torch
    import torch.distributed as dist

    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m, r = float(parts[0]), float(parts[1]), int(parts[2], 16)
            except ValueError:
                continue
            mx = max(mx, m)
            if r & 0x1:  # idle sample: not under load
                continue
            sm.append(s)
            for bit, name in REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# synthetic inputs on device
# ---------------------------------------------------------------------------

def flux_inputs(rows, cols, lo, hi, layer, device):
    """Two consecutive denoising-step activations of one layer, shard [lo:hi]."""
    import torch

    out = []
    g = torch.Generator(device=device).manual_seed(1000 * layer)
    a = torch.empty(rows, 1, device=device).log_normal_(0.0, 0.25, generator=g)
    c = torch.empty(1, cols, device=device).log_normal_(0.0, 1.0, generator=g)
    x = a * c * torch.randn(rows, cols, device=device, generator=g)
    out.append(x.to(torch.bfloat16)[lo:hi].contiguous())
    g2 = torch.Generator(device=device).manual_seed(1000 * layer + 1)
    x = x + 0.1 * a * c * torch.randn(rows, cols, device=device, generator=g2)
    out.append(x.to(torch.bfloat16)[lo:hi].contiguous())
    return out


# ---------------------------------------------------------------------------
# CPU path — cpu_baseline and --impl reference
# ---------------------------------------------------------------------------

def _cpu_worker(conn, gate, impl):
    """One host process: per request, build one rank-layer channel set and time
    one compressed step of it (encode own shard + (world-1) peer decodes, or one
    loopback decode at world 1).  Setup and the raw warmup step are untimed."""
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    import numpy as np

    if impl == "reference":
        from oracle.build_ref import import_reference

        cx, pl, _ = import_reference()
    else:
        from oracle import cc_oracle as O
    while True:
        req = conn.recv()
        if req is None:
            return
        rows, cols, world, codec, seed = req
        n = rows // world
        rng = np.random.Generator(np.random.PCG64(seed))
        a = rng.lognormal(0.0, 0.25, (n, 1)).astype(np.float32)
        c = rng.lognormal(0.0, 1.0, (1, cols)).astype(np.float32)
        x0 = (a * c * rng.standard_normal((n, cols), dtype=np.float32)).astype(np.float32)
        x1 = (x0 + 0.1 * a * c * rng.standard_normal((n, cols), dtype=np.float32)).astype(np.float32)
        peers = max(1, world - 1)
        if impl == "reference":
            spec = cx.CompressorSpec(cx.CompressorKind(codec))
            mode = pl.PipelineMode.RESIDUAL_WITH_FEEDBACK
            snd = pl.LayerState(mode, 1, np.zeros((n, cols), np.float32))
            rcv = [pl.LayerState(mode, 1, np.zeros((n, cols), np.float32)) for _ in range(peers)]
            p0, _ = pl.encode_step(snd, x0, spec)
            m0 = pl.message_for(1, 1, p0)
            for r in rcv:
                pl.decode_step(r, m0)

            def unit():
                p1, _ = pl.encode_step(snd, x1, spec)
                m1 = pl.message_for(2, 1, p1)
                for r in rcv:
                    pl.decode_step(r, m1)
        else:
            cdc = O.Codec({"sign1bit": O.SIGN1, "quant2bit": O.QUANT2}.get(codec, O.QUANT2))
            snd = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((n, cols), np.float32))
            rcv = [O.Channel(O.WITH_FEEDBACK, 1, np.zeros((n, cols), np.float32)) for _ in range(peers)]
            t0 = O.send(snd, x0, cdc)
            for r in rcv:
                O.receive(r, 1, True, O.RAW, t0[1], O.Codec(O.RAW))

            def unit():
                tg, body, _ = O.send(snd, x1, cdc)
                for r in rcv:
                    O.receive(r, 2, False, tg, body, cdc)
        gate.wait()
        start = time.perf_counter()
        unit()
        conn.send((start, time.perf_counter()))


class CpuPath:
    """`procs` persistent host processes (spawned, one per core, single-threaded
    numpy) running the CPU path concurrently; perf_counter is CLOCK_MONOTONIC, so
    spans from different processes share one time base."""

    def __init__(self, procs):
        import multiprocessing as mp

        from oracle.build_ref import import_reference

        self.impl = "reference" if import_reference() is not None else "port"
        ctx = mp.get_context("spawn")
        self.procs = procs
        self.gate = ctx.Barrier(procs)
        self.conns, self.workers = [], []
        for _ in range(procs):
            parent, child = ctx.Pipe()
            w = ctx.Process(target=_cpu_worker, args=(child, self.gate, self.impl), daemon=True)
            w.start()
            self.conns.append(parent)
            self.workers.append(w)

    def measure(self, rows, cols, world, codec, seed=17):
        """One step of `procs` concurrent rank-layer units: (activation GB/s, wall s)."""
        for i, c in enumerate(self.conns):
            c.send((rows, cols, world, codec, seed + i))
        spans = [c.recv() for c in self.conns]
        wall = max(e for _, e in spans) - min(s for s, _ in spans)
        return self.procs * 2 * rows * cols / wall / 1e9, wall

    def close(self):
        for c in self.conns:
            c.send(None)
        for w in self.workers:
            w.join(timeout=10)

    def describe(self, rows, cols, world, codec, wall):
        src = ("oracle/_ref: the unmodified reference package (compactcomm.pipeline.encode_step / decode_step)"
               if self.impl == "reference" else "oracle/cc_oracle.py numpy restatement of pipeline.encode_step/decode_step")
        work = (f"encode_step own [{rows // world},{cols}] shard + {world - 1} peer decode_step" if world > 1
                else f"encode_step + loopback decode_step [{rows},{cols}]")
        return (f"{self.procs} concurrent rank-layer units ({work}, {codec} residual+EF) on {self.procs} "
                f"single-threaded host processes, {wall:.2f} s wall per step; {src}")


def run_reference(a, world, rank):
    """Reference arm: the reference's CPU path on the host cores (rank 0 only)."""
    if rank != 0:
        return
    procs = a.cpu_procs or os.cpu_count() or 1
    cpu = CpuPath(procs)
    try:
        for _ in range(a.warmup):
            cpu.measure(a.rows, a.cols, world, a.codec)
        walls = [cpu.measure(a.rows, a.cols, world, a.codec)[1] for _ in range(a.steps)]
    finally:
        cpu.close()
    ms = statistics.mean(walls) * 1e3
    value = procs * 2 * a.rows * a.cols / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic FLUX-like activations (log-normal token x channel "
                                                     "scales, 10% step drift)",
        "config": bench_config(a, world),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": procs, "kind": cpu.impl,
                         "sample": cpu.describe(a.rows, a.cols, world, a.codec, statistics.mean(walls))},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_b200(a, world, rank):
    import torch

    from paper_2507_17511_b200 import _lib
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200.comm import PatchParallelExchange, RingExchange, shard_bounds

    lib = _lib.load()
    if a.pdl is not None:
        lib.cc_set_pdl(int(a.pdl))
    dev = torch.device("cuda", torch.cuda.current_device())
    spec = cx.CompressorSpec(cx.CompressorKind(a.codec))
    L, rows, cols = a.layers, a.rows, a.cols
    bounds = shard_bounds(rows, world) if world > 1 else [(0, rows)]
    lo, hi = bounds[rank]
    n_own = hi - lo
    Ex = RingExchange if a.topology == "ring" else PatchParallelExchange
    overlap = not a.no_overlap
    exs = []

    def make_exchanges():
        exs[:] = [Ex(rows, cols, spec, overlap=overlap) for _ in range(L)]
        for e in exs[1:]:
            e.streams = exs[0].streams  # one compute / comm / decode stream triple for the whole model
        return exs[0].streams

    streams = make_exchanges()
    inputs = [flux_inputs(rows, cols, lo, hi, layer, dev) for layer in range(L)]

    def one_step(par, skip_comm=False, k1=None, k2=None):
        for layer, e in enumerate(exs):
            e.step(inputs[layer][par], skip_comm=skip_comm, k1_events=None if k1 is None else k1[layer],
                   k2_events=None if k2 is None else k2[layer])

    def warm_up():
        one_step(0)  # protocol warmup (raw) step
        for s in range(a.warmup):
            one_step((s + 1) % 2)
        barrier(world)

    warm_up()

    def tev():
        # external: recorded as event nodes inside a CUDA-graph capture, so they time
        # the kernels of every replay
        return torch.cuda.Event(enable_timing=True, external=True)

    k1ev = [[(tev(), tev()) for _ in range(L)] for _ in range(2)]
    k2ev = [[(tev(), tev()) for _ in range(L)] for _ in range(2)]
    graphs = None
    if not a.no_graph:
        def capture(fn):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
                if os.environ.get("CC_BENCH_FAIL_CAPTURE"):  # exercises the eager fallback
                    raise RuntimeError("forced capture failure")
                torch.cuda.current_stream().wait_stream(streams.decode)
            return g

        try:
            graphs = {"main": [capture(lambda p=p: one_step(p)) for p in (0, 1)],
                      "timed": [capture(lambda p=p: one_step(p, k1=k1ev[p], k2=k2ev[p])) for p in (0, 1)]}
            if world > 1:
                graphs["nocomm"] = [capture(lambda p=p: one_step(p, skip_comm=True)) for p in (0, 1)]
            for e in exs:
                e.after_capture()
            for gs in graphs.values():
                for g in gs:
                    g.replay()
            barrier(world)
        except Exception as exc:  # e.g. a collective that cannot be captured: measure eagerly
            import traceback
            traceback.print_exc()
            print(f"bench: CUDA-graph capture failed ({type(exc).__name__}: {exc}); timing eager launches",
                  file=sys.stderr, flush=True)
            graphs = None
            torch.cuda.synchronize()
            streams = make_exchanges()  # host step counters advanced inside the failed capture
            warm_up()

    if graphs is None:  # eager timing: plain events (external ones only time graph replays)
        k1ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
                for _ in range(2)]
        k2ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]
                for _ in range(2)]

    def run(kind, steps):
        for s in range(steps):
            if graphs is not None:
                graphs[kind][s % 2].replay()
            elif kind == "main":
                one_step(s % 2)
            elif kind == "nocomm":
                one_step(s % 2, skip_comm=True)
            else:
                one_step(s % 2, k1=k1ev[s % 2], k2=k2ev[s % 2])

    K = a.steps
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier(world)
        start.record(streams.compute)
        run("main", K)
        streams.compute.wait_stream(streams.decode)
        end.record(streams.compute)
        barrier(world)
    ms = max_over_ranks(start.elapsed_time(end) / K, world)
    # kernels launched inside the timed region: one captured step's launches per replay
    n1 = lib.cc_launch_count()
    one_step(0)
    barrier(world)
    launches = (lib.cc_launch_count() - n1) * K

    # per-kernel durations, two ways:
    #  (a) events recorded inside the replayed graph around every K1 / K2 (the event
    #      nodes serialise the graph, so these include node-launch gaps: an upper bound)
    #  (b) graphs of the L layers' K1 launches alone / K2 launches alone on private
    #      state copies, replayed back to back: K1 / K2 as they run in a graph step
    k1s, k2s = [], []
    for s in range(K):
        if graphs is None:
            one_step(s % 2, k1=k1ev[s % 2], k2=k2ev[s % 2])
        else:
            graphs["timed"][s % 2].replay()
        torch.cuda.synchronize()
        k1s += [b.elapsed_time(e) for b, e in k1ev[s % 2]]
        k2s += [b.elapsed_time(e) for b, e in k2ev[s % 2]]
    k1_ev_ms, k2_ev_ms = statistics.mean(k1s), statistics.mean(k2s)
    k1_ms, k2_ms = kernel_graph_times(exs, inputs, spec, K) if (world == 1 and graphs is not None) else (None, None)
    if k1_ms is None:
        k1_ms, k2_ms = k1_ev_ms, k2_ev_ms
    barrier(world)

    act_bytes = L * 2 * rows * cols
    value = world * act_bytes / (ms / 1e3) / 1e9

    exposed_us = bf16_ag = comp_ag = None
    if world > 1:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        t0.record(streams.compute)
        run("nocomm", K)
        streams.compute.wait_stream(streams.decode)
        t1.record(streams.compute)
        barrier(world)
        ms_nc = max_over_ranks(t0.elapsed_time(t1) / K, world)
        exposed_us = max(0.0, (ms - ms_nc)) * 1e3 / L
        bf16_ag = allgather_us(n_own * cols * 2, world, L, K)
        comp_ag = allgather_us(exs[0].wire_bytes(False, False), world, L, K)

    bits = BITS[a.codec]
    s_own = n_own * cols
    k1_bytes = s_own * (18 + bits / 8) + 4 * (n_own + cols)
    n_peer_elems = (rows - n_own) * cols if world > 1 else rows * cols
    k2_bytes = n_peer_elems * (8 + bits / 8)
    path_bytes = k1_bytes + k2_bytes
    peaks = json.load(open(MEASURED)) if os.path.exists(MEASURED) else {}
    peak = peaks.get("hbm_gbs", 7672.0)
    k1_gbs = k1_bytes / (k1_ms / 1e3) / 1e9
    traffic = None
    if os.path.exists(TRAFFIC):
        tr = json.load(open(TRAFFIC))
        traffic = tr.get(f"{a.codec}_{world}")

    consistency = check_consistency(exs, inputs, world)
    e2e = None if a.no_e2e else measure_e2e(exs, inputs, streams, world, K, L, rows, cols)
    used_graph = graphs is not None
    sim = None
    if world == 1 and not a.no_sim:
        del graphs
        sim = {f"patch{P}": sim_rank_measure("patch", P, "quant2bit", L, rows, cols) for P in (2, 4, 8)}
        sim["ulysses8"] = sim_rank_measure("ulysses", 8, "sign1bit", L, rows, cols)
        sim["topk1pct_patch8"] = sim_rank_measure("patch", 8, "topk", L, rows, cols, spec_kw={"keep_fraction": 0.01})
        sim["topk10pct_patch8"] = sim_rank_measure("patch", 8, "topk", L, rows, cols, spec_kw={"keep_fraction": 0.1})
        sim["lowrank_r8_patch4"] = sim_rank_measure("patch", 4, "lowrank", 8, rows, cols, steps=5, warmup=3,
                                                    spec_kw={"rank": 8, "iterations": 2})
    cpu = None
    if not a.no_cpu and rank == 0:
        procs = a.cpu_procs or min(os.cpu_count() or 1, 16)
        cp = CpuPath(procs)
        try:
            v, wall = cp.measure(rows, cols, world, a.codec)
        finally:
            cp.close()
        cpu = {"value": v, "unit": "GB/s", "cores": procs, "kind": cp.impl,
               "sample": cp.describe(rows, cols, world, a.codec, wall)}
    barrier(world)

    line = {
        "metric": METRIC,
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic FLUX-like activations (log-normal token x channel scales, 10% step drift)",
        "config": bench_config(a, world),
        "value_is": "aggregate over ranks: every rank reconstructs the full activation per layer (per_gpu_gbs x n_gpus)",
        "per_gpu_gbs": value / world,
        "exposed_comm_us_per_layer": exposed_us,
        "bf16_allgather_us_per_layer": bf16_ag,
        "compressed_allgather_us_per_layer": comp_ag,
        "run": {"overlap": overlap, "cuda_graph": used_graph},
        "kernels": {"k1_encode_ms": k1_ms, "k1_gbs": k1_gbs, "k2_decode_ms": k2_ms,
                    "k2_gbs": k2_bytes / (k2_ms / 1e3) / 1e9, "k2_frac": k2_bytes / (k2_ms / 1e3) / 1e9 / peak,
                    "k1_in_step_events_ms": k1_ev_ms, "k2_in_step_events_ms": k2_ev_ms,
                    "timing": "k1/k2_*_ms: graphs of the L layers' K1 (resp. K2) launches alone on private "
                              "state copies, replayed back to back (events around the replay, / L); "
                              "*_in_step_events_ms: events recorded around every K1 / K2 inside the "
                              "replayed step graph (event nodes add node-launch gaps: upper bounds)",
                    "path_ideal_ms_per_layer": path_bytes / (peak * 1e9) * 1e3,
                    "path_frac": (path_bytes / (peak * 1e9) * 1e3) / (ms / L)},
        "roofline": {"bound": "hbm", "achieved": k1_gbs, "peak": peak, "unit": "GB/s", "frac": k1_gbs / peak,
                     "traffic": traffic, "kernel": "K1 encode_step (k1_resident: residual -> scales -> quantize/pack -> state update, one "
                               "persistent launch, residual kept on chip)",
                     "algorithmic_bytes_per_launch": k1_bytes, "peak_source": "MEASURED_PEAKS.json hbm_gbs"
                     if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "consistency": consistency,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "per_rank_sim": sim,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def kernel_graph_times(exs, inputs, spec, K):
    """K1 alone and K2 alone as they run in a CUDA-graph step: the L layers' encode_step
    launches (resp. loopback decodes) captured into one graph on PRIVATE copies of the
    layers' state (the benchmarked exchanges are not advanced), replayed K times
    back to back; ms per launch.  World size 1 only (the loopback receiver)."""
    import torch

    from paper_2507_17511_b200 import pipeline as pl

    L = len(exs)
    rows, cols = exs[0].rows, exs[0].cols
    sts = []
    for e in exs:  # private sender state at the exchange's current step
        st = pl.LayerState.__new__(pl.LayerState)
        st.mode, st.warmup_steps, st.step = e.sender.mode, e.sender.warmup_steps, e.sender.step
        st.base, st.feedback = e.sender.base.clone(), e.sender.feedback.clone()
        st.ref = None if e.sender.ref is None else e.sender.ref.clone()
        st._rec = None
        sts.append(st)
    bodies = [torch.empty_like(e.sendbuf) for e in exs]
    bases = [e.loop_base.clone() for e in exs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        nb = [0] * L
        for i in range(L):  # one eager step each: workspaces exist before the capture
            p, _ = pl.encode_step(sts[i], inputs[i][i % 2], spec, body_out=bodies[i])
            nb[i] = p.body.numel()
        g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=s):
            for i in range(L):
                pl.encode_step(sts[i], inputs[i][i % 2], spec, body_out=bodies[i])
        with torch.cuda.graph(g2, stream=s):
            for i in range(L):
                exs[i].engine.decode(spec, False, False, 1, [rows], cols, [bodies[i][:nb[i]]], [bases[i]])
        out = []
        for g in (g1, g2):
            g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(K):
                g.replay()
            b.record(s)
            b.synchronize()
            out.append(a.elapsed_time(b) / (K * L))
    torch.cuda.current_stream().wait_stream(s)
    del g1, g2, sts, bodies, bases
    return out[0], out[1]


def check_consistency(exs, inputs, world):
    """Outside the timed region: two more eager steps; every rank's blake2b digest
    of the full reconstruction must agree (mesh.py:237, 320-324), and at world 1 the
    loopback receiver must mirror the sender bit for bit (pipeline.py:193-194)."""
    import torch
    import torch.distributed as dist

    L = len(exs)
    layers = sorted({0, L // 2, L - 1})
    agree, checks = True, 0
    for s in range(2):
        for layer, e in enumerate(exs):
            e.step(inputs[layer][s])
        torch.cuda.synchronize()
        digs = [exs[i].digest() for i in layers]
        if world > 1:
            allv = [None] * world
            dist.all_gather_object(allv, digs)
            agree &= all(v == allv[0] for v in allv)
        else:
            agree &= all(torch.equal(exs[i].loop_base, exs[i].sender.base) for i in layers)
        checks += len(layers)
    return {"digests_agree" if world > 1 else "receiver_mirrors_sender": bool(agree), "layer_steps_checked": checks}


def allgather_us(nbytes, world, L, K):
    """µs per layer of L back-to-back NCCL all-gathers of `nbytes` per rank,
    replayed from a CUDA graph (the bf16 baseline the compression replaces, or the
    compressed bodies alone)."""
    import torch
    import torch.distributed as dist

    src = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty(world * nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        dist.all_gather_into_tensor(dst, src)
    barrier(world)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(L):
            dist.all_gather_into_tensor(dst, src)
    g.replay()
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(K):
        g.replay()
    t1.record()
    barrier(world)
    return max_over_ranks(t0.elapsed_time(t1) * 1e3 / (K * L), world)


def measure_e2e(exs, inputs, streams, world, K, L, rows, cols):
    """Public API with HOST buffers: H2D of each layer's bf16 shard from pinned
    memory, exchange step, D2H of the packed body and the StepRecord."""
    import torch

    host_in = [[x.cpu().pin_memory() for x in inp] for inp in inputs]
    dev_in = [torch.empty_like(inp[0]) for inp in inputs]
    body_n = [e.sendbuf.numel() for e in exs]
    host_body = [torch.empty(n, dtype=torch.uint8).pin_memory() for n in body_n]
    host_rec = [torch.empty(2, dtype=torch.float64).pin_memory() for _ in exs]
    copy = torch.cuda.Stream(exs[0].device)
    h2d = d2h = 0
    ev_in = [torch.cuda.Event() for _ in exs]

    def step(s):
        nonlocal h2d, d2h
        h2d = d2h = 0
        for layer, e in enumerate(exs):
            with torch.cuda.stream(copy):
                copy.wait_stream(streams.compute)  # previous user of dev_in finished (K1 read it)
                dev_in[layer].copy_(host_in[layer][s % 2], non_blocking=True)
                ev_in[layer].record(copy)
            streams.compute.wait_event(ev_in[layer])
            e.step(dev_in[layer])
            nb = e.last_nbytes
            with torch.cuda.stream(streams.compute):
                host_body[layer][:nb].copy_(e.sendbuf[:nb], non_blocking=True)
                host_rec[layer].copy_(e.last_record._dev, non_blocking=True)
            h2d += dev_in[layer].numel() * 2
            d2h += nb + 16
        streams.compute.wait_stream(streams.decode)

    for s in range(2):
        step(s)
    barrier(world)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(streams.compute)
    for s in range(K):
        step(s)
    t1.record(streams.compute)
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1) / K, world)
    value = world * L * 2 * rows * cols / (ms / 1e3) / 1e9
    return {"value": value, "unit": "GB/s", "ms_per_step": ms, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h}


def sim_rank_measure(kind, P, codec, L, rows, cols, steps=5, warmup=3, spec_kw=None, graph=True):
    """One rank of a P-rank job on this single GPU (exchange `sim_world=(P, 0)`): K1 on
    the rank's shard (patch: [rows/P, cols]; Ulysses: P chunks [rows/P, cols/P]), the
    collective replaced by device copies of the rank's bodies into the receive slots,
    K2 over the P-1 peer slots (patch) / P chunks (Ulysses).  Returns ms per layer and
    per-GPU activation GB/s — the per-rank compute + landing-copy cost of configs 2-3,
    without NVLink transfer time.  CUDA-graph replay, 57 layer channels."""
    import torch

    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import linalg as la
    from paper_2507_17511_b200.comm import PatchParallelExchange, UlyssesAllToAll, shard_bounds

    dev = torch.device("cuda", torch.cuda.current_device())
    spec = cx.CompressorSpec(cx.CompressorKind(codec), **(spec_kw or {}))
    lowrank = spec.kind == cx.CompressorKind.LOWRANK
    n = rows // P
    if kind == "patch":
        exs = [PatchParallelExchange(rows, cols, spec, sim_world=(P, 0)) for _ in range(L)]
        lo, hi = shard_bounds(rows, P)[0]
    else:
        exs = [UlyssesAllToAll(n, cols, spec, sim_world=(P, 0)) for _ in range(L)]
        lo, hi = 0, n
    streams = exs[0].streams
    for e in exs[1:]:
        e.streams = streams
    inputs = [flux_inputs(rows, cols, lo, hi, layer, dev) for layer in range(L)]

    # low-rank: every layer channel draws its start block (cx:407) on the device from
    # the mesh key spawn_rng(seed, 6, rank, t) (mesh.py:193) with t advanced on the
    # device (linalg.DeviceKey), so the step is captured and replayed like the others
    keys = [la.DeviceKey(1000 * layer, 6, 0, 2, advance=True) for layer in range(L)] if lowrank else None

    def one_step(s):
        for layer, e in enumerate(exs):
            e.step(inputs[layer][s % 2], rng=keys[layer] if lowrank else None)

    for s in range(warmup + 1):
        one_step(s)
    torch.cuda.synchronize()
    graphs = []
    if graph:
        for par in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                one_step(par)
                torch.cuda.current_stream().wait_stream(streams.decode)
            graphs.append(g)
        for e in exs:
            if hasattr(e, "after_capture"):
                e.after_capture()
        for par in (0, 1):
            graphs[par].replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(steps):
        if graph:
            graphs[s % 2].replay()
        else:
            one_step(warmup + 1 + s)
    torch.cuda.current_stream().wait_stream(streams.decode)
    t1.record()
    torch.cuda.synchronize()
    ms_layer = t0.elapsed_time(t1) / steps / L
    out = {"ms_per_layer": round(ms_layer, 5), "gbs_per_gpu": round(2 * rows * cols / (ms_layer / 1e3) / 1e9, 1),
           "codec": spec.label() if hasattr(spec, "label") else codec, "shard": [n, cols if kind == "patch" else cols // P],
           "cuda_graph": graph}
    del exs, inputs, graphs
    torch.cuda.empty_cache()
    return out


def main():
    a = parse()
    if a.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(a, world, rank)
        return 0
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a)
    world, rank = dist_setup()
    if world != a.gpus:
        print(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}; measuring {world} ranks", file=sys.stderr, flush=True)
    run_b200(a, world, rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
