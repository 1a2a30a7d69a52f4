#!/usr/bin/env python3
"""Benchmark of the B200 fast-summation graph-Laplacian matvec.

Metric (BASELINE.json): fp64 Laplacian matvecs/s (+ Lanczos time-to-k and the
roofline fraction of the dominant kernel).  One step = one application of
L_s = I - D^-1/2 W D^-1/2 to a block of `nvec` seeded N(0,1) vectors on the
BASELINE configuration's synthetic point set.  Default workload: config 5
(`configs[4]`, the largest single-GPU configuration: a block of 16 vectors at
n = 10M points in 3-D, N = 64, m = 8); configs 1-4 are reported under
"also" with their Lanczos time-to-k (k = 10 / 10 / 4 / 20).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--weak]
                  [--impl b200|reference] [--emulate N]

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun environment
re-launches itself under `torch.distributed.run` with N ranks.  Points are
sharded by the internal spatial order, each rank spreads its slice, and one
NCCL allreduce per apply sums the truncated spectra (strong scaling at fixed n;
`--weak`: config 5 at 1.25M points per GPU).  Whole-job matvecs/s = the
vectors all ranks applied / the max over ranks of the device time.

`--impl reference`: the reference's own CPU implementation of the path
(/root/reference/proj compiled unchanged against shim headers, oracle/_ref;
else the oracle restatement), serial as the reference is, on rank 0 only.
The reference arm never loads the product library: its inputs come from the
same seeded generator linked into oracle/liboracle.so.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 2024
VEC_SEED = 99
STAGES = ("spread", "assemble", "fft_r2c", "multiply", "fft_c2r", "interp")
WEAK_PER_GPU = 1_250_000
METRIC = "fp64 Laplacian matvecs/sec"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--weak", action="store_true", help="config 5 at 1.25M points per GPU (weak scaling)")
    p.add_argument("--nvec", type=int, default=0, help="vectors per step (0: 16 for config 5, else 1)")
    p.add_argument("--no-lanczos", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0)
    p.add_argument("--also", default="1,2,3,4", help="comma list of extra configs measured after the main line "
                   "(device matvecs/s + Lanczos time-to-k), '' to skip")
    p.add_argument("--emulate", type=int, default=0,
                   help="single GPU: time the N-rank sharded path as an emulated shard group (per-rank compute "
                        "measured, NVLink allreduce modelled) and print a projected N-GPU line")
    p.add_argument("--force-sharded", action="store_true",
                   help=argparse.SUPPRESS)  # run the sharded (NCCL) path even at world size 1 (under torchrun)
    return p.parse_args()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N` outside torchrun: re-run this script with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def workload(args, world):
    """(config dict shared by both arms, n, nvec, info) -- from the oracle
    library's copy of the generator (no product import)."""
    from oracle import oracle as orc
    info = orc.workload_info(args.config)
    n = info["n"]
    if args.weak:
        if args.config != 5:
            raise SystemExit("--weak is defined for config 5 (1.25M points per GPU)")
        n = WEAK_PER_GPU * world
    nvec = args.nvec or (16 if args.config == 5 else 1)
    cfg = {"workload": f"config{args.config}", "n": n, "d": info["d"], "sigma": info["sigma"], "N": info["N"],
           "m": info["m"], "p": info["p"], "nvec": nvec, "op": "L_s x"}
    return cfg, n, nvec, info


def nodes_for(args, n):
    from oracle import oracle as orc
    return orc.workload_nodes(args.config, SEED, n=n if args.weak else 0)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---- clocks sampling (B200_PROFILING.md clocks line) ---------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self, t0, t1):
        win = [s for (t, s) in self.samples if t0 - 0.06 <= t <= t1 + 0.06] or [s for (_, s) in self.samples]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in win if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in win for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(win[0][1]) if win[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(win)}


# ---- algorithmic work of one spread / interpolation launch ----------------
def stage_work(geom, n, nvec):
    """Algorithmic bytes and flops per launch.

    flops: 2 n (2m)^d per vector and pass (window evaluation precomputed).
    bytes: the per-point inputs the pass must read -- coordinates-equivalent
    taps are not counted (§8d counts coordinates, 8 d bytes per point), x and
    s per vector (spread), x, s and y (interp) -- plus one grid write (spread)
    or read (interp) of M^d doubles per vector.
    """
    d, T, M = geom["d"], geom["taps"], geom["M"]
    flops = 2.0 * n * T ** d * nvec
    coords = 8.0 * n * d
    grid = 8.0 * M ** d
    spread_b = coords + nvec * (16.0 * n + grid)
    interp_b = coords + nvec * (24.0 * n + grid)
    return {"spread": (spread_b, flops), "interp": (interp_b, flops)}


# ---- the reference's CPU path (oracle/_ref if built, else the restatement) --
def cpu_backend():
    """(module, kind): oracle/_ref = the reference's own nfft/kernels/fastsum/
    graphop/spectral .cpp compiled unchanged against shim Eigen/FFTW headers
    (kind "reference"); without it the oracle restatement (kind "port")."""
    try:
        from oracle import ref as R
        if R.available():
            return R, "reference"
    except Exception:  # noqa: BLE001 - fall back to the restatement
        pass
    from oracle import oracle as orc
    return orc, "port"


class Pinned:
    """Run the serial CPU path pinned to one core."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.old)


def cpu_apply_seconds(X, info, budget_s):
    """Mean seconds of one L_s apply (one warm-up, then >= 2 timed applies,
    acceptance.cpp:400-404) and the setup seconds, on the serial CPU path."""
    R, _ = cpu_backend()
    t0 = time.perf_counter()
    op = R.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    setup = time.perf_counter() - t0
    x = np.random.default_rng(1).standard_normal(X.shape[0])
    op.apply_sym_laplacian(x)
    reps, t0 = 0, time.perf_counter()
    while True:
        op.apply_sym_laplacian(x)
        reps += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and reps >= 2) or reps >= 200:
            break
    return el / reps, setup, reps


def cpu_matvec_rate(config, X, info, budget_s):
    """matvecs/s of the serial CPU path on this workload.  Up to 400k points
    the full set is timed; beyond, two prefixes of the seeded point stream
    (n1, 2 n1 points: the same distribution) give t(n) = a + b n and the full
    size is extrapolated (a = the n-independent FFT/multiply part)."""
    _, kind = cpu_backend()
    n = X.shape[0]
    with Pinned() as pin:
        if n <= 400_000:
            t, setup, reps = cpu_apply_seconds(X, info, budget_s)
            desc = f"{reps} timed applies of L_s on all {n} points"
        else:
            n1 = 50_000 if (info["d"] == 3 and info["m"] >= 8) else 100_000
            t1, _, r1 = cpu_apply_seconds(X[:n1], info, budget_s / 2)
            t2, setup, r2 = cpu_apply_seconds(X[:2 * n1], info, budget_s / 2)
            b = (t2 - t1) / n1
            a = max(0.0, t1 - b * n1)
            t = a + b * n
            desc = (f"L_s applies timed on the first {n1} and {2 * n1} points of the same seeded stream "
                    f"({r1} / {r2} timed applies: {t1:.3f} s / {t2:.3f} s), t(n) = a + b n fitted and evaluated "
                    f"at n = {n} (a = {a:.4f} s, b = {b * 1e6:.3f} us/point)")
        core = pin.core
    return 1.0 / t, t, setup, f"{desc}; serial, pinned to core {core}", kind


def cpu_lanczos(config, budget_ok=True):
    """Lanczos time-to-k of the serial CPU path (commands.cpp:174-183 split:
    setup = plan + degrees, solve = lanczos_largest with Ritz vectors)."""
    from oracle import oracle as orc
    R, kind = cpu_backend()
    info = orc.workload_info(config)
    X = orc.workload_nodes(config, SEED)
    with Pinned() as pin:
        t0 = time.perf_counter()
        op = R.AdjacencyOperator(X, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
        setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        vals, _, iters, conv = op.lanczos_largest(info["k"], max_iter=1000, tol=1e-8, seed=1)
        solve = time.perf_counter() - t0
    return {"workload": f"config{config}", "n": X.shape[0], "k": info["k"], "tol": 1e-8, "setup_s": setup,
            "solve_s": solve, "total_s": setup + solve, "iterations": iters, "converged": bool(conv),
            "kind": kind, "cores": 1, "core": pin.core, "top_eig_A": [float(v) for v in vals[:3]]}


# ---- reference arm ---------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg, n, nvec, info = workload(args, world)
    X = nodes_for(args, n)
    # each timed "step" is the bounded CPU sample; its budget keeps the whole
    # --steps/--warmup run within a few minutes
    budget = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    rate, t, setup, desc, kind = cpu_matvec_rate(args.config, X, info, budget)
    value = rate
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "matvecs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * nvec * t, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded stand-in for the paper's datasets)", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "matvecs/s", "cores": 1, "kind": kind, "sample": desc,
                         "cpu": cpu_model(), "host_cores": os.cpu_count(), "setup_s": setup},
        "e2e": {"value": value, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- emulated N-rank path on one GPU (projection, not a measurement) -------
ALLREDUCE_BUSBW = 300e9   # B/s, conservative NCCL allreduce bus bandwidth on 8x B200 NVLink 5 / NVSwitch
ALLREDUCE_LAT = 20e-6     # s per allreduce (launch + ring/NVLS latency)


def run_emulated(args):
    """`--emulate N`: the sharded data path of N ranks as one ShardGroup on
    this GPU.  Every shard's two apply phases are timed with CUDA events (what
    rank r computes on its own GPU: its slice's spread / interpolation, its
    slab-pruned convolution, its assembly); the exchange is the window
    spectrum allreduce, modelled at ALLREDUCE_BUSBW.  Projected whole-job
    matvecs/s = nvec / (max over shards + modelled allreduce)."""
    import torch

    import paper_1808_04580_b200 as fgs
    world = args.emulate
    cfg, n, nvec, info = workload(args, world)
    X = nodes_for(args, n)
    params = fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0)
    kern = fgs.KernelSpec.gaussian(info["sigma"])
    t0 = time.perf_counter()
    grp = fgs.ShardGroup(X, kern, params, world=world)
    setup_s = time.perf_counter() - t0
    x = torch.from_numpy(np.ascontiguousarray(fgs.workload_vectors(n, nvec, VEC_SEED).T)).cuda()
    y = torch.empty_like(x)
    grp.profile(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, ld=n, reps=max(1, args.warmup))
    shard_ms, ex_ms = grp.profile(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, ld=n,
                                  reps=max(1, args.steps))
    N, M, d = info["N"], 2 * info["N"], info["d"]
    if d == 3:
        nw = N if M == N else N + 1
        ex_bytes = nw * nw * (N // 2 + 1) * 16 * nvec
    elif d == 2:
        ex_bytes = M * M * 8 * nvec
    else:
        ex_bytes = (N // 2 + 1) * 16 * nvec
    ar_ms = 1e3 * (ALLREDUCE_LAT + 2.0 * (world - 1) / world * ex_bytes / ALLREDUCE_BUSBW) if world > 1 else 0.0
    step_ms = float(np.max(shard_ms)) + ar_ms
    stats = [grp.stats(r) for r in range(world)]
    line = {
        "metric": METRIC, "mode": "emulated shard group on 1 GPU (projection, not a measured N-GPU run)",
        "projected_value": nvec / (step_ms * 1e-3), "unit": "matvecs/s", "n_gpus_projected": world,
        "scaling": "weak" if args.weak else "strong", "dtype": "f64", "config": cfg,
        "shard_ms": [float(v) for v in shard_ms], "max_shard_ms": float(np.max(shard_ms)),
        "mean_shard_ms": float(np.mean(shard_ms)), "allreduce_bytes": ex_bytes,
        "allreduce_ms_model": ar_ms, "allreduce_model": f"{ALLREDUCE_LAT * 1e6:.0f} us + 2(N-1)/N bytes / "
                                                         f"{ALLREDUCE_BUSBW / 1e9:.0f} GB/s",
        "device_sum_exchange_ms": ex_ms, "conv_planes": [s["conv_planes"] for s in stats],
        "n_local": [s["n_local"] for s in stats], "setup_s": setup_s,
    }
    print(json.dumps(line), flush=True)


# ---- B200 arm --------------------------------------------------------------
def lanczos_timing(op, info, warm=2):
    """Lanczos time-to-k as the reference's eigs command splits it
    (commands.cpp:174-183): `solve_s` is the first solve on a fresh handle
    (workspace allocation and graph capture included, what a one-shot run
    pays); `solve_s_warm` the median of `warm` further solves on the same
    handle.  Ritz vectors are formed and copied to the host every time
    (single device; sharded runs return the eigenvalues)."""
    import torch

    import paper_1808_04580_b200 as fgs
    times, li, pairs, phases = [], None, None, None
    for _ in range(1 + warm):
        li = fgs.LanczosInfo()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li,
                                    want_vectors=op.world == 1)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        phases = op.lanczos_stats()
    rec = {"k": info["k"], "tol": 1e-8, "solve_s": times[0],
           "solve_s_warm": float(np.median(times[1:])) if warm else None,
           "iterations": li.iterations, "converged": li.converged, "phases": phases,
           "top_eig_A": [float(v) for v in pairs.values[:3]]}
    return rec


def fresh_nccl_id(dist):
    """A new NCCL unique id from rank 0 for every sharded handle: an id
    bootstraps exactly one communicator (its root exits with it)."""
    import paper_1808_04580_b200 as fgs
    nid = [fgs.nccl_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(nid, src=0)
    return nid[0]


def make_op(X, info, dev, rank, world, nccl_id, sharded):
    import paper_1808_04580_b200 as fgs
    params = fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0)
    kernel = fgs.KernelSpec.gaussian(info["sigma"])
    if sharded:
        return fgs.AdjacencyOperator(X, kernel, params, device=dev, rank=rank, world=world, nccl_id=nccl_id)
    return fgs.AdjacencyOperator(X, kernel, params, device=dev)


def device_inputs(op, n, nvec, dev):
    """This rank's slice of the seeded vectors in the internal order."""
    import torch

    import paper_1808_04580_b200 as fgs
    xs_host = fgs.workload_vectors(n, nvec, VEC_SEED)
    xs_host = xs_host if xs_host.ndim == 2 else xs_host[:, None]
    nl = op.n_local
    x_int = torch.empty((nvec, nl), dtype=torch.float64, device=f"cuda:{dev}")
    for v in range(nvec):  # caller order -> this rank's slice of the internal order
        xc = torch.from_numpy(np.ascontiguousarray(xs_host[:, v])).to(f"cuda:{dev}")
        op.permute_device(xc.data_ptr(), x_int[v].data_ptr(), nvec=1, ld=n, direction=0)
    return xs_host, x_int


def secondary(cfg_id, steps, dev, rank, world, nccl_id, sharded, dist):
    """Device matvecs/s and Lanczos time-to-k of another BASELINE config on
    the same GPU(s) (graph replays, L2 flushed between steps)."""
    import torch

    import paper_1808_04580_b200 as fgs
    from oracle import oracle as orc
    info = orc.workload_info(cfg_id)
    nvec = 16 if cfg_id == 5 else 1
    X = orc.workload_nodes(cfg_id, SEED)
    n = X.shape[0]
    t0 = time.perf_counter()
    op = make_op(X, info, dev, rank, world, fresh_nccl_id(dist) if sharded else None, sharded)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    op.set_stream(stream.cuda_stream)
    _, xi = device_inputs(op, n, nvec, dev)
    yi = torch.empty_like(xi)
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def step():
        op.apply_device(fgs.OP_SYM_LAPLACIAN, xi.data_ptr(), yi.data_ptr(), nvec=nvec, ld=op.n_local,
                        internal_order=True)

    for _ in range(3):
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    for s0, s1 in ev:
        flush.zero_()
        s0.record(stream)
        step()
        s1.record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"workload": f"config{cfg_id}", "n": n, "d": info["d"], "N": info["N"], "m": info["m"], "nvec": nvec,
           "value": nvec / (ms / 1000.0), "unit": "matvecs/s", "ms_per_step": ms, "setup_s": setup_s}
    if cfg_id <= 4:
        out["lanczos"] = {"setup_s": setup_s, **lanczos_timing(op, info)}
    return out


def run_b200(args, rank, world, local_rank):
    import torch

    import paper_1808_04580_b200 as fgs
    dev = local_rank
    torch.cuda.set_device(dev)
    # the fp64 roofline denominator, measured before the workload heats the
    # part: the larger of the DFMA and DMMA microbenchmarks, best of three
    # (MEASURED_PEAKS.json carries no fp64 figure)
    fp64_tf = max(max(fgs.measure_fp64_peak(dev), fgs.measure_dmma_peak(dev)) for _ in range(3))
    cfg, n, nvec, info = workload(args, world)
    X = nodes_for(args, n)

    sharded = world > 1 or args.force_sharded
    dist, nccl_id = None, None
    if sharded:
        import torch.distributed as dist
        nccl_id = fresh_nccl_id(dist)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = make_op(X, info, dev, rank, world, nccl_id, sharded)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=dev)  # non-default: applies replay captured CUDA graphs
    torch.cuda.set_stream(stream)
    op.set_stream(stream.cuda_stream)
    nl = op.n_local
    geom = op.geometry()
    xs_host, x_int = device_inputs(op, n, nvec, dev)
    y_int = torch.empty_like(x_int)
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=f"cuda:{dev}")  # > 126 MB L2

    def step():
        op.apply_device(fgs.OP_SYM_LAPLACIAN, x_int.data_ptr(), y_int.data_ptr(), nvec=nvec, ld=nl,
                        internal_order=True)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = op.launch_count()
    clocks = ClockSampler(dev)
    clocks.start()
    time.sleep(0.15)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    w0 = time.time()
    for s, e in ev:
        flush.zero_()  # L2 flush between timed iterations (outside the events)
        s.record(stream)
        step()
        e.record(stream)
    torch.cuda.synchronize()
    w1 = time.time()
    if dist:
        dist.barrier()
    launches = op.launch_count() - launches0
    # per-kernel durations: K more steps with stage events between the
    # launches (direct launches on the same stream; CUDA events on the
    # launching stream)
    op.profile(True)
    for _ in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    op.profile(False)
    stage_ms, napp = op.profile_read()
    time.sleep(0.1)
    clocks.stop()
    total_ms = sum(s.elapsed_time(e) for s, e in ev)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = nvec * args.steps / (total_ms / 1000.0)

    # ---- roofline of the dominant kernel (per-launch averages) --------------
    peaks, peak_src = measured_peaks()
    per_launch = {k: stage_ms[i] / max(1, napp) for i, k in enumerate(STAGES)}
    work = stage_work(geom, nl, nvec)
    dom = max(("spread", "interp"), key=lambda k: per_launch[k])
    b, f = work[dom]
    t = per_launch[dom] * 1e-3
    t_hbm = b / (peaks["hbm_gbs"] * 1e9)
    t_fp = f / (fp64_tf * 1e12)
    if t_fp >= t_hbm:
        roof = {"bound": "tensor", "achieved": f / t / 1e12, "peak": fp64_tf, "unit": "TFLOP/s",
                "frac": (f / t / 1e12) / fp64_tf, "traffic": None, "pipe": "fp64 tensor cores (DMMA m8n8k4)",
                "peak_source": "fp64 microbenchmarks on this B200 before the run: max(DFMA, DMMA m8n8k4), best of 3 "
                               "(MEASURED_PEAKS.json has no fp64 entry; its bf16 figure does not apply to an fp64 "
                               "kernel)"}
    else:
        roof = {"bound": "hbm", "achieved": b / t / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": (b / t / 1e9) / peaks["hbm_gbs"], "traffic": None,
                "peak_source": f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json)"}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(f"config{args.config}", {}).get(dom)
        if tr and not args.weak and world == 1:
            roof["traffic"] = tr["dram_bytes"]
            roof["traffic_source"] = f"ncu --set full, {tr['source']} ({tr['kernel']}), dram read+write per launch"
    except (OSError, ValueError):
        pass
    step_flops = 2 * work["spread"][1]
    roof.update({"kernel": dom, "launch_ms": per_launch[dom], "algorithmic_bytes": b, "algorithmic_flops": f,
                 "t_roof_ms": 1e3 * max(t_hbm, t_fp), "stage_ms_per_step": {k: per_launch[k] for k in STAGES},
                 "step_fp64_frac": step_flops / (ms_per_step * 1e-3) / (fp64_tf * 1e12)})

    # ---- end to end through the public API with pinned host buffers ---------
    e2e = None
    if not args.no_e2e:
        if not sharded:
            import ctypes as C
            hx = torch.from_numpy(np.asfortranarray(xs_host).T.copy()).pin_memory()  # [nvec][n] = column-major
            hy = torch.empty_like(hx).pin_memory()
            L = fgs.lib()
            xp = C.cast(hx.data_ptr(), C.POINTER(C.c_double))
            yp = C.cast(hy.data_ptr(), C.POINTER(C.c_double))
            for _ in range(2):
                L.fgs_adjacency_apply(op.handle, fgs.OP_SYM_LAPLACIAN, xp, yp, nvec, C.c_int64(n))
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(args.steps):
                st = L.fgs_adjacency_apply(op.handle, fgs.OP_SYM_LAPLACIAN, xp, yp, nvec, C.c_int64(n))
                assert st == 0, L.fgs_last_error()
            s1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = s0.elapsed_time(s1) / args.steps
            path = "fgs_adjacency_apply (C ABI) with pinned host x/y in caller order"
        else:
            # sharded handles take device vectors in the internal order (the
            # public multi-GPU API, fgs_adjacency_apply_device): each rank
            # streams its slice vector by vector -- H2D on one stream, the
            # apply on the handle's stream, D2H on a third, ping-pong device
            # buffers (two cached apply graphs) -- so copies overlap applies
            hx = x_int.cpu().pin_memory()
            hy = torch.empty_like(hx).pin_memory()
            xb = [torch.empty(nl, dtype=torch.float64, device=f"cuda:{dev}") for _ in range(2)]
            yb = [torch.empty(nl, dtype=torch.float64, device=f"cuda:{dev}") for _ in range(2)]
            s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
            ev_in = [torch.cuda.Event() for _ in range(nvec)]
            ev_ap = [torch.cuda.Event() for _ in range(nvec)]
            ev_out = [torch.cuda.Event() for _ in range(nvec)]

            def e2e_step():
                for v in range(nvec):
                    b = v & 1
                    if v >= 2:
                        s_in.wait_event(ev_ap[v - 2])  # xb[b] read by apply v - 2
                    with torch.cuda.stream(s_in):
                        xb[b].copy_(hx[v], non_blocking=True)
                    ev_in[v].record(s_in)
                    stream.wait_event(ev_in[v])
                    if v >= 2:
                        stream.wait_event(ev_out[v - 2])  # yb[b] downloaded
                    op.apply_device(fgs.OP_SYM_LAPLACIAN, xb[b].data_ptr(), yb[b].data_ptr(), nvec=1, ld=nl,
                                    internal_order=True)
                    ev_ap[v].record(stream)
                    s_out.wait_event(ev_ap[v])
                    with torch.cuda.stream(s_out):
                        hy[v].copy_(yb[b], non_blocking=True)
                    ev_out[v].record(s_out)
                stream.wait_event(ev_out[nvec - 1])
                stream.wait_event(ev_in[nvec - 1])

            for _ in range(2):
                e2e_step()
            torch.cuda.synchronize()
            dist.barrier()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(args.steps):
                e2e_step()
                stream.synchronize()
            s1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([s0.elapsed_time(s1) / args.steps], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
            path = ("per rank: pinned slice, vector-by-vector H2D / fgs_adjacency_apply_device (sharded, internal "
                    "order) / D2H on three streams; max over ranks")
        e2e = {"value": nvec / (e2e_ms / 1000.0), "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n * nvec,
               "d2h_bytes_per_step": 8 * n * nvec, "ms_per_step": e2e_ms, "path": path}
    del op
    torch.cuda.synchronize()

    # ---- secondary configurations with Lanczos time-to-k -------------------
    also = []
    if args.also:
        for c in [int(c) for c in args.also.split(",") if c.strip()]:
            if c == args.config and not args.weak:
                continue
            try:
                also.append(secondary(c, 10 if c != 5 else 2, dev, rank, world, nccl_id, sharded, dist))
            except Exception as ex:  # noqa: BLE001 - report, do not lose the main line
                also.append({"workload": f"config{c}", "error": str(ex)[:300]})
    lanczos = None
    if not args.no_lanczos and args.config <= 4 and not args.weak:
        try:
            op = make_op(X, info, dev, rank, world, fresh_nccl_id(dist) if sharded else None, sharded)
            op.set_stream(stream.cuda_stream)
            lanczos = {"setup_s": setup_s, **lanczos_timing(op, info)}
            lanczos["total_s"] = setup_s + lanczos["solve_s"]
            del op
        except Exception as ex:  # noqa: BLE001
            lanczos = {"error": str(ex)[:300]}

    # ---- CPU baseline (rank 0, N = 1): matvecs/s + Lanczos time-to-k ---------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, _, csetup, desc, kind = cpu_matvec_rate(args.config, X, info, args.cpu_seconds)
        cpu = {"value": rate, "unit": "matvecs/s", "cores": 1, "kind": kind, "sample": desc,
               "cpu": cpu_model(), "host_cores": os.cpu_count(), "setup_s": csetup}
        if not args.no_lanczos:
            cpu["lanczos"] = []
            for c in (1, 2):
                try:
                    cpu["lanczos"].append(cpu_lanczos(c))
                except Exception as ex:  # noqa: BLE001
                    cpu["lanczos"].append({"workload": f"config{c}", "error": str(ex)[:300]})

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "matvecs/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded stand-in for the paper's datasets)", "config": cfg,
            "parallelism": f"points sharded x{world} (NCCL)" if sharded else "single GPU",
            "l2": "flushed (256 MB write) between timed steps, outside the events",
            "vectors": ("value: device-resident block in the handle's internal (spatially sorted) order, the "
                        "order the Lanczos basis is kept in (fgs_adjacency_apply_device); e2e: host vectors in "
                        "the caller's order, permuted inside the handle"),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(w0, w1), "lanczos": lanczos, "setup_s": setup_s, "also": also,
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.emulate:
        run_emulated(args)
        return
    import torch
    import torch.distributed as dist
    distributed = world > 1 or args.force_sharded
    if distributed:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if distributed:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
