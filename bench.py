#!/usr/bin/env python3
"""Benchmark of the B200 fast-summation graph-Laplacian matvec.

Metric (BASELINE.json): fp64 Laplacian matvecs/s (+ Lanczos time-to-k and the
roofline fraction of the dominant kernel).  One step = one application of
L_s = I - D^-1/2 W D^-1/2 to a block of `nvec` seeded N(0,1) vectors (1 for
configs 1-4, 16 for config 5) on the BASELINE configuration's synthetic point
set.  Default workload: configs[1] (config 2, 100k points in 2-D).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

Multi-GPU: launched by torchrun, one process per GPU; points are sharded by
the internal spatial order and the truncated spectrum is summed with NCCL
(strong scaling, whole-job matvecs/s, max over ranks of device time).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 2024
STAGES = ("spread", "assemble", "fft_r2c", "multiply", "fft_c2r", "interp")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--nvec", type=int, default=0, help="vectors per step (0: 16 for config 5, else 1)")
    p.add_argument("--no-lanczos", action="store_true")
    p.add_argument("--force-sharded", action="store_true",
                   help=argparse.SUPPRESS)  # run the sharded (NCCL) path even at world size 1 (under torchrun)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--also", default="4", help="comma list of extra configs measured after the main line "
                   "(device matvecs/s + Lanczos time-to-k), '' to skip; N=1 only")
    return p.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ---- clocks sampling (B200_PROFILING.md clocks line) ---------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._proc = None
        self._t = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
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
def stage_work(geom, n, nvec, scaled_input=True):
    """bytes and flops the kernels must move / execute per launch.

    spread: taps n*d*T*8 (read once per block of vectors), x (+ s) per vector,
            item boxes written per vector; flops 2*n*T^d per vector.
    interp: taps, item boxes read, x, s, y per vector; flops 2*n*T^d per vector.
    """
    d, T = geom["d"], geom["taps"]
    taps = n * d * T * 8
    vec = n * 8
    box = geom["items"] * geom["box_stride"] * 8
    flops = 2.0 * n * T ** d * nvec
    spread_b = taps + nvec * (vec * (2 if scaled_input else 1) + box)
    interp_b = taps + nvec * (box + 3 * vec)
    return {"spread": (spread_b, flops), "interp": (interp_b, flops)}


# ---- CPU side: the oracle restatement (the reference is not buildable) ----
def cpu_matvecs_per_s(config, X, info, nvec, budget_s):
    """Serial oracle (kind "port") on the same nodes; bounded sample.  Returns
    (matvecs/s, sample description, setup seconds)."""
    from oracle import oracle as orc
    n = X.shape[0]
    sub = X
    scale = 1.0
    if n > 500_000:  # bounded sample: a point subsample, extrapolated linearly in n
        idx = np.random.default_rng(config).choice(n, 500_000 if info["d"] < 3 or info["m"] < 8 else 200_000,
                                                   replace=False)
        sub = X[np.sort(idx)]
        scale = sub.shape[0] / n
    t0 = time.perf_counter()
    ref = orc.AdjacencyOperator(sub, 0, info["sigma"], N=info["N"], m=info["m"], p=info["p"])
    setup = time.perf_counter() - t0
    x = np.random.default_rng(1).standard_normal(sub.shape[0])
    ref.apply_sym_laplacian(x)  # warm-up (acceptance.cpp:400-404)
    reps, t0 = 0, time.perf_counter()
    while True:
        ref.apply_sym_laplacian(x)
        reps += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and reps >= 2) or reps >= 500:
            break
    per = el / reps
    rate = scale / per
    desc = (f"serial oracle port, {reps} matvecs of L_s on {sub.shape[0]} points"
            + (f" (random subsample of {n}, throughput scaled by n_sample/n)" if scale < 1 else "")
            + f", 1 thread, config {config}")
    return rate, desc, setup


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---- reference arm ---------------------------------------------------------
def run_reference(args, rank, world):
    import paper_1808_04580_b200 as fgs
    if rank != 0:
        return
    info = fgs.workload_info(args.config)
    nvec = args.nvec or (16 if args.config == 5 else 1)
    X = fgs.workload_nodes(args.config, SEED)
    from oracle import oracle as orc
    n = X.shape[0]
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    rate, desc, setup = cpu_matvecs_per_s(args.config, X, info, nvec, budget)
    value = rate * 1.0
    line = {
        "impl": "reference", "metric": "fp64 Laplacian matvecs/sec", "value": value, "unit": "matvecs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * nvec / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded stand-in for the paper's datasets)",
        "config": {"workload": f"config{args.config}", "n": n, "d": info["d"], "sigma": info["sigma"],
                   "N": info["N"], "m": info["m"], "p": info["p"], "nvec": nvec},
        "cpu_baseline": {"value": value, "unit": "matvecs/s", "cores": 1, "kind": "port",
                         "sample": desc + "; reference C++ is not buildable here (Eigen3/FFTW3 absent)",
                         "cpu": cpu_model(), "host_cores": os.cpu_count(), "setup_s": setup},
        "e2e": {"value": value, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- secondary configurations (reported under "also") ----------------------
def secondary(cfg, steps, dev):
    """Device matvecs/s and Lanczos time-to-k of another BASELINE config on
    the same GPU (graph replays, L2 flushed between steps)."""
    import torch
    import paper_1808_04580_b200 as fgs
    info = fgs.workload_info(cfg)
    nvec = 16 if cfg == 5 else 1
    X = fgs.workload_nodes(cfg, SEED)
    n = X.shape[0]
    t0 = time.perf_counter()
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]),
                               fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0), device=dev)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    op.set_stream(stream.cuda_stream)
    xh = fgs.workload_vectors(n, nvec, 99)
    xh = xh if xh.ndim == 2 else xh[:, None]
    xc = torch.from_numpy(np.asfortranarray(xh).T.copy()).to(f"cuda:{dev}")
    xi = torch.empty((nvec, n), dtype=torch.float64, device=f"cuda:{dev}")
    for v in range(nvec):
        op.permute_device(xc[v].data_ptr(), xi[v].data_ptr(), nvec=1, ld=n, direction=0)
    yi = torch.empty_like(xi)
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def step():
        op.apply_device(fgs.OP_SYM_LAPLACIAN, xi.data_ptr(), yi.data_ptr(), nvec=nvec, ld=n, internal_order=True)

    for _ in range(3):
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for s0, s1 in ev:
        flush.zero_()
        s0.record(stream)
        step()
        s1.record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    out = {"workload": f"config{cfg}", "n": n, "d": info["d"], "N": info["N"], "m": info["m"], "nvec": nvec,
           "value": nvec / (ms / 1000.0), "unit": "matvecs/s", "ms_per_step": ms, "setup_s": setup_s}
    if cfg <= 4:
        out["lanczos"], _ = lanczos_timing(op, info)
    return out


def lanczos_timing(op, info, warm=2):
    """Lanczos time-to-k as the reference's eigs command splits it
    (commands.cpp:174-183): `solve_s` is the first solve on a fresh handle
    (workspace allocation and graph capture included, what a one-shot run
    pays); `solve_s_warm` the median of `warm` further solves on the same
    handle.  Ritz vectors are formed and copied to the host every time."""
    import torch

    import paper_1808_04580_b200 as fgs
    times, li, pairs, phases = [], None, None, None
    for _ in range(1 + warm):
        li = fgs.LanczosInfo()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        phases = op.lanczos_stats()
    rec = {"k": info["k"], "tol": 1e-8, "solve_s": times[0],
           "solve_s_warm": float(np.median(times[1:])) if warm else None,
           "iterations": li.iterations, "converged": li.converged, "phases": phases}
    return rec, pairs


# ---- B200 arm --------------------------------------------------------------
def run_b200(args, rank, world, local_rank):
    import torch
    import paper_1808_04580_b200 as fgs
    dev = local_rank
    torch.cuda.set_device(dev)
    info = fgs.workload_info(args.config)
    nvec = args.nvec or (16 if args.config == 5 else 1)
    X = fgs.workload_nodes(args.config, SEED)
    n = X.shape[0]
    params = fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0)
    kernel = fgs.KernelSpec.gaussian(info["sigma"])

    sharded = world > 1 or args.force_sharded
    dist = None
    if sharded:
        import torch.distributed as dist
        nid = [fgs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        nccl_id = nid[0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if sharded:
        op = fgs.AdjacencyOperator(X, kernel, params, device=dev, rank=rank, world=world, nccl_id=nccl_id)
    else:
        op = fgs.AdjacencyOperator(X, kernel, params, device=dev)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=dev)  # non-default: applies replay captured CUDA graphs
    torch.cuda.set_stream(stream)
    op.set_stream(stream.cuda_stream)
    nl = op.n_local
    geom = op.geometry()

    # device-resident inputs in the internal order (this rank's slice)
    xs_host = fgs.workload_vectors(n, nvec, 99)
    xs_host = xs_host if xs_host.ndim == 2 else xs_host[:, None]
    x_caller = torch.from_numpy(np.asfortranarray(xs_host).T.copy()).to(f"cuda:{dev}")  # [nvec][n]
    x_int = torch.empty((nvec, nl), dtype=torch.float64, device=f"cuda:{dev}")
    for v in range(nvec):  # caller order -> this rank's slice of the internal order
        op.permute_device(x_caller[v].data_ptr(), x_int[v].data_ptr(), nvec=1, ld=n, direction=0)
    y_int = torch.empty_like(x_int)
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=f"cuda:{dev}")  # > 126 MB L2

    def step():
        op.apply_device(fgs.OP_SYM_LAPLACIAN, x_int.data_ptr(), y_int.data_ptr(), nvec=nvec, ld=nl,
                        internal_order=True)

    for _ in range(args.warmup):
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
    # per-kernel durations: the same K steps again with stage events between
    # the launches (direct launches; kernel durations do not depend on graph
    # vs direct launch)
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
    fp64_tf = fgs.measure_fp64_peak(dev)
    per_launch = {k: stage_ms[i] / max(1, napp) for i, k in enumerate(STAGES)}
    work = stage_work(geom, nl, nvec)
    dom = max(("spread", "interp"), key=lambda k: per_launch[k])
    b, f = work[dom]
    t = per_launch[dom] * 1e-3
    t_hbm = b / (peaks["hbm_gbs"] * 1e9)
    t_fp = f / (fp64_tf * 1e12)
    if t_fp >= t_hbm:
        roof = {"bound": "fp64", "achieved": f / t / 1e12, "peak": fp64_tf, "unit": "TFLOP/s",
                "frac": (f / t / 1e12) / fp64_tf, "traffic": None,
                "peak_source": "fp64 DFMA microbenchmark on this B200 (not in MEASURED_PEAKS.json)"}
    else:
        roof = {"bound": "hbm", "achieved": b / t / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": (b / t / 1e9) / peaks["hbm_gbs"], "traffic": None,
                "peak_source": f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json)"}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(f"config{args.config}", {}).get(dom)
        if tr:
            roof["traffic"] = tr["dram_bytes"] * (nvec if args.config != 5 else 1)
            roof["traffic_source"] = f"ncu --set full, {tr['source']} ({tr['kernel']}), dram read+write per launch"
    except (OSError, ValueError):
        pass
    roof.update({"kernel": dom, "launch_ms": per_launch[dom], "algorithmic_bytes": b, "algorithmic_flops": f,
                 "t_roof_ms": 1e3 * max(t_hbm, t_fp), "frac_of_max_roof": max(t_hbm, t_fp) / t,
                 "stage_ms_per_step": {k: per_launch[k] for k in STAGES}})

    # ---- end to end through the public API with pinned host buffers ---------
    e2e = None
    if not sharded:
        hx = torch.from_numpy(np.asfortranarray(xs_host)).pin_memory()
        hy = torch.empty_like(hx).pin_memory()
        import ctypes as C
        L = fgs.lib()
        xp = C.cast(hx.data_ptr(), C.POINTER(C.c_double))
        yp = C.cast(hy.data_ptr(), C.POINTER(C.c_double))
        for _ in range(args.warmup):
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
        e2e = {"value": nvec / (e2e_ms / 1000.0), "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n * nvec,
               "d2h_bytes_per_step": 8 * n * nvec, "ms_per_step": e2e_ms,
               "path": "fgs_adjacency_apply (C ABI) with pinned host x/y, caller order"}

    else:
        # sharded handles take device vectors in the internal order (the
        # public multi-GPU API, fgs_adjacency_apply_device): each rank uploads
        # its slice from pinned memory, applies, downloads; max over ranks
        hx = x_int.cpu().pin_memory()
        hy = torch.empty_like(hx).pin_memory()
        for _ in range(args.warmup):
            x_int.copy_(hx, non_blocking=True)
            step()
            hy.copy_(y_int, non_blocking=True)
        torch.cuda.synchronize()
        dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            x_int.copy_(hx, non_blocking=True)
            step()
            hy.copy_(y_int, non_blocking=True)
            stream.synchronize()
        s1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([s0.elapsed_time(s1) / args.steps], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        e2e = {"value": nvec / (e2e_ms / 1000.0), "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n * nvec,
               "d2h_bytes_per_step": 8 * n * nvec, "ms_per_step": e2e_ms,
               "path": "per rank: pinned slice H2D + fgs_adjacency_apply_device (sharded, internal order) + D2H; "
                       "max over ranks"}

    # ---- Lanczos time-to-k (spectral.cpp:141-256 via the device path) -------
    lanczos = None
    if not sharded and not args.no_lanczos and args.config <= 4:
        rec, pairs = lanczos_timing(op, info)
        lanczos = {"setup_s": setup_s, **rec, "total_s": setup_s + rec["solve_s"],
                   "smallest_laplacian_eigs": [1.0 - v for v in pairs.values[:4].tolist()]}

    # ---- CPU baseline (rank 0, N=1) ----------------------------------------
    cpu = None
    if not sharded and not args.no_cpu:
        rate, desc, csetup = cpu_matvecs_per_s(args.config, X, info, nvec, args.cpu_seconds)
        cpu = {"value": rate, "unit": "matvecs/s", "cores": 1, "kind": "port", "sample": desc,
               "cpu": cpu_model(), "host_cores": os.cpu_count(), "setup_s": csetup}

    also = []
    if not sharded and args.also:
        for cfg in [int(c) for c in args.also.split(",") if c.strip()]:
            if cfg != args.config:
                try:
                    also.append(secondary(cfg, 10 if cfg != 5 else 2, dev))
                except Exception as e:  # noqa: BLE001 - report, do not lose the main line
                    also.append({"workload": f"config{cfg}", "error": str(e)[:200]})

    if rank == 0:
        line = {
            "metric": "fp64 Laplacian matvecs/sec", "value": value, "unit": "matvecs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded stand-in for the paper's datasets)",
            "config": {"workload": f"config{args.config}", "n": n, "d": info["d"], "sigma": info["sigma"],
                       "N": info["N"], "m": info["m"], "p": info["p"], "nvec": nvec, "op": "L_s x",
                       "parallelism": f"points sharded x{world}" if sharded else "single GPU",
                       "l2": "flushed (256 MB write) between timed steps, outside the events"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(w0, w1), "lanczos": lanczos, "setup_s": setup_s, "also": also,
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if (world > 1 or args.force_sharded) and args.impl == "b200":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world, local_rank)
    if (world > 1 or args.force_sharded) and args.impl == "b200":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
