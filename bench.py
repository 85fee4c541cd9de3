#!/usr/bin/env python3
"""LOBPCG hot-path benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "C2"): A = s*L7 on a 128^3 grid,
s = (N+1)^2, m = 10, Jacobi, B = I, tol 1e-8, max_iter 300, X0 = PCG64(0)
uniform(-1,1) built on the host (setup, not timed).  A "step" is one LOBPCG
iteration of the hot loop (lobpcg.py:418-540) on that state.

  value     iterations/s with the state resident in HBM (device-timed with
            CUDA events around K steps; every iteration includes its host
            small-matrix work and D2H/H2D of the small matrices)
  e2e       iterations/s of the public solve() call on host buffers: H2D of
            X0, all 300 iterations, exit refresh and D2H of the eigenvectors
  roofline  dominant kernel, algorithmic bytes / CUDA-event duration
  cpu_baseline  the CPU oracle (numpy/OpenBLAS restatement of the reference)
            on a bounded sample of C2 iterations, all host cores

--impl reference runs the CPU oracle alone (the reference is a Python
package; its restatement oracle/lobpcg_oracle.py is pinned bit-exact to it).
Multi-GPU (torchrun, N>1): weak scaling, one distributed solve on a
128 x 128 x 128N grid split in z-slabs (one C2-sized slab per GPU; halo
send/recv and Gram all-reduce over NCCL); value = N x global it/s
(C2-slab-iterations/s), max-over-ranks time.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_GRID, M_BLOCK, TOL, MAX_ITER, SEED = 128, 10, 1e-8, 300, 0
METRIC = "LOBPCG iterations/s & time-to-tol, 3-D 7-pt Laplacian; stencil HBM GB/s vs peak"
WORKLOAD = "C2: 128^3 7-pt Laplacian (scaled 1/h^2), m=10, Jacobi, B=I, tol 1e-8, max_iter 300"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_dict(n_gpus):
    return {
        "workload": WORKLOAD,
        "grid": [N_GRID] * 3,
        "block_size": M_BLOCK,
        "preconditioner": "jacobi",
        "tol": TOL,
        "max_iter": MAX_ITER,
        "seed": SEED,
        "l2": "inputs larger than L2 (10 live 168 MB blocks per iteration >> 126 MB L2)",
        "parallelism": (f"z-slab x{n_gpus} (grid 128x128x{128 * n_gpus}, one C2-size slab per "
                        "GPU, NCCL halo + Gram all-reduce)") if n_gpus > 1 else "single GPU",
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region.

    NVML in-process (nvidia_ml_py; cheap, no fork of this large process while
    the host side of the iteration runs); nvidia-smi as fallback."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period=0.05):
        self.index = index
        self.period = period
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            handle = None
            try:
                import torch

                uuid = str(torch.cuda.get_device_properties(index).uuid)
                handle = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
            except Exception:
                handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = (pynvml, handle)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flags = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        return [str(sm), str(mx)] + ["Active" if r & f else "Not Active" for f in flags]

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5).stdout.strip()
        return [v.strip() for v in out.split(",")] if out else None

    def _run(self):
        if os.environ.get("B2L_BENCH_NOCLOCK") == "1":   # diagnostic: sampler off
            return
        while True:
            try:
                row = self._sample_nvml() if self._nvml else self._sample_smi()
                if row:
                    self.rows.append(row)
            except Exception:
                pass
            if self._stop.wait(self.period if self._nvml else 0.2):
                break

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}


# ------------------------------------------------------------ CPU oracle
def cpu_oracle_sample(iters, threads_note):
    """Time `iters` C2 iterations of the CPU oracle; returns it/s."""
    from oracle import lobpcg_oracle as orc

    r = orc.laplacian_case(N_GRID, M_BLOCK, tol=TOL, max_iter=iters, seed=SEED,
                           record=False, timer=True)
    ts = r.iter_times
    # iteration i runs from ts[i] to ts[i+1]; the last stamp opens the final
    # (exit) check, so use the completed gaps.
    gaps = np.diff(ts)
    return float(len(gaps) / gaps.sum()), len(gaps)


REF_MAX_STEPS, REF_MAX_WARMUP = 12, 2


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    # a C2 iteration takes ~1.5 s on the host: the CPU arm times a bounded
    # sample of the same iteration sequence so the run ends within minutes
    warm, steps = min(args.warmup, REF_MAX_WARMUP), min(args.steps, REF_MAX_STEPS)
    total = warm + steps
    from oracle import lobpcg_oracle as orc

    r = orc.laplacian_case(N_GRID, M_BLOCK, tol=TOL, max_iter=total, seed=SEED,
                           record=False, timer=True)
    ts = np.array(r.iter_times)
    timed = ts[warm:warm + steps + 1]
    dt = float(timed[-1] - timed[0])
    k = len(timed) - 1
    value = k / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "it/s",
        "n_gpus": args.gpus, "steps": k, "warmup": warm,
        "ms_per_step": 1e3 * dt / k, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(1),
        "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "kind": "port",
                         "sample": f"C2 iterations {warm}..{warm + k} of the CPU "
                                   "oracle (numpy/OpenBLAS restatement, bit-exact to the reference)"},
        "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_0705_2626_b200 as pk
    from paper_0705_2626_b200 import device as dv

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    s = float((N_GRID + 1) ** 2)
    if world > 1:
        # weak scaling: a 128 x 128 x (128 P) grid, one C2-sized z-slab per
        # GPU, one-plane halos + Gram all-reduces over NCCL
        from paper_0705_2626_b200.distributed import SlabLaplacian3D, slab_initial_block

        A = SlabLaplacian3D((N_GRID, N_GRID, N_GRID * world), scale=s)
        x0 = slab_initial_block(A.grid, A.part, M_BLOCK, SEED)
        n = A.local_rows
    else:
        n = N_GRID ** 3
        A = pk.Laplacian3D((N_GRID,) * 3, scale=s)
        x0 = np.random.Generator(np.random.PCG64(SEED)).uniform(-1.0, 1.0, size=(n, M_BLOCK))
    T = pk.jacobi_preconditioner(A)
    cfg = pk.SolverConfig(block_size=M_BLOCK, tol=TOL, max_iter=MAX_ITER, seed=SEED)

    def new_run():
        return pk.LOBPCGRun(A, t=T, x0=x0, config=cfg)

    # ---- device-resident timing of K iterations
    # A full (gen-2) collection of the interpreter's import-time objects takes
    # 0.1-0.6 s and lands at an arbitrary step; collect once and freeze them
    # (no effect on the GPU work or the library's own host code).
    import gc

    gc.collect()
    gc.freeze()
    # Warm the drift-repair path (lobpcg.py:419-428) on a throw-away run first:
    # its first execution in a process has a variable one-time cost (measured
    # 3 ms .. 0.66 s on this pool) that must not land in the timed region.
    tmp = new_run()
    tmp.step()
    tmp._refresh_ritz(tmp._gram_xx())
    del tmp
    torch.cuda.synchronize()
    run = new_run()
    for _ in range(args.warmup):
        if not run.step():
            run = new_run()
    if run.it + args.steps > MAX_ITER:
        run = new_run()
    run_it0 = run.it
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    from paper_0705_2626_b200 import _lib

    nlib = _lib.load()
    launches0 = nlib.b2l_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trace = os.environ.get("B2L_BENCH_TRACE") == "1"
    stamps = []
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            run.step()
            if trace:
                stamps.append(time.perf_counter())
        e1.record()
        torch.cuda.synchronize()
    if trace and len(stamps) > 1:
        dts = np.diff(stamps) * 1e3
        worst = np.argsort(dts)[::-1][:5]
        print("trace: slowest steps " + ", ".join(f"({i + 1}, {dts[i]:.2f} ms)" for i in worst),
              file=sys.stderr, flush=True)
    launches = nlib.b2l_launch_count() - launches0   # every kernel of libb200lobpcg
    ms = e0.elapsed_time(e1)
    barrier()
    ms_all = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_all = float(t.item())
    value = world * args.steps / (ms_all / 1e3)

    # ---- per-kernel durations (CUDA events on the launching stream)
    ktimes = {}

    def timer(name, fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        ktimes.setdefault(name, []).append((a, b))
        return r

    run2 = new_run()
    for _ in range(3):
        run2.step()
    with pk.device_options(timer=timer):
        for _ in range(args.steps):
            run2.step()
    torch.cuda.synchronize()
    kt = {k: [a.elapsed_time(b) for a, b in v] for k, v in ktimes.items()}
    ld = dv.even(M_BLOCK)
    k_act = M_BLOCK  # C2 never locks within 300 iterations (reference run)
    # algorithmic bytes per launch (blocks counted at k=m columns)
    alg = {
        # K1 (+K5b): read W, write A W (the X read for [X W]^T A W is extra)
        "stencil": 16.0 * n * k_act,
        "residual": 8.0 * n * (2 * M_BLOCK + k_act),
        "update": 8.0 * n * (2 * M_BLOCK + 4 * k_act + 4 * M_BLOCK),
        # F1: read X, AX, W, AW, P_J, AP_J; write X', AX', P', AP', W'
        "step": 8.0 * n * (6 * M_BLOCK + 5 * k_act),
    }
    # the per-step big gram reads X, W, P, AW, AP; the drift gram reads X
    gram_calls = kt.get("gram", [])
    per = {}
    for name in ("stencil", "residual", "update", "step"):
        if kt.get(name):
            d = float(np.mean(kt[name]))
            per[name] = {"ms": d, "gbs": alg[name] / (d / 1e3) / 1e9, "calls": len(kt[name])}
    if gram_calls:
        db = float(np.mean(gram_calls))
        per["gram"] = {"ms": db, "gbs": 8.0 * n * (3 * M_BLOCK + 2 * k_act) / (db / 1e3) / 1e9,
                       "calls": len(gram_calls)}
    if kt.get("gram_drift"):
        dd = float(np.mean(kt["gram_drift"]))
        per["gram_drift"] = {"ms": dd, "gbs": 8.0 * n * M_BLOCK / (dd / 1e3) / 1e9,
                             "calls": len(kt["gram_drift"])}
    total_ms = {k: v["ms"] * v["calls"] for k, v in per.items()}
    dom = max(total_ms, key=total_ms.get) if total_ms else "stencil"
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    prof = ROOT / "profiles" / "ncu_traffic.json"
    traffic = None
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": per[dom]["gbs"], "peak": peak,
                "unit": "GB/s", "frac": per[dom]["gbs"] / peak, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                "kernels": per,
                "stencil_frac_of_8TBs": per.get("stencil", {}).get("gbs", 0.0) / 8000.0}

    # ---- e2e through the public API on host buffers: X0 from pinned host
    # memory, eigenvectors back to host memory, both inside the timed call.
    # One short untimed warm-up solve first (same shapes: it primes the
    # caching host/device allocators, the tensor-map and kernel caches).
    x0_host = torch.from_numpy(np.ascontiguousarray(x0)).pin_memory()
    warm_cfg = pk.SolverConfig(block_size=M_BLOCK, tol=TOL, max_iter=3, seed=SEED)
    del run, run2
    pk.solve(A, t=T, x0=x0_host, config=warm_cfg)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = pk.solve(A, t=T, x0=x0_host, config=cfg)
    vecs = rep.eigenvectors  # numpy: D2H inside solve()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    it_used = rep.iterations_used
    e2e_val = world * it_used / e2e_s
    exact = pk.exact_eigenvalues(A.grid, M_BLOCK, scale=s)

    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(config_dict(world), timed_iterations=[run_it0, run_it0 + args.steps]),
        "e2e": {"value": e2e_val, "unit": "it/s",
                "h2d_bytes_per_step": int(x0.nbytes / max(it_used, 1)),
                "d2h_bytes_per_step": int(vecs.nbytes / max(it_used, 1)),
                "solve_seconds": e2e_s, "iterations": it_used, "status": rep.status,
                "time_to_max_iter_s": e2e_s,
                "max_rel_err_vs_closed_form": float(np.max(np.abs(rep.eigenvalues - exact) / exact))},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        v, k = cpu_oracle_sample(args.cpu_iters, cores)
        line["cpu_baseline"] = {"value": v, "unit": "it/s", "cores": cores, "kind": "port",
                                "sample": f"{k} C2 iterations (after init) of the CPU oracle, "
                                          "numpy/OpenBLAS on all host cores"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # default: the C2 run after a warm-up of 15 iterations (iterations
    # 15..300, including its later drift repairs), ~0.2 s of device time
    ap.add_argument("--steps", type=int, default=285)
    ap.add_argument("--warmup", type=int, default=15)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
