#!/usr/bin/env python
"""Benchmark of the B200 LLG step (BASELINE.json metric: LLG cell-updates/s and % of HBM
roofline) on the 512x512x8 fp32 thin-film scaling point (BASELINE configs[2], the north
star's target configuration; SP#3 material, random initial state, no applied field).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--workload ...]

One process per GPU (torchrun for N > 1). N = 1 runs the 512x512x8 f32 headline; N > 1 runs
BASELINE configs[4], 2048x2048x64 f32 split into z-slabs over the ranks (NCCL all-to-all
transposes + halo; scaling "strong"), unless --workload picks another grid (grids that fit one
GPU then run as N independent replicas, scaling "weak"). Time = max over ranks of the
CUDA-event time of K graph-replayed steps; value = cell-updates of the whole job / that time.
Initial state: the reference generator (random_unit_field, proj/src/validate.cpp:21-39,
seed 20240 + nx) via libmmb.so's host utility.
--impl reference times the reference's own CPU solver (oracle/_ref: the reference sources
compiled in place with the FFTW-API shim) on the host cores, rank 0 only.
Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, precision)
    "512x512x8_f32": (512, 512, 8, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, "f32"),
    "1024x1024x32_f32": (1024, 1024, 32, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, "f32"),
    "256x256x1_f32": (256, 256, 1, 3.0, 1.3e7, 800.0, 0.0, 0.5, 5e-6, "f32"),
    "256x256x1_f64": (256, 256, 1, 3.0, 1.3e7, 800.0, 0.0, 0.5, 5e-6, "f64"),
    "sp4_128x32x1_f64": (128, 32, 1, 3.90625, 1.3e7, 800.0, 0.0, 0.5, 5e-6, "f64"),
    # the reference's own benchmark verb: SP#3 cube relaxation n^3 (proj/src/benchmark.cpp)
    "sp3_64_f32": (64, 64, 64, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, "f32"),
    "sp3_64_f64": (64, 64, 64, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, "f64"),
    "sp3_128_f32": (128, 128, 128, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, "f32"),
    # BASELINE configs[4]: slab-sharded across the GPUs of the box (strong scaling)
    "2048x2048x64_f32": (2048, 2048, 64, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, "f32"),
}
SHARDED = {"2048x2048x64_f32"}
METRIC = "LLG cell-updates/s"
UNIT = "cell-updates/s"


def algorithmic_bytes(nx, ny, nz, w):
    """SURVEY.md §8(d) canonical per-step bytes and the per-kernel split (one HBM read and
    write per stage of the pruned r2c pipeline; tensor = 6 real octants)."""
    n = nx * ny * nz
    lx = 1 if nx == 1 else 1 << math.ceil(math.log2(2 * nx - 1))
    ly = 1 if ny == 1 else 1 << math.ceil(math.log2(2 * ny - 1))
    lz = 1 if nz == 1 else 1 << math.ceil(math.log2(2 * nz - 1))
    xh = 1 if lx == 1 else lx // 2 + 1
    yh = 1 if ly == 1 else ly // 2 + 1
    zh = 1 if lz == 1 else lz // 2 + 1
    half = 3 * xh * ny * nz * 2 * w          # live half-spectrum rows (complex)
    padded = 3 * xh * ly * nz * 2 * w        # after the y-forward
    tensor = 6 * xh * yh * zh * w
    k = {"x_fwd": 3 * n * w + half, "x_inv": half + 3 * n * w, "llg": 9 * n * w}
    canonical = sum(k.values()) + (2 * half + tensor if nz == 1 else 2 * half + 4 * padded + tensor)
    # per-kernel algorithmic bytes of the kernels each path actually launches
    k["y_mac"] = k["yz"] = 2 * half + tensor          # fused: padded spectrum stays on chip
    k["xstep"] = 2 * half + 6 * n * w                 # fused x^-1 + LLG + x: S in/out, M in/out
    k["y_fwd"] = half + padded
    k["z_mac"] = 2 * padded + tensor
    k["y_inv"] = padded + half
    # SURVEY §8(d)'s canonical stage bytes of the stages each fused kernel implements (the
    # north-star pipeline K1 x-fwd, K2 y-fwd, K3 z+MAC, K4 y-inv, K5 x-inv, K6 local terms)
    if nz > 1:
        k2 = half + padded
        k3 = 2 * padded + tensor
        k4 = padded + half
    else:  # nz == 1: one fused y pass (forward, MAC, inverse) reads and writes the half spectrum
        k2, k3, k4 = half, tensor, half
    k["canonical"] = {"yz": k2 + k3 + k4, "xstep": k["x_inv"] + k["llg"] + k["x_fwd"],
                      "y_fwd": k2, "z_mac": k3, "y_inv": k4}
    return canonical, k


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: an NVML
    poller thread (~1 kHz) started right before and stopped right after it (the timed regions
    are a few ms long, shorter than nvidia-smi's sampling period). Falls back to nvidia-smi
    polling every 100 ms when NVML is unavailable."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self.thread = None
        self.stop = False
        self.proc = None
        self.path = None

    def _poll(self, nv, h):
        while not self.stop:
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.nv = nv
            self.thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.thread.start()
            while not self.samples:  # the poller is running before the timed region starts
                time.sleep(0.0002)
            return self
        except Exception:
            self.thread = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.thread:
            self.stop = True
            self.thread.join(timeout=5)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def mark(self):
        """Call right before and right after the timed call: the summary then covers the
        samples between the two marks."""
        self.marks = getattr(self, "marks", []) + [len(self.samples)]

    def summary(self):
        if self.thread is not None or self.samples:
            marks = getattr(self, "marks", [])
            win = self.samples[marks[0]:marks[1]] if len(marks) >= 2 and marks[1] > marks[0] else self.samples
            if not win:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
            sm = [s for s, _ in win]
            bits = 0
            for _, r in win:
                bits |= r
            reasons = sorted(n for n, c in self.NAMES if bits & getattr(self.nv, c, 0))
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                    "samples": len(sm), "sm_mhz_min": min(sm),
                    "source": "NVML poller (~1 kHz) between the marks around the timed call"}
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [r for r in rows if r[2].isdigit() and int(r[2]) > 0] or rows
        sm = [int(r[0]) for r in load if r[0].isdigit()]
        mx = [int(r[1]) for r in rows if r[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(load)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        ndev = max(1, torch.cuda.device_count())
        if world <= ndev:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
        else:
            # more ranks than GPUs (only to exercise the multi-rank code path on a small box):
            # ranks share devices, collectives over gloo; timings are then contended
            local = local % ndev
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, v):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, v):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def random_state(nx, ny, nz, ms, prec, z0=0, nz_local=None):
    """The reference generator's field (seed 20240 + nx), planes
    [z0, z0 + nz_local), from libmmb.so's host utility mmb_random_unit_field."""
    from paper_1501_07293_b200 import Precision, random_unit_field
    return random_unit_field(nx, ny, nz, ms, 20240 + nx, Precision.f32 if prec == "f32" else Precision.f64,
                             z0=z0, nz_local=nz_local)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def pcie_copy_ms(nbytes, dtype):
    """Device time of one pinned H2D plus one pinned D2H of `nbytes` each (cudaMemcpyAsync
    through torch): the floor of an e2e step that moves M in and out over PCIe."""
    import torch
    n = nbytes // np.dtype(dtype).itemsize
    h_in = torch.empty(n, dtype=torch.float32 if dtype == np.float32 else torch.float64, pin_memory=True)
    h_out = torch.empty_like(h_in).pin_memory()
    d = torch.empty_like(h_in, device="cuda")
    for _ in range(2):
        d.copy_(h_in, non_blocking=True)
        h_out.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record()
    for _ in range(reps):
        d.copy_(h_in, non_blocking=True)
        h_out.copy_(d, non_blocking=True)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def profile_summary(workload):
    """ncu-derived DRAM traffic per launch of the dominant kernel, if committed."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload, {})
    except Exception:
        return {}


def cpu_reference_time(wl, warmup=1, measure=3, serial_measure=2):
    """The reference's Simulation<T>::step() (oracle/_ref) on the host cores, timed as
    proj/src/benchmark.cpp:40-46 does (make_simulation per backend, warm-up steps, then
    steady-clock time of the measured steps; setup excluded), on a bounded sample: `measure`
    steps on the parallel backend with every host thread and `serial_measure` steps on the
    serial backend (1 core). FFTs are single-threaded in both, as in the reference."""
    # every host thread (torchrun exports OMP_NUM_THREADS=1 per rank; only rank 0 runs this, and
    # libgomp reads the variable when the reference library loads it below)
    cores = int(os.environ.get("MMB_REF_THREADS", len(os.sched_getaffinity(0))))
    os.environ["OMP_NUM_THREADS"] = str(cores)
    from oracle import ref
    nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, prec = WORKLOADS[wl]
    if not ref.available():
        raise RuntimeError("oracle/_ref/libmmsim_ref.so missing (build with make -C oracle)")
    P = ref.Problem(nx, ny, nz, delta, a_ex, ms, hk, alpha, dt)
    m0 = ref.random_unit_field(nx, ny, nz, ms, 20240 + nx, np.float64 if prec == "f64" else np.float32)
    n = nx * ny * nz
    rows = []
    for backend, steps, ncores in (("parallel", measure, cores), ("serial", serial_measure, 1)):
        if steps <= 0:
            continue
        t0 = time.perf_counter()
        sim = ref.RefSimulation(P, prec, backend=backend)
        setup = time.perf_counter() - t0
        sim.set_m(m0)
        for _ in range(warmup):
            sim.step(1)
        t1 = time.perf_counter()
        for _ in range(steps):
            sim.step(1)
        t = time.perf_counter() - t1
        rows.append({"backend": backend, "cores": ncores, "warmup": warmup, "steps": steps,
                     "ms_per_step": 1e3 * t / steps, "value": n * steps / t, "setup_s": round(setup, 2)})
        del sim
    par = rows[0]
    return {"value": par["value"], "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"reference Simulation<{'float' if prec == 'f32' else 'double'}>::step() on {nx}x{ny}x{nz}, "
                      f"timed as benchmark.cpp:40-46: {warmup} warm-up + {par['steps']} measured steps on the "
                      f"parallel backend ({cores} threads; FFTs single-threaded, FFTW-API shim), setup excluded"
                      + (f"; serial row: {warmup} + {rows[1]['steps']} steps on 1 core" if len(rows) > 1 else ""),
            "ms_per_step": par["ms_per_step"], "steps": par["steps"], "rows": rows,
            "cpu_model": cpu_model(), "nproc": os.cpu_count()}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    wl = args.workload
    nx, ny, nz, *_ , prec = WORKLOADS[wl]
    if wl in SHARDED:
        line = {"metric": METRIC, "impl": "reference", "unavailable":
                f"the reference layout needs ~181 GB of host memory at {wl} (SURVEY.md §8(d)); no CPU run"}
        print(json.dumps(line), flush=True)
        return 0
    # the reference arm times a bounded sample: per step ~2 s (parallel) / ~4 s (serial) at 512x512x8
    measure = max(1, min(args.steps, int(os.environ.get("MMB_REF_STEPS", "10"))))
    c = cpu_reference_time(wl, warmup=1, measure=measure, serial_measure=min(3, measure))
    line = {"metric": METRIC, "value": c["value"], "unit": UNIT, "n_gpus": world, "steps": c["steps"],
            "warmup": 1, "ms_per_step": c["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "impl": "reference",
            "config": {"workload": wl, "nx": nx, "ny": ny, "nz": nz, "parallelism": "host cores"},
            "cpu_baseline": c,
            "e2e": {"value": c["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_b200_sharded(args, world, rank, local):
    """BASELINE configs[4]: one global grid split into z-slabs over the ranks (NCCL transposes
    and halo exchange); value = global cell-updates / max-over-ranks device time."""
    from paper_1501_07293_b200 import Grid, MaterialParams, Precision, ProblemSpec
    from paper_1501_07293_b200.simulation import make_sharded_simulation, nccl_unique_id
    import torch
    import torch.distributed as dist
    wl = args.workload
    nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, prec = WORKLOADS[wl]
    w = 4 if prec == "f32" else 8
    n = nx * ny * nz
    nid = torch.zeros(128, dtype=torch.uint8,
                      device="cuda" if world > 1 and dist.get_backend() == "nccl" else "cpu")
    if rank == 0:
        nid[:] = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8)
    if world > 1:
        dist.broadcast(nid, 0)
    spec = ProblemSpec(name=wl, grid=Grid(nx, ny, nz, delta), material=MaterialParams(a_ex, ms, hk, alpha), dt=dt)
    sim = make_sharded_simulation(spec, Precision.f32 if prec == "f32" else Precision.f64, rank, world,
                                  bytes(nid.cpu().numpy()), device=local)
    sim.set_magnetization(random_state(nx, ny, nz, ms, prec, z0=sim.z0, nz_local=sim.nz_local))
    barrier(world)
    with ClockSampler(local) as clk:
        sim.time_steps(max(3, args.warmup))
        barrier(world)
        clk.mark()
        t_ms = sim.time_steps(args.steps)
        clk.mark()
    t_ms = max_over_ranks(world, t_ms)
    value = n * args.steps / (t_ms * 1e-3)
    ms_step = t_ms / args.steps
    b_alg, _ = algorithmic_bytes(nx, ny, nz, w)
    peak, peak_kind = load_peaks()
    achieved = b_alg / (ms_step * 1e-3) / 1e9
    # e2e: each rank moves its slab host->device and back around every step
    pin = torch.empty((3, sim.nz_local, ny, nx), dtype=torch.float32 if prec == "f32" else torch.float64,
                      pin_memory=True).numpy()
    sim.get_m_into(pin)
    e_steps = max(1, min(args.steps, 5))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e_steps):
        sim.set_m_from(pin)
        sim.step(1)
        sim.get_m_into(pin)
    te = max_over_ranks(world, time.perf_counter() - t0)
    slab_bytes = 3 * sim.nz_local * ny * nx * w
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
                "config": {"workload": wl, "nx": nx, "ny": ny, "nz": nz, "delta_nm": delta,
                           "parallelism": (f"z-slabs x{world} (chunked NCCL all-to-all overlapped with the y/z "
                                           "kernels, NCCL halo planes)" if world > 1
                                           else "single GPU (one slab: no exchange)"),
                           "l2": "working set >> 126 MB L2; no flush", "cells": n},
                "roofline": {"bound": "hbm", "kernel": "sharded_step", "achieved": achieved / world,
                             "peak": peak, "unit": "GB/s", "frac": achieved / world / peak, "traffic": None,
                             "alg_bytes": b_alg, "peak_kind": peak_kind,
                             "note": "canonical step bytes (SURVEY §8(d)) per GPU over the step time"},
                "cpu_baseline": {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                 "sample": "N/A: the reference layout needs ~181 GB at 2048x2048x64 (SURVEY §8(d))"},
                "e2e": {"value": n * e_steps / te, "unit": UNIT, "h2d_bytes_per_step": slab_bytes * world,
                        "d2h_bytes_per_step": slab_bytes * world,
                        "api": "mmb_set_m + mmb_step(1) + mmb_get_m per step on every rank's slab"},
                "gpu_launches": sim.launches_per_step() * args.steps,
                "clocks": clk.summary(), "device_bytes": sim.device_bytes(), "path": sim.path_info()}
        print(json.dumps(line), flush=True)
    barrier(world)
    return 0


def run_b200(args, world, rank, local):
    if args.workload in SHARDED:
        return run_b200_sharded(args, world, rank, local)
    from paper_1501_07293_b200 import (Grid, MaterialParams, Precision, ProblemSpec, make_simulation)
    import torch
    wl = args.workload
    nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, prec = WORKLOADS[wl]
    dtype = np.float32 if prec == "f32" else np.float64
    w = 4 if prec == "f32" else 8
    n = nx * ny * nz
    spec = ProblemSpec(name=wl, grid=Grid(nx, ny, nz, delta), material=MaterialParams(a_ex, ms, hk, alpha),
                       dt=dt)
    sim = make_simulation(spec, precision=Precision.f32 if prec == "f32" else Precision.f64, device=local)
    m0 = random_state(nx, ny, nz, ms, prec)
    sim.set_magnetization(m0)

    # ---- device-resident throughput (value). The warm-up steps run right before the timed
    # ones (after the clock sampler started), so the SMs are at their load clock when the
    # timed region begins.
    barrier(world)
    with ClockSampler(local) as clk:
        sim.time_steps(max(3, args.warmup))
        clk.mark()
        t_ms = sim.time_steps(args.steps)
        clk.mark()
    t_ms = max_over_ranks(world, t_ms)
    value = n * args.steps * world / (t_ms * 1e-3)
    ms_step = t_ms / args.steps

    # ---- per-kernel times (events between the kernels of replayed graphs) for the roofline
    prof = sim.profile_step(max(16, min(args.steps, 64)))
    b_alg, kbytes = algorithmic_bytes(nx, ny, nz, w)
    peak, peak_kind = load_peaks()
    top = max(prof, key=prof.get)
    achieved = kbytes[top] / (prof[top] * 1e-3) / 1e9
    ps = profile_summary(wl)
    traffic = ps.get(top, {}).get("dram_bytes") if ps else None
    roof = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "alg_bytes": kbytes[top],
            "kernel_ms": prof[top], "peak_kind": peak_kind,
            "step": {"alg_bytes": b_alg, "achieved": b_alg / (ms_step * 1e-3) / 1e9,
                     "frac": b_alg / (ms_step * 1e-3) / 1e9 / peak},
            "kernels_ms": prof}
    # the same kernel credited with SURVEY §8(d)'s canonical bytes of the stages it fuses (the
    # bytes the north-star stage pipeline moves for them; the fused kernel moves `alg_bytes`)
    cb = kbytes.get("canonical", {}).get(top)
    if cb:
        roof["canonical_stages"] = {"alg_bytes": cb, "achieved": cb / (prof[top] * 1e-3) / 1e9,
                                    "frac": cb / (prof[top] * 1e-3) / 1e9 / peak}
    # The FFT and LLG kernels are bounded by instruction issue, not by HBM: the warp
    # instructions ncu counted per launch against the issue limit of 4 per clock per SM (148 SMs
    # at the SM clock sampled during the timed region), over this run's kernel time.
    wi = ps.get(top, {}).get("warp_inst") if ps else None
    if wi:
        roof["issue"] = {"warp_inst": wi, "sm_mhz": clk.summary().get("sm_mhz") or 1965.0,
                         "limit_us": wi / (148 * 4 * (clk.summary().get("sm_mhz") or 1965.0)),
                         "frac": wi / (148 * 4 * (clk.summary().get("sm_mhz") or 1965.0)) / (prof[top] * 1e3),
                         "source": "ncu smsp__inst_executed.sum per launch (profiles/ncu_summary.json)"}

    # ---- end to end through the public API with host buffers (pinned): per step
    # H2D of M, one step, D2H of M
    pin_in = torch.empty((3, nz, ny, nx), dtype=torch.float32 if prec == "f32" else torch.float64,
                         pin_memory=True).numpy()
    pin_out = torch.empty_like(torch.from_numpy(pin_in)).pin_memory().numpy()
    pin_in[...] = m0
    for _ in range(2):
        sim.set_m_from(pin_in)
        sim.step(1)
        sim.get_m_into(pin_out)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.set_m_from(pin_in)
        sim.step(1)
        sim.get_m_into(pin_out)
    te_sync = max_over_ranks(world, time.perf_counter() - t0)
    # the same per-step traffic through the stream-ordered calls: the upload of step i+1, the
    # step and the download of step i overlap (PCIe is full duplex); one synchronise at the end
    for _ in range(2):
        sim.set_m_async(pin_in)
        sim.step(1)
        sim.get_m_async(pin_out)
    sim.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sim.set_m_async(pin_in)
        sim.step(1)
        sim.get_m_async(pin_out)
    sim.synchronize()
    te = max_over_ranks(world, time.perf_counter() - t0)
    copy_ms = pcie_copy_ms(3 * n * w, dtype)
    # a streaming run through the public API: M uploaded once, then mmb_run with a <m> record
    # (device -> host, 24 bytes) after every step, delivered through the device record ring
    from paper_1501_07293_b200 import RunOptions
    recs = []
    barrier(world)
    t0 = time.perf_counter()
    sim.set_m_from(pin_in)
    sim.run(RunOptions(steps=args.steps, cadence=1, sink=recs.append))
    tr = max_over_ranks(world, time.perf_counter() - t0)
    e2e = {"value": n * args.steps * world / te, "unit": UNIT,
           "h2d_bytes_per_step": 3 * n * w, "d2h_bytes_per_step": 3 * n * w,
           "api": "mmb_set_m_async + mmb_step(1) + mmb_get_m_async per step, mmb_synchronize at the end "
                  "(libmmb.so C-ABI via ctypes)",
           "ms_per_step": 1e3 * te / args.steps,
           "sync": {"value": n * args.steps * world / te_sync, "ms_per_step": 1e3 * te_sync / args.steps,
                    "api": "mmb_set_m + mmb_step(1) + mmb_get_m per step (each call synchronises)",
                    "pcie_floor_ms": copy_ms + ms_step},
           "note": "per step: pinned H2D of M (25 MB), one graph-replayed step, pinned D2H of M (25 MB); the "
                   "stream-ordered calls overlap step i's download with step i+1's upload and step; "
                   "sync.pcie_floor_ms = device time of the two copies back to back + the step",
           "run_records": {"value": n * args.steps * world / tr, "unit": UNIT,
                           "h2d_bytes": 3 * n * w, "d2h_bytes_per_step": 24, "records": len(recs),
                           "api": "mmb_set_m once + mmb_run(steps, cadence 1, record callback)"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_time(wl, warmup=1, measure=3, serial_measure=2)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
                "config": {"workload": wl, "nx": nx, "ny": ny, "nz": nz, "delta_nm": delta,
                           "material": "SP#3 (Ms=1000, A=1e-11 J/m, Hk=100, alpha=0.5)"
                           if nz > 1 else "permalloy (Ms=800, A=1.3e-11 J/m)",
                           "initial_state": "seeded random unit field",
                           "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                           "l2": "per-step working set (spectrum scratch + M/H + tensor) > 126 MB L2; no flush",
                           "cells": n},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": sim.launches_per_step() * args.steps,
                "clocks": clk.summary(),
                "device_bytes": sim.device_bytes(), "path": sim.path_info()}
        print(json.dumps(line), flush=True)
    barrier(world)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: 512x512x8_f32 on one GPU, 2048x2048x64_f32 z-slabs on N > 1")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    world, rank, local = dist_setup() if args.impl == "b200" else (
        int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if args.workload is None:
        args.workload = "512x512x8_f32" if world == 1 else "2048x2048x64_f32"
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_b200(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
