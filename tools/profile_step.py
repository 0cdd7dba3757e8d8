"""Minimal driver for ncu: build one Simulation for a bench workload, take `steps` graph
steps, synchronise. Setup launches 11 kernels (twiddles x3, tensor octant, cs tables x3,
axis transforms x3, finalize); each step launches Simulation.launches_per_step() kernels."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS, random_state  # noqa: E402
from paper_1501_07293_b200 import Grid, MaterialParams, Precision, ProblemSpec, make_simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="512x512x8_f32")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, prec = WORKLOADS[a.workload]
spec = ProblemSpec(name=a.workload, grid=Grid(nx, ny, nz, delta), material=MaterialParams(a_ex, ms, hk, alpha), dt=dt)
sim = make_simulation(spec, precision=Precision.f32 if prec == "f32" else Precision.f64)
sim.set_magnetization(random_state(nx, ny, nz, ms, prec))
sim.step(a.steps)
sim.synchronize()
print("ok", a.workload, sim.launches_per_step(), "launches/step")
