"""Per-kernel device times (mmb_profile_step) and the step time for one bench workload."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS, algorithmic_bytes, random_state  # noqa: E402
from paper_1501_07293_b200 import Grid, MaterialParams, Precision, ProblemSpec, make_simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="512x512x8_f32")
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, prec = WORKLOADS[a.workload]
spec = ProblemSpec(name=a.workload, grid=Grid(nx, ny, nz, delta), material=MaterialParams(a_ex, ms, hk, alpha), dt=dt)
sim = make_simulation(spec, precision=Precision.f32 if prec == "f32" else Precision.f64)
sim.set_magnetization(random_state(nx, ny, nz, ms, prec))
sim.time_steps(3)
t = sim.time_steps(a.steps) / a.steps
prof = sim.profile_step(a.steps)
_, kb = algorithmic_bytes(nx, ny, nz, 4 if prec == "f32" else 8)
print(a.workload, "step %.3f ms" % t)
for k, v in prof.items():
    print("  %-8s %8.3f ms  %6.2f GB  %6.2f TB/s" % (k, v, kb.get(k, 0) / 1e9, kb.get(k, 0) / (v * 1e-3) / 1e12))
