"""Device time per step of the slab-sharded pipeline run as emulated ranks on one GPU (all
ranks' kernels and exchanges on one device): transposes vs peer mode (MMB_SHARD_PEER)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS, random_state  # noqa: E402
from paper_1501_07293_b200 import Grid, MaterialParams, Precision, ProblemSpec  # noqa: E402
from paper_1501_07293_b200.simulation import make_emulated_sharded_simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="1024x1024x32_f32")
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, prec = WORKLOADS[a.workload]
spec = ProblemSpec(name=a.workload, grid=Grid(nx, ny, nz, delta), material=MaterialParams(a_ex, ms, hk, alpha), dt=dt)
sim = make_emulated_sharded_simulation(spec, Precision.f32, a.world)
sim.set_magnetization(random_state(nx, ny, nz, ms, prec))
sim.time_steps(2)
t = sim.time_steps(a.steps) / a.steps
print(f"{a.workload} world {a.world} peer={os.environ.get('MMB_SHARD_PEER', '0')} chunks={os.environ.get('MMB_SHARD_CHUNKS', '4')}: {t:.3f} ms/step "
      f"(all ranks on one GPU)")
