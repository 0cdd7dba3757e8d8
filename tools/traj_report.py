"""SP#4 <m>(t) parity report (B200 vs the reference's own full-precision trajectories in
tests/golden/traj_*.tsv and the reference fixture). Prints one line per case."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1501_07293_b200 import RunOptions  # noqa: E402
from tests.helpers import b200, sp4  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def crossing(rows, reversal=50000, dt=5e-6):
    for i in range(1, len(rows)):
        if rows[i - 1, 0] <= reversal:
            continue
        a, b = rows[i - 1, 1], rows[i, 1]
        if a > 0.0 and b <= 0.0:
            return (rows[i - 1, 0] + a / (a - b) * (rows[i, 0] - rows[i - 1, 0])) * dt - reversal * dt
    return float("nan")


fixture = np.loadtxt(os.path.join(GOLD, "sp4_field1_reference.tsv"))
print(f"reference fixture (6 decimals, FFTW build): crossing {crossing(fixture):.5f} ns after reversal")
for path in ("fast", "general"):
    os.environ.pop("MMB_GENERAL_PATH", None)
    if path == "general":
        os.environ["MMB_GENERAL_PATH"] = "1"
    for name, grid, prec in [("sp4_166_f64", (166, 42, 3.0), "f64"), ("sp4_128_f64", (128, 32, 3.90625), "f64"),
                             ("sp4_166_f32", (166, 42, 3.0), "f32"), ("sp4_128_f32", (128, 32, 3.90625), "f32")]:
        want = np.loadtxt(os.path.join(GOLD, f"traj_{name}.tsv"), comments="#")
        sim = b200(sp4(*grid), prec)
        recs = []
        t0 = time.perf_counter()
        sim.run(RunOptions(steps=150000, cadence=1000, sink=recs.append))
        wall = time.perf_counter() - t0
        got = np.array([[r.step, r.mx, r.my, r.mz] for r in recs])
        dev = np.max(np.abs(got[:, 1:] - want[:, 1:]))
        extra = ""
        if name == "sp4_166_f64":
            post = got[:, 0] > 50000
            extra = f" | vs fixture: max|d<m>| {np.max(np.abs(got[:, 1:] - fixture[:, 1:])):.2e}, " \
                    f"post-reversal max|d<my>| {np.max(np.abs(got[post, 2] - fixture[post, 2])):.2e}"
        print(f"{path:7s} {name}: max|<m>_B200 - <m>_ref| over 150 records = {dev:.3e} "
              f"(tol {'1e-6' if prec == 'f64' else '1e-3'}); crossing {crossing(got):.5f} ns "
              f"(ref {crossing(want):.5f}); 150000 steps in {wall:.2f} s{extra}", flush=True)
