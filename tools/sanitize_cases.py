"""Small runs of every kernel variant for compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [--quick]

Each case builds a Simulation (or an emulated sharded one), takes 2 steps, evaluates H_eff and
prints its path_info, so the log names the variants that ran under the tool."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1501_07293_b200 import (FieldSchedule, Grid, MaterialParams, Precision, ProblemSpec,  # noqa: E402
                                   ScheduleStage, make_simulation, random_unit_field)
from paper_1501_07293_b200.simulation import make_emulated_sharded_simulation  # noqa: E402

# (nx, ny, nz, precision, env)
CASES = [
    (24, 12, 4, "f32", {}),                          # fused y/z, Lz = 16, small x tile
    (24, 12, 1, "f64", {}),                          # fused y/z nz = 1, f64
    (200, 300, 8, "f32", {}),                        # PB = 128 x tile
    (512, 512, 8, "f32", {}),                        # headline: PB = 224 x tile (14 rows)
    (700, 20, 1, "f32", {}),                         # Lx = 2048 lane-pair x tile
    (600, 300, 8, "f32", {}),                        # Lx = 2048 WIDE x tile
    (40, 600, 9, "f32", {}),                         # streaming y/z, Ly = 2048 lane pairs
    (1100, 24, 9, "f32", {}),                        # Lx = 4096 x tile
    (40, 24, 9, "f64", {}),                          # streaming y/z f64
    (16, 12, 3, "f32", {"MMB_GENERAL_PATH": "1"}),   # general 6-kernel pipeline
]
SHARDED = [((40, 24, 9), 3, "f32", "0"), ((32, 16, 8), 2, "f32", "1")]


def spec(nx, ny, nz):
    return ProblemSpec(name="san", grid=Grid(nx, ny, nz, 1.0), material=MaterialParams(1.3e7, 800.0, 30.0, 0.5),
                       schedule=FieldSchedule([ScheduleStage(0, 100, (10.0, -20.0, 5.0))]), dt=5e-6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="skip the largest grids")
    a = ap.parse_args()
    for nx, ny, nz, prec, env in CASES:
        if a.quick and nx * ny * nz > 200_000:
            continue
        for k in ("MMB_GENERAL_PATH", "MMB_BIG_PATH"):
            os.environ.pop(k, None)
        os.environ.update(env)
        p = Precision.f64 if prec == "f64" else Precision.f32
        sim = make_simulation(spec(nx, ny, nz), precision=p)
        sim.set_magnetization(random_unit_field(nx, ny, nz, 800.0, 20240 + nx, p))
        sim.step(2)
        sim.effective_field()
        sim.synchronize()
        print("ok", sim.path_info(), flush=True)
    for (nx, ny, nz), world, prec, peer in SHARDED:
        os.environ["MMB_SHARD_PEER"] = peer
        os.environ.pop("MMB_GENERAL_PATH", None)
        if nz > 8:
            os.environ["MMB_BIG_PATH"] = "1"
        p = Precision.f64 if prec == "f64" else Precision.f32
        sim = make_emulated_sharded_simulation(spec(nx, ny, nz), p, world)
        sim.set_magnetization(random_unit_field(nx, ny, nz, 800.0, 20240 + nx, p))
        sim.step(2)
        sim.energy()
        sim.synchronize()
        print("ok", sim.path_info(), flush=True)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
