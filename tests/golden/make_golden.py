"""Generates the committed golden fixtures under tests/golden/ from the reference itself
(compiled in place by oracle/Makefile -> oracle/_ref/libmmsim_ref.so; needs /root/reference,
i.e. run in the build container, never on the GPU box).

    python tests/golden/make_golden.py fields            # small H_eff / step vectors (seconds)
    python tests/golden/make_golden.py traj sp4_128_f64  # full SP#4 trajectories (minutes)
    python tests/golden/make_golden.py fixture           # copy of the reference's own SP#4 TSV
    python tests/golden/make_golden.py film film256_f32  # 256x256x1 film relaxation (~45 min)
    python tests/golden/make_golden.py crit6             # acceptance criterion 6 energies (minutes)

Trajectory runs replay the reference's Simulation<T>::run exactly (proj/src/llg.cpp:110-124)
with cadence 1000 and record <m> with %.17g so the B200 run can be compared at 1e-6.
"""
from __future__ import annotations

import os
import shutil
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import mmsim_oracle as O  # noqa: E402
from oracle import ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name -> (nx, ny, nz, delta, precision)
TRAJ = {
    "sp4_166_f64": (166, 42, 1, 3.0, "f64"),
    "sp4_166_f32": (166, 42, 1, 3.0, "f32"),
    "sp4_128_f64": (128, 32, 1, 3.90625, "f64"),
    "sp4_128_f32": (128, 32, 1, 3.90625, "f32"),
}

# Small grids for field/step vectors: (nx, ny, nz, delta, a_ex, ms, hk, alpha, applied, seed)
FIELD_CASES = [
    (1, 1, 1, 2.0, 0.0, 800.0, 0.0, 0.5, (50.0, 0.0, 0.0), 1),
    (7, 1, 1, 1.0, 1.3e7, 800.0, 0.0, 0.5, (0.0, 0.0, 0.0), 2),
    (1, 6, 2, 1.0, 1.3e7, 800.0, 20.0, 0.5, (5.0, -3.0, 1.0), 3),
    (5, 3, 2, 3.0, 1.3e7, 800.0, 0.0, 0.5, (-19.576, 3.422, 0.0), 4),
    (8, 8, 4, 1.0, 1e7, 1000.0, 100.0, 0.5, (0.0, 0.0, 0.0), 5),
    (16, 12, 3, 2.5, 1.3e7, 800.0, 40.0, 0.3, (10.0, 20.0, -5.0), 6),
    (33, 17, 1, 3.0, 1.3e7, 800.0, 0.0, 0.5, (100.0, 100.0, 100.0), 7),
]


def sp4_problem(nx, ny, nz, delta):
    g, mat, dt, stages, steps, cad = O.standard_problem_4()
    return ref.Problem(nx, ny, nz, delta, mat.a_ex, mat.ms, mat.hk, mat.alpha, dt, stages), steps, cad


def make_fixture():
    src = "/root/reference/proj/tests/fixtures/sp4_field1_reference.tsv"
    shutil.copyfile(src, os.path.join(HERE, "sp4_field1_reference.tsv"))
    print("copied", src)


def make_fields():
    out = {}
    for idx, (nx, ny, nz, delta, a_ex, ms, hk, alpha, applied, seed) in enumerate(FIELD_CASES):
        stage = O.Stage(0, 1_000_000, applied)
        P = ref.Problem(nx, ny, nz, delta, a_ex, ms, hk, alpha, 5e-6, [stage])
        for prec in ("f64", "f32"):
            dt = np.float64 if prec == "f64" else np.float32
            m = ref.random_unit_field(nx, ny, nz, ms, 20240 + nx + seed, dt)
            h = ref.heff(P, m, applied)
            sim = ref.RefSimulation(P, prec)
            sim.set_m(m)
            sim.step(10)
            key = f"c{idx}_{prec}"
            out[key + "_m0"] = m
            out[key + "_heff"] = h
            out[key + "_m10"] = sim.get_m()
            out[key + "_avg10"] = np.array(sim.average_unit())
    out["cases"] = np.array([list(c[:8]) + list(c[8]) + [c[9]] for c in FIELD_CASES], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "fields_small.npz"), **out)
    print("wrote fields_small.npz", len(out))


# BASELINE configs[1]: 256x256x1 film, SURVEY.md §8(d) input (2): SP#3 overrides nx=ny=256, nz=1,
# delta=3, a_ex=1.3e7, ms=800, hk=0, alpha=0.5, dt=5e-6, no field; random start from the
# reference generator (proj/src/validate.cpp:21-39) with seed 20240 + nx; 20 000 steps at
# cadence 100.
FILM = {"film256_f32": "f32", "film256_f64": "f64"}
FILM_STEPS, FILM_CADENCE = 20000, 100


def film_problem():
    return ref.Problem(256, 256, 1, 3.0, 1.3e7, 800.0, 0.0, 0.5, 5e-6, [])


def make_film(name):
    prec = FILM[name]
    P = film_problem()
    sim = ref.RefSimulation(P, prec, backend="parallel")
    sim.set_m(ref.random_unit_field(256, 256, 1, 800.0, 20240 + 256, np.float64 if prec == "f64" else np.float32))
    recs = []
    t0 = time.time()
    sim.run(FILM_STEPS, FILM_CADENCE, records=recs)
    path = os.path.join(HERE, f"traj_{name}.tsv")
    with open(path, "w") as f:
        f.write(f"# reference Simulation<{'double' if prec == 'f64' else 'float'}>::run, film 256x256x1 delta=3 "
                f"a_ex=1.3e7 ms=800 hk=0 alpha=0.5 dt=5e-6, random_unit_field seed 20496, cadence "
                f"{FILM_CADENCE}, shim FFT; {time.time() - t0:.0f}s\n")
        for s_, mx, my, mz in recs:
            f.write(f"{s_}\t{mx:.17g}\t{my:.17g}\t{mz:.17g}\n")
    print("wrote", path, len(recs), f"{time.time() - t0:.0f}s")


def make_crit6():
    """Acceptance criterion 6 (proj/tests/acceptance.cpp:307-336): SP#3 16^3 f64 from uniform
    +x, energy after each of 200 bursts of 100 steps, final max torque."""
    P = ref.Problem(16, 16, 16, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5, [])
    sim = ref.RefSimulation(P, "f64")
    rows = [(0, sim.energy()) + sim.average_unit()]
    for _ in range(200):
        sim.run(100, 0)
        rows.append((sim.step_index(), sim.energy()) + sim.average_unit())
    path = os.path.join(HERE, "crit6_sp3_16_f64.tsv")
    with open(path, "w") as f:
        f.write(f"# reference Simulation<double> SP#3 16^3 (criterion 6): step, energy, <m>; final max_torque "
                f"{sim.max_torque():.17g}\n")
        for r in rows:
            f.write("\t".join([str(r[0])] + [f"{v:.17g}" for v in r[1:]]) + "\n")
    print("wrote", path, len(rows))


def make_traj(name):
    nx, ny, nz, delta, prec = TRAJ[name]
    P, steps, cad = sp4_problem(nx, ny, nz, delta)
    sim = ref.RefSimulation(P, prec)
    recs = []
    t0 = time.time()
    sim.run(steps, cad, records=recs)
    path = os.path.join(HERE, f"traj_{name}.tsv")
    with open(path, "w") as f:
        f.write(f"# reference Simulation<{ 'double' if prec == 'f64' else 'float'}>::run, SP#4 "
                f"{nx}x{ny}x{nz} delta={delta}, dt=5e-6, cadence {cad}, shim FFT; "
                f"{time.time() - t0:.0f}s\n")
        for s, mx, my, mz in recs:
            f.write(f"{s}\t{mx:.17g}\t{my:.17g}\t{mz:.17g}\n")
    print("wrote", path, len(recs), f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "fields"
    if what == "fields":
        make_fields()
    elif what == "fixture":
        make_fixture()
    elif what == "film":
        for n in sys.argv[2:] or list(FILM):
            make_film(n)
    elif what == "crit6":
        make_crit6()
    elif what == "traj":
        for n in sys.argv[2:] or list(TRAJ):
            make_traj(n)
    else:
        raise SystemExit(f"unknown target {what}")
