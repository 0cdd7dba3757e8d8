"""Shared builders: one problem description -> the B200 Simulation and the reference oracle."""
import numpy as np

from oracle import mmsim_oracle as O
from paper_1501_07293_b200 import (FieldSchedule, Grid, MaterialParams, Precision, ProblemSpec,
                                   ScheduleStage, make_simulation)


def spec(nx, ny, nz, delta, a_ex=1.3e7, ms=800.0, hk=0.0, alpha=0.5, dt=5e-6, stages=(),
         init=(1.0, 0.0, 0.0)):
    return ProblemSpec(name="t", grid=Grid(nx, ny, nz, delta),
                       material=MaterialParams(a_ex, ms, hk, alpha), initial_direction=init,
                       schedule=FieldSchedule([ScheduleStage(*s) if isinstance(s, tuple) else s
                                               for s in stages]), dt=dt, steps=0, cadence=1)


def b200(sp, prec="f64"):
    return make_simulation(sp, precision=Precision.f64 if prec == "f64" else Precision.f32)


def ref_problem(ref, sp):
    g, m = sp.grid, sp.material
    stages = [O.Stage(s.start, s.end, tuple(s.field), s.ramp, tuple(s.field_end), s.alpha_override)
              for s in sp.schedule.stages()]
    return ref.Problem(g.nx, g.ny, g.nz, g.delta, m.a_ex, m.ms, m.hk, m.alpha, sp.dt, stages,
                       init=tuple(sp.initial_direction))


def sp4(nx=166, ny=42, delta=3.0):
    stages = [ScheduleStage(0, 4000, (100.0, 100.0, 100.0)),
              ScheduleStage(4000, 6000, (100.0, 100.0, 100.0), True, (0.0, 0.0, 0.0)),
              ScheduleStage(50001, 150001, (-19.576, 3.422, 0.0), alpha_override=0.02)]
    return spec(nx, ny, 1, delta, 1.3e7, 800.0, 0.0, 0.5, 5e-6, stages)


def octant_from_shifted(t, nx, ny, nz):
    """Reference shifted tensor [6][2nz][2ny][2nx] -> non-negative octant [6][nz][ny][nx]."""
    return np.ascontiguousarray(t[:, nz - 1: 2 * nz - 1, ny - 1: 2 * ny - 1, nx - 1: 2 * nx - 1])


def rel(a, b):
    return O.max_relative_error(a, b)
