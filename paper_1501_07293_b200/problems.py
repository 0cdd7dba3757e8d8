"""Problem description types — Python mirror of the reference's host-side spec types.

Grid               proj/include/mmsim/grid.hpp:21-52
MaterialParams     proj/include/mmsim/material.hpp:13-34
ScheduleStage      proj/include/mmsim/schedule.hpp:14-27
FieldSchedule      proj/include/mmsim/schedule.hpp:36-48, proj/src/schedule.cpp:8-26
ProblemSpec        proj/include/mmsim/problems.hpp:15-24
standard_problem_4 proj/src/problems.cpp:7-42
standard_problem_3_benchmark proj/src/problems.cpp:44-58

Pure host data (no arithmetic on the hot path); validation messages and exception types
follow the reference (std::invalid_argument -> ValueError).
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

Vec3 = Tuple[float, float, float]

K_MU0 = 1.256636
K_GAMMA_MU0 = 0.221


@dataclass
class Grid:
    nx: int = 1
    ny: int = 1
    nz: int = 1
    delta: float = 1.0  # nm, cubic cells

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1 or self.nz < 1:
            raise ValueError("Grid: cell counts must be >= 1")
        if not self.delta > 0.0:
            raise ValueError("Grid: cell edge length must be > 0")

    def cell_count(self) -> int:
        return self.nx * self.ny * self.nz

    def index(self, i: int, j: int, k: int) -> int:
        return i + self.nx * (j + self.ny * k)

    def same_shape(self, o: "Grid") -> bool:
        return (self.nx, self.ny, self.nz) == (o.nx, o.ny, o.nz)

    @property
    def shape(self):  # numpy (z, y, x)
        return (self.nz, self.ny, self.nx)


@dataclass
class MaterialParams:
    a_ex: float = 0.0
    ms: float = 1.0
    hk: float = 0.0
    alpha: float = 1.0

    def validate(self):
        if not self.ms > 0.0:
            raise ValueError("MaterialParams: ms must be > 0")
        if self.a_ex < 0.0:
            raise ValueError("MaterialParams: a_ex must be >= 0")
        if self.hk < 0.0:
            raise ValueError("MaterialParams: hk must be >= 0")
        if not self.alpha > 0.0:
            raise ValueError("MaterialParams: alpha must be > 0")

    def exchange_coefficient(self, delta: float) -> float:
        return 2.0 * self.a_ex / (K_MU0 * self.ms * self.ms * delta * delta)

    def ku(self) -> float:
        return 0.5 * self.hk * K_MU0 * self.ms


@dataclass
class ScheduleStage:
    start: int = 0
    end: int = 0
    field: Vec3 = (0.0, 0.0, 0.0)
    ramp: bool = False
    field_end: Vec3 = (0.0, 0.0, 0.0)
    alpha_override: Optional[float] = None

    def value_at(self, step: int) -> Vec3:
        if not self.ramp:
            return tuple(self.field)
        f = float(step - self.start) / float(self.end - self.start)
        return tuple(a + f * (b - a) for a, b in zip(self.field, self.field_end))


class FieldSchedule:
    def __init__(self, stages: Optional[List[ScheduleStage]] = None):
        st = sorted((copy.copy(s) for s in (stages or [])), key=lambda s: s.start)
        for i, s in enumerate(st):
            if s.end <= s.start:
                raise ValueError("FieldSchedule: stage range must be nonempty")
            if i > 0 and s.start < st[i - 1].end:
                raise ValueError("FieldSchedule: stage ranges must be disjoint")
        self._stages = st

    def stages(self) -> List[ScheduleStage]:
        return self._stages

    def empty(self) -> bool:
        return not self._stages

    def at(self, step: int):
        for s in self._stages:
            if step < s.start:
                break
            if step < s.end:
                return s.value_at(step), s.alpha_override
        return (0.0, 0.0, 0.0), None


@dataclass
class ProblemSpec:
    name: str = ""
    grid: Grid = field(default_factory=Grid)
    material: MaterialParams = field(default_factory=MaterialParams)
    initial_direction: Vec3 = (1.0, 0.0, 0.0)
    schedule: FieldSchedule = field(default_factory=FieldSchedule)
    dt: float = 0.0
    steps: int = 0
    cadence: int = 1


def standard_problem_4() -> ProblemSpec:
    p = ProblemSpec(name="sp4", grid=Grid(166, 42, 1, 3.0),
                    material=MaterialParams(a_ex=1.3e7, ms=800.0, hk=0.0, alpha=0.5),
                    initial_direction=(1.0, 0.0, 0.0), dt=5e-6, steps=150000, cadence=1000)
    p.schedule = FieldSchedule([
        ScheduleStage(0, 4000, (100.0, 100.0, 100.0)),
        ScheduleStage(4000, 6000, (100.0, 100.0, 100.0), ramp=True, field_end=(0.0, 0.0, 0.0)),
        ScheduleStage(50001, p.steps + 1, (-19.576, 3.422, 0.0), alpha_override=0.02),
    ])
    return p


def standard_problem_3_benchmark(n: int) -> ProblemSpec:
    if n < 1:
        raise ValueError("standard_problem_3_benchmark: n must be >= 1")
    return ProblemSpec(name="sp3", grid=Grid(n, n, n, 1.0),
                       material=MaterialParams(a_ex=1e7, ms=1000.0, hk=100.0, alpha=0.5),
                       initial_direction=(1.0, 0.0, 0.0), dt=1e-5, steps=20000, cadence=100)
