"""Host-side mirror of the reference's simulation front end over the B200 C-ABI.

Simulation      <- mmsim::SimulationBase / Simulation<T>  proj/include/mmsim/llg.hpp:56-115
make_simulation <- mmsim::make_simulation                 proj/src/llg.cpp:163-168
RunOptions, TrajectoryRecord, Precision, Backend          proj/include/mmsim/llg.hpp:33-51,
                                                          proj/include/mmsim/backend.hpp:17

Every call goes through libmmb.so (include/mmb.h); the hot path is the sm_100a kernels in
csrc/. There is no CPU fallback: constructing a Simulation without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from .problems import ProblemSpec, Vec3


class Precision(enum.Enum):
    f32 = "f32"
    f64 = "f64"


class Backend(enum.Enum):
    serial = "serial"
    parallel = "parallel"
    b200 = "b200"


def precision_from_string(name: str) -> Precision:
    try:
        return Precision(name)
    except ValueError:
        raise ValueError(f"unknown precision '{name}' (expected f32 or f64)") from None


def backend_from_string(name: str) -> Backend:
    try:
        return Backend(name)
    except ValueError:
        raise ValueError(f"unknown backend '{name}' (expected serial, parallel or b200)") from None


@dataclass
class TrajectoryRecord:
    step: int = 0
    mx: float = 0.0
    my: float = 0.0
    mz: float = 0.0


@dataclass
class RunOptions:
    steps: int = 0
    cadence: int = 1
    sink: Optional[Callable[[TrajectoryRecord], None]] = None
    stop_torque: Optional[float] = None


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Simulation:
    """Simulation<T> on one B200: state (M ping-pong, spectral scratch, tensor spectrum) lives
    in HBM; step() enqueues one CUDA-graph replay of the fused per-step kernels."""

    def __init__(self, spec: ProblemSpec, precision: Precision = Precision.f64, device: int = 0,
                 _create=None):
        spec.material.validate()
        self._spec = spec
        self._precision = precision
        self.dtype = np.float64 if precision == Precision.f64 else np.float32
        L = _lib.load()
        g, m = spec.grid, spec.material
        desc = _lib.MmbDesc(g.nx, g.ny, g.nz, g.delta, m.a_ex, m.ms, m.hk, m.alpha, spec.dt,
                            (C.c_double * 3)(*spec.initial_direction),
                            _lib.MMB_F64 if precision == Precision.f64 else _lib.MMB_F32, device)
        stages = spec.schedule.stages()
        arr = (_lib.MmbStage * max(1, len(stages)))()
        for i, s in enumerate(stages):
            arr[i] = _lib.MmbStage(s.start, s.end, (C.c_double * 3)(*s.field), int(s.ramp),
                                   (C.c_double * 3)(*s.field_end), int(s.alpha_override is not None),
                                   float(s.alpha_override or 0.0))
        self._h = C.c_void_p()
        self._L = L
        if _create is None:
            _lib.check(L.mmb_create(C.byref(desc), arr, len(stages), C.byref(self._h)))
        else:
            _lib.check(_create(L, C.byref(desc), arr, len(stages), C.byref(self._h)))
        z0, nzl = C.c_int(), C.c_int()
        _lib.check(L.mmb_slab(self._h, C.byref(z0), C.byref(nzl)))
        self.z0, self.nz_local = z0.value, nzl.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.mmb_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- SimulationBase -------------------------------------------------------------------
    def step(self, n: int = 1) -> None:
        _lib.check(self._L.mmb_step(self._h, n))

    def run(self, opts: RunOptions) -> int:
        records: List[TrajectoryRecord] = []
        sink = opts.sink

        def cb(_u, step, mx, my, mz):
            if sink is not None:
                sink(TrajectoryRecord(step, mx, my, mz))

        fn = _lib.RECORD_FN(cb) if sink is not None else _lib.RECORD_FN()
        done = C.c_longlong()
        st = -1.0 if opts.stop_torque is None else float(opts.stop_torque)
        _lib.check(self._L.mmb_run(self._h, opts.steps, opts.cadence, st, fn, None, C.byref(done)))
        del records
        return done.value

    def step_index(self) -> int:
        v = C.c_longlong()
        _lib.check(self._L.mmb_step_index(self._h, C.byref(v)))
        return v.value

    def average_unit(self) -> Vec3:
        out = (C.c_double * 3)()
        _lib.check(self._L.mmb_average(self._h, out))
        return (out[0], out[1], out[2])

    def energy(self) -> float:
        v = C.c_double()
        _lib.check(self._L.mmb_energy(self._h, C.byref(v)))
        return v.value

    def max_torque(self) -> float:
        v = C.c_double()
        _lib.check(self._L.mmb_max_torque(self._h, C.byref(v)))
        return v.value

    def last_torque_sq(self) -> float:
        v = C.c_double()
        _lib.check(self._L.mmb_last_torque_sq(self._h, C.byref(v)))
        return v.value

    def spec(self) -> ProblemSpec:
        return self._spec

    def backend(self) -> Backend:
        return Backend.b200

    def precision(self) -> Precision:
        return self._precision

    # ---- state access (Simulation<T>::magnetization) ---------------------------------------
    def _shape(self):
        g = self._spec.grid
        return (3, self.nz_local, g.ny, g.nx)

    def magnetization(self) -> np.ndarray:
        out = np.empty(self._shape(), dtype=self.dtype)
        _lib.check(self._L.mmb_get_m(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def set_magnetization(self, m: np.ndarray) -> None:
        m = np.ascontiguousarray(m, dtype=self.dtype).reshape(self._shape())
        _lib.check(self._L.mmb_set_m(self._h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2])))

    def get_m_into(self, out: np.ndarray) -> None:
        """Device->host copy into a caller-owned (ideally pinned) array [3, nz, ny, nx]."""
        _lib.check(self._L.mmb_get_m(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))

    def set_m_from(self, m: np.ndarray) -> None:
        _lib.check(self._L.mmb_set_m(self._h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2])))

    def set_m_async(self, m: np.ndarray) -> None:
        """Stream-ordered upload from a caller-owned (ideally pinned) [3, nz, ny, nx] array that
        must stay valid and unchanged until synchronize()."""
        _lib.check(self._L.mmb_set_m_async(self._h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2])))

    def get_m_async(self, out: np.ndarray) -> None:
        """Stream-ordered download of the state at this point of the sequence into a
        caller-owned array, complete after synchronize()."""
        _lib.check(self._L.mmb_get_m_async(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))

    # ---- parity hooks -----------------------------------------------------------------------
    def effective_field(self) -> np.ndarray:
        out = np.empty(self._shape(), dtype=self.dtype)
        _lib.check(self._L.mmb_effective_field(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def demag_field(self, m: np.ndarray) -> np.ndarray:
        m = np.ascontiguousarray(m, dtype=self.dtype).reshape(self._shape())
        out = np.empty(self._shape(), dtype=self.dtype)
        _lib.check(self._L.mmb_demag_field(self._h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2]),
                                           _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out

    def tensor_octant(self) -> np.ndarray:
        g = self._spec.grid
        out = np.empty((6, g.nz, g.ny, g.nx), dtype=np.float64)
        _lib.check(self._L.mmb_tensor_octant(self._h, _ptr(out)))
        return out

    def upload_tensor_octant(self, entries: np.ndarray) -> None:
        e = np.ascontiguousarray(entries, dtype=np.float64)
        _lib.check(self._L.mmb_upload_tensor_octant(self._h, _ptr(e)))

    # ---- measurement -----------------------------------------------------------------------
    def synchronize(self):
        _lib.check(self._L.mmb_synchronize(self._h))

    def time_steps(self, n: int) -> float:
        v = C.c_float()
        _lib.check(self._L.mmb_time_steps(self._h, n, C.byref(v)))
        return v.value

    def profile_step(self, n: int):
        ms = (C.c_float * 16)()
        cnt = C.c_int()
        names = C.create_string_buffer(512)
        _lib.check(self._L.mmb_profile_step(self._h, n, ms, 16, C.byref(cnt), names, 512))
        return dict(zip(names.value.decode().split(";"), [ms[i] for i in range(cnt.value)]))

    def launches_per_step(self) -> int:
        v = C.c_int()
        _lib.check(self._L.mmb_launches_per_step(self._h, C.byref(v)))
        return v.value

    def device_bytes(self) -> int:
        v = C.c_size_t()
        _lib.check(self._L.mmb_device_bytes(self._h, C.byref(v)))
        return v.value

    def path_info(self) -> str:
        """The demag path and kernel variants (templates, tiles, grids) this handle runs."""
        buf = C.create_string_buffer(1024)
        _lib.check(self._L.mmb_path_info(self._h, buf, 1024))
        return buf.value.decode()


def random_unit_field(nx: int, ny: int, nz: int, ms: float, seed: int, precision: Precision = Precision.f64,
                      z0: int = 0, nz_local: Optional[int] = None) -> np.ndarray:
    """The reference's seeded random start (random_unit_field, proj/src/validate.cpp:21-39),
    generated by libmmb.so's host utility: [3, nz_local, ny, nx] for planes [z0, z0 + nz_local)
    of the global nx x ny x nz field."""
    nzl = nz - z0 if nz_local is None else nz_local
    plane = nx * ny
    dt = np.float64 if precision == Precision.f64 else np.float32
    out = np.empty((3, nzl, ny, nx), dtype=dt)
    _lib.check(_lib.load().mmb_random_unit_field(seed, ms, z0 * plane, nzl * plane,
                                                  _lib.MMB_F64 if precision == Precision.f64 else _lib.MMB_F32,
                                                  _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
    return out


def nccl_unique_id() -> bytes:
    """128-byte NCCL id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = C.create_string_buffer(128)
    _lib.check(_lib.load().mmb_nccl_unique_id(buf))
    return buf.raw


def make_sharded_simulation(spec: ProblemSpec, precision: Precision, rank: int, world: int,
                            nccl_id: bytes, device: int = 0) -> Simulation:
    """One rank of the z-slab decomposition (one process per GPU, NCCL exchanges). The
    handle's magnetization() / set_magnetization() cover its slab [z0, z0 + nz_local)."""
    def create(L, desc, arr, n, out):
        return L.mmb_create_sharded(desc, arr, n, rank, world, nccl_id, out)
    return Simulation(spec, precision, device, _create=create)


def make_emulated_sharded_simulation(spec: ProblemSpec, precision: Precision, world: int,
                                     device: int = 0) -> Simulation:
    """All `world` ranks of the decomposition on one device (device-copy exchanges)."""
    def create(L, desc, arr, n, out):
        return L.mmb_create_emulated(desc, arr, n, world, out)
    return Simulation(spec, precision, device, _create=create)


def make_simulation(spec: ProblemSpec, backend: Backend = Backend.b200,
                    precision: Precision = Precision.f64, device: int = 0) -> Simulation:
    """make_simulation (proj/src/llg.cpp:163-168). Only the b200 backend lives here; the
    reference's serial/parallel CPU backends are the reference itself."""
    if backend != Backend.b200:
        raise ValueError(f"backend '{backend.value}' is the reference CPU solver; this package "
                         "provides backend 'b200'")
    return Simulation(spec, precision, device)
