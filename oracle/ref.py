"""oracle/ref.py — TEST INFRASTRUCTURE ONLY: ctypes access to the UNMODIFIED reference solver
compiled in place (oracle/Makefile -> oracle/_ref/libmmsim_ref.so, reference sources +
FFTW-API shim + oracle/ref_driver.cpp). Used by tests/ as the parity checker and by
bench.py's reference / cpu_baseline arm. Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libmmsim_ref.so")
REFERENCE_ROOT = "/root/reference/proj"


class RefProblem(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("delta", C.c_double),
        ("a_ex", C.c_double), ("ms", C.c_double), ("hk", C.c_double), ("alpha", C.c_double),
        ("dt", C.c_double),
        ("init_x", C.c_double), ("init_y", C.c_double), ("init_z", C.c_double),
        ("nstages", C.c_int),
        ("start", C.POINTER(C.c_longlong)), ("end", C.POINTER(C.c_longlong)),
        ("field", C.POINTER(C.c_double)), ("ramp", C.POINTER(C.c_int)),
        ("field_end", C.POINTER(C.c_double)), ("has_alpha", C.POINTER(C.c_int)),
        ("alpha_override", C.POINTER(C.c_double)),
    ]


RECORD_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_longlong, C.c_double, C.c_double, C.c_double)

_lib = None


def build() -> bool:
    """Build oracle/_ref from /root/reference when the sources are present (this container).
    On the GPU box the prebuilt .so travels with the repo snapshot."""
    if os.path.exists(REFERENCE_ROOT):
        subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)
    return os.path.exists(LIB_PATH)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp, i, d, ll = C.c_void_p, C.c_int, C.c_double, C.c_longlong
        P = C.POINTER(RefProblem)
        L.ref_last_error.restype = C.c_char_p
        L.ref_sim_create.argtypes = [P, i, i, C.POINTER(vp)]
        L.ref_sim_free.argtypes = [vp]
        L.ref_sim_set_m.argtypes = [vp, vp, vp, vp]
        L.ref_sim_get_m.argtypes = [vp, vp, vp, vp]
        L.ref_sim_step.argtypes = [vp, ll]
        L.ref_sim_step_index.argtypes = [vp]
        L.ref_sim_step_index.restype = ll
        L.ref_sim_average.argtypes = [vp, C.POINTER(d)]
        L.ref_sim_energy.argtypes = [vp, C.POINTER(d)]
        L.ref_sim_max_torque.argtypes = [vp, C.POINTER(d)]
        L.ref_sim_run.argtypes = [vp, ll, ll, d, RECORD_FN, vp, C.POINTER(ll)]
        L.ref_heff.argtypes = [P, i, C.POINTER(d), i, vp, vp, vp, vp, vp, vp]
        L.ref_demag_direct.argtypes = [P] + [vp] * 6
        L.ref_tensor_entry.argtypes = [i, i, i, d, C.POINTER(d)]
        L.ref_build_tensor.argtypes = [i, i, i, d, vp]
        L.ref_random_unit_field.argtypes = [ll, d, C.c_uint, vp, vp, vp]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


class Problem:
    """Flat problem description (grid, material, dt, schedule) shared by the reference driver,
    the NumPy restatement and the B200 product API in tests."""

    def __init__(self, nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, stages=(), init=(1.0, 0.0, 0.0)):
        self.nx, self.ny, self.nz, self.delta = nx, ny, nz, delta
        self.a_ex, self.ms, self.hk, self.alpha, self.dt = a_ex, ms, hk, alpha, dt
        self.stages = list(stages)
        self.init = tuple(init)
        self._keep = []

    @property
    def n(self):
        return self.nx * self.ny * self.nz

    def c_struct(self) -> RefProblem:
        ns = len(self.stages)
        arr = lambda t, v: (t * max(1, len(v)))(*v)  # noqa: E731
        start = arr(C.c_longlong, [s.start for s in self.stages])
        end = arr(C.c_longlong, [s.end for s in self.stages])
        field = arr(C.c_double, [x for s in self.stages for x in s.field])
        ramp = arr(C.c_int, [int(s.ramp) for s in self.stages])
        fend = arr(C.c_double, [x for s in self.stages for x in s.field_end])
        has = arr(C.c_int, [int(s.alpha_override is not None) for s in self.stages])
        aov = arr(C.c_double, [s.alpha_override or 0.0 for s in self.stages])
        self._keep = [start, end, field, ramp, fend, has, aov]
        return RefProblem(self.nx, self.ny, self.nz, self.delta, self.a_ex, self.ms, self.hk,
                          self.alpha, self.dt, *self.init, ns, start, end, field, ramp, fend,
                          has, aov)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class RefSimulation:
    """The reference's Simulation<T> (proj/src/llg.cpp) driven through oracle/ref_driver.cpp."""

    def __init__(self, prob: Problem, precision: str = "f64", backend: str = "serial"):
        self.prob = prob
        self.dtype = np.float64 if precision == "f64" else np.float32
        self._h = C.c_void_p()
        st = prob.c_struct()
        _check(lib().ref_sim_create(C.byref(st), int(precision == "f64"), int(backend == "parallel"),
                                    C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().ref_sim_free(self._h)
            self._h = C.c_void_p()

    def shape(self):
        return (self.prob.nz, self.prob.ny, self.prob.nx)

    def set_m(self, m: np.ndarray):
        m = np.ascontiguousarray(m, dtype=self.dtype).reshape(3, -1)
        _check(lib().ref_sim_set_m(self._h, _ptr(m[0]), _ptr(m[1]), _ptr(m[2])))

    def get_m(self) -> np.ndarray:
        out = np.empty((3, self.prob.n), dtype=self.dtype)
        _check(lib().ref_sim_get_m(self._h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2])))
        return out.reshape((3,) + self.shape())

    def step(self, n: int = 1):
        _check(lib().ref_sim_step(self._h, n))

    def step_index(self) -> int:
        return lib().ref_sim_step_index(self._h)

    def average_unit(self):
        out = (C.c_double * 3)()
        _check(lib().ref_sim_average(self._h, out))
        return tuple(out)

    def energy(self) -> float:
        v = C.c_double()
        _check(lib().ref_sim_energy(self._h, C.byref(v)))
        return v.value

    def max_torque(self) -> float:
        v = C.c_double()
        _check(lib().ref_sim_max_torque(self._h, C.byref(v)))
        return v.value

    def run(self, steps: int, cadence: int = 1, stop_torque: Optional[float] = None, records=None) -> int:
        recs = records if records is not None else []

        def cb(_u, step, mx, my, mz):
            recs.append((step, mx, my, mz))

        fn = RECORD_FN(cb)
        done = C.c_longlong()
        _check(lib().ref_sim_run(self._h, steps, cadence, -1.0 if stop_torque is None else stop_torque,
                                 fn, None, C.byref(done)))
        return done.value


def heff(prob: Problem, m: np.ndarray, applied=(0.0, 0.0, 0.0), parts: int = 15) -> np.ndarray:
    """H_eff as llg.cpp:52-55 assembles it (parts bitmask: 1 demag, 2 exchange, 4 anisotropy,
    8 applied)."""
    dtype = m.dtype
    m = np.ascontiguousarray(m).reshape(3, -1)
    h = np.empty_like(m)
    st = prob.c_struct()
    app = (C.c_double * 3)(*applied)
    _check(lib().ref_heff(C.byref(st), int(dtype == np.float64), app, parts, _ptr(m[0]), _ptr(m[1]),
                          _ptr(m[2]), _ptr(h[0]), _ptr(h[1]), _ptr(h[2])))
    return h.reshape((3, prob.nz, prob.ny, prob.nx))


def demag_direct(prob: Problem, m: np.ndarray) -> np.ndarray:
    m = np.ascontiguousarray(m, dtype=np.float64).reshape(3, -1)
    h = np.empty_like(m)
    st = prob.c_struct()
    _check(lib().ref_demag_direct(C.byref(st), _ptr(m[0]), _ptr(m[1]), _ptr(m[2]), _ptr(h[0]),
                                  _ptr(h[1]), _ptr(h[2])))
    return h.reshape((3, prob.nz, prob.ny, prob.nx))


def tensor_entry(I, J, K, delta):
    out = (C.c_double * 6)()
    _check(lib().ref_tensor_entry(I, J, K, delta, out))
    return tuple(out)


def build_tensor(nx, ny, nz, delta) -> np.ndarray:
    out = np.empty((6, 2 * nz, 2 * ny, 2 * nx))
    _check(lib().ref_build_tensor(nx, ny, nz, delta, _ptr(out)))
    return out


def random_unit_field(nx, ny, nz, ms, seed, dtype=np.float64) -> np.ndarray:
    """The reference's seeded random start (proj/src/validate.cpp:21-39): mt19937 + libstdc++
    uniform_real_distribution(-1, 1), computed in f64 and cast to T."""
    n = nx * ny * nz
    out = np.empty((3, n))
    lib().ref_random_unit_field(n, ms, seed, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return out.astype(dtype).reshape((3, nz, ny, nx))
