"""ctypes binding of libmmb.so (include/mmb.h). The product path has no CPU fallback: if the
library is missing or no CUDA device is usable, calls raise instead of degrading."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MMB_LIB", os.path.join(HERE, "libmmb.so"))  # override: variants

MMB_OK, MMB_ERROR_ARGUMENT, MMB_ERROR_CONFIG, MMB_ERROR_NUMERICAL = 0, 1, 2, 3
MMB_ERROR_IO, MMB_ERROR_NOMEM, MMB_ERROR_VALIDATION, MMB_ERROR_INTERNAL, MMB_ERROR_CUDA = 4, 5, 6, 7, 8
MMB_F32, MMB_F64 = 0, 1

EXPORTS = [
    "mmb_status_string", "mmb_last_error", "mmb_version", "mmb_create", "mmb_free", "mmb_set_m",
    "mmb_get_m", "mmb_step", "mmb_step_index", "mmb_average", "mmb_energy", "mmb_max_torque",
    "mmb_last_torque_sq", "mmb_run", "mmb_synchronize", "mmb_effective_field", "mmb_demag_field",
    "mmb_tensor_octant", "mmb_upload_tensor_octant", "mmb_time_steps", "mmb_profile_step",
    "mmb_launches_per_step", "mmb_device_bytes", "mmb_nccl_unique_id", "mmb_create_sharded",
    "mmb_create_emulated", "mmb_slab", "mmb_validate", "mmb_string_free", "mmb_path_info",
    "mmb_random_unit_field", "mmb_set_m_async", "mmb_get_m_async",
]


class MmbDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("delta", C.c_double),
        ("a_ex", C.c_double), ("ms", C.c_double), ("hk", C.c_double), ("alpha", C.c_double),
        ("dt", C.c_double),
        ("init_dir", C.c_double * 3),
        ("precision", C.c_int),
        ("device", C.c_int),
    ]


class MmbStage(C.Structure):
    _fields_ = [
        ("start", C.c_longlong), ("end", C.c_longlong),
        ("field", C.c_double * 3),
        ("ramp", C.c_int),
        ("field_end", C.c_double * 3),
        ("has_alpha", C.c_int),
        ("alpha_override", C.c_double),
    ]


RECORD_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_longlong, C.c_double, C.c_double, C.c_double)

_lib = None


class MmbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class NumericalError(MmbError):
    pass


def load():
    """Load libmmb.so (building it first when the sources are newer / it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    L = C.CDLL(LIB_PATH)
    vp, i, d, ll, sz = C.c_void_p, C.c_int, C.c_double, C.c_longlong, C.c_size_t
    for name, res in [("mmb_status_string", C.c_char_p), ("mmb_last_error", C.c_char_p),
                      ("mmb_version", C.c_char_p)]:
        getattr(L, name).restype = res
    L.mmb_status_string.argtypes = [i]
    L.mmb_create.argtypes = [C.POINTER(MmbDesc), C.POINTER(MmbStage), i, C.POINTER(vp)]
    L.mmb_free.argtypes = [vp]
    L.mmb_free.restype = None
    L.mmb_set_m.argtypes = [vp, vp, vp, vp]
    L.mmb_get_m.argtypes = [vp, vp, vp, vp]
    L.mmb_set_m_async.argtypes = [vp, vp, vp, vp]
    L.mmb_get_m_async.argtypes = [vp, vp, vp, vp]
    L.mmb_step.argtypes = [vp, ll]
    L.mmb_step_index.argtypes = [vp, C.POINTER(ll)]
    L.mmb_average.argtypes = [vp, C.POINTER(d)]
    L.mmb_energy.argtypes = [vp, C.POINTER(d)]
    L.mmb_max_torque.argtypes = [vp, C.POINTER(d)]
    L.mmb_last_torque_sq.argtypes = [vp, C.POINTER(d)]
    L.mmb_run.argtypes = [vp, ll, ll, d, RECORD_FN, vp, C.POINTER(ll)]
    L.mmb_synchronize.argtypes = [vp]
    L.mmb_effective_field.argtypes = [vp, vp, vp, vp]
    L.mmb_demag_field.argtypes = [vp] + [vp] * 6
    L.mmb_tensor_octant.argtypes = [vp, vp]
    L.mmb_upload_tensor_octant.argtypes = [vp, vp]
    L.mmb_time_steps.argtypes = [vp, ll, C.POINTER(C.c_float)]
    L.mmb_profile_step.argtypes = [vp, ll, C.POINTER(C.c_float), i, C.POINTER(i), C.c_char_p, sz]
    L.mmb_launches_per_step.argtypes = [vp, C.POINTER(i)]
    L.mmb_device_bytes.argtypes = [vp, C.POINTER(sz)]
    L.mmb_path_info.argtypes = [vp, C.c_char_p, sz]
    L.mmb_random_unit_field.argtypes = [C.c_uint, d, ll, ll, i, vp, vp, vp]
    L.mmb_nccl_unique_id.argtypes = [C.c_char_p]
    L.mmb_create_sharded.argtypes = [C.POINTER(MmbDesc), C.POINTER(MmbStage), i, i, i, C.c_char_p,
                                     C.POINTER(vp)]
    L.mmb_create_emulated.argtypes = [C.POINTER(MmbDesc), C.POINTER(MmbStage), i, i, C.POINTER(vp)]
    L.mmb_slab.argtypes = [vp, C.POINTER(i), C.POINTER(i)]
    L.mmb_validate.argtypes = [C.POINTER(C.c_void_p)]
    L.mmb_string_free.argtypes = [C.c_void_p]
    L.mmb_string_free.restype = None
    _lib = L
    return L


def check(rc: int):
    if rc != MMB_OK:
        L = load()
        msg = L.mmb_last_error().decode()
        if rc == MMB_ERROR_NUMERICAL:
            raise NumericalError(rc, msg)
        if rc == MMB_ERROR_ARGUMENT:
            raise ValueError(msg)
        if rc == MMB_ERROR_NOMEM:
            raise MemoryError(msg)
        raise MmbError(rc, f"{L.mmb_status_string(rc).decode()}: {msg}")
