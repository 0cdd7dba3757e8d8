"""Device self-check suite (mmb_validate): the reference's `validate` verb
(mmsim_validate, proj/src/capi.cpp:286-298; run_validation, proj/src/validate.cpp:84-189)
evaluated on the B200 — tensor invariants from the device prism-sum kernel, the spectral
demag path against an O(N^2) device direct sum, linearity and shape factors."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List

from . import _lib


@dataclass
class ValidationReport:
    passed: bool
    text: str

    @property
    def lines(self) -> List[str]:
        return self.text.splitlines()

    def all_passed(self) -> bool:
        return self.passed


def run_validation() -> ValidationReport:
    L = _lib.load()
    out = C.c_void_p()
    rc = L.mmb_validate(C.byref(out))
    text = C.string_at(out.value).decode() if out.value else ""
    if out.value:
        L.mmb_string_free(out)
    if rc not in (_lib.MMB_OK, _lib.MMB_ERROR_VALIDATION):
        _lib.check(rc)
    return ValidationReport(rc == _lib.MMB_OK, text)
