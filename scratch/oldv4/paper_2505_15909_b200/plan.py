"""Selective per-layer / per-module precision (plan.hpp:84-110) via the C-ABI.

The grammar, resolution and effective-bits accounting are implemented once, in
C++ (csrc/dropin/plan.cpp); this module is the Python binding plus the
per-linear kernel choice (W4 or W8 variant) a decode stack needs.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

MODULES = ("qkv_proj", "attn_out_proj", "ffn_up", "ffn_down")  # ModuleId 1..4, types.hpp:46-51


def resolve(text: str, layers: int):
    """-> (table uint8[layers, 4] of 4/8, canonical text).  PlanError on bad input."""
    from . import _check, lib
    table = np.zeros(max(layers, 0) * 4, np.uint8)
    canon = C.create_string_buffer(1024)
    off = C.c_int64(-1)
    st = lib().rtnq_plan_resolve(text.encode(), layers, table.ctypes.data_as(C.c_void_p), canon,
                                 1024, C.byref(off))
    if st:
        from .errors import PlanError
        msg = lib().rtnq_last_error().decode()
        if st == 4:
            raise PlanError(msg, None if off.value < 0 else off.value)
        _check(st)
    return table.reshape(max(layers, 0), 4), canon.value.decode()


def canonical(text: str) -> str:
    return resolve(text, 0)[1]


def effective_bits(table, rows4, cols4, g=128, include_scales=False) -> float:
    from . import _check, lib
    t = np.ascontiguousarray(table, dtype=np.uint8).ravel()
    layers = t.size // 4
    r = np.ascontiguousarray(rows4, dtype=np.int64)
    c = np.ascontiguousarray(cols4, dtype=np.int64)
    out = C.c_double()
    _check(lib().rtnq_effective_bits(t.ctypes.data_as(C.c_void_p), layers,
                                     r.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p),
                                     g, int(include_scales), C.byref(out)))
    return out.value
