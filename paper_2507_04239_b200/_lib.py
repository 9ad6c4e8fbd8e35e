"""ctypes binding of the C ABI in include/power_attention_b200.h.

The product path has exactly one implementation: the in-tree CUDA library
``libpa_b200.so``.  If it is missing or no CUDA device is present, every call
raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import InvalidSpec, KernelError, OddPowerWithNormalize, ShapeMismatch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PA_B200_LIB") or os.path.join(HERE, "libpa_b200.so")

PA_F32, PA_BF16, PA_F16, PA_F64 = 0, 1, 2, 3
PA_FLAG_DETERMINISTIC, PA_FLAG_STRICT_TC, PA_FLAG_KEY_SUM = 1, 2, 4

_ERRORS = {
    1: InvalidSpec,
    2: ShapeMismatch,
    3: KernelError,
    4: InvalidSpec,
    5: KernelError,
    6: OddPowerWithNormalize,
}


class PaSpPart(ctypes.Structure):
    """pa_sp_part: this rank's chunk range inside the whole sequence."""

    _fields_ = [("chunk0", ctypes.c_int32), ("nchunks", ctypes.c_int32)]


class PaProblem(ctypes.Structure):
    _fields_ = [
        ("b", ctypes.c_int32),
        ("t", ctypes.c_int32),
        ("h", ctypes.c_int32),
        ("d", ctypes.c_int32),
        ("e", ctypes.c_int32),
        ("p", ctypes.c_int32),
        ("chunk", ctypes.c_int32),
        ("normalize", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("gated", ctypes.c_int32),
        ("has_scale", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("scale", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()

_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_PP = ctypes.POINTER(PaProblem)

_SIGS = {
    "pa_feature_dim": (_I64, [_I32, _I32]),
    "pa_feature_table": (ctypes.c_int, [_I32, _I32, _VP, _VP]),
    "pa_uses_tensor_cores": (ctypes.c_int, [_PP]),
    "pa_expansion_dim": (_I64, [_I32, _I32, _I32, _I32]),
    "pa_expansion_table": (ctypes.c_int, [_I32, _I32, _I32, _I32, _VP, _VP]),
    "pa_update_state_table": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I64, _I32, _VP, _VP, _VP, _VP, _VP,
                                              _VP, _VP, _I32, _VP]),
    "pa_query_state_table": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I64, _I32, _VP, _VP, _VP, _VP, _VP,
                                             _VP, _VP, _I32, _VP]),
    "pa_fwd_workspace_bytes": (_SZ, [_PP]),
    "pa_bwd_workspace_bytes": (_SZ, [_PP]),
    "pa_power_full_fwd": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "pa_power_full_bwd": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                          _VP, _VP, _VP, _SZ, _VP]),
    "pa_power_logspace_fwd": (ctypes.c_int, [_PP, ctypes.c_double, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "pa_fwd_zero_denominators": (ctypes.c_int, [_PP, _VP, _VP, ctypes.POINTER(_I32)]),
    "pa_update_state": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _VP, _VP, _VP, _VP,
                                        _VP, _I32, _VP]),
    "pa_query_state": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _VP, _VP, _VP, _VP,
                                       _VP, _I32, _VP]),
    "pa_discumsum": (ctypes.c_int, [_I32, _I64, _I64, _I32, _VP, _VP, _VP, _VP]),
    "pa_profile_enable": (ctypes.c_int, [_I32]),
    "pa_profile_reset": (None, []),
    "pa_profile_read": (ctypes.c_int, [_VP, _VP, _VP, _I32]),
    "pa_sp_state_floats": (_SZ, [_PP]),
    "pa_sp_fwd_local": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP, _VP]),
    "pa_sp_fwd_finish": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP, _VP]),
    "pa_sp_bwd_local": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _SZ, _VP,
                                        _VP]),
    "pa_sp_bwd_finish": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                         _VP, _VP, _SZ, _VP, _VP]),
    "pa_sp_combine": (ctypes.c_int, [_PP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "pa_last_error": (ctypes.c_char_p, []),
    "pa_launch_count": (_I64, []),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load (once) and return the CUDA library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise KernelError(
                    f"CUDA library {path} is not built; run "
                    "`python -m paper_2507_04239_b200.build` (no CPU fallback exists)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().pa_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, KernelError)(f"{what}: {msg}")


def launch_count() -> int:
    return int(load().pa_launch_count())


def profile_enable(on: bool) -> None:
    load().pa_profile_enable(1 if on else 0)


def profile_reset() -> None:
    load().pa_profile_reset()


def profile_read() -> dict:
    """{stage: (milliseconds, launches)} accumulated since the last reset."""
    import numpy as np

    cap = 64
    names = ctypes.create_string_buffer(32 * cap)
    ms = np.zeros(cap, dtype=np.float64)
    cnt = np.zeros(cap, dtype=np.int64)
    n = load().pa_profile_read(names, ms.ctypes.data_as(ctypes.c_void_p),
                               cnt.ctypes.data_as(ctypes.c_void_p), cap)
    raw = names.raw
    out = {}
    for i in range(n):
        nm = raw[32 * i: 32 * i + 32].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out
