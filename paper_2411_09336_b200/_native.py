"""ctypes binding of libmpskq.so (the C ABI declared in include/mpskq.h).

The library is loaded from the package directory; there is no fallback: if
it is missing the import of every GPU entry point fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# MPSKQ_LIB overrides the in-tree library (A/B experiments only)
LIB_PATH = Path(os.environ.get("MPSKQ_LIB") or Path(__file__).resolve().parent / "libmpskq.so")

OK = 0
ERR_INVALID = -1
ERR_CUDA = -2
ERR_CAPACITY = -3
ERR_NUMERIC = -4
ERR_NOMEM = -5
STATE_OK, STATE_CAPACITY, STATE_NONFINITE, STATE_NOCONV = 0, 1, 2, 3
OP_H, OP_RZ, OP_RXX, OP_SWAP, OP_QRL, OP_QRR, OP_U1, OP_U2 = 1, 2, 3, 4, 5, 6, 7, 8
ABSORB_LEFT = 1

GATE_H, GATE_RZ, GATE_RXX, GATE_SWAP = 0, 1, 2, 3
KIND_TRAIN, KIND_TEST = 0, 1
OUT_KERNEL, OUT_AMPLITUDE = 0, 1

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p

_SIGNATURES = {
    "mpskq_abi_version": (C.c_int, []),
    "mpskq_last_error": (C.c_char_p, []),
    "mpskq_device_count": (C.c_int, []),
    "mpskq_feature_map_topology": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _i32p, C.c_int64, _i64p, _i64p],
    ),
    "mpskq_feature_map_angles": (
        C.c_int,
        [_f64p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double, _f64p],
    ),
    "mpskq_feature_map_coefficients_device": (
        C.c_int,
        [_vp, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double, _vp, _vp, _vp],
    ),
    "mpskq_half_angle_coefficients": (C.c_int, [_f64p, C.c_int64, _f64p]),
    "mpskq_program_compile": (
        C.c_int,
        [C.c_int, C.c_int64, _i32p, _i32p, _i32p, _i32p, _i32p, C.c_int64, _i64p, _i64p, _i64p],
    ),
    "mpskq_batch_layout": (C.c_int, [C.c_int, C.c_int, _i64p, _i64p]),
    "mpskq_supported_chi_caps": (C.c_int, [_i32p, C.c_int, C.POINTER(C.c_int)]),
    "mpskq_simulate": (
        C.c_int,
        [C.c_int, C.c_int, _vp, C.c_int64, C.c_int64, _vp, C.c_int64, C.c_int64, C.c_double,
         C.c_int, _vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "mpskq_run_program": (
        C.c_int,
        [C.c_int, C.c_int, _vp, C.c_int64, C.c_int64, _vp, C.c_int64, C.c_int64, C.c_double,
         C.c_int, _vp, C.c_int64, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "mpskq_relayout": (
        C.c_int,
        [C.c_int, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp, _vp, C.c_int64, _vp, _vp],
    ),
    "mpskq_svd_truncated_batched": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int64, _vp, C.c_double, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "mpskq_overlap": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp,
         C.c_int64, C.c_int, C.c_int, _vp, C.c_int64, _vp],
    ),
    "mpskq_pack_exact": (C.c_int, [C.c_int, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp, _vp, _vp]),
    "mpskq_unpack_exact": (C.c_int, [C.c_int, C.c_int64, _vp, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp]),
    "mpskq_owned_rows": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_int, _i64p]),
    "mpskq_overlap_owned_rows": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp, C.c_int64, C.c_int, C.c_int,
         _vp, _vp, _vp, _vp],
    ),
    "mpskq_assemble_rows": (
        C.c_int,
        [C.c_int, C.c_int64, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp],
    ),
    "mpskq_overlap_host": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp, _vp],
    ),
    "mpskq_overlap_tiles": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int, _i32p, C.c_int64, _i64p, _i32p, _i32p],
    ),
    "mpskq_gram_host": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _f64p,
         C.c_int64, _f64p, C.c_int64, _f64p, _vp, _f64p],
    ),
    "mpskq_sm_clock_khz": (C.c_int, []),
    "mpskq_fp64_probe": (C.c_int, [C.c_int, C.c_int64, _vp, _vp]),
}

_lib = None


def lib():
    """The loaded library (built in-tree by paper_2411_09336_b200.build)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2411_09336_b200.build` "
                "(the GPU path has no CPU fallback)"
            )
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.mpskq_abi_version() != 1:
            raise RuntimeError("libmpskq ABI version mismatch")
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(status: int) -> None:
    """Map a C status to the reference's exception types."""
    if status == OK:
        return
    msg = (lib().mpskq_last_error() or b"").decode(errors="replace")
    if status in (ERR_INVALID, ERR_NUMERIC):
        raise ValueError(msg)
    if status == ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libmpskq status {status}: {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def supported_chi_caps() -> list[int]:
    buf = np.zeros(16, dtype=np.int32)
    n = C.c_int(0)
    check(lib().mpskq_supported_chi_caps(ptr(buf, C.c_int32), 16, C.byref(n)))
    return [int(x) for x in buf[: n.value]]
