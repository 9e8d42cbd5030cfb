"""ctypes binding of libpilc_sm100a.so (include/pilc.h).

The shared library is built in-tree by `__graft_entry__.build()` /
`make -C paper_2206_05279_b200/csrc`. There is no fallback: if the library is
missing or no sm_100 device is visible, the first GPU call raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PILC_LIB_PATH: an alternative build of the same library (A/B timing of
# kernel variants); the in-tree build by default
LIB_PATH = os.environ.get("PILC_LIB_PATH") or os.path.join(HERE, "libpilc_sm100a.so")

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64

# name -> (restype, argtypes)
_SIGS = {
    "pilc_version": (ctypes.c_char_p, []),
    "pilc_device_arch": (ctypes.c_int, []),
    "pilc_set_tuning": (ctypes.c_int, [I32, I32]),
    "pilc_twar_forward": (ctypes.c_int, [P, P, I64, I32, I32, P, P]),
    "pilc_twar_decode": (ctypes.c_int, [P, P, P, I64, I32, I32, P, P]),
    "pilc_rans_encode": (ctypes.c_int, [P, P, P, P, I64, I64, I32, P, I32, I32, I32, P, I64, P, P, P]),
    "pilc_rans_decode": (ctypes.c_int, [P, P, P, P, P, P, I64, I64, I32, P, I32, I32, P, P, P, P]),
    "pilc_model_floats": (I64, [I32, I32, I32, I32]),
    "pilc_model_pack": (ctypes.c_int, [P, I32, I32, I32, I32, P]),
    "pilc_vq_workspace_bytes": (I64, [I64, I32, I32, I32, I32, I32, I32]),
    "pilc_vq_encode": (ctypes.c_int, [P, I64, I32, I32, P, I32, I32, I32, I32, P, I64, P, P, P]),
    "pilc_vq_encode_exact": (ctypes.c_int, [P, I64, I32, I32, P, I32, I32, I32, I32, P, I64, P, P, P]),
    "pilc_vq_fast_decoder": (ctypes.c_int, [I32, I32, I32, I32, I32, I32]),
    "pilc_vq_argmin": (ctypes.c_int, [P, I64, P, I32, I32, I32, I32, P, P]),
    "pilc_vq_argmin_tc_workspace": (I64, [I64]),
    "pilc_vq_argmin_tc": (ctypes.c_int, [P, I64, P, I32, I32, I32, I32, P, I64, P, P]),
    "pilc_vq_decode": (ctypes.c_int, [P, I64, I32, I32, P, I32, I32, I32, I32, P, I32, P, I64, P, P, P, P, P]),
    "pilc_vq_decode_exact": (ctypes.c_int, [P, I64, I32, I32, P, I32, I32, I32, I32, P, I32, P, I64, P, P, P, P, P]),
    "pilc_static_scale": (ctypes.c_int, [P, I64, I64, P, I32, P, P]),
    "pilc_container_sizes": (ctypes.c_int, [P, P, I64, I32, I64, P, P, P]),
    "pilc_container_pack": (ctypes.c_int, [P, I32, P, P, I32, I64, I64, I32, P, I64, P, P, P, I64, P, P, P, P, P]),
    "pilc_container_parse": (ctypes.c_int, [P, P, I64, ctypes.c_uint64, ctypes.c_uint64, I32, P, P]),
    "pilc_container_lanes": (ctypes.c_int, [P, P, P, P, I64, I32, I32, I32, I32, P, P, P, P, P]),
    "pilc_container_summary": (ctypes.c_int, [P, P, P, I64, P, P]),
    "pilc_crc32": (ctypes.c_int, [P, P, P, I64, P, P]),
    "pilc_sched_crc": (ctypes.c_int, [P, P, I64, I64, P, P]),
    "pilc_prof_reset": (None, [I32]),
    "pilc_prof_launches": (I64, []),
    "pilc_prof_categories": (I32, []),
    "pilc_prof_name": (ctypes.c_char_p, [I32]),
    "pilc_prof_read": (ctypes.c_int, [I32, P, P, P]),
    "pilc_prof_count": (I64, []),
    "pilc_prof_record": (ctypes.c_int, [I64, P, P, P]),
}

# pilc_header (include/pilc.h), 72 bytes
HEADER_DTYPE = np.dtype(
    [
        ("status", "<i4"), ("aux", "<i4"),
        ("backend", "u1"), ("M", "u1"), ("pad_rule", "u1"), ("flags", "u1"),
        ("width", "<u4"), ("height", "<u4"),
        ("lanes", "<u2"), ("static_d", "<u2"), ("D", "<u2"), ("reserved", "<u2"),
        ("params_hash_off", "<u4"), ("model_hash_off", "<u4"),
        ("idx_table_off", "<u4"), ("res_table_off", "<u4"),
        ("sched_crc", "<u4"), ("payload_off", "<u4"), ("grid_crc", "<u4"),
        ("idx_bytes", "<u8"), ("res_bytes", "<u8"),
    ],
    align=True,
)
assert HEADER_DTYPE.itemsize == 72

# pilc_summary (include/pilc.h)
SUMMARY_DTYPE = np.dtype([("n_bad", "<i4"), ("uniform", "<i4"), ("h0", HEADER_DTYPE), ("grid", "u1", 2 + 8 * 256),
                          ("pad", "u1", 6)], align=True)
assert SUMMARY_DTYPE.itemsize == 2136

ST_NAMES = {
    0: "OK", 1: "TRUNCATED", 2: "BAD_MAGIC", 3: "BAD_VERSION", 4: "CRC", 5: "BAD_BACKEND",
    6: "BAD_M", 7: "BAD_PAD", 8: "BAD_FLAGS", 9: "BAD_DIMS", 10: "GRID_TRUNC", 11: "STATIC_D",
    12: "IDX_LENS", 13: "RES_LENS", 14: "PAYLOAD_LEN", 15: "GRID_EMPTY", 16: "GRID_VALUE",
    17: "GRID_ORDER", 18: "GRID_GEOM", 20: "LANE_HDR", 21: "LANE_TRUNC",
    22: "LANE_LEN", 23: "STATE_RANGE", 24: "UNDERFLOW", 25: "END_STATE", 26: "PARAMS_HASH",
    27: "MODEL_HASH",
}

_lib = None


class LibraryError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load the CUDA library (raises LibraryError if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise LibraryError(f"{name} failed with status {rc} ({['OK', 'E_ARG', 'E_CUDA', 'E_UNSUPPORTED'][rc] if rc < 4 else rc})")
    return rc


TUNE_BLOCK_FUSION = 0
TUNE_DEC_TRUNK = 1
TUNE_ENC_TRUNK = 2
TUNE_DEC_UPHEAD = 3


def set_tuning(key: int, value: int) -> int:
    """pilc_set_tuning: returns the previous value."""
    prev = load().pilc_set_tuning(key, value)
    if prev < 0:
        raise ValueError(f"unknown tuning key {key}")
    return prev


def prof_reset(timing: bool) -> None:
    load().pilc_prof_reset(1 if timing else 0)


def prof_launches() -> int:
    return int(load().pilc_prof_launches())


def prof_read() -> dict:
    """{kernel: (launches, total_ms, work_units)} since the last reset."""
    lib = load()
    out = {}
    for c in range(lib.pilc_prof_categories()):
        n, ms, u = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        call("pilc_prof_read", c, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(u))
        if n.value:
            out[lib.pilc_prof_name(c).decode()] = (n.value, ms.value, u.value)
    return out


def prof_records() -> list:
    """[(kernel, ms, work_units)] per launch, in launch order."""
    lib = load()
    out = []
    for i in range(lib.pilc_prof_count()):
        c, ms, u = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
        call("pilc_prof_record", i, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(u))
        out.append((lib.pilc_prof_name(c.value).decode(), ms.value, u.value))
    return out


def version() -> str:
    return load().pilc_version().decode()
