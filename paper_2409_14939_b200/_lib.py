"""ctypes binding of libfastgl_b200.so (the C ABI in include/fastgl_b200.h).

The library is built in-tree (``python -m paper_2409_14939_b200._build`` or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or a call fails, the error propagates.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import CapacityError, ConfigError, MiniGLError, NotFoundError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "libfastgl_b200.so"

FGL_OK = 0
_ERRORS = {
    -1: ValidationError,
    -2: CapacityError,
    -3: NotFoundError,
    -4: ConfigError,
    -5: MiniGLError,
    -6: ConfigError,
}

c_i32p = C.POINTER(C.c_int32)
c_i64p = C.POINTER(C.c_int64)
vp = C.c_void_p


class FglGraph(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int64),
        ("num_edges", C.c_int64),
        ("row_offsets", vp),
        ("col_indices", vp),
        ("edge_weights", vp),
    ]


class FglSampleOut(C.Structure):
    _fields_ = [
        ("tgt", vp), ("src", vp), ("wgt", vp), ("edge_cap", C.c_int64),
        ("tgt_row", vp), ("src_row", vp), ("tgt_front", vp), ("src_front", vp),
        ("unique_nodes", vp), ("unique_cap", C.c_int64),
        ("frontier", vp), ("frontier_stride", C.c_int64),
        ("seed_rows", vp), ("seed_front", vp), ("counts", vp),
    ]


# name -> (restype, argtypes); every entry is declared in include/fastgl_b200.h
SIGNATURES = {
    "fgl_last_error": (C.c_char_p, []),
    "fgl_version": (C.c_int, []),
    "fgl_launch_count": (C.c_int64, []),
    "fgl_device_check": (C.c_int, [C.c_int]),
    "fgl_sample_bounds": (C.c_int, [C.c_int64, c_i64p, C.c_int32, c_i32p, C.c_int32, c_i64p]),
    "fgl_sample_window": (C.c_int, [
        C.POINTER(FglGraph), vp, vp, C.c_int64, C.c_int32, vp, c_i32p, C.c_int32,
        C.POINTER(FglSampleOut), vp, C.c_int64, vp]),
    "fgl_philox_words": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, vp, vp]),
    "fgl_philox_bench": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, vp, vp]),
    "fgl_profile": (C.c_int, [C.c_int32]),
    "fgl_depth_relayout_ws_bytes": (C.c_int64, [C.c_int64]),
    "fgl_depth_relayout": (C.c_int, [vp, C.c_int32, C.c_int32, vp, C.c_int64, vp, vp, C.c_int64, vp, C.c_int64,
                                     vp, vp, vp, C.c_int64, vp, vp, vp, C.c_int64, vp]),
    "fgl_add_rows": (C.c_int, [vp, C.c_int64, vp, C.c_int64, C.c_int64, C.c_int32, vp]),
    "fgl_walk_ws_bytes": (C.c_int64, [C.c_int64, C.c_int64]),
    "fgl_sample_walk": (C.c_int, [C.POINTER(FglGraph), vp, C.c_int64, C.c_int32, C.c_uint64, C.c_uint64, vp, vp, vp, C.c_int64,
                                  vp, vp, C.c_int64, vp, vp, C.c_int64, vp]),
    "fgl_profile_read": (C.c_int, [C.c_int64, vp, vp, vp, vp]),
    "fgl_csr_offsets_sorted": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, vp, vp]),
    "fgl_stable_group_ws_bytes": (C.c_int64, [C.c_int64]),
    "fgl_stable_group": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp, vp, vp, C.c_int64, vp]),
    "fgl_gather_i32_f32": (C.c_int, [vp, C.c_int64, vp, vp, vp, vp, vp]),
    "fgl_prepare_layer_ws_bytes": (C.c_int64, [C.c_int64, C.c_int64, C.c_int64]),
    "fgl_prepare_layer_grouped_ws_bytes": (C.c_int64, [C.c_int64, C.c_int64, C.c_int64]),
    "fgl_prepare_layer_grouped": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, vp, vp, vp, vp,
                                            vp, vp, vp, C.c_int64, vp]),
    "fgl_prepare_layer": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, vp, vp,
                                    vp, vp, vp, vp, C.c_int64, vp]),
    "fgl_spmm_ids": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int64, vp, C.c_int64, vp, C.c_int64, C.c_int32, vp,
                               C.c_int64, C.c_int32, vp]),
    "fgl_spmm": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int64, vp, C.c_int64, vp, C.c_int64,
                           vp, C.c_int64, C.c_int32, vp]),
    "fgl_spmm_gather": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int64, vp, C.c_int64, C.c_int64, vp, C.c_int64,
                                  C.c_int32, C.c_int32, vp]),
    "fgl_dense_fwd": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int32, vp, vp, C.c_int32, vp,
                                C.c_int64, C.c_int32, vp]),
    "fgl_dense_bwd_ws_bytes": (C.c_int64, [C.c_int32, C.c_int32]),
    "fgl_dense_bwd": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int32, vp, C.c_int32, vp,
                                C.c_int64, vp, C.c_int64, vp, vp, vp, C.c_int64, vp, C.c_int64,
                                vp]),
    "fgl_dense_dgrad": (C.c_int, [vp, C.c_int64, vp, C.c_int64, C.c_int64, vp, C.c_int32, C.c_int32, vp, C.c_int64,
                                  vp]),
    "fgl_dense_fallback_count": (C.c_int64, []),
    "fgl_set_dense_ctas": (C.c_int, [C.c_int32]),
    "fgl_capture_begin": (C.c_int, [vp]),
    "fgl_capture_end_launch": (C.c_int, [vp, vp]),
    "fgl_exec_create": (C.c_int, [vp]),
    "fgl_exec_destroy": (C.c_int, [vp]),
    "fgl_capture_abort": (C.c_int, [vp]),
    "fgl_capture_stats": (C.c_int, [vp]),
    "fgl_event_create": (C.c_int, [vp]),
    "fgl_event_destroy": (C.c_int, [vp]),
    "fgl_event_record_ext": (C.c_int, [vp, vp]),
    "fgl_stream_wait_ext": (C.c_int, [vp, vp]),
    "fgl_softmax_xent_ws_bytes": (C.c_int64, []),
    "fgl_softmax_xent": (C.c_int, [vp, C.c_int64, vp, C.c_int64, vp, vp, C.c_int64, C.c_int32,
                                   vp, C.c_int64, vp, vp, C.c_int64, vp]),
    "fgl_top_layer_ws_bytes": (C.c_int64, [C.c_int64, C.c_int32, C.c_int32]),
    "fgl_top_layer": (C.c_int, [vp, C.c_int64, vp, C.c_int64, vp, vp, C.c_int64, C.c_int32, C.c_int32, vp, vp, vp,
                                C.c_int64, vp, vp, vp, vp, C.c_int64, vp, vp, vp, C.c_int64, vp, vp]),
    "fgl_top_layer_reduce": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, vp, vp, vp, vp, vp]),
    "fgl_sgd": (C.c_int, [vp, vp, C.c_int64, C.c_float, vp]),
    "fgl_fill_rows": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int32, vp, C.c_int32, vp]),
    "fgl_idmap_ws_bytes": (C.c_int64, [C.c_int64, C.c_int64]),
    "fgl_idmap_build": (C.c_int, [vp, C.c_int64, C.c_int32, C.c_int64, C.c_int32, vp, vp, vp, vp,
                                  C.c_int64, vp]),
    "fgl_idmap_lookup": (C.c_int, [vp, vp, C.c_int64, C.c_int32, C.c_int32, vp, C.c_int64, vp, vp,
                                   vp]),
    "fgl_sample_ws_bitmaps": (C.c_int, [C.c_int64, C.c_int32, C.c_int64, C.c_int64, c_i64p]),
    "fgl_match_counts": (C.c_int, [vp, C.c_int64, C.c_int32, vp, vp]),
    "fgl_mark_bitmaps": (C.c_int, [vp, vp, C.c_int32, C.c_int64, C.c_int64, vp, vp]),
    "fgl_bitmap_test": (C.c_int, [vp, C.c_int64, vp, vp, vp]),
    "fgl_gather_rows": (C.c_int, [vp, C.c_int64, C.c_int32, vp, C.c_int64, vp, vp, C.c_int64,
                                  vp, C.c_int64, vp, C.c_int64, vp, vp]),
    "fgl_host_register": (C.c_int, [vp, C.c_int64, vp]),
    "fgl_host_unregister": (C.c_int, [vp]),
    "fgl_gather_rows_cached": (C.c_int, [vp, C.c_int64, C.c_int32, vp, C.c_int64, vp, vp, C.c_int64,
                                         vp, C.c_int64, vp, vp, vp, C.c_int64, vp, C.c_int64, vp, vp, vp]),
}

_lib = None


def lib():
    """Load (once) and return the library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise MiniGLError(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback for the B200 hot path)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(rc: int, what: str = ""):
    """Map an FGL_E_* return code to the reference's exception type."""
    if rc == FGL_OK:
        return
    msg = lib().fgl_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, MiniGLError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


def status_error(code: int, what: str):
    """Raise for a device-side status word written by a kernel."""
    if code == 0:
        return
    raise _ERRORS.get(int(code), MiniGLError)(f"{what}: device status {int(code)}")


def i64_array(values):
    arr = (C.c_int64 * len(values))(*[int(v) for v in values])
    return arr


def i32_array(values):
    return (C.c_int32 * len(values))(*[int(v) for v in values])
