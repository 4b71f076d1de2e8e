"""ctypes binding of the C ABI in include/spdkfac.h (lib/libspdkfac.so).

There is no fallback: if the library is missing or the device is not an
sm_100 B200, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ.get("SPDKFAC_LIB", _HERE / "lib" / "libspdkfac.so"))

OK, ERR_NOT_PD, ERR_SHAPE, ERR_ARG, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED = range(7)
ROWS, CONV_A, SPATIAL, CONV_A_NHWC, SPATIAL_NHWC = 0, 1, 2, 3, 4


class FactorGeom(C.Structure):
    _fields_ = [("layout", C.c_int32), ("n", C.c_int64), ("c", C.c_int64), ("h", C.c_int64), ("w", C.c_int64),
                ("kh", C.c_int32), ("kw", C.c_int32), ("stride_h", C.c_int32), ("stride_w", C.c_int32),
                ("pad_h", C.c_int32), ("pad_w", C.c_int32), ("dil_h", C.c_int32), ("dil_w", C.c_int32)]


_vp, _i32, _i64, _f32, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_size_t
_pp = C.POINTER(C.c_void_p)
_pi32 = C.POINTER(C.c_int32)

# name -> (restype, argtypes); must match include/spdkfac.h exactly
SIGNATURES = {
    "spdkfac_last_error": (C.c_char_p, []),
    "spdkfac_version": (C.c_int, []),
    "spdkfac_device_supported": (C.c_int, []),
    "spdkfac_stats_reset": (None, [C.c_int]),
    "spdkfac_stats_launches": (C.c_uint64, []),
    "spdkfac_stats_reserve": (C.c_int, [C.c_int]),
    "spdkfac_stats_read": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(_i64), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
    "spdkfac_stats_set_probes": (C.c_int, [C.c_int, C.c_int]),
    "spdkfac_factor_dims": (C.c_int, [C.POINTER(FactorGeom), C.POINTER(_i64), C.POINTER(_i64)]),
    "spdkfac_factor_workspace_size": (_sz, [C.POINTER(FactorGeom)]),
    "spdkfac_factor_plan_create": (C.c_int, [C.POINTER(_vp), C.POINTER(FactorGeom), _vp, _sz, _vp]),
    "spdkfac_factor_plan_run": (C.c_int, [_vp, _vp, _f32, _f32, _f32, _vp, _vp]),
    "spdkfac_factor_plan_stage": (C.c_int, [_vp, _vp, _vp]),
    "spdkfac_factor_plan_compute": (C.c_int, [_vp, _f32, _f32, _f32, _vp, _vp]),
    "spdkfac_factor_plan_destroy": (None, [_vp]),
    "spdkfac_factor_group_workspace_size": (_sz, [C.c_int, C.POINTER(FactorGeom)]),
    "spdkfac_factor_group_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.POINTER(FactorGeom), _pp,
                                              C.POINTER(C.c_float), _vp, _sz, _vp]),
    "spdkfac_factor_group_stage": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "spdkfac_factor_group_compute": (C.c_int, [_vp, _f32, _f32, _vp]),
    "spdkfac_factor_group_destroy": (None, [_vp]),
    "spdkfac_factor_group_describe": (C.c_int, [_vp, C.c_int, C.POINTER(_i64)]),
    "spdkfac_pack_upper_f32": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "spdkfac_unpack_upper_f32": (C.c_int, [_vp, _i64, _vp, _i64, _vp]),
    "spdkfac_pack_upper_batched_f32": (C.c_int, [C.c_int, _pi32, _pp, _pp, _vp]),
    "spdkfac_unpack_upper_batched_f32": (C.c_int, [C.c_int, _pi32, _pp, _pp, _vp]),
    "spdkfac_inverse_workspace_size": (_sz, [C.c_int, _pi32]),
    "spdkfac_inverse_plan_create": (C.c_int, [C.POINTER(_vp), C.c_int, _pi32, _pp, _pp, _vp, _vp, _sz, _vp]),
    "spdkfac_inverse_plan_run": (C.c_int, [_vp, _f32, _vp]),
    "spdkfac_inverse_plan_destroy": (None, [_vp]),
    "spdkfac_precond_workspace_size": (_sz, [C.c_int, _pi32, _pi32]),
    "spdkfac_precond_plan_create": (C.c_int, [C.POINTER(_vp), C.c_int, _pi32, _pi32, _vp, _sz, _vp]),
    "spdkfac_precond_plan_run": (C.c_int, [_vp, _pp, _pp, _pp, _pp, _f32, _pp, _vp]),
    "spdkfac_precond_plan_stage_inverses": (C.c_int, [_vp, C.c_int, C.c_int, _pi32, _pp, _vp]),
    "spdkfac_precond_plan_stage_packed": (C.c_int, [_vp, C.c_int, C.c_int, _pi32, _pp, _pp, _vp]),
    "spdkfac_precond_plan_destroy": (None, [_vp]),
    "spdkfac_comm_unique_id": (C.c_int, [_vp]),
    "spdkfac_comm_create": (C.c_int, [C.POINTER(_vp), _vp, C.c_int, C.c_int]),
    "spdkfac_comm_allreduce_sum_f32": (C.c_int, [_vp, _vp, _sz, _vp]),
    "spdkfac_comm_bcast_f32": (C.c_int, [_vp, _vp, _sz, C.c_int, _vp]),
    "spdkfac_comm_reduce_sum_f32": (C.c_int, [_vp, _vp, _sz, C.c_int, _vp]),
    "spdkfac_comm_group_start": (C.c_int, []),
    "spdkfac_comm_group_end": (C.c_int, []),
    "spdkfac_comm_destroy": (None, [_vp]),
    "spdkfac_peer_alloc": (C.c_int, [_sz, C.POINTER(_vp)]),
    "spdkfac_peer_free": (C.c_int, [_vp]),
    "spdkfac_peer_handle": (C.c_int, [_vp, _vp]),
    "spdkfac_peer_open": (C.c_int, [_vp, C.POINTER(_vp)]),
    "spdkfac_peer_close": (C.c_int, [_vp]),
    "spdkfac_peer_copy": (C.c_int, [_vp, _vp, _sz, _vp]),
    "spdkfac_peer_scatter_f32": (C.c_int, [_pp, C.c_int, _vp, _i64, _vp]),
    "spdkfac_peer_epoch_advance": (C.c_int, [_vp, _vp]),
    "spdkfac_peer_signal": (C.c_int, [_pp, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "spdkfac_peer_wait_sum": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, C.c_double, _vp, _vp, _i64,
                                        C.c_int, _vp, _i64, _vp]),
}

_lib = None


class LibraryError(RuntimeError):
    pass


def load(require_device: bool = False):
    """Load (once) and return the ctypes library; raise loudly if absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise LibraryError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device and not _lib.spdkfac_device_supported():
        raise LibraryError("libspdkfac requires an sm_100 (B200) CUDA device")
    return _lib


STAT_CATEGORIES = ("factor_stage", "factor_syrk", "factor_reduce", "inv_small", "inv_pivot", "inv_panel",
                   "inv_update", "inv_unpack_finalize", "precond_split", "precond_gemm", "precond_apply", "pack")


def stats_reset(timing=False, reserve: int = 0) -> None:
    """timing: False / True (all categories) / iterable of category names."""
    if timing is True:
        mask = -1
    elif not timing:
        mask = 0
    else:
        mask = 0
        for name in timing:
            mask |= 1 << STAT_CATEGORIES.index(name)
    lib = load()
    if reserve:
        check(lib.spdkfac_stats_reserve(int(reserve)), "stats reserve")
    lib.spdkfac_stats_reset(mask)


def stats_probes(categories=(), slots: int = 4096) -> None:
    """Time the given categories with in-kernel launch probes (no events; see include/spdkfac.h)."""
    mask = 0
    for name in categories:
        mask |= 1 << STAT_CATEGORIES.index(name)
    check(load().spdkfac_stats_set_probes(mask, int(slots)), "stats probes")


def stats() -> dict:
    """Per-category {ms, launches, flops, bytes} since the last stats_reset (synchronises)."""
    lib = load()
    out = {}
    for i, name in enumerate(STAT_CATEGORIES):
        ms, n, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        check(lib.spdkfac_stats_read(i, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by)), "stats")
        out[name] = {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}
    out["total_launches"] = int(lib.spdkfac_stats_launches())
    return out


def last_error() -> str:
    msg = load().spdkfac_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc in (ERR_SHAPE, ERR_ARG):
        raise ValueError(msg)
    raise LibraryError(f"spdkfac error {rc}: {msg}")


def ptr_array(ptrs):
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i32_array(vals):
    arr = (C.c_int32 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
