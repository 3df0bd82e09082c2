"""ctypes loader for libfsgpu.so (built in-tree by paper_2405_07989_b200/build.py).

Argument marshalling only: every step of the enumeration runs inside the library's CUDA
kernels.  If the shared library is missing this module raises -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfsgpu.so")

FS_OK, FS_EINVAL, FS_ERANGE, FS_ECUDA, FS_ENOMEM, FS_ENODEV = 0, -1, -2, -3, -4, -5
FS_PRED_LEN_LE, FS_PRED_LEN_GE, FS_PRED_LEN_EQ, FS_PRED_COORD_GE = 1, 2, 3, 4
FS_CONSUMER_COUNT, FS_CONSUMER_HIST, FS_CONSUMER_ANY, FS_CONSUMER_ROWS = 0, 1, 2, 3
FS_MAX_D = 16
FS_ORDER_CANONICAL, FS_ORDER_ANY, FS_ORDER_INCREASING = 0, 1, 2
FS_TAIL_ROWS, FS_TAIL_CLOSED, FS_TAIL_SKIP_OFF, FS_TAIL_SKIP_PAPER = 0, 1, 2, 3
FS_GENORDER_GIVEN, FS_GENORDER_AUTO = 0, 1
FS_ROWS_BATCH, FS_ROWS_STAGED = 0, 1
FS_SLICES_AUTO, FS_SLICES_COST, FS_SLICES_UNIFORM = 0, 1, 2
FS_WALK_AUTO, FS_WALK_RESIDUE = 0, 1

u64 = ctypes.c_uint64
i64 = ctypes.c_int64
u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
vp = ctypes.c_void_p


class ExecT(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int),
        ("cuda_stream", ctypes.c_void_p),
        ("rank", ctypes.c_int),
        ("world", ctypes.c_int),
        ("slice_units", ctypes.c_uint64),
        ("ctas_per_sm", ctypes.c_int),
        ("order", ctypes.c_int),
        ("tail", ctypes.c_int),
        ("gen_order", ctypes.c_int),
        ("rows_impl", ctypes.c_int),
        ("slicing", ctypes.c_int),
        ("walk", ctypes.c_int),
        ("reserved", ctypes.c_int * 2),
    ]


class PlanInfoT(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64),
        ("d", ctypes.c_int),
        ("consumer", ctypes.c_int),
        ("level", ctypes.c_int),
        ("total_units", ctypes.c_uint64),
        ("total_rows", ctypes.c_uint64),
        ("unit_begin", ctypes.c_uint64),
        ("unit_end", ctypes.c_uint64),
        ("row_begin", ctypes.c_uint64),
        ("row_end", ctypes.c_uint64),
        ("slice_units", ctypes.c_uint64),
        ("num_slices", ctypes.c_uint64),
        ("hist_len", ctypes.c_uint64),
        ("grid", ctypes.c_uint32),
        ("block", ctypes.c_uint32),
        ("nodes_per_level", ctypes.c_uint64 * FS_MAX_D),
        ("table_bytes", ctypes.c_uint64),
        ("state_block", ctypes.c_uint32),
        ("cost_slices", ctypes.c_uint32),
        ("dead_levels", ctypes.c_uint32),
    ]


EXPORTS = {
    # name: (restype, argtypes)
    "fs_count": (ctypes.c_int, [u64, u32p, ctypes.c_int, u64p]),
    "fs_length_set": (ctypes.c_int, [u64, u32p, ctypes.c_int, vp, u64]),
    "fs_any": (ctypes.c_int, [u64, u32p, ctypes.c_int, ctypes.c_int, u64, ctypes.POINTER(ctypes.c_int), u32p]),
    "fs_enumerate": (i64, [u64, u32p, ctypes.c_int, ctypes.c_int, vp, u64]),
    "fs_count_ex": (ctypes.c_int, [u64, u32p, ctypes.c_int, ctypes.POINTER(ExecT), u64p]),
    "fs_length_set_ex": (ctypes.c_int, [u64, u32p, ctypes.c_int, ctypes.POINTER(ExecT), vp, u64]),
    "fs_any_ex": (ctypes.c_int, [u64, u32p, ctypes.c_int, ctypes.POINTER(ExecT), ctypes.c_int, u64,
                                 ctypes.POINTER(ctypes.c_int), u32p]),
    "fs_enumerate_ex": (i64, [u64, u32p, ctypes.c_int, ctypes.c_int, vp, u64, ctypes.POINTER(ExecT), u64p]),
    "fs_enumerate_filtered_ex": (i64, [u64, u32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u64, vp, u64,
                                       ctypes.POINTER(ExecT)]),
    "fs_plan_create": (ctypes.c_int, [u64, u32p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ExecT),
                                      ctypes.POINTER(vp)]),
    "fs_plan_info": (ctypes.c_int, [vp, ctypes.POINTER(PlanInfoT)]),
    "fs_plan_count_async": (ctypes.c_int, [vp, vp]),
    "fs_plan_hist_async": (ctypes.c_int, [vp, vp, u64]),
    "fs_plan_any_async": (ctypes.c_int, [vp, ctypes.c_int, u64, vp, vp]),
    "fs_plan_enumerate_async": (ctypes.c_int, [vp, ctypes.c_int, vp, u64]),
    "fs_plan_last_launches": (ctypes.c_int, [vp]),
    "fs_plan_rows_check": (ctypes.c_int, [vp]),
    "fs_plan_destroy": (None, [vp]),
    "fs_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "fs_version": (ctypes.c_int, []),
    # test/introspection (include/fsgpu_debug.h)
    "fsdbg_host_model": (ctypes.c_int, [vp, u64p, u64p, u64, ctypes.c_int, vp, u64, u64p, u32p]),
    "fsdbg_host_any": (ctypes.c_int, [vp, ctypes.c_int, u64, ctypes.POINTER(ctypes.c_int), u32p]),
    "fsdbg_unrank": (ctypes.c_int, [vp, u64, u32p, ctypes.POINTER(ctypes.c_int64)]),
    "fsdbg_magic": (ctypes.c_int, [ctypes.c_uint32, u32p, u32p]),
    "fsdbg_magic_div": (ctypes.c_uint32, [ctypes.c_uint32, ctypes.c_uint32]),
    "fsdbg_claim_slice": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]),
    "fsdbg_total_launches": (ctypes.c_uint64, []),
    "fsdbg_count_slices": (ctypes.c_int, [vp, vp, vp]),
    "fsdbg_slice_start": (ctypes.c_int, [vp, u64, u64p, u32p]),
    "fsdbg_microbench": (ctypes.c_int, [ctypes.c_int, u64, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double)]),
}

_lib = None


def lib():
    """Load libfsgpu.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                "libfsgpu.so not found at %s: build it with `python -m paper_2405_07989_b200.build` "
                "(there is no CPU fallback)" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class FsError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> int:
    if rc >= 0:
        return rc
    msg = lib().fs_strerror(rc).decode()
    text = "%s failed: %s (%d)" % (what or "fsgpu", msg, rc)
    if rc == FS_EINVAL:
        raise ValueError(text)
    if rc == FS_ERANGE:
        raise OverflowError(text)
    raise FsError(text)


def gens_array(gens):
    g = [int(x) for x in gens]
    for x in g:
        if x < 0 or x >= 2 ** 32:
            raise ValueError("generator out of uint32 range: %r" % x)
    return (ctypes.c_uint32 * max(1, len(g)))(*g), len(g)
