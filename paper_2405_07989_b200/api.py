"""Python binding of the C ABI (include/fsgpu.h) -- same names, argument marshalling only.

PyTorch provides device memory (torch tensors' data_ptr()) and streams; every step of the
enumeration runs in libfsgpu.so's CUDA kernels.  Calls raise if the library or a CUDA
device is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

from . import _lib as L


def _torch():
    import torch

    return torch


def _exec(device: Optional[int] = None, stream=None, rank: int = 0, world: int = 1,
          slice_units: int = 0, ctas_per_sm: int = 0, order: int = 0, tail: int = 0,
          gen_order: int = 0, rows_impl: int = 0, slicing: int = 0, walk: int = 0) -> L.ExecT:
    ex = L.ExecT()
    ex.device = -1 if device is None else int(device)
    ex.cuda_stream = None if stream is None else ctypes.c_void_p(int(stream))
    ex.rank = int(rank)
    ex.world = int(world)
    ex.slice_units = int(slice_units)
    ex.ctas_per_sm = int(ctas_per_sm)
    ex.order = int(order)
    ex.tail = int(tail)
    ex.gen_order = int(gen_order)
    ex.rows_impl = int(rows_impl)
    ex.slicing = int(slicing)
    ex.walk = int(walk)
    return ex


def _stream_handle(stream):
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------ north_star entry points
def fs_count(n: int, gens: Sequence[int]) -> int:
    """|Z(n, gens)|, computed on the current CUDA device."""
    g, d = L.gens_array(gens)
    out = ctypes.c_uint64(0)
    L.check(L.lib().fs_count(int(n), g, d, ctypes.byref(out)), "fs_count")
    return int(out.value)


def hist_len(n: int, gens: Sequence[int]) -> int:
    return int(n) // min(int(x) for x in gens) + 1


def fs_length_set(n: int, gens: Sequence[int], hist=None):
    """Length histogram h[l] = #{a in Z : sum a = l}, l = 0..floor(n/min g), as an int64
    CUDA tensor (the u64 counts of fs_length_set reinterpreted)."""
    torch = _torch()
    g, d = L.gens_array(gens)
    cap = hist_len(n, gens)
    if hist is None:
        hist = torch.empty(cap, dtype=torch.int64, device="cuda")
    L.check(L.lib().fs_length_set(int(n), g, d, ctypes.c_void_p(hist.data_ptr()), hist.numel()),
            "fs_length_set")
    return hist


def fs_any(n: int, gens: Sequence[int], pred: int, pred_arg: int) -> Tuple[bool, Optional[List[int]]]:
    """(found, witness): does some factorization satisfy the predicate."""
    g, d = L.gens_array(gens)
    found = ctypes.c_int(0)
    wit = (ctypes.c_uint32 * max(1, d))()
    L.check(L.lib().fs_any(int(n), g, d, int(pred), int(pred_arg), ctypes.byref(found), wit), "fs_any")
    return bool(found.value), ([int(x) for x in wit[:d]] if found.value else None)


def fs_enumerate(n: int, gens: Sequence[int], B: int = 16, cap: Optional[int] = None, out=None):
    """Rows of Z in canonical decreasing-lex order.  Returns (|Z|, rows) where rows is a
    uint16/int32 CUDA tensor of shape [min(cap, |Z|), d] (raw little-endian u16/u32 words).

    If cap is None, |Z| is obtained from a plan first (exact DP) and every row is written."""
    torch = _torch()
    g, d = L.gens_array(gens)
    if cap is None:
        cap = Plan(n, gens, L.FS_CONSUMER_ROWS).info["total_rows"]
    dt = torch.uint16 if B == 16 else torch.int32
    if out is None:
        out = torch.empty((max(0, int(cap)), d), dtype=dt, device="cuda")
    total = L.check(L.lib().fs_enumerate(int(n), g, d, int(B), ctypes.c_void_p(out.data_ptr()), int(cap)),
                    "fs_enumerate")
    return int(total), out[: min(int(cap), int(total))]


# ------------------------------------------------------------------ _ex variants
def fs_count_ex(n, gens, *, device=None, stream=None, rank=0, world=1, slice_units=0, ctas_per_sm=0,
                tail=L.FS_TAIL_ROWS, gen_order=L.FS_GENORDER_GIVEN, slicing=L.FS_SLICES_AUTO, walk=L.FS_WALK_AUTO) -> int:
    g, d = L.gens_array(gens)
    ex = _exec(device, _stream_handle(stream), rank, world, slice_units, ctas_per_sm, 0, tail, gen_order, 0, slicing,
               walk)
    out = ctypes.c_uint64(0)
    L.check(L.lib().fs_count_ex(int(n), g, d, ctypes.byref(ex), ctypes.byref(out)), "fs_count_ex")
    return int(out.value)


def fs_length_set_ex(n, gens, hist=None, *, device=None, stream=None, rank=0, world=1, slice_units=0,
                     ctas_per_sm=0, gen_order=L.FS_GENORDER_GIVEN, tail=L.FS_TAIL_ROWS, slicing=L.FS_SLICES_AUTO,
                     walk=L.FS_WALK_AUTO):
    torch = _torch()
    g, d = L.gens_array(gens)
    ex = _exec(device, _stream_handle(stream), rank, world, slice_units, ctas_per_sm, 0, tail, gen_order, 0, slicing,
               walk)
    if hist is None:
        hist = torch.empty(hist_len(n, gens), dtype=torch.int64,
                           device="cuda" if device is None else "cuda:%d" % device)
    L.check(L.lib().fs_length_set_ex(int(n), g, d, ctypes.byref(ex), ctypes.c_void_p(hist.data_ptr()),
                                     hist.numel()), "fs_length_set_ex")
    return hist


def fs_any_ex(n, gens, pred, pred_arg, *, device=None, stream=None, rank=0, world=1, slice_units=0,
              ctas_per_sm=0, gen_order=L.FS_GENORDER_GIVEN, tail=L.FS_TAIL_ROWS, slicing=L.FS_SLICES_AUTO):
    g, d = L.gens_array(gens)
    ex = _exec(device, _stream_handle(stream), rank, world, slice_units, ctas_per_sm, 0, tail, gen_order, 0, slicing)
    found = ctypes.c_int(0)
    wit = (ctypes.c_uint32 * max(1, d))()
    L.check(L.lib().fs_any_ex(int(n), g, d, ctypes.byref(ex), int(pred), int(pred_arg), ctypes.byref(found),
                              wit), "fs_any_ex")
    return bool(found.value), ([int(x) for x in wit[:d]] if found.value else None)


def fs_enumerate_ex(n, gens, B=16, cap=None, out=None, *, device=None, stream=None, rank=0, world=1,
                    slice_units=0, ctas_per_sm=0, order=L.FS_ORDER_CANONICAL, gen_order=L.FS_GENORDER_GIVEN,
                    rows_impl=L.FS_ROWS_BATCH):
    """This rank's block of rows.  Returns (rank_rows, global_row_offset, rows_tensor).
    order=FS_ORDER_ANY: warp-compacted (M2) layout, same multiset of rows, arbitrary order.
    rows_impl: FS_ROWS_BATCH (default) or FS_ROWS_STAGED (the round-1 kernels)."""
    torch = _torch()
    g, d = L.gens_array(gens)
    ex = _exec(device, _stream_handle(stream), rank, world, slice_units, ctas_per_sm, order, 0, gen_order,
               rows_impl)
    if cap is None:
        info = Plan(n, gens, L.FS_CONSUMER_ROWS, rank=rank, world=world).info
        cap = info["row_end"] - info["row_begin"]
    dt = torch.uint16 if B == 16 else torch.int32
    if out is None:
        out = torch.empty((max(0, int(cap)), d), dtype=dt,
                          device="cuda" if device is None else "cuda:%d" % device)
    off = ctypes.c_uint64(0)
    rows = L.check(L.lib().fs_enumerate_ex(int(n), g, d, int(B), ctypes.c_void_p(out.data_ptr()), int(cap),
                                           ctypes.byref(ex), ctypes.byref(off)), "fs_enumerate_ex")
    return int(rows), int(off.value), out[: min(int(cap), int(rows))]


def fs_enumerate_filtered(n, gens, pred, pred_arg, B=16, cap=None, out=None, *, device=None, stream=None, rank=0,
                          world=1, slice_units=0, ctas_per_sm=0, gen_order=L.FS_GENORDER_GIVEN):
    """Rows of (this rank's share of) Z(n, gens) satisfying pred(pred_arg), in arbitrary order
    (SURVEY 8(f) NEXT-4).  Returns (matches, rows_tensor); rows_tensor holds all matches when
    they fit in cap (default: counted first, then allocated exactly), else it is empty."""
    torch = _torch()
    g, d = L.gens_array(gens)
    ex = _exec(device, _stream_handle(stream), rank, world, slice_units, ctas_per_sm, L.FS_ORDER_ANY, 0, gen_order)
    fn = L.lib().fs_enumerate_filtered_ex
    if cap is None:
        cap = L.check(fn(int(n), g, d, int(B), int(pred), int(pred_arg), None, 0, ctypes.byref(ex)),
                      "fs_enumerate_filtered_ex")
    dt = torch.uint16 if B == 16 else torch.int32
    if out is None:
        out = torch.empty((max(1, int(cap)), d), dtype=dt, device="cuda" if device is None else "cuda:%d" % device)
    m = L.check(fn(int(n), g, d, int(B), int(pred), int(pred_arg), ctypes.c_void_p(out.data_ptr()), int(cap),
                   ctypes.byref(ex)), "fs_enumerate_filtered_ex")
    return int(m), out[: int(m) if m <= cap else 0]


# ------------------------------------------------------------------ plans
class Plan:
    """Host work (validation, constants, exact DP tables, partition) done once; kernels
    enqueued asynchronously on `stream` with results left in device tensors."""

    def __init__(self, n: int, gens: Sequence[int], consumer: int = L.FS_CONSUMER_COUNT, *,
                 device: Optional[int] = None, stream=None, rank: int = 0, world: int = 1,
                 slice_units: int = 0, ctas_per_sm: int = 0, order: int = 0, tail: int = 0,
                 gen_order: int = 0, rows_impl: int = 0, slicing: int = 0, walk: int = 0):
        self.n = int(n)
        self.gens = tuple(int(x) for x in gens)
        self.consumer = consumer
        g, d = L.gens_array(gens)
        self._stream = stream
        ex = _exec(device, _stream_handle(stream), rank, world, slice_units, ctas_per_sm, order, tail, gen_order,
                   rows_impl, slicing, walk)
        h = ctypes.c_void_p()
        L.check(L.lib().fs_plan_create(self.n, g, d, int(consumer), ctypes.byref(ex), ctypes.byref(h)),
                "fs_plan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().fs_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def info(self) -> dict:
        inf = L.PlanInfoT()
        L.check(L.lib().fs_plan_info(self._h, ctypes.byref(inf)), "fs_plan_info")
        out = {k: getattr(inf, k) for k, _ in L.PlanInfoT._fields_ if k != "nodes_per_level"}
        out["nodes_per_level"] = [int(inf.nodes_per_level[i]) for i in range(inf.level + 1)]
        return out

    def count_async(self, out):
        return L.check(L.lib().fs_plan_count_async(self._h, ctypes.c_void_p(out.data_ptr())), "count_async")

    def hist_async(self, out):
        return L.check(L.lib().fs_plan_hist_async(self._h, ctypes.c_void_p(out.data_ptr()), out.numel()),
                       "hist_async")

    def any_async(self, pred: int, arg: int, found, witness=None):
        w = ctypes.c_void_p(witness.data_ptr()) if witness is not None else None
        return L.check(L.lib().fs_plan_any_async(self._h, int(pred), int(arg), ctypes.c_void_p(found.data_ptr()),
                                                 w), "any_async")

    def enumerate_async(self, B: int, out, cap: int):
        return L.check(L.lib().fs_plan_enumerate_async(self._h, int(B), ctypes.c_void_p(out.data_ptr()), int(cap)),
                       "enumerate_async")

    def rows_check(self) -> None:
        """Wait for the plan's stream and check the order=any (M2) cursor invariant (raises)."""
        L.check(L.lib().fs_plan_rows_check(self._h), "fs_plan_rows_check")

    def last_launches(self) -> int:
        return int(L.lib().fs_plan_last_launches(self._h))


def sort_rows_desc(rows):
    """Canonical (decreasing lex) order of a [N, d] row tensor on the device -- used to
    verify the order=any (M2) layout.  Stable sorts from the last coordinate to the first."""
    torch = _torch()
    x = rows.to(torch.int64)
    idx = torch.arange(x.shape[0], device=x.device)
    for j in range(x.shape[1] - 1, -1, -1):
        order = torch.sort(x[idx, j], descending=True, stable=True).indices
        idx = idx[order]
    return x[idx].to(rows.dtype)
