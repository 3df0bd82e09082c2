"""Test-side helpers for include/fsgpu_debug.h (host model, unrank, magic division)."""
import ctypes

from paper_2405_07989_b200 import _lib as L
from paper_2405_07989_b200.api import Plan


def host_model(n, gens, consumer=L.FS_CONSUMER_COUNT, *, rank=0, world=1, slice_units=0, B=16, cap=None,
               want_hist=False, want_rows=False, want_slices=False, tail=0, gen_order=0, slicing=0, walk=0):
    """Run the kernels' per-lane code on the host (sequential, slice by slice)."""
    p = Plan(n, gens, consumer, rank=rank, world=world, slice_units=slice_units, tail=tail, gen_order=gen_order,
             slicing=slicing, walk=walk)
    info = p.info
    d = len(gens)
    cnt = ctypes.c_uint64(0)
    hist = (ctypes.c_uint64 * info["hist_len"])() if want_hist else None
    rows = None
    if want_rows:
        if cap is None:
            cap = info["unit_end"] - info["unit_begin"] if consumer == L.FS_CONSUMER_ROWS else info["total_rows"]
        rows = ctypes.create_string_buffer(max(1, cap * d * B // 8))
    ns = info["num_slices"]
    sc = (ctypes.c_uint64 * max(1, ns))() if want_slices else None
    sf = (ctypes.c_uint32 * max(1, ns * d))() if want_slices else None
    rc = L.lib().fsdbg_host_model(p.handle, ctypes.byref(cnt), hist, info["hist_len"] if want_hist else 0, B,
                                  ctypes.cast(rows, ctypes.c_void_p) if rows is not None else None,
                                  cap or 0, sc, sf)
    L.check(rc, "fsdbg_host_model")
    out = {"count": cnt.value, "info": info}
    if want_hist:
        out["hist"] = [int(x) for x in hist]
    if want_rows:
        out["rows"] = rows.raw[: min(cap, cnt.value) * d * B // 8]
    if want_slices:
        out["slice_counts"] = [int(x) for x in sc[:ns]]
        out["slice_first"] = [tuple(int(x) for x in sf[i * d:(i + 1) * d]) for i in range(ns)]
    return out


def host_any(n, gens, pred, arg, *, tail=0, gen_order=0, slice_units=0, rank=0, world=1):
    """(found, witness) of the any-predicate through the host model (per row, or per node in
    closed form with tail=FS_TAIL_CLOSED)."""
    p = Plan(n, gens, L.FS_CONSUMER_ANY, rank=rank, world=world, slice_units=slice_units, tail=tail,
             gen_order=gen_order)
    d = len(gens)
    found = ctypes.c_int(0)
    wit = (ctypes.c_uint32 * max(1, d))()
    L.check(L.lib().fsdbg_host_any(p.handle, int(pred), int(arg), ctypes.byref(found), wit), "fsdbg_host_any")
    return bool(found.value), ([int(x) for x in wit[:d]] if found.value else None)


def unrank(plan, unit):
    d = len(plan.gens)
    pre = (ctypes.c_uint32 * max(1, d))()
    row = ctypes.c_int64(0)
    L.check(L.lib().fsdbg_unrank(plan.handle, unit, pre, ctypes.byref(row)), "fsdbg_unrank")
    return [int(x) for x in pre[: max(0, d - 2)]], int(row.value)


def magic(g):
    m = ctypes.c_uint32(0)
    sh = ctypes.c_uint32(0)
    L.check(L.lib().fsdbg_magic(g, ctypes.byref(m), ctypes.byref(sh)), "fsdbg_magic")
    return m.value, sh.value
