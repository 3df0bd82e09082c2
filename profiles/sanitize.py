"""Every kernel of libfsgpu.so on small instances, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck).  Results are checked against the oracle, so a run that completes is
also a parity run.  Usage: compute-sanitizer --tool <tool> python profiles/sanitize.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2405_07989_b200 import _lib as L  # noqa: E402
from paper_2405_07989_b200 import api  # noqa: E402

CASES = [(1000, (6, 9, 20)), (600, (11, 13, 17, 19, 23)), (300, (3, 5, 7, 11)), (400, (13, 14, 20, 22, 23, 24, 35, 39)),
         (500, (11, 13, 17, 18, 24)), (2000, (1, 1, 2, 997, 1000)), (0, (3, 5, 7)), (7, (4, 6)), (12, (4,)),
         (1000, (6, 10))]
if os.environ.get("FS_SAN_QUICK"):  # racecheck is ~100x slower: the first, smaller instances
    CASES = [(300, (6, 9, 20)), (250, (11, 13, 17, 19, 23)), (150, (3, 5, 7, 11)), (250, (13, 14, 20, 22, 23, 24, 35, 39)),
             (200, (11, 13, 17, 18, 24)), (7, (4, 6)), (12, (4,))]
GO, TC = L.FS_GENORDER_AUTO, L.FS_TAIL_CLOSED
kernels = 0
for n, g in CASES:
    d = len(g)
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    rows16 = oracle.rows(n, g, B=16) if max(n // x for x in g) <= 65535 else None
    rows32 = oracle.rows(n, g, B=32)
    # count: per-row, closed (residue and state form), skip ablations, uniform / cost / tiny slices, ranks
    for kw in (dict(), dict(tail=TC), dict(tail=TC, gen_order=GO), dict(tail=L.FS_TAIL_SKIP_OFF),
               dict(tail=L.FS_TAIL_SKIP_PAPER), dict(tail=TC, slice_units=3), dict(tail=TC, slicing=L.FS_SLICES_COST),
               dict(tail=TC, gen_order=GO, slicing=L.FS_SLICES_COST)):
        assert api.fs_count_ex(n, g, **kw) == want["count"], (n, g, kw)
        assert sum(api.fs_count_ex(n, g, rank=r, world=3, **kw) for r in range(3)) == want["count"]
    # histogram: per-row and closed
    for kw in (dict(), dict(tail=TC), dict(tail=TC, gen_order=GO), dict(tail=TC, slice_units=5)):
        h = api.fs_length_set_ex(n, g, **kw)
        assert [int(x) for x in h.cpu().tolist()][: len(want["hist"])] == want["hist"], (n, g, kw)
    # any: per-row and closed
    lmax = max(i for i, v in enumerate(want["hist"]) if v) if want["count"] else 0
    for kw in (dict(), dict(tail=TC, gen_order=GO)):
        f, w = api.fs_any_ex(n, g, L.FS_PRED_LEN_GE, lmax, **kw)
        assert f == bool(want["count"])
        f, w = api.fs_any_ex(n, g, L.FS_PRED_LEN_GE, lmax + 1, **kw)
        assert not f
    # materialise: batch and staged kernels, all orders, both widths, a forced small slice size
    for B, want_rows in ((16, rows16), (32, rows32)):
        if want_rows is None:
            continue
        for impl in (L.FS_ROWS_BATCH, L.FS_ROWS_STAGED):
            for T in (0, 64):
                r, off, t = api.fs_enumerate_ex(n, g, B=B, rows_impl=impl, slice_units=T)
                assert t.contiguous().cpu().numpy().tobytes() == want_rows
                r, off, t = api.fs_enumerate_ex(n, g, B=B, rows_impl=impl, slice_units=T, order=L.FS_ORDER_ANY)
                assert api.sort_rows_desc(t).contiguous().cpu().numpy().tobytes() == want_rows
                r, off, t = api.fs_enumerate_ex(n, g, B=B, rows_impl=impl, slice_units=T,
                                                order=L.FS_ORDER_INCREASING)
                assert r == want["count"]
        m, t = api.fs_enumerate_filtered(n, g, L.FS_PRED_LEN_GE, lmax, B=B)
        assert (m >= 1) == bool(want["count"])
    # slice audit kernel
    if d >= 3:
        p = api.Plan(n, g, L.FS_CONSUMER_COUNT, tail=TC, slicing=L.FS_SLICES_COST)
        S = p.info["num_slices"]
        c = torch.zeros(1, dtype=torch.int64, device="cuda")
        sc = torch.zeros(max(1, S), dtype=torch.int64, device="cuda")
        L.check(L.lib().fsdbg_count_slices(p.handle, ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(sc.data_ptr())),
                "audit")
        torch.cuda.synchronize()
        assert int(c.item()) == int(sc.sum().item()) == want["count"]
torch.cuda.synchronize()
print("sanitize workload ok: %d launches" % L.lib().fsdbg_total_launches(), flush=True)
