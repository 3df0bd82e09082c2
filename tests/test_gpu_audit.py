"""GPU: the device slice audit (include/fsgpu_debug.h fsdbg_count_slices).

The bounds of PAPER.md:196-200 must partition the lex order: every factorization is counted by
exactly one slice.  The closed-tail count kernel writes every slice's row count on the device;
each must equal the number of oracle rows between the slice's first node and the next slice's
(oracle.gf.prefix_ranker: the canonical index of the first row with a prefix), for uniform and
equal-cost slices, whole instances and rank shares."""
import ctypes

import pytest

from oracle import gf
from paper_2405_07989_b200 import _lib as L
from paper_2405_07989_b200 import api
from paper_2405_07989_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [W.C2, W.Instance("C3s", 1500, W.C3.gens), W.Instance("C5s", 3000, W.C5.gens),
         W.Instance("d4", 700, (7, 11, 13, 17)), W.Instance("cd", 2500, (11, 13, 17, 18, 24)),
         W.Instance("d6", 400, (5, 6, 9, 10, 14, 15))]


def _slice_starts(p, rank):
    info = p.info
    d = len(p.gens)
    out = []
    for sl in range(info["num_slices"]):
        u = ctypes.c_uint64(0)
        pre = (ctypes.c_uint32 * max(1, d))()
        L.check(L.lib().fsdbg_slice_start(p.handle, sl, ctypes.byref(u), pre), "fsdbg_slice_start")
        out.append((u.value, tuple(int(x) for x in pre[: d - 2])))
    return out


@pytest.mark.parametrize("inst", CASES, ids=lambda i: i.name)
@pytest.mark.parametrize("slicing", [L.FS_SLICES_UNIFORM, L.FS_SLICES_COST])
@pytest.mark.parametrize("world", [1, 3])
def test_slice_audit(inst, slicing, world):
    n, g = inst.n, inst.gens
    rank_of = gf.prefix_ranker(n, g)  # the stream runs the given order here
    total = gf.count(n, g)
    seen = 0
    for r in range(world):
        p = api.Plan(n, g, L.FS_CONSUMER_COUNT, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_GIVEN,
                     slicing=slicing, rank=r, world=world)
        info = p.info
        S = info["num_slices"]
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        sc = torch.zeros(max(1, S), dtype=torch.int64, device="cuda")
        L.check(L.lib().fsdbg_count_slices(p.handle, ctypes.c_void_p(cnt.data_ptr()), ctypes.c_void_p(sc.data_ptr())),
                "fsdbg_count_slices")
        torch.cuda.synchronize()
        got = [int(x) for x in sc[:S].cpu().tolist()]
        starts = _slice_starts(p, r)
        bounds = [rank_of(pre) if u < info["total_units"] else total for u, pre in starts]
        if info["unit_end"] >= info["total_units"]:
            end = total
        else:  # the next rank's first node
            from tests.fsdbg import unrank
            end = rank_of(unrank(p, info["unit_end"])[0])
        want = [b - a for a, b in zip(bounds, bounds[1:] + [end])]
        assert got == want
        assert sum(got) == int(cnt.item())
        if S:
            assert bounds[0] == seen  # ranks tile the lex order
        seen = end if S else seen
    assert seen == total
