"""GPU: complete (not sampled) checks of every materialise layout at HBM-roofline sizes.

C2-L (824,598,466 rows, 8.25 GB of u16 rows) and C2-XL (2,597,173,872 rows, 26 GB) -- the
sizes bench.py times -- in all three layouts (canonical M1, order = any M2, increasing lex;
PAPER.md:55 "saving the factorizations", P:97 increasing order).  Every row is checked on the
device: its coordinates satisfy sum a_i g_i = n (the definition of Z), and its
canonical rank

    rank(a) = sum_{k < d-1} |Z(R_k - (a_k + 1) g_k, (g_k..g_d))|,  R_k = n - sum_{j<k} a_j g_j

(the number of factorizations lex-greater than a: those that agree with a before coordinate k
and exceed it at k) is computed from the oracle's suffix count tables (oracle.gf.suffix_tables).
The ranks must be exactly 0..|Z|-1 in order (canonical), reversed (increasing), or a
permutation of the rank's block (order = any).  This identifies every row, so it is as strong as
a byte comparison with the sorted oracle output."""
import pytest

from oracle import gf
from paper_2405_07989_b200 import _lib as L
from paper_2405_07989_b200 import api
from paper_2405_07989_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CHUNK = 1 << 26


def _suffix(inst, dev):
    S = gf.suffix_tables(inst.n, inst.gens)  # S[k][r] = |Z(r, gens[k:])|
    return torch.tensor([[int(v) for v in row] for row in S], dtype=torch.int64, device=dev)


def _ranks(rows, inst, S):
    """(canonical rank, phi == n) of every row of a [N, d] u16 tensor, chunked."""
    n, g = inst.n, inst.gens
    d = len(g)
    out = torch.empty(rows.shape[0], dtype=torch.int64, device=rows.device)
    for i in range(0, rows.shape[0], CHUNK):
        a = rows[i:i + CHUNK].to(torch.int64)
        R = torch.full((a.shape[0],), n, dtype=torch.int64, device=a.device)
        rk = torch.zeros_like(R)
        for k in range(d - 1):
            r = R - (a[:, k] + 1) * g[k]
            rk += torch.where(r >= 0, S[k][r.clamp(min=0)], torch.zeros_like(r))
            R -= a[:, k] * g[k]
        # the last coordinate closes the sum exactly: phi(a) = n
        assert bool((R == a[:, d - 1] * g[d - 1]).all()), "a row with phi != n"
        assert bool((R >= 0).all())
        out[i:i + CHUNK] = rk
    return out


def _check_perm(rk, lo, hi):
    """rk is a permutation of lo..hi-1"""
    assert rk.numel() == hi - lo
    assert int(rk.min().item()) >= lo and int(rk.max().item()) < hi
    seen = torch.zeros(hi - lo, dtype=torch.bool, device=rk.device)
    seen[rk - lo] = True
    assert bool(seen.all())


@pytest.mark.parametrize("inst", [W.C2L, W.C2XL], ids=lambda i: i.name)
def test_materialise_all_layouts_complete(inst):
    dev = torch.device("cuda")
    S = _suffix(inst, dev)
    total = int(S[0][inst.n].item())
    out = torch.empty((total, inst.d), dtype=torch.uint16, device=dev)
    ar = None
    for order in (L.FS_ORDER_CANONICAL, L.FS_ORDER_INCREASING, L.FS_ORDER_ANY):
        out.view(torch.int16).fill_(-1)  # nothing stale from the previous layout can pass
        rows, off, t = api.fs_enumerate_ex(inst.n, inst.gens, B=16, out=out, cap=total, order=order)
        assert rows == total and off == 0 and t.shape[0] == total
        rk = _ranks(t, inst, S)
        if order == L.FS_ORDER_ANY:
            _check_perm(rk, 0, total)
        else:
            if ar is None:
                ar = torch.arange(total, dtype=torch.int64, device=dev)
            want = ar if order == L.FS_ORDER_CANONICAL else (total - 1) - ar
            assert torch.equal(rk, want)
        del rk
    del out, ar
    torch.cuda.empty_cache()


def test_materialise_plan_async_any_c2l_world2():
    """The plan/async path bench.py times (order = any, M2) with the cursor check, per rank of a
    2-way partition: each rank's rows are exactly its contiguous block of canonical ranks."""
    inst = W.C2L
    dev = torch.device("cuda")
    S = _suffix(inst, dev)
    total = int(S[0][inst.n].item())
    for r in range(2):
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, rank=r, world=2, order=L.FS_ORDER_ANY)
        info = p.info
        rows = info["row_end"] - info["row_begin"]
        out = torch.full((rows, inst.d), -1, dtype=torch.int16, device=dev).view(torch.uint16)
        p.enumerate_async(16, out, rows)
        p.rows_check()
        _check_perm(_ranks(out, inst, S), info["row_begin"], info["row_end"])
        del out
    assert info["row_end"] == total
    torch.cuda.empty_cache()
