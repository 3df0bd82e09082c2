"""GPU: counter widths and the range limits (SURVEY 8(c) edge battery).

A lane's slice can hold far more than 2^32 factorizations (a node holds up to ~n/(g_{d-1} s)
rows and a slice up to 2^24 nodes), so every per-lane counter must be folded into 64 bits
before it can wrap.  These instances put > 2^32 rows into one slice, one group or one node,
through every count / histogram / any path, and check the exact results against closed
forms (C(n+2, 2) for (1,1,1); the oracle's two-generator congruence sum for d = 3).  The
boundary n + max g = 2^31 - 1 (accepted; 2^31 rejected) is exercised at d = 3, where the
level-0 DP table is stored compactly."""
from math import comb

import pytest

import oracle
from oracle import gf
from paper_2405_07989_b200 import _lib as L
from paper_2405_07989_b200 import api

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CLOSED, ROWS = L.FS_TAIL_CLOSED, L.FS_TAIL_ROWS
GIVEN, AUTO = L.FS_GENORDER_GIVEN, L.FS_GENORDER_AUTO


def test_count_2p28_ones():
    n = 2 ** 28
    want = comb(n + 2, 2)  # |Z(n, (1,1,1))| = C(n + d - 1, d - 1)
    assert want > 2 ** 55
    assert api.fs_count(n, (1, 1, 1)) == want
    assert api.fs_count_ex(n, (1, 1, 1), tail=CLOSED, gen_order=GIVEN) == want


def test_length_set_2p28_ones():
    """Every row of Z(n, (1,1,1)) has length n: one bin holds all C(n+2, 2) rows (the 64-bit
    difference array and the chunked finalize scan at 2^28 + 1 bins, dstride = 1)."""
    n = 2 ** 28
    want = comb(n + 2, 2)
    h = api.fs_length_set(n, (1, 1, 1))
    assert h.numel() == n + 1
    assert int(h[n].item()) == want
    assert int((h != 0).sum().item()) == 1
    del h
    torch.cuda.empty_cache()


def test_count_one_slice_many_rows():
    """A single slice of 100001 nodes holding 5,000,150,001 rows (> 2^32)."""
    n = 100000
    want = comb(n + 2, 2)
    assert want == 5000150001
    for go in (GIVEN, AUTO):
        assert api.fs_count_ex(n, (1, 1, 1), slice_units=1 << 24, tail=CLOSED, gen_order=go) == want
    h = api.fs_length_set_ex(n, (1, 1, 1), slice_units=1 << 24, tail=CLOSED, gen_order=AUTO)
    assert int(h[n].item()) == want and int(h.sum().item()) == want


@pytest.mark.parametrize("T", [0, 1 << 24])
def test_count_group_path_large(T):
    """(1,1,2) in the given order: s = 2, so the closed-tail count runs the paired group table
    (cc_group2); nodes hold up to 2^25 rows, 16-node groups up to 2^29, slices far more."""
    n = 2 ** 26
    want = sum(n - 2 * x + 1 for x in range(n // 2 + 1))  # a_3 = x, (a_1, a_2) on n - 2x
    assert want == gf.count_d3(n, (2, 1, 1))
    assert api.fs_count_ex(n, (1, 1, 2), slice_units=T, tail=CLOSED, gen_order=GIVEN) == want
    # the histogram of the same instance: lengths n - x (a_3 = x), n - 2x + 1 rows each
    h = api.fs_length_set_ex(n, (1, 1, 2), slice_units=T, tail=CLOSED, gen_order=GIVEN)
    idx = torch.arange(n // 2, n + 1, device=h.device)
    exp = 2 * idx - n + 1  # length l = n - x  ->  rows n - 2x + 1 = 2l - n + 1
    assert torch.equal(h[n // 2:], exp.to(h.dtype))
    assert int(h[: n // 2].abs().sum().item()) == 0


def test_count_rows_tail_large_nodes():
    """Per-row tail: 32-bit per-iteration counters folded into 64 bits (2^20-row nodes)."""
    n = 2 ** 20
    want = comb(n + 2, 2)
    assert api.fs_count_ex(n, (1, 1, 1), tail=ROWS, gen_order=GIVEN) == want


D3_BOUNDARY = [
    (2 ** 31 - 1 - 1000, (1, 1, 1000)),    # auto order runs (1000, 1, 1)
    (2 ** 31 - 1 - 1000, (997, 999, 1000)),
    (2 ** 31 - 1 - 65537, (65537, 3, 5)),
]


@pytest.mark.parametrize("n,g", D3_BOUNDARY)
def test_d3_boundary_count(n, g):
    assert n + max(g) == 2 ** 31 - 1
    want = gf.count_d3(n, sorted(g, reverse=True))
    assert api.fs_count(n, g) == want
    with pytest.raises(OverflowError):
        api.fs_count(n + 1, g)  # n + max g = 2^31


def test_d3_boundary_any_and_rows(oracle_mod):
    n, g = 2 ** 31 - 1 - 1000, (1000, 1, 1)
    X = n // 1000
    found, wit = api.fs_any(n, g, L.FS_PRED_LEN_GE, n)  # (0, n, 0) has length n
    assert found and sum(a * b for a, b in zip(wit, g)) == n and sum(wit) >= n
    found, wit = api.fs_any(n, g, L.FS_PRED_LEN_LE, X + (n - 1000 * X) - 1)  # below the minimum length
    assert not found
    found, wit = api.fs_any(n, g, L.FS_PRED_LEN_LE, X + (n - 1000 * X))
    assert found and sum(wit) == X + (n - 1000 * X)
    # the first 1000 canonical rows (u32): boxes a_1 = X, X - 1 of the oracle
    total, rows = api.fs_enumerate(n, g, B=32, cap=1000)
    assert total == gf.count_d3(n, g)
    assert rows.contiguous().cpu().numpy().tobytes() == oracle.rows(n, g, B=32, cap=1000, box=((), X - 1, X))
