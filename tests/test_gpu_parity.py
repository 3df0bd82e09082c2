"""GPU parity: the CUDA path, called through the C ABI (python binding), against the oracle
on the same seeded inputs.  Integer results must be bit-exact; rows byte-identical."""
import hashlib
import json
import os
import random
import struct

import pytest

import oracle
from oracle import gf
from paper_2405_07989_b200 import _lib as L
from paper_2405_07989_b200 import api
from paper_2405_07989_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    with open(os.path.join(GOLD, name + ".json")) as f:
        return json.load(f)


def rows_bytes(t):
    return t.contiguous().cpu().numpy().tobytes()


def hist_list(t, L_):
    return [int(x) for x in t[:L_].cpu().tolist()]


def suite(count, seed, d_max, g_max, n_max, max_rows):
    out = []
    for inst in W.random_instances(count * 4, seed=seed, d_max=d_max, g_max=g_max, n_max=n_max):
        if gf.count(inst.n, inst.gens) <= max_rows:
            out.append(inst)
        if len(out) == count:
            break
    return out


EDGE = [W.Instance("n0", 0, (3, 5, 7)), W.Instance("n0d1", 0, (4,)), W.Instance("d1", 12, (4,)),
        W.Instance("d1x", 13, (4,)), W.Instance("d2", 1000, (6, 10)), W.Instance("d2c", 997, (1, 1)),
        W.Instance("rep", 30, (2, 2, 2, 2)), W.Instance("empty", 7, (4, 6)), W.Instance("lt", 2, (3, 5, 7)),
        W.Instance("ones", 12, (1, 1, 1, 1, 1)), W.Instance("unsorted", 200, (20, 6, 9)),
        W.Instance("biglast", 500, (3, 7, 499)), W.Instance("g1last", 40, (5, 7, 1)),
        W.Instance("d16", 40, tuple(range(2, 18))), W.Instance("d16b", 30, (3,) * 8 + (5,) * 8),
        W.Instance("huge_gA", 60000, (7, 9000, 11)), W.Instance("huge_s", 70000, (3, 5, 65537)),
        W.Instance("C1", 1000, (6, 9, 20)), W.Instance("McN44", 44, (6, 9, 20)),
        W.Instance("cd6", 800, (11, 13, 17, 18, 24)), W.Instance("cd10", 700, (6, 10, 15, 4, 14))]
RAND = suite(50, seed=0, d_max=8, g_max=40, n_max=400, max_rows=300000)
ALL = EDGE[:-2] + RAND[:19] + EDGE[-2:] + RAND[19:]  # the non-coprime-tail pair within ALL[:40]
assert all(gf.count(i.n, i.gens) <= 300000 for i in EDGE), "edge instances must stay oracle-sized"
ids = lambda i: "%s_%d_%s" % (i.name, i.n, "-".join(map(str, i.gens)))


@pytest.mark.parametrize("inst", ALL, ids=ids)
def test_count_hist_rows(oracle_mod, inst):
    n, g = inst.n, inst.gens
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    assert api.fs_count(n, g) == want["count"]
    h = api.fs_length_set(n, g)
    assert hist_list(h, len(want["hist"])) == want["hist"]
    for B in (16, 32):
        if B == 16 and max(n // x for x in g) > 65535:
            with pytest.raises(OverflowError):
                api.fs_enumerate(n, g, B=B)
            continue
        total, rows = api.fs_enumerate(n, g, B=B)
        assert total == want["count"]
        assert rows_bytes(rows) == oracle.rows(n, g, B=B)


@pytest.mark.parametrize("inst", ALL[:30], ids=ids)
@pytest.mark.parametrize("T", [1, 5])
def test_tiny_slices(oracle_mod, inst, T):
    """Force many tiny slices: per-slice boundaries must neither lose nor duplicate rows."""
    n, g = inst.n, inst.gens
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    assert api.fs_count_ex(n, g, slice_units=T) == want["count"]
    h = api.fs_length_set_ex(n, g, slice_units=T)
    assert hist_list(h, len(want["hist"])) == want["hist"]
    rows, off, t = api.fs_enumerate_ex(n, g, B=32, slice_units=8 * T)
    assert rows == want["count"] and off == 0
    assert rows_bytes(t) == oracle.rows(n, g, B=32)


@pytest.mark.parametrize("inst", ALL, ids=ids)
def test_count_closed_tail(oracle_mod, inst):
    n, g = inst.n, inst.gens
    want = oracle.count(n, g)
    for go in (L.FS_GENORDER_GIVEN, L.FS_GENORDER_AUTO):
        for T in (0, 1, 5, 37):
            assert api.fs_count_ex(n, g, slice_units=T, tail=L.FS_TAIL_CLOSED, gen_order=go) == want
        parts = [api.fs_count_ex(n, g, rank=r, world=3, tail=L.FS_TAIL_CLOSED, gen_order=go) for r in range(3)]
        assert sum(parts) == want


@pytest.mark.parametrize("inst", ALL, ids=ids)
def test_count_skip_ablation(oracle_mod, inst):
    n, g = inst.n, inst.gens
    want = oracle.count(n, g)
    for tail in (L.FS_TAIL_SKIP_OFF, L.FS_TAIL_SKIP_PAPER):
        for T in (0, 2):
            assert api.fs_count_ex(n, g, slice_units=T, tail=tail) == want


@pytest.mark.parametrize("inst", ALL, ids=ids)
def test_hist_closed_tail(oracle_mod, inst):
    n, g = inst.n, inst.gens
    want = oracle.hist(n, g)
    for go in (L.FS_GENORDER_GIVEN, L.FS_GENORDER_AUTO):
        for T in (0, 1, 5):
            h = api.fs_length_set_ex(n, g, slice_units=T, gen_order=go, tail=L.FS_TAIL_CLOSED)
            assert hist_list(h, len(want)) == want
    hs = [api.fs_length_set_ex(n, g, rank=r, world=3, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO)
          for r in range(3)]
    assert hist_list(sum(hs), len(want)) == want


@pytest.mark.parametrize("inst", ALL, ids=ids)
def test_generator_order_auto(oracle_mod, inst):
    """NEXT-2 (stream over the largest generators first): same count / histogram / any, rows in
    the caller's coordinates (M2 layout), witnesses and COORD_GE indices in caller order."""
    n, g = inst.n, inst.gens
    AUTO = L.FS_GENORDER_AUTO
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    assert api.fs_count_ex(n, g, gen_order=AUTO) == want["count"]
    assert api.fs_count_ex(n, g, gen_order=AUTO, tail=L.FS_TAIL_CLOSED) == want["count"]
    h = api.fs_length_set_ex(n, g, gen_order=AUTO)
    assert hist_list(h, len(want["hist"])) == want["hist"]
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), len(g), 32)
    for pred, arg in [(L.FS_PRED_COORD_GE, ((len(g) - 1) << 32) | 2), (L.FS_PRED_COORD_GE, 1),
                      (L.FS_PRED_LEN_EQ, sum(rows[len(rows) // 2]) if rows else 1)]:
        found, wit = api.fs_any_ex(n, g, pred, arg, gen_order=AUTO)
        assert found == any(oracle.pred_holds(r, pred, arg) for r in rows)
        if found:
            assert tuple(wit) in set(rows) and oracle.pred_holds(wit, pred, arg)
    B = 32
    for impl in (L.FS_ROWS_BATCH, L.FS_ROWS_STAGED):  # the staged kernel runs the permuted order
        nr, off, t = api.fs_enumerate_ex(n, g, B=B, order=L.FS_ORDER_ANY, gen_order=AUTO, rows_impl=impl)
        assert nr == len(rows)
        assert rows_bytes(api.sort_rows_desc(t)) == oracle.rows(n, g, B=B)


def test_c5_auto_order_full():
    g = gold("C5")
    AUTO = L.FS_GENORDER_AUTO
    assert api.fs_count_ex(W.C5.n, W.C5.gens, gen_order=AUTO) == g["count"]
    assert api.fs_count_ex(W.C5.n, W.C5.gens, gen_order=AUTO, tail=L.FS_TAIL_CLOSED) == g["count"]
    h = api.fs_length_set_ex(W.C5.n, W.C5.gens, gen_order=AUTO)
    assert hist_list(h, 20001) == g["hist"]
    found, wit = api.fs_any_ex(W.C5.n, W.C5.gens, L.FS_PRED_LEN_LE, 20, gen_order=AUTO)
    assert found and wit == [0, 0, 0, 0, 20]
    assert not api.fs_any_ex(W.C5.n, W.C5.gens, L.FS_PRED_LEN_LE, 19, gen_order=AUTO)[0]


@pytest.mark.parametrize("inst", ALL[:40], ids=ids)
def test_any(oracle_mod, inst):
    n, g = inst.n, inst.gens
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), len(g), 32)
    lens = sorted(sum(r) for r in rows)
    preds = [(L.FS_PRED_LEN_LE, lens[0] if lens else 0), (L.FS_PRED_LEN_LE, max(0, (lens[0] if lens else 1) - 1)),
             (L.FS_PRED_LEN_GE, lens[-1] if lens else 0), (L.FS_PRED_LEN_EQ, lens[len(lens) // 2] if lens else 3),
             (L.FS_PRED_COORD_GE, ((len(g) - 1) << 32) | 2), (L.FS_PRED_COORD_GE, (0 << 32) | 1)]
    # closed tail decides LEN_EQ by solving l0 + j (t - s) = X, COORD_GE at the extreme row:
    # every length and every coordinate index, around the attained bounds
    d = len(g)
    distinct = sorted(set(lens))
    preds += [(L.FS_PRED_LEN_EQ, x) for x in distinct[:3] + distinct[-3:]]
    preds += [(L.FS_PRED_LEN_EQ, distinct[0] - 1 if distinct else 0), (L.FS_PRED_LEN_GE, lens[-1] + 1 if lens else 1)]
    for i in range(d):
        top = max((r[i] for r in rows), default=0)
        preds += [(L.FS_PRED_COORD_GE, (i << 32) | top), (L.FS_PRED_COORD_GE, (i << 32) | (top + 1))]
    rowset = set(rows)
    runs = [lambda pr, a: api.fs_any(n, g, pr, a),
            lambda pr, a: api.fs_any_ex(n, g, pr, a),
            lambda pr, a: api.fs_any_ex(n, g, pr, a, tail=L.FS_TAIL_CLOSED),
            lambda pr, a: api.fs_any_ex(n, g, pr, a, tail=L.FS_TAIL_CLOSED, slice_units=1)]
    for pred, arg in preds:
        want = any(oracle.pred_holds(r, pred, arg) for r in rows)
        for run in runs:
            found, wit = run(pred, arg)
            assert found == want, (pred, arg)
            if found:
                assert sum(a * b for a, b in zip(wit, g)) == n
                assert oracle.pred_holds(wit, pred, arg)
                assert tuple(wit) in rowset


def _pack(rows, d, B):
    fmt = "<%d%s" % (d, "H" if B == 16 else "I")
    return b"".join(struct.pack(fmt, *r) for r in rows)


@pytest.mark.parametrize("inst", ALL[:40], ids=ids)
def test_rows_filtered(oracle_mod, inst):
    """Filtered materialise (NEXT-4): exactly the oracle rows satisfying the predicate (sorted =
    the canonical order of that subset), for every predicate kind around the attained bounds,
    both coordinate widths, given and auto generator order, tiny slices, and the count-only /
    too-small-cap contract."""
    n, g = inst.n, inst.gens
    d = len(g)
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), d, 32)
    lens = sorted(set(sum(r) for r in rows)) or [0]
    preds = [(L.FS_PRED_LEN_LE, lens[0]), (L.FS_PRED_LEN_LE, lens[len(lens) // 2]), (L.FS_PRED_LEN_GE, lens[-1]),
             (L.FS_PRED_LEN_EQ, lens[len(lens) // 2]), (L.FS_PRED_LEN_EQ, lens[0] - 1 if lens[0] else 1 << 40),
             (L.FS_PRED_COORD_GE, ((d - 1) << 32) | 2), (L.FS_PRED_COORD_GE, (0 << 32) | 1)]
    for i in range(d):
        top = max((r[i] for r in rows), default=0)
        preds.append((L.FS_PRED_COORD_GE, (i << 32) | max(0, top - 1)))
    for B in (16, 32):
        if B == 16 and max(n // x for x in g) > 65535:
            continue
        for k, (pred, arg) in enumerate(preds):
            want = [r for r in rows if oracle.pred_holds(r, pred, arg)]
            kw = [{}, {"gen_order": L.FS_GENORDER_AUTO}, {"slice_units": 64}][k % 3]
            m, t = api.fs_enumerate_filtered(n, g, pred, arg, B=B, **kw)
            assert m == len(want), (pred, arg)
            assert rows_bytes(api.sort_rows_desc(t)) == _pack(want, d, B)
            if want:  # too small a cap: the count, nothing written
                m2, t2 = api.fs_enumerate_filtered(n, g, pred, arg, B=B, cap=len(want) - 1)
                assert m2 == len(want) and t2.shape[0] == 0


def test_rows_filtered_c2(oracle_mod):
    """C2 (681,152 rows): one length class, sharded over 3 virtual ranks."""
    n, g = W.C2.n, W.C2.gens
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=16), 5, 16)
    X = 120
    want = [r for r in rows if sum(r) == X]
    got = []
    for r in range(3):
        m, t = api.fs_enumerate_filtered(n, g, L.FS_PRED_LEN_EQ, X, B=16, rank=r, world=3)
        got += oracle.rows_as_tuples(rows_bytes(t), 5, 16)
    assert sorted(got, reverse=True) == want


@pytest.mark.parametrize("inst", ALL[:40], ids=ids)
def test_rows_order_any(oracle_mod, inst):
    """M2 layout (warp-aggregated compaction): same multiset of rows; sorted = canonical."""
    n, g = inst.n, inst.gens
    for B in (16, 32):
        if B == 16 and max(n // x for x in g) > 65535:
            continue
        rows, off, t = api.fs_enumerate_ex(n, g, B=B, order=L.FS_ORDER_ANY)
        assert rows == oracle.count(n, g)
        assert rows_bytes(api.sort_rows_desc(t)) == oracle.rows(n, g, B=B)


@pytest.mark.parametrize("inst", ALL[:40], ids=ids)
@pytest.mark.parametrize("impl", [L.FS_ROWS_BATCH, L.FS_ROWS_STAGED])
def test_rows_impls(oracle_mod, inst, impl):
    """Both materialise kernels, both layouts, several slice sizes (many claims, partial warp
    claims, a ragged last slice for the tail kernel): byte-identical canonical rows."""
    n, g = inst.n, inst.gens
    for B in (16, 32):
        if B == 16 and max(n // x for x in g) > 65535:
            continue
        want = oracle.rows(n, g, B=B)
        rb = len(g) * B // 8
        rev = b"".join(want[i:i + rb] for i in range(len(want) - rb, -1, -rb)) if want else b""
        for T in (64, 192, 0):
            rows, off, t = api.fs_enumerate_ex(n, g, B=B, slice_units=T, rows_impl=impl)
            assert rows_bytes(t) == want
            # increasing lex order: the canonical rows reversed; cap = the smallest rows
            rows, off, t = api.fs_enumerate_ex(n, g, B=B, slice_units=T, rows_impl=impl,
                                               order=L.FS_ORDER_INCREASING)
            assert rows_bytes(t) == rev and off == 0
            cap = len(want) // rb // 3
            rows, off, t = api.fs_enumerate_ex(n, g, B=B, slice_units=T, rows_impl=impl, cap=cap,
                                               order=L.FS_ORDER_INCREASING)
            assert rows_bytes(t) == rev[: cap * rb]
            rows, off, t = api.fs_enumerate_ex(n, g, B=B, slice_units=T, rows_impl=impl, order=L.FS_ORDER_ANY)
            assert rows_bytes(api.sort_rows_desc(t)) == want


@pytest.mark.parametrize("impl", [L.FS_ROWS_BATCH, L.FS_ROWS_STAGED])
def test_rows_impls_c2(oracle_mod, impl):
    """C2 (681,152 rows): every supported batch shape's neighbour d = 5 at B = 16/32, both
    layouts, several world sizes (rank blocks with ragged ends)."""
    n, g = W.C2.n, W.C2.gens
    for B in (16, 32):
        want = oracle.rows(n, g, B=B)
        for world in (1, 3):
            blob, blob_any, inc = b"", [], {}
            for r in range(world):
                rows, off, t = api.fs_enumerate_ex(n, g, B=B, rank=r, world=world, rows_impl=impl)
                blob += rows_bytes(t)
                rows, off, t = api.fs_enumerate_ex(n, g, B=B, rank=r, world=world, rows_impl=impl,
                                                   order=L.FS_ORDER_INCREASING)
                inc[off] = rows_bytes(t)
                rows, off, t = api.fs_enumerate_ex(n, g, B=B, rank=r, world=world, rows_impl=impl,
                                                   order=L.FS_ORDER_ANY)
                blob_any.append(rows_bytes(api.sort_rows_desc(t)))
            assert blob == want
            assert b"".join(blob_any) == want
            rb = 5 * B // 8
            assert b"".join(inc[k] for k in sorted(inc)) == b"".join(
                want[i:i + rb] for i in range(len(want) - rb, -1, -rb))


def test_rows_order_any_c2(oracle_mod):
    n, g = W.C2.n, W.C2.gens
    rows, off, t = api.fs_enumerate_ex(n, g, B=16, order=L.FS_ORDER_ANY)
    s = rows_bytes(api.sort_rows_desc(t))
    assert hashlib.sha256(s).hexdigest() == "af101488b41676e1839ebcca06e795af9c2a2d2b278c6f7e0e584315721eb01e"
    with pytest.raises(OverflowError):  # compaction needs room for every row
        api.fs_enumerate_ex(n, g, B=16, cap=rows - 1, order=L.FS_ORDER_ANY)


def test_cap_truncation(oracle_mod):
    n, g = W.C2.n, W.C2.gens
    full = oracle.rows(n, g, B=16)
    rb = 2 * len(g)
    for cap in (0, 1, 7, 8, 9, 1000, 12345, 681151):
        total, t = api.fs_enumerate(n, g, B=16, cap=cap)
        assert total == 681152
        assert rows_bytes(t) == full[: cap * rb]


def test_c2_rows_golden(oracle_mod):
    n, g = W.C2.n, W.C2.gens
    for B, sha in ((16, "af101488b41676e1839ebcca06e795af9c2a2d2b278c6f7e0e584315721eb01e"),
                   (32, "bf19f5cf473192f1055dba45a72442114f083eb5f912b14b8ee16e513ebf2ffd")):
        total, t = api.fs_enumerate(n, g, B=B)
        b = rows_bytes(t)
        assert b == oracle.rows(n, g, B=B)
        assert hashlib.sha256(b).hexdigest() == sha


def test_c1_all_consumers(oracle_mod):
    n, g = W.C1.n, W.C1.gens
    assert api.fs_count(n, g) == 465
    h = api.fs_length_set(n, g)
    assert hist_list(h, 167) == gold("C1")["hist"]
    total, t = api.fs_enumerate(n, g, B=16)
    assert rows_bytes(t) == oracle.rows(n, g, B=16)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_virtual_ranks(oracle_mod, world):
    """Rank r of W run one after another on one GPU: partials combine to the whole."""
    for inst in [W.C1, W.C2] + RAND[:8]:
        n, g = inst.n, inst.gens
        want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
        assert sum(api.fs_count_ex(n, g, rank=r, world=world) for r in range(world)) == want["count"]
        hs = [api.fs_length_set_ex(n, g, rank=r, world=world) for r in range(world)]
        assert hist_list(sum(hs), len(want["hist"])) == want["hist"]
        blob, nxt = b"", 0
        for r in range(world):
            rows, off, t = api.fs_enumerate_ex(n, g, B=16, rank=r, world=world)
            assert off == nxt
            nxt += rows
            blob += rows_bytes(t)
        assert blob == oracle.rows(n, g, B=16)


# ------------------------------------------------------------------ full-size configs
def test_c3_count_full():
    assert api.fs_count(W.C3.n, W.C3.gens) == gold("C3")["count"] == 100032405189
    assert api.fs_count_ex(W.C3.n, W.C3.gens, tail=L.FS_TAIL_CLOSED) == 100032405189


def test_c4_hist_full():
    h = api.fs_length_set(W.C4.n, W.C4.gens)  # default: generator order auto, closed tail
    assert hist_list(h, 329) == gold("C3")["hist"]
    for go in (0, 1):
        for tail in (0, 1):
            h = api.fs_length_set_ex(W.C4.n, W.C4.gens, gen_order=go, tail=tail)
            assert hist_list(h, 329) == gold("C3")["hist"], (go, tail)


@pytest.mark.parametrize("world", [2, 8])
def test_c4_virtual_ranks(world):
    hs = [api.fs_length_set_ex(W.C4.n, W.C4.gens, rank=r, world=world) for r in range(world)]
    assert hist_list(sum(hs), 329) == gold("C3")["hist"]


def test_c5_count_hist_full():
    g = gold("C5")
    assert api.fs_count(W.C5.n, W.C5.gens) == g["count"] == 4055053706
    h = api.fs_length_set(W.C5.n, W.C5.gens)
    assert hist_list(h, 20001) == g["hist"]


def test_c5_any_predicates():
    n, g = W.C5.n, W.C5.gens
    found, wit = api.fs_any(n, g, L.FS_PRED_LEN_LE, 20)      # P_late: unique witness, lex-last row
    assert found and wit == [0, 0, 0, 0, 20]
    found, wit = api.fs_any(n, g, L.FS_PRED_LEN_LE, 19)      # P_none
    assert not found and wit is None
    found, wit = api.fs_any(n, g, L.FS_PRED_LEN_GE, 19995)   # P_first
    assert found and sum(wit) >= 19995 and sum(a * b for a, b in zip(wit, g)) == n
    # the per-row tail, generator order auto (the closed tail is fs_any's default)
    AUTO = L.FS_GENORDER_AUTO
    found, wit = api.fs_any_ex(n, g, L.FS_PRED_LEN_LE, 20, gen_order=AUTO)
    assert found and wit == [0, 0, 0, 0, 20]
    assert not api.fs_any_ex(n, g, L.FS_PRED_LEN_LE, 19, gen_order=AUTO)[0]
    found, wit = api.fs_any_ex(n, g, L.FS_PRED_LEN_EQ, 10001, gen_order=AUTO, tail=L.FS_TAIL_CLOSED)
    assert found and sum(wit) == 10001 and sum(a * b for a, b in zip(wit, g)) == n


def test_c2l_rows_sampled(oracle_mod):
    """C2-L (824,598,466 rows, 8.25 GB of u16): sampled prefix boxes equal the oracle's box
    rows at the GF-computed canonical offsets; global invariants checked on the device."""
    n, g = W.C2L.n, W.C2L.gens
    total, t = api.fs_enumerate(n, g, B=16)
    assert total == 824598466 and t.shape == (total, 5)
    rng = random.Random(0)
    for _ in range(6):
        a1 = rng.randint(0, n // g[0])
        a2 = rng.randint(0, (n - a1 * g[0]) // g[1])
        box = ((a1,), a2, a2)
        want = oracle.rows(n, g, B=16, box=box)
        off = gf.rows_before_prefix(n, g, (a1, a2))
        cnt = len(want) // 10
        assert rows_bytes(t[off:off + cnt]) == want
    # every row sums to n; strictly decreasing lex (checked in chunks on the GPU)
    gt = torch.tensor(g, dtype=torch.int64, device="cuda")
    chunk = 1 << 26
    prev = None
    for s in range(0, total, chunk):
        x = t[s:s + chunk].to(torch.int64)
        assert bool(((x * gt).sum(1) == n).all())
        if prev is not None:
            x = torch.cat([prev, x])
        key = x[:, 0] * (1 << 48) + x[:, 1] * (1 << 36) + x[:, 2] * (1 << 24) + x[:, 3] * (1 << 12) + x[:, 4]
        assert bool((key[1:] < key[:-1]).all())
        prev = x[-1:]
    del t
    torch.cuda.empty_cache()


def test_plan_async_and_launch_count():
    p = api.Plan(W.C2.n, W.C2.gens, L.FS_CONSUMER_COUNT)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    before = L.lib().fsdbg_total_launches()
    for _ in range(3):
        p.count_async(out)
        assert p.last_launches() == 1
    torch.cuda.synchronize()
    assert int(out.item()) == 681152
    # 3 count kernels + the plan's one-time slice-start table (built at upload; two kernels
    # for equal-cost slices)
    assert L.lib().fsdbg_total_launches() - before == 3 + (2 if p.info["cost_slices"] else 1)


def test_errors_on_gpu():
    with pytest.raises(ValueError):
        api.fs_count(10, (2, 0))
    with pytest.raises(OverflowError):
        api.fs_enumerate(70000, (1, 2), B=16)
    t = torch.empty(100, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):  # misaligned output
        L.check(L.lib().fs_enumerate(10, (api.ctypes.c_uint32 * 2)(2, 3), 2, 16,
                                     api.ctypes.c_void_p(t.data_ptr() + 2), 2))
    h = torch.empty(3, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):  # hist_cap too small
        api.fs_length_set(100, (3, 5), hist=h)


@pytest.mark.parametrize("inst", [i for i in ALL if len(i.gens) >= 4][:30], ids=ids)
def test_cost_slices(oracle_mod, inst):
    """Equal-cost slices forced at small sizes (automatic only when a rank holds many more runs
    than lanes): slices cut at run starts by a cost-space unrank on the device, node counts
    from the slice-start table, empty slices skipped -- count, histogram and any, both tails,
    given and auto generator order, 1 and 3 ranks."""
    n, g = inst.n, inst.gens
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    C = L.FS_SLICES_COST
    for go in (L.FS_GENORDER_GIVEN, L.FS_GENORDER_AUTO):
        for tail in (L.FS_TAIL_ROWS, L.FS_TAIL_CLOSED):
            assert api.fs_count_ex(n, g, tail=tail, gen_order=go, slicing=C) == want["count"]
            parts = [api.fs_count_ex(n, g, rank=r, world=3, tail=tail, gen_order=go, slicing=C) for r in range(3)]
            assert sum(parts) == want["count"]
            h = api.fs_length_set_ex(n, g, tail=tail, gen_order=go, slicing=C)
            assert hist_list(h, len(want["hist"])) == want["hist"]
        lmax = max(i for i, v in enumerate(want["hist"]) if v) if want["count"] else 0
        found, wit = api.fs_any_ex(n, g, L.FS_PRED_LEN_GE, lmax, tail=L.FS_TAIL_CLOSED, gen_order=go, slicing=C)
        assert found == bool(want["count"])
        if found:
            assert sum(a * b for a, b in zip(wit, g)) == n and sum(wit) >= lmax


def _state_form_instances():
    """Instances whose fs_length_set runs the state-form histogram (hq_group): random ones with
    gcd(g_{d-1}, g_d) = 1 in stream order (both signs of t - s), plus C3's generators."""
    out = [W.Instance("C3g650", 650, W.C3.gens), W.Instance("C3g1100", 1100, W.C3.gens)]
    for inst in W.random_instances(400, seed=5, d_max=7, g_max=30, n_max=350):
        if len(out) == 14:
            break
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_HIST, tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO)
        if p.info["state_block"] and gf.count(inst.n, inst.gens) <= 3000000:
            out.append(inst)
    return out


@pytest.mark.parametrize("inst", _state_form_instances(), ids=ids)
def test_hist_state_form_vs_residue_form(oracle_mod, inst):
    """The state-form histogram walk equals the residue-form walk and the exact histogram, for
    the default slices, tiny slices (many run starts inside blocks) and 3 virtual ranks."""
    n, g = inst.n, inst.gens
    want = gf.hist(n, g)
    kw = dict(tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO)
    assert api.Plan(n, g, L.FS_CONSUMER_HIST, **kw).info["state_block"] == 8
    for T in (0, 1, 7):
        h = api.fs_length_set_ex(n, g, slice_units=T, **kw)
        assert hist_list(h, len(want)) == want, T
    h = api.fs_length_set_ex(n, g, walk=L.FS_WALK_RESIDUE, **kw)
    assert hist_list(h, len(want)) == want
    tot = [0] * len(want)
    for r in range(3):
        h = hist_list(api.fs_length_set_ex(n, g, rank=r, world=3, **kw), len(want))
        tot = [a + b for a, b in zip(tot, h)]
    assert tot == want


def _next3_instances():
    """Non-coprime trailing generators in stream order (NEXT-3): the last two share a
    factor (live-node walks of every closed consumer), or the last k >= 3 do (dead-subtree skip
    in the generic ascend), for given and largest-first order."""
    rng = random.Random(31)
    out = [W.Instance("cd2a", 700, (11, 13, 17, 18, 24)), W.Instance("cd2b", 500, (7, 9, 10, 4, 6)),
           W.Instance("cd3a", 600, (5, 7, 6, 9, 12)), W.Instance("cd3b", 420, (7, 5, 12, 18, 30, 24)),
           W.Instance("cd4", 300, (9, 8, 12, 16, 20, 4)), W.Instance("cdall", 360, (6, 10, 14, 22)),
           # g_{d-1} > 64 with a common divisor: no live-node pair table, the NEXT-3 kernel
           # variant walks the plain pair table (a routing bug found in round 2)
           W.Instance("cdwide", 900, (5, 7, 6, 66, 132)), W.Instance("cdwide2", 800, (3, 11, 70, 140, 210))]
    while len(out) < 20:
        d = rng.randint(4, 7)
        f = rng.choice((2, 3, 4, 6))
        k = rng.randint(2, d - 1)
        g = tuple([rng.randint(1, 25) for _ in range(d - k)] + [f * rng.randint(1, 8) for _ in range(k)])
        n = rng.randint(50, 420)
        if gf.count(n, g) <= 400000:
            out.append(W.Instance("cdr%d" % len(out), n, g))
    return out


@pytest.mark.parametrize("inst", _next3_instances(), ids=ids)
def test_next3_common_divisor_all_consumers(oracle_mod, inst):
    """Every consumer on instances whose trailing generators share a factor: count (rows and
    closed tails), histogram (closed: live-node table), any (closed: live-node step), and the
    materialised rows, against the oracle; tiny slices and 3 virtual ranks for the skips."""
    n, g = inst.n, inst.gens
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    for go in (L.FS_GENORDER_GIVEN, L.FS_GENORDER_AUTO):
        for T in (0, 1, 5):
            for tail in (L.FS_TAIL_ROWS, L.FS_TAIL_CLOSED):
                assert api.fs_count_ex(n, g, slice_units=T, tail=tail, gen_order=go) == want["count"], (go, T, tail)
            h = api.fs_length_set_ex(n, g, slice_units=T, tail=L.FS_TAIL_CLOSED, gen_order=go)
            assert hist_list(h, len(want["hist"])) == want["hist"], (go, T)
        tot = sum(api.fs_count_ex(n, g, rank=r, world=3, tail=L.FS_TAIL_CLOSED, gen_order=go) for r in range(3))
        assert tot == want["count"]
        ls = [i for i, v in enumerate(want["hist"]) if v]
        if ls:
            for pred, arg, exp in ((L.FS_PRED_LEN_GE, ls[-1], True), (L.FS_PRED_LEN_GE, ls[-1] + 1, False),
                                   (L.FS_PRED_LEN_LE, ls[0], True), (L.FS_PRED_LEN_EQ, ls[len(ls) // 2], True)):
                f, wit = api.fs_any_ex(n, g, pred, arg, tail=L.FS_TAIL_CLOSED, gen_order=go, slice_units=3)
                assert f == exp, (pred, arg)
                if f:
                    assert sum(a * b for a, b in zip(wit, g)) == n
    r, off, t = api.fs_enumerate_ex(n, g, B=32)
    assert r == want["count"] and rows_bytes(t) == oracle.rows(n, g, B=32)
