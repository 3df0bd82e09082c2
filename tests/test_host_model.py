"""CPU checks of the CUDA path's host logic: the exact DP tables, slice unranking, the
per-lane successor (csrc/fs_core.cuh, executed on the host by fsdbg_host_model) and the
W-way partition, all against the oracle.  No GPU needed; no kernel is launched."""
import random

import pytest

import oracle
from oracle import gf
from paper_2405_07989_b200 import _lib as L
from paper_2405_07989_b200 import workloads as W
from paper_2405_07989_b200.api import Plan

from .fsdbg import host_any, host_model, magic, unrank


def small_instances(count, seed, d_max=6, g_max=30, n_max=300, max_rows=20000):
    out = []
    for inst in W.random_instances(count * 3, seed=seed, d_max=d_max, g_max=g_max, n_max=n_max):
        if gf.count(inst.n, inst.gens) <= max_rows:
            out.append(inst)
        if len(out) == count:
            break
    out += [W.Instance("n0", 0, (3, 5, 7)), W.Instance("d1", 12, (4,)), W.Instance("d1x", 13, (4,)),
            W.Instance("d2", 100, (6, 10)), W.Instance("rep", 30, (2, 2, 2, 2)),
            W.Instance("empty", 7, (4, 6)), W.Instance("ones", 12, (1, 1, 1, 1, 1)),
            W.Instance("unsorted", 200, (20, 6, 9)), W.Instance("big_last", 500, (3, 7, 499)),
            W.Instance("g1_last", 40, (5, 7, 1)), W.Instance("C1", 1000, (6, 9, 20))]
    return out


INSTANCES = small_instances(60, seed=0)


def test_library_exports_every_declared_symbol():
    import re
    import os
    lib = L.lib()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    names = set()
    for h in ("fsgpu.h", "fsgpu_debug.h"):
        src = open(os.path.join(root, "include", h)).read()
        names |= set(re.findall(r"\b((?:fs|fsdbg)_[a-z0-9_]+)\s*\(", src))
    assert len(names) >= 20
    for nm in sorted(names):
        assert hasattr(lib, nm), nm
    assert lib.fs_version() == 10000
    assert set(L.EXPORTS) <= names


@pytest.mark.parametrize("inst", INSTANCES, ids=lambda i: "%s_%d_%s" % (i.name, i.n, "-".join(map(str, i.gens))))
def test_host_model_matches_oracle(oracle_mod, inst):
    n, g = inst.n, inst.gens
    want_rows = oracle.rows(n, g, B=32)
    want_hist = oracle.hist(n, g)
    for T in (0, 1, 3):
        r = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=T, want_hist=True, want_rows=True, B=32)
        assert r["count"] == len(want_rows) // (4 * len(g))
        assert r["info"]["total_rows"] == r["count"]
        assert r["hist"] == want_hist
        # count-sliced plans visit slices in order, so rows come out canonical too
        assert r["rows"] == want_rows
    for T in (8, 16):
        r = host_model(n, g, L.FS_CONSUMER_ROWS, slice_units=T, want_rows=True, B=32)
        assert r["rows"] == want_rows


@pytest.mark.parametrize("inst", INSTANCES, ids=lambda i: "%s" % i.name)
def test_closed_tail_count(oracle_mod, inst):
    """NEXT-1 closed-form tail: same count, and the same per-slice counts, as the row steps."""
    n, g = inst.n, inst.gens
    want = oracle.count(n, g)
    for T in (0, 1, 2, 7):
        a = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=T, want_slices=True, tail=L.FS_TAIL_CLOSED)
        b = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=T, want_slices=True)
        assert a["count"] == want == b["count"]
        if T:  # forced uniform slices: the same slices (automatic ones are cut by kernel-specific costs)
            assert a["slice_counts"] == b["slice_counts"]


@pytest.mark.parametrize("inst", INSTANCES, ids=lambda i: "%s" % i.name)
def test_skip_ablation_count(oracle_mod, inst):
    """Skip=off / Skip=paper candidate loops (the paper's literal index-(d-1) loop): same
    count and per-slice counts as the modulo-skip-at-entry rows."""
    n, g = inst.n, inst.gens
    want = oracle.count(n, g)
    for tail in (L.FS_TAIL_SKIP_OFF, L.FS_TAIL_SKIP_PAPER):
        for go in (0, 1):
            a = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=3, want_slices=True, tail=tail, gen_order=go)
            b = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=3, want_slices=True, gen_order=go)
            assert a["count"] == want
            assert a["slice_counts"] == b["slice_counts"]


@pytest.mark.parametrize("inst", INSTANCES, ids=lambda i: "%s" % i.name)
def test_closed_tail_hist(oracle_mod, inst):
    """Closed-tail histogram: strided difference array of each node's length progression."""
    n, g = inst.n, inst.gens
    want = oracle.hist(n, g)
    for go in (0, 1):
        for T in (0, 1, 5):
            r = host_model(n, g, L.FS_CONSUMER_HIST, slice_units=T, want_hist=True, tail=L.FS_TAIL_CLOSED,
                           gen_order=go)
            assert r["hist"] == want


@pytest.mark.parametrize("inst", INSTANCES[:40] + INSTANCES[-11:], ids=lambda i: "%s" % i.name)
def test_any_predicate_rows_and_closed(oracle_mod, inst):
    """fs_any's decision per row (tail rows) and per node in closed form (tail closed: the
    extreme row of the node's progression, LEN_EQ solved for j) against the oracle's rows,
    for every predicate kind around the attained bounds, given and auto generator order."""
    n, g = inst.n, inst.gens
    d = len(g)
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), d, 32)
    lens = sorted(set(sum(r) for r in rows))
    preds = [(L.FS_PRED_LEN_LE, 0), (L.FS_PRED_LEN_GE, 1 << 33), (L.FS_PRED_LEN_EQ, 1 << 41)]
    for x in lens[:2] + lens[-2:] + lens[len(lens) // 2:len(lens) // 2 + 1]:
        preds += [(L.FS_PRED_LEN_LE, x), (L.FS_PRED_LEN_LE, x - 1), (L.FS_PRED_LEN_GE, x), (L.FS_PRED_LEN_GE, x + 1),
                  (L.FS_PRED_LEN_EQ, x), (L.FS_PRED_LEN_EQ, x + 1)]
    for i in range(d):
        top = max((r[i] for r in rows), default=0)
        preds += [(L.FS_PRED_COORD_GE, (i << 32) | top), (L.FS_PRED_COORD_GE, (i << 32) | (top + 1)),
                  (L.FS_PRED_COORD_GE, (i << 32) | (top // 2))]
    rowset = set(rows)
    for pred, arg in preds:
        if arg < 0:
            continue
        want = any(oracle.pred_holds(r, pred, arg) for r in rows)
        for tail in (L.FS_TAIL_ROWS, L.FS_TAIL_CLOSED):
            for go in (L.FS_GENORDER_GIVEN, L.FS_GENORDER_AUTO):
                found, wit = host_any(n, g, pred, arg, tail=tail, gen_order=go, slice_units=3)
                assert found == want, (pred, arg, tail, go)
                if found:
                    assert tuple(wit) in rowset and oracle.pred_holds(wit, pred, arg)


@pytest.mark.parametrize("inst", INSTANCES, ids=lambda i: "%s" % i.name)
def test_generator_order_auto(oracle_mod, inst):
    """NEXT-2: the stream over a permutation of the generators gives the same count and
    histogram, and the same multiset of rows in the caller's coordinates."""
    n, g = inst.n, inst.gens
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    for tail in (0, 1):
        r = host_model(n, g, L.FS_CONSUMER_COUNT, gen_order=L.FS_GENORDER_AUTO, tail=tail, slice_units=3,
                       want_hist=(tail == 0))
        assert r["count"] == want["count"]
        if tail == 0:
            assert r["hist"] == want["hist"]
    r = host_model(n, g, L.FS_CONSUMER_COUNT, gen_order=L.FS_GENORDER_AUTO, want_rows=True, B=32)
    got = sorted(oracle.rows_as_tuples(r["rows"], len(g), 32), reverse=True)
    assert got == oracle.rows_as_tuples(oracle.rows(n, g, B=32), len(g), 32)


def test_generator_order_choice():
    # C5: largest generators first collapses 6.7e11 nodes to 7.7e5
    p = Plan(W.C5.n, W.C5.gens, gen_order=L.FS_GENORDER_AUTO)
    assert p.info["nodes_per_level"][-1] < 10 ** 6
    assert p.info["total_rows"] == 4055053706
    q = Plan(W.C3.n, W.C3.gens, gen_order=L.FS_GENORDER_AUTO)
    assert q.info["nodes_per_level"][-1] < Plan(W.C3.n, W.C3.gens).info["nodes_per_level"][-1]
    # canonical materialise never permutes
    r = Plan(W.C5.n, W.C5.gens, L.FS_CONSUMER_ROWS, gen_order=L.FS_GENORDER_AUTO)
    assert r.info["nodes_per_level"][-1] > 10 ** 11


@pytest.mark.parametrize("inst", INSTANCES[:30], ids=lambda i: "%s" % i.name)
def test_slices_exact_and_gap_free(oracle_mod, inst):
    """Per-slice row counts equal the oracle's rows in that lex range: no gaps, no overlap."""
    n, g = inst.n, inst.gens
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), len(g), 32)
    r = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=2, want_slices=True, want_rows=True, B=32)
    assert sum(r["slice_counts"]) == len(rows)
    pos = 0
    for cnt, first in zip(r["slice_counts"], r["slice_first"]):
        if cnt:
            assert rows[pos] == first
        pos += cnt
    # row-sliced plans: every slice holds exactly T rows except the last
    rr = host_model(n, g, L.FS_CONSUMER_ROWS, slice_units=8, want_slices=True)
    sc, T = rr["slice_counts"], rr["info"]["slice_units"]
    assert T % 64 == 0
    assert all(c == T for c in sc[:-1]) and (not sc or 1 <= sc[-1] <= T)


@pytest.mark.parametrize("inst", [i for i in INSTANCES if len(i.gens) >= 4][:30], ids=lambda i: "%s" % i.name)
def test_cost_slices_exact_and_gap_free(oracle_mod, inst):
    """Equal-cost slices (automatic slicing of node-unit plans, d >= 4): cut at run starts by a
    cost-space unrank; the per-slice counts and first rows tile the oracle's rows exactly (empty
    slices -- two cost targets inside one run -- hold nothing), for every tail and rank."""
    n, g = inst.n, inst.gens
    rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), len(g), 32)
    for tail in (L.FS_TAIL_ROWS, L.FS_TAIL_CLOSED):
        for world in (1, 3):
            pos = 0
            for rank in range(world):
                r = host_model(n, g, L.FS_CONSUMER_COUNT, rank=rank, world=world, want_slices=True, tail=tail,
                               slicing=L.FS_SLICES_COST)
                i = r["info"]
                assert i["num_slices"] >= (1 if i["unit_end"] > i["unit_begin"] else 0)
                for cnt, first in zip(r["slice_counts"], r["slice_first"]):
                    if cnt and tail == L.FS_TAIL_ROWS:  # (the closed tail records no rows)
                        assert rows[pos] == first
                    pos += cnt
            assert pos == len(rows)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_concatenates(oracle_mod, world):
    for inst in INSTANCES[:25]:
        n, g = inst.n, inst.gens
        want = oracle.rows(n, g, B=16)
        got = b""
        total = 0
        for rank in range(world):
            r = host_model(n, g, L.FS_CONSUMER_ROWS, rank=rank, world=world, want_rows=True, B=16)
            info = r["info"]
            assert info["row_begin"] == total
            total += r["count"]
            got += r["rows"]
        assert got == want
        # count plans: partial counts sum to |Z|
        s = sum(host_model(n, g, L.FS_CONSUMER_COUNT, rank=k, world=world)["count"] for k in range(world))
        assert s == gf.count(n, g)


def test_unrank_rows_equals_oracle_row(oracle_mod):
    rng = random.Random(0)
    for inst in INSTANCES[:30]:
        n, g = inst.n, inst.gens
        d = len(g)
        if d < 2:
            continue
        rows = oracle.rows_as_tuples(oracle.rows(n, g, B=32), d, 32)
        if not rows:
            continue
        p = Plan(n, g, L.FS_CONSUMER_ROWS)
        for r in rng.sample(range(len(rows)), min(10, len(rows))):
            prefix, j = unrank(p, r)
            assert tuple(prefix) == rows[r][: d - 2]
            # row j of the node: the valid a_{d-1} values are a*, a*-s, ...
            same = [x for x in rows if x[: d - 2] == rows[r][: d - 2]]
            assert same[j] == rows[r]


def test_dp_totals_and_nodes(oracle_mod):
    for inst in INSTANCES:
        n, g = inst.n, inst.gens
        info = Plan(n, g).info
        assert info["total_rows"] == gf.count(n, g)
        d = len(g)
        if d >= 2:
            # nodes at level k = #(a_1..a_k) with sum <= n = sum_{r<=n} |Z(r, g_1..g_k)|
            for k, nk in enumerate(info["nodes_per_level"]):
                assert nk == sum(gf.count_table(n, g[:k])) if k else nk == 1
            assert info["total_units"] == info["nodes_per_level"][d - 2]  # node units


def test_full_size_plans():
    """Plans of the full-size configs: exact totals (vs oracle.gf) and slice sizing."""
    for name in ("C2", "C2L", "C2XL", "C3", "C5"):
        inst = W.CONFIGS[name]
        info = Plan(inst.n, inst.gens).info
        assert info["total_rows"] == gf.count(inst.n, inst.gens)
        assert info["num_slices"] >= 1
        ri = Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS).info
        assert ri["total_units"] == ri["total_rows"] == info["total_rows"]
        assert ri["slice_units"] % 8 == 0


def test_magic_division():
    rng = random.Random(1)
    gs = list(range(1, 2000)) + [rng.randint(2, 2 ** 31 - 1) for _ in range(300)] + [2 ** k for k in range(31)] + \
         [2 ** k + 1 for k in range(30)] + [2 ** k - 1 for k in range(2, 31)]
    xs_fixed = [0, 1, 2, 3, 2 ** 31 - 1, 2 ** 31 - 2, 2 ** 30, 2 ** 30 - 1]
    for g in gs:
        m, sh = magic(g)
        assert 0 < m < 2 ** 32
        xs = xs_fixed + [rng.randint(0, 2 ** 31 - 1) for _ in range(40)] + [g * k + r for k in (1, 7, 1000) for r in (-1, 0, 1) if 0 <= g * k + r < 2 ** 31]
        for x in xs:
            assert (x * m) >> sh == x // g, (g, x)


def test_validation_errors():
    with pytest.raises(ValueError):
        Plan(10, (2, 0, 3))
    with pytest.raises(ValueError):
        Plan(10, ())
    with pytest.raises(ValueError):
        Plan(10, tuple(range(1, 18)))
    with pytest.raises(OverflowError):
        Plan(2 ** 31 - 10, (3, 20))
    Plan(2 ** 31 - 21, (20, 3))  # n + max g = 2^31 - 1: accepted (d = 2, no tables)
    with pytest.raises(ValueError):
        Plan(10, (2, 3), rank=2, world=2)


def test_filtered_and_order_argument_checks():
    """fs_enumerate_filtered_ex rejects a bad width / predicate / misaligned buffer before any
    GPU work (FS_EINVAL on any machine); the exec struct carries the rows_impl field."""
    import ctypes

    g = (ctypes.c_uint32 * 3)(6, 9, 20)
    fn = L.lib().fs_enumerate_filtered_ex
    ex = L.ExecT()
    ex.device, ex.world = -1, 1
    assert fn(1000, g, 3, 8, L.FS_PRED_LEN_EQ, 100, None, 0, ctypes.byref(ex)) == L.FS_EINVAL  # B
    assert fn(1000, g, 3, 16, 0, 100, None, 0, ctypes.byref(ex)) == L.FS_EINVAL  # predicate
    assert fn(1000, g, 3, 16, 9, 100, None, 0, ctypes.byref(ex)) == L.FS_EINVAL
    assert fn(1000, g, 3, 16, L.FS_PRED_LEN_EQ, 100, ctypes.c_void_p(8), 10, ctypes.byref(ex)) == L.FS_EINVAL
    names = [f for f, _ in L.ExecT._fields_]
    assert "rows_impl" in names and names.index("rows_impl") == names.index("gen_order") + 1


def test_range_boundary_d3_plans():
    """n + max g = 2^31 - 1 at d = 3 (SURVEY 8(c) edge battery): the level-0 DP table is
    compact (floor(n / g_1) + 1 entries), so the plan exists when g_1 is large; the host model
    of the closed-tail count (64-bit node counts) matches the oracle's congruence sum.  With
    g_1 = 1 the level-0 table would need 2^31 entries: FS_ERANGE."""
    n = 2 ** 31 - 1 - 1000
    want = gf.count_d3(n, (1000, 1, 1))
    p = Plan(n, (1, 1, 1000), tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO)
    assert p.info["total_rows"] == want
    assert host_model(n, (1, 1, 1000), tail=L.FS_TAIL_CLOSED, gen_order=L.FS_GENORDER_AUTO)["count"] == want
    with pytest.raises(OverflowError):
        Plan(n, (1, 1, 1000), gen_order=L.FS_GENORDER_GIVEN)
    with pytest.raises(OverflowError):
        Plan(n + 1, (1000, 1, 1))


def test_host_model_group_counts_beyond_32_bits():
    """The table-driven closed-tail count on the host in the kernel's counter widths (32-bit
    group sums folded into 64 bits): one slice of (1,1,2) at n = 2^22 holds 4.4e12 rows."""
    n = 2 ** 22
    want = sum(n - 2 * x + 1 for x in range(n // 2 + 1))
    assert want > 2 ** 32
    for T in (0, 1 << 24):
        r = host_model(n, (1, 1, 2), tail=L.FS_TAIL_CLOSED, slice_units=T)
        assert r["count"] == want
    assert host_model(100000, (1, 1, 1), tail=L.FS_TAIL_CLOSED, slice_units=1 << 24)["count"] == 5000150001


def test_hist_state_form_host_replay(oracle_mod):
    """The state-form histogram table (fs_host.cu, hq_group) replayed on the host: every
    instance's histogram equals the oracle's, the residue-form walk gives the same, and every
    difference update stays inside the kernel's shared array with its margins (else ERANGE)."""
    import random

    rng = random.Random(11)
    used = 0
    signs = set()
    tried = 0
    while used < 40 and tried < 4000:
        tried += 1
        d = rng.randint(3, 7)
        g = [rng.randint(1, 30) for _ in range(d)]
        n = rng.randint(0, 300)
        go = rng.randint(0, 1)
        p = Plan(n, g, L.FS_CONSUMER_HIST, tail=L.FS_TAIL_CLOSED, gen_order=go)
        if not p.info["state_block"]:
            continue
        used += 1
        want = oracle.hist(n, g)
        for T in (0, 1, 9):
            r = host_model(n, g, L.FS_CONSUMER_HIST, slice_units=T, want_hist=True, tail=L.FS_TAIL_CLOSED,
                           gen_order=go)
            assert r["info"]["state_block"] == 8
            assert r["hist"] == want, (n, g, go, T)
        r = host_model(n, g, L.FS_CONSUMER_HIST, want_hist=True, tail=L.FS_TAIL_CLOSED, gen_order=go,
                       walk=L.FS_WALK_RESIDUE)
        assert r["info"]["state_block"] == 0 and r["hist"] == want
        gi = sorted(g, reverse=True) if go else g
        signs.add((gi[-2] > gi[-1]))
    assert used == 40 and signs == {True, False}


def test_hist_state_form_c3_gens(oracle_mod):
    """C3's generators (largest-first: g_{d-1}, g_d = 14, 13, dl = +1) at oracle-sized n."""
    for n in (300, 650):
        r = host_model(n, W.C3.gens, L.FS_CONSUMER_HIST, want_hist=True, tail=L.FS_TAIL_CLOSED,
                       gen_order=L.FS_GENORDER_AUTO)
        assert r["info"]["state_block"] == 8
        assert r["hist"] == oracle.hist(n, W.C3.gens)


def _cd_instances():
    """Instances whose last k >= 3 generators share a factor (NEXT-3 beyond the last two),
    in stream order for gen_order given and auto."""
    rng = random.Random(23)
    out = [(300, (5, 7, 6, 9, 12), 0), (260, (11, 4, 6, 10, 8), 0), (240, (7, 5, 12, 18, 30, 24), 0),
           (180, (3, 10, 15, 20, 25), 1), (200, (9, 8, 12, 16, 20, 4), 0)]
    while len(out) < 24:
        d = rng.randint(4, 7)
        f = rng.choice((2, 3, 4, 6))
        k = rng.randint(3, d - 1)
        g = [rng.randint(1, 25) for _ in range(d - k)] + [f * rng.randint(1, 8) for _ in range(k)]
        out.append((rng.randint(0, 260), tuple(g), rng.randint(0, 1)))
    return out


@pytest.mark.parametrize("case", _cd_instances(), ids=lambda c: "%d_%s_go%d" % (c[0], "-".join(map(str, c[1])), c[2]))
def test_dead_subtree_skip(oracle_mod, case):
    """NEXT-3 for k >= 3 trailing generators (fs_core.cuh ascend_cd): every consumer's host model
    with the dead-subtree skip equals the oracle, at tiny slices (budgets ending inside a
    skipped subtree) and over 3 ranks, and the plan reports the skipped levels."""
    n, g, go = case
    want = oracle.run(n, g, hist_len=oracle.hist_len_for(n, g))
    levels = Plan(n, g, L.FS_CONSUMER_COUNT, gen_order=go).info["dead_levels"]
    from math import gcd

    def mask(gi):
        m = 0
        for q in range(len(gi) - 3):
            G = 0
            for x in gi[q + 1:]:
                G = gcd(G, x)
            m |= (G > 1) << q
        return m

    # (auto order keeps the given order unless largest-first has fewer level-L nodes)
    assert levels == mask(list(g)) or (go and levels == mask(sorted(g, reverse=True)))
    for T in (0, 1, 3, 7):
        for tail in (L.FS_TAIL_ROWS, L.FS_TAIL_CLOSED):
            r = host_model(n, g, L.FS_CONSUMER_COUNT, slice_units=T, tail=tail, gen_order=go, want_slices=True)
            assert r["count"] == want["count"], (T, tail)
        r = host_model(n, g, L.FS_CONSUMER_HIST, slice_units=T, want_hist=True, tail=L.FS_TAIL_CLOSED, gen_order=go)
        assert r["hist"] == want["hist"], T
    tot = sum(host_model(n, g, L.FS_CONSUMER_COUNT, rank=r, world=3, tail=L.FS_TAIL_CLOSED, gen_order=go)["count"]
              for r in range(3))
    assert tot == want["count"]
    if not go:
        r = host_model(n, g, L.FS_CONSUMER_ROWS, slice_units=8, want_rows=True, B=32)
        assert r["rows"] == oracle.rows(n, g, B=32)
    lmax = max((i for i, v in enumerate(want["hist"]) if v), default=0)
    f, _ = host_any(n, g, L.FS_PRED_LEN_GE, lmax, tail=L.FS_TAIL_CLOSED, gen_order=go, slice_units=3)
    assert f == bool(want["count"])


def test_any_claim_order():
    """The any-predicate's claim order (fs_core.cuh claim_slice, compiled into libfsgpu): for
    every slice count S the 2^bits claims map onto [0, S) exactly once (no slice skipped or
    taken twice), claim 0 is the lex-first slice and claim 1 the lex-last, and both halves are
    walked in bit-reversed order (claims 2, 3 are the middles)."""
    f = L.lib().fsdbg_claim_slice
    none = (1 << 64) - 1
    for S in list(range(1, 130)) + [1000, 4097, 65536, 100003]:
        bits = max(0, (S - 1).bit_length())
        got = [f(i, bits, S) for i in range(1 << bits)]
        live = [g for g in got if g != none]
        assert sorted(live) == list(range(S)), S
        if S >= 2:
            assert got[0] == 0 and got[1] == S - 1
        if S >= 8:  # the middles (the back half holds floor(S/2) slices)
            mid = 1 << (bits - 2)
            assert got[2] == (mid if mid < (S + 1) // 2 else none)
            assert got[3] == (S - 1 - mid if mid < S // 2 else none)
