"""oracle/gf.py -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Exact big-integer counts of Z(n, g) from the generating function

    sum_n |Z(n, g)| x^n = prod_i 1 / (1 - x^{g_i})

(the definition of Z, Sec. 1, read as a coefficient extraction), and the
length histogram from the bivariate generating function

    sum_{n,l} #{a in Z(n,g) : sum a_i = l} x^n y^l = prod_i 1 / (1 - x^{g_i} y).

Both are computed by the textbook coin-change recurrence (multiply by one factor
1/(1 - x^g y) at a time: T[r] += T[r - g], shifted by one in l for the bivariate case).
Python ints only, so nothing can overflow.  This module is independent of oracle/enum.c
(it never enumerates) and of the CUDA path (it shares no code with it).

Used for full-size counts/histograms that the nested-loop oracle cannot finish
(configs C3-C5, hours of enumeration), and for the lex offset of a prefix box so that
sampled rows of a huge enumeration can be compared with oracle/enum.c's box output.
"""
from __future__ import annotations

from typing import List, Sequence


def count(n: int, gens: Sequence[int]) -> int:
    """|Z(n, gens)|: coefficient of x^n in prod 1/(1 - x^g)."""
    if any(int(g) <= 0 for g in gens):
        raise ValueError("generators must be positive")
    T = [0] * (n + 1)
    T[0] = 1
    for g in gens:
        g = int(g)
        for r in range(g, n + 1):
            T[r] += T[r - g]
    return T[n]


def count_table(n: int, gens: Sequence[int]) -> List[int]:
    """[|Z(r, gens)| for r in 0..n]."""
    T = [0] * (n + 1)
    T[0] = 1
    for g in gens:
        g = int(g)
        for r in range(g, n + 1):
            T[r] += T[r - g]
    return T


def hist(n: int, gens: Sequence[int], length: int | None = None) -> List[int]:
    """h[l] = #{a in Z(n, gens) : sum a = l} for l in 0..length-1.

    length defaults to floor(n / min(gens)) + 1 (no factorization is longer)."""
    if any(int(g) <= 0 for g in gens):
        raise ValueError("generators must be positive")
    if length is None:
        length = n // min(int(g) for g in gens) + 1
    import numpy as np

    # H[r][l]: object arrays keep exact Python ints
    H = np.zeros((n + 1, length), dtype=object)
    H[0, 0] = 1
    for g in gens:
        g = int(g)
        for r in range(g, n + 1):
            # multiplying by 1/(1 - x^g y): H[r][l] += H[r-g][l-1]
            H[r, 1:] += H[r - g, :-1]
    return [int(v) for v in H[n]]


def hist_u64(n: int, gens: Sequence[int], length: int | None = None) -> List[int]:
    """Same as hist() but vectorised with numpy uint64 for large n (C3/C5 sizes).

    Every intermediate H[r][l] counts factorizations of r <= n with lengths l using a
    sub-multiset of the generators, so it is bounded by the final column sums; the
    result is cross-checked against count() (exact Python ints) so an overflow could not
    pass silently."""
    import numpy as np

    if length is None:
        length = n // min(int(g) for g in gens) + 1
    H = np.zeros((n + 1, length), dtype=np.uint64)
    H[0, 0] = 1
    for g in gens:
        g = int(g)
        # rows r in [j*g, (j+1)*g) depend only on rows r-g of the previous block
        for start in range(g, n + 1, g):
            stop = min(start + g, n + 1)
            H[start:stop, 1:] += H[start - g:stop - g, :-1]
    out = [int(v) for v in H[n]]
    total = count(n, gens)
    if sum(out) != total:
        raise OverflowError("hist_u64 overflowed (sum %d != count %d)" % (sum(out), total))
    return out


def suffix_tables(n: int, gens: Sequence[int]) -> List[List[int]]:
    """S[k][r] = |Z(r, gens[k:])| for k = 0..d (S[d][r] = [r == 0])."""
    d = len(gens)
    S: List[List[int]] = [None] * (d + 1)  # type: ignore
    cur = [0] * (n + 1)
    cur[0] = 1
    S[d] = list(cur)
    for k in range(d - 1, -1, -1):
        g = int(gens[k])
        cur = list(cur)
        for r in range(g, n + 1):
            cur[r] += cur[r - g]
        S[k] = cur
    return S


def rows_before_prefix(n: int, gens: Sequence[int], prefix: Sequence[int]) -> int:
    """Number of factorizations that come strictly before every row starting with
    `prefix` in decreasing lexicographic order, i.e. the 0-based canonical row index of
    the first row with that prefix (if any)."""
    S = suffix_tables(n, gens)
    R = n
    before = 0
    for k, x in enumerate(prefix):
        g = int(gens[k])
        # rows with a_k > x (and the same earlier coordinates) come first
        top = R // g
        for y in range(top, x, -1):
            before += S[k + 1][R - y * g]
        R -= x * g
        if R < 0:
            raise ValueError("prefix overshoots n")
    return before


def work_tables(n: int, gens: Sequence[int]) -> List[List[int]]:
    """Wk[k][r] = #(a_k..a_{d-2}) with sum_j a_j g_j <= r (0-based k), i.e. the number of
    innermost-loop iterations the nested-loop oracle performs below a level-k prefix with
    residual r.  Wk[d-1][r] = 1."""
    d = len(gens)
    out: List[List[int]] = [None] * d  # type: ignore
    cur = [1] * (n + 1)  # below level d-1: the single last-coordinate test
    out[d - 1] = list(cur)
    # Z-counts of the suffix (g_k..g_{d-2}) summed over residual <= r
    z = [0] * (n + 1)
    z[0] = 1
    for k in range(d - 2, -1, -1):
        g = int(gens[k])
        for r in range(g, n + 1):
            z[r] += z[r - g]
        acc, pref = 0, [0] * (n + 1)
        for r in range(n + 1):
            acc += z[r]
            pref[r] = acc
        out[k] = pref
    return out


def count_pair(n: int, a: int, b: int) -> int:
    """|Z(n, (a, b))| = #{(x, y) >= 0 : a x + b y = n}, solved as a linear congruence (the
    definition of Z, for d = 2): with h = gcd(a, b), no solution unless h | n;
    else x must satisfy (a/h) x = n/h (mod b/h), i.e. x = x0 + k b/h with
    x0 = (n/h) (a/h)^{-1} mod (b/h), and 0 <= x <= floor(n / a)."""
    from math import gcd

    if n < 0:
        return 0
    h = gcd(a, b)
    if n % h:
        return 0
    a1, b1, n1 = a // h, b // h, n // h
    x0 = (n1 * pow(a1, -1, b1)) % b1 if b1 > 1 else 0
    top = n1 // a1
    return 0 if x0 > top else (top - x0) // b1 + 1


def count_d3(n: int, gens: Sequence[int]) -> int:
    """|Z(n, (g1, g2, g3))| as the sum over a_1 of the two-generator counts of the residual
    (Z(n, g) is the disjoint union over a_1 of {a_1} x Z(n - a_1 g_1, (g_2, g_3))).  O(n / g_1)
    Python steps: usable for d = 3 instances with n near 2^31 when g_1 is large, where the
    coin-change DP (count) would need O(n) memory and time."""
    g1, g2, g3 = (int(x) for x in gens)
    return sum(count_pair(n - x * g1, g2, g3) for x in range(n // g1 + 1))


def prefix_ranker(n: int, gens: Sequence[int]):
    """rows_before_prefix with the suffix tables computed once: returns rank(prefix) = the number
    of factorizations lex-greater (decreasing-lex order) than every row that
    starts with `prefix`, i.e. the canonical index of the first such row.  Rows lex-greater
    agree with the prefix before some coordinate k and exceed it there:
        rank(p) = sum_k sum_{y > p_k} |Z(R_k - y g_k, gens[k+1:])| = sum_k |Z(R_k - (p_k + 1) g_k, gens[k:])|
    (R_k = n - sum_{j<k} p_j g_j; the second form sums the first over y by the coin recurrence)."""
    S = suffix_tables(n, gens)

    def rank(prefix: Sequence[int]) -> int:
        R, before = n, 0
        for k, x in enumerate(prefix):
            g = int(gens[k])
            r = R - (int(x) + 1) * g
            if r >= 0:
                before += S[k][r]
            R -= int(x) * g
            if R < 0:
                raise ValueError("prefix overshoots n")
        return before

    return rank
