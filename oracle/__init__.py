"""oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, single-threaded CPU implementation of what the GPU path computes, written
from the paper and sharing no code with `paper_2405_07989_b200/`:

* `oracle/enum.c` (loaded here through ctypes): the definition of Z(n, g)
  (Sec. 1) as descending nested loops, i.e. rows in decreasing
  lexicographic order, with the four stream consumers of PAPER.md:55
  (count, length histogram, any-predicate, saved rows) and a prefix-box restriction for
  sampled checks of huge instances.
* `oracle/gf.py`: exact big-integer generating-function counts and length histograms
  (coefficient extraction from prod 1/(1 - x^g) and prod 1/(1 - x^g y)).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its cpu_baseline and
`--impl reference` legs) may import this package.  The product path never does.

Pins (tests/test_oracle.py, `-m "not gpu"`): brute force over the full box
prod [0, floor(n/g_i)] on tiny inputs; closed forms (|Z(n,(1,2))| = floor(n/2)+1,
|Z(n,(1..1))| = C(n+d-1, d-1), Popoviciu's formula, d = 1, n = 0, gcd(g) not dividing n);
PAPER.md Table 1 cardinalities; SPEC.md worked examples; invariants (row sums,
strict descent, no duplicates); SURVEY.md Sec. 8(c) golden hashes, derived independently.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

from . import gf  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "enum.c")
_LIB = os.path.join(_HERE, "liboracle.so")

PRED_NONE, PRED_LEN_LE, PRED_LEN_GE, PRED_LEN_EQ, PRED_COORD_GE = 0, 1, 2, 3, 4
TOO_LARGE = -2


class OracleTooLarge(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle/enum.c with plain gcc (-O2, no vectorisation tricks needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u64, u32p, u64p = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64)
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [
            u64, u32p, ctypes.c_int,
            ctypes.c_int, u32p, u64, u64,
            u64,
            u64p,
            u64p, u64,
            ctypes.c_int, u64, ctypes.POINTER(ctypes.c_int), u32p,
            ctypes.c_void_p, ctypes.c_int, u64,
        ]
        _lib = lib
    return _lib


def _gens(g: Sequence[int]):
    arr = (ctypes.c_uint32 * len(g))(*[int(x) for x in g])
    return arr


def run(n: int, g: Sequence[int], *, box: Optional[Tuple[Sequence[int], int, int]] = None,
        hist_len: int = 0, pred: int = PRED_NONE, pred_arg: int = 0,
        rows_B: int = 0, cap: int = 0, ceiling: int = 0):
    """Run the nested-loop oracle once.  Returns dict(count, hist, found, witness, rows)."""
    lib = _load()
    d = len(g)
    ga = _gens(g)
    if box is None:
        plen, pref, lo, hi = -1, None, 0, 0
    else:
        prefix, lo, hi = box
        plen = len(prefix)
        pref = _gens(prefix) if plen else None
    cnt = ctypes.c_uint64(0)
    hist = (ctypes.c_uint64 * hist_len)() if hist_len else None
    found = ctypes.c_int(0)
    wit = (ctypes.c_uint32 * d)()
    rows = None
    if rows_B:
        rows = ctypes.create_string_buffer(max(1, cap * d * rows_B // 8))
    rc = lib.oracle_run(n, ga, d, plen, pref, lo, hi, ceiling, ctypes.byref(cnt),
                        hist, hist_len, pred, pred_arg, ctypes.byref(found), wit,
                        ctypes.cast(rows, ctypes.c_void_p) if rows is not None else None,
                        rows_B if rows_B else 16, cap)
    if rc == TOO_LARGE:
        raise OracleTooLarge("oracle too large")
    if rc < 0:
        raise ValueError("oracle: invalid arguments (rc=%d)" % rc)
    out = {"count": cnt.value, "found": bool(found.value)}
    if hist_len:
        out["hist"] = [int(v) for v in hist]
    if pred:
        out["witness"] = [int(v) for v in wit] if found.value else None
    if rows_B:
        nrows = min(cap, cnt.value)
        out["rows"] = rows.raw[: nrows * d * rows_B // 8]
    return out


def count(n: int, g: Sequence[int], ceiling: int = 0) -> int:
    return run(n, g, ceiling=ceiling)["count"]


def hist_len_for(n: int, g: Sequence[int]) -> int:
    return n // min(int(x) for x in g) + 1


def hist(n: int, g: Sequence[int], ceiling: int = 0) -> List[int]:
    return run(n, g, hist_len=hist_len_for(n, g), ceiling=ceiling)["hist"]


def any_pred(n: int, g: Sequence[int], pred: int, arg: int, ceiling: int = 0):
    r = run(n, g, pred=pred, pred_arg=arg, ceiling=ceiling)
    return r["found"], r["witness"]


def rows(n: int, g: Sequence[int], B: int = 16, cap: Optional[int] = None, ceiling: int = 0,
         box=None) -> bytes:
    if cap is None:
        cap = run(n, g, ceiling=ceiling, box=box)["count"]
    return run(n, g, rows_B=B, cap=cap, ceiling=ceiling, box=box)["rows"]


def rows_as_tuples(raw: bytes, d: int, B: int = 16) -> List[Tuple[int, ...]]:
    import struct
    w = B // 8
    fmt = "<" + ("H" if B == 16 else "I") * d
    step = d * w
    return [struct.unpack_from(fmt, raw, i) for i in range(0, len(raw), step)]


def pred_holds(row: Sequence[int], pred: int, arg: int) -> bool:
    """The predicate semantics, restated for checking witnesses."""
    s = sum(row)
    if pred == PRED_LEN_LE:
        return s <= arg
    if pred == PRED_LEN_GE:
        return s >= arg
    if pred == PRED_LEN_EQ:
        return s == arg
    if pred == PRED_COORD_GE:
        i, k = arg >> 32, arg & 0xFFFFFFFF
        return i < len(row) and row[i] >= k
    raise ValueError(pred)
