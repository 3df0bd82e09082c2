// fs_core.cuh -- the per-lane successor stream of the factorization-set enumeration.
//
// One "lane" (a GPU thread, or the host model in csrc/fs_host.cu) owns one bounded slice of
// the decreasing-lexicographic order of Z(n, (g_1..g_d)) (Sec. 4: a bound
// partitions the lex order into disjoint worker slices) and walks it with the successor of
// PAPER.md Alg. 3.1, state in registers.
//
// Notation (0-based arrays, 1-based in comments to match the paper):
//   d generators g_1..g_d, node level L = d-2.  A "node" is a prefix (a_1..a_L) with residual
//   R_L = n - sum_{j<=L} a_j g_j >= 0.  Below a node the paper's stream runs the index-(d-1)
//   candidates a_{d-1} = ceil/floor(R_L/g_{d-1}) .. 0 with a_d solved by division
//   (decrementAndSolve).  We apply the paper's modulo optimisation at run
//   entry: the valid a_{d-1} of a node are exactly a*, a*-s, a*-2s, ... >= 0 with
//   s = g_d / gcd(g_{d-1}, g_d) (the additive order of g_{d-1} mod g_d), and a*
//   is found from the residue rho = R_L mod g_{d-1} by a table lookup k0(rho), a* = A - k0,
//   A = floor(R_L / g_{d-1}).  Every valid factorization of the node is then one "row".
//
//   The paper's overshoot candidate (.., ceil(R/g), 0, ..) is invalid unless the division is
//   exact, in which case it equals the floor candidate; its successor is the floor candidate
//   with one more coordinate solved.  The lane goes straight to the floor
//   candidate: it visits every node the paper's stream visits, in the same order, and emits
//   the same factorizations in the same order (Thm. 3.2/3.3).
//
// Units and slices: a slice is a range of units of the stream.  Count / histogram / any
// plans use NODE units (alpha = 1, beta = 0): a slice owns whole nodes with all their rows.
// Materialise plans use ROW units (alpha = 0, beta = 1): a slice owns exactly T rows, so it
// writes them at exact canonical offsets.  The exact DP tables U[k][r] (units below a
// level-k node with residual r) let a lane jump to any unit index (unrank) and run exactly
// `budget` units, so slices are disjoint, gap-free and equal in work (a finer, exact form of
// the paper's bound splitting, and of its "better work division").
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define FS_HD __host__ __device__ __forceinline__
#else
#define FS_HD inline
#endif

#ifndef FS_MAX_D
#define FS_MAX_D 16
#endif

namespace fs {

constexpr uint32_t kNone = 0x7FFFFFFFu;  // "no valid a_{d-1} in this node"

// 31-bit magic division: q = floor(x / g) for x < 2^31 via one 32x32->64 multiply and a
// shift: l = ceil(log2 g), m = floor(2^(31+l)/g) + 1 < 2^32, sh = 31 + l.  (m g = 2^(31+l)
// + e with 0 < e <= 2^l, so x m / 2^(31+l) = x/g + x e/(g 2^(31+l)) and the error term is
// < 1/g for x < 2^31.)
struct Div {
  uint32_t m, sh;
};

FS_HD uint32_t divq(uint32_t x, Div v) { return (uint32_t)(((uint64_t)x * v.m) >> v.sh); }

// Instance constants as the lanes see them (passed by value in the kernel parameters).
struct Consts {
  uint32_t n;
  int d;
  uint32_t g[FS_MAX_D];
  Div dv[FS_MAX_D];
  uint32_t gA, gB;       // g_{d-1}, g_d
  uint32_t h, s, t, inv; // h = gcd(gA,gB), s = gB/h, t = gA/h, inv = t^{-1} mod s
  Div dvA, dvB, dvH, dvS;
  uint32_t delta, q;     // g_L mod gA, g_L / gA (L >= 1)
  uint32_t cB;           // gA mod gB (skip ablation: residue step of one a_{d-1} decrement)
  uint32_t alpha, beta;  // units per node entry / per row
  uint32_t ktab_len;     // 0: k0 by arithmetic; else words of the node tables (below)
  uint32_t adv_off;      // word offset of the advance table inside ktab (8 B aligned)
  uint32_t cadv_off;     // word offset of the closed-tail group table (0: none; see fs_host.cu)
  uint32_t cadv_words;   // words per group-table entry: 2 (count, packed histogram) or 4 (histogram)
  uint32_t cadv_packed;  // histogram entry {link, (s - k0) | (ad0 - k0 + 2^15) << 16}
  uint32_t mhi;          // ceil(2^32 / s) for the group table's umulhi division
  uint32_t t2_off;       // word offset of the count's one-level ascend table (0: none; fs_host.cu)
  uint32_t cadv2_off;    // word offset of the count's paired closed-tail table (0: none; fs_host.cu)
  uint32_t cadv2_skip;   // 1: that table walks live nodes only (8 words per entry; NEXT-3)
  uint32_t t3_off;       // word offset of the count's two-level ascend table (0: none; fs_host.cu)
  uint32_t hadv_off;     // word offset of the histogram's 8-copy closed-tail table (0: none; fs_host.cu)
  uint32_t hadv_skip;    // 1: that table walks live nodes only (gcd(g_{d-1}, g_d) > 1; NEXT-3)
  uint32_t qtab_off;     // word offset of the count's state-pair table (0: none; fs_host.cu)
  uint32_t q1_off;       // word offset of its single-step table
  uint32_t t2q_off;      // word offset of the count's one-level ascend table in state form (0: none)
  uint32_t hq_off;       // word offset of the histogram's state-form table (0: none; fs_host.cu)
  uint32_t hq_bias;      // its difference-array index bias (s - 1: rowless nodes reach index -(s-1))
  uint32_t radv_off;     // word offset of the materialise advance table (0: none; fs_host.cu):
                         //   4 words per rho {next | inc << 11, k0(next), ad0(next), 0}
  // NEXT-3 for k >= 3 trailing generators: bit j (0-based coordinate j <= L - 2) set
  // when G_j = gcd(g_{j+1}, .., g_d) > 1 -- a node (a_1..a_j) whose residual G_j does not divide
  // roots a subtree without factorizations, which advance_cd() skips (charging its DP units)
  uint32_t cd_mask;
  uint32_t cd_g[FS_MAX_D];
  Div cd_dv[FS_MAX_D];
  int32_t dl;            // t - s: change of a row's length from one valid a_{d-1} to the next
  uint32_t dstride;      // stride of the closed-tail length-difference array (|dl|, or 1 if 0)
  uint8_t perm[FS_MAX_D];  // internal coordinate j is the caller's coordinate perm[j]
  uint32_t permuted;       // perm is not the identity
  const uint64_t *U;     // DP tables: V0[x] = U[0][n - x g_1] (u0_len entries), then U[1..L-1][0..n]
  uint32_t u0_len;       // floor(n / g_1) + 1
  // node tables (device or host), for rho in [0, g_{d-1}) (g_{d-1} <= 2048):
  //   ktab[rho]                     = k0(rho)
  //   ktab[adv_off + 2 rho]         = next(rho) | (q + carry(rho)) << 11,
  //                                   next = (rho + delta) mod g_{d-1}
  //   ktab[adv_off + 2 rho + 1]     = k0(next(rho))
  // i.e. one 8 B load performs a node advance's residue and quotient update and the new
  // node's entry.
  const uint32_t *ktab;
};

#ifdef __CUDA_ARCH__
FS_HD uint64_t ldU(const uint64_t *p) { return __ldg(p); }
#else
FS_HD uint64_t ldU(const uint64_t *p) { return *p; }
#endif

// smallest k >= 0 with g_d | rho + k g_{d-1}, or kNone (P:172 congruence)
FS_HD uint32_t k0_arith(uint32_t rho, const Consts &c) {
  uint32_t rq = divq(rho, c.dvH);
  if (rq * c.h != rho) return kNone;
  uint32_t rs = rq - divq(rq, c.dvS) * c.s;
  uint32_t neg = rs ? c.s - rs : 0u;
  return (uint32_t)(((uint64_t)neg * c.inv) % c.s);
}

template <int D>
struct Lane {
  static constexpr int L = D - 2;
  static constexpr int LA = (D - 2) > 0 ? (D - 2) : 1;
  uint32_t a[LA];  // a_1..a_L
  uint32_t R[LA];  // R_1..R_L
  uint32_t A, rho; // floor(R_L / g_{d-1}), R_L mod g_{d-1}
  int32_t cur;     // current row's a_{d-1} (< 0: none left in this node)
  uint32_t ad;     // unused placeholder (a_d is solved on demand by row_ad())
  uint32_t lsum;   // a_1 + .. + a_L (tracked when the consumer needs lengths/coordinates)
  // Lazy counters of the fast path: k = node advances still allowed before a sync (at most
  // min(budget, a_L)); kb = its value at the last sync.  Between syncs, a_L, lsum and (node
  // units) the budget are behind by (kb - k); see sync_k / cur_aL / cur_lsum.
  uint32_t k, kb;
  uint32_t e;      // skip ablation only: (R_L - a_{d-1} g_{d-1}) mod g_d of the current candidate
};

template <int D>
FS_HD uint32_t cur_aL(const Lane<D> &st) {  // a_L as of now
  if constexpr (D >= 3)
    return st.a[D - 3] - (st.kb - st.k);
  else
    return 0;
}
template <int D>
FS_HD uint32_t cur_lsum(const Lane<D> &st) {
  return st.lsum - (st.kb - st.k);
}
// row coordinate j < L as of now
template <int D>
FS_HD uint32_t cur_coord(const Lane<D> &st, int j) {
  if constexpr (D >= 3)
    return j == D - 3 ? cur_aL<D>(st) : st.a[j];
  else
    return 0;
}

// Apply the fast path's pending advances to a_L, lsum and the budget, and re-arm k.
template <int D, int ALPHA>
FS_HD void sync_k(Lane<D> &st, uint32_t &budget) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    const uint32_t used = st.kb - st.k;
    st.a[L - 1] -= used;
    st.lsum -= used;
    if (ALPHA) budget -= used;
    const uint32_t al = st.a[L - 1];
    st.k = ALPHA ? (budget < al ? budget : al) : al;
    st.kb = st.k;
  } else {
    st.k = st.kb = 0;
  }
}

// Node-table lookups: k0(rho), and step(rho) = the advance transition (next residue, carry,
// k0 of the next residue) -- from the tables (host vector, or a shared-memory copy on the
// device), or by arithmetic when g_{d-1} is too large for a table.
struct Adv {
  uint32_t next, k0, inc;  // next residue, k0(next), increment of floor(R_L / g_{d-1})
};
constexpr uint32_t kAdvBits = 11;  // next < 2^11 in the packed table word
constexpr uint32_t kCAdvShift = 16;  // count group table: byte offset < 2^16 below the increment
FS_HD uint32_t adv_pack(uint32_t next, uint32_t inc) { return next | (inc << kAdvBits); }
FS_HD Adv adv_unpack(uint32_t w0, uint32_t w1) {
  return Adv{w0 & ((1u << kAdvBits) - 1u), w1, w0 >> kAdvBits};
}
struct KTabPtr {
  const uint32_t *p;
  uint32_t adv_off;
  FS_HD uint32_t operator()(uint32_t rho, const Consts &) const { return p[rho]; }
  FS_HD Adv step(uint32_t rho, const Consts &) const {
    return adv_unpack(p[adv_off + 2 * rho], p[adv_off + 2 * rho + 1]);
  }
};
struct KTabArith {
  FS_HD uint32_t operator()(uint32_t rho, const Consts &c) const { return k0_arith(rho, c); }
  FS_HD Adv step(uint32_t rho, const Consts &c) const {
    uint32_t r2 = rho + c.delta;
    const uint32_t cy = r2 >= c.gA ? 1u : 0u;
    r2 -= cy ? c.gA : 0u;
    return Adv{r2, k0_arith(r2, c), c.q + cy};
  }
};

// Node entry: solve the first valid a_{d-1} of the node (modulo skip at run entry).
template <int D, bool NEED_AD, class KT>
FS_HD void entry(Lane<D> &st, const Consts &c, const KT &kt) {
  const uint32_t k = kt(st.rho, c);
  st.cur = (int32_t)st.A - (int32_t)k;  // A <= n < 2^31 - 1, so kNone gives cur < 0
  (void)NEED_AD;
}

// The last coordinate of the current row, solved by division (decrementAndSolve):
// a_d = (R_L - a_{d-1} g_{d-1}) / g_d, exact for a valid row.
// (R_L = A g_{d-1} + rho, so R_L - a_{d-1} g_{d-1} = (A - a_{d-1}) g_{d-1} + rho.)
template <int D>
FS_HD uint32_t row_ad(const Lane<D> &st, const Consts &c) {
  return divq((st.A - (uint32_t)st.cur) * c.gA + st.rho, c.dvB);
}

// Deeper ascend of Alg. 3.1 steps 2-11: rightmost nonzero index i < L, a_i -= 1,
// re-solve a_{i+1}..a_L greedily (floor) -- returns false at end of stream.
// (CC: Consts, or any struct with the same g / dv / gA / dvA members, e.g. a register copy)
template <int D, class CC = Consts>
FS_HD bool ascend(Lane<D> &st, const CC &c) {
  constexpr int L = D - 2;
  if constexpr (L <= 1) {
    return false;
  } else {
    if (st.a[L - 2] > 0) {  // common case: one level up
      st.a[L - 2]--;
      uint32_t r = st.R[L - 2] + c.g[L - 2];
      st.R[L - 2] = r;
      uint32_t x = divq(r, c.dv[L - 1]);
      st.a[L - 1] = x;
      r -= x * c.g[L - 1];
      st.R[L - 1] = r;
      uint32_t A = divq(r, c.dvA);
      st.A = A;
      st.rho = r - A * c.gA;
      st.lsum = st.lsum - 1 + x;
      return true;
    }
    int k = -1;
#pragma unroll
    for (int j = 0; j < L - 2; ++j)
      if (st.a[j] > 0) k = j;
    if (k < 0) return false;
#pragma unroll
    for (int j = 0; j < L - 2; ++j)
      if (j == k) {
        st.a[j]--;
        st.R[j] += c.g[j];
      }
    uint32_t lsum = 0;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      if (j > k) {
        uint32_t r = st.R[j - 1];
        uint32_t x = divq(r, c.dv[j]);
        st.a[j] = x;
        st.R[j] = r - x * c.g[j];
      }
      lsum += st.a[j];
    }
    uint32_t r = st.R[L - 1];
    uint32_t A = divq(r, c.dvA);
    st.A = A;
    st.rho = r - A * c.gA;
    st.lsum = lsum;
    return true;
  }
}

// Move to the next node in decreasing lex order; false at end of stream.
template <int D>
FS_HD bool advance(Lane<D> &st, const Consts &c) {
  constexpr int L = D - 2;
  if constexpr (L == 0) {
    return false;
  } else {
    if (st.a[L - 1] > 0) {
      st.a[L - 1]--;
      st.R[L - 1] += c.g[L - 1];
      uint32_t r2 = st.rho + c.delta;
      uint32_t carry = r2 >= c.gA ? 1u : 0u;
      st.rho = carry ? r2 - c.gA : r2;
      st.A += c.q + carry;
      st.lsum--;
      return true;
    }
    return ascend<D>(st, c);
  }
}

// NEXT-3 beyond the last two generators ("the same applies if the last n generators
// share a common denominator"): after an ascend, a node (a_1..a_j), j <= L - 1, whose residual
// is not a multiple of G_j = gcd(g_{j+1}, .., g_d) has no factorization below it.  The lane is at
// the first node of that subtree (the ascend re-solved every deeper coordinate greedily), so
// the subtree's units -- U[j][R_j] - U[j][R_j - g_j] from the exact DP, node entries for
// count / hist / any plans, rows (none) for materialise -- are charged at once, the deeper
// coordinates are zeroed (the lane stands on the subtree's last node) and the ascend repeats.
// Returns false at end of stream, or when the slice's budget ends inside a dead subtree.
// (0-based below: coordinate q <= L - 2 has residual R[q] and divisor cd_g[q].)
// The level an ascend from this state decrements: the rightmost nonzero a[q], q <= L - 2.
template <int D>
FS_HD int ascend_level(const Lane<D> &st) {
  constexpr int L = D - 2;
  int k = -1;
#pragma unroll
  for (int j = 0; j < L - 1; ++j)
    if (st.a[j] > 0) k = j;
  return k;
}

template <int D, int ALPHA>
FS_HD bool ascend_cd(Lane<D> &st, const Consts &c, uint32_t &budget) {
  constexpr int L = D - 2;
  if constexpr (L >= 2) {
    for (;;) {
      const int k = ascend_level<D>(st);
      if (!ascend<D>(st, c)) return false;
      // the new subtrees are those at levels k .. L - 2 (the lane stands on their first node)
      int j = -1;
#pragma unroll
      for (int q = 0; q < L - 1; ++q)
        if (j < 0 && q >= k && ((c.cd_mask >> q) & 1u) && st.R[q] != divq(st.R[q], c.cd_dv[q]) * c.cd_g[q]) j = q;
      if (j < 0) return true;
      if (ALPHA) {
        uint64_t u;
        if (j == 0) {
          const uint32_t top = divq(c.n, c.dv[0]), x = st.a[0];
          u = ldU(c.U + x) - (x < top ? ldU(c.U + x + 1) : 0ull);
        } else {
          const uint64_t *Uj = c.U + c.u0_len + (uint64_t)(j - 1) * ((uint64_t)c.n + 1);
          const uint32_t r = st.R[j];
          u = ldU(Uj + r) - (r >= c.g[j] ? ldU(Uj + r - c.g[j]) : 0ull);
        }
        if (u >= budget) {  // the slice ends inside the dead subtree: nothing left to emit
          budget = 0;
          return false;
        }
        budget -= (uint32_t)u;
      }
      uint32_t lsum = 0;
#pragma unroll
      for (int q = 0; q < L; ++q) {
        if (q > j) {
          st.a[q] = 0;
          st.R[q] = st.R[q - 1];
        }
        lsum += st.a[q];
      }
      st.lsum = lsum;
    }
  } else {
    (void)budget;
    return ascend<D>(st, c);
  }
}

template <int D, int ALPHA>
FS_HD bool advance_cd(Lane<D> &st, const Consts &c, uint32_t &budget) {
  constexpr int L = D - 2;
  if constexpr (L >= 2) {
    if (c.cd_mask && st.a[L - 1] == 0) return ascend_cd<D, ALPHA>(st, c, budget);
  }
  return advance<D>(st, c);
}

// Position the lane at global unit index u (exact, from the DP tables), perform the node
// entry, and return the offset of u inside the node's unit list (0 = the entry unit when
// alpha = 1).
template <int D, bool NEED_AD, class KT>
FS_HD uint64_t unrank(Lane<D> &st, const Consts &c, const KT &kt, uint64_t u) {
  constexpr int L = D - 2;
  uint32_t R = c.n;
  uint32_t lsum = 0;
  const uint64_t stride = (uint64_t)c.n + 1;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    // level 0 is stored compactly (entry x = U[0][n - x g_1]); levels >= 1 in full
    const uint64_t *Uk = k == 0 ? c.U : c.U + c.u0_len + (uint64_t)(k - 1) * stride;
    const uint32_t g = c.g[k];
    uint32_t top = divq(R, c.dv[k]);
    // cum(x) = U[k][R - x g] = units of the subtrees a_k in [x, top]; nonincreasing in x.
    uint32_t lo = 0, hi = top + 1;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (ldU(Uk + (k == 0 ? mid : R - mid * g)) > u)
        lo = mid;
      else
        hi = mid;
    }
    if (lo < top) u -= ldU(Uk + (k == 0 ? lo + 1 : R - (lo + 1) * g));
    st.a[k] = lo;
    R -= lo * g;
    st.R[k] = R;
    lsum += lo;
  }
  uint32_t A = divq(R, c.dvA);
  st.A = A;
  st.rho = R - A * c.gA;
  st.lsum = lsum;
  st.k = st.kb = 0;
  entry<D, NEED_AD>(st, c, kt);
  return u;
}

// Unit range [u, e) of slice `sl` of a rank's range [unit0, unit1).  Node-unit plans cut the
// range in three phases (guided slices, fs_host.cu): n0 slices of 4T units, n1 of 2T, then slices
// of T -- large slices while there is plenty of work (fewer refills), small ones at the end (a
// short tail); row-unit plans and forced slice sizes use n0 = n1 = 0 (uniform T).
FS_HD void slice_range(uint64_t unit0, uint64_t unit1, uint64_t T, uint64_t n0, uint64_t n1, uint64_t sl,
                       uint64_t &u, uint64_t &e) {
  uint64_t off, len;
  if (sl < n0) {
    off = sl * 4 * T;
    len = 4 * T;
  } else if (sl < n0 + n1) {
    off = n0 * 4 * T + (sl - n0) * 2 * T;
    len = 2 * T;
  } else {
    off = n0 * 4 * T + n1 * 2 * T + (sl - n0 - n1) * T;
    len = T;
  }
  u = unit0 + off;
  e = u + len < unit1 ? u + len : unit1;
}

// Equal-COST slicing (node-unit plans, L >= 2; fs_host.cu).  CW[k][r] = cost below a level-k
// prefix with residual r: w_node per level-L node plus w_run per run (a level-(L-1) prefix: the
// level-L nodes it holds plus its ascend), stored like U (level 0 compactly: entry x =
// CW[0][n - x g_1]).  cost_boundary(target) is the node-unit index of the start of the run in
// which the lex-ordered cumulative cost passes `target` (the total units for target >= total
// cost); pre[0..L-1] receives that run's first node (a_L at its maximum).  Rank partitions and
// slices both cut the lex order there, so every slice starts at a run start.
template <int D>
FS_HD uint64_t cost_boundary(const Consts &c, const uint64_t *CW, uint64_t target, uint32_t *pre) {
  constexpr int L = D - 2;
  uint64_t units = 0;
  if constexpr (L >= 2) {
    const uint64_t stride = (uint64_t)c.n + 1;
    uint32_t R = c.n;
    uint64_t rem = target;
    if (target >= ldU(CW)) {  // past the end: no run
      for (int k = 0; k < L; ++k) pre[k] = 0;
      return ldU(c.U);
    }
#pragma unroll
    for (int k = 0; k < L - 1; ++k) {
      const uint64_t *Ck = k == 0 ? CW : CW + c.u0_len + (uint64_t)(k - 1) * stride;
      const uint64_t *Uk = k == 0 ? c.U : c.U + c.u0_len + (uint64_t)(k - 1) * stride;
      const uint32_t g = c.g[k];
      const uint32_t top = divq(R, c.dv[k]);
      // cost of the subtrees a_k >= x is Ck[R - x g] (nonincreasing in x): the largest x whose
      // subtrees a_k >= x cost more than rem holds the boundary
      uint32_t lo = 0, hi = top + 1;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ldU(Ck + (k == 0 ? mid : R - mid * g)) > rem)
          lo = mid;
        else
          hi = mid;
      }
      if (lo < top) {
        rem -= ldU(Ck + (k == 0 ? lo + 1 : R - (lo + 1) * g));
        units += ldU(Uk + (k == 0 ? lo + 1 : R - (lo + 1) * g));
      }
      R -= lo * g;
      pre[k] = lo;
    }
    pre[L - 1] = divq(R, c.dv[L - 1]);  // the run's first node: a_L at its maximum
  }
  return units;
}

FS_HD uint64_t bitrev_bits(uint64_t x, uint32_t bits) {
#ifdef __CUDA_ARCH__
  return bits ? (__brevll(x) >> (64 - bits)) : 0ull;
#else
  uint64_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1ull) << (bits - 1u - i);
  return r;
#endif
}

// Any-predicate claim order (KParams::permute): both ends of the lex order early.  Even claims
// walk the front half of the S slices in bit-reversed order, odd claims the back half mirrored
// -- claim 0 is the lex-first slice, claim 1 the lex-last, then the middles -- so a witness
// near either end (C5 P_first / P_late) is met in the first wave and every region is sampled
// early.  A bijection of [0, S) over the 2^bits claims; the rest map to ~0 (skipped).
FS_HD uint64_t claim_slice(uint64_t idx, uint32_t bits, uint64_t S) {
  const uint64_t j = bitrev_bits(idx >> 1, bits ? bits - 1u : 0u);
  if (idx & 1ull) return j < (S >> 1) ? S - 1ull - j : ~0ull;
  return j < ((S + 1ull) >> 1) ? j : ~0ull;
}

// Cost target of the start of slice j of an equal-cost guided slicing of [cb, ce): P phases of
// Lp slices, phase k's slices of cost 2^(P-1-k) c with c = (ce - cb) / (Lp (2^P - 1)).
FS_HD uint64_t cost_target(uint64_t cb, uint64_t ce, uint64_t Lp, uint64_t P, uint64_t S, uint64_t j) {
  // P phases of Lp slices each; phase k's slices weigh 2^(P-1-k) (S = P Lp; slice S is the end)
  (void)S;
  const uint64_t k = j / Lp, i = j - k * Lp;
  const uint64_t f = k >= P ? Lp * ((1ull << P) - 1) : Lp * ((1ull << P) - (1ull << (P - k))) + i * (1ull << (P - 1 - k));
  return cb + (uint64_t)((unsigned __int128)(ce - cb) * f / (Lp * ((1ull << P) - 1)));
}

// After unrank(): node-unit plans (alpha = 1) start at the node's entry, which is consumed
// here (returns 1); row-unit plans (alpha = 0) skip to row `off` of the node (returns 0).
template <int D, bool NEED_AD>
FS_HD uint32_t position_in_node(Lane<D> &st, const Consts &c, uint64_t off) {
  if (c.alpha) return 1;  // off == 0: node units never split a node
  st.cur -= (int32_t)((uint32_t)off * c.s);
  return 0;
}

// A lane needs a new slice when its budget is spent and -- for node-unit slices, whose last
// node's rows all belong to the slice -- its current node has no rows left.
template <int D, int ALPHA>
FS_HD bool needs_refill(const Lane<D> &st, uint32_t budget) {
  return ALPHA ? (budget == 0 && st.cur < 0) : (budget == 0);
}

// Slow step, for a lane whose node is exhausted and whose level-L coordinate is 0: Alg. 3.1
// steps 2-11 at an index i < L (ascend() re-solves a_{i+1}..a_L greedily), then the new
// node's entry (one ENTRY unit).  It never emits: the node's first row, if any, is emitted
// by the next fast_step, so every emission happens with the warp converged.
// (CD = false: without the k >= 3 dead-subtree skip -- the kernels instantiate it only in their
// NEXT-3 variants, so the common kernels keep the short ascend)
template <int D, bool NEED_AD, int ALPHA, bool CD = true, class KT>
FS_HD void slow_step(Lane<D> &st, const Consts &c, const KT &kt, uint32_t &budget) {
  if (!(CD ? advance_cd<D, ALPHA>(st, c, budget) : advance<D>(st, c))) {
    budget = 0;  // end of stream
    return;
  }
  entry<D, NEED_AD>(st, c, kt);
  budget -= ALPHA;
}

// Branch-free fast step for SIMT lanes.  Every lane does, under predicates:
//   - a row lane (cur >= 0) emits its row and steps a_{d-1} -= s;
//   - a lane with budget whose node is exhausted and whose level-L coordinate a_L > 0
//     advances to the next node (a_L -= 1, residual += g_L, incremental floor/residue of R_L
//     by g_{d-1}), solves the node's first valid row through k0 and emits it (row units:
//     budget permitting).
// Lanes that need the rare ascend (a_L = 0) or end of stream do nothing here and are left for
// slow_step() (needs_slow()).
template <int D, bool NEED_AD, int ALPHA, class KT, class Emit>
FS_HD void fast_step(Lane<D> &st, const Consts &c, const KT &kt, uint32_t &budget, Emit &emit) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    // k > 0 <=> a_L > 0 and (node units) budget left, as of the last sync
    const bool fa = st.cur < 0 && st.k != 0;
    // one table load: next residue of R_L + g_L mod g_{d-1}, the carry into floor(R_L/g_{d-1}),
    // and k0 of the next residue (all lanes load; only advancing lanes commit)
    const Adv w = kt.step(st.rho, c);
    if (fa) {  // advance (a_L -= 1, R_L += g_L, lazily via k) and entry of the new node
      st.k -= 1u;
      st.rho = w.next;
      st.A += w.inc;
      st.cur = (int32_t)st.A - (int32_t)w.k0;
    }
  }
  // node units: every row of an entered node belongs to the slice; row units: budget-limited
  const bool em = ALPHA ? (st.cur >= 0) : (st.cur >= 0 && budget != 0);
  emit.cond(em, st, c);
  if (em) {
    st.cur -= (int32_t)c.s;
    if (!ALPHA) budget -= 1u;
  }
}

// NEXT-1 of SURVEY Sec. 8(f) (the paper's "dynamic behavior" future work, in its
// cheapest closed form): for the COUNT consumer a node's valid a_{d-1} form the progression
// a*, a*-s, ..., so its rows are counted in O(1) as floor(a*/s) + 1 (one magic division)
// instead of one step per row.  Node-unit slices only (a slice owns whole nodes), so the
// slice boundaries are those of fast_step.
//
// Node consumers (NodeEmit::node(em, st, c, rows) receives the whole progression at once):
// the count adds `rows`; the length histogram adds the progression's lengths
// l_j = l_0 + j (t - s), j < rows, as two updates of a strided difference array.
template <int D, class KT, class NodeEmit>
FS_HD void fast_step_closed(Lane<D> &st, const Consts &c, const KT &kt, uint32_t &budget, NodeEmit &ne) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    const bool fa = st.cur < 0 && st.k != 0;
    const Adv w = kt.step(st.rho, c);
    if (fa) {
      st.k -= 1u;
      st.rho = w.next;
      st.A += w.inc;
      st.cur = (int32_t)st.A - (int32_t)w.k0;
    }
  }
  const bool em = st.cur >= 0;  // node units: the node's rows all belong to this slice
  const uint32_t rows = divq((uint32_t)(em ? st.cur : 0), c.dvS) + 1u;
  ne.node(em, st, c, rows);
  if (em) st.cur = -1;
}

// Count-only closed step: rows = floor(max(cur + s, 0) / s), which is floor(a*/s) + 1 for a
// node with rows (cur = a* >= 0) and 0 otherwise (cur < 0), so no compare/select is needed
// (cur + s <= n + g_d < 2^31 keeps the magic division exact).  One node can hold up to
// ~n / (g_{d-1} s) < 2^31 rows, so the count is accumulated in 64 bits here.
template <int D, class KT>
FS_HD void fast_step_count_closed(Lane<D> &st, const Consts &c, const KT &kt, uint64_t &cnt) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    const bool fa = st.cur < 0 && st.k != 0;
    const Adv w = kt.step(st.rho, c);
    if (fa) {
      st.k -= 1u;
      st.rho = w.next;
      st.A += w.inc;
      st.cur = (int32_t)st.A - (int32_t)w.k0;
    }
  }
  const int32_t x = st.cur + (int32_t)c.s;
  cnt += divq((uint32_t)(x > 0 ? x : 0), c.dvS);
  st.cur = -1;
}

// NEXT-1 for the any-predicate (fs_any): a node's rows j < rows are (a_1..a_L, a* - j s,
// ad* + j t) with lengths l0 + j (t - s), so each predicate of fs_any holds for some row of the
// node iff it holds at the row where the tested quantity is extreme -- or, for LEN_EQ, at the
// one j solving l0 + j (t - s) = X.  Decided in O(1) per node; jw = a witness row's index.
// (COORD_GE's coordinate index is the stream's internal index, remapped on the host.)
template <int D>
FS_HD bool any_closed_pick(const Lane<D> &st, const Consts &c, uint32_t rows, int pred, uint64_t arg,
                           uint32_t &jw) {
  const uint32_t ad = row_ad<D>(st, c);  // a_d of row 0 (a_{d-1} = a* = cur)
  const int64_t l0 = (int64_t)cur_lsum<D>(st) + (int64_t)(uint32_t)st.cur + (int64_t)ad;
  const int64_t dl = c.dl;
  const uint32_t last = rows - 1u;
  switch (pred) {
    case FS_PRED_LEN_LE:
      jw = dl >= 0 ? 0u : last;
      return (uint64_t)(l0 + (int64_t)jw * dl) <= arg;
    case FS_PRED_LEN_GE:
      jw = dl > 0 ? last : 0u;
      return (uint64_t)(l0 + (int64_t)jw * dl) >= arg;
    case FS_PRED_LEN_EQ: {
      if (arg >= (1ull << 40)) return false;  // lengths are < 2^32
      const int64_t diff = (int64_t)arg - l0;
      if (dl == 0) {
        jw = 0u;
        return diff == 0;
      }
      if (diff % dl != 0) return false;
      const int64_t j = diff / dl;
      if (j < 0 || j > (int64_t)last) return false;
      jw = (uint32_t)j;
      return true;
    }
    default: {
      const uint32_t i = (uint32_t)(arg >> 32), k = (uint32_t)(arg & 0xffffffffu);
      if (i + 2u < (uint32_t)D) {
        jw = 0u;
        return cur_coord<D>(st, (int)i) >= k;
      }
      if (i + 2u == (uint32_t)D) {  // a_{d-1}: largest at row 0
        jw = 0u;
        return (uint32_t)st.cur >= k;
      }
      if (i + 1u == (uint32_t)D) {  // a_d: largest at the last row
        jw = last;
        return (uint64_t)ad + (uint64_t)last * c.t >= (uint64_t)k;
      }
      return false;
    }
  }
}

struct NodeCount {
  uint32_t n;
  template <int D>
  FS_HD void node(bool em, const Lane<D> &, const Consts &, uint32_t rows) {
    n += em ? rows : 0u;
  }
};

// The two difference-array updates of a node's length progression: +v at lo, -v at hi
// (hi = lo + rows * dstride).  dl == 0: all rows share one length (v = rows, stride 1).
template <int D>
FS_HD void hist_diff_updates(const Lane<D> &st, const Consts &c, uint32_t rows, uint32_t &lo, uint32_t &hi,
                             uint32_t &v) {
  const uint32_t l0 = cur_lsum<D>(st) + (uint32_t)st.cur + row_ad<D>(st, c);
  if (c.dl == 0) {
    lo = l0;
    hi = l0 + 1u;
    v = rows;
  } else {
    lo = c.dl > 0 ? l0 : l0 - (rows - 1u) * (uint32_t)(-c.dl);
    hi = lo + rows * c.dstride;
    v = 1u;
  }
}

// Skip ablation: the paper's literal index-(d-1) loop.  A node's
// candidates a_{d-1} = A, A-1, ..., 0 are visited one per step and tested by the residue
// e = (R_L - a_{d-1} g_{d-1}) mod g_d (Skip=off); with PAPER, a valid candidate is followed
// by a jump of s (the paper's modulo optimisation; single steps once a_{d-1} < s,
// SURVEY 8c #9).  Count consumer, node units; same slices and result as the other tails.
template <int D>
FS_HD void enter_candidates(Lane<D> &st, const Consts &c) {
  st.cur = (int32_t)st.A;
  st.e = st.rho - divq(st.rho, c.dvB) * c.gB;
}

template <int D, bool PAPER, class KT>
FS_HD void fast_step_cand(Lane<D> &st, const Consts &c, const KT &kt, uint32_t &budget, uint32_t &cnt) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    const bool fa = st.cur < 0 && st.k != 0;
    const Adv w = kt.step(st.rho, c);
    if (fa) {
      st.k -= 1u;
      st.rho = w.next;
      st.A += w.inc;
      st.cur = (int32_t)st.A;
      st.e = w.next - divq(w.next, c.dvB) * c.gB;
    }
  }
  if (st.cur >= 0) {
    const bool valid = st.e == 0;
    cnt += valid ? 1u : 0u;
    if (PAPER && valid && st.cur >= (int32_t)c.s) {
      st.cur -= (int32_t)c.s;  // the next candidate is valid again
    } else {
      st.cur -= 1;
      const uint32_t e2 = st.e + c.cB;
      st.e = e2 >= c.gB ? e2 - c.gB : e2;
    }
  }
  (void)budget;
}

// (called after sync_k)
template <int D>
FS_HD bool needs_slow(const Lane<D> &st, uint32_t budget) {
  constexpr int L = D - 2;
  if constexpr (L >= 1)
    return budget != 0 && st.cur < 0 && st.a[L - 1] == 0;
  else
    return budget != 0 && st.cur < 0;
}

// units below a node with residual r (the DP base): alpha + beta * #valid a_{d-1}
FS_HD uint64_t node_units_host(uint32_t r, const Consts &c, const uint32_t *ktab) {
  uint32_t A = r / c.gA, rho = r % c.gA;
  uint32_t k = ktab ? ktab[rho] : k0_arith(rho, c);
  uint64_t rows = 0;
  if (k != kNone && k <= A) rows = (A - k) / c.s + 1;
  return (uint64_t)c.alpha + (uint64_t)c.beta * rows;
}

}  // namespace fs
