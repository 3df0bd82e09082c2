// fs_host.cu -- host side of the CUDA path: instance validation (PAPER.md:28 footnote 1 --
// generators taken as given), device constants (magic division, modulo-skip congruence
// constants), the exact DP tables that size the slices (not in the paper; serves
// its "work division improvement"), the W-way partition of the lex order
// (P:196-200), device upload, and the host model used by CPU tests.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/fsgpu.h"
#include "../../include/fsgpu_debug.h"
#include "fs_core.cuh"
#include "fs_internal.h"

using fs::Consts;
using fs::Div;

typedef unsigned __int128 u128;


fs::Div fs_make_div(uint32_t g) {
  uint32_t l = 0;
  while (((uint64_t)1 << l) < g) ++l;  // l = ceil(log2 g)
  uint64_t m = (((uint64_t)1 << (31 + l)) / g) + 1;
  Div v;
  v.m = (uint32_t)m;
  v.sh = 31 + l;
  return v;
}

static uint32_t gcd32(uint32_t a, uint32_t b) {
  while (b) {
    uint32_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// inverse of t modulo s (gcd(t, s) = 1); s == 1 -> 0
static uint32_t inv_mod(uint32_t t, uint32_t s) {
  if (s == 1) return 0;
  int64_t r0 = s, r1 = t % s, x0 = 0, x1 = 1;
  while (r1) {
    int64_t qq = r0 / r1, tmp = r0 - qq * r1;
    r0 = r1;
    r1 = tmp;
    tmp = x0 - qq * x1;
    x0 = x1;
    x1 = tmp;
  }
  int64_t v = x0 % (int64_t)s;
  if (v < 0) v += s;
  return (uint32_t)v;
}

static uint64_t ceil_div_u64(uint64_t a, uint64_t b) { return a / b + (a % b ? 1 : 0); }

// target number of resident lanes used to size slices when the caller does not (a B200
// holds 148 SMs x 2048 threads; the persistent grid uses about half that at ~64 regs)
static const uint64_t kTargetLanes = 148ull * 1024ull;
#ifndef FS_SLICES_PER_LANE
#define FS_SLICES_PER_LANE 16
#endif
static const uint64_t kSlicesPerLane = FS_SLICES_PER_LANE;

int fs_validate_and_build(fs_plan *p, uint64_t n, const uint32_t *gens, int d, int consumer,
                          const fs_exec_t *ex) {
  if (d < 1 || d > FS_MAX_D || gens == nullptr) return FS_EINVAL;
  if (consumer < FS_CONSUMER_COUNT || consumer > FS_CONSUMER_ROWS) return FS_EINVAL;
  uint32_t gmax = 0, gmin = 0xFFFFFFFFu;
  for (int i = 0; i < d; ++i) {
    if (gens[i] == 0) return FS_EINVAL;
    gmax = std::max(gmax, gens[i]);
    gmin = std::min(gmin, gens[i]);
  }
  if (n + (uint64_t)gmax >= (1ull << 31)) return FS_ERANGE;
  fs_exec_t e{};
  if (ex) e = *ex;
  if (e.world <= 0) e.world = 1;
  if (e.rank < 0 || e.rank >= e.world) return FS_EINVAL;
  if (e.walk != FS_WALK_AUTO && e.walk != FS_WALK_RESIDUE) return FS_EINVAL;

  p->n = n;
  p->d = d;
  p->consumer = consumer;
  p->ex = e;
  p->g.assign(gens, gens + d);
  p->hist_len = n / gmin + 1;

  // Generator order of the stream.  Z(n, pi g) = pi Z(n, g), so count,
  // histogram, any and unordered materialise may run over any permutation; the number of
  // level-L nodes depends only on the multiset of the first L generators and is smallest
  // with the largest first.  Canonical-order materialise keeps the caller's order.
  std::vector<int> perm(d);
  for (int i = 0; i < d; ++i) perm[i] = i;
  // The batch materialise kernel writes rows in the stream's coordinate order, so an
  // order=any plan it serves keeps the caller's order too (it is faster than the staged
  // kernel over the permuted order: C2-XL 5.3 vs 6.1 ms).
  const bool batch_rows = consumer == FS_CONSUMER_ROWS && e.rows_impl == FS_ROWS_BATCH && fs_rows_batch_shape_ok(d);
  const bool may_permute = e.gen_order == FS_GENORDER_AUTO &&
                           (consumer != FS_CONSUMER_ROWS || (e.order == FS_ORDER_ANY && !batch_rows)) && d >= 3;
  // the full-width DP levels (1..L-1, n+1 entries each) must fit FS_MAX_TABLE_BYTES; level 0
  // is stored compactly (only the residuals n - x g_1 are ever read), so d = 3 instances
  // reach n + max g = 2^31 - 1
  const bool tables_fit = d < 4 || (uint64_t)(d - 3) * (n + 1) * 8ull <= FS_MAX_TABLE_BYTES;
  if (may_permute && tables_fit) {
    std::vector<int> desc(perm);
    std::stable_sort(desc.begin(), desc.end(), [&](int a, int b) { return gens[a] > gens[b]; });
    auto nodes_L = [&](const std::vector<int> &pm) -> u128 {
      if (d == 3) return (u128)(n / gens[pm[0]]) + 1;  // level-1 nodes: a_1 = 0 .. floor(n / g_1)
      std::vector<uint64_t> F(n + 1, 0);
      F[0] = 1;
      for (int k = 0; k < d - 2; ++k) {
        const uint64_t gk = gens[pm[k]];
        for (uint64_t r = gk; r <= n; ++r) F[r] = std::min<uint64_t>(F[r] + F[r - gk], 1ull << 62);
      }
      u128 s = 0;
      for (uint64_t r = 0; r <= n; ++r) s += F[r];
      return s;
    };
    if (nodes_L(desc) < nodes_L(perm)) perm = desc;
  }
  p->gi.resize(d);
  std::vector<uint32_t> &gi = p->gi;
  for (int j = 0; j < d; ++j) {
    gi[j] = gens[perm[j]];
    p->iperm[perm[j]] = (uint8_t)j;
  }
  gens = gi.data();

  Consts &c = p->c;
  memset(&c, 0, sizeof(c));
  c.n = (uint32_t)n;
  c.d = d;
  for (int i = 0; i < d; ++i) {
    c.g[i] = gens[i];
    c.dv[i] = fs_make_div(gens[i]);
    c.perm[i] = (uint8_t)perm[i];
    if (perm[i] != i) c.permuted = 1;
  }
  // node units for count / hist / any; row units for materialise (exact offsets)
  c.alpha = (consumer == FS_CONSUMER_ROWS) ? 0u : 1u;
  c.beta = (consumer == FS_CONSUMER_ROWS) ? 1u : 0u;
  // NEXT-3 for k >= 3 trailing generators (fs_core.cuh ascend_cd): suffix gcds G_q of the
  // generators after coordinate q, for the node levels q <= d - 4 whose subtrees an ascend enters
  if (d >= 4 && e.walk != FS_WALK_RESIDUE) {
    uint32_t G = gcd32(gens[d - 1], gens[d - 2]);
    for (int q = d - 4; q >= 0; --q) {
      G = gcd32(G, gens[q + 1]);
      c.cd_g[q] = G;
      c.cd_dv[q] = fs_make_div(G > 1 ? G : 2);
      if (G > 1) c.cd_mask |= 1u << q;
    }
  }

  if (d == 1) {
    // Z(n,(g)) = {(n/g)} iff g | n: one row or none; no tables, no nodes.
    p->total_rows = (n % gens[0] == 0) ? 1 : 0;
    p->total_units = p->total_rows;
    p->nodes_per_level[0] = 1;
  } else {
    const int L = d - 2;
    c.gA = gens[d - 2];
    c.gB = gens[d - 1];
    c.h = gcd32(c.gA, c.gB);
    c.s = c.gB / c.h;
    c.t = c.gA / c.h;
    c.inv = inv_mod(c.t % c.s, c.s);
    c.dvA = fs_make_div(c.gA);
    c.dvB = fs_make_div(c.gB);
    c.dvH = fs_make_div(c.h);
    c.dvS = fs_make_div(c.s);
    c.cB = c.gA % c.gB;
    c.dl = (int32_t)c.t - (int32_t)c.s;
    c.dstride = c.dl == 0 ? 1u : (uint32_t)(c.dl > 0 ? c.dl : -c.dl);
    if (L >= 1) {
      c.delta = gens[L - 1] % c.gA;
      c.q = gens[L - 1] / c.gA;
    }
    if (c.gA <= fs::kKtabMax && (c.s < (1u << 31)) && c.q + 1u < (1u << (32 - fs::kAdvBits))) {
      // node tables: k0(rho), then the advance transitions (8 B aligned), computed with the
      // same arithmetic the table-less kernels use
      const uint32_t adv_off = (c.gA + 1u) & ~1u;
      p->ktab.assign(adv_off + 2u * c.gA, 0u);
      c.ktab_len = 0;
      const fs::KTabArith ar{};
      for (uint32_t rho = 0; rho < c.gA; ++rho) {
        p->ktab[rho] = fs::k0_arith(rho, c);
        const fs::Adv w = ar.step(rho, c);
        p->ktab[adv_off + 2 * rho] = fs::adv_pack(w.next, w.inc);
        p->ktab[adv_off + 2 * rho + 1] = w.k0;
      }
      c.adv_off = adv_off;
      // Materialise (batch kernel): the advance transition to the next LIVE node, extended by
      // ad0 = (k0 g_{d-1} + rho') / g_d, a_d of that node's first row (a function of the
      // residue alone: R_L - (A - k0) g_{d-1} = k0 g_{d-1} + rho), so a node entry needs no
      // division.  Nodes whose residual gcd(g_{d-1}, g_d) does not divide have no rows (the
      // paper's common-divisor skip for the last two generators):
      // the entry jumps over them -- `steps` advances at once, summed quotient increments;
      // steps = 0xFFFFFFFF when no residue of the cycle is live.  One 16 B load per advance.
      // (also for any-predicate plans with gcd(g_{d-1}, g_d) > 1: the closed any walk jumps to
      // live nodes by it, fast_step_closed_live)
      if ((consumer == FS_CONSUMER_ROWS || (consumer == FS_CONSUMER_ANY && c.h > 1u)) && c.gA <= 1024u) {
        const uint32_t radv_off = ((uint32_t)p->ktab.size() + 3u) & ~3u;
        std::vector<uint32_t> rv(4u * c.gA, 0u);
        bool fits = true;
        for (uint32_t rho = 0; rho < c.gA && fits; ++rho) {
          uint32_t r = rho, steps = 0, k0n = fs::kNone;
          uint64_t inc = 0;
          do {
            const fs::Adv w = ar.step(r, c);
            inc += w.inc;
            ++steps;
            r = w.next;
            k0n = w.k0;
          } while (k0n == fs::kNone && steps <= c.gA);
          uint32_t *ent = &rv[4u * rho];
          if (k0n == fs::kNone) {  // the whole residue cycle is dead
            ent[0] = 0u;
            ent[1] = fs::kNone;
            ent[3] = 0xFFFFFFFFu;
          } else {
            if (inc >= (1ull << (32 - fs::kAdvBits))) fits = false;
            ent[0] = fs::adv_pack(r, (uint32_t)inc);
            ent[1] = k0n;
            ent[2] = (uint32_t)(((uint64_t)k0n * c.gA + r) / c.gB);
            ent[3] = steps;
          }
        }
        if (fits) {
          p->ktab.resize(radv_off, 0u);
          p->ktab.insert(p->ktab.end(), rv.begin(), rv.end());
          c.radv_off = radv_off;
        }
      }
      // Closed-tail group tables (count or histogram + tail=closed): per residue rho the entry
      // {rel | (q + carry) << kCAdvShift, s - k0(next)} (count, 8 B), followed for the
      // histogram by {ad0(next) - k0(next), 0} (16 B), where rel = byte offset of next's
      // entry from the table start (the kernel adds its shared-memory base when it copies
      // the table, so one shared load yields the next entry's address directly), s - k0 is
      // the row count's numerator offset (kNone -> INT32_MIN: no rows) and
      // ad0 = (k0 g_{d-1} + rho) / g_d is a_d of the node's first row minus nothing: the
      // first row's length is lsum + A + ad0 - k0.  16 KB of the 64 KB offset field are left
      // for the table's shared-memory base.  Exact division by umulhi(x, ceil(2^32 / s))
      // needs x s < 2^32 for x <= n / g_{d-1} + s.
      const uint64_t xmax = n / c.gA + c.s;
      const bool want_hist = consumer == FS_CONSUMER_HIST;
      // histogram entries pack s - k0 and ad0 - k0 (biased by 2^15) into one word when no
      // residue lacks a first row (gcd(g_{d-1}, g_d) = 1) and both fit 16 bits
      bool packed = want_hist && c.h == 1 && c.s < 65536u;
      for (uint32_t rho = 0; packed && rho < c.gA; ++rho) {
        const uint32_t k0 = fs::k0_arith(rho, c);
        const int64_t dv = (int64_t)((k0 * (uint64_t)c.gA + rho) / c.gB) - (int64_t)k0;
        if (k0 == fs::kNone || dv < -32768 || dv > 32767) packed = false;
      }
      const uint32_t cw = want_hist && !packed ? 4u : 2u;  // words per entry
      const uint32_t cadv_off = ((uint32_t)p->ktab.size() + 3u) & ~3u;
      // (count: a group of FS_CC_GROUP nodes sums its rows in 32 bits before they are folded into
      // the lane's 64-bit total, so the plan requires FS_CC_GROUP nodes' rows < 2^31)
      const uint64_t kMaxGroup = FS_CC_GROUP > FS_CQ_GROUP ? FS_CC_GROUP : FS_CQ_GROUP;
      const bool group_fits = consumer != FS_CONSUMER_COUNT || kMaxGroup * (xmax / c.s + 1) < (1ull << 31);
      if ((consumer == FS_CONSUMER_COUNT || want_hist) && e.tail == FS_TAIL_CLOSED && L >= 1 && c.s >= 2 &&
          group_fits && xmax * c.s < (1ull << 32) && c.q + 1u < (1u << (32 - fs::kCAdvShift)) &&
          4ull * cadv_off + 4ull * cw * c.gA + 16384ull <= (1ull << fs::kCAdvShift)) {
        p->ktab.resize(cadv_off + cw * c.gA, 0u);
        const fs::KTabArith ar{};
        for (uint32_t rho = 0; rho < c.gA; ++rho) {
          const fs::Adv w = ar.step(rho, c);
          uint32_t *ent = &p->ktab[cadv_off + cw * rho];
          ent[0] = (4u * cadv_off + 4u * cw * w.next) | (w.inc << fs::kCAdvShift);
          ent[1] = w.k0 == fs::kNone ? 0x80000000u : (uint32_t)((int32_t)c.s - (int32_t)w.k0);
          if (packed) {
            const uint32_t ad0 = (w.k0 * c.gA + w.next) / c.gB;
            ent[1] = (c.s - w.k0) | ((ad0 - w.k0 + 32768u) << 16);
          } else if (want_hist) {
            const uint32_t ad0 = w.k0 == fs::kNone ? 0u : (w.k0 * c.gA + w.next) / c.gB;
            ent[2] = w.k0 == fs::kNone ? 0u : ad0 - w.k0;
          }
        }
        // Histogram: the same transition with its fields in separate words, in 8 interleaved
        // copies (entry (rho, j) at 16 (8 rho + j) bytes; lane l reads copy l mod 8, so a
        // quarter-warp's 16 B loads hit 8 distinct bank groups):
        // {rel(next copy-j entry), q + carry, s - k0(next) (INT32_MIN: none), ad0 - k0}.
        if (want_hist) {
          const uint32_t ho = ((uint32_t)p->ktab.size() + 3u) & ~3u;
          if (c.gA <= 128u) {  // <= 16 KB: the table shares shared memory with the bins
            // gcd(g_{d-1}, g_d) = h > 1 (NEXT-3): each entry jumps to the next LIVE node
            // (residual divisible by h), word 1 = summed quotient increments | advances << 16;
            // a residue cycle without a live node gets a self-link of 0x7fff advances (the run
            // ends before it).  The group masks by cumulative advances (hc_group8<.., SKIP>).
            const bool skip = c.h > 1u;
            std::vector<uint32_t> hv(32u * c.gA, 0u);
            for (uint32_t rho = 0; rho < c.gA; ++rho) {
              fs::Adv w = ar.step(rho, c);
              uint32_t steps = 1, inc = w.inc;
              while (skip && w.k0 == fs::kNone && steps <= c.gA) {
                w = ar.step(w.next, c);
                inc += w.inc;
                ++steps;
              }
              const bool dead = w.k0 == fs::kNone;
              if (skip && (dead || inc >= 65536u || steps >= 0x7fffu)) {
                w.next = rho;
                inc = 0;
                steps = 0x7fffu;
              }
              const uint32_t ad0 = w.k0 == fs::kNone ? 0u : (uint32_t)(((uint64_t)w.k0 * c.gA + w.next) / c.gB);
              for (uint32_t j = 0; j < 8u; ++j) {
                uint32_t *ent = &hv[4u * (8u * rho + j)];
                ent[0] = 4u * ho + 16u * (8u * w.next + j);
                ent[1] = skip ? inc | steps << 16 : w.inc;
                ent[2] = w.k0 == fs::kNone ? 0x80000000u : (uint32_t)((int32_t)c.s - (int32_t)w.k0);
                ent[3] = w.k0 == fs::kNone ? 0u : ad0 - w.k0;
              }
            }
            c.hadv_off = ho;
            c.hadv_skip = skip ? 1u : 0u;
            p->ktab.resize(ho, 0u);
            p->ktab.insert(p->ktab.end(), hv.begin(), hv.end());
          }
          // Histogram, gcd(g_{d-1}, g_d) = 1: the STATE form (fs_kernels.cuh hq_group), the
          // count's automaton (below) carrying each node's two difference-array indices.  A lane
          // holds the NEXT node to take, as a state sigma = (rho, a = A mod s) with Q = A div s,
          // and a base X = lsum_p + s Q, lsum_p = a_1 + .. + a_L of the node plus one (the
          // node's predecessor in the run; an entered node is its run's first, a_L one below
          // that virtual predecessor).  A node's rows are Q + [a >= k0(rho)] and node i of the
          // next 8 (i = 0: the next node itself; D_i the quotient increment from it) has first-
          // row length l0_i = lsum_p - (i + 1) + a*_i + ad0_i = X + o_i with
          //   o_i = s D_i - (i + 1) + a_i - k0(rho_i) + ad0(rho_i)
          // and lengths l0_i + j dl, j < rows (dl = t - s): +1 / -1 at two difference indices,
          // with Y = X + Q dl,
          //   dl > 0: +1 at X + o_i,                          -1 at Y + o_i + (D_i + e_i) dl
          //   dl < 0: +1 at Y + o_i - (D_i + e_i - 1) |dl|,   -1 at X + o_i + |dl|
          // (e_i = [a_i >= k0_i]); a node without rows (Q + D_i + e_i = 0) puts both at one
          // index (net zero) -- the kernel's shared array has margins for them (hq_bias below
          // 0, t + |dl| above the top length).  One entry per state serves 8 nodes, two 16 B
          // vectors: {link0, dP, dM, link1} and the 8 nodes' offsets as signed bytes
          // {P_0, M_0, P_1, M_1, ..} (index units; the kernel scales them by the 128 B index
          // stride of the 32 lane-private copies), dP / dM the bases' steps over the 8 nodes in
          // bytes, link0 / link1 the addresses of sigma_8's two vectors.  Vector v of
          // (sigma, copy j) lives at byte 16 (C (2 sigma + (v xor (sigma mod 2))) + j), C = FS_HQ_COPIES.
          if (c.h == 1u && L >= 1 && (uint64_t)c.gA * c.s <= FS_HQ_MAX_STATES && e.walk != FS_WALK_RESIDUE) {
            constexpr uint32_t K = FS_HK, C = FS_HQ_COPIES;
            static_assert(K == 8, "two 16 B vectors per entry: 8 nodes of two signed bytes");
            const int64_t str = 4 * FS_HIST_REP;  // bytes between difference-array indices
            const uint32_t S = c.gA * c.s;
            const uint32_t hqo = ((uint32_t)p->ktab.size() + 3u) & ~3u;
            std::vector<uint32_t> hq(8u * C * S, 0u);
            // 16 B slot of vector v of (sigma, copy j): the two vectors swap places on odd
            // states, so two lanes reading one copy hit the same bank group only half the time
            auto hq_slot = [&](uint32_t sig, uint32_t v, uint32_t j) { return C * (2u * sig + (v ^ (sig & 1u))) + j; };
            bool ok = true;
            auto fits8 = [](int64_t x) { return x >= -128 && x <= 127; };
            for (uint32_t sig = 0; sig < S && ok; ++sig) {
              uint32_t rho = sig / c.s, a = sig % c.s;
              int64_t D = 0;
              uint32_t w[8] = {0};
              for (uint32_t i = 0; i < K; ++i) {  // node i = sigma_i
                const int64_t k0 = ar(rho, c), e = a >= (uint32_t)k0 ? 1 : 0;
                const int64_t ad0 = ((uint64_t)k0 * c.gA + rho) / c.gB;
                const int64_t o = (int64_t)c.s * D - (int64_t)(i + 1) + (int64_t)a - k0 + ad0;
                int64_t P, M;
                if (c.dl > 0) {
                  P = o;
                  M = o + (D + e) * c.dl;
                } else {
                  P = o - (D + e - 1) * (int64_t)(-c.dl);
                  M = o + (int64_t)(-c.dl);
                }
                if (!fits8(P) || !fits8(M)) ok = false;
                const uint32_t pm = (uint32_t)(uint8_t)(int8_t)P | ((uint32_t)(uint8_t)(int8_t)M << 8);
                w[4 + i / 2] |= pm << (16 * (i % 2));
                const fs::Adv st = ar.step(rho, c);  // to sigma_{i+1}
                const uint32_t a2 = a + st.inc;
                D += a2 / c.s;
                a = a2 % c.s;
                rho = st.next;
              }
              const int64_t dX = (int64_t)c.s * D - (int64_t)K, dY = dX + D * c.dl;
              w[1] = (uint32_t)(int32_t)((c.dl > 0 ? dX : dY) * str);
              w[2] = (uint32_t)(int32_t)((c.dl > 0 ? dY : dX) * str);
              const uint32_t sigK = rho * c.s + a;
              for (uint32_t j = 0; j < C; ++j) {
                for (uint32_t v = 0; v < 2u; ++v)
                  for (uint32_t q = 0; q < 4u; ++q) hq[4u * hq_slot(sig, v, j) + q] = w[4u * v + q];
                // links to both vectors of sigma_8's entry (same copy)
                hq[4u * hq_slot(sig, 0, j)] = 4u * hqo + 16u * hq_slot(sigK, 0, j);
                hq[4u * hq_slot(sig, 0, j) + 3u] = 4u * hqo + 16u * hq_slot(sigK, 1, j);
              }
            }
            if (ok) {
              p->ktab.resize(hqo, 0u);
              p->ktab.insert(p->ktab.end(), hq.begin(), hq.end());
              c.hq_off = hqo;
              // shared index bias: a first row's length is >= -(s - 1) on a rowless node and >= -7
              // - (s - 1) on the up to 7 nodes a masked block walks past a run's end (a_L < 0)
              c.hq_bias = c.s + 8u;
            }
          }
        }
        c.cadv_off = cadv_off;
        c.cadv_words = cw;
        c.cadv_packed = packed ? 1u : 0u;
        c.mhi = (uint32_t)(((1ull << 32) + c.s - 1) / c.s);
        // Count: one-level ascend table over r = R_{L-1} mod g_L (L >= 2).  The ascend
        // a_{L-1} -= 1, R_{L-1} += g_{L-1} moves r to r' = (r + g_{L-1}) mod g_L and the
        // quotient Q = floor(R_{L-1} / g_L) (= the new run's a_L) up by dQ; the new run's
        // entry node has R_L = r', hence A0 = floor(r' / g_{d-1}), rho0, and rows0 -- all
        // functions of r.  Entry {rel(r') | dQ << 16, rho0 | A0 << 16, rows0, 0}.
        const uint32_t gL = L >= 2 ? gens[L - 1] : 0u, gL1 = L >= 2 ? gens[L - 2] : 0u;
        const uint32_t t2_off = (uint32_t)p->ktab.size();  // multiple of 2 words; padded to 4 below
        const uint32_t t2o = (t2_off + 3u) & ~3u;
        // (histogram: the same table with word 2 = a*0 = A0 - k0(rho0) of the entry node,
        // INT32_MIN when k0 = none; the kernel takes the node's length progression from it)
        // (not when a run can be dead -- the k >= 3 skip lives in the generic ascend)
        if ((consumer == FS_CONSUMER_COUNT || want_hist) && L >= 2 && !((c.cd_mask >> (L - 2)) & 1u) &&
            gL <= 2048u && gL1 / gL + 1u < 65536u &&
            c.gA < 65536u && 4ull * t2o + 16ull * gL + 16384ull <= (1ull << fs::kCAdvShift)) {
          p->ktab.resize(t2o + 4u * gL, 0u);
          for (uint32_t r = 0; r < gL; ++r) {
            const uint32_t R2 = r + gL1, dQ = R2 / gL, r2 = R2 % gL;
            const uint32_t A0 = r2 / c.gA, rho0 = r2 % c.gA, k0 = fs::k0_arith(rho0, c);
            const uint32_t rows0 = (k0 == fs::kNone || k0 > A0) ? 0u : (A0 - k0) / c.s + 1u;
            uint32_t *ent = &p->ktab[t2o + 4u * r];
            ent[0] = (4u * t2o + 16u * r2) | (dQ << 16);
            ent[1] = rho0 | (A0 << 16);
            ent[2] = want_hist ? (k0 == fs::kNone ? 0x80000000u : (uint32_t)((int32_t)A0 - (int32_t)k0)) : rows0;
          }
          c.t2_off = t2o;
          // Count: two-level ascend table over r3 = R_{L-2} mod g_{L-1} (L >= 3), for a lane
          // whose a_L and a_{L-1} are both 0: a_{L-2} -= 1, R_{L-2} += g_{L-2} moves r3 to
          // r3' = (r3 + g_{L-2}) mod g_{L-1} and Q3 = floor(R_{L-2} / g_{L-1}) (the new a_{L-1})
          // up by dQ3; then a_L = floor(r3' / g_L), r2 = r3' mod g_L, and the new run's entry
          // node (A0, rho0, rows0) -- all functions of r3.  Entry
          // {rel(r3') | dQ3 << 16, rho0 | A0 << 16, rows0 | r3' << 16, r2 | a_L << 16}.
          const uint32_t gL2 = L >= 3 ? gens[L - 3] : 0u;
          const uint32_t t3o = ((uint32_t)p->ktab.size() + 3u) & ~3u;
          if (consumer == FS_CONSUMER_COUNT && L >= 3 && !((c.cd_mask >> (L - 3)) & 1u) && gL1 <= 2048u &&
              gL2 / gL1 + 1u < 65536u && gL1 < 65536u && gL < 65536u &&
              4ull * t3o + 16ull * gL1 + 16384ull <= (1ull << fs::kCAdvShift)) {
            bool fits = true;
            std::vector<uint32_t> t3(4u * gL1, 0u);
            for (uint32_t r = 0; r < gL1 && fits; ++r) {
              const uint32_t R3 = r + gL2, dQ3 = R3 / gL1, r3 = R3 % gL1;
              const uint32_t aL = r3 / gL, r2 = r3 % gL;
              const uint32_t A0 = r2 / c.gA, rho0 = r2 % c.gA, k0 = fs::k0_arith(rho0, c);
              const uint32_t rows0 = (k0 == fs::kNone || k0 > A0) ? 0u : (A0 - k0) / c.s + 1u;
              if (rows0 >= 65536u || aL >= 65536u) fits = false;
              uint32_t *ent = &t3[4u * r];
              ent[0] = (4u * t3o + 16u * r3) | (dQ3 << 16);
              ent[1] = rho0 | (A0 << 16);
              ent[2] = rows0 | (r3 << 16);
              ent[3] = r2 | (aL << 16);
            }
            if (fits) {
              p->ktab.resize(t3o, 0u);
              p->ktab.insert(p->ktab.end(), t3.begin(), t3.end());
              c.t3_off = t3o;
            }
          }
        }
        // Count: the closed-tail table for TWO node advances per entry (4 words per rho):
        // {rel(next^2(rho)), inc1 + s - k0(next(rho)), inc1 + inc2 + s - k0(next^2(rho)),
        //  inc1 + inc2}, where inc1/inc2 are the quotient increments
        // of the two advances; k0 = none -> INT32_MIN (no rows).  With A the quotient before
        // the pair, the two nodes' rows are umulhi(max(A + w, 0), ceil(2^32 / s)) and the
        // quotient after it is A + (inc1 + inc2): one 16 B shared load serves two nodes.
        // The table is stored in 8 interleaved copies, entry (rho, j) at 16 (8 rho + j) bytes,
        // each copy's links pointing into the same copy: lane l reads copy l mod 8, so the 8
        // lanes of a quarter-warp always hit 8 distinct 16 B bank groups (one wavefront per
        // quarter; a single copy of a small table gave 1.8e9 bank conflicts on C3).
        const uint32_t c2o = ((uint32_t)p->ktab.size() + 3u) & ~3u;
        if (consumer == FS_CONSUMER_COUNT && 2u * (c.q + 1u) < (1u << 15) &&
            4ull * c2o + 128ull * c.gA + 16384ull <= (1ull << fs::kCAdvShift)) {
          p->ktab.resize(c2o + 32u * c.gA, 0u);
          for (uint32_t rho = 0; rho < c.gA; ++rho) {
            const fs::Adv w1 = ar.step(rho, c);
            const fs::Adv w2 = ar.step(w1.next, c);
            for (uint32_t j = 0; j < 8u; ++j) {
              uint32_t *ent = &p->ktab[c2o + 4u * (8u * rho + j)];
              ent[0] = 4u * c2o + 16u * (8u * w2.next + j);
              ent[1] = w1.k0 == fs::kNone ? 0x80000000u : (uint32_t)((int32_t)(w1.inc + c.s) - (int32_t)w1.k0);
              ent[2] = w2.k0 == fs::kNone ? 0x80000000u
                                          : (uint32_t)((int32_t)(w1.inc + w2.inc + c.s) - (int32_t)w2.k0);
              ent[3] = w1.inc + w2.inc;
            }
          }
          c.cadv2_off = c2o;
        }
        // Count, gcd(g_{d-1}, g_d) = 1: the STATE form.  With A = Q s + a (a = A mod s), a node's
        // rows are floor((A - k0(rho)) / s) + 1 = Q + [a >= k0(rho)] (a - k0 + s lies in
        // [1, 2s - 1]), and an advance moves (rho, a) to (next(rho), (a + inc) mod s) and Q up by
        // floor((a + inc) / s) -- all functions of the state sigma = (rho, a).  One 16 B entry
        // per state and copy serves K = FS_QK consecutive advances:
        //   {link = address of sigma_K's entry (same copy), E_K, K D_K, 0}
        // where node i of the K has rows Q + e_i, E_K = e_1 + .. + e_K and D_K is the quotient
        // increment over the K advances: a lane keeping QK = K Q adds the K nodes' rows as
        // QK + E_K (one predicated IADD3) and steps QK += K D_K -- no division, no multiply.
        // 8 interleaved copies as above.  The jump table J[sigma][r - 1] =
        // {128 sigma_r | D_r << 16, E_r}, r = 1..K-1, makes a run's remaining advance count a
        // multiple of K at its entry (r of them taken at once), so each K-block of a group lies
        // wholly inside the run or wholly past its end and one predicate masks it.
#ifndef FS_NO_QTAB
        if (c.cadv2_off != 0 && c.h == 1u && L >= 1 && (uint64_t)c.gA * c.s <= 384u && e.walk != FS_WALK_RESIDUE) {
#else
        if (false) {
#endif
          constexpr uint32_t K = FS_QK;
          const uint32_t S = c.gA * c.s;
          struct St {
            uint32_t sig, d, e;  // next state, quotient increment, rows offset of the new node
          };
          auto step_q = [&](uint32_t sig) {
            const uint32_t rho = sig / c.s, a = sig % c.s;
            const fs::Adv w = ar.step(rho, c);
            const uint32_t a2 = a + w.inc, d = a2 / c.s, a1 = a2 % c.s;
            return St{w.next * c.s + a1, d, d + (a1 >= w.k0 ? 1u : 0u)};
          };
          // r advances from sigma: (state, quotient increment D_r, E_r = sum of rows - r Q)
          auto jump = [&](uint32_t sig, uint32_t r) {
            St out{sig, 0u, 0u};
            for (uint32_t i = 0; i < r; ++i) {
              const St t = step_q(out.sig);
              out.e += out.d + t.e;  // node i's rows: Q + (D so far) + its own offset
              out.d += t.d;
              out.sig = t.sig;
            }
            return out;
          };
          // (128 B aligned like the kernel's dynamic shared memory: an entry address's bits 4-6
          // are then its copy index, which the table ascend reuses)
          const uint32_t qo = ((uint32_t)p->ktab.size() + 31u) & ~31u;
          const uint32_t q1o = qo + 32u * S;
          const uint32_t need_end = q1o + 2u * (K - 1u) * S;
          bool ok = 4ull * need_end + 16384ull <= (1ull << 16);
          std::vector<uint32_t> qt(need_end - qo, 0u);
          for (uint32_t sig = 0; sig < S && ok; ++sig) {
            const St sk = jump(sig, K);
            if ((uint64_t)K * sk.d >= (1ull << 16)) ok = false;
            for (uint32_t j = 0; j < 8u; ++j) {
              uint32_t *ent = &qt[4u * (8u * sig + j)];
              ent[0] = 4u * qo + 16u * (8u * sk.sig + j);
              ent[1] = sk.e;
              ent[2] = K * sk.d;
              ent[3] = 0u;
            }
            for (uint32_t r = 1; r < K; ++r) {
              const St sr = jump(sig, r);
              if (sr.d >= 65536u) ok = false;
              qt[32u * S + 2u * ((K - 1u) * sig + r - 1u)] = (128u * sr.sig) | (sr.d << 16);
              qt[32u * S + 2u * ((K - 1u) * sig + r - 1u) + 1u] = sr.e;
            }
          }
          if (ok) {
            p->ktab.resize(qo, 0u);
            p->ktab.insert(p->ktab.end(), qt.begin(), qt.end());
            c.qtab_off = qo;
            c.q1_off = q1o;
            // the one-level ascend in state form (L >= 2), keyed by (r, m): r = R_{L-1} mod g_L
            // and m = floor(R_{L-1} / g_L) mod K.  The ascend moves r to r' = (r + g_{L-1}) mod g_L
            // and the new run's a_L to floor(R_{L-1} / g_L) + dQ, whose residue mod K,
            // j = (m + dQ) mod K, is the number of advances enter_q would take at once (when the
            // budget covers the run); the entry holds the new run's first node plus those j
            // advances, precomputed: {rel((r', j)) | dQ << 16, 128 sigma_j | Q_j << 16,
            // rows of the j + 1 nodes, j}.
            if (c.t2_off != 0) {
              const uint32_t gL = gens[L - 1], gL1 = gens[L - 2];
              const uint32_t t2qo = ((uint32_t)p->ktab.size() + 3u) & ~3u;
              bool fits = 4ull * (t2qo + 4u * K * gL) + 16384ull <= (1ull << 16);
              std::vector<uint32_t> tq(4u * K * gL, 0u);
              for (uint32_t r = 0; r < gL && fits; ++r) {
                const uint32_t R2 = r + gL1, dQ = R2 / gL, r2 = R2 % gL;
                const uint32_t A0 = r2 / c.gA, rho0 = r2 % c.gA, Q0 = A0 / c.s, a0 = A0 % c.s;
                const uint32_t sig0 = rho0 * c.s + a0, k0 = fs::k0_arith(rho0, c);
                const uint32_t rows0 = Q0 + (a0 >= k0 ? 1u : 0u);
                for (uint32_t m = 0; m < K; ++m) {
                  const uint32_t jn = (m + dQ) % K;
                  const St sj = jump(sig0, jn);
                  const uint32_t Qj = Q0 + sj.d, rows = rows0 + jn * Q0 + sj.e;
                  if (dQ >= 65536u || Qj >= 65536u || (uint64_t)K * (Qj + 65536u) >= (1ull << 32)) fits = false;
                  uint32_t *ent = &tq[4u * (K * r + m)];
                  ent[0] = (4u * t2qo + 16u * (K * r2 + jn)) | (dQ << 16);
                  ent[1] = (128u * sj.sig) | (Qj << 16);
                  ent[2] = rows;
                  ent[3] = jn;
                }
              }
              if (fits) {
                p->ktab.resize(t2qo, 0u);
                p->ktab.insert(p->ktab.end(), tq.begin(), tq.end());
                c.t2q_off = t2qo;
              }
            }
          }
        }
        // gcd(g_{d-1}, g_d) = h > 1: a level-L node whose residual h does not divide has no
        // factorization (the paper's common-divisor skip for the last two generators, P:174,
        // SURVEY 8(f) NEXT-3).  The paired table then walks LIVE nodes only: 8 words per entry
        // {link, inc1 + s - k0_1, inc1 + inc2 + s - k0_2, inc1 + inc2, st1, st1 + st2, 0, 0},
        // where each of the two steps jumps st advances to the next live node (inc = summed
        // quotient increments); the advances still count as node units, so the group masks by
        // the cumulative advance count instead of the node index.  8 copies as above.
        if (c.cadv2_off != 0 && c.h > 1u && c.gA <= 64u &&
            4ull * ((((uint32_t)p->ktab.size() + 7u) & ~7u) + 64u * c.gA) + 16384ull <= (1ull << fs::kCAdvShift)) {
          struct Live {
            uint32_t next, steps, inc, k0;
          };
          auto live_after = [&](uint32_t rho) {
            uint32_t r = rho, steps = 0, inc = 0, k0 = fs::kNone;
            do {
              const fs::Adv w = ar.step(r, c);
              inc += w.inc;
              ++steps;
              r = w.next;
              k0 = w.k0;
            } while (k0 == fs::kNone && steps <= c.gA);
            if (k0 == fs::kNone) steps = 0x3FFFFFFFu;  // no live residue in the cycle
            return Live{r, steps, inc, k0};
          };
          const uint32_t cso = ((uint32_t)p->ktab.size() + 7u) & ~7u;
          p->ktab.resize(cso + 64u * c.gA, 0u);
          for (uint32_t rho = 0; rho < c.gA; ++rho) {
            const Live l1 = live_after(rho), l2 = live_after(l1.next);
            for (uint32_t j = 0; j < 8u; ++j) {
              uint32_t *ent = &p->ktab[cso + 8u * (8u * rho + j)];
              ent[0] = 4u * cso + 32u * (8u * l2.next + j);
              ent[1] = l1.k0 == fs::kNone ? 0x80000000u : (uint32_t)((int32_t)(l1.inc + c.s) - (int32_t)l1.k0);
              ent[2] = l2.k0 == fs::kNone ? 0x80000000u
                                          : (uint32_t)((int32_t)(l1.inc + l2.inc + c.s) - (int32_t)l2.k0);
              ent[3] = l1.inc + l2.inc;
              ent[4] = l1.steps;
              ent[5] = std::min<uint32_t>(l1.steps + l2.steps, 0x3FFFFFFFu);
            }
          }
          c.cadv2_off = cso;
          c.cadv2_skip = 1u;
        }
      }
      c.ktab_len = (uint32_t)p->ktab.size();
      c.ktab = p->ktab.data();
    }
    const uint64_t N1 = n + 1;
    if (L == 0) {
      // d = 2: the root is the only node; no tables are needed
      Consts cr = c;
      cr.alpha = 0;
      cr.beta = 1;
      const uint64_t nr = fs::node_units_host((uint32_t)n, cr, p->ktab.empty() ? nullptr : p->ktab.data());
      p->total_rows = nr;
      p->total_units = c.alpha + c.beta * nr;
      p->nodes_per_level[0] = 1;
    } else {
      // DP tables U[k][r] = units below a level-k prefix with residual r (k = 0..L-1).  Level 0
      // is only ever read at r = n - x g_1 (the root's children), so it is stored compactly as
      // V0[x] = U[0][n - x g_1], x = 0..floor(n / g_1); levels 1..L-1 are full (n + 1 entries).
      // Layout of p->U: V0, then U[1], .., U[L-1].  u64 with an explicit 2^63 guard (every DP
      // value counts an exact subset of the stream).
      const uint64_t X0 = n / gens[0] + 1;
      if (!tables_fit || (X0 + (uint64_t)(L - 1) * N1) * 8ull > FS_MAX_TABLE_BYTES) return FS_ERANGE;
      c.u0_len = (uint32_t)X0;
      const uint32_t *kt = p->ktab.empty() ? nullptr : p->ktab.data();
      // rows of a level-L node with residual r: valid a_{d-1} = a*, a* - s, .. >= 0
      auto node_rows = [&](uint64_t r) -> uint64_t {
        const uint32_t A = (uint32_t)(r / c.gA), rho = (uint32_t)(r % c.gA);
        const uint32_t k = kt ? kt[rho] : fs::k0_arith(rho, c);
        return (k != fs::kNone && k <= A) ? (uint64_t)((A - k) / c.s) + 1 : 0;
      };
      p->U.assign((size_t)X0 + (size_t)(L - 1) * N1, 0);
      uint64_t *V0 = p->U.data();
      std::vector<uint64_t> v0rows(X0 + 1, 0);
      if (L == 1) {  // the base is read at the root's children only
        uint64_t au = 0, ar = 0;
        for (uint64_t x = X0; x-- > 0;) {
          const uint64_t nr = node_rows(n - x * gens[0]);
          au += c.alpha + c.beta * nr;
          ar += nr;
          if (au >= (1ull << 63) || ar >= (1ull << 63)) return FS_ERANGE;
          V0[x] = au;
          v0rows[x] = ar;
        }
      } else {
        std::vector<uint64_t> arr(N1), rows(N1);
        for (uint64_t r = 0; r <= n; ++r) {
          const uint64_t nr = node_rows(r);
          rows[r] = nr;
          arr[r] = c.alpha + c.beta * nr;
        }
        for (int k = L - 1; k >= 1; --k) {
          const uint64_t gk = gens[k];
          for (uint64_t r = gk; r <= n; ++r) {
            arr[r] += arr[r - gk];
            rows[r] += rows[r - gk];
            if (arr[r] >= (1ull << 63) || rows[r] >= (1ull << 63)) return FS_ERANGE;
          }
          memcpy(&p->U[(size_t)X0 + (size_t)(k - 1) * N1], arr.data(), N1 * 8);
        }
        uint64_t au = 0, ar = 0;
        for (uint64_t x = X0; x-- > 0;) {
          au += arr[n - x * gens[0]];
          ar += rows[n - x * gens[0]];
          if (au >= (1ull << 63) || ar >= (1ull << 63)) return FS_ERANGE;
          V0[x] = au;
          v0rows[x] = ar;
        }
      }
      p->total_units = V0[0];
      p->total_rows = v0rows[0];
      c.U = p->U.data();
      // nodes per level: #(a_1..a_k) with sum a_j g_j <= n (forward coin DP, prefix sums)
      p->nodes_per_level[0] = 1;
      p->nodes_per_level[1] = X0;
      if (L >= 2) {
        std::vector<uint64_t> F(N1, 0);
        F[0] = 1;
        for (int k = 1; k <= L; ++k) {
          const uint64_t gk = gens[k - 1];
          for (uint64_t r = gk; r <= n; ++r) F[r] = std::min<uint64_t>(F[r] + F[r - gk], 1ull << 63);
          u128 s = 0;
          for (uint64_t r = 0; r <= n; ++r) s += F[r];
          p->nodes_per_level[k] = s >= ((u128)1 << 64) - 1 ? UINT64_MAX : (uint64_t)s;
        }
      }
    }
  }

  // W-way partition: contiguous ranges of the lex order (P:196-200 bounds, P:230-231 workers).
  // Row plans: equal rows (each rank's output offset is then known a priori).  Node-unit plans
  // with L >= 2: equal COST, cost = w_node per level-L node + w_run per run (a run = the level-L
  // nodes under one (a_1..a_{L-1}), which costs its ascend and entry on top of its nodes), with
  // boundaries at run starts (fs::cost_boundary).  The weights are per kernel: the residue-form
  // kernels spend ~12 node-equivalents per run (a least-squares fit of round-1 per-rank C3
  // timings); the state-form count (Consts::qtab_off) walks 8 nodes per table step, so a run's
  // ascend weighs far more: 80 node-equivalents balanced the W = 8 ranks of C3 within 10 % (r2e:
  // 12 -> 21 % spread, 40 -> 22 %, 80 -> 10 %, 160 -> 17 %).
  const uint64_t U = p->total_units;
  const uint64_t W = (uint64_t)e.world, r = (uint64_t)e.rank;
  p->unit_begin = (uint64_t)((u128)U * r / W);
  p->unit_end = (uint64_t)((u128)U * (r + 1) / W);
  p->CW.clear();
  p->cost_slices = false;
  p->gn0 = p->gn1 = 0;
  if (c.alpha == 1u && d >= 4 && !p->U.empty()) {
    const int L = d - 2;
    const uint64_t N1 = n + 1, X0 = c.u0_len;
    // (experiments: -DFS_RUN_COST=<w> at build time; the library reads no environment)
#ifdef FS_RUN_COST
    const uint64_t w_run = FS_RUN_COST;
#else
    const uint64_t w_run = c.qtab_off ? 80 : 12;
#endif
    // CW (same layout as U): levels L-1 .. 1 in full, level 0 compactly
    std::vector<uint64_t> arr(N1);
    for (uint64_t x = 0; x <= n; ++x) arr[x] = 1;  // one node
    p->CW.assign((size_t)X0 + (size_t)(L - 1) * N1, 0);
    bool ok = true;
    for (int k = L - 1; k >= 1 && ok; --k) {
      const uint64_t gk = gens[k];
      for (uint64_t x = gk; x <= n; ++x) arr[x] += arr[x - gk];
      if (k == L - 1)
        for (uint64_t x = 0; x <= n; ++x) arr[x] += w_run;  // each length-(L-1) prefix is a run
      for (uint64_t x = 0; x <= n; ++x)
        if (arr[x] >= (1ull << 62)) ok = false;
      memcpy(&p->CW[(size_t)X0 + (size_t)(k - 1) * N1], arr.data(), N1 * 8);
    }
    uint64_t acc = 0;
    for (uint64_t x = X0; x-- > 0 && ok;) {
      acc += arr[n - x * gens[0]];
      if (acc >= (1ull << 62)) ok = false;
      p->CW[x] = acc;
    }
    if (!ok) {
      p->CW.clear();
    } else {
      c.U = p->U.data();
      const uint64_t C = p->CW[0];
      uint32_t pre[FS_MAX_D];
      p->cost_begin = (uint64_t)((u128)C * r / W);
      p->cost_end = (uint64_t)((u128)C * (r + 1) / W);
      if (W > 1) {
        p->unit_begin = fs_host_cost_boundary(p, p->cost_begin, pre);
        p->unit_end = r + 1 == W ? U : fs_host_cost_boundary(p, p->cost_end, pre);
      }
    }
  }
  if (consumer == FS_CONSUMER_ROWS) {
    p->row_begin = p->unit_begin;
    p->row_end = p->unit_end;
  }
  // slice size
  const uint64_t span = p->unit_end - p->unit_begin;
  uint64_t T = e.slice_units;
  if (T == 0) T = std::max<uint64_t>(1, ceil_div_u64(span, kTargetLanes * kSlicesPerLane));
  T = std::min<uint64_t>(T, 1ull << 24);
  // materialise: small slices by default -- the 32 lanes of a warp write 32 consecutive slices,
  // and the closer their segments lie the better the DRAM write locality.  Canonical order
  // (M1): 64 rows (two 32-row flush groups per slice, so a warp's 32 segments of a flush are
  // 640 B apart), entered from the slice-start table (L + 1 words per 64 rows, +4 % bytes read)
  // when it fits FS_M1_TABLE_MB: C2-XL 4.79 -> 4.47 ms (T = 1088 -> 512 rows in round 1: 5.12
  // -> 4.91 ms; 128 rows + table 4.62; 128 rows by unrank 5.16).  Increasing order the same,
  // from a table of its mirrored slicing (fs_build_slice_starts; 64 rows by unrank: 6.3 vs 5.0
  // ms); order = any writes whole-warp blocks and keeps the larger slices (4.13 vs 4.26 ms).
  if (consumer == FS_CONSUMER_ROWS && e.slice_units == 0 && e.order != FS_ORDER_ANY) {
    const uint64_t t64 = ceil_div_u64(span, 64) * (uint64_t)(d - 1) * 4u;  // table bytes at T = 64
    T = std::min<uint64_t>(T, d >= 3 && t64 <= ((uint64_t)FS_M1_TABLE_MB << 20) ? 64 : 512);
  }
  if (consumer == FS_CONSUMER_ROWS) T = (T + 63) & ~63ull;  // slices start 128 B aligned
  p->T = T;
  p->num_slices = span ? ceil_div_u64(span, T) : 0;
  if (!p->CW.empty() && e.slice_units == 0 && span && e.slicing != FS_SLICES_UNIFORM) {
    // Equal-cost, guided slices (node units): the rank's cost range is cut at run starts into
    // P = 6 phases of one slice per resident lane each, every phase's slices half the cost of the
    // previous phase's (the first take half the rank).  Equal cost balances lanes whatever the lex
    // region (runs are short where a_1 is large, long where it is small); the large early slices
    // keep refills (claim + slice entry, ~100 warp instructions) at 6 per lane, and the last
    // slices are 1/63 of a lane's work, so the tail is short (round 1 / early round 2: 3 phases of
    // 4c, 2c, c with 12c per lane -- a 3x longer last slice; W = 8 virtual ranks of C3 lost ~0.09
    // ms per rank to it; finer slices in all phases cost more in refills than they saved).  A slice's first
    // node prefix and its node count come from the slice-start table (fs_build_slice_starts).
    // Slices are cut at run starts only, so this needs many more runs than lanes (C5, 231 runs of
    // ~3300 nodes, keeps uniform node slices, which split runs: 0.07 ms vs 0.36 ms).
#ifndef FS_GUIDED_PHASES
#define FS_GUIDED_PHASES 6  // phases of the guided slices, each slice half the cost of the last phase's
#endif
    const uint64_t S2 = FS_GUIDED_PHASES * kTargetLanes;
    const uint64_t runs_share = (uint64_t)((u128)p->nodes_per_level[d - 3] * (p->cost_end - p->cost_begin) /
                                           std::max<uint64_t>(1, p->CW[0]));
    // a slice's node count (< its cost + one run) must fit the kernel's 32-bit budget
    const bool forced = e.slicing == FS_SLICES_COST;  // (tests: at any size, S2 <= runs / 2)
    const uint64_t s2 = forced ? std::max<uint64_t>(1, std::min<uint64_t>(S2, runs_share / 2)) : S2;
    // automatic: for the closed-tail kernels, whose per-run cost the weights model (the per-row
    // kernels keep node slices: C3 per-row count 190 ms with them, 210 ms with cost slices)
    const bool closed_kernel = e.tail == FS_TAIL_CLOSED && (consumer == FS_CONSUMER_COUNT || consumer == FS_CONSUMER_HIST);
    // P phases of Lp slices: the first slices take half of the rank's cost (2^(P-1) / (2^P - 1)),
    // each later phase's slices half the cost of the phase before, so the last slices are
    // short (a short tail) while the refills stay at P per lane
    const uint64_t P = FS_GUIDED_PHASES, Lp = std::max<uint64_t>(1, s2 / P);
    if ((forced || (closed_kernel && runs_share >= 8 * kTargetLanes)) &&
        (p->cost_end - p->cost_begin) / Lp + n + 1024 < (1ull << 31)) {
      p->gn0 = Lp;
      p->gn1 = P;
      p->num_slices = P * Lp;
      p->cost_slices = true;
      p->T = std::max<uint64_t>(1, span / p->num_slices);  // reported average
    }
  }
  return FS_OK;
}

uint64_t fs_host_cost_boundary(const fs_plan *p, uint64_t target, uint32_t *pre) {
  fs::Consts c = p->c;
  c.U = p->U.data();
  switch (p->d) {
#define FS_CASE(DD) \
  case DD:          \
    return fs::cost_boundary<DD>(c, p->CW.data(), target, pre);
    FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
  }
  return 0;
}

void fs_plan_free_device(fs_plan *p) {
  if (!p->uploaded) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  if (p->U_dev) cudaFree(p->U_dev);
  if (p->CW_dev) cudaFree(p->CW_dev);
  p->CW_dev = nullptr;
  if (p->ktab_dev) cudaFree(p->ktab_dev);
  if (p->scratch_dev) cudaFree(p->scratch_dev);
  if (p->diff_dev) cudaFree(p->diff_dev);
  if (p->starts_dev) {
    if (p->starts_async)
      cudaFreeAsync(p->starts_dev, p->stream);  // back to the pool, stream-ordered after the plan's work
    else
      cudaFree(p->starts_dev);
  }
  p->diff_dev = nullptr;
  p->starts_dev = nullptr;
  p->U_dev = nullptr;
  p->ktab_dev = nullptr;
  p->scratch_dev = nullptr;
  p->uploaded = false;
  if (prev >= 0) cudaSetDevice(prev);
}

int fs_plan_upload_impl(fs_plan *p) {
  if (p->uploaded) return FS_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    return FS_ENODEV;
  }
  int dev = p->ex.device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) return FS_ECUDA;
  }
  if (dev >= ndev) return FS_EINVAL;
  if (cudaSetDevice(dev) != cudaSuccess) return FS_ECUDA;
  p->device = dev;
  p->stream = (cudaStream_t)p->ex.cuda_stream;
  if (!p->U.empty()) {
    if (cudaMalloc(&p->U_dev, p->U.size() * 8) != cudaSuccess) return FS_ENOMEM;
    if (cudaMemcpyAsync(p->U_dev, p->U.data(), p->U.size() * 8, cudaMemcpyHostToDevice, p->stream) !=
        cudaSuccess)
      return FS_ECUDA;
  }
  if (p->cost_slices) {
    if (cudaMalloc(&p->CW_dev, p->CW.size() * 8) != cudaSuccess) return FS_ENOMEM;
    if (cudaMemcpyAsync(p->CW_dev, p->CW.data(), p->CW.size() * 8, cudaMemcpyHostToDevice, p->stream) != cudaSuccess)
      return FS_ECUDA;
  }
  if (!p->ktab.empty()) {
    if (cudaMalloc(&p->ktab_dev, p->ktab.size() * 4) != cudaSuccess) return FS_ENOMEM;
    if (cudaMemcpyAsync(p->ktab_dev, p->ktab.data(), p->ktab.size() * 4, cudaMemcpyHostToDevice,
                        p->stream) != cudaSuccess)
      return FS_ECUDA;
  }
  if (cudaMalloc(&p->scratch_dev, fs::kScratchBytes) != cudaSuccess) return FS_ENOMEM;
  p->uploaded = true;
  return fs_build_slice_starts(p);
}

// ------------------------------------------------------------------ host model (tests only)
namespace {

struct HostSink {
  int d = 0;
  const uint8_t *perm = nullptr;  // internal coordinate j -> caller coordinate perm[j]
  uint64_t count = 0;
  uint64_t *hist = nullptr;
  uint64_t hist_cap = 0;
  int B = 0;
  unsigned char *rows = nullptr;
  uint64_t cap = 0;
  uint64_t slice_rows = 0;
  std::vector<int64_t> diffv;
  int64_t *diff = nullptr;
  std::vector<int64_t> hq_sh;  // state-form histogram: one lane-copy of the kernel's shared array
  bool hq_bad = false;
  uint32_t first[FS_MAX_D];
  bool have_first = false;
  // any-predicate (fsdbg_host_any): pred_arg in the caller's coordinates; pred_arg_int with
  // COORD_GE's index remapped to the stream's order (closed-form node test)
  int pred = 0;
  uint64_t pred_arg = 0, pred_arg_int = 0;
  bool found = false;
  uint32_t wit[FS_MAX_D];
  void hit(const uint32_t *v) {  // v in the caller's coordinates
    if (found) return;
    found = true;
    memcpy(wit, v, sizeof(uint32_t) * d);
  }
  void put(const uint32_t *vi) {
    uint32_t v[FS_MAX_D];
    for (int j = 0; j < d; ++j) v[perm ? perm[j] : j] = vi[j];
    if (pred) {
      uint64_t len = 0;
      for (int i = 0; i < d; ++i) len += v[i];
      bool ok = false;
      const uint64_t ci = pred_arg >> 32;
      switch (pred) {
        case FS_PRED_LEN_LE: ok = len <= pred_arg; break;
        case FS_PRED_LEN_GE: ok = len >= pred_arg; break;
        case FS_PRED_LEN_EQ: ok = len == pred_arg; break;
        default: ok = ci < (uint64_t)d && v[ci] >= (uint32_t)(pred_arg & 0xffffffffu);
      }
      if (ok) hit(v);
    }
    uint64_t len = 0;
    for (int i = 0; i < d; ++i) len += v[i];
    if (hist && len < hist_cap) hist[len]++;
    if (rows && count < cap) {
      const int w = B / 8;
      unsigned char *q = rows + count * (uint64_t)d * w;
      for (int i = 0; i < d; ++i)
        for (int b = 0; b < w; ++b) q[i * w + b] = (unsigned char)((v[i] >> (8 * b)) & 0xff);
    }
    if (!have_first) {
      memcpy(first, v, sizeof(uint32_t) * d);
      have_first = true;
    }
    ++count;
    ++slice_rows;
  }
};

template <int D>
struct HostEmit {
  HostSink *sink;
  FS_HD void cond(bool em, const fs::Lane<D> &st, const fs::Consts &c) {
#ifndef __CUDA_ARCH__
    if (!em) return;
    uint32_t v[FS_MAX_D];
    for (int j = 0; j < D - 2; ++j) v[j] = fs::cur_coord<D>(st, j);
    v[D - 2] = (uint32_t)st.cur;
    v[D - 1] = fs::row_ad<D>(st, c);
    sink->put(v);
#endif
  }
};

// closed-tail node consumer of the host model: the count, and the length histogram through
// the same strided difference array the kernels use (resolved by host_finish_diff)
struct HostNodeSink {
  const fs_plan *p;
  HostSink *sink;
  uint64_t n;
  template <int D>
  void node(bool em, const fs::Lane<D> &st, const fs::Consts &c, uint32_t rows) {
    if (!em) return;
    n += rows;
    if (sink->pred) {  // the kernels' closed-form any test of the node
      uint32_t j;
      if (fs::any_closed_pick<D>(st, c, rows, sink->pred, sink->pred_arg_int, j)) {
        uint32_t vi[FS_MAX_D], v[FS_MAX_D];
        for (int q = 0; q < D - 2; ++q) vi[q] = fs::cur_coord<D>(st, q);
        vi[D - 2] = (uint32_t)st.cur - j * c.s;
        vi[D - 1] = fs::row_ad<D>(st, c) + j * c.t;
        for (int q = 0; q < D; ++q) v[c.perm[q]] = vi[q];
        sink->hit(v);
      }
    }
    if (sink->diff) {
      uint32_t lo, hi, v;
      fs::hist_diff_updates<D>(st, c, rows, lo, hi, v);
      sink->diff[lo] += (int64_t)v;
      sink->diff[hi] -= (int64_t)v;
    }
  }
};

// The state-form histogram (fs_kernels.cuh hq_group / enter_h) replayed on the host
// for one lane and one slice, reading the same table words (links are byte offsets from the
// table start; copy j = lane mod FS_HQ_COPIES), with the kernel's shared index arithmetic: every
// update lands in `sh` (one lane-copy of the shared array, index = address / stride), and the
// replay fails (bad) if an address leaves the array or is not index-aligned (masked nodes of a
// block included).  Ascends take the generic ascend (the kernel's t2 ascend table is pinned
// separately).
template <int D, class KT>
void host_hist_tables_slice(const fs_plan *p, const KT &ktab, fs::Lane<D> &st, uint32_t &budget, uint32_t j,
                            std::vector<int64_t> &sh, bool &bad) {
  const fs::Consts &c = p->c;
  const uint32_t *W = p->ktab.data();
  constexpr int L = D - 2;
  constexpr uint32_t K = FS_HK, C = FS_HQ_COPIES, STR = 4u * FS_HIST_REP;
  uint32_t h = 0, h1 = 0, bP = 0, bM = 0;
  auto upd = [&](uint32_t addr, int64_t v) {
    if (addr % STR != 0u || addr / STR >= sh.size()) {
      bad = true;
      return;
    }
    sh[addr / STR] += v;
  };
  // enter_h: the entered node (A, rho; entry unit not charged) becomes the next node to take,
  // a_L and lsum those of its virtual predecessor (one more)
  auto enter = [&]() {
    if constexpr (L >= 1) {
      st.a[L - 1] += 1u;
      st.lsum += 1u;
    }
    st.cur = -1;
    fs::sync_k<D, 1>(st, budget);
    const uint32_t Q = st.A / c.s, a = st.A % c.s;
    const uint32_t X = STR * (st.lsum + c.s * Q + c.hq_bias);
    const uint32_t Y = X + STR * Q * (uint32_t)c.dl;
    const uint32_t sig = st.rho * c.s + a;
    h = c.hq_off + 4u * (C * (2u * sig + (sig & 1u)) + j);
    h1 = c.hq_off + 4u * (C * (2u * sig + (1u - (sig & 1u))) + j);
    bP = c.dl > 0 ? X : Y;
    bM = c.dl > 0 ? Y : X;
  };
  enter();
  while (!fs::needs_refill<D, 1>(st, budget)) {
    const uint32_t kk = st.k;
    for (uint32_t v = 0; v < FS_HQ_GROUP / K; ++v) {  // hq_group: masked 8-node blocks
      if (kk <= K * v) break;
      const uint32_t *w = W + h, *w1 = W + h1;
      for (uint32_t i = 0; i < K; ++i) {
        const uint32_t pm = w1[i / 2u] >> (16u * (i % 2u));
        const uint32_t aP = bP + STR * (uint32_t)(int32_t)(int8_t)(pm & 0xffu);
        upd(aP, 1);  // masked nodes (past the run or slice): -1 on the same index, net zero
        upd(K * v + i < kk ? bM + STR * (uint32_t)(int32_t)(int8_t)((pm >> 8) & 0xffu) : aP, -1);
      }
      h = w[0] / 4u;
      h1 = w[3] / 4u;
      bP += w[1];
      bM += w[2];
    }
    st.k = kk > FS_HQ_GROUP ? kk - FS_HQ_GROUP : 0u;
    fs::sync_k<D, 1>(st, budget);
    if (!fs::needs_slow<D>(st, budget)) continue;
    if (!fs::advance_cd<D, 1>(st, c, budget)) {  // (a_L = 0: the ascend) end of stream or slice
      budget = 0;
      break;
    }
    enter();
  }
}

// The kernels' count-only closed tail with the tables (fs_kernels.cuh cc_group2, t2_ascend,
// t3_ascend) replayed on the host for one lane, reading the same host table words: the link
// words hold byte offsets from the table start (the kernels add their shared-memory base), and
// the lane's copy of the paired table is j = lane mod 8.  Returns the slice's rows.
template <int D, class KT>
uint64_t host_count_tables_slice(const fs_plan *p, const KT &ktab, fs::Lane<D> &st, uint32_t &budget, uint32_t j) {
  const fs::Consts &c = p->c;
  const uint32_t *W = p->ktab.data();
  constexpr int L = D - 2;
  const bool qform = c.qtab_off != 0;  // the kernel's state form (cq_group, enter_q, t2q_ascend)
  const uint32_t G = qform ? FS_CQ_GROUP : FS_CC_GROUP;
  const uint32_t t2off = qform ? c.t2q_off : c.t2_off;
  uint64_t n = 0;
  uint32_t hq = 0, Q = 0;  // state form: word index of the lane's state entry, quotient
  auto take_entry = [&]() {
    const int32_t x = st.cur + (int32_t)c.s;
    st.cur = -1;
    n += fs::divq((uint32_t)(x > 0 ? x : 0), c.dvS);
  };
  constexpr uint32_t K = FS_QK;
  // fs_kernels.cuh enter_q: the entered node (A, rho) as a state; r = st.k mod K advances now
  auto enter_q_from = [&](uint32_t sig128, uint32_t q) {
    const uint32_t r = st.k % K;
    if (r) {
      const uint32_t *w = W + c.q1_off + 2u * ((K - 1u) * (sig128 / 128u) + r - 1u);
      n += (uint64_t)r * q + w[1];
      q += w[0] >> 16;
      sig128 = w[0] & 0xffffu;
      st.k -= r;
    }
    Q = K * q;  // the group keeps QK = K Q
    hq = c.qtab_off + (sig128 + 16u * j) / 4u;
  };
  auto enter_q = [&]() {
    if (!qform) return;
    const uint32_t q = fs::divq(st.A, c.dvS);
    enter_q_from(128u * (st.rho * c.s + (st.A - q * c.s)), q);
  };
  uint32_t t2w = 0, q2 = 0, t3w = 0, q3 = 0;  // word indices of the t2 / t3 entries
  auto t2_sync = [&]() {
    if constexpr (D >= 4) {
      if (!c.t2_off) return;
      const uint32_t R1 = st.R[L - 2];
      q2 = fs::divq(R1, c.dv[L - 1]);
      const uint32_t r = R1 - q2 * c.g[L - 1];
      t2w = t2off + (qform ? 4u * (K * r + (q2 & (K - 1u))) : 4u * r);
    }
  };
  auto t3_sync = [&]() {
    if constexpr (D >= 5) {
      if (!c.t3_off) return;
      const uint32_t R3 = st.R[L - 3];
      q3 = fs::divq(R3, c.dv[L - 2]);
      t3w = c.t3_off + 4u * (R3 - q3 * c.g[L - 2]);
    }
  };
  take_entry();
  t2_sync();
  t3_sync();
  enter_q();
  while (!fs::needs_refill<D, 1>(st, budget)) {
    uint32_t gsum = 0;  // the kernel's 32-bit group sum (folded into 64 bits per group)
    if (qform) {  // cq_group: G nodes in blocks of K, one predicate per block (kk = 0 mod K)
      const uint32_t kk = st.k;
      for (uint32_t v = 0; v < G / K; ++v) {
        const uint32_t *w = W + hq;
        hq = w[0] / 4u;
        if (K * v < kk) gsum += Q + w[1];  // Q holds K Q here
        Q += w[2];
      }
      st.k = kk > G ? kk - G : 0u;
    } else if constexpr (D >= 3) {  // cc_group2: G nodes, two per paired-table entry
      const bool skip = c.cadv2_skip != 0;
      const uint32_t ew = skip ? 8u : 4u;  // words per entry
      uint32_t h = c.cadv2_off + ew * (8u * st.rho + j);
      uint32_t A = st.A;
      const uint32_t kk = st.k;
      uint32_t cum = 0;  // advances taken (skip form), else 2 per pair
      for (uint32_t v = 0; v < G / 2; ++v) {
        const uint32_t *w = W + h;
        h = w[0] / 4u;
        int32_t x1 = (int32_t)(A + w[1]), x2 = (int32_t)(A + w[2]);
        x1 = x1 > 0 ? x1 : 0;
        x2 = x2 > 0 ? x2 : 0;
        A += w[3];
        const uint32_t c1 = skip ? cum + w[4] : 2u * v + 1u, c2 = skip ? cum + w[5] : 2u * v + 2u;
        if (c1 <= kk) gsum += (uint32_t)(((uint64_t)(uint32_t)x1 * c.mhi) >> 32);
        if (c2 <= kk) gsum += (uint32_t)(((uint64_t)(uint32_t)x2 * c.mhi) >> 32);
        cum = c2;
      }
      st.rho = (h - c.cadv2_off) / (8u * ew);
      st.A = A;
      st.k = kk > cum ? kk - cum : 0u;
    }
    n += gsum;
    fs::sync_k<D, 1>(st, budget);
    if (fs::needs_slow<D>(st, budget)) {
      bool done = false;
      if constexpr (D >= 4) {
        if (c.t2_off && st.a[L - 2] > 0u && (!qform || c.t2q_off)) {  // t2_ascend / t2q_ascend
          const uint32_t *w = W + t2w;
          t2w = (w[0] & 0xffffu) / 4u;
          q2 += w[0] >> 16;
          st.a[L - 2] -= 1u;
          st.R[L - 2] += c.g[L - 2];
          st.a[L - 1] = q2;
          st.lsum = st.lsum - 1u + q2;
          st.cur = -1;
          budget -= 1u;
          fs::sync_k<D, 1>(st, budget);
          if (qform && st.k == st.a[L - 1]) {  // t2q_ascend: entry node + j advances, precomputed
            n += w[2];
            Q = K * (w[1] >> 16);
            hq = c.qtab_off + ((w[1] & 0xffffu) + 16u * j) / 4u;
            st.k -= w[3];
          } else if (qform) {  // the budget ends inside the run: the entry node, then enter_q
            const uint32_t r2 = (t2w - t2off) / 4u / K;  // R_L of the new run's first node
            const uint32_t A0 = r2 / c.gA, rho0 = r2 % c.gA, q0 = A0 / c.s, a0 = A0 % c.s;
            n += q0 + (a0 >= ktab(rho0, c) ? 1u : 0u);
            enter_q_from(128u * (rho0 * c.s + a0), q0);
          } else {
            st.rho = w[1] & 0xffffu;
            st.A = w[1] >> 16;
            n += w[2];
          }
          done = true;
        }
      }
      if constexpr (D >= 5) {
        if (!done && c.t3_off && st.a[L - 2] == 0u && st.a[L - 3] > 0u) {  // t3_ascend
          const uint32_t *w = W + t3w;
          t3w = (w[0] & 0xffffu) / 4u;
          q3 += w[0] >> 16;
          st.a[L - 3] -= 1u;
          st.R[L - 3] += c.g[L - 3];
          st.a[L - 2] = q3;
          st.R[L - 2] = w[2] >> 16;
          const uint32_t aL = w[3] >> 16;
          st.a[L - 1] = aL;
          st.lsum = st.lsum - 1u + q3 + aL;
          st.rho = w[1] & 0xffffu;
          st.A = w[1] >> 16;
          st.cur = -1;
          n += w[2] & 0xffffu;
          q2 = aL;
          t2w = t2off + (qform ? 4u * (K * (w[3] & 0xffffu) + (aL & (K - 1u))) : 4u * (w[3] & 0xffffu));
          budget -= 1u;
          fs::sync_k<D, 1>(st, budget);
          enter_q();
          done = true;
        }
      }
      if (!done) {
        fs::slow_step<D, true, 1>(st, c, ktab, budget);
        fs::sync_k<D, 1>(st, budget);
        take_entry();
        t2_sync();
        t3_sync();
        enter_q();
      }
    }
  }
  return n;
}

// The batch materialise kernel's row stream (fs_rows_batch.cuh rb_ensure_row) replayed on the
// host for one full row slice: table advances from the radv entry of the current residue
// (next residue, quotient increment, k0 and a_d of the next node's first row), generic ascend
// otherwise; one row per step.  Pins the radv table against the oracle on the CPU.
template <int D, class KT>
void host_rows_batch_slice(const fs_plan *p, const KT &ktab, fs::Lane<D> &st, uint32_t rows, HostSink &sink) {
  const fs::Consts &c = p->c;
  const uint32_t *W = p->ktab.data();
  constexpr int L = D - 2;
  uint32_t ad = fs::divq((st.A - (uint32_t)st.cur) * c.gA + st.rho, c.dvB);
  for (uint32_t r = 0; r < rows; ++r) {
    if constexpr (L >= 1) {
      while (st.cur < 0) {
        const uint32_t *w = W + c.radv_off + 4u * st.rho;
        if (st.a[L - 1] >= w[3]) {  // to the next live node, w[3] advances at once
          st.a[L - 1] -= w[3];
          st.rho = w[0] & ((1u << fs::kAdvBits) - 1u);
          st.A += w[0] >> fs::kAdvBits;
          st.cur = (int32_t)st.A - (int32_t)w[1];
          ad = w[2];
        } else {  // the rest of the run is dead (or empty): ascend
          st.lsum -= st.a[L - 1];
          st.a[L - 1] = 0u;
          if (!fs::ascend<D>(st, c)) return;  // end of stream (not inside a full slice)
          st.cur = (int32_t)st.A - (int32_t)ktab(st.rho, c);
          ad = fs::divq((st.A - (uint32_t)st.cur) * c.gA + st.rho, c.dvB);
        }
      }
    }
    uint32_t v[FS_MAX_D];
    for (int q = 0; q < L; ++q) v[q] = st.a[q];
    v[D - 2] = (uint32_t)st.cur;
    v[D - 1] = ad;
    sink.put(v);
    st.cur -= (int32_t)c.s;
    ad += c.t;
  }
}

template <int D, int ALPHA, class KT>
void host_model_d(const fs_plan *p, const KT &ktab, HostSink &sink, uint64_t *slice_counts, uint32_t *slice_first) {
  const Consts &c = p->c;
  for (uint64_t sl = 0; sl < p->num_slices; ++sl) {
    uint64_t u, e;
    if (p->cost_slices) {  // the slice-start table's cost boundaries (fs_build_slice_starts)
      uint32_t pre[FS_MAX_D];
      const uint64_t S = p->num_slices;
      u = sl == 0 ? p->unit_begin
                  : fs_host_cost_boundary(p, fs::cost_target(p->cost_begin, p->cost_end, p->gn0, p->gn1, S, sl), pre);
      e = sl + 1 == S ? p->unit_end
                      : fs_host_cost_boundary(p, fs::cost_target(p->cost_begin, p->cost_end, p->gn0, p->gn1, S, sl + 1), pre);
      if (e <= u) {  // an empty slice (two targets inside one run)
        if (slice_counts) slice_counts[sl] = 0;
        if (slice_first)
          for (int i = 0; i < D; ++i) slice_first[sl * D + i] = 0xFFFFFFFFu;
        continue;
      }
    } else {
      fs::slice_range(p->unit_begin, p->unit_end, p->T, p->gn0, p->gn1, sl, u, e);
    }
    uint32_t budget = (uint32_t)(e - u);
    fs::Lane<D> st;
    uint64_t off = fs::unrank<D, true>(st, c, ktab, u);
    budget -= fs::position_in_node<D, true>(st, c, off);
    fs::sync_k<D, ALPHA>(st, budget);
    sink.slice_rows = 0;
    sink.have_first = false;
    HostEmit<D> emit{&sink};
    // the kernels' schedule: branch-free fast steps, slow_step() for lanes needing an ascend
    if (ALPHA && p->consumer == FS_CONSUMER_COUNT &&
        (p->ex.tail == FS_TAIL_SKIP_OFF || p->ex.tail == FS_TAIL_SKIP_PAPER)) {
      const bool paper = p->ex.tail == FS_TAIL_SKIP_PAPER;
      uint64_t cnt = 0;
      fs::enter_candidates<D>(st, c);
      while (!fs::needs_refill<D, ALPHA>(st, budget)) {
        uint32_t step_cnt = 0;  // the kernel's 32-bit per-iteration counter
        if (paper)
          fs::fast_step_cand<D, true>(st, c, ktab, budget, step_cnt);
        else
          fs::fast_step_cand<D, false>(st, c, ktab, budget, step_cnt);
        cnt += step_cnt;
        fs::sync_k<D, ALPHA>(st, budget);
        if (fs::needs_slow<D>(st, budget)) {
          fs::slow_step<D, true, ALPHA>(st, c, ktab, budget);
          fs::enter_candidates<D>(st, c);
          fs::sync_k<D, ALPHA>(st, budget);
        }
      }
      sink.count += cnt;
      sink.slice_rows = cnt;
    } else if (ALPHA &&
               (p->consumer == FS_CONSUMER_COUNT || p->consumer == FS_CONSUMER_HIST || p->consumer == FS_CONSUMER_ANY) &&
               p->ex.tail == FS_TAIL_CLOSED) {
      HostNodeSink ns{p, &sink, 0};
      const bool count_only = p->consumer == FS_CONSUMER_COUNT && !sink.pred;
      if (count_only && p->c.cadv2_off != 0) {  // the kernel's table-driven group form
        ns.n += host_count_tables_slice<D>(p, ktab, st, budget, (uint32_t)(sl & 7u));
        budget = 0;
        st.cur = -1;
      }
      if (sink.diff && !sink.hq_sh.empty()) {  // the kernel's state-form histogram
        budget += 1u;  // (position_in_node charged the entry unit: enter_h takes it as a node)
        host_hist_tables_slice<D>(p, ktab, st, budget, (uint32_t)(sl % FS_HQ_COPIES), sink.hq_sh, sink.hq_bad);
        budget = 0;
        st.cur = -1;
      }
      while (!fs::needs_refill<D, ALPHA>(st, budget)) {
        if (count_only) {  // the kernels' count-only closed step
          uint64_t cnt = 0;
          fs::fast_step_count_closed<D>(st, c, ktab, cnt);
          ns.n += cnt;
        } else {
          fs::fast_step_closed<D>(st, c, ktab, budget, ns);
        }
        fs::sync_k<D, ALPHA>(st, budget);
        if (fs::needs_slow<D>(st, budget)) {
          fs::slow_step<D, true, ALPHA>(st, c, ktab, budget);
          fs::sync_k<D, ALPHA>(st, budget);
        }
      }
      sink.count += ns.n;
      sink.slice_rows = ns.n;
    } else if (!ALPHA && p->c.radv_off != 0 && p->ex.rows_impl == FS_ROWS_BATCH && !p->c.permuted) {
      // the batch kernel's stream (its own row-unit slices: st is at row `off` of the node)
      host_rows_batch_slice<D>(p, ktab, st, budget, sink);
    } else {
      while (!fs::needs_refill<D, ALPHA>(st, budget)) {
        fs::fast_step<D, true, ALPHA>(st, c, ktab, budget, emit);
        fs::sync_k<D, ALPHA>(st, budget);
        if (fs::needs_slow<D>(st, budget)) {
          fs::slow_step<D, true, ALPHA>(st, c, ktab, budget);
          fs::sync_k<D, ALPHA>(st, budget);
        }
      }
    }
    if (slice_counts) slice_counts[sl] = sink.slice_rows;
    if (slice_first) {
      for (int i = 0; i < D; ++i) slice_first[sl * D + i] = sink.have_first ? sink.first[i] : 0xFFFFFFFFu;
    }
  }
}

template <int D, class KT>
void host_model_kt(const fs_plan *p, const KT &kt, HostSink &sink, uint64_t *sc, uint32_t *sf) {
  if (p->c.alpha)
    host_model_d<D, 1>(p, kt, sink, sc, sf);
  else
    host_model_d<D, 0>(p, kt, sink, sc, sf);
}

template <int D>
void host_model_alpha(const fs_plan *p, HostSink &sink, uint64_t *sc, uint32_t *sf) {
  if (!p->ktab.empty())
    host_model_kt<D>(p, fs::KTabPtr{p->ktab.data(), p->c.adv_off}, sink, sc, sf);
  else
    host_model_kt<D>(p, fs::KTabArith{}, sink, sc, sf);
}

}  // namespace

extern "C" int fsdbg_host_model(const fs_plan *p, uint64_t *count_out, uint64_t *hist, uint64_t hist_cap,
                                int B, void *rows, uint64_t cap, uint64_t *slice_counts,
                                uint32_t *slice_first_row) {
  if (!p) return FS_EINVAL;
  if (rows && B != 16 && B != 32) return FS_EINVAL;
  HostSink sink;
  sink.d = p->d;
  sink.perm = p->c.perm;
  sink.hist = hist;
  sink.hist_cap = hist_cap;
  sink.B = B;
  sink.rows = (unsigned char *)rows;
  sink.cap = cap;
  if (hist) memset(hist, 0, hist_cap * 8);
  const bool closed_hist = hist && p->consumer == FS_CONSUMER_HIST && p->ex.tail == FS_TAIL_CLOSED && p->d >= 2;
  if (closed_hist) {
    sink.diffv.assign(p->hist_len + p->c.dstride + 1, 0);
    sink.diff = sink.diffv.data();
    const fs_hist_shape hs = fs_hist_closed_shape(p);
    if (hs.hq) sink.hq_sh.assign(hs.slen, 0);
  }
  if (p->d == 1) {
    // one slice, one unit at most
    for (uint64_t sl = 0; sl < p->num_slices; ++sl) {
      sink.slice_rows = 0;
      sink.have_first = false;
      uint32_t v = (uint32_t)(p->n / p->g[0]);
      sink.put(&v);
      if (slice_counts) slice_counts[sl] = sink.slice_rows;
      if (slice_first_row) slice_first_row[sl] = v;
    }
  } else {
    switch (p->d) {
#define FS_CASE(DD) \
  case DD:          \
    host_model_alpha<DD>(p, sink, slice_counts, slice_first_row); \
    break;
      FS_CASE(2) FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
      FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
      default:
        return FS_EINVAL;
    }
  }
  if (closed_hist && !sink.hq_sh.empty()) {  // the shared array's indices hq_bias + l; margins net to zero
    const fs_hist_shape hs = fs_hist_closed_shape(p);
    for (uint64_t i = 0; i < sink.hq_sh.size(); ++i) {
      const int64_t l = (int64_t)i - (int64_t)hs.sbias;
      if (l >= 0 && l < (int64_t)hs.diff_len)
        sink.diff[l] += sink.hq_sh[i];
      else if (sink.hq_sh[i] != 0)
        sink.hq_bad = true;
    }
    if (sink.hq_bad) return FS_ERANGE;  // the replay left the kernel's shared array
  }
  if (closed_hist) {  // strided prefix sums of the difference array
    const uint64_t L = p->hist_len, S = p->c.dstride;
    for (uint64_t r = 0; r < S && r < L; ++r) {
      int64_t acc = 0;
      for (uint64_t l = r; l < L; l += S) {
        acc += sink.diff[l];
        if (l < hist_cap) hist[l] = (uint64_t)acc;
      }
    }
  }
  if (count_out) *count_out = sink.count;
  return FS_OK;
}

// The any-predicate through the host model: per row (tail rows) or per node in closed form
// (tail closed, any_closed_pick), in the kernels' schedule.  *found_out and one witness row
// (caller's coordinates; which one is unspecified, as for fs_any).
extern "C" int fsdbg_host_any(const fs_plan *p, int pred, uint64_t pred_arg, int *found_out, uint32_t *witness) {
  if (!p || !found_out || pred < FS_PRED_LEN_LE || pred > FS_PRED_COORD_GE) return FS_EINVAL;
  if (p->consumer != FS_CONSUMER_ANY) return FS_EINVAL;
  HostSink sink;
  sink.d = p->d;
  sink.perm = p->c.perm;
  sink.pred = pred;
  sink.pred_arg = pred_arg;
  sink.pred_arg_int = pred_arg;
  if (pred == FS_PRED_COORD_GE && (pred_arg >> 32) < (uint64_t)p->d)
    sink.pred_arg_int = ((uint64_t)p->iperm[pred_arg >> 32] << 32) | (pred_arg & 0xffffffffull);
  if (p->d == 1) {
    for (uint64_t sl = 0; sl < p->num_slices; ++sl) {
      uint32_t v = (uint32_t)(p->n / p->g[0]);
      sink.put(&v);
    }
  } else {
    switch (p->d) {
#define FS_CASE(DD) \
  case DD:          \
    host_model_alpha<DD>(p, sink, nullptr, nullptr); \
    break;
      FS_CASE(2) FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
      FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
      default:
        return FS_EINVAL;
    }
  }
  *found_out = sink.found ? 1 : 0;
  if (sink.found && witness) memcpy(witness, sink.wit, sizeof(uint32_t) * p->d);
  return FS_OK;
}

namespace {
template <int D>
int unrank_host(const fs_plan *p, uint64_t unit, uint32_t *prefix_out, int64_t *row_out) {
  fs::Lane<D> st;
  uint64_t off = p->ktab.empty() ? fs::unrank<D, true>(st, p->c, fs::KTabArith{}, unit)
                                 : fs::unrank<D, true>(st, p->c, fs::KTabPtr{p->ktab.data(), p->c.adv_off}, unit);
  for (int j = 0; j < D - 2; ++j) prefix_out[j] = st.a[j];
  *row_out = p->c.alpha ? -1 : (int64_t)off;
  return FS_OK;
}
}  // namespace

extern "C" int fsdbg_unrank(const fs_plan *p, uint64_t unit, uint32_t *prefix_out, int64_t *row_in_node_out) {
  if (!p || !prefix_out || !row_in_node_out) return FS_EINVAL;
  if (unit >= p->total_units) return FS_ERANGE;
  if (p->d == 1) {
    *row_in_node_out = 0;
    return FS_OK;
  }
  switch (p->d) {
#define FS_CASE(DD) \
  case DD:          \
    return unrank_host<DD>(p, unit, prefix_out, row_in_node_out);
    FS_CASE(2) FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
  }
  return FS_EINVAL;
}

extern "C" int fsdbg_magic(uint32_t g, uint32_t *m_out, uint32_t *sh_out) {
  if (g == 0 || g >= (1u << 31)) return FS_EINVAL;
  Div v = fs_make_div(g);
  if (m_out) *m_out = v.m;
  if (sh_out) *sh_out = v.sh;
  return FS_OK;
}

extern "C" uint32_t fsdbg_magic_div(uint32_t x, uint32_t g) { return fs::divq(x, fs_make_div(g)); }
extern "C" uint64_t fsdbg_claim_slice(uint64_t idx, uint32_t bits, uint64_t S) { return fs::claim_slice(idx, bits, S); }

// The closed-tail histogram's launch shape.  32-bit shared difference bins only while one
// inner-loop iteration of a CTA (256 lanes x FS_CC_GROUP nodes, <= 2^29 at < 2^17 rows per node)
// changes a bin by less than the kernel's 2^30 drain guard, so a bin stays below 2^31; else
// 64-bit global atomics.  Group-form kernels spread the shared updates over 32 lane-private
// copies (one bank each: no bank conflicts) when they fit; the state form (hq_group) needs
// them (its table offsets are pre-multiplied by the copies' index stride) and margins for
// rowless nodes (shared index = length + hq_bias, up to the top length + t + dstride).
fs_hist_shape fs_hist_closed_shape(const fs_plan *p) {
  fs_hist_shape h{};
  h.diff_len = (uint32_t)(p->hist_len + p->c.dstride);
  const uint64_t max_node_rows = (p->n / p->c.gA) / (p->c.s ? p->c.s : 1) + 1;
  h.hist_smem = h.diff_len <= fs::kHistSmemMax && max_node_rows < (1ull << 17) ? 1u : 0u;
  h.hist_rep = (h.hist_smem && p->c.cadv_off && (size_t)(h.diff_len + 1) * FS_HIST_REP * 4 <= fs::kHistRepBytes)
                   ? (uint32_t)FS_HIST_REP : 1u;
  h.slen = h.diff_len + 1u;
  h.sbias = 0;
  // (top: a node's first-row or lowest-row length is <= lsum + R_L / g_{d-1} + t; on a masked
  // node up to 7 advances past a run's end R_L grows by up to 7 g_L: ceil(7 g_L / g_{d-1}) more)
  const uint64_t gL = p->d >= 3 ? p->c.g[p->d - 3] : 0;
  const uint64_t slen_hq =
      (uint64_t)p->c.hq_bias + p->hist_len + p->c.t + p->c.dstride + (7 * gL + p->c.gA - 1) / p->c.gA + 1;
  if (p->c.hq_off && h.hist_rep == (uint32_t)FS_HIST_REP && slen_hq * FS_HIST_REP * 4 <= fs::kHistRepBytes) {
    h.hq = 1;
    h.slen = (uint32_t)slen_hq;
    h.sbias = p->c.hq_bias;
  }
  return h;
}

