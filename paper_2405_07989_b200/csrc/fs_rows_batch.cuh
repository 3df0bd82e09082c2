// fs_rows_batch.cuh -- materialise (the paper's "saving the factorizations",
// P:55) with one row per lane per step, in lockstep across the warp.
//
// Row-unit slices hold exactly T rows (T a multiple of 64), so once every lane of a warp has a
// full slice, every lane emits exactly one row per step: the step first moves an exhausted
// lane to the next node that has rows (Alg. 3.1 at index L -- a 16 B shared-table advance --
// or the rare ascend at an index < L, with the modulo skip applied at entry,
// P:170-176), then takes the node's next row (a_{d-1} -= s, a_d += t).  Because the row index
// inside a batch is a compile-time constant, a batch of NB rows (NB * row_bytes a multiple of
// 16) is assembled in registers with fixed shifts, written to the lane's shared-memory slot
// with 16 B stores (a lane stride of an odd number of 16 B units keeps each quarter-warp on
// distinct banks), and after NBUF batches the warp copies all 32 slots out with 16 B stores:
//   canonical (M1): lane l's slot goes to its slice's exact byte offset (a contiguous
//                   segment of NBUF * NB rows per lane),
//   any (M2):       the warp reserves 32 * NBUF * NB rows on the front cursor with one
//                   atomicAdd and writes its whole staging area as ONE contiguous block.
// The rank's ragged last slice (< T rows) is written by fs_rows_tail_kernel.
// MODE 2 (increasing lex order, "could readily be modified to proceed in increasing
// order"): the same stream written mirrored -- output row p holds canonical row E-1-p of the
// enumerated range [0, E); slices are anchored at the output side (slice j = output rows
// [jT, jT + T) = canonical rows [E - jT - T, E - jT)), rows inside a batch and batches inside
// a group are placed in reverse, so every group is still one aligned 16 B-multiple segment;
// the ragged slice (canonical rows [0, E - nfull T)) goes to the tail kernel.
#pragma once

#include "fs_kernels.cuh"

namespace fs {

constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }

#ifndef FS_RB_BLOCK
#define FS_RB_BLOCK 128  // threads per CTA of the batch kernel (measured: 128 > 192 > 256)
#endif
constexpr int kRbBlock = FS_RB_BLOCK;
#ifndef FS_RB_TMA
// M1 / increasing order: per-lane bulk (TMA, cp.async.bulk) copies of each group's segment
// instead of the warp's LDS/STG copy loop.  Measured on C2-XL (r2f): 4.87 ms with it vs 4.78 ms
// without (and 640 B segments: 7.0 ms, fewer resident warps), so the copy instructions are not
// what holds M1 at 0.83 of the copy peak; kept as an option, off by default.
#define FS_RB_TMA 0
#endif
constexpr bool kRbTma = FS_RB_TMA != 0;

#ifndef FS_RB_GMAX
#define FS_RB_GMAX 320  // bytes per lane per flush group (upper bound)
#endif

template <int D, int B>
struct RowsBatchGeom {
  static constexpr int RB = D * (B / 8);              // row bytes
  static constexpr int NB = 16 / cgcd(RB, 16);        // rows per 16 B-aligned batch (1, 2, 4 or 8)
  static constexpr int BB = NB * RB;                  // batch bytes
  static constexpr int BW = BB / 4;                   // batch words
  static constexpr bool kOk = D >= 2 && BB <= 112;    // register budget of the batch
  static constexpr int nbuf_(int p) { return (2 * p * NB <= 64 && 2 * p * BB <= FS_RB_GMAX) ? nbuf_(2 * p) : p; }
  static constexpr int NBUF = nbuf_(1);               // batches per flush group (power of two)
  static constexpr int GR = NB * NBUF;                // rows per lane per group (divides 64)
  static constexpr int FG = NBUF * BB;                // bytes per lane per group
  static constexpr int C = FG / 16;                   // 16 B chunks per lane per group
  static constexpr int STRIDE = (C & 1) ? FG : FG + 16;  // odd number of 16 B units
  static constexpr size_t kWarpStage = 32u * STRIDE;
  // group copy: chunk q = 32 it + lane -> slot l = q / C, part = q % C.  (32 it) mod C cycles
  // with period NPH, so per lane the NPH (slot delta, part) offsets are precomputed once and a
  // chunk's addresses are one add each (when NPH is small enough to keep them in registers)
  static constexpr int NPH = C / cgcd(32, C);
  static constexpr bool kPhase = NPH <= 8;
  static constexpr size_t smem_stage(int warps) { return (size_t)warps * kWarpStage; }
};

__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  FS_CHK_SMEM(a, 16);
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 lds128_nv(uint32_t a) {
  uint4 v;
  FS_CHK_SMEM(a, 16);
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// Node transition with the first row's a_d, as an entry for a residue rho: the next residue,
// the increment of floor(R_L / g_{d-1}), k0 of the next residue and a_d of the next node's
// first row.  Shared-memory table (one 16 B load, issued right after the previous advance so
// its latency is off the row loop's critical path) or arithmetic.
struct RAdvSmem {
  using Ent = uint4;
  uint32_t base;  // shared-window address of the radv table
  __device__ __forceinline__ Ent load(uint32_t rho, const Consts &) const { return lds128_nv(base + rho * 16u); }
  __device__ __forceinline__ static uint32_t next(const Ent &e) { return e.x & ((1u << kAdvBits) - 1u); }
  __device__ __forceinline__ static uint32_t inc(const Ent &e) { return e.x >> kAdvBits; }
  __device__ __forceinline__ static uint32_t k0(const Ent &e) { return e.y; }
  __device__ __forceinline__ static uint32_t ad0(const Ent &e) { return e.z; }
  __device__ __forceinline__ static uint32_t steps(const Ent &e) { return e.w; }
};
struct RAdvArith {
  struct Ent {
    uint32_t nx, in, k, a, st;
  };
  // the same transition by arithmetic: advance until a live residue (at most g_{d-1} steps)
  __device__ __forceinline__ Ent load(uint32_t rho, const Consts &c) const {
    uint32_t r = rho, inc = 0, steps = 0;
    Adv w;
    do {
      w = KTabArith{}.step(r, c);
      inc += w.inc;
      ++steps;
      r = w.next;
    } while (w.k0 == kNone && steps <= c.gA);
    if (w.k0 == kNone) steps = 0xFFFFFFFFu;
    return Ent{r, inc, w.k0, divq(w.k0 * c.gA + r, c.dvB), steps};  // a: garbage when k0 = none
  }
  __device__ __forceinline__ static uint32_t next(const Ent &e) { return e.nx; }
  __device__ __forceinline__ static uint32_t inc(const Ent &e) { return e.in; }
  __device__ __forceinline__ static uint32_t k0(const Ent &e) { return e.k; }
  __device__ __forceinline__ static uint32_t ad0(const Ent &e) { return e.a; }
  __device__ __forceinline__ static uint32_t steps(const Ent &e) { return e.st; }
};

// Register copy of the constants the row step and ascend() read.  They are staged through
// shared memory and read back once: ptxas would otherwise re-load a kernel parameter (LDCU)
// at every use inside the row loop (it sees through register moves and shuffles).
template <int D>
struct RegC {
  static constexpr int LA = Lane<D>::LA;
  uint32_t g[LA];
  Div dv[LA];
  uint32_t gA;
  Div dvA, dvB;
  static constexpr int kWords = 3 * LA + 5;
  // w: kWords words of shared memory; every thread calls put() then (after a barrier) get()
  __device__ __forceinline__ static void put(const Consts &c, uint32_t *w) {
    if (threadIdx.x == 0) {
      for (int j = 0; j < LA; ++j) {
        w[3 * j] = c.g[j];
        w[3 * j + 1] = c.dv[j].m;
        w[3 * j + 2] = c.dv[j].sh;
      }
      w[3 * LA] = c.gA;
      w[3 * LA + 1] = c.dvA.m;
      w[3 * LA + 2] = c.dvA.sh;
      w[3 * LA + 3] = c.dvB.m;
      w[3 * LA + 4] = c.dvB.sh;
    }
  }
  __device__ __forceinline__ void get(const uint32_t *w) {
#pragma unroll
    for (int j = 0; j < LA; ++j) {
      g[j] = w[3 * j];
      dv[j].m = w[3 * j + 1];
      dv[j].sh = w[3 * j + 2];
    }
    gA = w[3 * LA];
    dvA.m = w[3 * LA + 1];
    dvA.sh = w[3 * LA + 2];
    dvB.m = w[3 * LA + 3];
    dvB.sh = w[3 * LA + 4];
  }
};

// a_d of the current row by division (slice entry and after an ascend only)
template <int D, class CC>
__device__ __forceinline__ uint32_t rb_solve_ad(const Lane<D> &st, const CC &c) {
  return divq((st.A - (uint32_t)st.cur) * c.gA + st.rho, c.dvB);
}

// Make the lane's current row valid: while its node is exhausted, move to the next node in
// decreasing lex order (Alg. 3.1 at index L by table, or an ascend at an index < L) and
// enter it with the modulo skip.  Inside a full row slice the stream cannot end here.
// (R_L is not tracked: ascend() re-derives it from R_{L-1}.)  `wn` is the transition entry
// of the current residue; it is refreshed whenever rho changes.
template <int D, class KT, class RA, class CC>
__device__ __forceinline__ void rb_slow(Lane<D> &st, uint32_t &ad, typename RA::Ent &wn, const Consts &c,
                                        const CC &rc, const KT &kt, const RA &ra) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    if (st.cur >= 0) return;
    while (st.cur < 0) {
      if (st.a[L - 1] >= RA::steps(wn)) {  // to the next live node (NEXT-3 skip of dead ones)
        st.a[L - 1] -= RA::steps(wn);
        st.rho = RA::next(wn);
        st.A += RA::inc(wn);
        st.cur = (int32_t)st.A - (int32_t)RA::k0(wn);
        ad = RA::ad0(wn);
      } else {  // the rest of the run is dead (or empty): ascend
        st.lsum -= st.a[L - 1];
        st.a[L - 1] = 0u;
        if (!ascend<D>(st, rc)) {  // end of stream: impossible inside a full slice
          st.cur = 0x3fffffff;
          break;
        }
        st.cur = (int32_t)st.A - (int32_t)kt(st.rho, c);
        ad = rb_solve_ad<D>(st, rc);
      }
      wn = ra.load(st.rho, c);
    }
  }
}

// The common case branch-free: a lane whose node is exhausted and whose a_L > 0 advances one
// node under a predicate, from the prefetched entry, and issues the load of the next entry;
// the rare lanes that land on a node without rows or need an ascend are finished by rb_slow()
// behind one warp vote.
template <int D, class KT, class RA, class CC>
__device__ __forceinline__ void rb_ensure_row(Lane<D> &st, uint32_t &ad, typename RA::Ent &wn, const Consts &c,
                                              const CC &rc, const KT &kt, const RA &ra) {
  constexpr int L = D - 2;
  if constexpr (L >= 1) {
    if (st.cur < 0 && st.a[L - 1] >= RA::steps(wn)) {
      st.a[L - 1] -= RA::steps(wn);
      st.rho = RA::next(wn);
      st.A += RA::inc(wn);
      st.cur = (int32_t)st.A - (int32_t)RA::k0(wn);
      ad = RA::ad0(wn);
      wn = ra.load(st.rho, c);
    }
    if (__any_sync(kFull, st.cur < 0)) rb_slow<D>(st, ad, wn, c, rc, kt, ra);
  }
}

template <int D, int B, int MODE, bool KTAB>
__global__ void __launch_bounds__(kRbBlock, 1) fs_rows_batch_kernel(const KParams P) {
  using G = RowsBatchGeom<D, B>;
  constexpr bool ANY = MODE == 1, REV = MODE == 2;
  constexpr int L = D - 2;
  extern __shared__ __align__(128) unsigned char smem[];  // (128: the same start as every kernel's dynamic array)
  const Consts &c = P.c;
  uint32_t *ktab_s = reinterpret_cast<uint32_t *>(smem);
  const uint32_t kt_words = (c.ktab_len + 3u) & ~3u;
  for (uint32_t i = threadIdx.x; i < c.ktab_len; i += blockDim.x) ktab_s[i] = c.ktab[i];
  __shared__ uint32_t kc[RegC<D>::kWords + 2];
  RegC<D>::put(c, kc);
  if (threadIdx.x == 0) {
    kc[RegC<D>::kWords] = c.s;
    kc[RegC<D>::kWords + 1] = c.t;
  }
  __syncthreads();
  RegC<D> rc;
  rc.get(kc);
  const uint32_t s = kc[RegC<D>::kWords], t = kc[RegC<D>::kWords + 1];
  unsigned char *stage = reinterpret_cast<unsigned char *>(ktab_s + kt_words);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t wstage = (uint32_t)__cvta_generic_to_shared(stage + (size_t)warp * G::kWarpStage);
  const uint32_t myslot = wstage + (uint32_t)lane * G::STRIDE;

  using KT = typename std::conditional<KTAB, KTabSmem, KTabArith>::type;
  KT kt;
  const uint32_t ktab_base = (uint32_t)__cvta_generic_to_shared(ktab_s);
  if constexpr (KTAB) {
    kt.base = ktab_base;
    kt.adv = ktab_base + 4u * c.adv_off;
  }
  using RA = typename std::conditional<KTAB, RAdvSmem, RAdvArith>::type;
  RA ra;
  if constexpr (KTAB) ra.base = ktab_base + 4u * c.radv_off;

  Lane<D> st;
#pragma unroll
  for (int j = 0; j < Lane<D>::LA; ++j) {
    st.a[j] = 0;
    st.R[j] = 0;
  }
  st.A = st.rho = 0;
  st.cur = 0;
  st.k = st.kb = 0;
  st.lsum = 0;
  uint32_t ad = 0;
  typename RA::Ent wn = ra.load(0u, c);
  const uint32_t groups = (uint32_t)(P.T / (uint64_t)G::GR);
#ifdef FS_CHECK
  const uint64_t out_bytes = (ANY ? P.rank_rows : P.unit1 - P.unit0) * (uint64_t)G::RB;  // (FS_CHECK)
#endif


  for (;;) {
    // one claim of 32 consecutive full slices per warp
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(P.queue, 32ull);
    base = __shfl_sync(kFull, base, 0);
    if (base >= P.num_slices) break;
    const uint64_t idx = base + (uint64_t)lane;
    const bool live = idx < P.num_slices;
    const uint64_t rem = P.num_slices - base;
    const uint32_t nlive = rem < 32u ? (uint32_t)rem : 32u;
    if (live) {
      // REV: slice idx = output rows [idx T, idx T + T) = canonical rows E - idx T - T ..
      const uint64_t u = REV ? P.unit1 - (idx + 1) * P.T : P.unit0 + idx * P.T;
      // (the slice-start table holds the canonical slicing, or for REV the mirrored one: its
      // full slices end at unit_end, slice idx is entry starts_rev - 1 - idx)
      const uint64_t te = REV ? P.starts_rev - 1u - idx : idx;
      const uint64_t off = (P.starts && (!REV || P.starts_rev))
                               ? start_from_table<D, true>(st, c, kt, P.starts + te * (uint64_t)starts_stride<D>(c))
                               : unrank<D, true>(st, c, kt, u);
      st.cur -= (int32_t)((uint32_t)off * s);  // row units: skip to row `off` of the node
      ad = rb_solve_ad<D>(st, c);
    } else {
      st.cur = 0x3fffffff;  // an idle lane: a node that never runs out (never flushed)
      if constexpr (L >= 1) st.a[L - 1] = 0;
    }
    wn = ra.load(st.rho, c);
    // destination of the claim: M1 -- lane l's slice starts at byte (base + l) T RB of the
    // rank's block; M2 -- one reservation of nlive * T rows for the whole claim (filled
    // completely, group by group), so the front cursor sees one atomic per claim
    unsigned char *dst0;
    if (ANY) {
      unsigned long long blk = 0;
      if (lane == 0) blk = atomicAdd(P.front, (unsigned long long)nlive * P.T);
      blk = __shfl_sync(kFull, blk, 0);
      dst0 = P.rows_out + blk * (uint64_t)G::RB;
    } else {
      dst0 = P.rows_out + base * P.T * (uint64_t)G::RB;
    }
    const uint64_t SS = P.T * (uint64_t)G::RB;  // M1: bytes per slice
    // per-lane copy offsets for the NPH phases of q = 32 it + lane (see RowsBatchGeom)
    uint32_t so[G::kPhase ? G::NPH : 1], go[G::kPhase ? G::NPH : 1];
    if constexpr (G::kPhase) {
#pragma unroll
      for (int ph = 0; ph < G::NPH; ++ph) {
        const uint32_t x = (uint32_t)((32 * ph) % G::C) + (uint32_t)lane;
        const uint32_t dl = x / (uint32_t)G::C, part = x - dl * (uint32_t)G::C;
        so[ph] = dl * G::STRIDE + 16u * part;
        go[ph] = (uint32_t)(dl * SS) + 16u * part;  // M1 (a slice is far below 4 GB)
      }
    }
    __syncwarp();
    for (uint32_t grp = 0; grp < groups; ++grp) {
      // M1 / increasing order with per-lane bulk copies: the previous group's copy must have
      // read the lane's slot before the slot is overwritten
      if (!ANY && kRbTma) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll 1
      for (int b = 0; b < G::NBUF; ++b) {
        uint32_t wd[G::BW];
#pragma unroll
        for (int i = 0; i < G::BW; ++i) wd[i] = 0u;  // halves are OR-ed in (REV fills odd halves first)
#pragma unroll
        for (int u = 0; u < G::NB; ++u) {
          rb_ensure_row<D>(st, ad, wn, c, rc, kt, ra);
          uint32_t v[D];
#pragma unroll
          for (int j = 0; j < L; ++j) v[j] = st.a[j];
          v[D - 2] = (uint32_t)st.cur;
          v[D - 1] = ad;
          const int us = REV ? G::NB - 1 - u : u;  // the row's slot in the batch
#pragma unroll
          for (int j = 0; j < D; ++j) {
            if (B == 32) {
              wd[us * D + j] = v[j];
            } else {
              const int h = us * D + j;
              wd[h >> 1] |= (h & 1) ? v[j] << 16 : v[j];
            }
          }
          st.cur -= (int32_t)s;
          ad += t;
        }
        const uint32_t bs = REV ? (uint32_t)(G::NBUF - 1 - b) : (uint32_t)b;  // the batch's slot
#pragma unroll
        for (int i = 0; i < G::BW / 4; ++i)
          sts128(myslot + bs * G::BB + 16u * i, wd[4 * i], wd[4 * i + 1], wd[4 * i + 2], wd[4 * i + 3]);
      }
      if (!ANY && kRbTma) {
        // M1 / increasing order: each live lane's group is ONE contiguous segment of FG bytes at
        // its slice's exact offset -- stored by the TMA engine with one bulk copy from the lane's
        // slot (cp.async.bulk, 16 B-aligned, FG a multiple of 16) instead of the warp's LDS/STG
        // copy loop; the fence orders the lane's st.shared before the async-proxy read.
        if ((uint32_t)lane < nlive) {
          unsigned char *gdst = dst0 + (uint64_t)lane * SS +
                                (REV ? (P.T - (uint64_t)(grp + 1) * G::GR) * (uint64_t)G::RB : (uint64_t)grp * G::FG);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(myslot),
                       "n"(G::FG)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        continue;
      }
      __syncwarp();
      if (G::kPhase && nlive == 32u) {  // every slot live: addresses by phase, no checks
        unsigned char *gdst = dst0 + (ANY ? (uint64_t)grp * 32u * G::FG
                                          : REV ? (P.T - (uint64_t)(grp + 1) * G::GR) * (uint64_t)G::RB
                                                : (uint64_t)grp * G::FG);
        if (ANY) gdst += 16u * (uint32_t)lane;
        // it = blk NPH + ph: slot base b = blk (32 NPH / C) + (32 ph) / C (32 NPH is a multiple
        // of C); the phase loop is unrolled, the block loop is not (loads stay few in flight)
        constexpr uint32_t kBStep = (uint32_t)(32 * G::NPH / G::C);
#pragma unroll 1
        for (uint32_t blk = 0; blk < (uint32_t)(G::C / G::NPH); ++blk) {
#pragma unroll
          for (int ph = 0; ph < G::NPH; ++ph) {
            const uint32_t b = blk * kBStep + (uint32_t)((32 * ph) / G::C);
            const uint4 v = lds128_nv(wstage + b * G::STRIDE + so[G::kPhase ? ph : 0]);
            if (ANY) {
              FS_CHK_GMEM(gdst + 512u * (blk * G::NPH + (uint32_t)ph), P.rows_out, out_bytes, 16);
              __stcs(reinterpret_cast<uint4 *>(gdst + 512u * (blk * G::NPH + (uint32_t)ph)), v);
            } else {
              FS_CHK_GMEM(gdst + b * SS + go[G::kPhase ? ph : 0], P.rows_out, out_bytes, 16);
              __stcs(reinterpret_cast<uint4 *>(gdst + b * SS + go[G::kPhase ? ph : 0]), v);
            }
          }
        }
      } else if (ANY) {
        uint4 *dst = reinterpret_cast<uint4 *>(dst0 + (uint64_t)grp * nlive * G::FG);
#pragma unroll 4
        for (int it = 0; it < G::C; ++it) {
          const uint32_t q = (uint32_t)it * 32u + (uint32_t)lane;
          const uint32_t l = q / (uint32_t)G::C, part = q - l * (uint32_t)G::C;
          if (l < nlive) {
            FS_CHK_GMEM(dst + q, P.rows_out, out_bytes, 16);
            __stcs(dst + q, lds128_nv(wstage + l * G::STRIDE + part * 16u));
          }
        }
      } else {
        // REV: group grp of slice j = output rows [jT + T - (grp+1) GR, jT + T - grp GR)
        unsigned char *dst = dst0 + (REV ? (P.T - (uint64_t)(grp + 1) * G::GR) * (uint64_t)G::RB
                                         : (uint64_t)grp * G::FG);
#pragma unroll 4
        for (int it = 0; it < G::C; ++it) {
          const uint32_t q = (uint32_t)it * 32u + (uint32_t)lane;
          const uint32_t l = q / (uint32_t)G::C, part = q - l * (uint32_t)G::C;
          if (l < nlive) {
            FS_CHK_GMEM(dst + l * SS + part * 16u, P.rows_out, out_bytes, 16);
            __stcs(reinterpret_cast<uint4 *>(dst + l * SS + part * 16u), lds128_nv(wstage + l * G::STRIDE + part * 16u));
          }
        }
      }
      __syncwarp();
    }
  }
  if (!ANY && kRbTma) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // all copies complete
}

// The rank's ragged slice: canonical rows [unit0 + first, unit0 + first + rows) (fewer than
// T), split across the threads of one CTA; each thread unranks its first row and stores its
// rows coordinate by coordinate (M1: at their canonical offsets; M2: at the back of the rank's
// block, where the back cursor grows down from rank_rows; REV: mirrored).
template <int D, int B, int MODE>
__global__ void fs_rows_tail_kernel(const KParams P, uint64_t first, uint64_t rows) {
  constexpr bool ANY = MODE == 1, REV = MODE == 2;
  const Consts &c = P.c;
  const uint64_t E = P.unit1 - P.unit0;
  const uint64_t per = (rows + blockDim.x - 1) / blockDim.x;
  const uint64_t r0 = (uint64_t)threadIdx.x * per;
  if (ANY && threadIdx.x == 0) atomicAdd(P.back, (unsigned long long)rows);
  if (r0 >= rows) return;
  const uint64_t r1 = r0 + per < rows ? r0 + per : rows;
  Lane<D> st;
  KTabArith kt;
  RAdvArith ra;
  const uint64_t u = P.unit0 + first + r0;
  const uint64_t off = unrank<D, true>(st, c, kt, u);
  st.cur -= (int32_t)((uint32_t)off * c.s);
  uint32_t ad = rb_solve_ad<D>(st, c);
  RAdvArith::Ent wn = ra.load(st.rho, c);
  const uint64_t out_row = ANY ? (P.rank_rows - rows + r0) : REV ? E - 1 - (first + r0) : (first + r0);
  unsigned char *q = P.rows_out + out_row * (uint64_t)(D * (B / 8));
  const int64_t step = REV ? -(int64_t)(D * (B / 8)) : (int64_t)(D * (B / 8));
  for (uint64_t r = r0; r < r1; ++r) {
    rb_slow<D>(st, ad, wn, c, c, kt, ra);  // per thread (threads diverge here)
    uint32_t v[D];
#pragma unroll
    for (int j = 0; j < D - 2; ++j) v[j] = st.a[j];
    v[D - 2] = (uint32_t)st.cur;
    v[D - 1] = ad;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (B == 16)
        reinterpret_cast<uint16_t *>(q)[j] = (uint16_t)v[j];
      else
        reinterpret_cast<uint32_t *>(q)[j] = v[j];
    }
    q += step;
    st.cur -= (int32_t)c.s;
    ad += c.t;
  }
}

}  // namespace fs
