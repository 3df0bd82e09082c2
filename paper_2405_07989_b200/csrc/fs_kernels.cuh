// fs_kernels.cuh -- persistent sm_100a kernels: one successor stream per thread over DP-sized,
// disjoint lex slices pulled from an atomic work queue (replaces the paper's host-side
// splitWork + 1024-launch cadence), four consumers:
//   COUNT  per-lane u32 slice counters -> u64 -> warp shuffle reduction -> 1 atomic / warp
//   HIST   length histogram in shared-memory u32 bins (overflow-guarded) -> u64 global
//   ANY    predicate, CAS-published witness, bit-reversed claim order + flag polling for
//          early exit
//   ROWS   packed u16/u32 rows at exact canonical offsets: per-lane 256 B shared-memory ring,
//          completed 128 B halves copied warp-cooperatively with coalesced 16 B stores.
// All integer ALU work; no tensor cores (the path is not a dense contraction).
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/fsgpu.h"
#include "fs_core.cuh"
#include "fs_internal.h"

namespace fs {

// FS_CHECK builds (tests only; compute-sanitizer is closed on the GPU pool): every shared-memory
// table load / store / reduction of the kernels is checked against the CTA's dynamic shared
// memory and every global row store against the launch's output range; a violation traps.
#ifdef FS_CHECK
}  // namespace fs
#include <cstdio>
namespace fs {
extern __shared__ __align__(128) unsigned char fs_chk_dyn[];
__device__ __forceinline__ void fs_chk_smem(uint32_t a, uint32_t n, int line) {
  const uint32_t lo = (uint32_t)__cvta_generic_to_shared(fs_chk_dyn);
  uint32_t sz;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(sz));
  if (a < lo || a + n > lo + sz) {
    printf("FS_CHECK shared [%u, +%u) outside [%u, %u) at line %d (block %d thread %d)\n", a, n, lo, lo + sz, line,
           (int)blockIdx.x, (int)threadIdx.x);
    __trap();
  }
}
__device__ __forceinline__ void fs_chk_gmem(const void *p, const void *lo, uint64_t bytes, uint32_t n, int line) {
  const char *q = static_cast<const char *>(p), *b = static_cast<const char *>(lo);
  if (q < b || q + n > b + bytes) {
    printf("FS_CHECK global offset %lld (+%u) outside [0, %llu) at line %d\n", (long long)(q - b), n,
           (unsigned long long)bytes, line);
    __trap();
  }
}
#define FS_CHK_SMEM(a, n) fs_chk_smem((uint32_t)(a), (n), __LINE__)
#define FS_CHK_GMEM(p, lo, bytes, n) fs_chk_gmem((p), (lo), (bytes), (n), __LINE__)
#else
#define FS_CHK_SMEM(a, n) ((void)0)
#define FS_CHK_GMEM(p, lo, bytes, n) ((void)0)
#endif

// node tables in shared memory (copied once per CTA)
struct KTabSmem {
  uint32_t base;  // shared-window address of the k0 table
  uint32_t adv;   // shared-window address of the advance table (8 B aligned)
  __device__ __forceinline__ uint32_t operator()(uint32_t rho, const Consts &) const {
    uint32_t v;
    FS_CHK_SMEM(base + rho * 4u, 4);
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + rho * 4u));
    return v;
  }
  __device__ __forceinline__ Adv step(uint32_t rho, const Consts &) const {
    uint32_t w0, w1;
    FS_CHK_SMEM(adv + rho * 8u, 8);
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(adv + rho * 8u));
    return adv_unpack(w0, w1);
  }
};

constexpr unsigned kFull = 0xffffffffu;

// Slice entry from the precomputed slice-start table (stride L words for node-unit plans, L + 1
// for row-unit plans): the first node's prefix a_1..a_L (independent loads) and, for row
// units, the row offset inside the node; the residuals are re-derived -- the state unrank()
// would produce.  Returns the offset (node units: 0, the slice starts at a node's entry).
template <int D>
__device__ __forceinline__ uint32_t starts_stride(const Consts &c, int cost_slices = 0) {
  return (uint32_t)(D - 2) + (c.alpha && !cost_slices ? 0u : 1u);
}
template <int D, bool NEED_AD, class KT>
__device__ __forceinline__ uint64_t start_from_table(Lane<D> &st, const Consts &c, const KT &kt, const uint32_t *p) {
  constexpr int L = D - 2;
  uint32_t R = c.n, lsum = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const uint32_t a = __ldg(p + k);
    st.a[k] = a;
    R -= a * c.g[k];
    st.R[k] = R;
    lsum += a;
  }
  const uint32_t A = divq(R, c.dvA);
  st.A = A;
  st.rho = R - A * c.gA;
  st.lsum = lsum;
  st.k = st.kb = 0;
  entry<D, NEED_AD>(st, c, kt);
  return c.alpha ? 0u : __ldg(p + L);
}

// Equal-cost slices (KParams::cost_slices): one thread per slice finds the slice's first node
// by a cost-space unrank (fs::cost_boundary, at a run start) and stores its prefix; the second
// kernel stores each slice's node count (next start - this start) in word L.
template <int D>
__global__ void fs_slice_starts_cost_kernel(const KParams P, const uint64_t *CW, uint64_t cb, uint64_t ce,
                                            uint32_t *out, unsigned long long *ustart) {
  constexpr int L = D - 2;
  for (uint64_t sl = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; sl < P.num_slices;
       sl += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t pre[L > 0 ? L : 1];
    const uint64_t u = cost_boundary<D>(P.c, CW, cost_target(cb, ce, P.gn0, P.gn1, P.num_slices, sl), pre);
#pragma unroll
    for (int k = 0; k < L; ++k) out[sl * (L + 1) + k] = pre[k];
    ustart[sl] = u;
  }
}
template <int D>
__global__ void fs_slice_budgets_kernel(const KParams P, uint32_t *out, const unsigned long long *ustart) {
  constexpr int L = D - 2;
  for (uint64_t sl = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; sl < P.num_slices;
       sl += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = sl + 1 < P.num_slices ? ustart[sl + 1] : P.unit1;
    out[sl * (L + 1) + L] = (uint32_t)(e - ustart[sl]);
  }
}

// One thread per slice: unrank the slice's first unit and store the node prefix (plan setup).
template <int D>
__global__ void fs_slice_starts_kernel(const KParams P, uint32_t *out) {
  constexpr int L = D - 2;
  const uint32_t stride = starts_stride<D>(P.c);
  for (uint64_t sl = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; sl < P.num_slices;
       sl += (uint64_t)gridDim.x * blockDim.x) {
    Lane<D> st;
    KTabArith kt;
    uint64_t u, e;
    slice_range(P.unit0, P.unit1, P.T, P.gn0, P.gn1, sl, u, e);
    const uint64_t off = unrank<D, false>(st, P.c, kt, u);
#pragma unroll
    for (int k = 0; k < L; ++k) out[sl * stride + k] = st.a[k];
    if (!P.c.alpha) out[sl * stride + L] = (uint32_t)off;
  }
}

#ifndef FS_CC_INNER
// closed-tail count: steps between the warp's slice-refill checks (16 groups of the state form).
// Round 1 (pair form): 128 vs 64, fewer votes per node (C3 12.63 -> 12.51 ms).  Round 2 (state
// form, geometric guided slices; C3 one A/B, W = 1 / virtual W = 8 rank): 64 -> 3.87 / 0.613 ms,
// 128 -> 3.68 / 0.566, 256 -> 3.58 / 0.544, 512 -> 3.53 / 0.539, 1024 -> 3.51 / 0.550 ms.  A tiny
// instance pays a longer idle tail after its last slices (C5, 0.77 M nodes).  (A runtime bound
// instead of this constant cost the count loop 9 %.)
#define FS_CC_INNER 512
#endif
// (the count's B = 32 variant -- small or uniform slices, NEXT-3 -- checks every 128 steps: a
// lane that finishes a slice of a few hundred nodes would otherwise idle for most of 512)
#ifndef FS_HC_INNER
// closed-tail histogram, B = 16 kernel (equal-cost guided slices): steps between the warp's
// refill checks.  C4, one A/B: 64 -> 17.33 ms, 128 -> 16.90, 256 -> 16.69, 512 -> 16.60 (W = 8
// virtual rank at 256: 2.35 -> 2.25 ms); uniform-slice plans run the B = 32 kernel (64)
#define FS_HC_INNER 256
#endif
template <int CONS, int B = 16>
struct Inner {
  static constexpr int value = CONS == kConsCountClosed ? (B == 16 ? FS_CC_INNER : 128)
                               : CONS == kConsHistClosed && B == 16 ? FS_HC_INNER
                                                                    : 64;
};

// ---------------------------------------------------------------- consumers
// Per-lane row counter of the count consumers.  32 bits inside one inner-loop iteration only:
// it is folded into the lane's 64-bit total after every iteration (a per-row step adds at most
// 1 per step; a closed-tail group at most FS_CC_GROUP nodes' rows, which the plan bounds below
// 2^31, fs_host.cu; the t2/t3 ascend tables add < 2^16).  Node entries, whose rows are
// unbounded, go straight to the 64-bit total.
template <int D>
struct EmitCount {
  uint32_t n;
  __device__ __forceinline__ void cond(bool em, const Lane<D> &, const Consts &) { n += em ? 1u : 0u; }
  __device__ __forceinline__ void node(bool em, const Lane<D> &, const Consts &, uint32_t rows) {
    n += em ? rows : 0u;
  }
};

// Closed-tail histogram: a node's lengths form l_0 + j (t - s); two atomics on a strided
// difference array (shared-memory u32 with wrap-around, or global u64) replace one per row.
template <int D>
struct EmitHistClosed {
  uint32_t *diff;  // shared: this lane's copy (index i at diff[i * rep])
  unsigned long long *gdiff;
  uint32_t smem;
  uint32_t rep;    // shared copies (1, or 32 lane-private ones)
  uint32_t n;
  __device__ __forceinline__ void node(bool em, const Lane<D> &st, const Consts &c, uint32_t rows) {
    if (!em) return;
    uint32_t lo, hi, v;
    hist_diff_updates<D>(st, c, rows, lo, hi, v);
    if (smem) {
      FS_CHK_SMEM(__cvta_generic_to_shared(&diff[lo * rep]), 4);
      FS_CHK_SMEM(__cvta_generic_to_shared(&diff[hi * rep]), 4);
      atomicAdd(&diff[lo * rep], v);
      atomicAdd(&diff[hi * rep], 0u - v);
    } else {
      atomicAdd(&gdiff[lo], (unsigned long long)v);
      atomicAdd(&gdiff[hi], 0ull - (unsigned long long)v);
    }
    n += rows;
  }
};

template <int D>
struct EmitHist {
  uint32_t *bins;
  unsigned long long *gbins;
  uint32_t smem;
  uint32_t n;
  __device__ __forceinline__ void cond(bool em, const Lane<D> &st, const Consts &c) {
    if (!em) return;
    const uint32_t l = cur_lsum<D>(st) + (uint32_t)st.cur + row_ad<D>(st, c);  // length = sum_i a_i
    if (smem) {
      FS_CHK_SMEM(__cvta_generic_to_shared(&bins[l]), 4);
      atomicAdd(&bins[l], 1u);
    } else
      atomicAdd(&gbins[l], 1ull);
    ++n;
  }
};

template <int D>
__device__ __forceinline__ uint32_t coord(const Lane<D> &st, uint32_t i, uint32_t ad) {
  uint32_t v = ad;
  if (i == D - 2) v = (uint32_t)st.cur;
#pragma unroll
  for (int j = 0; j < D - 2; ++j)
    if (i == (uint32_t)j) v = cur_coord<D>(st, j);
  return v;
}

// pred(row) for the current row (a_d = ad): the fs_any predicates ("setting a boolean
// variable based on a predicate"); COORD_GE's index is the stream's internal coordinate.
template <int D>
__device__ __forceinline__ bool pred_row_holds(const Lane<D> &st, uint32_t ad, int pred, uint64_t arg) {
  const uint64_t len = (uint64_t)cur_lsum<D>(st) + (uint32_t)st.cur + ad;
  switch (pred) {
    case FS_PRED_LEN_LE: return len <= arg;
    case FS_PRED_LEN_GE: return len >= arg;
    case FS_PRED_LEN_EQ: return len == arg;
    default: {
      const uint32_t i = (uint32_t)(arg >> 32);
      return i < (uint32_t)D && coord<D>(st, i, ad) >= (uint32_t)(arg & 0xffffffffu);
    }
  }
}

template <int D>
struct EmitAny {
  int pred;
  uint64_t arg;
  int *found;
  uint32_t *wit;
  bool hit;
  __device__ __forceinline__ void cond(bool em, const Lane<D> &st, const Consts &c) {
    if (!em) return;
    const uint32_t ad = row_ad<D>(st, c);
    const bool ok = pred_row_holds<D>(st, ad, pred, arg);
    if (ok && !hit) {
      hit = true;
      if (atomicCAS(found, 0, 1) == 0 && wit) {  // caller's coordinate order
#pragma unroll
        for (int j = 0; j < D - 2; ++j) wit[c.perm[j]] = cur_coord<D>(st, j);
        wit[c.perm[D - 2]] = (uint32_t)st.cur;
        wit[c.perm[D - 1]] = ad;
      }
    }
  }
  // closed tail (fast_step_closed): the node's rows decided at once (any_closed_pick)
  __device__ __forceinline__ void node(bool em, const Lane<D> &st, const Consts &c, uint32_t rows) {
    if (!em || hit) return;
    uint32_t j;
    if (!any_closed_pick<D>(st, c, rows, pred, arg, j)) return;
    hit = true;
    if (atomicCAS(found, 0, 1) == 0 && wit) {
      const uint32_t ad = row_ad<D>(st, c);
#pragma unroll
      for (int q = 0; q < D - 2; ++q) wit[c.perm[q]] = cur_coord<D>(st, q);
      wit[c.perm[D - 2]] = (uint32_t)st.cur - j * c.s;
      wit[c.perm[D - 1]] = ad + j * c.t;
    }
  }
};

// Store one row (D coordinates, caller order) at a shared-memory address q.  B = 16: q is
// 2-byte aligned; adjacent coordinates are packed into 32-bit stores on the 4-byte-aligned
// side of the row (D/2 + 1 stores instead of D) -- shared-memory wavefronts are what bound
// the materialise kernels.  B = 32: one 32-bit store per coordinate.
template <int D, int B>
__device__ __forceinline__ void store_row(unsigned char *q, const uint32_t (&v)[D]) {
  if (B == 32) {
#pragma unroll
    for (int i = 0; i < D; ++i) *reinterpret_cast<uint32_t *>(q + 4 * i) = v[i];
  } else if ((reinterpret_cast<uintptr_t>(q) & 2u) == 0) {
#pragma unroll
    for (int i = 0; i + 1 < D; i += 2) *reinterpret_cast<uint32_t *>(q + 2 * i) = (v[i] & 0xffffu) | (v[i + 1] << 16);
    if (D & 1) *reinterpret_cast<uint16_t *>(q + 2 * (D - 1)) = (uint16_t)v[D - 1];
  } else {
    *reinterpret_cast<uint16_t *>(q) = (uint16_t)v[0];
#pragma unroll
    for (int i = 1; i + 1 < D; i += 2) *reinterpret_cast<uint32_t *>(q + 2 * i) = (v[i] & 0xffffu) | (v[i + 1] << 16);
    if (!(D & 1)) *reinterpret_cast<uint16_t *>(q + 2 * (D - 1)) = (uint16_t)v[D - 1];
  }
}

template <int D>
__device__ __forceinline__ void row_values(const Lane<D> &st, const Consts &c, uint32_t (&v)[D]) {
#pragma unroll
  for (int j = 0; j < D - 2; ++j) v[j] = cur_coord<D>(st, j);
  v[D - 2] = (uint32_t)st.cur;
  v[D - 1] = row_ad<D>(st, c);
}

// M1 (canonical order).  Rows are appended LINEARLY to the lane's staging buffer at byte w
// (w < 2 kHalf before a write, so a row never wraps and every coordinate is one STS with an
// immediate offset).  When w crosses kHalf, half 0 is complete; when it crosses 2 kHalf,
// half 1 is complete and the bytes that spilled past it are moved to the front (half 0 was
// flushed one group earlier).  Completed halves are copied by the warp to their exact
// canonical byte offsets.
template <int D, int B>
struct EmitRows {
  static constexpr uint32_t kRB = D * (B / 8);
  unsigned char *buf;
  uint32_t w;           // write position in buf
  uint64_t gpos;        // canonical byte offset of buf[0] in the output
  uint64_t slice_goff;  // byte offset of the slice in the output
  bool pend;
  uint32_t pend_soff, pend_len;
  uint64_t pend_goff;
  __device__ __forceinline__ void put(unsigned char *q, int i, uint32_t v) {
    if (B == 16)
      *reinterpret_cast<uint16_t *>(q + 2 * i) = (uint16_t)v;
    else
      *reinterpret_cast<uint32_t *>(q + 4 * i) = v;
  }
  __device__ __forceinline__ void start(uint64_t goff) {
    slice_goff = goff;
    gpos = goff;
    w = 0;
  }
  __device__ __forceinline__ void cond(bool em, const Lane<D> &st, const Consts &c) {
    if (!em) return;
    uint32_t v[D];
    row_values<D>(st, c, v);
    store_row<D, B>(buf + w, v);
    const uint32_t nw = w + kRB;
    const bool c0 = w < kHalf && nw >= kHalf;          // half 0 complete
    const bool c1 = w < 2 * kHalf && nw >= 2 * kHalf;  // half 1 complete (both, for rows > kHalf)
    if (c0 || c1) {
      pend = true;
      pend_soff = c0 ? 0u : kHalf;
      pend_len = (c0 && c1) ? 2 * kHalf : kHalf;
      pend_goff = gpos + pend_soff;
    }
    w = nw;
  }
  // after the group's flush: move the bytes that spilled past the two halves to the front
  // (a group writes at most max(kHalf, one row) bytes, so w < 2 kHalf + 64 here)
  __device__ __forceinline__ void rebase() {
    if (w >= 2 * kHalf) {
      for (uint32_t i = 2 * kHalf; i < w; i += 2)
        *reinterpret_cast<uint16_t *>(buf + (i - 2 * kHalf)) = *reinterpret_cast<const uint16_t *>(buf + i);
      gpos += 2 * kHalf;
      w -= 2 * kHalf;
    }
  }
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// M2 (order = any): warp-aggregated compaction.  Each fast step, the warp's valid rows are
// ranked with one ballot and appended contiguously to the warp's shared buffer; when the
// buffer is nearly full the warp reserves a block of 8k rows with ONE atomicAdd on the front
// cursor (8 rows keep every block 16 B aligned) and writes it with coalesced 16 B stores.
#ifndef FS_M2_TH
#define FS_M2_TH 6  // reserve when the ring holds FS_M2_TH / 8 of its capacity
#endif
// shared-memory stores/loads by 32-bit shared-window address
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  FS_CHK_SMEM(a, 2);
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  FS_CHK_SMEM(a, 4);
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  FS_CHK_SMEM(a, 16);
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  FS_CHK_SMEM(a, 2);
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
// keep a value in a register (the compiler may not re-derive it inside the loop)
__device__ __forceinline__ void pin(uint32_t &x) { asm volatile("" : "+r"(x)); }

template <int D, int B>
struct EmitCompact {
  // M2 (order = any): each warp appends its rows to a RING in shared memory (kRing bytes, a
  // whole number of 8-row blocks, so a row never straddles the wrap and every 8-row block is
  // a multiple of 16 B).  Once the ring holds FS_M2_TH/8 of its capacity the warp reserves
  // those rows (a multiple of 8) on the front cursor with one atomicAdd whose result is not
  // waited for: the warp keeps enumerating, and writes the reserved rows out (coalesced 16 B
  // streaming stores) only when the ring runs out of room, so the atomic's latency under
  // contention is hidden behind enumeration.  Each warp's final < 8 rows go to the back
  // cursor; front and back meet exactly at the rank's row count.
  static constexpr uint32_t kRB = D * (B / 8);
  static constexpr uint32_t kBlk = 8 * kRB;
  static constexpr uint32_t kRing = (kWarpBuf / kBlk) * kBlk;
  static constexpr uint32_t kCap = kRing / kRB;
  uint32_t sbuf;            // shared-window address of the warp's ring
  uint32_t head, tail;      // warp-uniform row counters: rows [head, tail) are in the ring
  uint32_t hpos, wpos;      // byte positions of rows head and tail in the ring
  uint32_t resv;            // rows reserved by the pending atomic (0: none)
  unsigned long long roff;  // lane 0: row offset returned by the pending atomic
  uint32_t poff[D];         // byte offset of internal coordinate j in the caller's row
  __device__ __forceinline__ void init(const Consts &c, const unsigned char *buf) {
    sbuf = (uint32_t)__cvta_generic_to_shared(buf);
    pin(sbuf);
    head = tail = hpos = wpos = resv = 0;
    roff = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      poff[j] = (uint32_t)c.perm[j] * (B / 8);
      pin(poff[j]);
    }
  }
  __device__ __forceinline__ uint32_t rows() const { return tail - head; }
  __device__ __forceinline__ void put(uint32_t a, uint32_t v) {
    if (B == 16)
      sts16(a, v);
    else
      sts32(a, v);
  }
  int filt_pred;        // 0: every row; else only rows satisfying this fs_any predicate (NEXT-4)
  uint64_t filt_arg;
  bool count_only;      // filtered pass 1: count the warp's matching rows, write nothing
  __device__ __forceinline__ void cond(bool em, const Lane<D> &st, const Consts &c) {
    if (filt_pred) em = em && pred_row_holds<D>(st, row_ad<D>(st, c), filt_pred, filt_arg);
    const unsigned m = __ballot_sync(kFull, em);
    if (count_only) {
      tail += (uint32_t)__popc(m);
      return;
    }
    if (em) {  // coordinates written at the caller's positions (generator order may differ)
      uint32_t pos = wpos + (uint32_t)__popc(m & lanemask_lt()) * kRB;
      if (pos >= kRing) pos -= kRing;
      const uint32_t q = sbuf + pos;
      const uint32_t ad = row_ad<D>(st, c);
      if (c.permuted) {
#pragma unroll
        for (int j = 0; j < D - 2; ++j) put(q + poff[j], cur_coord<D>(st, j));
        put(q + poff[D - 2], (uint32_t)st.cur);
        put(q + poff[D - 1], ad);
      } else if (B == 32) {
#pragma unroll
        for (int j = 0; j < D - 2; ++j) sts32(q + 4 * j, cur_coord<D>(st, j));
        sts32(q + 4 * (D - 2), (uint32_t)st.cur);
        sts32(q + 4 * (D - 1), ad);
      } else {  // u16 rows: adjacent coordinates packed into 32-bit stores
        uint32_t v[D];
#pragma unroll
        for (int j = 0; j < D - 2; ++j) v[j] = cur_coord<D>(st, j);
        v[D - 2] = (uint32_t)st.cur;
        v[D - 1] = ad;
        if ((q & 2u) == 0) {
#pragma unroll
          for (int i = 0; i + 1 < D; i += 2) sts32(q + 2 * i, (v[i] & 0xffffu) | (v[i + 1] << 16));
          if (D & 1) sts16(q + 2 * (D - 1), v[D - 1]);
        } else {
          sts16(q, v[0]);
#pragma unroll
          for (int i = 1; i + 1 < D; i += 2) sts32(q + 2 * i, (v[i] & 0xffffu) | (v[i + 1] << 16));
          if (!(D & 1)) sts16(q + 2 * (D - 1), v[D - 1]);
        }
      }
    }
    const uint32_t nr = (uint32_t)__popc(m);
    tail += nr;
    wpos += nr * kRB;
    if (wpos >= kRing) wpos -= kRing;
  }
  __device__ __forceinline__ void reserve(const KParams &P) {
    const uint32_t k = rows() & ~7u;
    if (k == 0) return;
    resv = k;
    if ((threadIdx.x & 31) == 0) roff = atomicAdd(P.front, (unsigned long long)k);
  }
  // converged: copy the reserved rows [head, head + resv) to their global offset
  __device__ __forceinline__ void write_out(const KParams &P) {
    __syncwarp();
    const unsigned long long off = __shfl_sync(kFull, roff, 0);
    const uint32_t chunks = resv * kRB / 16u;
    uint4 *dst = reinterpret_cast<uint4 *>(P.rows_out + off * kRB);
    const int lane = threadIdx.x & 31;
    for (uint32_t i = (uint32_t)lane; i < chunks; i += 32u) {
      uint32_t sp = hpos + 16u * i;
      if (sp >= kRing) sp -= kRing;
      __stcs(dst + i, lds128(sbuf + sp));
    }
    __syncwarp();
    head += resv;
    hpos += resv * kRB;
    if (hpos >= kRing) hpos -= kRing;
    resv = 0;
  }
  // converged; keeps room for `room` more rows
  __device__ __forceinline__ void flush(const KParams &P, bool final, uint32_t room = 32) {
    if (count_only) return;
    if (resv && (final || rows() + room > kCap)) write_out(P);
    if (!resv && (final || rows() >= kCap * FS_M2_TH / 8u || rows() + room > kCap)) {
      reserve(P);
      if (resv && (final || rows() + room > kCap)) write_out(P);
    }
  }
  // converged, at warp exit: the final < 8 rows go to the back cursor with plain stores
  __device__ __forceinline__ void finish(const KParams &P) {
    if (count_only) {
      if ((threadIdx.x & 31) == 0 && rows()) atomicAdd(P.front, (unsigned long long)rows());
      return;
    }
    flush(P, true);
    __syncwarp();  // the ring's last rows were written by other lanes (cond), possibly without a flush
    const uint32_t r = rows();
    if (r == 0) return;
    const int lane = threadIdx.x & 31;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(P.back, (unsigned long long)r);
    b = __shfl_sync(kFull, b, 0);
    const uint64_t pos = P.rank_rows - b - r;
    unsigned char *dst = P.rows_out + pos * kRB;
    for (uint32_t i = 2u * lane; i < r * kRB; i += 64u) {
      uint32_t sp = hpos + i;
      if (sp >= kRing) sp -= kRing;
      *reinterpret_cast<uint16_t *>(dst + i) = (uint16_t)lds16(sbuf + sp);
    }
    head = tail;
  }
};

// Warp-cooperative copy of every lane's pending staging segment (a multiple of 16 B, at most
// 2 kHalf): 8 segments per round, 4 lanes per segment, 16 B per lane per iteration.  Pending
// lanes publish their lane id at their rank in a per-warp slot table, so consumer lanes find
// the segment they copy with one shared-memory load.
__device__ __forceinline__ void warp_flush(bool &pend, uint32_t soff, uint64_t goff, uint32_t len,
                                           const unsigned char *warp_stage, unsigned char *out,
                                           unsigned char *slot) {
  const unsigned pm = __ballot_sync(kFull, pend);
  if (!pm) return;
  constexpr int kLanesPerSeg = 4, kSegs = 32 / kLanesPerSeg;
  const int lane = threadIdx.x & 31, sub = lane / kLanesPerSeg, j = lane % kLanesPerSeg;
  if (pend) slot[__popc(pm & lanemask_lt())] = (unsigned char)lane;
  __syncwarp();
  const int npend = __popc(pm);
  for (int base = 0; base < npend; base += kSegs) {
    const int seg = base + sub;
    const int src = seg < npend ? (int)slot[seg] : -1;
    const int sl = src < 0 ? 0 : src;
    const uint32_t s_soff = __shfl_sync(kFull, soff, sl);
    const uint32_t s_len = __shfl_sync(kFull, len, sl);
    const uint64_t s_goff = __shfl_sync(kFull, goff, sl);
    if (src >= 0) {  // a segment is at most 2 kHalf = 128 B: at most two 16 B chunks per lane
#pragma unroll
      for (int q = 0; q < (int)(2 * kHalf / (16u * kLanesPerSeg)); ++q) {
        const uint32_t o = (uint32_t)j * 16u + (uint32_t)q * 16u * kLanesPerSeg;
        if (o < s_len) {
          const uint32_t *r = reinterpret_cast<const uint32_t *>(warp_stage + src * kLaneStride + s_soff + o);
          uint4 v;
          v.x = r[0];
          v.y = r[1];
          v.z = r[2];
          v.w = r[3];
          __stcs(reinterpret_cast<uint4 *>(out + s_goff + o), v);
        }
      }
    }
  }
  __syncwarp();
  pend = false;
}

// ROWS: the lane's slice is complete -- the bytes [w & ~(kHalf-1), w) of its last half: the
// 16 B-aligned part goes to the warp flush, a ragged tail (only at the very end of the
// rank's block) is stored byte by byte.
template <int D, int B>
__device__ __forceinline__ void rows_slice_done(const KParams &P, EmitRows<D, B> &er, bool &fin, uint32_t &fin_soff,
                                                uint64_t &fin_goff, uint32_t &fin_len) {
  const uint32_t w = er.w;
  const uint32_t hstart = w & ~(kHalf - 1);
  const uint32_t plen = w - hstart;
  const uint32_t alen = plen & ~15u;
  for (uint32_t b = alen; b < plen; ++b) P.rows_out[er.gpos + hstart + b] = er.buf[hstart + b];
  if (alen) {
    fin = true;
    fin_soff = hstart;
    fin_goff = er.gpos + hstart;
    fin_len = alen;
  }
}

// The closed-tail node step over the live-node advance table (Consts::radv_off, built for an
// any-predicate plan when gcd(g_{d-1}, g_d) > 1: NEXT-3): one 16 B entry jumps `steps`
// advances to the next node whose residual that gcd divides (summed quotient increments, its
// k0); when fewer than `steps` advances are left (or the cycle holds no live node) the rest of
// the run has no rows and the lane goes to its ascend.
template <int D, class NodeEmit>
__device__ __forceinline__ void fast_step_closed_live(Lane<D> &st, const Consts &c, uint32_t rtab, NodeEmit &ne) {
  if (st.cur < 0 && st.k != 0u) {
    uint32_t w0, w1, w2, w3;
    FS_CHK_SMEM(rtab + 16u * st.rho, 16);
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(rtab + 16u * st.rho));
    (void)w2;
    if (w3 <= st.k) {
      st.k -= w3;
      st.rho = w0 & ((1u << kAdvBits) - 1u);
      st.A += w0 >> kAdvBits;
      st.cur = (int32_t)st.A - (int32_t)w1;
    } else {
      st.k = 0u;
    }
  }
  const bool em = st.cur >= 0;
  const uint32_t rows = divq((uint32_t)(em ? st.cur : 0), c.dvS) + 1u;
  ne.node(em, st, c, rows);
  if (em) st.cur = -1;
}


// Count with the closed tail, group form (Consts::cadv_off != 0): the entered node's rows
// are taken at once, so a group step is only "advance and count": k (= min(budget, a_L)
// at the last sync) bounds the valid steps; the others run on harmlessly (a residue stays a
// residue) and are masked out of the sum.  Per step: one LDS.64 (next entry's shared
// address + quotient increment, s - k0(next)), one add, one max, one umulhi-accumulate.
template <int D>
__device__ __forceinline__ uint32_t take_entry_rows(Lane<D> &st, const Consts &c) {
  const int32_t x = st.cur + (int32_t)c.s;
  st.cur = -1;
  return divq((uint32_t)(x > 0 ? x : 0), c.dvS);
}

template <int D, class E>
__device__ __forceinline__ void take_entry_hist(Lane<D> &st, const Consts &c, E &e) {
  const bool em = st.cur >= 0;
  const uint32_t rows = divq((uint32_t)(em ? st.cur : 0), c.dvS) + 1u;
  e.node(em, st, c, rows);
  st.cur = -1;
}

// Count: the one-level ascend (a_{L-1} -= 1, R_{L-1} += g_{L-1}, a_L = floor(R_{L-1}/g_L) and
// the entry of the new run) as one LDS.128 of the ascend table (Consts::t2_off, fs_host.cu),
// instead of two magic divisions and the k0 lookup.  t2a/q2 track r = R_{L-1} mod g_L and
// Q = floor(R_{L-1} / g_L); t2_sync re-derives them after a refill or a deeper ascend.
template <int D>
__device__ __forceinline__ bool t2_can_ascend(const Lane<D> &st) {
  if constexpr (D >= 4)
    return st.a[D - 4] > 0u;
  else
    return false;
}
template <int D, bool QFORM = false>
__device__ __forceinline__ void t2_sync(const Lane<D> &st, const Consts &c, uint32_t t2base, uint32_t &t2a,
                                        uint32_t &q2) {
  if constexpr (D >= 4) {
    constexpr int L = D - 2;
    const uint32_t R1 = st.R[L - 2];
    q2 = divq(R1, c.dv[L - 1]);
    const uint32_t r = R1 - q2 * c.g[L - 1];
    // state form (t2q): entries keyed by (r, q2 mod FS_QK)
    t2a = t2base + (QFORM ? 16u * (FS_QK * r + (q2 & (FS_QK - 1u))) : 16u * r);
  }
}
template <int D>
__device__ __forceinline__ void t2_ascend(Lane<D> &st, const Consts &c, uint32_t &t2a, uint32_t &q2,
                                          uint32_t &cnt) {
  if constexpr (D >= 4) {
    constexpr int L = D - 2;
    const uint4 w = lds128(t2a);
    t2a = w.x & ((1u << kCAdvShift) - 1u);
    q2 += w.x >> 16;
    st.a[L - 2] -= 1u;
    st.R[L - 2] += c.g[L - 2];
    st.a[L - 1] = q2;
    st.lsum = st.lsum - 1u + q2;
    st.rho = w.y & 0xffffu;
    st.A = w.y >> 16;
    st.cur = -1;  // the entry node's rows are taken here
    cnt += w.z;
  }
}

// Count: the two-level ascend (a_L = a_{L-1} = 0: a_{L-2} -= 1, re-solve a_{L-1} and a_L,
// enter the new run) as one LDS.128 of the t3 table (Consts::t3_off, fs_host.cu) instead of
// the generic ascend's rightmost-nonzero search and four magic divisions.  t3a/q3 track
// r3 = R_{L-2} mod g_{L-1} and Q3 = floor(R_{L-2} / g_{L-1}); the t2 state follows from the
// entry.  (0-based: a[L-3] is a_{L-2}.)
template <int D>
__device__ __forceinline__ bool t3_can_ascend(const Lane<D> &st) {
  if constexpr (D >= 5)
    return st.a[D - 4] == 0u && st.a[D - 5] > 0u;
  else
    return false;
}
template <int D>
__device__ __forceinline__ void t3_sync(const Lane<D> &st, const Consts &c, uint32_t t3base, uint32_t &t3a,
                                        uint32_t &q3) {
  if constexpr (D >= 5) {
    constexpr int L = D - 2;
    const uint32_t R3 = st.R[L - 3];
    q3 = divq(R3, c.dv[L - 2]);
    t3a = t3base + 16u * (R3 - q3 * c.g[L - 2]);
  }
}
template <int D, bool QFORM = false>
__device__ __forceinline__ void t3_ascend(Lane<D> &st, const Consts &c, uint32_t &t3a, uint32_t &q3, uint32_t t2base,
                                          uint32_t &t2a, uint32_t &q2, uint32_t &cnt) {
  if constexpr (D >= 5) {
    constexpr int L = D - 2;
    const uint4 w = lds128(t3a);
    t3a = w.x & ((1u << kCAdvShift) - 1u);
    q3 += w.x >> 16;
    st.a[L - 3] -= 1u;
    st.R[L - 3] += c.g[L - 3];
    st.a[L - 2] = q3;
    st.R[L - 2] = w.z >> 16;
    const uint32_t aL = w.w >> 16;
    st.a[L - 1] = aL;
    st.lsum = st.lsum - 1u + q3 + aL;
    st.rho = w.y & 0xffffu;
    st.A = w.y >> 16;
    st.cur = -1;  // the entry node's rows are taken here
    cnt += w.z & 0xffffu;
    q2 = aL;
    t2a = t2base + (QFORM ? 16u * (FS_QK * (w.w & 0xffffu) + (aL & (FS_QK - 1u))) : 16u * (w.w & 0xffffu));
  }
}

// Histogram: the one-level ascend by the same table (word 2 = a*0 of the new run's entry
// node); the entry's length progression is then taken by take_entry_hist.
template <int D>
__device__ __forceinline__ void t2_ascend_hist(Lane<D> &st, const Consts &c, uint32_t &t2a, uint32_t &q2) {
  if constexpr (D >= 4) {
    constexpr int L = D - 2;
    const uint4 w = lds128(t2a);
    t2a = w.x & ((1u << kCAdvShift) - 1u);
    q2 += w.x >> 16;
    st.a[L - 2] -= 1u;
    st.R[L - 2] += c.g[L - 2];
    st.a[L - 1] = q2;
    st.lsum = st.lsum - 1u + q2;
    st.rho = w.y & 0xffffu;
    st.A = w.y >> 16;
    st.cur = (int32_t)w.z;
  }
}

// Count, STATE form (Consts::qtab_off, fs_host.cu): between groups a lane keeps its node as a
// state sigma = (rho, A mod s) -- held as the shared address of its entry in the lane's copy of
// the state table, in st.rho -- and K times its quotient, QK = K floor(A / s), in st.A (K =
// FS_QK).  A node's rows are Q + e with e from the table, so a block of K advances costs one
// LDS.128, one predicate, one predicated add (QK + E_K) and one add (QK += K D_K): no division,
// no multiply.  enter_q converts the entered node (A, rho) to that form and takes the run's
// first r = st.k mod K advances at once (jump table), so every later K-block lies wholly inside
// the run or wholly past its end and one predicate masks it.
template <int D>
__device__ __forceinline__ void enter_q_from(Lane<D> &st, uint32_t sig128, uint32_t q, uint32_t qbase_lane,
                                             uint32_t q1base, uint32_t &cnt) {
  constexpr uint32_t K = FS_QK;
  const uint32_t r = st.k & (K - 1u);
  if (r) {
    uint32_t w0, w1;
    FS_CHK_SMEM(q1base + 8u * ((K - 1u) * (sig128 >> 7) + r - 1u), 8);
    asm("ld.shared.v2.u32 {%0, %1}, [%2];"
        : "=r"(w0), "=r"(w1)
        : "r"(q1base + 8u * ((K - 1u) * (sig128 >> 7) + r - 1u)));
    cnt += r * q + w1;
    q += w0 >> 16;
    sig128 = w0 & 0xffffu;
    st.k -= r;  // applied to a_L and the budget by the next sync_k
  }
  st.rho = qbase_lane + sig128;
  st.A = K * q;
}

template <int D>
__device__ __forceinline__ void enter_q(Lane<D> &st, const Consts &c, uint32_t qbase_lane, uint32_t q1base,
                                        uint32_t &cnt) {
  const uint32_t q = divq(st.A, c.dvS);
  enter_q_from<D>(st, 128u * (st.rho * c.s + (st.A - q * c.s)), q, qbase_lane, q1base, cnt);
}

template <int D, int G>
__device__ __forceinline__ void cq_group(Lane<D> &st, uint32_t &cnt) {
  constexpr uint32_t K = FS_QK;
  static_assert(G % K == 0, "nodes per group must be a multiple of FS_QK");
  uint32_t h = st.rho, QK = st.A;
  const uint32_t kk = st.k;  // a multiple of K (enter_q)
  uint32_t n = cnt;
#pragma unroll
  for (int v = 0; v < G / (int)K; ++v) {
    uint32_t w0, w1, w2, w3;
    FS_CHK_SMEM(h, 16);
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(h));
    (void)w3;
    h = w0;
    // n += QK + E_K for a block inside the run
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\tsetp.lt.u32 p, %1, %2;\n\tadd.u32 t, %3, %4;\n\t@p add.u32 %0, %0, t;\n\t}"
        : "+r"(n)
        : "r"(K * (uint32_t)v), "r"(kk), "r"(QK), "r"(w1));
    QK += w2;
  }
  cnt = n;
  st.rho = h;
  st.A = QK;
  st.k = kk > (uint32_t)G ? kk - (uint32_t)G : 0u;
}

// The one-level ascend in state form (Consts::t2q_off), keyed by r = R_{L-1} mod g_L and
// m = floor(R_{L-1} / g_L) mod K: the new run's first node plus the j = a_L mod K advances that
// enter_q would take, precomputed (one LDS.128).  When the slice's budget ends inside the new run
// (once per slice) the entry node is taken and enter_q runs with the budget's remainder instead.
template <int D>
__device__ __forceinline__ void t2q_ascend(Lane<D> &st, const Consts &c, uint32_t ktab_base, uint32_t t2base,
                                           uint32_t &t2a, uint32_t &q2, uint32_t &budget, uint32_t qbase_lane,
                                           uint32_t q1base, uint32_t &cnt) {
  if constexpr (D >= 4) {
    constexpr int L = D - 2;
    constexpr uint32_t K = FS_QK;
    const uint4 w = lds128(t2a);
    t2a = w.x & ((1u << kCAdvShift) - 1u);
    q2 += w.x >> 16;
    st.a[L - 2] -= 1u;
    st.R[L - 2] += c.g[L - 2];
    st.a[L - 1] = q2;
    st.cur = -1;
    budget -= 1u;  // the entry node
    sync_k<D, 1>(st, budget);
    if (st.k == q2) {
      cnt += w.z;
      st.rho = (w.y & 0xffffu) + (st.rho & (16u * 7u));  // sigma_j's entry in the lane's copy
      st.A = K * (w.y >> 16);
      st.k -= w.w;
    } else {
      const uint32_t r2 = (t2a - t2base) / (16u * K);  // R_L of the new run's first node
      const uint32_t A0 = divq(r2, c.dvA), rho0 = r2 - A0 * c.gA;
      const uint32_t q0 = divq(A0, c.dvS), a0 = A0 - q0 * c.s;
      uint32_t k0;
      FS_CHK_SMEM(ktab_base + 4u * rho0, 4);
      asm("ld.shared.u32 %0, [%1];" : "=r"(k0) : "r"(ktab_base + 4u * rho0));  // k0 table
      cnt += q0 + (a0 >= k0 ? 1u : 0u);
      enter_q_from<D>(st, 128u * (rho0 * c.s + a0), q0, qbase_lane, q1base, cnt);
    }
  }
}

template <int D, int G>
__device__ __forceinline__ void cc_group(Lane<D> &st, const Consts &c, uint32_t tab, uint32_t &cnt) {
  if constexpr (D >= 3) {
    uint32_t h = tab + 8u * st.rho;
    uint32_t A = st.A;
    const uint32_t kk = st.k;
    uint32_t n = cnt;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      uint32_t w0, w1;
      FS_CHK_SMEM(h, 8);
      asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(h));
      h = w0 & ((1u << kCAdvShift) - 1u);
      A += w0 >> kCAdvShift;
      int32_t x = (int32_t)(A + w1);
      x = x > 0 ? x : 0;
      // n += umulhi(x, ceil(2^32/s)) for the valid steps u < kk (predicated multiply-add)
      asm("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %2, %3;\n\t@p mad.hi.u32 %0, %1, %4, %0;\n\t}"
          : "+r"(n)
          : "r"((uint32_t)x), "r"((uint32_t)u), "r"(kk), "r"(c.mhi));
    }
    cnt = n;
    st.rho = (h - tab) >> 3;
    st.A = A;
    st.k = kk > (uint32_t)G ? kk - (uint32_t)G : 0u;
  }
}

// The same group over the paired table (Consts::cadv2_off): one LDS.128 per TWO nodes gives
// the link two advances ahead, both nodes' row-count numerators relative to the quotient
// before the pair, and the pair's quotient increment -- per node: half a shared load, half an
// add, one add-max, one predicated umulhi-accumulate.  (The predicated mad.hi's register moves
// run on the FMA pipe; a select-masked form with fewer instructions loads the ALU pipe, which
// is the busier one, and measured 5 % slower.)
// The paired group over the live-node table (Consts::cadv2_skip, gcd(g_{d-1}, g_d) > 1): each
// step jumps to the next live node; the validity mask compares the cumulative advance count
// (node units) with kk.
template <int D, int G>
__device__ __forceinline__ void cc_group2_skip(Lane<D> &st, const Consts &c, uint32_t tab2, uint32_t &cnt) {
  if constexpr (D >= 3) {
    uint32_t h = tab2 + 32u * (8u * st.rho + (threadIdx.x & 7u));
    uint32_t A = st.A;
    const uint32_t kk = st.k;
    uint32_t n = cnt, cum = 0;
#pragma unroll
    for (int v = 0; v < G / 2; ++v) {
      uint32_t w0, w1, w2, w3, w4, w5, w6, w7;
      FS_CHK_SMEM(h, 16);
      asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(h));
      FS_CHK_SMEM(h + 16u, 16);
      asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w4), "=r"(w5), "=r"(w6), "=r"(w7) : "r"(h + 16u));
      (void)w6;
      (void)w7;
      h = w0;
      int32_t x1 = (int32_t)(A + w1), x2 = (int32_t)(A + w2);
      x1 = x1 > 0 ? x1 : 0;
      x2 = x2 > 0 ? x2 : 0;
      A += w3;
      const uint32_t c1 = cum + w4, c2 = cum + w5;
      if (c1 <= kk) n += __umulhi((uint32_t)x1, c.mhi);
      if (c2 <= kk) n += __umulhi((uint32_t)x2, c.mhi);
      cum = c2;
    }
    cnt = n;
    st.rho = (h - tab2) >> 8;
    st.A = A;
    st.k = kk > cum ? kk - cum : 0u;
  }
}

template <int D, int G>
__device__ __forceinline__ void cc_group2(Lane<D> &st, const Consts &c, uint32_t tab2, uint32_t &cnt) {
  static_assert(G % 2 == 0, "nodes per group must be even");
  if constexpr (D >= 3) {
    uint32_t h = tab2 + 16u * (8u * st.rho + (threadIdx.x & 7u));  // the lane's copy (bank group)
    uint32_t A = st.A;
    const uint32_t kk = st.k;
    uint32_t n = cnt;
#pragma unroll
    for (int v = 0; v < G / 2; ++v) {
      uint32_t w0, w1, w2, w3;
      FS_CHK_SMEM(h, 16);
      asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(h));
      h = w0;  // the link alone (no mask): the ALU pipe is the busy one
      int32_t x1 = (int32_t)(A + w1), x2 = (int32_t)(A + w2);
      x1 = x1 > 0 ? x1 : 0;
      x2 = x2 > 0 ? x2 : 0;
      A += w3;
      asm("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %2, %3;\n\t@p mad.hi.u32 %0, %1, %4, %0;\n\t}"
          : "+r"(n)
          : "r"((uint32_t)x1), "r"((uint32_t)(2 * v)), "r"(kk), "r"(c.mhi));
      asm("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %2, %3;\n\t@p mad.hi.u32 %0, %1, %4, %0;\n\t}"
          : "+r"(n)
          : "r"((uint32_t)x2), "r"((uint32_t)(2 * v + 1)), "r"(kk), "r"(c.mhi));
    }
    cnt = n;
    st.rho = (h - tab2) >> 7;
    st.A = A;
    st.k = kk > (uint32_t)G ? kk - (uint32_t)G : 0u;
  }
}

// Length histogram with the closed tail, group form (Consts::cadv_off set for a histogram
// plan): per node one shared load gives the next entry's address, the quotient increment,
// s - k0 and ad0 - k0 (packed into one word when both fit 16 bits), so the node's first-row
// length is l0 = lsum + A + (ad0 - k0) with lsum = lsum0 - 1 - u at step u, and its lengths
// l0 + j (t - s), j < rows, are two updates of the strided difference array, done only by
// valid steps of nodes with rows (ptxas never predicates ATOMS, so this is a short branch;
// unconditional updates of rowless / masked steps measured 23 % slower: the shared atomics
// bound this kernel).  With KParams::hist_rep = 32 every lane updates its own bank-private
// copy (index i of lane l at word 32 i + l), which removed the bank conflicts (8e9 -> 7e7 on
// C4).
struct HcConsts {
  uint32_t dbase;  // shared address of this lane's copy of diff[0]
  uint32_t dstr;   // bytes between consecutive indices (4 * copies)
  uint32_t sstr;   // dstr * |t - s|: address step of one row along the length progression
};
__device__ __forceinline__ HcConsts hc_consts(const Consts &c, uint32_t diff, uint32_t rep) {
  HcConsts k;
  k.dbase = diff + (rep > 1u ? 4u * (threadIdx.x & (rep - 1u)) : 0u);
  k.dstr = 4u * rep;
  k.sstr = k.dstr * (uint32_t)(c.dl < 0 ? -c.dl : c.dl);
  return k;
}

// DLS = sign of t - s.  The node's lengths l0 + j (t - s), j < rows, as difference updates:
//   t > s: +1 at l0, -1 at l0 + rows (t - s);  t < s: -1 at l0 + (s - t), +1 at that minus
//   rows (s - t);  t = s: +rows at l0, -rows at l0 + 1.
template <int D, int G, bool PACKED, int DLS>
__device__ __forceinline__ void hc_group(Lane<D> &st, const Consts &c, uint32_t tab, const HcConsts &k,
                                         uint32_t &nrows) {
  if constexpr (D >= 3) {
    constexpr uint32_t kEnt = PACKED ? 8u : 16u;
    uint32_t h = tab + kEnt * st.rho;
    uint32_t A = st.A;
    const uint32_t kk = st.k;
    // address of index l0 is base0 + dstr * (A + w2 - u): l0 = lsum0 - 1 - u + A + (ad0 - k0)
    const uint32_t bofs = st.lsum - 1u - (PACKED ? 32768u : 0u) + (DLS < 0 ? (uint32_t)(-c.dl) : 0u);
    const uint32_t base0 = k.dbase + k.dstr * bofs;
    uint32_t n = nrows;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      uint32_t w0, w1, w2;
      if (PACKED) {
        uint32_t p1;
        FS_CHK_SMEM(h, 8);
        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(p1) : "r"(h));
        w1 = p1 & 0xffffu;  // s - k0 >= 1: no residue lacks a row
        w2 = p1 >> 16;      // ad0 - k0 + 2^15
      } else {
        uint32_t w3;
        FS_CHK_SMEM(h, 16);
        asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(h));
        (void)w3;
      }
      h = w0 & ((1u << kCAdvShift) - 1u);
      A += w0 >> kCAdvShift;
      const int32_t y = (int32_t)(A + w1);
      const uint32_t rows = __umulhi((uint32_t)(y > 0 ? y : 0), c.mhi);
      if ((uint32_t)u < kk && rows != 0u) {  // valid step with rows: both updates
        n += rows;
        const uint32_t a0 = base0 + k.dstr * (A + w2 - (uint32_t)u);  // l0 (t < s: l0 + s - t)
        if (DLS > 0) {
          FS_CHK_SMEM(a0, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(1u) : "memory");
          FS_CHK_SMEM(a0 + rows * k.sstr, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0 + rows * k.sstr), "r"(0xffffffffu) : "memory");
        } else if (DLS < 0) {
          FS_CHK_SMEM(a0 - rows * k.sstr, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0 - rows * k.sstr), "r"(1u) : "memory");
          FS_CHK_SMEM(a0, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(0xffffffffu) : "memory");
        } else {
          FS_CHK_SMEM(a0, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(rows) : "memory");
          FS_CHK_SMEM(a0 + k.dstr, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0 + k.dstr), "r"(0u - rows) : "memory");
        }
      }
    }
    nrows = n;
    st.rho = (h - tab) / kEnt;
    st.A = A;
    st.k = kk > (uint32_t)G ? kk - (uint32_t)G : 0u;
  }
}

// The histogram group over the 8-copy table (Consts::hadv_off): fields in separate words
// (no unpacking on the ALU pipe) and a bank-group-private copy per quarter-warp lane.
// SKIP (Consts::hadv_skip, gcd(g_{d-1}, g_d) > 1, NEXT-3): each step jumps to the next live node
// (word 1 = quotient increment | advances << 16); the cumulative advance count cum replaces
// u + 1 in the first-row length and in the validity mask.
template <int D, int G, int DLS, bool SKIP = false>
__device__ __forceinline__ void hc_group8(Lane<D> &st, const Consts &c, uint32_t tab, const HcConsts &k,
                                          uint32_t &nrows) {
  if constexpr (D >= 3) {
    uint32_t h = tab + 16u * (8u * st.rho + (threadIdx.x & 7u));
    uint32_t A = st.A;
    const uint32_t kk = st.k;
    // address of index l0 is base0 + dstr * (A + w3 - u): l0 = lsum0 - 1 - u + A + (ad0 - k0)
    const uint32_t bofs = st.lsum - 1u + (DLS < 0 ? (uint32_t)(-c.dl) : 0u);
    const uint32_t base0 = k.dbase + k.dstr * bofs;
    uint32_t n = nrows, cum = 0;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      uint32_t w0, w1, w2, w3;
      FS_CHK_SMEM(h, 16);
      asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(h));
      h = w0;
      if (SKIP) {
        A += w1 & 0xffffu;
        cum += w1 >> 16;
      } else {
        A += w1;
      }
      const int32_t y = (int32_t)(A + w2);
      const uint32_t rows = __umulhi((uint32_t)(y > 0 ? y : 0), c.mhi);
      const bool ok = SKIP ? cum <= kk : (uint32_t)u < kk;
      if (ok && rows != 0u) {  // valid step with rows: both updates
        n += rows;
        const uint32_t a0 = base0 + k.dstr * (A + w3 - (SKIP ? cum - 1u : (uint32_t)u));  // l0 (t < s: l0 + s - t)
        if (DLS > 0) {
          FS_CHK_SMEM(a0, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(1u) : "memory");
          FS_CHK_SMEM(a0 + rows * k.sstr, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0 + rows * k.sstr), "r"(0xffffffffu) : "memory");
        } else if (DLS < 0) {
          FS_CHK_SMEM(a0 - rows * k.sstr, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0 - rows * k.sstr), "r"(1u) : "memory");
          FS_CHK_SMEM(a0, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(0xffffffffu) : "memory");
        } else {
          FS_CHK_SMEM(a0, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(rows) : "memory");
          FS_CHK_SMEM(a0 + k.dstr, 4);
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0 + k.dstr), "r"(0u - rows) : "memory");
        }
      }
    }
    nrows = n;
    st.rho = (h - tab) >> 7;
    st.A = A;
    if (SKIP)
      st.k = kk > cum ? kk - cum : 0u;
    else
      st.k = kk > (uint32_t)G ? kk - (uint32_t)G : 0u;
  }
}

template <int D, int G, bool PACKED>
__device__ __forceinline__ void hc_group_dl(Lane<D> &st, const Consts &c, uint32_t tab, const HcConsts &k,
                                            uint32_t &nrows) {
  if (c.dl > 0)
    hc_group<D, G, PACKED, 1>(st, c, tab, k, nrows);
  else if (c.dl < 0)
    hc_group<D, G, PACKED, -1>(st, c, tab, k, nrows);
  else
    hc_group<D, G, PACKED, 0>(st, c, tab, k, nrows);
}

// Length histogram, STATE form (Consts::hq_off, KParams::hist_hq; table layout in fs_host.cu).
// Between groups a lane keeps its node as the shared address of its state's entry (st.rho) and
// two byte addresses in its lane-private difference-array copy, bP (st.A) and bM: node i of
// the next 8 puts +1 at bP + 128 P_i and -1 at bM + 128 M_i, with P_i / M_i signed bytes of the
// entry's second vector -- per node two byte extracts (PRMT), two scaled adds (LEA) and two
// shared reductions; no division, no multiply.  Blocks past the end of the run or slice are
// skipped (one branch per block); inside the last block a node past the end puts its -1 on its
// own +1 index (one select per node; the shared array's margins hold those indices), so no node
// needs a separate tail pass.
template <int I>
__device__ __forceinline__ void hq_node(uint32_t bP, uint32_t bM, uint32_t w, bool ok) {
  constexpr uint32_t kSelP = (2u * I) | ((2u * I + 8u) << 4) | ((2u * I + 8u) << 8) | ((2u * I + 8u) << 12);
  constexpr uint32_t kSelM = (2u * I + 1u) | ((2u * I + 9u) << 4) | ((2u * I + 9u) << 8) | ((2u * I + 9u) << 12);
  uint32_t p, m;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(p) : "r"(w), "n"(kSelP));  // sign-extended byte 2I
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(m) : "r"(w), "n"(kSelM));  // sign-extended byte 2I + 1
  const uint32_t aP = bP + (p << 7);
  const uint32_t aM = ok ? bM + (m << 7) : aP;  // a masked node: +1 and -1 on one index
  FS_CHK_SMEM(aP, 4);
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(aP), "r"(1u) : "memory");
  FS_CHK_SMEM(aM, 4);
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(aM), "r"(0xffffffffu) : "memory");
}

template <int D, int G>
__device__ __forceinline__ void hq_group(Lane<D> &st, uint32_t &h1, uint32_t &bM, uint32_t &nrows) {
  constexpr uint32_t K = FS_HK;
  static_assert(K == 8, "two 16 B vectors per entry: 8 nodes of two signed bytes");
  static_assert(4u * FS_HIST_REP == 128u, "offsets are scaled by the 32 copies' 128 B index stride");
  static_assert(G % K == 0, "nodes per group must be a multiple of FS_HK");
  uint32_t h = st.rho, hv = h1, bP = st.A, m = bM;
  const uint32_t kk = st.k;
#pragma unroll
  for (int v = 0; v < G / (int)K; ++v) {
    if (kk > K * (uint32_t)v) {
      const uint4 w0 = lds128(h), w1 = lds128(hv);
      const uint32_t b = K * (uint32_t)v;
      hq_node<0>(bP, m, w1.x, b + 0u < kk);
      hq_node<1>(bP, m, w1.x, b + 1u < kk);
      hq_node<0>(bP, m, w1.y, b + 2u < kk);
      hq_node<1>(bP, m, w1.y, b + 3u < kk);
      hq_node<0>(bP, m, w1.z, b + 4u < kk);
      hq_node<1>(bP, m, w1.z, b + 5u < kk);
      hq_node<0>(bP, m, w1.w, b + 6u < kk);
      hq_node<1>(bP, m, w1.w, b + 7u < kk);
      h = w0.x;
      hv = w0.w;
      bP += w0.y;
      m += w0.z;
    }
  }
  st.rho = h;
  h1 = hv;
  st.A = bP;
  bM = m;
  const uint32_t done = kk < (uint32_t)G ? kk : (uint32_t)G;
  st.k = kk - done;
  nrows += done;  // (dl != 0: a node changes any difference index by at most 1)
}

// A lane that has just entered a node (A, rho; its entry unit not charged to the budget) takes
// it as the NEXT node of the state walk: a_L and lsum become those of the node's virtual
// predecessor in the run (one more), so the walk's lazy counters charge the node like an
// advance; then the state sigma = (rho, A mod s), Q = floor(A / s), X = lsum + s Q and
// Y = X + Q dl as addresses in the lane's difference-array copy (dbase: shared index 0;
// length l lives at index l + hq_bias).
template <int D, int ALPHA>
__device__ __forceinline__ void enter_h(Lane<D> &st, const Consts &c, uint32_t hq_lane, uint32_t dbase,
                                        uint32_t &h1, uint32_t &bM, uint32_t &budget) {
  constexpr uint32_t STR = 4u * FS_HIST_REP;
  if constexpr (D >= 3) {
    st.a[D - 3] += 1u;
    st.lsum += 1u;
  }
  st.cur = -1;
  sync_k<D, ALPHA>(st, budget);
  const uint32_t Q = divq(st.A, c.dvS), a = st.A - Q * c.s;
  const uint32_t X = dbase + STR * (st.lsum + c.s * Q + c.hq_bias);
  const uint32_t Y = X + STR * Q * (uint32_t)c.dl;
  const uint32_t sig = st.rho * c.s + a, e0 = hq_lane + 32u * FS_HQ_COPIES * sig;
  st.rho = e0 + ((sig & 1u) ? 16u * FS_HQ_COPIES : 0u);  // vector 0 (the vectors swap on odd states)
  h1 = e0 + ((sig & 1u) ? 0u : 16u * FS_HQ_COPIES);
  st.A = c.dl > 0 ? X : Y;
  bM = c.dl > 0 ? Y : X;
}

template <int D, int CONS, int B, bool KTAB>
__global__ void __launch_bounds__(kBlock, (CONS == kConsRowsAny || CONS == FS_CONSUMER_ROWS ? 4
                                           : CONS == kConsCountClosed              ? (D <= 9 ? FS_CC_MINB : 1)
                                           : CONS == kConsHistClosed               ? (D <= 9 ? FS_HC_MINB : 1)
                                                                                   : 1))
    fs_enum_kernel(const KParams P) {
  constexpr bool CAND = CONS == kConsCountSkipOff || CONS == kConsCountSkipPaper;
  constexpr bool COUNTLIKE = CONS == FS_CONSUMER_COUNT || CONS == kConsCountClosed || CAND;
  constexpr bool NEED_AD = !COUNTLIKE;
  constexpr bool HISTLIKE = CONS == FS_CONSUMER_HIST || CONS == kConsHistClosed;
  constexpr bool ANYLIKE = CONS == FS_CONSUMER_ANY || CONS == kConsAnyClosed;
  constexpr int ALPHA = (CONS == FS_CONSUMER_ROWS || CONS == kConsRowsAny) ? 0 : 1;
  // the closed-tail consumers' NEXT-3 variant (B = 32): live-node walks when
  // gcd(g_{d-1}, g_d) > 1 and the k >= 3 dead-subtree skip in the ascend (Consts::cd_mask)
  constexpr bool N3 = B == 32 && (CONS == kConsCountClosed || CONS == kConsHistClosed || CONS == kConsAnyClosed);
  constexpr int INNER = Inner<CONS, B>::value;
  // ROWS: a lane completes at most one ring half in kHalf / row_bytes steps, so the warp
  // flushes pending halves once per that many steps.
  constexpr int kRowsPerHalf = (int)(kHalf / (D * (B / 8))) > 0 ? (int)(kHalf / (D * (B / 8))) : 1;
  constexpr int UNROLL = CONS == FS_CONSUMER_ROWS                               ? kRowsPerHalf
                         : (CONS == kConsCountClosed || CONS == kConsHistClosed) ? FS_CC_GROUP
                                                                                 : 4;
  extern __shared__ __align__(128) unsigned char smem[];  // (128: fs_host.cu qtab alignment)
  __shared__ unsigned int hist_guard;
  const Consts &c = P.c;

  uint32_t *ktab_s = reinterpret_cast<uint32_t *>(smem);
  const uint32_t kt_words = (c.ktab_len + 3u) & ~3u;
  uint32_t *hist_s = ktab_s + kt_words;
  const uint32_t hist_words =
      !(HISTLIKE && P.hist_smem) ? 0u
      : ((CONS == kConsHistClosed ? P.diff_slen * P.hist_rep : P.hist_len) + 3u) & ~3u;
  unsigned char *stage = reinterpret_cast<unsigned char *>(hist_s + hist_words);

  const uint32_t ktab_base = (uint32_t)__cvta_generic_to_shared(ktab_s);
  // count-only group table (closed tail): its link words get the table's shared address
  const bool cfast = KTAB && CONS == kConsCountClosed && c.cadv_off != 0 && ktab_base < 16384u;
  const bool hfast = KTAB && CONS == kConsHistClosed && c.cadv_off != 0 && P.hist_smem && ktab_base < 16384u;
  // count in state form (cq_group); its table ascend needs the table 128 B aligned (fs_host.cu)
  // (the state form only in the count's B = 16 kernel: its B = 32 variant walks the residue form)
  const bool qfast = B == 16 && cfast && c.qtab_off != 0 && ((ktab_base + 4u * c.qtab_off) & 127u) == 0u;
  const bool t2fast = cfast && D >= 4 && c.t2_off != 0 && (!qfast || c.t2q_off != 0);
  const bool t2h = hfast && D >= 4 && c.t2_off != 0;  // histogram: one-level ascend by table
  const bool hqf = hfast && P.hist_hq && c.hq_off != 0;  // histogram in state form (hq_group)
  const uint32_t hq_lane = ktab_base + 4u * c.hq_off + 16u * (threadIdx.x & (FS_HQ_COPIES - 1u));
  uint32_t hq_bm = 0, hq_h1 = 0;  // state form: -1 base address (bP lives in st.A), second vector's address
  const uint32_t t2base = ktab_base + 4u * (qfast ? c.t2q_off : c.t2_off);
  const uint32_t qbase_lane = ktab_base + 4u * c.qtab_off + 16u * (threadIdx.x & 7u);
  const uint32_t q1base = ktab_base + 4u * c.q1_off;
  uint32_t t2a = t2base, q2 = 0;  // count: ascend-table entry of r = R_{L-1} mod g_L, Q = R_{L-1} / g_L
  const bool t3fast = t2fast && D >= 5 && c.t3_off != 0;
  const uint32_t t3base = ktab_base + 4u * c.t3_off;
  uint32_t t3a = t3base, q3 = 0;  // count: two-level ascend entry of r3 = R_{L-2} mod g_{L-1}, Q3
  for (uint32_t i = threadIdx.x; i < c.ktab_len; i += blockDim.x) {
    uint32_t v = c.ktab[i];
    // link words (byte offsets of table entries) get the table's shared-memory base
    if ((cfast || hfast) && i >= c.cadv_off && i < c.cadv_off + c.cadv_words * c.gA &&
        (i - c.cadv_off) % c.cadv_words == 0u)
      v += ktab_base;
    if ((cfast || hfast) && c.t2_off != 0u && D >= 4 && i >= c.t2_off && i < c.t2_off + 4u * c.g[D >= 4 ? D - 3 : 0] &&
        ((i - c.t2_off) & 3u) == 0u)
      v += ktab_base;
    if (cfast && c.cadv2_off != 0u &&
        (c.cadv2_skip ? (i >= c.cadv2_off && i < c.cadv2_off + 64u * c.gA && ((i - c.cadv2_off) & 7u) == 0u)
                      : (i >= c.cadv2_off && i < c.cadv2_off + 32u * c.gA && ((i - c.cadv2_off) & 3u) == 0u)))
      v += ktab_base;
    if (hfast && c.hadv_off != 0u && i >= c.hadv_off && i < c.hadv_off + 32u * c.gA && ((i - c.hadv_off) & 3u) == 0u)
      v += ktab_base;
    if (cfast && c.t3_off != 0u && D >= 5 && i >= c.t3_off && i < c.t3_off + 4u * c.g[D >= 5 ? D - 4 : 0] &&
        ((i - c.t3_off) & 3u) == 0u)
      v += ktab_base;
    if (cfast && c.qtab_off != 0u && i >= c.qtab_off && i < c.q1_off && ((i - c.qtab_off) & 3u) == 0u) v += ktab_base;
    if (hqf && i >= c.hq_off && i < c.hq_off + 8u * FS_HQ_COPIES * c.gA * c.s) {  // link0 / link1 of vector 0
      const uint32_t r = i - c.hq_off, sig = r / (8u * FS_HQ_COPIES), slot = (r / 4u) % (2u * FS_HQ_COPIES);
      if (slot / FS_HQ_COPIES == (sig & 1u) && ((r & 3u) == 0u || (r & 3u) == 3u)) v += ktab_base;
    }
    if (cfast && c.t2q_off != 0u && D >= 4 && i >= c.t2q_off && i < c.t2q_off + 4u * FS_QK * c.g[D >= 4 ? D - 3 : 0] &&
        ((i - c.t2q_off) & 3u) == 0u)
      v += ktab_base;
    // (word 1's state field 128 sigma_j becomes the address of sigma_j's copy-0 entry: the
    // ascend adds the lane's copy offset from its current state address -- the tables fit the
    // first 64 KB, so the 16-bit field cannot carry into Q_j)
    if (cfast && c.t2q_off != 0u && c.qtab_off != 0u && D >= 4 && i >= c.t2q_off &&
        i < c.t2q_off + 4u * FS_QK * c.g[D >= 4 ? D - 3 : 0] && ((i - c.t2q_off) & 3u) == 1u)
      v += ktab_base + 4u * c.qtab_off;
    ktab_s[i] = v;
  }
  if (HISTLIKE) {
    for (uint32_t i = threadIdx.x; i < hist_words; i += blockDim.x) hist_s[i] = 0u;
    if (threadIdx.x == 0) hist_guard = 0u;
  }
  __syncthreads();

  using KT = typename std::conditional<KTAB, KTabSmem, KTabArith>::type;
  KT kt;
  if constexpr (KTAB) {
    kt.base = ktab_base;
    kt.adv = kt.base + 4u * c.adv_off;
    pin(kt.base);
    pin(kt.adv);
  }
  const int lane = threadIdx.x & 31;
  Lane<D> st;
#pragma unroll
  for (int j = 0; j < Lane<D>::LA; ++j) {
    st.a[j] = 0;
    st.R[j] = 0;
  }
  st.A = 0;
  st.rho = 0;  // keeps k0 lookups of idle lanes inside the table
  st.cur = -1;
  st.ad = 0;
  st.lsum = 0;
  st.k = st.kb = 0;
  // state form: a lane without a slice still walks the table (masked) -- start it on a valid state
  if (qfast) st.rho = qbase_lane;
  uint32_t budget = 0;
  bool alive = true;
  uint64_t acc = 0;

  EmitCount<D> e_count{0};
  EmitHist<D> e_hist{hist_s, P.hist_out, P.hist_smem, 0};
  const uint32_t hrep = CONS == kConsHistClosed && P.hist_rep > 1u ? P.hist_rep : 1u;
  // (shared index = difference index + diff_sbias: the state form's margin below index 0)
  EmitHistClosed<D> e_hcl{hist_s + P.diff_sbias * hrep + (hrep > 1u ? (threadIdx.x & (hrep - 1u)) : 0u), P.diff_out,
                          P.hist_smem, hrep, 0};
  const HcConsts hck = hc_consts(c, (uint32_t)__cvta_generic_to_shared(hist_s), hrep);
  EmitAny<D> e_any{P.pred, P.pred_arg, P.found, P.witness, false};
  EmitRows<D, B> e_rows;
  e_rows.buf = stage + threadIdx.x * kLaneStride;
  e_rows.start(0);
  e_rows.pend_len = kHalf;
  e_rows.pend = false;
  e_rows.pend_soff = 0;
  e_rows.pend_goff = 0;
  bool fin = false;
  uint32_t fin_soff = 0, fin_len = 0;
  uint64_t fin_goff = 0;
  const unsigned char *warp_stage = stage + (threadIdx.x & ~31) * kLaneStride;
  // per-warp slot table of the M1 flush, after the staging buffers
  unsigned char *wslot = stage + kBlock * kLaneStride + (threadIdx.x >> 5) * 32;
  EmitCompact<D, B> e_cmp;
  e_cmp.init(c, stage + (threadIdx.x >> 5) * kWarpBuf);
  e_cmp.filt_pred = P.filt_pred;
  e_cmp.filt_arg = P.filt_arg;
  e_cmp.count_only = P.count_only != 0;

  // slice audit (KParams::slice_counts, closed-tail count): the lane's current slice and its
  // running total at the slice's start, in shared memory (touched at refills only)
  __shared__ unsigned long long audit_s[CONS == kConsCountClosed ? 2 * kBlock : 1];
  if (CONS == kConsCountClosed && P.slice_counts) audit_s[2 * threadIdx.x] = ~0ull;
  for (;;) {
    const bool need = alive && needs_refill<D, ALPHA>(st, budget);
    const unsigned needm = __ballot_sync(kFull, need);
    if (CONS == kConsCountClosed && P.slice_counts && need) {  // the lane's slice is complete
      const unsigned long long sl0 = audit_s[2 * threadIdx.x];
      if (sl0 != ~0ull) P.slice_counts[sl0] = acc + e_count.n - audit_s[2 * threadIdx.x + 1];
    }
    if (needm) {
      const int leader = __ffs(needm) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(P.queue, (unsigned long long)__popc(needm));
      base = __shfl_sync(kFull, base, leader);
      if (need) {
        const uint64_t idx = base + (uint64_t)__popc(needm & ((1u << lane) - 1u));
        if (idx >= P.num_claims) {
          alive = false;
        } else {
          const uint64_t sl = P.permute ? claim_slice(idx, P.claim_bits, P.num_slices) : idx;
          uint64_t u = 0, e = 0;
          if (P.cost_slices) {  // equal-cost slices: node count from the slice-start table
            if (sl < P.num_slices) e = __ldg(P.starts + sl * (uint64_t)(D - 2 + 1) + (D - 2));
          } else if (sl < P.num_slices) {
            slice_range(P.unit0, P.unit1, P.T, P.gn0, P.gn1, sl, u, e);
            e -= u;
          }
          if (CONS == kConsCountClosed && P.slice_counts) {
            audit_s[2 * threadIdx.x] = e != 0 ? sl : ~0ull;
            audit_s[2 * threadIdx.x + 1] = acc + e_count.n;
          }
          if (e != 0) {  // (an empty cost slice -- two targets inside one run -- is skipped)
            budget = (uint32_t)e;
            const uint64_t off =
                P.starts ? start_from_table<D, NEED_AD>(st, c, kt, P.starts + sl * (uint64_t)starts_stride<D>(c, P.cost_slices))
                         : unrank<D, NEED_AD>(st, c, kt, u);
            budget -= position_in_node<D, NEED_AD>(st, c, off);
            if (CAND) enter_candidates<D>(st, c);
            sync_k<D, ALPHA>(st, budget);
            if (CONS == FS_CONSUMER_ROWS) e_rows.start((u - P.unit0) * (uint64_t)EmitRows<D, B>::kRB);
            if (cfast) acc += take_entry_rows<D>(st, c);
            if (qfast) t2_sync<D, true>(st, c, t2base, t2a, q2);
            else if (t2fast || t2h) t2_sync<D>(st, c, t2base, t2a, q2);
            if (t3fast) t3_sync<D>(st, c, t3base, t3a, q3);
            if (qfast) enter_q<D>(st, c, qbase_lane, q1base, e_count.n);
            if (hqf) {  // (position_in_node charged the entry unit: the walk takes it as a node)
              budget += 1u;
              enter_h<D, ALPHA>(st, c, hq_lane, hck.dbase, hq_h1, hq_bm, budget);
            } else if (hfast) {
              take_entry_hist<D>(st, c, e_hcl);
            }
          }
        }
      }
    }
    if (ANYLIKE) {
      int f = 0;
      if (lane == 0) f = *reinterpret_cast<volatile int *>(P.found);
      f = __shfl_sync(kFull, f, 0);
      if (f) {
        alive = false;
        budget = 0;
        st.cur = -1;
        st.k = st.kb = 0;
      }
    }
    if (__ballot_sync(kFull, alive) == 0) break;

#pragma unroll 1
    for (int it = 0; it < INNER; it += UNROLL) {
      const bool had = budget != 0;
      // UNROLL branch-free fast steps, then one (warp-uniform) check for lanes parked on an
      // ascend; the rare slow lanes run the generic successor step together.
      if (CONS == kConsCountClosed && B == 16 && qfast) {
        cq_group<D, FS_CQ_GROUP>(st, e_count.n);
      } else if (CONS == kConsCountClosed && B == 32 && cfast && c.cadv2_off != 0u && c.cadv2_skip &&
                 (UNROLL % 2) == 0) {
        // (the count ignores B: its B = 32 instantiation is the live-node walk, Consts::cadv2_skip,
        // so the common kernel carries none of that code)
        cc_group2_skip<D, (UNROLL % 2) == 0 ? UNROLL : 2>(st, c, ktab_base + 4u * c.cadv2_off, e_count.n);
      } else if (cfast && c.cadv2_off != 0u && (UNROLL % 2) == 0) {
        cc_group2<D, (UNROLL % 2) == 0 ? UNROLL : 2>(st, c, ktab_base + 4u * c.cadv2_off, e_count.n);
      } else if (cfast) {
        cc_group<D, UNROLL>(st, c, ktab_base + 4u * c.cadv_off, e_count.n);
      } else if (N3 && CONS == kConsAnyClosed && KTAB && c.radv_off != 0u) {  // live nodes only (NEXT-3)
        const uint32_t rt = ktab_base + 4u * c.radv_off;
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) fast_step_closed_live<D>(st, c, rt, e_any);
      } else if (CONS == kConsAnyClosed) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) fast_step_closed<D>(st, c, kt, budget, e_any);
      } else if (hqf) {
        hq_group<D, FS_HQ_GROUP>(st, hq_h1, hq_bm, e_hcl.n);
      } else if (hfast && c.hadv_off != 0u) {
        const uint32_t htab = ktab_base + 4u * c.hadv_off;
        if (N3 && c.hadv_skip) {  // (gcd(g_{d-1}, g_d) > 1 implies s < g_d, t - s of either sign)
          if (c.dl > 0)
            hc_group8<D, UNROLL, 1, true>(st, c, htab, hck, e_hcl.n);
          else if (c.dl < 0)
            hc_group8<D, UNROLL, -1, true>(st, c, htab, hck, e_hcl.n);
          else
            hc_group8<D, UNROLL, 0, true>(st, c, htab, hck, e_hcl.n);
        } else if (c.dl > 0)
          hc_group8<D, UNROLL, 1>(st, c, htab, hck, e_hcl.n);
        else if (c.dl < 0)
          hc_group8<D, UNROLL, -1>(st, c, htab, hck, e_hcl.n);
        else
          hc_group8<D, UNROLL, 0>(st, c, htab, hck, e_hcl.n);
      } else if (hfast) {
        if (c.cadv_packed)
          hc_group_dl<D, UNROLL, true>(st, c, ktab_base + 4u * c.cadv_off, hck, e_hcl.n);
        else
          hc_group_dl<D, UNROLL, false>(st, c, ktab_base + 4u * c.cadv_off, hck, e_hcl.n);
      } else {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (CONS == FS_CONSUMER_COUNT) {
          fast_step<D, NEED_AD, ALPHA>(st, c, kt, budget, e_count);
        } else if (CONS == kConsCountClosed) {
          fast_step_count_closed<D>(st, c, kt, acc);
        } else if (CONS == kConsCountSkipOff) {
          fast_step_cand<D, false>(st, c, kt, budget, e_count.n);
        } else if (CONS == kConsCountSkipPaper) {
          fast_step_cand<D, true>(st, c, kt, budget, e_count.n);
        } else if (CONS == kConsHistClosed) {
          fast_step_closed<D>(st, c, kt, budget, e_hcl);
        } else if (CONS == FS_CONSUMER_HIST) {
          fast_step<D, NEED_AD, ALPHA>(st, c, kt, budget, e_hist);
        } else if (CONS == FS_CONSUMER_ANY) {
          fast_step<D, NEED_AD, ALPHA>(st, c, kt, budget, e_any);
        } else if (CONS == kConsRowsAny) {
          fast_step<D, NEED_AD, ALPHA>(st, c, kt, budget, e_cmp);
          // per-step check only when the warp buffer cannot hold a whole group of rows
          if (EmitCompact<D, B>::kCap < 32u * UNROLL + 8u) e_cmp.flush(P, false);
        } else {
          fast_step<D, NEED_AD, ALPHA>(st, c, kt, budget, e_rows);
        }
      }
      }
      if (CONS == kConsRowsAny && EmitCompact<D, B>::kCap >= 32u * UNROLL + 8u) e_cmp.flush(P, false, 32u * UNROLL);
      if (CONS == FS_CONSUMER_ROWS) {
        if (had && budget == 0) rows_slice_done(P, e_rows, fin, fin_soff, fin_goff, fin_len);
        warp_flush(e_rows.pend, e_rows.pend_soff, e_rows.pend_goff, e_rows.pend_len, warp_stage, P.rows_out, wslot);
        warp_flush(fin, fin_soff, fin_goff, fin_len, warp_stage, P.rows_out, wslot);
        e_rows.rebase();
      }
      sync_k<D, ALPHA>(st, budget);
      const bool slow = needs_slow<D>(st, budget);
      if (__any_sync(kFull, slow)) {
        if (slow && hqf) {  // state-form histogram: the ascend, the new run's entry node is the next node
          bool ok = true;
          if (t2h && t2_can_ascend<D>(st)) {
            t2_ascend_hist<D>(st, c, t2a, q2);
          } else {
            ok = N3 ? advance_cd<D, ALPHA>(st, c, budget) : advance<D>(st, c);
            if (t2h) t2_sync<D>(st, c, t2base, t2a, q2);
          }
          if (ok)
            enter_h<D, ALPHA>(st, c, hq_lane, hck.dbase, hq_h1, hq_bm, budget);
          else
            budget = 0;  // end of stream
        } else if (slow) {
          if (t2fast && t2_can_ascend<D>(st)) {  // one-level ascend by table (count)
            if (qfast) {
              t2q_ascend<D>(st, c, ktab_base, t2base, t2a, q2, budget, qbase_lane, q1base, e_count.n);
            } else {
              t2_ascend<D>(st, c, t2a, q2, e_count.n);
              budget -= 1u;
              sync_k<D, ALPHA>(st, budget);
            }
          } else if (t2h && t2_can_ascend<D>(st)) {  // one-level ascend by table (histogram)
            t2_ascend_hist<D>(st, c, t2a, q2);
            budget -= 1u;
            sync_k<D, ALPHA>(st, budget);
          } else if (t3fast && t3_can_ascend<D>(st)) {  // two-level ascend by table (count)
            if (qfast)
              t3_ascend<D, true>(st, c, t3a, q3, t2base, t2a, q2, e_count.n);
            else
              t3_ascend<D>(st, c, t3a, q3, t2base, t2a, q2, e_count.n);
            budget -= 1u;
            sync_k<D, ALPHA>(st, budget);
            if (qfast) enter_q<D>(st, c, qbase_lane, q1base, e_count.n);
          } else {
          slow_step<D, NEED_AD, ALPHA, N3>(st, c, kt, budget);
          if (CAND) enter_candidates<D>(st, c);
          sync_k<D, ALPHA>(st, budget);
          if (cfast) acc += take_entry_rows<D>(st, c);
          if (qfast) t2_sync<D, true>(st, c, t2base, t2a, q2);
          else if (t2fast || t2h) t2_sync<D>(st, c, t2base, t2a, q2);
          if (t3fast) t3_sync<D>(st, c, t3base, t3a, q3);
          if (qfast) enter_q<D>(st, c, qbase_lane, q1base, e_count.n);
          }
          if (hfast) take_entry_hist<D>(st, c, e_hcl);
          if (CONS == FS_CONSUMER_ROWS && budget == 0) rows_slice_done(P, e_rows, fin, fin_soff, fin_goff, fin_len);
        }
        if (CONS == FS_CONSUMER_ROWS) {
          warp_flush(e_rows.pend, e_rows.pend_soff, e_rows.pend_goff, e_rows.pend_len, warp_stage, P.rows_out, wslot);
          warp_flush(fin, fin_soff, fin_goff, fin_len, warp_stage, P.rows_out, wslot);
        }
      }
      if (COUNTLIKE) {  // fold the iteration's 32-bit count into the lane's 64-bit total
        acc += e_count.n;
        e_count.n = 0;
      }
      if (HISTLIKE && P.hist_smem && (!hqf || it + UNROLL >= INNER)) {
        // overflow guard of the 32-bit shared bins / difference array: the rows added by the
        // warp this iteration (an upper bound of any bin's change) are summed per CTA, and
        // every 2^30 of them the bins are drained to global memory (as sign-extended values
        // for the difference array).  The plan bounds one iteration's rows per CTA far below
        // 2^30 (fs_capi.cu), so no bin can pass 2^31 between drains.  (State form: nodes, at
        // most 1 per index each, counted over the whole inner loop -- <= 2^15 per CTA.)
        const uint32_t mine = CONS == kConsHistClosed ? e_hcl.n : e_hist.n;
        e_hist.n = 0;
        e_hcl.n = 0;
        const uint32_t wsum = __reduce_add_sync(kFull, mine);
        if (lane == 0 && wsum) {
          const uint32_t old = atomicAdd(&hist_guard, wsum);
          if ((old >> 30) != ((old + wsum) >> 30)) {
            if (CONS == kConsHistClosed) {
              for (uint32_t i = 0; i < P.diff_len * hrep; ++i) {
                const int32_t v = (int32_t)atomicExch(&hist_s[i + P.diff_sbias * hrep], 0u);
                if (v) atomicAdd(&P.diff_out[i / hrep], (unsigned long long)(long long)v);
              }
            } else {
              for (uint32_t i = 0; i < P.hist_len; ++i) {
                const uint32_t v = atomicExch(&hist_s[i], 0u);
                if (v) atomicAdd(&P.hist_out[i], (unsigned long long)v);
              }
            }
          }
        }
      }
      if (ANYLIKE && e_any.hit) {
        budget = 0;
        st.cur = -1;
        st.k = st.kb = 0;
        alive = false;
      }
    }
  }

  // ---------------------------------------------------------------- epilogue
  if (CONS == kConsRowsAny) e_cmp.finish(P);
  if (COUNTLIKE) {
    acc += e_count.n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0 && acc) atomicAdd(P.count_out, (unsigned long long)acc);
  }
  if (CONS == FS_CONSUMER_HIST && P.hist_smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P.hist_len; i += blockDim.x) {
      const uint32_t v = hist_s[i];
      if (v) atomicAdd(&P.hist_out[i], (unsigned long long)v);
    }
  }
  if (CONS == kConsHistClosed && P.hist_smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P.diff_len; i += blockDim.x) {
      int64_t v = 0;
      for (uint32_t j = 0; j < hrep; ++j)  // lane-private copies, rotated so lanes hit distinct banks
        v += (int32_t)hist_s[(i + P.diff_sbias) * hrep + ((j + threadIdx.x) & (hrep - 1u))];
      if (v) atomicAdd(&P.diff_out[i], (unsigned long long)v);
    }
  }
}

// d = 1: Z(n,(g)) = {(n/g)} iff g | n.  One thread; the rank owning unit 0 emits it.
template <int CONS, int B>
__global__ void fs_d1_kernel(const KParams P) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (!(P.unit0 == 0 && P.unit1 > 0)) return;
  const uint32_t x = P.c.n / P.c.g[0];
  if (CONS == FS_CONSUMER_COUNT || CONS == kConsCountClosed || CONS == kConsCountSkipOff ||
      CONS == kConsCountSkipPaper)
    atomicAdd(P.count_out, 1ull);
  if (CONS == FS_CONSUMER_HIST || CONS == kConsHistClosed) atomicAdd(&P.hist_out[x], 1ull);
  if (CONS == FS_CONSUMER_ANY || CONS == kConsAnyClosed) {
    bool ok;
    switch (P.pred) {
      case FS_PRED_LEN_LE: ok = x <= P.pred_arg; break;
      case FS_PRED_LEN_GE: ok = x >= P.pred_arg; break;
      case FS_PRED_LEN_EQ: ok = x == P.pred_arg; break;
      default: ok = (P.pred_arg >> 32) == 0 && x >= (uint32_t)(P.pred_arg & 0xffffffffu);
    }
    if (ok && atomicCAS(P.found, 0, 1) == 0 && P.witness) P.witness[0] = x;
  }
  if (CONS == FS_CONSUMER_ROWS || CONS == kConsRowsAny) {
    if (CONS == kConsRowsAny) atomicAdd(P.front, 1ull);
    if (B == 16)
      *reinterpret_cast<uint16_t *>(P.rows_out) = (uint16_t)x;
    else
      *reinterpret_cast<uint32_t *>(P.rows_out) = x;
  }
}

// Closed-tail histogram: hist[l] = sum of diff[k] over k <= l, k = l mod dstride.
static __global__ void fs_hist_finalize_kernel(const unsigned long long *diff, unsigned long long *hist, uint32_t hist_len,
                                        uint32_t dstride) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < dstride && r < hist_len; r += gridDim.x * blockDim.x) {
    unsigned long long acc = 0;
    for (uint32_t l = r; l < hist_len; l += dstride) {
      acc += diff[l];
      hist[l] = acc;
    }
  }
}

static size_t smem_bytes(const KParams &kp, int consumer) {
  size_t b = (size_t)((kp.c.ktab_len + 3u) & ~3u) * 4;
  if (consumer == FS_CONSUMER_HIST && kp.hist_smem) b += (size_t)((kp.hist_len + 3u) & ~3u) * 4;
  if (consumer == kConsHistClosed && kp.hist_smem)
    b += (size_t)((kp.diff_slen * (kp.hist_rep > 1u ? kp.hist_rep : 1u) + 3u) & ~3u) * 4;
  if (consumer == FS_CONSUMER_ROWS) b += (size_t)kBlock * kLaneStride + (kBlock / 32) * 32;
  if (consumer == kConsRowsAny) b += (size_t)(kBlock / 32) * kWarpBuf;
  return b;
}

template <int D, int CONS, int B, bool KTAB>
static int launch_t(fs_plan *p, const KParams &kp, cudaStream_t stream, bool query_only, uint32_t *grid_out) {
  auto kern = fs_enum_kernel<D, CONS, B, KTAB>;
  const size_t smem = smem_bytes(kp, CONS);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return FS_ECUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem) != cudaSuccess) return FS_ECUDA;
  if (per_sm < 1) return FS_ECUDA;
  if (p->ex.ctas_per_sm > 0 && p->ex.ctas_per_sm < per_sm) per_sm = p->ex.ctas_per_sm;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) return FS_ECUDA;
  uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
  // never more CTAs than the slices can feed
  const uint64_t need_ctas = (kp.num_claims + kBlock - 1) / kBlock;
  if (grid > need_ctas) grid = need_ctas ? need_ctas : 1;
  if (grid_out) *grid_out = (uint32_t)grid;
  if (query_only) return FS_OK;
  kern<<<(unsigned)grid, kBlock, smem, stream>>>(kp);
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  return FS_OK;
}

template <int CONS, int B>
static int launch_d1(const KParams &kp, cudaStream_t stream, bool query_only, uint32_t *grid_out) {
  if (grid_out) *grid_out = 1;
  if (query_only) return FS_OK;
  fs_d1_kernel<CONS, B><<<1, 32, 0, stream>>>(kp);
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  return FS_OK;
}

template <int CONS, int B, bool KTAB>
static int dispatch_d(fs_plan *p, const KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  switch (p->d) {
    case 1: return launch_d1<CONS, B>(kp, s, q, g);
#define FS_CASE(DD) \
  case DD:          \
    return launch_t<DD, CONS, B, KTAB>(p, kp, s, q, g);
    FS_CASE(2) FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
  }
  return FS_EINVAL;
}

template <int CONS, int B>
static int dispatch_kt(fs_plan *p, const KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  return kp.c.ktab_len ? dispatch_d<CONS, B, true>(p, kp, s, q, g) : dispatch_d<CONS, B, false>(p, kp, s, q, g);
}

}  // namespace fs
