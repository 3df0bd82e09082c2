// fs_internal.h -- plan object and kernel launch parameters shared by the host code
// (fs_host.cu), the kernels (fs_kernels.cu) and the C ABI (fs_capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <vector>

#include "../../include/fsgpu.h"
#include "fs_core.cuh"

namespace fs {

constexpr int kBlock = 256;          // threads per persistent CTA
#ifndef FS_CC_GROUP
#define FS_CC_GROUP 16  // steps per group of the closed-tail count (cc_group)
#endif
#ifndef FS_QK
// nodes per entry of the count's state-form table (cq_group; a power of two).  C3 (r2b/r2c):
// K = 2: 9.45 ms, 4: 7.0 ms, 8: 5.0 ms (with 32-node groups)
#define FS_QK 8
#endif
#ifndef FS_CQ_GROUP
#define FS_CQ_GROUP 32  // nodes per group of the state-form count (C3: 16 -> 5.93, 32 -> 5.0, 64 -> 5.41 ms)
#endif
#ifndef FS_CC_MINB
// __launch_bounds__ min blocks per SM of the closed-tail count kernel (d <= 9).  Round 1 (pair
// table with umulhi): 5 CTAs of 256 threads (<= 48 registers) beat 4 (C3 14.7 -> 13.8 ms).  The
// state-form walk (cq_group) needs a few more registers: at 5 it spills (10.66 ms), at 4 it does
// not (9.07 ms, r2b).  Larger d keep the compiler's choice (no spills).
#define FS_CC_MINB 4
#endif
// Materialise (M1) per-lane staging: two 64 B halves + room for one row spilling past them
// (rows are <= 64 B); lane stride 196 B = 49 words (odd) so lanes at equal positions hit
// distinct shared-memory banks (measured faster than a 16 B-aligned stride with LDS.128).
constexpr uint32_t kHalf = 64;                    // flush granule: one completed half
constexpr uint32_t kStageBytes = 2 * kHalf + 64;  // 192 B usable per lane
constexpr uint32_t kLaneStride = kStageBytes + 4;
constexpr uint32_t kKtabMax = 2048;  // node tables in shared memory if g_{d-1} <= this (<= 24 KB)
constexpr uint32_t kHistSmemMax = 24576;  // u32 histogram bins kept in shared memory
constexpr uint32_t kHistRepBytes = 49152; // lane-private difference-array copies if they fit in this
#ifndef FS_HIST_REP
#define FS_HIST_REP 32  // difference-array copies per CTA (lane l uses copy l mod FS_HIST_REP)
#endif
#ifndef FS_HK
#define FS_HK 8  // advances per entry of the histogram's state-form table (hq_group)
#endif
#ifndef FS_HQ_COPIES
#define FS_HQ_COPIES 4  // interleaved copies of that table (lane l reads copy l mod FS_HQ_COPIES)
#endif
#ifndef FS_HQ_GROUP
#define FS_HQ_GROUP 16  // nodes per group of the state-form histogram (C4: 16 -> 18.8, 32 -> 19.1, 64 -> 23.4 ms)
#endif
#ifndef FS_HQ_MAX_STATES
#define FS_HQ_MAX_STATES 512  // g_{d-1} s bound for that table (48 FS_HQ_COPIES bytes per state)
#endif
#ifndef FS_M1_TABLE_MB
#define FS_M1_TABLE_MB 1024  // slice-start table cap for canonical materialise at 64-row slices
#endif
#ifndef FS_HC_MINB
#define FS_HC_MINB 1  // __launch_bounds__ min blocks per SM of the closed-tail histogram kernel (d <= 9)
#endif
constexpr int kConsRowsAny = 4;           // internal consumer: materialise, order = any (M2)
#ifndef FS_WARPBUF
#define FS_WARPBUF 6144
#endif
constexpr uint32_t kWarpBuf = FS_WARPBUF;  // M2 per-warp compaction ring (bytes)
constexpr size_t kScratchBytes = 2048;    // per-plan device scratch (queue, results, M2 cursors)
constexpr int kConsCountClosed = 5;       // internal consumer: count with the closed-form tail
constexpr int kConsHistClosed = 6;        // internal consumer: histogram with the closed-form tail
constexpr int kConsAnyClosed = 9;         // internal consumer: any-predicate with the closed-form tail
constexpr int kConsCountSkipOff = 7;      // internal consumer: count, Skip=off ablation
constexpr int kConsCountSkipPaper = 8;    // internal consumer: count, Skip=paper ablation

// Everything a kernel needs, by value (fits the 4 KB parameter space comfortably).
struct KParams {
  Consts c;
  uint64_t unit0, unit1;     // this rank's unit range (global unit indices)
  uint64_t T;                // units per slice (the last phase's, for guided slices)
  uint64_t gn0, gn1;         // uniform slices: 0, 0 (node-space phases of slice_range, unused)
  int cost_slices;           // slices from the slice-start table: L prefix words + node count
  uint64_t num_slices;
  uint64_t num_claims;       // num_slices, or the next power of two when claims are permuted
  uint32_t claim_bits;       // log2(num_claims) when permuted
  int permute;               // bit-reversed claim order (any-predicate)
  unsigned long long *queue; // work-queue head (zeroed before launch)
  // consumers
  unsigned long long *count_out;
  unsigned long long *hist_out;
  uint32_t hist_len;
  uint32_t hist_smem;        // 1: bins in shared memory
  int pred;
  uint64_t pred_arg;
  int *found;
  uint32_t *witness;
  unsigned char *rows_out;
  uint32_t row_bytes;
  // M2 (order = any): front cursor (rows, grows up in 8-row blocks) and back cursor (rows,
  // grows down from rank_rows for each warp's final < 8 rows); must meet exactly.
  unsigned long long *front;
  unsigned long long *back;
  uint64_t rank_rows;
  // closed-tail histogram: strided difference array (hist_len + dstride entries, signed
  // values stored as two's-complement u64), resolved by the finalize kernel
  unsigned long long *diff_out;
  uint32_t diff_len;
  uint32_t hist_rep;  // closed-tail histogram: 32 = one difference-array copy per lane (bank-private), else 1
  uint32_t hist_hq;   // closed-tail histogram in state form (Consts::hq_off, hist_rep = FS_HIST_REP)
  uint32_t diff_slen; // shared difference-array entries per copy (diff_len + 1, or with the state form's margins)
  uint32_t diff_sbias;// shared index of global difference index 0 (0, or Consts::hq_bias)
  // node-unit plans: the prefix a_1..a_L of every slice's first node (num_slices x L words,
  // built once per plan by fs_build_slice_starts), so a refill is L independent loads instead
  // of the unrank's O(L log n) dependent ones; nullptr = unrank
  // filtered materialise (M2 staged kernel): only rows satisfying
  // filt_pred(filt_arg) are compacted; count_only = pass 1 (count them into *front)
  int filt_pred;
  uint64_t filt_arg;
  int count_only;
  const uint32_t *starts;
  uint64_t starts_rev;  // increasing-order materialise: the table's full slices (entry nfull - 1 - idx), else 0
  // audit (debug, count consumers with the closed tail): per-slice row counts, or nullptr
  unsigned long long *slice_counts;
};

}  // namespace fs

struct fs_plan {
  uint64_t n = 0;
  int d = 0;
  int consumer = 0;
  fs_exec_t ex{};
  std::vector<uint32_t> g;        // generators as given by the caller
  std::vector<uint32_t> gi;       // generators in the internal (stream) order
  uint8_t iperm[FS_MAX_D] = {0};  // caller coordinate i is internal coordinate iperm[i]
  fs::Consts c{};                 // host copy (U/ktab point at host vectors)
  std::vector<uint64_t> U;        // L * (n+1)
  std::vector<uint32_t> ktab;     // g_{d-1} entries or empty
  uint64_t total_units = 0, total_rows = 0;
  uint64_t unit_begin = 0, unit_end = 0;
  uint64_t row_begin = 0, row_end = 0;
  uint64_t T = 1, num_slices = 0;
  uint64_t gn0 = 0, gn1 = 0;  // cost slices: S0 slices of cost 4c, S1 of 2c, then c (else 0, 0)
  std::vector<uint64_t> CW;   // cost tables (fs::cost_boundary; layout of U), node-unit plans, L >= 2
  bool cost_slices = false;   // equal-cost guided slices: prefix + node count per slice in the table
  uint64_t cost_begin = 0, cost_end = 0;  // this rank's cost range
  uint64_t *CW_dev = nullptr;
  uint64_t hist_len = 0;
  uint64_t nodes_per_level[FS_MAX_D] = {0};
  // device side
  int device = -1;
  cudaStream_t stream = nullptr;
  uint64_t *U_dev = nullptr;
  uint32_t *ktab_dev = nullptr;
  unsigned long long *scratch_dev = nullptr;  // [0] queue head, [1..] spare
  unsigned long long *diff_dev = nullptr;     // closed-tail histogram difference array
  uint32_t *starts_dev = nullptr;             // slice-start table, or nullptr
  bool starts_async = false;                  // starts_dev came from cudaMallocAsync (pool)
  bool uploaded = false;
  uint32_t grid = 0, block = fs::kBlock;
  int last_launches = 0;
};

// host helpers (fs_host.cu)
uint64_t fs_host_cost_boundary(const fs_plan *p, uint64_t target, uint32_t *pre);
int fs_validate_and_build(fs_plan *p, uint64_t n, const uint32_t *gens, int d, int consumer,
                          const fs_exec_t *ex);
int fs_plan_upload_impl(fs_plan *p);
void fs_plan_free_device(fs_plan *p);
fs::Div fs_make_div(uint32_t g);

// kernel launchers (fs_kernels.cu); return FS_OK or an error
int fs_launch(fs_plan *p, int consumer, int B, const fs::KParams &kp_template, cudaStream_t stream);
int fs_occupancy_grid(fs_plan *p, int consumer, int B, uint32_t *grid_out);
// closed-tail histogram finalize (1 or 3 launches); scratch: fs_hist_finalize_scratch() u64s
int fs_launch_hist_finalize(const fs::KParams &kp, unsigned long long *scratch, cudaStream_t stream, int *launches);
uint64_t fs_hist_finalize_scratch(uint64_t hist_len, uint32_t dstride);
// closed-tail histogram launch shape (fs_plan_hist_async, and the host model that replays it):
// global difference entries, whether the state form runs, and its shared entries per copy
struct fs_hist_shape {
  uint32_t diff_len, hist_smem, hist_rep, hq, slen, sbias;
};
fs_hist_shape fs_hist_closed_shape(const fs_plan *p);
// builds p->starts_dev on p->stream (node-unit plans with L >= 1; skipped when too large)
int fs_build_slice_starts(fs_plan *p);
extern std::atomic<unsigned long long> g_fs_total_launches;  // launches enqueued by the library (all threads)
// lockstep batch materialise kernel (fs_k_rowsb.cu)
bool fs_rows_batch_supported(const fs_plan *p, int B);
bool fs_rows_batch_shape_ok(int d);
int fs_launch_rows_reverse(unsigned char *out, uint64_t rows, uint32_t rb, cudaStream_t stream);  // some B in {16, 32} has a batch kernel for d coordinates
// mode: 0 canonical (M1), 1 order any (M2), 2 increasing lex order (mirrored M1)
int fs_dispatch_rows_batch(fs_plan *p, int B, int mode, const fs::KParams &kp, cudaStream_t s, bool query_only,
                           uint32_t *grid_out, int *launches);
