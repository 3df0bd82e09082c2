/*
 * fsgpu_debug.h -- TEST/INTROSPECTION entry points of libfsgpu.so.  Not part of the
 * product path: fs_count/fs_length_set/fs_any/fs_enumerate never call these.
 *
 * fsdbg_host_model runs the SAME per-lane successor code the kernels run
 * (csrc/fs_core.cuh: slice unranking from the DP tables, slice entry, Alg. 3.1 successor
 * with the modulo skip applied at run entry, consumers) sequentially on the host, slice by
 * slice.  It exists so that the slicing/successor logic can be checked against the oracle
 * on a machine without a GPU.  It is slow and single-threaded and is not a fallback: the
 * python package never routes a user call to it.
 */
#ifndef FSGPU_DEBUG_H
#define FSGPU_DEBUG_H

#include <stdint.h>
#include "fsgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Runs every slice of the plan (this rank's share) on the host.
 *   count_out        : rows emitted (all consumers)
 *   hist (nullable)  : uint64[hist_cap] length histogram
 *   rows (nullable)  : B-bit rows, rank block order, at most cap rows
 *   slice_counts     : uint64[num_slices] rows emitted by each slice (nullable)
 *   slice_first_row  : uint32[num_slices * d] first row (a vector) of each slice that
 *                      emitted one, else all 0xFFFFFFFF (nullable)
 * Returns FS_OK or an error. */
int fsdbg_host_model(const fs_plan *plan, uint64_t *count_out, uint64_t *hist, uint64_t hist_cap,
                     int B, void *rows, uint64_t cap, uint64_t *slice_counts, uint32_t *slice_first_row);

/* The any-predicate through the same host model (plan made for FS_CONSUMER_ANY): per row with
 * tail = FS_TAIL_ROWS, per node in closed form (the kernels' any_closed_pick) with tail =
 * FS_TAIL_CLOSED.  *found_out = 1 iff some row satisfies pred; then witness (d host uint32,
 * caller's coordinates, may be NULL) receives one such row.  pred/pred_arg as for fs_any. */
int fsdbg_host_any(const fs_plan *plan, int pred, uint64_t pred_arg, int *found_out, uint32_t *witness);

/* Host unranking: the lane state at unit `unit` (global unit index) -> the prefix vector
 * a_1..a_L, the row offset within the node (or -1 for the node-entry unit).  Returns
 * FS_OK.  prefix_out: uint32[d]. */
int fsdbg_unrank(const fs_plan *plan, uint64_t unit, uint32_t *prefix_out, int64_t *row_in_node_out);

/* The 31-bit magic division constants the kernels use for divisor g (m, sh) and the
 * quotient they produce for x (x < 2^31). */
int fsdbg_magic(uint32_t g, uint32_t *m_out, uint32_t *sh_out);
uint32_t fsdbg_magic_div(uint32_t x, uint32_t g);
/* The any-predicate's claim order (fs_core.cuh claim_slice): the slice claim idx maps to, of S
 * slices with 2^bits >= S claims; ~0 for a claim that maps to no slice. */
uint64_t fsdbg_claim_slice(uint64_t idx, uint32_t bits, uint64_t S);

/* Roofline microbenchmarks on the current device.  kind 0: IADD3 chains, 1: IMAD chains,
 * 2: 1:1 IADD3/IMAD mix, 3: LOP3 chains -> *result_out = INT32 lane-ops per clock per SM
 * (from clock64), *aux_out = Tops/s (from CUDA events).  kind 4: coalesced 16 B streaming
 * stores over `param` bytes (0 = 8 GiB) -> *result_out = GB/s (best of 5), *aux_out = bytes. */
int fsdbg_microbench(int kind, uint64_t param, double *result_out, double *aux_out);

/* Slice audit on the device (the bounds partition the lex order into
 * disjoint slices, so every factorization belongs to exactly one of them): runs the plan's
 * closed-tail count (tail = FS_TAIL_CLOSED, node-unit plan) and writes, besides the total to
 * count_dev (device uint64[1]), every slice's row count to slice_counts_dev (device
 * uint64[num_slices], zeroed first; an empty slice stays 0).  FS_EINVAL for other plans. */
int fsdbg_count_slices(fs_plan *plan, uint64_t *count_dev, uint64_t *slice_counts_dev);

/* Host computation of the plan's slicing: the first node-unit index of slice sl (uniform or
 * equal-cost slices) in *unit_out and, for d >= 3, that node's prefix a_1..a_L (stream order)
 * in prefix_out (uint32[d], may be NULL).  FS_EINVAL if sl >= num_slices. */
int fsdbg_slice_start(const fs_plan *plan, uint64_t sl, uint64_t *unit_out, uint32_t *prefix_out);

/* Device count of the launches the library made since load (all plans). */
uint64_t fsdbg_total_launches(void);

#ifdef __cplusplus
}
#endif

#endif
