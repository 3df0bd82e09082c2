/*
 * fsgpu.h -- C ABI of libfsgpu.so: parallel bounded lexicographic enumeration of the
 * factorization set on NVIDIA B200 (sm_100a).
 *
 * The problem (Sec. 1):
 *
 *     Z(n, (g_1..g_d)) = { (a_1..a_d) in N^d : a_1 g_1 + ... + a_d g_d = n }
 *
 * for any positive generators g_i, "regardless of order, setwise coprimality, or
 * minimality, including outright repeated generators" (footnote 1).
 * Generators are used AS GIVEN: no sorting, dedup or gcd reduction; coordinate i of every
 * output row belongs to gens[i].
 *
 * The stream consumers are those of PAPER.md:55 (Sec. 2): counting the results, a
 * boolean predicate over the results, and saving the results; plus the length histogram
 * (length of a = sum_i a_i) named by BASELINE.json's north_star.
 *
 * Canonical order: strictly DECREASING lexicographic order in the user's coordinate order
 * ("We compute candidates in lexicographic decreasing order").
 *
 * Execution: every entry point runs on the GPU (one successor stream per thread over
 * disjoint, DP-sized lexicographic slices).  There is no CPU fallback: with
 * no usable CUDA device the calls return FS_ENODEV.
 *
 * Ownership: `gens` is read during the call only.  `*_dev` pointers are caller-allocated
 * device memory on the selected device (e.g. torch.empty(..., device="cuda").data_ptr()).
 * The library allocates only internal scratch (DP tables, a work-queue word, counters),
 * owned by an fs_plan or freed before the call returns.
 *
 * Errors (checked before any GPU work, in this order):
 *   FS_EINVAL  d < 1 or d > FS_MAX_D; gens == NULL; some g_i == 0 (Z would be infinite);
 *              B not in {16, 32}; hist_cap too small; unknown predicate or consumer;
 *              out_dev not 16-byte aligned; world < 1 or rank outside [0, world).
 *   FS_ERANGE  n + max_i g_i >= 2^31 (device arithmetic is u32 with exact 31-bit magic
 *              division); B == 16 and some floor(n/g_i) > 65535; a DP total >= 2^63;
 *              the DP tables would exceed FS_MAX_TABLE_BYTES; order=any with cap < |Z|.
 *   FS_ENODEV  no CUDA device / driver.
 *   FS_ECUDA, FS_ENOMEM  CUDA runtime failure / device allocation failure.
 * Negative return values are these codes; fs_strerror() names them.
 */
#ifndef FSGPU_H
#define FSGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_MAX_D 16
#define FS_MAX_TABLE_BYTES (8ull << 30)

enum {
    FS_OK = 0,
    FS_EINVAL = -1,
    FS_ERANGE = -2,
    FS_ECUDA = -3,
    FS_ENOMEM = -4,
    FS_ENODEV = -5
};

/* any-predicates ("a boolean variable based on a predicate's value").
 * LEN_* compare the length l(a) = sum_i a_i with pred_arg; COORD_GE tests
 * a_i >= k with pred_arg = (i << 32) | k, i 0-based. */
enum {
    FS_PRED_LEN_LE = 1,
    FS_PRED_LEN_GE = 2,
    FS_PRED_LEN_EQ = 3,
    FS_PRED_COORD_GE = 4
};

/* consumers: what a plan's kernel does with each factorization */
enum {
    FS_CONSUMER_COUNT = 0,
    FS_CONSUMER_HIST = 1,
    FS_CONSUMER_ANY = 2,
    FS_CONSUMER_ROWS = 3
};

/* Execution options for the _ex variants and plans.  Zero-initialise, then set fields.
 *   device      CUDA device ordinal; -1 = the current device.
 *   cuda_stream cudaStream_t the work is ordered on; NULL = legacy default stream.
 *   rank/world  compute only rank's share of a world-way partition of the canonical lex
 *               order (contiguous, equal DP weight; PAPER.md:196-200 bounds, 230-231
 *               distributed workers).  world = 0 is treated as 1.
 *   slice_units target units per slice (0 = automatic); rows per slice for ROWS plans
 *               (rounded up to a multiple of 64).  Tests force tiny slices with it.
 *   ctas_per_sm persistent CTAs per SM (0 = occupancy maximum).
 *   order       materialise layout: FS_ORDER_CANONICAL (0, default) writes every row at its
 *               exact canonical offset; FS_ORDER_ANY (1) compacts rows per warp with
 *               warp-aggregated atomics into an arbitrary order (the same multiset of rows;
 *               requires cap >= the rank's rows, else FS_ERANGE); FS_ORDER_INCREASING (2)
 *               writes the rows in increasing lex order ("could readily be
 *               modified to proceed in increasing order"): the first cap rows of that order,
 *               and the _ex offset is the block's position in it (total - row_end).
 *   tail        count / histogram / any: FS_TAIL_ROWS (0, default) steps through every valid
 *               factorization of a node (one modulo-skip step per row); FS_TAIL_CLOSED (1)
 *               takes a node's rows at once (the closed form of the
 *               paper's suffix-set idea): the count adds floor(a* / s) + 1,
 *               the histogram adds the node's length progression l0 + j (t - s) as two
 *               difference-array updates, the any-predicate tests the progression's extreme
 *               row (or solves LEN_EQ for j).  Same result.
 *               Count-only ablations of PAPER.md Alg. 3.1's index-(d-1) loop (SURVEY 8(a)
 *               A6, E2): FS_TAIL_SKIP_OFF (2) visits every candidate a_{d-1} and tests it;
 *               FS_TAIL_SKIP_PAPER (3) adds the paper's modulo jump after a valid candidate.
 *   gen_order   FS_GENORDER_GIVEN (0, default) runs the stream over the generators in the
 *               caller's order; FS_GENORDER_AUTO (1) lets count / hist / any and order=any
 *               materialise run it over a permutation that minimises the number of nodes
 *               (largest generators first; "regardless of
 *               order").  Results are reported in the caller's coordinates (witnesses,
 *               COORD_GE predicates, row coordinates); canonical-order materialise always
 *               uses the given order.
 *   rows_impl   materialise kernel: FS_ROWS_BATCH (0, default) -- every lane emits exactly
 *               one row per step into a 16 B-aligned register batch, whole batches go to a
 *               per-lane shared-memory slot with 16 B stores and the warp copies all 32
 *               lanes' slots out with coalesced 16 B stores (row shapes whose batch is at
 *               most 112 B; others use the next kernel); FS_ROWS_STAGED (1) -- the round-1
 *               kernels (per-step emission, per-lane linear staging / per-warp ring).
 *   slicing     node-unit plans (count / hist / any) with slice_units = 0:
 *               FS_SLICES_AUTO (0) cuts the rank's range into equal-COST slices at run starts
 *               (cost = level-L nodes + a per-run weight; guided: large slices first, small
 *               ones last) when d >= 4 and the range holds many more runs than lanes, else into
 *               equal node-count slices; FS_SLICES_COST (1) / FS_SLICES_UNIFORM (2) force one
 *               of the two (tests).  Same results either way. */
typedef struct {
    int device;
    void *cuda_stream;
    int rank;
    int world;
    uint64_t slice_units;
    int ctas_per_sm;
    int order;
    int tail;
    int gen_order;
    int rows_impl;
    int slicing;
    int walk;          /* FS_WALK_*: state-form table walks where they fit (auto), or the residue
                          form (ablation: one table step per node) */
    int reserved[2];
} fs_exec_t;

enum { FS_ORDER_CANONICAL = 0, FS_ORDER_ANY = 1, FS_ORDER_INCREASING = 2 };
enum { FS_TAIL_ROWS = 0, FS_TAIL_CLOSED = 1, FS_TAIL_SKIP_OFF = 2, FS_TAIL_SKIP_PAPER = 3 };
enum { FS_GENORDER_GIVEN = 0, FS_GENORDER_AUTO = 1 };
enum { FS_ROWS_BATCH = 0, FS_ROWS_STAGED = 1 };
enum { FS_SLICES_AUTO = 0, FS_SLICES_COST = 1, FS_SLICES_UNIFORM = 2 };
enum { FS_WALK_AUTO = 0, FS_WALK_RESIDUE = 1 };

/* ---------------------------------------------------------------------------------
 * north_star entry points: current CUDA device, default stream, whole instance.
 * All are synchronous: they return after the result is available.  They pick the fastest
 * exact configuration: fs_count / fs_length_set / fs_any run the stream with
 * gen_order = FS_GENORDER_AUTO and tail = FS_TAIL_CLOSED; fs_enumerate
 * keeps the caller's generator order (it defines the canonical row order).  The _ex
 * variants run exactly the configuration their fs_exec_t asks for.
 * --------------------------------------------------------------------------------- */

/* |Z(n, gens)| into *count_out (host).  Z(n, g) = {a in N^d : sum_i a_i g_i = n} is the
 * factorization set of PAPER.md:29-31 (Sec. 1); the count is the paper's "incrementing a
 * counter" consumer of the lexicographic stream (Sec. 2), over the stream of Alg. 3.1
 * with the modulo optimisation and disjoint bounded slices (P:196-200,
 * Sec. 4).  Errors: FS_EINVAL (d < 1 or > 16, gens NULL, a g_i = 0, count_out NULL),
 * FS_ERANGE (n + max g >= 2^31, |Z| >= 2^63), FS_ECUDA / FS_ENODEV / FS_ENOMEM. */
int fs_count(uint64_t n, const uint32_t *gens, int d, uint64_t *count_out);

/* hist_dev[l] = #{a in Z : sum_i a_i = l} for l = 0 .. floor(n / min g); entries beyond
 * that up to hist_cap are zeroed.  hist_dev: device uint64[hist_cap],
 * hist_cap >= floor(n / min g) + 1 (else FS_EINVAL).  The length set of the north_star
 * ("length" = sum a_i; the paper names no length consumer -- a counter per
 * length), over the same stream and slices as fs_count.  Errors as fs_count. */
int fs_length_set(uint64_t n, const uint32_t *gens, int d, uint64_t *hist_dev, uint64_t hist_cap);

/* *found_out = 1 iff some a in Z satisfies pred; if so and witness_or_null != NULL, one
 * such a (d host uint32; WHICH witness is unspecified) is written there.  The paper's
 * "setting a boolean variable based on a predicate" consumer, with early exit: slices
 * are claimed from both ends of the lex order inward (P:196-200 slices).  pred: FS_PRED_*;
 * pred_arg: the length bound, or (i << 32) | k for a_i >= k.  Errors as fs_count, plus
 * FS_EINVAL for an unknown pred or found_out NULL. */
int fs_any(uint64_t n, const uint32_t *gens, int d, int pred, uint64_t pred_arg,
           int *found_out, uint32_t *witness_or_null);

/* Writes the first min(cap, |Z|) rows of Z in canonical (decreasing lex) order to
 * out_dev: row-major, d coordinates per row, little-endian uint16 (B = 16) or uint32
 * (B = 32), no padding (row r at byte r * d * B/8).  Returns |Z| (>= 0, snprintf
 * convention: truncation is not an error) or an FS_E* code.  out_dev must be 16-byte
 * aligned (device memory, caller-owned).  The paper's "saving the factorizations" consumer
 * (its per-thread buffers, are replaced by exact DP row offsets); the order
 * is the paper's decreasing lexicographic order.  Errors as fs_count, plus FS_EINVAL
 * for B not 16 | 32 or out_dev NULL with cap > 0, FS_ERANGE for B = 16 with a coordinate
 * above 65535. */
int64_t fs_enumerate(uint64_t n, const uint32_t *gens, int d, int B, void *out_dev, uint64_t cap);

/* ---------------------------------------------------------------------------------
 * _ex variants: explicit device/stream, and a rank's share of a world-way partition.
 * With world > 1 the outputs are the RANK'S PARTIAL results (count, histogram, any flag,
 * or its contiguous block of rows); the caller combines them (python/dist: NCCL
 * all_reduce / all_gather).  Still synchronous.
 * --------------------------------------------------------------------------------- */
int fs_count_ex(uint64_t n, const uint32_t *gens, int d, const fs_exec_t *ex, uint64_t *count_out);
int fs_length_set_ex(uint64_t n, const uint32_t *gens, int d, const fs_exec_t *ex,
                     uint64_t *hist_dev, uint64_t hist_cap);
int fs_any_ex(uint64_t n, const uint32_t *gens, int d, const fs_exec_t *ex, int pred,
              uint64_t pred_arg, int *found_out, uint32_t *witness_or_null);
/* Writes this rank's rows (its contiguous block of the canonical order, at most cap of
 * them) to out_dev; *global_row_offset_out (may be NULL) receives the canonical index of
 * the block's first row.  Returns the number of rows in the rank's block (before cap). */
int64_t fs_enumerate_ex(uint64_t n, const uint32_t *gens, int d, int B, void *out_dev,
                        uint64_t cap, const fs_exec_t *ex, uint64_t *global_row_offset_out);

/* Filtered materialise (the paper's consumers combine saving with a
 * predicate): the rows of this rank's share of Z(n, gens) that satisfy
 * pred(pred_arg) -- the fs_any predicates, COORD_GE's index in the caller's coordinates --
 * packed like fs_enumerate's rows (B = 16 | 32) but in ARBITRARY order (warp-aggregated
 * compaction, the order = any layout; sorting them gives the canonical order).  Two passes
 * over the rank's slices: the first counts the matching rows, the second writes them (only
 * if they fit).  Returns the number of matching rows m >= 0 and writes all m rows when
 * m <= cap, none otherwise; or an FS_E* code (FS_EINVAL: bad B / predicate / alignment;
 * FS_ERANGE as fs_enumerate).  out_dev: caller-owned device memory, 16-byte aligned, cap rows;
 * may be NULL when cap = 0 (count only). */
int64_t fs_enumerate_filtered_ex(uint64_t n, const uint32_t *gens, int d, int B, int pred,
                                 uint64_t pred_arg, void *out_dev, uint64_t cap,
                                 const fs_exec_t *ex);

/* ---------------------------------------------------------------------------------
 * Plans: host work (validation, constants, exact DP tables, partition) done once;
 * kernels enqueued asynchronously on ex->cuda_stream with results left in DEVICE memory,
 * so a collective (NCCL) can follow on the same stream and the launch can be captured in
 * a CUDA graph.  A plan's device scratch is reused across runs; runs on one plan must be
 * stream-ordered (one at a time).
 * --------------------------------------------------------------------------------- */
typedef struct fs_plan fs_plan;

typedef struct {
    uint64_t n;
    int d;
    int consumer;
    int level;                  /* node level L = max(d - 2, 0) */
    uint64_t total_units;       /* units of the whole instance (entries+rows, or rows) */
    uint64_t total_rows;        /* |Z(n, gens)| (from the exact DP) */
    uint64_t unit_begin, unit_end; /* this rank's unit range */
    uint64_t row_begin, row_end;   /* this rank's rows (ROWS plans; else 0,0) */
    uint64_t slice_units;
    uint64_t num_slices;
    uint64_t hist_len;          /* floor(n / min g) + 1 */
    uint32_t grid, block;       /* persistent launch shape */
    uint64_t nodes_per_level[FS_MAX_D]; /* #prefixes (a_1..a_k) with residual >= 0, k = 0..L */
    uint64_t table_bytes;
    uint32_t state_block;       /* count and histogram plans: level-L nodes per table step of the
                                   state-form walk, 0 if the plan does not use it */
    uint32_t cost_slices;       /* 1: equal-cost slices (slice-start table of two kernels) */
    uint32_t dead_levels;       /* bit q: coordinate q's subtrees are skipped when the gcd of the
                                   generators after it does not divide their residual (NEXT-3) */
} fs_plan_info_t;

int fs_plan_create(uint64_t n, const uint32_t *gens, int d, int consumer, const fs_exec_t *ex,
                   fs_plan **plan_out);
int fs_plan_info(const fs_plan *plan, fs_plan_info_t *info_out);
/* count_dev: device uint64[1], overwritten with the rank's count. */
int fs_plan_count_async(fs_plan *plan, uint64_t *count_dev);
/* hist_dev: device uint64[hist_cap], overwritten with the rank's histogram. */
int fs_plan_hist_async(fs_plan *plan, uint64_t *hist_dev, uint64_t hist_cap);
/* found_dev: device int32[1]; witness_dev: device uint32[d] or NULL. */
int fs_plan_any_async(fs_plan *plan, int pred, uint64_t pred_arg, int *found_dev, uint32_t *witness_dev);
/* writes min(cap, rank rows) rows of the rank's block to out_dev (16-byte aligned). */
int fs_plan_enumerate_async(fs_plan *plan, int B, void *out_dev, uint64_t cap);
/* ROWS plans, after fs_plan_enumerate_async: waits for the plan's stream, then checks the
 * order = any (M2) exactness invariant -- the front cursor (8-row blocks growing up) and the
 * back cursor (each warp's final < 8 rows, growing down from the rank's row count) must meet
 * exactly, so every row was written exactly once (every bound
 * factorization is saved exactly once).  FS_OK (also for other orders, and before any run),
 * FS_ECUDA if the cursors did not meet or the copy failed, FS_EINVAL for a non-ROWS plan. */
int fs_plan_rows_check(fs_plan *plan);
/* number of kernel launches the last *_async call enqueued (for launch accounting) */
int fs_plan_last_launches(const fs_plan *plan);
void fs_plan_destroy(fs_plan *plan);

const char *fs_strerror(int code);
/* library version, e.g. 10000 for 1.0.0 */
int fs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FSGPU_H */
