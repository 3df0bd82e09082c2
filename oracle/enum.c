/*
 * oracle/enum.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU enumerator of the factorization set
 *
 *     Z(n, (g_1..g_d)) = { a in N^d : sum_i a_i g_i = n }          (Sec. 1)
 *
 * written as the definition itself: nested loops over a_1..a_{d-1}, each descending from
 * floor(R/g_k) to 0 (so rows come out in strictly decreasing lexicographic order, the
 * order of PAPER.md:97, Sec. 3.2), with a_d fixed by divisibility.  There is no
 * overshoot candidate, no modulo skip, no DP and no table: nothing here is shared with
 * the CUDA path (paper_2405_07989_b200/), and the CUDA path never includes or links it.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.
 *
 * Consumers (Sec. 2: "saving the factorizations ... incrementing a counter
 * ... setting a boolean variable based on a predicate"):
 *   count   : |Z|
 *   hist    : hist[l] = #{a in Z : sum_i a_i = l}, l = 0..hist_len-1 (length set)
 *   any     : OR over Z of pred(a); stops at the first witness (returns it)
 *   rows    : packed little-endian rows, B = 16 or 32 bits per coordinate, first `cap` rows
 *
 * Restrictions (for sampled checks at full size):
 *   prefix box: the first `plen` coordinates are fixed to prefix[0..plen-1] and coordinate
 *               plen (0-based) is restricted to [box_lo, box_hi]; plen = -1 means no box.
 *
 * Errors: returns ORC_TOO_LARGE when more than `work_ceiling` innermost iterations would
 * be needed ("oracle too large"), ORC_EINVAL on bad arguments.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_TOO_LARGE (-2)
#define ORC_FOUND 1

enum { ORC_PRED_NONE = 0, ORC_PRED_LEN_LE = 1, ORC_PRED_LEN_GE = 2, ORC_PRED_LEN_EQ = 3,
       ORC_PRED_COORD_GE = 4 };

typedef struct {
    uint64_t n;
    const uint32_t *g;
    int d;
    /* consumers */
    uint64_t count;
    uint64_t *hist;
    uint64_t hist_len;
    int pred;
    uint64_t pred_arg;
    int found;
    uint32_t *witness;
    void *rows;
    int B;
    uint64_t cap;
    /* box */
    int plen;
    const uint32_t *prefix;
    uint64_t box_lo, box_hi;
    /* work accounting */
    uint64_t work, ceiling;
    int too_large;
    uint64_t a[64];
} orc_t;

static int pred_holds(const orc_t *s) {
    uint64_t len = 0;
    for (int i = 0; i < s->d; i++) len += s->a[i];
    switch (s->pred) {
    case ORC_PRED_LEN_LE: return len <= s->pred_arg;
    case ORC_PRED_LEN_GE: return len >= s->pred_arg;
    case ORC_PRED_LEN_EQ: return len == s->pred_arg;
    case ORC_PRED_COORD_GE: {
        uint64_t i = s->pred_arg >> 32, k = s->pred_arg & 0xffffffffull;
        return i < (uint64_t)s->d && s->a[i] >= k;
    }
    default: return 0;
    }
}

/* one factorization a[0..d-1] has been found: hand it to every consumer */
static void emit(orc_t *s) {
    if (s->rows && s->count < s->cap) {
        if (s->B == 16) {
            uint8_t *p = (uint8_t *)s->rows + s->count * (uint64_t)s->d * 2;
            for (int i = 0; i < s->d; i++) {
                p[2 * i] = (uint8_t)(s->a[i] & 0xff);
                p[2 * i + 1] = (uint8_t)((s->a[i] >> 8) & 0xff);
            }
        } else {
            uint8_t *p = (uint8_t *)s->rows + s->count * (uint64_t)s->d * 4;
            for (int i = 0; i < s->d; i++)
                for (int b = 0; b < 4; b++) p[4 * i + b] = (uint8_t)((s->a[i] >> (8 * b)) & 0xff);
        }
    }
    if (s->hist) {
        uint64_t len = 0;
        for (int i = 0; i < s->d; i++) len += s->a[i];
        if (len < s->hist_len) s->hist[len] += 1;
    }
    if (s->pred != ORC_PRED_NONE && !s->found && pred_holds(s)) {
        s->found = 1;
        if (s->witness)
            for (int i = 0; i < s->d; i++) s->witness[i] = (uint32_t)s->a[i];
    }
    s->count += 1;
}

/* level k (0-based) with residual R = n - sum_{j<k} a_j g_j.  Descending loops. */
static void visit(orc_t *s, int k, uint64_t R) {
    if (s->too_large || s->found) return;
    uint64_t gk = s->g[k];
    if (k == s->d - 1) {
        /* last coordinate: fixed by divisibility */
        s->work += 1;
        if (s->work > s->ceiling) { s->too_large = 1; return; }
        if (R % gk == 0) {
            uint64_t x = R / gk;
            if (k == s->plen && (x < s->box_lo || x > s->box_hi)) return;
            if (k < s->plen && x != s->prefix[k]) return;
            s->a[k] = x;
            emit(s);
        }
        return;
    }
    uint64_t top = R / gk;
    uint64_t lo = 0;
    if (k < s->plen) {
        if (s->prefix[k] > top) return;
        top = s->prefix[k];
        lo = s->prefix[k];
    } else if (k == s->plen) {
        if (s->box_hi < top) top = s->box_hi;
        lo = s->box_lo;
        if (lo > top) return;
    }
    for (uint64_t x = top + 1; x-- > lo;) {
        s->a[k] = x;
        visit(s, k + 1, R - x * gk);
        if (s->too_large || s->found) return;
    }
}

/*
 * The single entry point.  Any consumer pointer may be NULL.  Returns ORC_OK (or
 * ORC_FOUND when a predicate witness was found), or a negative error.
 * count_out always receives the number of factorizations visited (all of Z, or of the
 * box, unless the predicate stopped the scan early).
 */
int oracle_run(uint64_t n, const uint32_t *g, int d,
               int plen, const uint32_t *prefix, uint64_t box_lo, uint64_t box_hi,
               uint64_t work_ceiling,
               uint64_t *count_out,
               uint64_t *hist, uint64_t hist_len,
               int pred, uint64_t pred_arg, int *found_out, uint32_t *witness,
               void *rows, int B, uint64_t cap) {
    if (d < 1 || d > 64 || g == NULL) return ORC_EINVAL;
    for (int i = 0; i < d; i++)
        if (g[i] == 0) return ORC_EINVAL;
    if (rows && B != 16 && B != 32) return ORC_EINVAL;
    if (plen >= d) return ORC_EINVAL;
    if (plen > 0 && prefix == NULL) return ORC_EINVAL;
    orc_t s;
    memset(&s, 0, sizeof(s));
    s.n = n; s.g = g; s.d = d;
    s.hist = hist; s.hist_len = hist_len;
    s.pred = pred; s.pred_arg = pred_arg; s.witness = witness;
    s.rows = rows; s.B = B; s.cap = cap;
    s.plen = plen; s.prefix = prefix; s.box_lo = box_lo; s.box_hi = box_hi;
    s.ceiling = work_ceiling ? work_ceiling : UINT64_MAX;
    if (hist) memset(hist, 0, hist_len * sizeof(uint64_t));
    visit(&s, 0, n);
    if (count_out) *count_out = s.count;
    if (found_out) *found_out = s.found;
    if (s.too_large) return ORC_TOO_LARGE;
    return s.found ? ORC_FOUND : ORC_OK;
}

/* ABI version of this test library */
uint64_t oracle_version(void) { return 1; }
