// fs_capi.cu -- the extern "C" boundary declared in include/fsgpu.h.
#include <cuda_runtime.h>

#include <vector>
#include <stdint.h>
#include <string.h>

#include <new>

#include "../../include/fsgpu.h"
#include "../../include/fsgpu_debug.h"
#include "fs_internal.h"

namespace {

// scratch layout (bytes): [0] queue u64, [8] count u64, [16] found i32, [64..128) witness,
// [1024] M2 front cursor, [1152] M2 back cursor (own 128 B lines: no contention with the queue)
constexpr size_t kOffCount = 8, kOffFound = 16, kOffWitness = 64, kOffFront = 1024, kOffBack = 1152;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (dev >= 0) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

fs::KParams base_params(const fs_plan *p) {
  fs::KParams kp;
  memset(&kp, 0, sizeof(kp));
  kp.c = p->c;
  kp.c.U = p->U_dev;
  kp.c.ktab = p->ktab_dev;
  kp.unit0 = p->unit_begin;
  kp.unit1 = p->unit_end;
  kp.T = p->T;
  kp.gn0 = p->gn0;
  kp.gn1 = p->gn1;
  kp.cost_slices = p->cost_slices ? 1 : 0;
  kp.num_slices = p->num_slices;
  kp.num_claims = p->num_slices;
  kp.queue = p->scratch_dev;
  kp.hist_len = (uint32_t)p->hist_len;
  kp.hist_smem = p->hist_len <= fs::kHistSmemMax ? 1u : 0u;
  kp.starts = p->starts_dev;
  return kp;
}

int prepare(fs_plan *p, bool rows) {
  if (!p) return FS_EINVAL;
  if (rows != (p->c.alpha == 0)) return FS_EINVAL;  // row-sliced vs unit-sliced plan
  int rc = fs_plan_upload_impl(p);
  if (rc != FS_OK) return rc;
  if (cudaSetDevice(p->device) != cudaSuccess) return FS_ECUDA;
  if (cudaMemsetAsync(p->scratch_dev, 0, 8, p->stream) != cudaSuccess) return FS_ECUDA;
  p->last_launches = 0;
  return FS_OK;
}

int finish(fs_plan *p, int rc) {
  if (rc == FS_OK) p->last_launches = 1;
  return rc;
}

int sync_plan(fs_plan *p) {
  cudaError_t e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) return FS_ECUDA;
  return FS_OK;
}

struct PlanHolder {
  fs_plan *p = nullptr;
  ~PlanHolder() { fs_plan_destroy(p); }
};

}  // namespace

extern "C" {

int fs_version(void) { return 10000; }

const char *fs_strerror(int code) {
  switch (code) {
    case FS_OK: return "ok";
    case FS_EINVAL: return "invalid argument";
    case FS_ERANGE: return "value out of the supported range";
    case FS_ECUDA: return "CUDA runtime error";
    case FS_ENOMEM: return "device out of memory";
    case FS_ENODEV: return "no CUDA device";
  }
  return "unknown error";
}

int fs_plan_create(uint64_t n, const uint32_t *gens, int d, int consumer, const fs_exec_t *ex, fs_plan **out) {
  if (!out) return FS_EINVAL;
  *out = nullptr;
  fs_plan *p = new (std::nothrow) fs_plan();
  if (!p) return FS_ENOMEM;
  int rc = fs_validate_and_build(p, n, gens, d, consumer, ex);
  if (rc != FS_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return FS_OK;
}

int fs_plan_info(const fs_plan *p, fs_plan_info_t *info) {
  if (!p || !info) return FS_EINVAL;
  memset(info, 0, sizeof(*info));
  info->n = p->n;
  info->d = p->d;
  info->consumer = p->consumer;
  info->level = p->d >= 2 ? p->d - 2 : 0;
  info->total_units = p->total_units;
  info->total_rows = p->total_rows;
  info->unit_begin = p->unit_begin;
  info->unit_end = p->unit_end;
  info->row_begin = p->row_begin;
  info->row_end = p->row_end;
  info->slice_units = p->T;
  info->num_slices = p->num_slices;
  info->hist_len = p->hist_len;
  info->grid = p->grid;
  info->block = p->block;
  for (int i = 0; i < FS_MAX_D; ++i) info->nodes_per_level[i] = p->nodes_per_level[i];
  info->table_bytes = p->U.size() * 8 + p->ktab.size() * 4;
  info->state_block = p->c.qtab_off ? (uint32_t)FS_QK
                      : (p->consumer == FS_CONSUMER_HIST && p->ex.tail == FS_TAIL_CLOSED && p->d >= 2 &&
                         fs_hist_closed_shape(p).hq) ? (uint32_t)FS_HK : 0u;
  info->cost_slices = p->cost_slices ? 1u : 0u;
  info->dead_levels = p->c.cd_mask;
  return FS_OK;
}

void fs_plan_destroy(fs_plan *p) {
  if (!p) return;
  fs_plan_free_device(p);
  delete p;
}

int fs_plan_last_launches(const fs_plan *p) { return p ? p->last_launches : 0; }

int fs_plan_count_async(fs_plan *p, uint64_t *count_dev) {
  if (!count_dev) return FS_EINVAL;
  int rc = prepare(p, false);
  if (rc != FS_OK) return rc;
  DeviceGuard g(p->device);
  if (cudaMemsetAsync(count_dev, 0, 8, p->stream) != cudaSuccess) return FS_ECUDA;
  fs::KParams kp = base_params(p);
  kp.count_out = reinterpret_cast<unsigned long long *>(count_dev);
  const int cons = p->ex.tail == FS_TAIL_CLOSED       ? fs::kConsCountClosed
                   : p->ex.tail == FS_TAIL_SKIP_OFF   ? fs::kConsCountSkipOff
                   : p->ex.tail == FS_TAIL_SKIP_PAPER ? fs::kConsCountSkipPaper
                                                      : FS_CONSUMER_COUNT;
  return finish(p, fs_launch(p, cons, 16, kp, p->stream));
}

// Slice audit (include/fsgpu_debug.h): the closed-tail count with every slice's row count written
// to slice_counts_dev[sl] (the lane that ran the slice stores it when the slice is complete).
int fsdbg_count_slices(fs_plan *p, uint64_t *count_dev, uint64_t *slice_counts_dev) {
  if (!count_dev || !slice_counts_dev) return FS_EINVAL;
  if (!p || p->ex.tail != FS_TAIL_CLOSED || p->c.alpha != 1u) return FS_EINVAL;
  int rc = prepare(p, false);
  if (rc != FS_OK) return rc;
  DeviceGuard g(p->device);
  if (cudaMemsetAsync(count_dev, 0, 8, p->stream) != cudaSuccess) return FS_ECUDA;
  if (p->num_slices &&
      cudaMemsetAsync(slice_counts_dev, 0, p->num_slices * 8, p->stream) != cudaSuccess)
    return FS_ECUDA;
  fs::KParams kp = base_params(p);
  kp.count_out = reinterpret_cast<unsigned long long *>(count_dev);
  kp.slice_counts = reinterpret_cast<unsigned long long *>(slice_counts_dev);
  return finish(p, fs_launch(p, fs::kConsCountClosed, 16, kp, p->stream));
}

// The first node-unit index of slice sl and that node's prefix a_1..a_L (host computation of the
// plan's slicing: uniform, or equal-cost boundaries).
int fsdbg_slice_start(const fs_plan *p, uint64_t sl, uint64_t *unit_out, uint32_t *prefix_out) {
  if (!p || !unit_out || sl >= p->num_slices) return FS_EINVAL;
  uint64_t u, e;
  uint32_t pre[FS_MAX_D];
  if (p->cost_slices) {
    u = fs_host_cost_boundary(p, fs::cost_target(p->cost_begin, p->cost_end, p->gn0, p->gn1, p->num_slices, sl), pre);
  } else {
    fs::slice_range(p->unit_begin, p->unit_end, p->T, p->gn0, p->gn1, sl, u, e);
  }
  *unit_out = u;
  if (prefix_out && p->d >= 3 && u < p->total_units) {
    int64_t row = 0;
    int rc = fsdbg_unrank(p, u, prefix_out, &row);
    if (rc != FS_OK) return rc;
  }
  return FS_OK;
}

int fs_plan_hist_async(fs_plan *p, uint64_t *hist_dev, uint64_t hist_cap) {
  if (!p || !hist_dev || hist_cap < p->hist_len) return FS_EINVAL;
  int rc = prepare(p, false);
  if (rc != FS_OK) return rc;
  DeviceGuard g(p->device);
  if (cudaMemsetAsync(hist_dev, 0, hist_cap * 8, p->stream) != cudaSuccess) return FS_ECUDA;
  fs::KParams kp = base_params(p);
  kp.hist_out = reinterpret_cast<unsigned long long *>(hist_dev);
  if (p->ex.tail == FS_TAIL_CLOSED && p->d >= 2) {
    // closed tail: strided difference array + finalize (two or four launches)
    const fs_hist_shape hs = fs_hist_closed_shape(p);
    kp.diff_len = hs.diff_len;
    kp.hist_smem = hs.hist_smem;
    kp.hist_rep = hs.hist_rep;
    kp.hist_hq = hs.hq;
    kp.diff_slen = hs.slen;
    kp.diff_sbias = hs.sbias;
    const uint64_t scratch = fs_hist_finalize_scratch(p->hist_len, p->c.dstride);
    if (!p->diff_dev && cudaMalloc(&p->diff_dev, ((size_t)kp.diff_len + scratch) * 8) != cudaSuccess) return FS_ENOMEM;
    if (cudaMemsetAsync(p->diff_dev, 0, (size_t)kp.diff_len * 8, p->stream) != cudaSuccess) return FS_ECUDA;
    kp.diff_out = p->diff_dev;
    rc = fs_launch(p, fs::kConsHistClosed, 16, kp, p->stream);
    if (rc != FS_OK) return rc;
    int fl = 0;
    rc = fs_launch_hist_finalize(kp, scratch ? p->diff_dev + kp.diff_len : nullptr, p->stream, &fl);
    if (rc == FS_OK) p->last_launches = 1 + fl;
    return rc;
  }
  // per-row histogram: one inner-loop iteration adds at most 4 rows per lane, far below the
  // drain guard's 2^30, whatever the instance
  return finish(p, fs_launch(p, FS_CONSUMER_HIST, 16, kp, p->stream));
}

int fs_plan_any_async(fs_plan *p, int pred, uint64_t pred_arg, int *found_dev, uint32_t *witness_dev) {
  if (!p || !found_dev) return FS_EINVAL;
  if (pred < FS_PRED_LEN_LE || pred > FS_PRED_COORD_GE) return FS_EINVAL;
  int rc = prepare(p, false);
  if (rc != FS_OK) return rc;
  DeviceGuard g(p->device);
  if (cudaMemsetAsync(found_dev, 0, 4, p->stream) != cudaSuccess) return FS_ECUDA;
  // (a witness is written only when found; zeroed so a copy of it is always defined)
  if (witness_dev && cudaMemsetAsync(witness_dev, 0, 4u * (size_t)p->d, p->stream) != cudaSuccess) return FS_ECUDA;
  fs::KParams kp = base_params(p);
  kp.pred = pred;
  kp.pred_arg = pred_arg;
  if (pred == FS_PRED_COORD_GE) {  // caller's coordinate index -> the stream's index
    const uint64_t i = pred_arg >> 32;
    if (i < (uint64_t)p->d) kp.pred_arg = ((uint64_t)p->iperm[i] << 32) | (pred_arg & 0xffffffffull);
  }
  kp.found = found_dev;
  kp.witness = witness_dev;
  // claim order from both ends, bit-reversed inside each half (fs_kernels.cuh claim_slice): every
  // region of the lex order, and both of its ends first, are sampled early (early exit)
  uint32_t bits = 0;
  while ((1ull << bits) < kp.num_slices) ++bits;
  kp.permute = 1;
  kp.claim_bits = bits;
  kp.num_claims = kp.num_slices ? (1ull << bits) : 0;
  // closed tail: each node decided at once (any_closed_pick), a kernel of its own
  return finish(p, fs_launch(p, p->ex.tail == FS_TAIL_CLOSED ? fs::kConsAnyClosed : FS_CONSUMER_ANY, 16, kp,
                             p->stream));
}

int fs_plan_enumerate_async(fs_plan *p, int B, void *out_dev, uint64_t cap) {
  if (!p || (B != 16 && B != 32)) return FS_EINVAL;
  if (((uintptr_t)out_dev & 15u) != 0) return FS_EINVAL;
  if (B == 16) {
    for (int i = 0; i < p->d; ++i)
      if (p->n / p->g[i] > 65535) return FS_ERANGE;
  }
  int rc = prepare(p, true);
  if (rc != FS_OK) return rc;
  DeviceGuard g(p->device);
  fs::KParams kp = base_params(p);
  const uint64_t span = p->unit_end - p->unit_begin;
  const uint64_t take = cap < span ? cap : span;
  if (take == 0) return finish(p, FS_OK);
  if (!out_dev) return FS_EINVAL;
  const bool incr = p->ex.order == FS_ORDER_INCREASING;
  if (p->ex.order != FS_ORDER_CANONICAL && p->ex.order != FS_ORDER_ANY && !incr) return FS_EINVAL;
  kp.unit1 = p->unit_begin + take;
  if (incr) {  // the first `take` rows in increasing order = the last `take` canonical rows
    kp.unit0 = p->unit_end - take;
    kp.unit1 = p->unit_end;
    // the table (64-row slices) holds the mirrored slicing: entry nfull - 1 - idx for slice idx
    if (p->T == 64 && kp.starts)
      kp.starts_rev = (p->unit_end - p->unit_begin) / p->T;
    else
      kp.starts = nullptr;
  }
  // canonical order (M1): the table only with its 64-row slices (fs_host.cu); at 512 rows it
  // measured slower (C2-XL 4.78 -> 4.97 ms, also with evict-first table loads, so not L2
  // pollution; cause not established), while M2 (whole-warp blocks) gains (4.06 -> 3.93 ms)
  if (p->ex.order == FS_ORDER_CANONICAL && p->T != 64) kp.starts = nullptr;
  kp.num_slices = (take + p->T - 1) / p->T;
  kp.num_claims = kp.num_slices;
  kp.rows_out = reinterpret_cast<unsigned char *>(out_dev);
  kp.row_bytes = (uint32_t)(p->d * (B / 8));
  if (p->ex.rows_impl == FS_ROWS_BATCH && fs_rows_batch_supported(p, B)) {
    // lockstep batch kernel over the full slices + the ragged-tail kernel
    kp.num_slices = take / p->T;
    kp.num_claims = kp.num_slices;
    if (p->ex.order == FS_ORDER_ANY) {
      if (take < span) return FS_ERANGE;
      char *base = reinterpret_cast<char *>(p->scratch_dev);
      if (cudaMemsetAsync(base + kOffFront, 0, kOffBack + 8 - kOffFront, p->stream) != cudaSuccess) return FS_ECUDA;
      kp.front = reinterpret_cast<unsigned long long *>(base + kOffFront);
      kp.back = reinterpret_cast<unsigned long long *>(base + kOffBack);
      kp.rank_rows = span;
    }
    int launches = 0;
    uint32_t grid = 0;
    rc = fs_dispatch_rows_batch(p, B, p->ex.order == FS_ORDER_ANY ? 1 : incr ? 2 : 0, kp, p->stream, false, &grid,
                                &launches);
    if (rc != FS_OK) return rc;
    p->grid = grid;
    g_fs_total_launches += (unsigned long long)launches;
    p->last_launches = launches;
    return FS_OK;
  }
  if (p->ex.order == FS_ORDER_ANY) {
    if (take < span) return FS_ERANGE;  // compaction writes all of the rank's rows
    char *base = reinterpret_cast<char *>(p->scratch_dev);
    if (cudaMemsetAsync(base + kOffFront, 0, kOffBack + 8 - kOffFront, p->stream) != cudaSuccess) return FS_ECUDA;
    kp.front = reinterpret_cast<unsigned long long *>(base + kOffFront);
    kp.back = reinterpret_cast<unsigned long long *>(base + kOffBack);
    kp.rank_rows = span;
    return finish(p, fs_launch(p, fs::kConsRowsAny, B, kp, p->stream));
  }
  if (incr) {  // staged kernel in canonical order, then the rows reversed in place
    kp.starts = nullptr;  // (a table of this plan holds the mirrored slicing)
    kp.starts_rev = 0;
    rc = fs_launch(p, FS_CONSUMER_ROWS, B, kp, p->stream);
    if (rc != FS_OK) return rc;
    rc = fs_launch_rows_reverse(kp.rows_out, take, kp.row_bytes, p->stream);
    if (rc != FS_OK) return rc;
    p->last_launches = 2;
    return FS_OK;
  }
  return finish(p, fs_launch(p, FS_CONSUMER_ROWS, B, kp, p->stream));
}

int fs_plan_rows_check(fs_plan *p) {
  if (!p || p->c.alpha != 0) return FS_EINVAL;
  if (!p->uploaded || p->ex.order != FS_ORDER_ANY || p->row_end == p->row_begin) return FS_OK;
  DeviceGuard g(p->device);
  if (sync_plan(p) != FS_OK) return FS_ECUDA;
  // M2 exactness check: the front and back cursors must meet at the rank's row count
  unsigned long long fr = 0, bk = 0;
  char *base = reinterpret_cast<char *>(p->scratch_dev);
  if (cudaMemcpy(&fr, base + kOffFront, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(&bk, base + kOffBack, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return FS_ECUDA;
  return fr + bk == p->row_end - p->row_begin ? FS_OK : FS_ECUDA;
}

// ------------------------------------------------------------------ synchronous entry points
int fs_count_ex(uint64_t n, const uint32_t *gens, int d, const fs_exec_t *ex, uint64_t *count_out) {
  if (!count_out) return FS_EINVAL;
  PlanHolder h;
  int rc = fs_plan_create(n, gens, d, FS_CONSUMER_COUNT, ex, &h.p);
  if (rc != FS_OK) return rc;
  rc = fs_plan_upload_impl(h.p);
  if (rc != FS_OK) return rc;
  DeviceGuard g(h.p->device);
  uint64_t *dev = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(h.p->scratch_dev) + kOffCount);
  rc = fs_plan_count_async(h.p, dev);
  if (rc != FS_OK) return rc;
  if (cudaMemcpyAsync(count_out, dev, 8, cudaMemcpyDeviceToHost, h.p->stream) != cudaSuccess) return FS_ECUDA;
  return sync_plan(h.p);
}

int fs_count(uint64_t n, const uint32_t *gens, int d, uint64_t *count_out) {
  fs_exec_t ex;
  memset(&ex, 0, sizeof(ex));
  ex.device = -1;
  ex.world = 1;
  ex.gen_order = FS_GENORDER_AUTO;  // exact for any order; fewest nodes first
  ex.tail = FS_TAIL_CLOSED;         // a node's rows counted by division (NEXT-1)
  return fs_count_ex(n, gens, d, &ex, count_out);
}

int fs_length_set_ex(uint64_t n, const uint32_t *gens, int d, const fs_exec_t *ex, uint64_t *hist_dev,
                     uint64_t hist_cap) {
  PlanHolder h;
  int rc = fs_plan_create(n, gens, d, FS_CONSUMER_HIST, ex, &h.p);
  if (rc != FS_OK) return rc;
  if (!hist_dev || hist_cap < h.p->hist_len) return FS_EINVAL;
  rc = fs_plan_hist_async(h.p, hist_dev, hist_cap);
  if (rc != FS_OK) return rc;
  DeviceGuard g(h.p->device);
  return sync_plan(h.p);
}

int fs_length_set(uint64_t n, const uint32_t *gens, int d, uint64_t *hist_dev, uint64_t hist_cap) {
  fs_exec_t ex;
  memset(&ex, 0, sizeof(ex));
  ex.device = -1;
  ex.world = 1;
  ex.gen_order = FS_GENORDER_AUTO;
  ex.tail = FS_TAIL_CLOSED;
  return fs_length_set_ex(n, gens, d, &ex, hist_dev, hist_cap);
}

int fs_any_ex(uint64_t n, const uint32_t *gens, int d, const fs_exec_t *ex, int pred, uint64_t pred_arg,
              int *found_out, uint32_t *witness_or_null) {
  if (!found_out) return FS_EINVAL;
  if (pred < FS_PRED_LEN_LE || pred > FS_PRED_COORD_GE) return FS_EINVAL;
  PlanHolder h;
  int rc = fs_plan_create(n, gens, d, FS_CONSUMER_ANY, ex, &h.p);
  if (rc != FS_OK) return rc;
  rc = fs_plan_upload_impl(h.p);
  if (rc != FS_OK) return rc;
  DeviceGuard g(h.p->device);
  char *base = reinterpret_cast<char *>(h.p->scratch_dev);
  int *fdev = reinterpret_cast<int *>(base + kOffFound);
  uint32_t *wdev = reinterpret_cast<uint32_t *>(base + kOffWitness);
  rc = fs_plan_any_async(h.p, pred, pred_arg, fdev, wdev);
  if (rc != FS_OK) return rc;
  if (cudaMemcpyAsync(found_out, fdev, 4, cudaMemcpyDeviceToHost, h.p->stream) != cudaSuccess) return FS_ECUDA;
  uint32_t wit[FS_MAX_D];
  if (witness_or_null &&
      cudaMemcpyAsync(wit, wdev, 4 * d, cudaMemcpyDeviceToHost, h.p->stream) != cudaSuccess)
    return FS_ECUDA;
  rc = sync_plan(h.p);
  if (rc != FS_OK) return rc;
  if (witness_or_null && *found_out) memcpy(witness_or_null, wit, 4 * d);
  return FS_OK;
}

int fs_any(uint64_t n, const uint32_t *gens, int d, int pred, uint64_t pred_arg, int *found_out,
           uint32_t *witness_or_null) {
  fs_exec_t ex;
  memset(&ex, 0, sizeof(ex));
  ex.device = -1;
  ex.world = 1;
  ex.gen_order = FS_GENORDER_AUTO;
  ex.tail = FS_TAIL_CLOSED;  // each node's rows decided at once (NEXT-1)
  return fs_any_ex(n, gens, d, &ex, pred, pred_arg, found_out, witness_or_null);
}

int64_t fs_enumerate_ex(uint64_t n, const uint32_t *gens, int d, int B, void *out_dev, uint64_t cap,
                        const fs_exec_t *ex, uint64_t *global_row_offset_out) {
  if (B != 16 && B != 32) return FS_EINVAL;
  PlanHolder h;
  int rc = fs_plan_create(n, gens, d, FS_CONSUMER_ROWS, ex, &h.p);
  if (rc != FS_OK) return rc;
  rc = fs_plan_enumerate_async(h.p, B, out_dev, cap);
  if (rc != FS_OK) return rc;
  if (h.p->uploaded) {
    DeviceGuard g(h.p->device);
    rc = sync_plan(h.p);
    if (rc != FS_OK) return rc;
    rc = fs_plan_rows_check(h.p);  // order = any: the M2 cursors met exactly
    if (rc != FS_OK) return rc;
  }
  if (global_row_offset_out)  // the block's first row in the requested order
    *global_row_offset_out = h.p->ex.order == FS_ORDER_INCREASING ? h.p->total_rows - h.p->row_end : h.p->row_begin;
  return (int64_t)(h.p->row_end - h.p->row_begin);
}

int64_t fs_enumerate_filtered_ex(uint64_t n, const uint32_t *gens, int d, int B, int pred, uint64_t pred_arg,
                                 void *out_dev, uint64_t cap, const fs_exec_t *ex) {
  if (B != 16 && B != 32) return FS_EINVAL;
  if (pred < FS_PRED_LEN_LE || pred > FS_PRED_COORD_GE) return FS_EINVAL;
  if (cap && (!out_dev || ((uintptr_t)out_dev & 15u) != 0)) return FS_EINVAL;
  fs_exec_t e;
  if (ex)
    e = *ex;
  else {
    memset(&e, 0, sizeof(e));
    e.device = -1;
    e.world = 1;
  }
  e.order = FS_ORDER_ANY;         // compaction: the matching rows' positions are not known a priori
  e.rows_impl = FS_ROWS_STAGED;   // per-step ballot compaction (emission is filtered per row)
  PlanHolder h;
  int rc = fs_plan_create(n, gens, d, FS_CONSUMER_ROWS, &e, &h.p);
  if (rc != FS_OK) return rc;
  fs_plan *p = h.p;
  if (B == 16) {
    for (int i = 0; i < p->d; ++i)
      if (p->n / p->g[i] > 65535) return FS_ERANGE;
  }
  const uint64_t span = p->unit_end - p->unit_begin;
  if (span == 0) return 0;
  if (p->d == 1) {  // Z = {(n/g)} iff g | n: decided on the host
    const uint64_t x = p->n / p->g[0];
    bool ok;
    switch (pred) {
      case FS_PRED_LEN_LE: ok = x <= pred_arg; break;
      case FS_PRED_LEN_GE: ok = x >= pred_arg; break;
      case FS_PRED_LEN_EQ: ok = x == pred_arg; break;
      default: ok = (pred_arg >> 32) == 0 && x >= (pred_arg & 0xffffffffull);
    }
    if (!ok) return 0;
    if (cap >= 1) {
      DeviceGuard g(p->device);
      if (B == 16) {
        const uint16_t v = (uint16_t)x;
        if (cudaMemcpy(out_dev, &v, 2, cudaMemcpyHostToDevice) != cudaSuccess) return FS_ECUDA;
      } else {
        const uint32_t v = (uint32_t)x;
        if (cudaMemcpy(out_dev, &v, 4, cudaMemcpyHostToDevice) != cudaSuccess) return FS_ECUDA;
      }
    }
    return 1;
  }
  unsigned long long cur[2] = {0, 0};
  uint64_t matches = 0;
  for (int pass = 0; pass < 2; ++pass) {
    rc = prepare(p, true);
    if (rc != FS_OK) return rc;
    DeviceGuard g(p->device);
    fs::KParams kp = base_params(p);
    kp.rows_out = reinterpret_cast<unsigned char *>(out_dev);
    kp.row_bytes = (uint32_t)(p->d * (B / 8));
    kp.filt_pred = pred;
    kp.filt_arg = pred_arg;
    if (pred == FS_PRED_COORD_GE) {  // caller's coordinate index -> the stream's index
      const uint64_t i = pred_arg >> 32;
      if (i < (uint64_t)p->d) kp.filt_arg = ((uint64_t)p->iperm[i] << 32) | (pred_arg & 0xffffffffull);
    }
    kp.count_only = pass == 0 ? 1 : 0;
    char *base = reinterpret_cast<char *>(p->scratch_dev);
    if (cudaMemsetAsync(base + kOffFront, 0, kOffBack + 8 - kOffFront, p->stream) != cudaSuccess) return FS_ECUDA;
    kp.front = reinterpret_cast<unsigned long long *>(base + kOffFront);
    kp.back = reinterpret_cast<unsigned long long *>(base + kOffBack);
    kp.rank_rows = matches;
    rc = fs_launch(p, fs::kConsRowsAny, B, kp, p->stream);
    if (rc != FS_OK) return rc;
    rc = sync_plan(p);
    if (rc != FS_OK) return rc;
    if (cudaMemcpy(&cur[0], base + kOffFront, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&cur[1], base + kOffBack, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      return FS_ECUDA;
    if (pass == 0) {
      matches = cur[0];
      if (matches == 0 || matches > cap) return (int64_t)matches;
    } else if (cur[0] + cur[1] != matches) {
      return FS_ECUDA;  // the cursors must meet exactly at the pass-1 count
    }
  }
  return (int64_t)matches;
}

int64_t fs_enumerate(uint64_t n, const uint32_t *gens, int d, int B, void *out_dev, uint64_t cap) {
  fs_exec_t ex;
  memset(&ex, 0, sizeof(ex));
  ex.device = -1;
  ex.world = 1;
  int64_t r = fs_enumerate_ex(n, gens, d, B, out_dev, cap, &ex, nullptr);
  return r;
}

uint64_t fsdbg_total_launches(void) { return g_fs_total_launches.load(); }

}  // extern "C"
