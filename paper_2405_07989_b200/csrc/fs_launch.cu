// fs_launch.cu -- consumer dispatch and launch accounting for the persistent kernels.
#include <cuda_runtime.h>

#include "../../include/fsgpu.h"
#include "fs_internal.h"

std::atomic<unsigned long long> g_fs_total_launches{0};

int fs_dispatch_count(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_hist(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_any(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_rows(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_hist_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_count_skip(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g,
                          bool paper);
int fs_dispatch_count_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_any_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);
int fs_dispatch_rowsany(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g);

static int dispatch(fs_plan *p, int consumer, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  switch (consumer) {
    case FS_CONSUMER_COUNT: return fs_dispatch_count(p, B, kp, s, q, g);
    case FS_CONSUMER_HIST: return fs_dispatch_hist(p, B, kp, s, q, g);
    case FS_CONSUMER_ANY: return fs_dispatch_any(p, B, kp, s, q, g);
    case fs::kConsAnyClosed: return fs_dispatch_any_closed(p, B, kp, s, q, g);
    case FS_CONSUMER_ROWS: return fs_dispatch_rows(p, B, kp, s, q, g);
    case fs::kConsRowsAny: return fs_dispatch_rowsany(p, B, kp, s, q, g);
    case fs::kConsCountClosed: return fs_dispatch_count_closed(p, B, kp, s, q, g);
    case fs::kConsCountSkipOff: return fs_dispatch_count_skip(p, B, kp, s, q, g, false);
    case fs::kConsCountSkipPaper: return fs_dispatch_count_skip(p, B, kp, s, q, g, true);
    case fs::kConsHistClosed: return fs_dispatch_hist_closed(p, B, kp, s, q, g);
  }
  return FS_EINVAL;
}

int fs_launch(fs_plan *p, int consumer, int B, const fs::KParams &kp, cudaStream_t stream) {
  uint32_t grid = 0;
  int rc = dispatch(p, consumer, B, kp, stream, false, &grid);
  if (rc == FS_OK) {
    p->grid = grid;
    ++g_fs_total_launches;
  }
  return rc;
}

int fs_occupancy_grid(fs_plan *p, int consumer, int B, uint32_t *grid_out) {
  fs::KParams kp{};
  kp.c = p->c;
  kp.num_claims = p->num_slices;
  kp.hist_len = (uint32_t)p->hist_len;
  kp.hist_smem = p->hist_len <= fs::kHistSmemMax;
  return dispatch(p, consumer, B, kp, nullptr, true, grid_out);
}
