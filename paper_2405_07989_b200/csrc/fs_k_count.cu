// fs_k_count.cu -- instantiates the persistent kernels of the count consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include "fs_kernels.cuh"

int fs_dispatch_count_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B;
  return fs::dispatch_kt<fs::kConsCountClosed, 16>(p, kp, s, q, g);
}

int fs_dispatch_count_skip(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g,
                          bool paper) {
  (void)B;
  return paper ? fs::dispatch_kt<fs::kConsCountSkipPaper, 16>(p, kp, s, q, g)
               : fs::dispatch_kt<fs::kConsCountSkipOff, 16>(p, kp, s, q, g);
}

int fs_dispatch_count(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B; return fs::dispatch_kt<FS_CONSUMER_COUNT, 16>(p, kp, s, q, g);
}
