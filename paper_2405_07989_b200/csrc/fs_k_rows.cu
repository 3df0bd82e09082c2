// fs_k_rows.cu -- instantiates the persistent kernels of the rows consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include "fs_kernels.cuh"

int fs_dispatch_rows(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  return B == 16 ? fs::dispatch_kt<FS_CONSUMER_ROWS, 16>(p, kp, s, q, g) : fs::dispatch_kt<FS_CONSUMER_ROWS, 32>(p, kp, s, q, g);
}
