// fs_k_hist.cu -- instantiates the persistent kernels of the hist consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include "fs_kernels.cuh"

int fs_dispatch_hist_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B;
  return fs::dispatch_kt<fs::kConsHistClosed, 16>(p, kp, s, q, g);
}

int fs_launch_hist_finalize(const fs::KParams &kp, cudaStream_t stream) {
  const uint32_t threads = 128;
  uint32_t blocks = (kp.c.dstride + threads - 1) / threads;
  if (blocks > 148) blocks = 148;
  if (blocks == 0) blocks = 1;
  fs::fs_hist_finalize_kernel<<<blocks, threads, 0, stream>>>(kp.diff_out, kp.hist_out, kp.hist_len, kp.c.dstride);
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  ++g_fs_total_launches;
  return FS_OK;
}

int fs_dispatch_hist(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B; return fs::dispatch_kt<FS_CONSUMER_HIST, 16>(p, kp, s, q, g);
}
