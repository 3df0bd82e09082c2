// fs_k_any.cu -- instantiates the persistent kernels of the any consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include "fs_kernels.cuh"

int fs_dispatch_any(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B; return fs::dispatch_kt<FS_CONSUMER_ANY, 16>(p, kp, s, q, g);
}

int fs_dispatch_any_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  // (B = 32: the NEXT-3 variant -- live-node step, k >= 3 dead-subtree skip)
  (void)B;
  return (p->c.h > 1u && p->c.radv_off) || p->c.cd_mask ? fs::dispatch_kt<fs::kConsAnyClosed, 32>(p, kp, s, q, g)
                                                        : fs::dispatch_kt<fs::kConsAnyClosed, 16>(p, kp, s, q, g);
}
