// fs_k_rowsany.cu -- instantiates the materialise kernels with order = any (M2: warp-aggregated
// atomic compaction), d = 1..16, both coordinate widths.
#include "fs_kernels.cuh"

int fs_dispatch_rowsany(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  return B == 16 ? fs::dispatch_kt<fs::kConsRowsAny, 16>(p, kp, s, q, g)
                 : fs::dispatch_kt<fs::kConsRowsAny, 32>(p, kp, s, q, g);
}
