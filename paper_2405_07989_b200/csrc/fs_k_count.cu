// fs_k_count.cu -- instantiates the persistent kernels of the count consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include <string.h>

#include "fs_kernels.cuh"

int fs_dispatch_count_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B;
  // B is meaningless for a count: the B = 32 instantiation walks live nodes only (NEXT-3)
  return p->c.cadv2_skip ? fs::dispatch_kt<fs::kConsCountClosed, 32>(p, kp, s, q, g)
                         : fs::dispatch_kt<fs::kConsCountClosed, 16>(p, kp, s, q, g);
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

// Slice-start table of a plan (node units: the first node's prefix; row units: also the row
// offset in it): launched once per plan at upload; refills then read L (+1) words instead of
// unranking (16 dependent-load binary searches
// per slice otherwise cost ~0.9 ms of latency per launch on C3, which dominates small shards).
int fs_build_slice_starts(fs_plan *p) {
  const int L = p->d - 2;
  if (L < 1 || p->num_slices == 0) return FS_OK;
  const uint64_t words = p->num_slices * (uint64_t)(L + (p->c.alpha ? 0 : 1));  // row units: + offset
  if (words * 4u > (256ull << 20)) return FS_OK;  // the unrank path instead
  // stream-ordered allocation from the device's memory pool (kept across plans: a one-shot
  // fs_count would otherwise pay a synchronous cudaMalloc/cudaFree of tens of MB per call)
  static bool pool_set[64] = {false};
  if (p->device >= 0 && p->device < 64 && !pool_set[p->device]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, p->device) == cudaSuccess) {
      uint64_t keep = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    pool_set[p->device] = true;
  }
  if (cudaMallocAsync(reinterpret_cast<void **>(&p->starts_dev), words * 4u, p->stream) != cudaSuccess) {
    cudaGetLastError();
    p->starts_dev = nullptr;
    return FS_OK;
  }
  p->starts_async = true;
  fs::KParams kp;
  memset(&kp, 0, sizeof(kp));
  kp.c = p->c;
  kp.c.U = p->U_dev;
  kp.c.ktab = p->ktab_dev;
  kp.unit0 = p->unit_begin;
  kp.unit1 = p->unit_end;
  kp.T = p->T;
  kp.num_slices = p->num_slices;
  uint64_t blocks = (p->num_slices + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  switch (p->d) {
#define FS_CASE(DD)                                                                                       \
  case DD:                                                                                                \
    fs::fs_slice_starts_kernel<DD><<<(unsigned)blocks, 256, 0, p->stream>>>(kp, p->starts_dev);         \
    break;
    FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
    default: return FS_OK;
  }
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  ++g_fs_total_launches;
  return FS_OK;
}
