// fs_k_count.cu -- instantiates the persistent kernels of the count consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include <string.h>

#include <mutex>

#include "fs_kernels.cuh"

int fs_dispatch_count_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B;
  // B is meaningless for a count.  B = 16: the state-form walk over equal-cost guided slices,
  // refill checks every FS_CC_INNER steps.  B = 32: the NEXT-3 variant (live-node walk, k >= 3
  // dead-subtree skip) and every plan with uniform slices (small instances: few runs per lane,
  // short slices), refill checks every 128 steps.
  const bool b16 = p->cost_slices && !p->c.cadv2_skip && !p->c.cd_mask;
  return b16 ? fs::dispatch_kt<fs::kConsCountClosed, 16>(p, kp, s, q, g)
             : fs::dispatch_kt<fs::kConsCountClosed, 32>(p, kp, s, q, g);
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

// The library's private stream-ordered memory pool on `device` (nullptr if it cannot be made).
static cudaMemPool_t fs_device_pool(int device) {
  constexpr int kMaxDev = 64;
  static std::once_flag once[kMaxDev];
  static cudaMemPool_t pools[kMaxDev];
  if (device < 0 || device >= kMaxDev) return nullptr;
  std::call_once(once[device], [device]() {
    cudaMemPoolProps props;
    memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t keep = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[device] = pool;
    } else {
      cudaGetLastError();
      pools[device] = nullptr;
    }
  });
  return pools[device];
}

// Equal-cost slices: the table is mandatory (it holds each slice's node count); built by a
// cost-space unrank per slice, then the node counts from consecutive starts.
static int build_cost_slice_starts(fs_plan *p, uint64_t words) {
  cudaMemPool_t pool = fs_device_pool(p->device);
  unsigned long long *ustart = nullptr;
  if (!pool ||
      cudaMallocFromPoolAsync(reinterpret_cast<void **>(&p->starts_dev), words * 4u, pool, p->stream) != cudaSuccess ||
      cudaMallocFromPoolAsync(reinterpret_cast<void **>(&ustart), p->num_slices * 8u, pool, p->stream) != cudaSuccess) {
    cudaGetLastError();
    if (p->starts_dev) cudaFreeAsync(p->starts_dev, p->stream);
    p->starts_dev = nullptr;
    return FS_ENOMEM;
  }
  p->starts_async = true;
  fs::KParams kp;
  memset(&kp, 0, sizeof(kp));
  kp.c = p->c;
  kp.c.U = p->U_dev;
  kp.c.ktab = p->ktab_dev;
  kp.unit0 = p->unit_begin;
  kp.unit1 = p->unit_end;
  kp.gn0 = p->gn0;
  kp.gn1 = p->gn1;
  kp.num_slices = p->num_slices;
  kp.cost_slices = 1;
  uint64_t blocks = (p->num_slices + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  switch (p->d) {
#define FS_CASE(DD)                                                                                              \
  case DD:                                                                                                       \
    fs::fs_slice_starts_cost_kernel<DD><<<(unsigned)blocks, 256, 0, p->stream>>>(kp, p->CW_dev, p->cost_begin,   \
                                                                                  p->cost_end, p->starts_dev, ustart); \
    fs::fs_slice_budgets_kernel<DD><<<(unsigned)blocks, 256, 0, p->stream>>>(kp, p->starts_dev, ustart);        \
    break;
    FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
    default: return FS_EINVAL;
  }
  cudaFreeAsync(ustart, p->stream);
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  g_fs_total_launches += 2;
  return FS_OK;
}

// Slice-start table of a plan (node units: the first node's prefix; row units: also the row
// offset in it): launched once per plan at upload; refills then read L (+1) words instead of
// unranking (16 dependent-load binary searches
// per slice otherwise cost ~0.9 ms of latency per launch on C3, which dominates small shards).
int fs_build_slice_starts(fs_plan *p) {
  const int L = p->d - 2;
  if (L < 1 || p->num_slices == 0) return FS_OK;
  // row units: + the row offset; equal-cost slices: + the slice's node count
  const uint64_t words = p->num_slices * (uint64_t)(L + (p->c.alpha && !p->cost_slices ? 0 : 1));
  if (p->cost_slices) return build_cost_slice_starts(p, words);
  // (at most 256 MB; canonical materialise at 64-row slices: FS_M1_TABLE_MB, fs_host.cu)
  const bool m1 = p->consumer == FS_CONSUMER_ROWS && p->ex.order != FS_ORDER_ANY && p->T == 64;
  if (words * 4u > ((uint64_t)(m1 ? FS_M1_TABLE_MB : 256) << 20)) return FS_OK;  // the unrank path instead
  // stream-ordered allocation from the library's own memory pool on the device (created once
  // per device, thread-safe; it keeps up to 1 GB cached across plans so a one-shot fs_count does
  // not pay a synchronous cudaMalloc/cudaFree of tens of MB per call).  The device's default
  // pool -- which torch or the caller may use -- is left untouched.
  cudaMemPool_t pool = fs_device_pool(p->device);
  if (!pool || cudaMallocFromPoolAsync(reinterpret_cast<void **>(&p->starts_dev), words * 4u, pool, p->stream) !=
                   cudaSuccess) {
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
  kp.gn0 = p->gn0;
  kp.gn1 = p->gn1;
  kp.num_slices = p->num_slices;
  if (m1 && p->ex.order == FS_ORDER_INCREASING) {
    // the mirrored slicing of increasing order: its full slices end at unit_end, so entry k
    // starts at unit_begin + (span mod T) + k T (the batch kernel reads entry nfull - 1 - idx)
    const uint64_t span = p->unit_end - p->unit_begin;
    kp.unit0 = p->unit_begin + span % p->T;
    kp.num_slices = span / p->T;
    if (kp.num_slices == 0) return FS_OK;
  }
  uint64_t blocks = (kp.num_slices + 255) / 256;
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
