// fs_k_rowsb.cu -- launches of the lockstep batch materialise kernel (fs_rows_batch.cuh) for
// M1 (canonical) and M2 (order = any), plus the ragged-tail kernel.
#include "fs_rows_batch.cuh"

namespace fs {

template <int D, int B, int MODE, bool KTAB>
static int rb_launch(fs_plan *p, const KParams &kp, cudaStream_t stream, bool query_only, uint32_t *grid_out,
                     int *launches) {
  using G = RowsBatchGeom<D, B>;
  if constexpr (!G::kOk) {
    return FS_EINVAL;
  } else {
    auto kern = fs_rows_batch_kernel<D, B, MODE, KTAB>;
    const size_t smem = (size_t)((kp.c.ktab_len + 3u) & ~3u) * 4 + G::smem_stage(kRbBlock / 32);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return FS_ECUDA;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRbBlock, smem) != cudaSuccess) return FS_ECUDA;
    if (per_sm < 1) return FS_ECUDA;
    if (p->ex.ctas_per_sm > 0 && p->ex.ctas_per_sm < per_sm) per_sm = p->ex.ctas_per_sm;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) return FS_ECUDA;
    uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
    const uint64_t need = (kp.num_slices + kRbBlock - 1) / kRbBlock;  // one slice per lane at least
    if (grid > need) grid = need ? need : 1;
    if (grid_out) *grid_out = (uint32_t)grid;
    if (query_only) return FS_OK;
    const uint64_t full_rows = kp.num_slices * kp.T;
    const uint64_t span = kp.unit1 - kp.unit0;
    if (kp.num_slices) {
      kern<<<(unsigned)grid, kRbBlock, smem, stream>>>(kp);
      if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
      ++*launches;
    }
    if (span > full_rows) {  // the ragged slice: the end of the range, or (MODE 2) its start
      fs_rows_tail_kernel<D, B, MODE><<<1, kBlock, 0, stream>>>(kp, MODE == 2 ? 0 : full_rows, span - full_rows);
      if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
      ++*launches;
    }
    return FS_OK;
  }
}

template <int B, int MODE, bool KTAB>
static int rb_dispatch_d(fs_plan *p, const KParams &kp, cudaStream_t s, bool q, uint32_t *g, int *n) {
  switch (p->d) {
#define FS_CASE(DD) \
  case DD:          \
    return rb_launch<DD, B, MODE, KTAB>(p, kp, s, q, g, n);
    FS_CASE(2) FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
  }
  return FS_EINVAL;
}

template <int B>
static bool rb_ok_b(int d) {
  switch (d) {
#define FS_CASE(DD) \
  case DD:          \
    return RowsBatchGeom<DD, B>::kOk;
    FS_CASE(2) FS_CASE(3) FS_CASE(4) FS_CASE(5) FS_CASE(6) FS_CASE(7) FS_CASE(8) FS_CASE(9)
    FS_CASE(10) FS_CASE(11) FS_CASE(12) FS_CASE(13) FS_CASE(14) FS_CASE(15) FS_CASE(16)
#undef FS_CASE
  }
  return false;
}

}  // namespace fs

// The batch kernel applies to row-unit plans in the caller's generator order whose row shape
// has a batch of at most 112 B (fs::RowsBatchGeom::kOk).
bool fs_rows_batch_supported(const fs_plan *p, int B) {
  if (p->d < 2 || p->c.permuted) return false;
  if (p->T % 64 != 0) return false;
  return B == 16 ? fs::rb_ok_b<16>(p->d) : fs::rb_ok_b<32>(p->d);
}

// Reverse `rows` rows of `rb` bytes in place (increasing-order fallback for row shapes the
// batch kernel does not cover).
static __global__ void fs_rows_reverse_kernel(unsigned char *out, uint64_t rows, uint32_t rb) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows / 2; i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned char *a = out + i * rb, *b = out + (rows - 1 - i) * rb;
    for (uint32_t k = 0; k < rb; k += 2) {  // rows are 2-byte aligned (u16 / u32 coordinates)
      const uint16_t x = *reinterpret_cast<uint16_t *>(a + k);
      *reinterpret_cast<uint16_t *>(a + k) = *reinterpret_cast<uint16_t *>(b + k);
      *reinterpret_cast<uint16_t *>(b + k) = x;
    }
  }
}

int fs_launch_rows_reverse(unsigned char *out, uint64_t rows, uint32_t rb, cudaStream_t stream) {
  if (rows < 2) return FS_OK;
  uint64_t blocks = (rows / 2 + 255) / 256;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  fs_rows_reverse_kernel<<<(unsigned)blocks, 256, 0, stream>>>(out, rows, rb);
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  ++g_fs_total_launches;
  return FS_OK;
}

bool fs_rows_batch_shape_ok(int d) { return fs::rb_ok_b<16>(d) || fs::rb_ok_b<32>(d); }

// kp.num_slices = number of FULL slices of T rows; rows [num_slices * T, unit1 - unit0) go to
// the tail kernel.  *launches counts the kernels enqueued.
int fs_dispatch_rows_batch(fs_plan *p, int B, int mode, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g,
                           int *launches) {
  const bool ktab = kp.c.ktab_len != 0 && kp.c.radv_off != 0;
#define FS_RB(BB, MM)                                                             \
  return ktab ? fs::rb_dispatch_d<BB, MM, true>(p, kp, s, q, g, launches) \
              : fs::rb_dispatch_d<BB, MM, false>(p, kp, s, q, g, launches);
  if (B == 16) {
    if (mode == 1) FS_RB(16, 1)
    if (mode == 2) FS_RB(16, 2)
    FS_RB(16, 0)
  }
  if (mode == 1) FS_RB(32, 1)
  if (mode == 2) FS_RB(32, 2)
  FS_RB(32, 0)
#undef FS_RB
}
