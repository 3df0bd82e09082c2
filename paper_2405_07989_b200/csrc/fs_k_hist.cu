// fs_k_hist.cu -- instantiates the persistent kernels of the hist consumer (d = 1..16, k0 table
// in shared memory or arithmetic).  One translation unit per consumer so nvcc compiles them in
// parallel.
#include "fs_kernels.cuh"

int fs_dispatch_hist_closed(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B;
  // (B = 16: equal-cost guided slices, refill checks every FS_HC_INNER steps; B = 32: the NEXT-3
  // variant -- live-node table walk, k >= 3 dead-subtree skip -- and uniform-slice plans, 64)
  const bool b16 = p->cost_slices && !p->c.hadv_skip && !p->c.cd_mask;
  return b16 ? fs::dispatch_kt<fs::kConsHistClosed, 16>(p, kp, s, q, g)
             : fs::dispatch_kt<fs::kConsHistClosed, 32>(p, kp, s, q, g);
}

// Closed-tail histogram finalize: hist[l] = sum of diff[k] over k <= l, k = l mod dstride (a
// prefix sum down each residue class).  Short classes (<= kFinChunk entries): one thread per
// class.  Long ones (e.g. a huge n with dstride = 1): the class is cut into chunks of kFinChunk
// entries -- chunk sums, an exclusive scan of the chunk sums per class, then each chunk's
// prefix sum from its offset (three launches; `scratch` holds fs_hist_finalize_scratch()
// entries).
static constexpr uint64_t kFinChunk = 4096;

static __global__ void fs_hist_chunk_sums_kernel(const unsigned long long *diff, unsigned long long *part,
                                                 uint64_t hist_len, uint32_t ds, uint64_t nchunks) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nchunks * ds;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ch = i / ds, r = i % ds;
    unsigned long long acc = 0;
    for (uint64_t l = r + ch * kFinChunk * ds, e = l + kFinChunk * ds; l < e && l < hist_len; l += ds) acc += diff[l];
    part[i] = acc;
  }
}

static __global__ void fs_hist_chunk_scan_kernel(unsigned long long *part, uint32_t ds, uint64_t nchunks) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < ds; r += gridDim.x * blockDim.x) {
    unsigned long long acc = 0;
    for (uint64_t ch = 0; ch < nchunks; ++ch) {
      const unsigned long long v = part[ch * ds + r];
      part[ch * ds + r] = acc;
      acc += v;
    }
  }
}

static __global__ void fs_hist_chunk_apply_kernel(const unsigned long long *diff, const unsigned long long *part,
                                                  unsigned long long *hist, uint64_t hist_len, uint32_t ds,
                                                  uint64_t nchunks) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nchunks * ds;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ch = i / ds, r = i % ds;
    unsigned long long acc = part[i];
    for (uint64_t l = r + ch * kFinChunk * ds, e = l + kFinChunk * ds; l < e && l < hist_len; l += ds) {
      acc += diff[l];
      hist[l] = acc;
    }
  }
}

static uint64_t fin_chunks(uint64_t hist_len, uint32_t ds) {
  const uint64_t rows = (hist_len + ds - 1) / ds;
  return rows <= kFinChunk ? 0 : (rows + kFinChunk - 1) / kFinChunk;
}

uint64_t fs_hist_finalize_scratch(uint64_t hist_len, uint32_t dstride) {
  return fin_chunks(hist_len, dstride) * (uint64_t)dstride;
}

int fs_launch_hist_finalize(const fs::KParams &kp, unsigned long long *scratch, cudaStream_t stream, int *launches) {
  const uint32_t threads = 128, ds = kp.c.dstride;
  const uint64_t nch = fin_chunks(kp.hist_len, ds);
  if (nch == 0) {
    uint32_t blocks = (ds + threads - 1) / threads;
    if (blocks > 148) blocks = 148;
    if (blocks == 0) blocks = 1;
    fs::fs_hist_finalize_kernel<<<blocks, threads, 0, stream>>>(kp.diff_out, kp.hist_out, kp.hist_len, ds);
    if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
    g_fs_total_launches += 1;
    *launches = 1;
    return FS_OK;
  }
  if (!scratch) return FS_EINVAL;
  uint64_t b = (nch * ds + threads - 1) / threads;
  const unsigned blocks = (unsigned)(b > 148ull * 16 ? 148ull * 16 : b);
  fs_hist_chunk_sums_kernel<<<blocks, threads, 0, stream>>>(kp.diff_out, scratch, kp.hist_len, ds, nch);
  fs_hist_chunk_scan_kernel<<<(ds + threads - 1) / threads < 148 ? (ds + threads - 1) / threads : 148, threads, 0,
                              stream>>>(scratch, ds, nch);
  fs_hist_chunk_apply_kernel<<<blocks, threads, 0, stream>>>(kp.diff_out, scratch, kp.hist_out, kp.hist_len, ds,
                                                             nch);
  if (cudaGetLastError() != cudaSuccess) return FS_ECUDA;
  g_fs_total_launches += 3;
  *launches = 3;
  return FS_OK;
}

int fs_dispatch_hist(fs_plan *p, int B, const fs::KParams &kp, cudaStream_t s, bool q, uint32_t *g) {
  (void)B; return fs::dispatch_kt<FS_CONSUMER_HIST, 16>(p, kp, s, q, g);
}
