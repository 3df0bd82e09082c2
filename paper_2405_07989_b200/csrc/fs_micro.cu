// fs_micro.cu -- microbenchmarks that measure the roofline denominators on the running B200
// (SURVEY Sec. 8(d) N3): INT32 lane-ops per clock per SM for the instruction classes the
// successor uses (IADD3 / LOP3 on the ALU pipe, IMAD on the FMA pipe, and a 1:1 mix), and the
// achievable HBM write bandwidth with coalesced 16 B streaming stores.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fsgpu.h"
#include "../../include/fsgpu_debug.h"

namespace {

constexpr int kMicroBlock = 256;

// 8 registers updated in a rotating chain x_i <- op(x_i, x_{i-1}): every intermediate value
// is consumed by the next instruction, so ptxas cannot fuse two PTX ops into one IADD3/LOP3
// and the SASS instruction count equals the PTX count (16 per inner iteration).
#define FS_OP_ADD(a, b) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b))
#define FS_OP_MAD(a, b) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(k))
#define FS_OP_XOR(a, b) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a) : "r"(b))
#define FS_ROUND(OPA, OPB) \
  OPA(x0, x7);             \
  OPB(x1, x0);             \
  OPA(x2, x1);             \
  OPB(x3, x2);             \
  OPA(x4, x3);             \
  OPB(x5, x4);             \
  OPA(x6, x5);             \
  OPB(x7, x6);

template <int MODE>
__global__ void __launch_bounds__(kMicroBlock) int_peak_kernel(uint32_t iters, uint32_t *sink,
                                                               unsigned long long *cycles) {
  uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
  const uint32_t k = blockIdx.x | 1u;
  __syncthreads();
  const long long t0 = clock64();
  for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (MODE == 0) {
        FS_ROUND(FS_OP_ADD, FS_OP_ADD)
      } else if (MODE == 1) {
        FS_ROUND(FS_OP_MAD, FS_OP_MAD)
      } else if (MODE == 2) {
        FS_ROUND(FS_OP_ADD, FS_OP_MAD)
      } else {
        FS_ROUND(FS_OP_XOR, FS_OP_XOR)
      }
    }
  }
  const long long t1 = clock64();
  const uint32_t v = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
  if (v == 0x12345678u) sink[0] = v;
  if (threadIdx.x == 0) atomicMax(cycles, (unsigned long long)(t1 - t0));
}

__global__ void __launch_bounds__(kMicroBlock) hbm_write_kernel(uint4 *out, uint64_t n16) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint4 v = make_uint4(threadIdx.x, blockIdx.x, 0x9e3779b9u, 0x7f4a7c15u);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) __stcs(out + i, v);
}

template <int MODE>
int run_int(double *ops_per_clk_sm, double *tops) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, int_peak_kernel<MODE>, kMicroBlock, 0);
  const int grid = sms * per_sm;
  uint32_t *sink = nullptr;
  unsigned long long *cyc = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess || cudaMalloc(&cyc, 8) != cudaSuccess) return FS_ENOMEM;
  const uint32_t iters = 1u << 16;
  int_peak_kernel<MODE><<<grid, kMicroBlock>>>(1024, sink, cyc);  // warm-up
  cudaMemset(cyc, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  int_peak_kernel<MODE><<<grid, kMicroBlock>>>(iters, sink, cyc);
  cudaEventRecord(b);
  if (cudaEventSynchronize(b) != cudaSuccess) return FS_ECUDA;
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long cycles = 0;
  cudaMemcpy(&cycles, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)grid * kMicroBlock * (double)iters * 16.0;
  *ops_per_clk_sm = ops / ((double)cycles * sms);
  *tops = ops / (ms * 1e-3) / 1e12;
  cudaFree(sink);
  cudaFree(cyc);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return FS_OK;
}

int run_hbm(uint64_t bytes, double *gbs) {
  uint4 *buf = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return FS_ENOMEM;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hbm_write_kernel, kMicroBlock, 0);
  const uint64_t n16 = bytes / 16;
  hbm_write_kernel<<<sms * per_sm, kMicroBlock>>>(buf, n16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    hbm_write_kernel<<<sms * per_sm, kMicroBlock>>>(buf, n16);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) return FS_ECUDA;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  *gbs = (double)(n16 * 16) / (best * 1e-3) / 1e9;
  cudaFree(buf);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return FS_OK;
}

}  // namespace

extern "C" int fsdbg_microbench(int kind, uint64_t param, double *result_out, double *aux_out) {
  if (!result_out || !aux_out) return FS_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return FS_ENODEV;
  }
  switch (kind) {
    case 0: return run_int<0>(result_out, aux_out);
    case 1: return run_int<1>(result_out, aux_out);
    case 2: return run_int<2>(result_out, aux_out);
    case 3: return run_int<3>(result_out, aux_out);
    case 4: *aux_out = (double)(param ? param : (8ull << 30)); return run_hbm(param ? param : (8ull << 30), result_out);
  }
  return FS_EINVAL;
}
