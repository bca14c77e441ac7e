// Probe: per-SM TMA load throughput from L2 (148 CTAs, one producer thread
// each) for 2-D boxes of `rows` x 512 B (the conv's B-stage shape) into a ring
// of 8 shared-memory slots; a slot is reused once its previous load completed.
//   tma_rate <rows per box> [iterations]
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void __launch_bounds__(32, 1) rate(const __grid_constant__ CUtensorMap map, int rows, int iters,
                                              int total_rows, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
  fence_barrier_init();
  const uint32_t bytes = (uint32_t)rows * 512u;
  uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long t0 = clock64();
  int r0 = (blockIdx.x * 97) % (total_rows - rows);
  for (int it = 0; it < iters; ++it) {
    const int s = it & 7;
    if (it >= 8) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
    mbar_arrive_expect_tx(&bar[s], bytes);
    tma_2d(sm + (size_t)s * bytes, &map, &bar[s], 0, r0);
    r0 += rows;
    if (r0 + rows > total_rows) r0 = 0;
  }
  for (int s = 0; s < 8; ++s) { mbar_wait(&bar[s], ph[s]); }
  out[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 16;
  const int iters = argc > 2 ? atoi(argv[2]) : 20000;
  const int total_rows = 8192;  // 4 MB source: L2-resident
  void* src;
  cudaMalloc(&src, (size_t)total_rows * 512);
  cudaMemset(src, 1, (size_t)total_rows * 512);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[2] = {512, (cuuint64_t)total_rows};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {256, (cuuint32_t)rows};  // 256 x 2-byte elements = 512 B per row
  cuuint32_t es[2] = {1, 1};
  dims[0] = 256;
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const size_t smem = 8 * (size_t)rows * 512;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rate<<<148, 32, smem>>>(map, rows, 100, total_rows, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<<<148, 32, smem>>>(map, rows, iters, total_rows, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148], mx = 0;
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)iters * rows * 512;
  printf("box %2d x 512 B (%5.1f KB), 8 in flight: %s  %.1f B/cycle per SM, %.2f TB/s chip\n", rows, rows * 0.5,
         cudaGetErrorString(e), bytes / (double)mx, bytes * 148 / (ms * 1e-3) / 1e12);
  return 0;
}
