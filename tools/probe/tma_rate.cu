// Probe: per-SM TMA load throughput from L2 (148 CTAs, one producer thread
// each) for 2-D boxes of `rows` x `row_bytes` (the conv's B stage: rows of
// 512 B) into a ring of `slots` shared-memory slots; a slot is reused once its
// previous load completed.
//   tma_rate <rows per box> [iterations] [row_bytes 512|1024|2048] [slots <= 16] [issuing warps <= 4]
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

__global__ void __launch_bounds__(128, 1) rate(const __grid_constant__ CUtensorMap map, int rows, int iters,
                                              int total_rows, unsigned long long* out, int row_bytes, int slots, int lanes) {
  extern __shared__ __align__(1024) uint8_t smem_all[];
  __shared__ uint64_t bars[8][16];
  // issuers: lane 0 of `warps` warps, or lanes 0..lanes-1 of warp 0 (each its own ring)
  const int w = lanes > 1 ? (int)(threadIdx.x & 31) : (int)(threadIdx.x >> 5);
  if (lanes > 1 ? (threadIdx.x >= (unsigned)lanes) : ((threadIdx.x & 31) != 0)) return;
  uint64_t* bar = bars[w];
  uint8_t* sm = smem_all + (size_t)w * slots * rows * row_bytes;
  for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1);
  fence_barrier_init();
  const uint32_t bytes = (uint32_t)rows * (uint32_t)row_bytes;
  uint32_t ph[16] = {};
  unsigned long long t0 = clock64();
  int r0 = (blockIdx.x * 97 + w * 1031) % (total_rows - rows);
  for (int it = 0; it < iters; ++it) {
    const int s = it % slots;
    if (it >= slots) { mbar_wait(&bar[s], ph[s]); ph[s] ^= 1; }
    mbar_arrive_expect_tx(&bar[s], bytes);
    tma_2d(sm + (size_t)s * bytes, &map, &bar[s], 0, r0);
    r0 += rows;
    if (r0 + rows > total_rows) r0 = 0;
  }
  for (int s = 0; s < slots && s < iters; ++s) { mbar_wait(&bar[s], ph[s]); }
  if (w == 0) out[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 16;
  const int iters = argc > 2 ? atoi(argv[2]) : 20000;
  const int row_bytes = argc > 3 ? atoi(argv[3]) : 512;
  const int slots = argc > 4 ? atoi(argv[4]) : 8;
  const int warps = argc > 5 ? atoi(argv[5]) : 1;  // issuing threads per SM (one per warp)
  const int lanes = argc > 6 ? atoi(argv[6]) : 1;  // or: this many lanes of ONE warp issue (warps = 1)
  const int total_rows = (4 << 20) / row_bytes;  // 4 MB source: L2-resident
  void* src;
  cudaMalloc(&src, (size_t)4 << 20);
  cudaMemset(src, 1, (size_t)4 << 20);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)row_bytes / 8, (cuuint64_t)total_rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {(cuuint32_t)row_bytes / 8, (cuuint32_t)rows};  // 8-byte elements
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const int issuers = lanes > 1 ? lanes : warps;
  const size_t smem = (size_t)issuers * slots * rows * row_bytes;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rate<<<148, 32 * warps, smem>>>(map, rows, 100, total_rows, d, row_bytes, slots, lanes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<<<148, 32 * warps, smem>>>(map, rows, iters, total_rows, d, row_bytes, slots, lanes);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148], mx = 0;
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)iters * rows * row_bytes * issuers;
  printf("%d issuer(s)%s: box %3d x %4d B (%5.1f KB), %2d in flight each: %s  %.1f B/cycle per SM (%.1f cycles per row), %.2f TB/s chip\n",
         issuers, lanes > 1 ? " (lanes of one warp)" : "", rows, row_bytes, rows * row_bytes / 1024.0, slots, cudaGetErrorString(e), bytes / (double)mx,
         (double)mx / ((double)iters * rows), bytes * 148 / (ms * 1e-3) / 1e12);
  return 0;
}
