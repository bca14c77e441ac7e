// Probe: sustained (power-capped) int8 MMA throughput of the fp32 mode's K step
// in two issue shapes with the SAME multiply-accumulate work (garbage smem
// operands, only timing and power matter). cta_group::2, M = 256, leader issues.
//   scheme 0 (shipped): 10 MMAs of N = 128, one per digit pair (i, j), into
//            level block L = i + j (4 blocks x 128 TMEM columns).
//   scheme 1: B digit planes concatenated along N so one A digit feeds up to
//            two level blocks per MMA: 4 MMAs of N = 256 + 2 of N = 128
//            (A_0 x [B0|B1], A_0 x [B2|B3], A_1 x [B0|B1], A_2 x [B0|B1],
//            A_1 x B2, A_3 x B0): 6 A-operand reads per K step instead of 10.
// Usage: mma_concat <ksteps> [scheme...]; prints TOPS (int8) over the launch.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

__global__ void __launch_bounds__(128, 1) rate(int scheme, long long ksteps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (i + 7919u * rank) * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    // A: 4 digit planes x 128 rows x 32 B (K-major, no swizzle, LBO 2048 = one 16-byte K chunk of 128 rows)
    const uint32_t a4 = (smem_u32(sm) & 0x3FFFFu) >> 4;
    const uint32_t b4 = (smem_u32(sm + 16384) & 0x3FFFFu) >> 4;
    const uint64_t at = smem_desc(0, 2048, 128, kSwizzleNone);
    const uint64_t bt64 = smem_desc(0, 64 * 16, 128, kSwizzleNone);    // 64 B rows per CTA (N = 128)
    const uint64_t bt128 = smem_desc(0, 128 * 16, 128, kSwizzleNone);  // 128 B rows per CTA (N = 256)
    const uint32_t id128 = instr_desc_i8(256u, 128u), id256 = instr_desc_i8(256u, 256u);
    unsigned long long t0 = clock64();
    for (long long it = 0; it < ksteps; ++it) {
      if (scheme == 0) {
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          const int L = q == 0 ? 0 : (q < 3 ? 1 : (q < 6 ? 2 : 3));
          const uint64_t a = at + a4 + (uint32_t)((q & 3) * 256);
          const uint64_t b = bt64 + b4 + (uint32_t)(((q >> 2) & 3) * 128);
          mma_i8_cg2(tmem + (uint32_t)(L * 128), a, b, id128, 1u);
        }
      } else {
        // B regions per CTA: R0 = 128 rows (4 KB), R1 = 128 rows, R2 = 64 rows, R3 = 64 rows
        const uint64_t r0 = bt128 + b4, r1 = bt128 + b4 + 256, r2 = bt64 + b4 + 512, r3 = bt64 + b4 + 640;
        mma_i8_cg2(tmem + 0, at + a4, r0, id256, 1u);          // A0 x [B0|B1] -> L0, L1
        mma_i8_cg2(tmem + 256, at + a4, r1, id256, 1u);        // A0 x [B2|B3] -> L2, L3
        mma_i8_cg2(tmem + 128, at + a4 + 256, r0, id256, 1u);  // A1 x [B0|B1] -> L1, L2
        mma_i8_cg2(tmem + 256, at + a4 + 512, r0, id256, 1u);  // A2 x [B0|B1] -> L2, L3
        mma_i8_cg2(tmem + 384, at + a4 + 256, r2, id128, 1u);  // A1 x B2 -> L3
        mma_i8_cg2(tmem + 384, at + a4 + 768, r3, id128, 1u);  // A3 x B0 -> L3
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  if (threadIdx.x == 0 && rank == 1) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

static void run(int scheme, long long ksteps) {
  unsigned long long* d;
  const int grid = 148;
  cudaMalloc(&d, grid * sizeof(unsigned long long));
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 65536 + 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, rate, scheme, ksteps, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 256 * 1280 * 32 * (double)ksteps * (grid / 2);
  printf("scheme %d: %s  %.0f TOPS (int8) over %.0f ms\n", scheme, cudaGetErrorString(e), ops / (ms * 1e-3) / 1e12, ms);
  cudaFree(d);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const long long ksteps = argc > 1 ? atoll(argv[1]) : 2000000;
  if (argc > 2) {
    for (int i = 2; i < argc; ++i) run(atoi(argv[i]), ksteps);
  } else {
    run(0, 20000);  // warm
    for (int r = 0; r < 3; ++r) { run(0, ksteps); run(1, ksteps); }
  }
  return 0;
}
