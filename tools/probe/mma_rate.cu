// Probe: steady-state tcgen05.mma issue rate for the shapes the conv kernel
// uses (garbage smem operands; only timing matters). One CTA per SM, one
// thread issues `iters` MMAs back to back, then commits and waits.
//   kind 0: i8  cta_group::1 M=128 N=n, 10 MMAs/step over 4 accumulators (Ozaki levels)
//   kind 1: f16 cta_group::1 M=128 N=n
//   kind 2: i8  cta_group::2 M=256 N=n (cluster of 2, leader issues)
//   kind 3: kind 0 plus a concurrent bulk-copy writer (4 x 16 KB in flight) into other smem
//   kind 4: the bulk-copy writer alone
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

template <int KIND>
__global__ void __launch_bounds__(128, 1) rate(int n, int iters, unsigned long long* out, const uint8_t* gsrc,
                                               volatile int* stop, int a_sbo) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[4];
  __shared__ int done_flag;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const bool cg2 = KIND == 2 || KIND == 5;
  const uint32_t rank = cg2 ? cluster_ctarank() : 0;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1);
    done_flag = 0;
    fence_barrier_init();
  }
  if (warp == 0) {
    if (cg2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(&slot, 512);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (cg2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if ((KIND == 3 || KIND == 4) && threadIdx.x == 32) {
    // writer: keep 4 x 16 KB bulk copies in flight into sm[65536..131072)
    unsigned long long t0 = clock64(), bytes = 0;
    uint32_t ph[4] = {0, 0, 0, 0};
    int pending[4] = {0, 0, 0, 0};
    const int ncopies = KIND == 4 ? iters : 1 << 30;
    for (int c = 0; c < ncopies; ++c) {
      const int s2 = c & 3;
      if (pending[s2]) { mbar_wait(&cbar[s2], ph[s2]); ph[s2] ^= 1; pending[s2] = 0; bytes += 16384; }
      if (KIND == 3 && *(volatile int*)&done_flag) break;
      mbar_arrive_expect_tx(&cbar[s2], 16384);
      bulk_load(sm + 65536 + s2 * 16384, gsrc + (size_t)((c * 16384) & ((1 << 20) - 1)), 16384, &cbar[s2]);
      pending[s2] = 1;
    }
    for (int s2 = 0; s2 < 4; ++s2)
      if (pending[s2]) mbar_wait(&cbar[s2], ph[s2]);
    unsigned long long t1 = clock64();
    out[148 + blockIdx.x] = (unsigned long long)((double)bytes / (double)(t1 - t0) * 1000.0);  // B/kclk
  }
  if (KIND != 4 && threadIdx.x == 0 && rank == 0) {
    const uint32_t a4 = (smem_u32(sm) & 0x3FFFFu) >> 4, b4 = (smem_u32(sm + 32768) & 0x3FFFFu) >> 4;
    const uint64_t at = smem_desc(0, 4096, (uint32_t)a_sbo, kSwizzleNone), bt = smem_desc(0, (uint32_t)n * 16u, 128, kSwizzleNone);
    const uint32_t m = (cg2 || KIND == 5) ? 256u : 128u;
    const uint32_t idesc = (KIND == 1 || KIND == 5) ? instr_desc(1u, m, (uint32_t)n) : instr_desc_i8(m, (uint32_t)n);
    const int nacc = (KIND == 1) ? 512 / n : (4 * n <= 512 ? 4 : 512 / n);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (KIND == 1 || KIND == 5) {  // 8 bf16 MMAs per iteration, 2 accumulators
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint64_t a = at + a4 + (uint32_t)((q & 1) * 2), b = bt + b4 + (uint32_t)((q & 1) * 2);
          if (KIND == 5) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (uint32_t)((q & 1) * n)),
                         "l"(a), "l"(b), "r"(idesc), "r"(1u) : "memory");
          } else {
            mma_bf16(tmem + (uint32_t)((q & 1) * n), a, b, idesc, 1u);
          }
        }
      } else {
        // 10 MMAs / K step into nacc accumulators (level L = i + j)
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          const int L = q == 0 ? 0 : (q < 3 ? 1 : (q < 6 ? 2 : 3));
          const uint32_t d = tmem + (uint32_t)((L % nacc) * n);
          const uint64_t a = at + a4 + (uint32_t)((q & 3) * 128), b = bt + b4 + (uint32_t)(((q >> 2) & 3) * 128);
          if (cg2) mma_i8_cg2(d, a, b, idesc, 1u);
          else mma_i8(d, a, b, idesc, 1u);
        }
      }
    }
    if (cg2)
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    else
      mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    *(volatile int*)&done_flag = 1;
  }
  if (cg2 && threadIdx.x == 0 && rank == 1) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  if (cg2) cluster_sync();
  if (warp == 0) {
    if (cg2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      tmem_dealloc(tmem, 512);
  }
}

template <int KIND>
void run(int n, int iters, int a_sbo = 128) {
  unsigned long long* d;
  const int grid = 148;
  cudaMalloc(&d, 2 * grid * sizeof(unsigned long long));
  cudaMemset(d, 0, 2 * grid * sizeof(unsigned long long));
  uint8_t* g;
  cudaMalloc(&g, 1 << 20);
  cudaMemset(g, 1, 1 << 20);
  int* stop;
  cudaMalloc(&stop, 4);
  cudaFuncSetAttribute(rate<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 2048);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 131072 + 2048;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (KIND == 2 || KIND == 5) ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, rate<KIND>, n, iters, d, (const uint8_t*)g, stop, a_sbo);  // warm
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, rate<KIND>, n, iters, d, (const uint8_t*)g, stop, a_sbo);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double wr = 0;
  for (int i = 0; i < grid; ++i) wr += h[148 + i] / 1000.0 / grid;
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double nmma = (double)iters * ((KIND == 1 || KIND == 5) ? 8 : 10);
  const double m = (KIND == 2 || KIND == 5) ? 256 : 128;
  const double kel = (KIND == 1 || KIND == 5) ? 16 : 32;
  const int issuers = (KIND == 2 || KIND == 5) ? grid / 2 : grid;
  const double ops = 2.0 * m * n * kel * nmma * issuers;
  printf("sbo %d kind %d n %3d: %s  %.1f cyc/MMA (leader)  %.0f TOPS over %.3f ms  writer %.1f B/clk\n", a_sbo, KIND, n,
         cudaGetErrorString(e), (double)mx / nmma, ops / (ms * 1e-3) / 1e12, ms, wr);
  cudaFree(d);
  cudaFree(g);
  cudaFree(stop);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  if (argc > 2) {  // long run (power-capped steady state)
    run<0>(128, iters);
    return 0;
  }
  run<5>(256, iters, 128);
  run<5>(256, iters, 192);
  run<1>(256, iters, 128);
  run<0>(128, iters, 128);
  run<0>(128, iters, 192);
  run<2>(128, iters, 128);
  run<2>(128, iters, 192);
  return 0;
}
