// Probe: cycles per tcgen05.mma (cta_group::2, M = 256) by kind, N and the
// number of accumulators the MMAs rotate over, with the conv kernel's
// halo-mode A geometry (K-major, no swizzle, SBO = halo row pitch, LBO = one
// channel-group plane). Garbage operands. The leader CTA's warp 0 runs the
// loop converged; elect.sync inside the asm issues (ptxas emits a bare
// UTC*MMA), operands are formed before the loop, so the loop is pure issue.
//   mma_geom [iters]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

template <int KIND>
__device__ __forceinline__ void mma_e(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  if constexpr (KIND == 0)
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, 1;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                 : "memory");
  else if constexpr (KIND == 1)
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                 : "memory");
  else
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, 1;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
                 : "memory");
}

template <int KIND, int NACC>
__global__ void __launch_bounds__(128, 1) rate(uint32_t n, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 200000 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
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
  const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);
  if (warp == 0 && rank == 0) {
    const uint32_t lbo = 10368, sbo = 192;
    const uint32_t a4 = ((smem_u32(sm) & 0x3FFFFu) >> 4) + 2;
    const uint32_t b4 = (smem_u32(sm + 160000) & 0x3FFFFu) >> 4;
    const uint64_t at = smem_desc(0, lbo, sbo, kSwizzleNone), bt = smem_desc(0, n / 2 * 16, 128, kSwizzleNone);
    const uint32_t idesc = KIND == 0 ? instr_desc_i8(256u, n) : instr_desc(KIND == 1 ? 1u : 2u, 256u, n);
    const uint32_t a_ks = 2 * (lbo >> 4);
    const uint64_t A0 = at + a4, A1 = A0 + a_ks, A2 = A1 + a_ks, A3 = A2 + a_ks;
    const uint64_t B0 = bt + b4, B1 = B0 + 128, B2 = B1 + 128, B3 = B2 + 128;
    const uint32_t D0 = tmem, D1 = tmem + (1 % NACC) * n, D2 = tmem + (2 % NACC) * n, D3 = tmem + (3 % NACC) * n;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      mma_e<KIND>(D0, A0, B0, idesc);
      mma_e<KIND>(D1, A1, B1, idesc);
      mma_e<KIND>(D2, A2, B2, idesc);
      mma_e<KIND>(D3, A3, B3, idesc);
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
    mbar_wait(&bar, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  if (warp == 0 && rank == 1) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int KIND, int NACC>
static void run(uint32_t n, int iters) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(rate<KIND, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, rate<KIND, NACC>, n, 200, d);
  cudaLaunchKernelEx(&cfg, rate<KIND, NACC>, n, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; i += 2) mx = h[i] > mx ? h[i] : mx;
  printf("kind %d N %3u accumulators %d: %s  %.1f cyc/MMA (nominal %.0f)\n", KIND, n, NACC, cudaGetErrorString(e),
         (double)mx / (4.0 * iters), n / 2.0);
  cudaFree(d);
}

template <int KIND>
static void sweep(int iters) {
  for (uint32_t n : {64u, 128u, 256u}) {
    run<KIND, 1>(n, iters);
    run<KIND, 2>(n, iters);
    if (n <= 128) run<KIND, 4>(n, iters);
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  sweep<0>(iters);
  sweep<1>(iters);
  sweep<2>(iters);
  return 0;
}
