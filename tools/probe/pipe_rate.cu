// Probe: MMA issue loop structure vs throughput (int8, M=128, N=128, 20 MMAs
// per stage, S-stage ring). No TMA: a "producer" lane re-arms full[s] as soon
// as the MMA commit frees empty[s]. Variants:
//   v0: one lane issues all MMAs, no barriers (ceiling)
//   v1: one lane, per-stage full wait + commit to empty (producer lane re-arms)
//   v2: converged warp + elect.sync per stage (the conv kernel's pattern)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

template <int V>
__global__ void __launch_bounds__(128, 1) pipe(int stages_total, int S, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = instr_desc_i8(128u, 128u);
  const uint64_t at = smem_desc(0, 2048, 128, kSwizzleNone), bt = smem_desc(0, 128 * 16, 128, kSwizzleNone);
  const uint32_t a4 = (smem_u32(sm) & 0x3FFFFu) >> 4, b4 = (smem_u32(sm + 32768) & 0x3FFFFu) >> 4;
  auto issue_stage = [&](int st) {
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
      for (int q = 0; q < 10; ++q) {
        const int L = q == 0 ? 0 : (q < 3 ? 1 : (q < 6 ? 2 : 3));
        mma_i8(tmem + (uint32_t)(L * 128), at + a4 + (uint32_t)((q & 3) * 128 + s2 * 256),
               bt + b4 + (uint32_t)(((q >> 2) & 3) * 128 + s2 * 256), idesc, 1u);
      }
  };
  if (warp == 0 && V > 0) {  // producer lane: re-arm full[s] once empty[s] completes
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int k = 0; k < stages_total; ++k) {
        mbar_wait(&empty[stage], ph ^ 1);
        mbar_arrive(&full[stage]);
        if (++stage == S) { stage = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    unsigned long long t0 = clock64();
    if (V == 0) {
      if (lane == 0) {
        for (int k = 0; k < stages_total; ++k) issue_stage(k);
        mma_commit(&done);
      }
    } else if (V == 1) {
      if (lane == 0) {
        int stage = 0;
        uint32_t ph = 0;
        for (int k = 0; k < stages_total; ++k) {
          mbar_wait(&full[stage], ph);
          tc_fence_after();
          issue_stage(k);
          mma_commit(&empty[stage]);
          if (++stage == S) { stage = 0; ph ^= 1; }
        }
        mma_commit(&done);
      }
    } else {
      int stage = 0;
      uint32_t ph = 0;
      for (int k = 0; k < stages_total; ++k) {
        mbar_wait(&full[stage], ph);
        tc_fence_after();
        if (elect_one()) {
          issue_stage(k);
          mma_commit(&empty[stage]);
          if (k == stages_total - 1) mma_commit(&done);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; ph ^= 1; }
      }
    }
    mbar_wait(&done, 0);
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int V>
void run(int stages_total, int S) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(pipe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
  pipe<V><<<148, 128, 65536 + 2048>>>(stages_total, S, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pipe<V><<<148, 128, 65536 + 2048>>>(stages_total, S, d);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148], mx = 0;
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("v%d S=%d: %s  %.1f cyc/MMA  %.3f ms\n", V, S, cudaGetErrorString(e), (double)mx / (stages_total * 20.0), ms);
  cudaFree(d);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int n = argc > 1 ? atoi(argv[1]) : 4000;
  run<0>(n, 3);
  run<1>(n, 3);
  run<2>(n, 3);
  run<1>(n, 6);
  run<2>(n, 6);
  run<2>(n, 2);
  return 0;
}
