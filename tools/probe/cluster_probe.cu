// Probe: cluster rank mapping and multicast bulk-copy semantics on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

__global__ void probe(int* out, const int* src) {
  __shared__ __align__(1024) int buf[256];
  __shared__ uint64_t bar;
  uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = -1;
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 1024);
    // rank r loads half r of src (512 B) multicast to both CTAs
    bulk_load_multicast(reinterpret_cast<char*>(buf) + rank * 512, reinterpret_cast<const char*>(src) + rank * 512, 512, &bar, 3);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  out[blockIdx.x * 260 + 0] = blockIdx.x;
  out[blockIdx.x * 260 + 1] = rank;
  out[blockIdx.x * 260 + 2] = (int)smem_u32(buf);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[blockIdx.x * 260 + 4 + i] = buf[i];
  cluster_sync();
}

int main() {
  int *out, *src;
  cudaMalloc(&out, 8 * 260 * 4);
  cudaMalloc(&src, 256 * 4);
  int h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1000 + i;
  cudaMemcpy(src, h, 1024, cudaMemcpyHostToDevice);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(8);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, probe, out, (const int*)src);
  printf("launch %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize();
  printf("sync %s\n", cudaGetErrorString(e));
  int ho[8 * 260];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  for (int b = 0; b < 8; ++b) {
    int bad = 0;
    for (int i = 0; i < 256; ++i) bad += ho[b * 260 + 4 + i] != 1000 + i;
    printf("block %d rank %d smem 0x%x bad %d first %d %d last %d\n", ho[b * 260], ho[b * 260 + 1], ho[b * 260 + 2], bad,
           ho[b * 260 + 4], ho[b * 260 + 4 + 128], ho[b * 260 + 4 + 255]);
  }
  return 0;
}
