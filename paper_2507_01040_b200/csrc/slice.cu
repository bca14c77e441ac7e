// slice.cu -- operand preparation for the fp32-accurate mode (kPrecFp32).
//
// Each fp32 value v is written as  v = s * sum_i d_i 2^(-7-8(i-1))  with a
// power-of-two scale s (per sample for activations, per output column for
// the expanded filter) and 4 balanced base-256 int8 digits (|error| <= s 2^-32,
// finer than the fp32 operands themselves near the scale). Digit products
// d_i w_j are then summed EXACTLY by tcgen05 kind::i8 into s32 TMEM
// accumulators, one per level L = i + j <= 3 (0-based; see conv_tc.cu);
// the truncating fp32 accumulation of the tf32/bf16 tensor-core paths never
// touches the result.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace cl {

__global__ void absmax_kernel(const float* __restrict__ x, long long per_sample, unsigned* __restrict__ amax) {
  const int b = blockIdx.y;
  const float* xs = x + (long long)b * per_sample;
  float m = 0.f;
  // samples need not start 16-byte aligned (1-D tensors): scalar head, float4 body, scalar tail
  long long head = (long long)((16 - (reinterpret_cast<uintptr_t>(xs) & 15)) & 15) / 4;
  if (head > per_sample) head = per_sample;
  const long long n4 = (per_sample - head) / 4;
  const float4* x4 = reinterpret_cast<const float4*>(xs + head);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n4; i += nth) {
    const float4 v = __ldg(x4 + i);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  if (tid < head) m = fmaxf(m, fabsf(xs[tid]));
  for (long long i = head + n4 * 4 + tid; i < per_sample; i += nth) m = fmaxf(m, fabsf(xs[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(amax + b, __float_as_uint(m));
}

cudaError_t launch_sample_absmax(const float* x, long long B, long long per_sample, unsigned* amax,
                                 cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(unsigned) * B, s);
  if (e != cudaSuccess) return e;
  long long want = (per_sample / 4 + 255) / 256;
  long long per = std::max<long long>(1, std::min<long long>(want, ((long long)num_sms() * 8 + B - 1) / B));
  dim3 grid((unsigned)per, (unsigned)B);
  absmax_kernel<<<grid, 256, 0, s>>>(x, per_sample, amax);
  count_launch();
  return cudaGetLastError();
}

// One thread per (b, g, p): the 16 K-elements of group g at pixel p
// (16/nb channels x nb blades) -> 4 digit planes (digit, b, g, p, 16 B).
__global__ void slice_input_kernel(const float* __restrict__ x, const unsigned* __restrict__ amax,
                                   int8_t* __restrict__ out, float* __restrict__ scale, int nb, long long B,
                                   int C, long long P, int G) {
  const long long total = B * G * P;
  const int cpg = 16 / nb;  // channels per group
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pp = i % P;
    const long long bg = i / P;
    const int g = (int)(bg % G);
    const long long b = bg / G;
    const float sc = pow2_scale_for(__uint_as_float(__ldg(amax + b)));
    if (g == 0 && pp == 0) scale[b] = sc;
    const float inv = 1.f / sc;  // exact (power of two)
    int8_t dg[4][16];
    for (int cl = 0; cl < cpg; ++cl) {
      const int c = g * cpg + cl;
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = 0.f;
      if (c < C) {
        const float* src = x + ((b * C + c) * P + pp) * nb;
        if (nb == 2) {
          const float2 q = __ldg(reinterpret_cast<const float2*>(src));
          v[0] = q.x; v[1] = q.y;
        } else {
          const float4 q0 = __ldg(reinterpret_cast<const float4*>(src));
          v[0] = q0.x; v[1] = q0.y; v[2] = q0.z; v[3] = q0.w;
          if (nb == 8) {
            const float4 q1 = __ldg(reinterpret_cast<const float4*>(src) + 1);
            v[4] = q1.x; v[5] = q1.y; v[6] = q1.z; v[7] = q1.w;
          }
        }
      }
      for (int j = 0; j < nb; ++j) {
        int8_t d[4];
        digits_b256<4>(v[j] * inv, d);
#pragma unroll
        for (int k = 0; k < 4; ++k) dg[k][cl * nb + j] = d[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4 u;
      u.x = (uint32_t)(uint8_t)dg[k][0] | ((uint32_t)(uint8_t)dg[k][1] << 8) | ((uint32_t)(uint8_t)dg[k][2] << 16) | ((uint32_t)(uint8_t)dg[k][3] << 24);
      u.y = (uint32_t)(uint8_t)dg[k][4] | ((uint32_t)(uint8_t)dg[k][5] << 8) | ((uint32_t)(uint8_t)dg[k][6] << 16) | ((uint32_t)(uint8_t)dg[k][7] << 24);
      u.z = (uint32_t)(uint8_t)dg[k][8] | ((uint32_t)(uint8_t)dg[k][9] << 8) | ((uint32_t)(uint8_t)dg[k][10] << 16) | ((uint32_t)(uint8_t)dg[k][11] << 24);
      u.w = (uint32_t)(uint8_t)dg[k][12] | ((uint32_t)(uint8_t)dg[k][13] << 8) | ((uint32_t)(uint8_t)dg[k][14] << 16) | ((uint32_t)(uint8_t)dg[k][15] << 24);
      reinterpret_cast<uint4*>(out)[(long long)k * total + i] = u;
    }
  }
}

cudaError_t launch_slice_input(const float* x, const unsigned* amax, int8_t* digits, float* scale, int nb,
                               long long B, int C, long long P, int G, cudaStream_t s) {
  const long long total = B * G * P;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  slice_input_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, amax, digits, scale, nb, B, C, P, G);
  count_launch();
  return cudaGetLastError();
}

// Per output column n = (co, t) of the expanded filter: power-of-two scale
// covering max_k |W[n, k]| (W entries are signed filter values, conv.py:188-202).
__global__ void weight_colscale_kernel(int g0, int g1, int g2, int k, const float* __restrict__ f, int C_in,
                                       int C_out, int Q, int N_pad, float* __restrict__ w_scale) {
  const int nb = 1 << k;
  const int gg[3] = {g0, g1, g2};
  const int n = blockIdx.x;
  const int co = n / nb, t = n % nb;
  float m = 0.f;
  if (co < C_out) {
    for (int idx = threadIdx.x; idx < C_in * nb * Q; idx += blockDim.x) {
      const int q = idx % Q;
      const int j = (idx / Q) % nb;
      const int ci = idx / (Q * nb);
      const int i = t ^ j;
      if (blade_coeff(i, j, gg, k) != 0)
        m = fmaxf(m, fabsf(__ldg(f + (((long long)i * C_in + ci) * C_out + co) * Q + q)));
    }
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    w_scale[n] = pow2_scale_for(m);
  }
}

cudaError_t launch_weight_colscale(const int* g, const ConvPlan& pl, const float* f, int C_in, int C_out,
                                   float* w_scale, cudaStream_t s) {
  const int N_pad = pl.n_ntiles * pl.n_tile;
  weight_colscale_kernel<<<N_pad, 256, 0, s>>>(g[0], g[1], g[2], pl.ka, f, C_in, C_out, pl.Q, N_pad, w_scale);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cl
