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

// One thread per (b, g, p): the 16 K-elements of group g at pixel p -> 4
// digit planes (digit, b, g, p, [ncol x] 16 B). Without a change of basis a
// group is 16/nb channels x nb blades; with one (bs.on) each pixel yields ncol
// rows, row c holding 16/w channels x the w transformed components
// x'[c*w + r] = sum_I T[c*w + r][I] x[I] (exact in fp64).
__global__ void slice_input_kernel(const float* __restrict__ x, const unsigned* __restrict__ amax,
                                   int8_t* __restrict__ out, float* __restrict__ scale, int nb, long long B,
                                   int C, long long P, int G, Basis bs) {
  const long long total = B * G * P;
  const int ncol = bs.on ? bs.ncol : 1;
  const int w = bs.on ? bs.w : nb;
  const int cpg = 16 / w;  // channels per group
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pp = i % P;
    const long long bg = i / P;
    const int g = (int)(bg % G);
    const long long b = bg / G;
    const float amx = __uint_as_float(__ldg(amax + b));
    const float sc = pow2_scale_for(bs.on ? 2.f * amx : amx);  // |x'| <= 2 max|x|
    if (g == 0 && pp == 0) scale[b] = sc;
    const double inv = 1.0 / (double)sc;  // exact (power of two)
    for (int col = 0; col < ncol; ++col) {
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
        for (int r = 0; r < w; ++r) {
          double xv;
          if (bs.on) {
            xv = 0.0;
            for (int I = 0; I < nb; ++I) {
              const int t = bs.T[(col * w + r) * 8 + I];
              if (t) xv += t > 0 ? (double)v[I] : -(double)v[I];
            }
          } else {
            xv = (double)v[r];
          }
          int8_t d[4];
          digits_b256_d<4>(xv * inv, d);
#pragma unroll
          for (int k = 0; k < 4; ++k) dg[k][cl * w + r] = d[k];
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t wd[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          wd[q] = (uint32_t)(uint8_t)dg[k][4 * q] | ((uint32_t)(uint8_t)dg[k][4 * q + 1] << 8) |
                  ((uint32_t)(uint8_t)dg[k][4 * q + 2] << 16) | ((uint32_t)(uint8_t)dg[k][4 * q + 3] << 24);
        reinterpret_cast<uint4*>(out)[((long long)k * total + i) * ncol + col] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
      }
    }
  }
}

cudaError_t launch_slice_input(const float* x, const unsigned* amax, int8_t* digits, float* scale, int nb,
                               long long B, int C, long long P, int G, const Basis& bs, cudaStream_t s) {
  const long long total = B * G * P;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  slice_input_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, amax, digits, scale, nb, B, C, P, G, bs);
  count_launch();
  return cudaGetLastError();
}

// Per output column n of the B operand: power-of-two scale covering
// max_k |W[n, k]|. Without a change of basis W is the expanded filter
// (conv.py:188-202, entries are signed filter values); with one, n = (co, r)
// and W[n, (q, ci, m)] = R(f[ci, co, q])[r][m] (see expand.cu).
__global__ void weight_colscale_kernel(Sig sg, const float* __restrict__ f, int C_in, int C_out, int Q,
                                       Basis bs, float* __restrict__ w_scale) {
  const int nb = 1 << sg.k;
  const int w = bs.on ? bs.w : nb;
  const int n = blockIdx.x;
  const int co = n / w, t = n % w;
  float m = 0.f;
  if (co < C_out) {
    for (int idx = threadIdx.x; idx < C_in * w * Q; idx += blockDim.x) {
      const int q = idx % Q;
      const int j = (idx / Q) % w;
      const int ci = idx / (Q * w);
      const double e = bs.on ? basis_entry(sg, bs, f, C_in, C_out, Q, co, t, ci, j, q)
                             : (double)expanded_entry(sg, f, nb, C_in, C_out, Q, co, t, ci, j, q);
      m = fmaxf(m, (float)fabs(e));
    }
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) m = fmaxf(m, red[ww]);
    // float rounding of |e| may round down: one more power of two of headroom is free
    w_scale[n] = pow2_scale_for(m * 1.0000002f);
  }
}

cudaError_t launch_weight_colscale(const int* g, const ConvPlan& pl, const float* f, int C_in, int C_out,
                                   float* w_scale, cudaStream_t s) {
  const int N_pad = pl.n_ntiles * pl.n_tile;
  Sig sg{{0, 0, 0}, pl.ka};
  for (int i = 0; i < pl.ka; ++i) sg.g[i] = g[i];
  weight_colscale_kernel<<<N_pad, 256, 0, s>>>(sg, f, C_in, C_out, pl.Q, pl.bs, w_scale);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cl
