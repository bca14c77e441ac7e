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
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace cl {

// Per-sample max |x| over the FINITE values, and a per-sample flag when the
// sample holds Inf / NaN (those are sliced as 0 and their receptive fields
// poisoned afterwards, poison_nonfinite_kernel). Block (j, b) reduces the j-th
// contiguous chunk of kAbsmaxU float4 per thread of sample b (many waves, one
// atomic per block). The grid is 1-D over (sample, chunk) pairs -- any B (a
// linear layer can have far more than gridDim.y's 65535 samples); launches of
// more than 2^31-1 blocks are split by the host with `blk0`.
constexpr int kAbsmaxU = 8;
__global__ void __launch_bounds__(256) absmax_kernel(const float* __restrict__ x, long long per_sample,
                                                     long long per, long long blk0, unsigned* __restrict__ amax,
                                                     unsigned* __restrict__ flags) {
  const long long bid = blk0 + (long long)blockIdx.x;
  const long long b = bid / per;
  const long long chunk = bid - b * per;
  const float* xs = x + b * per_sample;
  unsigned m = 0;    // max finite |x| as float bits
  unsigned any = 0;  // max |x| as float bits, NaN-sticky: >= 0x7f800000 iff a value is non-finite
  auto take = [&](float v) {
    m = max(m, finite_abs_bits(v));
    any = max(any, abs_bits(v));
  };
  // samples need not start 16-byte aligned (1-D tensors): scalar head, float4 body, scalar tail
  long long head = (long long)((16 - (reinterpret_cast<uintptr_t>(xs) & 15)) & 15) / 4;
  if (head > per_sample) head = per_sample;
  const long long n4 = (per_sample - head) / 4;
  const float4* x4 = reinterpret_cast<const float4*>(xs + head);
  const long long base = chunk * (256 * kAbsmaxU) + threadIdx.x;
  float4 v[kAbsmaxU];
#pragma unroll
  for (int u = 0; u < kAbsmaxU; ++u)
    v[u] = base + u * 256 < n4 ? __ldcs(x4 + base + u * 256) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int u = 0; u < kAbsmaxU; ++u) {
    take(v[u].x); take(v[u].y); take(v[u].z); take(v[u].w);
  }
  if (chunk == 0) {
    if (threadIdx.x < head) take(xs[threadIdx.x]);
    for (long long i = head + n4 * 4 + threadIdx.x; i < per_sample; i += blockDim.x) take(xs[i]);
  }
  __shared__ unsigned red[8], redn[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    any = max(any, __shfl_xor_sync(0xffffffffu, any, o));
  }
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = m; redn[threadIdx.x >> 5] = any; }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < 8; ++w) { m = max(m, red[w]); any = max(any, redn[w]); }
    atomicMax(amax + b, m);
    if (any >= 0x7f800000u) atomicOr(flags + b, 1u);
  }
}

cudaError_t launch_sample_absmax(const float* x, long long B, long long per_sample, unsigned* amax, unsigned* flags,
                                 cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  cudaError_t e;
  if (flags == amax + B) {  // adjacent arrays (the conv workspace layout): one memset
    e = cudaMemsetAsync(amax, 0, sizeof(unsigned) * 2 * B, s);
  } else if ((e = cudaMemsetAsync(amax, 0, sizeof(unsigned) * B, s)) == cudaSuccess) {
    e = cudaMemsetAsync(flags, 0, sizeof(unsigned) * B, s);
  }
  if (e != cudaSuccess) return e;
  const long long per = std::max<long long>(1, (per_sample / 4 + 256 * kAbsmaxU - 1) / (256 * kAbsmaxU));
  const long long total = per * B;
  for (long long b0 = 0; b0 < total; b0 += 0x7fffffffLL) {
    const long long n = std::min<long long>(0x7fffffffLL, total - b0);
    absmax_kernel<<<(unsigned)n, 256, 0, s>>>(x, per_sample, per, b0, amax, flags);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// One thread per (b, g, p): the 16 K-elements of group g at pixel p -> 4
// digit planes (digit, b, g, p, [ncol x] 16 B). Without a change of basis a
// group is 16/NB channels x NB blades; with one (BASIS) each pixel yields 2
// rows, row c holding 16/W channels x the W = NB/2 transformed components
// x'[c*W + r] = sum_I T[c*W + r][I] x[I].
// Integer-exact: X_I = rint(x_I 2^31 / s) (power-of-two scaling, one rounding),
// X' = sum_I T X_I in int32 (|X'| < 2^31 since s >= 2 max|x| 1.016), and the
// balanced base-256 digits are the two's-complement bytes of X'.
// FIXED: the (1,1,1) M2(C) basis found by find_basis, whose rows are sums /
// differences of blade pairs (2m, 2m+1): x' = (u0, -u3, v2, v1, u2, -u1, v0, v3)
// with u_m = X_2m + X_2m+1, v_m = X_2m - X_2m+1 (8 adds instead of 64 multiply-adds).
// One (b, g, p) item: the 16 K-elements of group g at pixel p of sample b ->
// 4 digit planes, with the sample's absmax `amx` (see slice_input_kernel).
// Balanced base-256 digits of X (|X| < 2^31 - 2^23): X = d0 + 2^8 d1 + 2^16 d2 + 2^24 d3
// with d0..d2 in [-128, 127]. Y = X + 0x808080 has the unsigned bytes d_k + 128
// (k < 3) and top byte d3, so the two's-complement digit bytes are the bytes
// of Y ^ 0x808080 -- the same digits as peeling d = sext(X & 255), X = (X - d) >> 8.
__device__ __forceinline__ uint32_t digits_of(int X) {
  return ((uint32_t)X + 0x808080u) ^ 0x808080u;
}

template <int NB, bool BASIS, bool FIXED>
__device__ __forceinline__ void slice_item(const float* __restrict__ x, float amx, int8_t* __restrict__ out,
                                           float* __restrict__ scale, long long b, int g, long long pp, int C,
                                           long long P, long long total, long long i, const Basis& bs) {
  constexpr int W = BASIS ? NB / 2 : NB;
  constexpr int NCOL = BASIS ? 2 : 1;
  constexpr int CPG = 16 / W;  // channels per group
  const float sc = pow2_scale_for(BASIS ? 2.f * amx : amx);  // |x'| <= 2 max|x|
  if (g == 0 && pp == 0) scale[b] = sc;
  const float mult = 2147483648.f / sc;  // 2^31 / s, exact power of two
  // Z[col][e]: the 4 balanced base-256 digits of element e of the 16-byte row,
  // as the bytes of one word (see digits_of)
  uint32_t Z[NCOL][16];
#pragma unroll
  for (int cl = 0; cl < CPG; ++cl) {
    const int c = g * CPG + cl;
    int X[NB];
    if (c < C) {
      const float* src = x + ((b * C + c) * P + pp) * NB;
      float v[NB];
      if constexpr (NB == 2) {
        const float2 q = __ldg(reinterpret_cast<const float2*>(src));
        v[0] = q.x; v[1] = q.y;
      } else {
#pragma unroll
        for (int h = 0; h < NB / 4; ++h) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(src) + h);
          v[4 * h] = q.x; v[4 * h + 1] = q.y; v[4 * h + 2] = q.z; v[4 * h + 3] = q.w;
        }
      }
#pragma unroll
      for (int I = 0; I < NB; ++I) X[I] = non_finite(v[I]) ? 0 : __float2int_rn(v[I] * mult);  // see finite_abs_bits
    } else {
#pragma unroll
      for (int I = 0; I < NB; ++I) X[I] = 0;
    }
#pragma unroll
    for (int col = 0; col < NCOL; ++col) {
#pragma unroll
      for (int r = 0; r < W; ++r) {
        int Xs;
        if constexpr (FIXED) {
          const int a = col * W + r;
          const int m = (a == 0 || a == 6) ? 0 : (a == 3 || a == 5) ? 1 : (a == 2 || a == 4) ? 2 : 3;
          const bool use_u = (a == 0 || a == 1 || a == 4 || a == 5);
          const int val = use_u ? X[2 * m] + X[2 * m + 1] : X[2 * m] - X[2 * m + 1];
          Xs = (a == 1 || a == 5) ? -val : val;
        } else if constexpr (BASIS) {
          Xs = 0;
#pragma unroll
          for (int I = 0; I < NB; ++I) Xs += (int)bs.T[(col * W + r) * 8 + I] * X[I];
        } else {
          Xs = X[r];
        }
        Z[col][cl * W + r] = digits_of(Xs);
      }
    }
  }
  // digit plane k holds digit 3-k (plane 0 = most significant): a 4x4 byte
  // transpose of every 4 consecutive elements, 8 byte permutes per 4 words
#pragma unroll
  for (int col = 0; col < NCOL; ++col) {
    uint32_t word[4][4];  // [digit plane][word]
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t t0 = __byte_perm(Z[col][4 * j], Z[col][4 * j + 1], 0x5140);  // b0 b0' b1 b1'
      const uint32_t t1 = __byte_perm(Z[col][4 * j], Z[col][4 * j + 1], 0x7362);  // b2 b2' b3 b3'
      const uint32_t t2 = __byte_perm(Z[col][4 * j + 2], Z[col][4 * j + 3], 0x5140);
      const uint32_t t3 = __byte_perm(Z[col][4 * j + 2], Z[col][4 * j + 3], 0x7362);
      word[3][j] = __byte_perm(t0, t2, 0x5410);  // digit 0 (least significant)
      word[2][j] = __byte_perm(t0, t2, 0x7632);
      word[1][j] = __byte_perm(t1, t3, 0x5410);
      word[0][j] = __byte_perm(t1, t3, 0x7632);  // digit 3
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      reinterpret_cast<uint4*>(out)[((long long)k * total + i) * NCOL + col] =
          make_uint4(word[k][0], word[k][1], word[k][2], word[k][3]);
  }
}

// One thread per (b, g, p): the 16 K-elements of group g at pixel p -> 4
// digit planes (digit, b, g, p, [ncol x] 16 B). Without a change of basis a
// group is 16/NB channels x NB blades; with one (BASIS) each pixel yields 2
// rows, row c holding 16/W channels x the W = NB/2 transformed components
// x'[c*W + r] = sum_I T[c*W + r][I] x[I].
// Integer-exact: X_I = rint(x_I 2^31 / s) (power-of-two scaling, one rounding),
// X' = sum_I T X_I in int32 (|X'| < 2^31 since s >= 2 max|x| 1.016), and the
// balanced base-256 digits are the two's-complement bytes of X'.
// FIXED: the (1,1,1) M2(C) basis found by find_basis, whose rows are sums /
// differences of blade pairs (2m, 2m+1): x' = (u0, -u3, v2, v1, u2, -u1, v0, v3)
// with u_m = X_2m + X_2m+1, v_m = X_2m - X_2m+1 (8 adds instead of 64 multiply-adds).
#ifndef CL_SLICE_MINB
#define CL_SLICE_MINB 3  // resident blocks per SM of the fixed-form kernel (A/B builds: -DCL_SLICE_MINB=n)
#endif
template <int NB, bool BASIS, bool FIXED = false>
__global__ void __launch_bounds__(256, FIXED ? CL_SLICE_MINB : 1) slice_input_kernel(const float* __restrict__ x,
                                                          const unsigned* __restrict__ amax,
                                                          int8_t* __restrict__ out, float* __restrict__ scale,
                                                          long long B, int C, long long P, int G, Basis bs) {
  const long long total = B * G * P;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long pp, b;
    int g;
    if (total <= 0xffffffffLL) {  // 32-bit division (uniform branch)
      const unsigned bg = (unsigned)i / (unsigned)P;
      pp = (unsigned)i - bg * (unsigned)P;
      b = bg / (unsigned)G;
      g = (int)(bg - (unsigned)b * (unsigned)G);
    } else {
      pp = i % P;
      const long long bg = i / P;
      g = (int)(bg % G);
      b = bg / G;
    }
    slice_item<NB, BASIS, FIXED>(x, __uint_as_float(__ldg(amax + b)), out, scale, b, g, pp, C, P, total, i, bs);
  }
}

// Small layers (launch-bound): absmax and slicing in ONE launch. A cluster of
// kSliceCluster CTAs per sample: each CTA takes the max over its share of the
// sample, the cluster combines the shares through distributed shared memory,
// then each CTA slices its share of the sample's (g, p) items. Replaces the
// memset + absmax + slice launches of the general path (which need a grid-wide
// max first).
constexpr int kSliceCluster = 8;
template <int NB, bool BASIS, bool FIXED = false>
__global__ void __launch_bounds__(256) absmax_slice_kernel(const float* __restrict__ x, int8_t* __restrict__ out,
                                                           float* __restrict__ scale, unsigned* __restrict__ flags,
                                                           long long B, int C, long long P, int G, Basis bs) {
  __shared__ unsigned red[8], redn[8];  // max finite |x| / max |x| (NaN-sticky) as float bits
  __shared__ float cmax, cany;
  const int rank = (int)cluster_ctarank();
  const long long b = blockIdx.x / kSliceCluster;
  const long long per_sample = (long long)C * P * NB;
  const float* xs = x + b * per_sample;
  unsigned m = 0, any = 0;
  const long long n0 = per_sample * rank / kSliceCluster, n1 = per_sample * (rank + 1) / kSliceCluster;
  for (long long i = n0 + threadIdx.x; i < n1; i += blockDim.x) {
    const float v = __ldg(xs + i);
    m = max(m, finite_abs_bits(v));
    any = max(any, abs_bits(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    any = max(any, __shfl_xor_sync(0xffffffffu, any, o));
  }
  if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = m; redn[threadIdx.x >> 5] = any; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned v = 0, vn = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { v = max(v, red[w]); vn = max(vn, redn[w]); }
    cmax = __uint_as_float(v);
    cany = __uint_as_float(vn);
  }
  cluster_sync();  // every CTA's share is in its cmax / cany
  if (threadIdx.x == 0) {
    unsigned v = 0, vn = 0;
    for (int r = 0; r < kSliceCluster; ++r) {
      v = max(v, __float_as_uint(ld_shared_cluster_f32(&cmax, r)));
      vn = max(vn, __float_as_uint(ld_shared_cluster_f32(&cany, r)));
    }
    red[0] = v;
    if (rank == 0) flags[b] = vn >= 0x7f800000u ? 1u : 0u;  // written every call: no zeroing launch
  }
  cluster_sync();  // peers done reading cmax (no CTA exits while it is read)
  __syncthreads();
  const float amx = __uint_as_float(red[0]);
  const long long total = B * G * P;
  const long long items = (long long)G * P;
  const long long i0 = items * rank / kSliceCluster, i1 = items * (rank + 1) / kSliceCluster;
  for (long long it = i0 + threadIdx.x; it < i1; it += blockDim.x) {
    const int g = (int)(it / P);
    const long long pp = it - (long long)g * P;
    const long long i = (b * G + g) * P + pp;
    slice_item<NB, BASIS, FIXED>(x, amx, out, scale, b, g, pp, C, P, total, i, bs);
  }
}

template <int NB, bool BASIS, bool FIXED>
static cudaError_t launch_fused_t(const float* x, int8_t* digits, float* scale, unsigned* flags, long long B, int C,
                                  long long P, int G, const Basis& bs, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * kSliceCluster));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSliceCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, absmax_slice_kernel<NB, BASIS, FIXED>, x, digits, scale, flags, B, C, P, G, bs);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

static bool fixed_111_basis(int nb, const Basis& bs) {
  static const int8_t kFixed[8][8] = {{1, 1, 0, 0, 0, 0, 0, 0},  {0, 0, 0, 0, 0, 0, -1, -1}, {0, 0, 0, 0, 1, -1, 0, 0},
                                      {0, 0, 1, -1, 0, 0, 0, 0}, {0, 0, 0, 0, 1, 1, 0, 0},   {0, 0, -1, -1, 0, 0, 0, 0},
                                      {1, -1, 0, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 1, -1}};
  static const bool no_fixed = CL_ENV("CL_NO_SLICE_FIXED") != nullptr;
  bool fixed = nb == 8 && bs.on && !no_fixed;
  for (int a = 0; a < 8 && fixed; ++a)
    for (int I = 0; I < 8 && fixed; ++I) fixed = bs.T[a * 8 + I] == kFixed[a][I];
  return fixed;
}

cudaError_t launch_absmax_slice(const float* x, int8_t* digits, float* scale, unsigned* flags, int nb, long long B,
                                int C, long long P, int G, const Basis& bs, cudaStream_t s) {
  if (B * G * P == 0) return cudaSuccess;
  if (bs.on) {
    if (nb == 4) return launch_fused_t<4, true, false>(x, digits, scale, flags, B, C, P, G, bs, s);
    if (fixed_111_basis(nb, bs)) return launch_fused_t<8, true, true>(x, digits, scale, flags, B, C, P, G, bs, s);
    return launch_fused_t<8, true, false>(x, digits, scale, flags, B, C, P, G, bs, s);
  }
  if (nb == 2) return launch_fused_t<2, false, false>(x, digits, scale, flags, B, C, P, G, bs, s);
  if (nb == 4) return launch_fused_t<4, false, false>(x, digits, scale, flags, B, C, P, G, bs, s);
  return launch_fused_t<8, false, false>(x, digits, scale, flags, B, C, P, G, bs, s);
}

cudaError_t launch_slice_input(const float* x, const unsigned* amax, int8_t* digits, float* scale, int nb,
                               long long B, int C, long long P, int G, const Basis& bs, cudaStream_t s) {
  const long long total = B * G * P;
  if (total == 0) return cudaSuccess;
  // One wave: blocks per SM from the occupancy calculator (the basis variants
  // are register-heavy). Unlike the activation, a many-wave grid (one item per
  // thread) measured slower here: 8.2 vs 7.0 ms per cfg5 tensor (each block
  // streams 4 input channels and 4 digit planes at once).
  auto grid = [&](auto kern) {
    const int per_sm = resident_blocks_per_sm(reinterpret_cast<const void*>(kern), 256, 0);
    long long blocks = (total + 255) / 256;
    const long long cap = (long long)num_sms() * per_sm;
    return (unsigned)(blocks > cap ? cap : blocks);
  };
  if (bs.on) {
    const bool fixed = fixed_111_basis(nb, bs);
    if (nb == 4) slice_input_kernel<4, true><<<grid(slice_input_kernel<4, true>), 256, 0, s>>>(x, amax, digits, scale, B, C, P, G, bs);
    else if (fixed) slice_input_kernel<8, true, true><<<grid(slice_input_kernel<8, true, true>), 256, 0, s>>>(x, amax, digits, scale, B, C, P, G, bs);
    else slice_input_kernel<8, true><<<grid(slice_input_kernel<8, true>), 256, 0, s>>>(x, amax, digits, scale, B, C, P, G, bs);
  } else {
    if (nb == 2) slice_input_kernel<2, false><<<grid(slice_input_kernel<2, false>), 256, 0, s>>>(x, amax, digits, scale, B, C, P, G, bs);
    else if (nb == 4) slice_input_kernel<4, false><<<grid(slice_input_kernel<4, false>), 256, 0, s>>>(x, amax, digits, scale, B, C, P, G, bs);
    else slice_input_kernel<8, false><<<grid(slice_input_kernel<8, false>), 256, 0, s>>>(x, amax, digits, scale, B, C, P, G, bs);
  }
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
  unsigned m = 0;  // max |entry| as float bits (NaN-sticky: a NaN filter gives a NaN scale)
  // under a change of basis all w columns of a channel share one scale, so the
  // epilogue can combine the two column terms of the inverse as exact integers
  const int t0 = bs.on ? 0 : t, t1 = bs.on ? w : t + 1;
  if (co < C_out) {
    for (int tt = t0; tt < t1; ++tt)
      for (int idx = threadIdx.x; idx < C_in * w * Q; idx += blockDim.x) {
        const int q = idx % Q;
        const int j = (idx / Q) % w;
        const int ci = idx / (Q * w);
        const double e = bs.on ? basis_entry(sg, bs, f, C_in, C_out, Q, co, tt, ci, j, q)
                               : (double)expanded_entry(sg, f, nb, C_in, C_out, Q, co, tt, ci, j, q);
        m = max(m, abs_bits((float)e));
      }
  }
  __shared__ unsigned red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) m = max(m, red[ww]);
    // float rounding of |e| may round down: one more power of two of headroom is free
    w_scale[n] = pow2_scale_for(__uint_as_float(m) * 1.0000002f);
  }
}

cudaError_t launch_weight_colscale(const int* g, const ConvPlan& pl, const float* f, int C_in, int C_out,
                                   float* w_scale, cudaStream_t s) {
  const int N_pad = pl.n_ntiles * pl.n_tile;
  const Sig sg = make_sig(g, pl.ka);
  weight_colscale_kernel<<<N_pad, 256, 0, s>>>(sg, f, C_in, C_out, pl.Q, pl.bs, w_scale);
  count_launch();
  return cudaGetLastError();
}

// Exact mode, non-finite inputs (after the conv): every output pixel whose
// receptive field holds an Inf / NaN input becomes NaN in all channels and
// blades -- what the reference's fp64 einsum gives there (a non-finite input
// times the Cayley tensor's structural zeros, conv.py:168-176) -- while every
// other output keeps its exact value (the slice pass encoded the non-finite
// inputs as 0). Samples without a flag return at once, so the launch is a few
// microseconds when the input is finite. `flags_out` (optional) marks the
// samples the next conv of a block must treat the same way.
__global__ void __launch_bounds__(256) poison_nonfinite_kernel(PoisonParams p) {
  const long long total = p.B * p.P_out;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / p.P_out;
    if (!__ldg(p.flags + b)) continue;
    const long long o = i - b * p.P_out;
    const int d = p.d_out;
    const int ox = (int)(o % d), oy = p.k >= 2 ? (int)((o / d) % d) : 0, oz = p.k == 3 ? (int)(o / ((long long)d * d)) : 0;
    const int qz_n = p.k == 3 ? p.d_filter : 1, qy_n = p.k >= 2 ? p.d_filter : 1;
    bool hit = false;
    for (int qz = 0; qz < qz_n && !hit; ++qz) {
      const int iz = oz + qz - (p.k == 3 ? p.pad : 0);
      if (iz < 0 || iz >= (p.k == 3 ? p.d_in : 1)) continue;
      for (int qy = 0; qy < qy_n && !hit; ++qy) {
        const int iy = oy + qy - (p.k >= 2 ? p.pad : 0);
        if (iy < 0 || iy >= (p.k >= 2 ? p.d_in : 1)) continue;
        for (int qx = 0; qx < p.d_filter && !hit; ++qx) {
          const int ix = ox + qx - p.pad;
          if (ix < 0 || ix >= p.d_in) continue;
          const long long pin = ((long long)iz * p.d_in + iy) * p.d_in + ix;
          for (int c = 0; c < p.C_in && !hit; ++c) {
            const float* xp = p.x + ((b * p.C_in + c) * p.P_in + pin) * p.nb;
            for (int j = 0; j < p.nb; ++j) hit = hit || non_finite(xp[j]);
          }
        }
      }
    }
    if (!hit) continue;
    for (int co = 0; co < p.C_out; ++co) {
      float* yp = p.y + ((b * p.C_out + co) * p.P_out + o) * p.nb;
      for (int t = 0; t < p.nb; ++t) yp[t] = __uint_as_float(0x7fc00000u);
    }
    if (p.flags_out) atomicOr(p.flags_out + b, 1u);
  }
}

cudaError_t launch_poison_nonfinite(const PoisonParams& p, cudaStream_t s) {
  const long long total = p.B * p.P_out;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  const long long cap = 8LL * num_sms();
  if (blocks > cap) blocks = cap;
  poison_nonfinite_kernel<<<(unsigned)blocks, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cl
