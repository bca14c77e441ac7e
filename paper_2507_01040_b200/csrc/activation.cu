// activation.cu -- (3) multivector activation, standalone (HBM-bound).
//
// Semantics of activation.py:142-162 applied per (b, c, p) as in the
// spatial fold of serve.py:108-117 (no fold is materialised: the gate is
// computed in place on the protocol layout (B, C, P, N_B)):
//   s = sum_k x[ki[k]] * w[c, k] + bias[c]   (Linear)
//   s = sum_k x[ki[k]]                        (Sum)
//   s = sum_k x[ki[k]] / K                    (Mean)
//   out[j] = x[j] * sigmoid(s)  for every blade j.
// The kernel-blade subset and the Linear weights are re-keyed once at create
// time to a dense (C, N_B) blade-ordered table (as activation.py:385-390 does
// for its specialised path), so the inner loop is branch-free for any K <= N_B
// and any C. Non-kernel blades are SELECTED out (kmask), not multiplied by a
// zero weight: the reference never reads them (activation.py:142-162), so an
// Inf / NaN there must not reach the gate (0 * Inf = NaN).
//
// One thread per multivector: 8 B (1-D), 16 B (2-D) or 32 B (3-D) of
// contiguous, aligned data -> 64/128-bit streaming loads/stores; 4 (8 in 1-D)
// multivectors in flight per thread; one contiguous chunk per block.
#include "common.cuh"
#include "internal.h"

#include <type_traits>

namespace cl {

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Exact unsigned division of n < 2^31 (host-side magic numbers, launch_act).
__device__ __forceinline__ unsigned udiv(unsigned n, unsigned mag, unsigned sh) {
  return (unsigned)(((unsigned long long)n * mag) >> sh);
}

// Each block gates one contiguous chunk of 256*U multivectors (no grid-stride
// loop, many waves): a block streams 16-32 KB of consecutive HBM, which kept
// DRAM pages open better than a grid-stride loop over a one-wave grid
// (tools/probe/act_variants.cu at cfg2: 6.2 vs 5.3-5.5 TB/s median). The
// channel of element i is ((i / P) % C); the block's first index is split
// once in 64 bits, the rest is 32-bit magic-number division.
template <int NB, int MODE, int U, bool FULL>
__global__ void __launch_bounds__(256) act_kernel(ActParams p) {
  using VT = typename std::conditional<NB == 2, float2, float4>::type;
  constexpr int V = NB == 2 ? 1 : NB / 4;  // vectors per multivector
  const long long base0 = (long long)blockIdx.x * (256 * U);
  const long long bc0 = base0 / p.P;                 // (b, c) plane of the chunk start
  const unsigned r0 = (unsigned)(base0 - bc0 * p.P);  // offset inside that plane (< P < 2^31)
  const unsigned c0 = (unsigned)(bc0 % p.C);
  const VT* __restrict__ x = reinterpret_cast<const VT*>(p.x);
  VT* __restrict__ y = reinterpret_cast<VT*>(p.y);
  VT v[U][V];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = base0 + u * 256 + threadIdx.x;
    if (i < p.n_mv) {
#pragma unroll
      for (int h = 0; h < V; ++h) {
        if constexpr (NB == 2) v[u][h] = __ldcs(x + i);
        else v[u][h] = ld_stream(x + i * V + h);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long i = base0 + u * 256 + threadIdx.x;
    if (i < p.n_mv) {
      // planes crossed since the chunk start (r0 + 256U < 2^31: P < 2^30)
      const unsigned k = udiv(r0 + (unsigned)(u * 256) + threadIdx.x, p.magP, p.shP);
      const unsigned ck = c0 + k;
      const unsigned c = ck - udiv(ck, p.magC, p.shC) * (unsigned)p.C;
      const float* w = p.w + c * NB;
      // every blade is a kernel blade (FULL), or a select keeps the others out
      auto acc = [&](float s, float xv, int j) {
        const float t = fmaf(xv, __ldg(w + j), s);
        return (FULL || ((p.kmask >> j) & 1u)) ? t : s;
      };
      float s = 0.f;
      if constexpr (NB == 2) {
        s = acc(s, v[u][0].x, 0);
        s = acc(s, v[u][0].y, 1);
      } else {
#pragma unroll
        for (int h = 0; h < V; ++h) {
          s = acc(s, v[u][h].x, 4 * h + 0);
          s = acc(s, v[u][h].y, 4 * h + 1);
          s = acc(s, v[u][h].z, 4 * h + 2);
          s = acc(s, v[u][h].w, 4 * h + 3);
        }
      }
      if (MODE == 0) s += __ldg(p.b + c);
      if (MODE == 2) s = s / p.Kf;
      const float gte = 1.f / (1.f + expf(-s));
#pragma unroll
      for (int h = 0; h < V; ++h) {
        VT o = v[u][h];
        if constexpr (NB == 2) {
          o.x *= gte; o.y *= gte;
          __stcs(y + i, o);
        } else {
          o.x *= gte; o.y *= gte; o.z *= gte; o.w *= gte;
          st_stream(y + i * V + h, o);
        }
      }
    }
  }
}

template <int NB, int MODE>
static cudaError_t launch_mode(const ActParams& p, cudaStream_t s) {
  constexpr int U = NB == 2 ? 8 : 4;
  const long long blocks = (p.n_mv + 256LL * U - 1) / (256LL * U);
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  if (p.kmask == (1u << NB) - 1u) act_kernel<NB, MODE, U, true><<<(unsigned)blocks, 256, 0, s>>>(p);
  else act_kernel<NB, MODE, U, false><<<(unsigned)blocks, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int NB>
static cudaError_t launch_nb(const ActParams& p, cudaStream_t s) {
  switch (p.mode) {
    case 0: return launch_mode<NB, 0>(p, s);
    case 1: return launch_mode<NB, 1>(p, s);
    default: return launch_mode<NB, 2>(p, s);
  }
}

// n < 2^31: with sh = 31 + ceil(log2 d) and mag = ceil(2^sh / d) < 2^32,
// (n * mag) >> sh == n / d exactly, because n * (mag * d - 2^sh) < 2^sh.
static void magic_div(unsigned d, unsigned* mag, unsigned* sh) {
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  *sh = 31 + l;
  *mag = (unsigned)(((1ull << *sh) + d - 1) / d);
}

cudaError_t launch_act(int nb, const ActParams& p0, cudaStream_t s) {
  if (p0.n_mv == 0) return cudaSuccess;
  if (p0.P < 1 || p0.P >= (1LL << 30) || p0.C < 1 || p0.C >= (1 << 30)) return cudaErrorInvalidValue;
  ActParams p = p0;
  magic_div((unsigned)p.P, &p.magP, &p.shP);
  magic_div((unsigned)p.C, &p.magC, &p.shC);
  if (nb == 2) {
    switch (p.mode) {
      case 0: return launch_mode<2, 0>(p, s);
      case 1: return launch_mode<2, 1>(p, s);
      default: return launch_mode<2, 2>(p, s);
    }
  }
  return nb == 4 ? launch_nb<4>(p, s) : launch_nb<8>(p, s);
}

// gate_preactivation (activation.py:110-117): s per (b, c, p) -- the kernel
// blades in the caller's order ki[0..K), Linear weights from the re-keyed
// table, + bias (Linear) or / K (Mean). gather_vpack (activation.py:99-107):
// the K kernel blades of every multivector, in ki order, (B, C, P, K).
// Diagnostic / property-check entry points (one thread per multivector).
template <int NB, bool GATHER>
__global__ void __launch_bounds__(256) act_aux_kernel(ActParams p) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < p.n_mv;
       i += (long long)gridDim.x * blockDim.x) {
    const float* xv = p.x + i * NB;
    if constexpr (GATHER) {
      for (int k = 0; k < p.K; ++k) p.y[i * p.K + k] = xv[p.ki[k]];
    } else {
      const int c = (int)((i / p.P) % p.C);
      float s = 0.f;
      for (int k = 0; k < p.K; ++k) {
        const float a = xv[p.ki[k]];
        s = p.mode == 0 ? fmaf(a, __ldg(p.w + c * NB + p.ki[k]), s) : s + a;
      }
      if (p.mode == 0) s += __ldg(p.b + c);
      else if (p.mode == 2) s = s / p.Kf;
      p.y[i] = s;
    }
  }
}

template <bool GATHER>
static cudaError_t launch_aux(int nb, const ActParams& p, cudaStream_t s) {
  if (p.n_mv == 0) return cudaSuccess;
  long long blocks = (p.n_mv + 255) / 256;
  blocks = blocks > 4LL * num_sms() * 8 ? 4LL * num_sms() * 8 : blocks;
  if (nb == 2) act_aux_kernel<2, GATHER><<<(unsigned)blocks, 256, 0, s>>>(p);
  else if (nb == 4) act_aux_kernel<4, GATHER><<<(unsigned)blocks, 256, 0, s>>>(p);
  else act_aux_kernel<8, GATHER><<<(unsigned)blocks, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_act_preact(int nb, const ActParams& p, cudaStream_t s) { return launch_aux<false>(nb, p, s); }
cudaError_t launch_act_gather(int nb, const ActParams& p, cudaStream_t s) { return launch_aux<true>(nb, p, s); }

}  // namespace cl
