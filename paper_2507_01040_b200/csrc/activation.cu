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
// time to a dense (C, N_B) blade-ordered table (zero for non-kernel blades,
// as activation.py:385-390 does for its specialised path), so the inner loop
// is branch-free for any K <= N_B and any C.
//
// One thread per multivector: 16 B (2-D) or 32 B (3-D) of contiguous,
// 16-byte-aligned data -> 128-bit streaming loads/stores; 4 multivectors in
// flight per thread; grid sized to a multiple of the SM count.
#include "common.cuh"
#include "internal.h"

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

// 1-D (N_B = 2): 8-byte multivectors, 8 in flight per thread.
template <int MODE>
__global__ void __launch_bounds__(256) act_kernel_nb2(ActParams p) {
  constexpr int U = 8;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float2* __restrict__ x = reinterpret_cast<const float2*>(p.x);
  float2* __restrict__ y = reinterpret_cast<float2*>(p.y);
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < p.n_mv; base += stride * U) {
    float2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < p.n_mv) v[u] = __ldcs(x + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < p.n_mv) {
        const int c = (int)((i / p.P) % p.C);
        float s = fmaf(v[u].x, __ldg(p.w + 2 * c), 0.f);
        s = fmaf(v[u].y, __ldg(p.w + 2 * c + 1), s);
        if (MODE == 0) s += __ldg(p.b + c);
        if (MODE == 2) s = s / p.Kf;
        const float gte = 1.f / (1.f + expf(-s));
        __stcs(y + i, make_float2(v[u].x * gte, v[u].y * gte));
      }
    }
  }
}

template <int NB, int MODE>
__global__ void __launch_bounds__(256) act_kernel(ActParams p) {
  constexpr int V = NB / 4;  // float4 per multivector
  constexpr int U = 4;       // multivectors in flight per thread
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float4* __restrict__ x = reinterpret_cast<const float4*>(p.x);
  float4* __restrict__ y = reinterpret_cast<float4*>(p.y);
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < p.n_mv;
       base += stride * U) {
    float4 v[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < p.n_mv) {
#pragma unroll
        for (int h = 0; h < V; ++h) v[u][h] = ld_stream(x + i * V + h);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = base + u * stride;
      if (i < p.n_mv) {
        const int c = (int)((i / p.P) % p.C);
        const float* w = p.w + c * NB;
        float s = 0.f;
#pragma unroll
        for (int h = 0; h < V; ++h) {
          s = fmaf(v[u][h].x, __ldg(w + 4 * h + 0), s);
          s = fmaf(v[u][h].y, __ldg(w + 4 * h + 1), s);
          s = fmaf(v[u][h].z, __ldg(w + 4 * h + 2), s);
          s = fmaf(v[u][h].w, __ldg(w + 4 * h + 3), s);
        }
        if (MODE == 0) s += __ldg(p.b + c);
        if (MODE == 2) s = s / p.Kf;
        const float gte = 1.f / (1.f + expf(-s));
#pragma unroll
        for (int h = 0; h < V; ++h) {
          float4 o = v[u][h];
          o.x *= gte; o.y *= gte; o.z *= gte; o.w *= gte;
          st_stream(y + i * V + h, o);
        }
      }
    }
  }
}

// Grid = exactly the resident capacity (one wave, no tail): blocks per SM
// from the occupancy calculator x SM count, capped by the work.
template <int NB, int MODE>
static cudaError_t launch_mode(const ActParams& p, cudaStream_t s) {
  static int per_sm = [] {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, act_kernel<NB, MODE>, 256, 0);
    return n > 0 ? n : 1;
  }();
  long long blocks = (p.n_mv + 256LL * 4 - 1) / (256LL * 4);
  const long long cap = (long long)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  act_kernel<NB, MODE><<<(unsigned)blocks, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_nb2_mode(const ActParams& p, cudaStream_t s) {
  static int per_sm = [] {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, act_kernel_nb2<MODE>, 256, 0);
    return n > 0 ? n : 1;
  }();
  long long blocks = (p.n_mv + 256LL * 8 - 1) / (256LL * 8);
  const long long cap = (long long)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  act_kernel_nb2<MODE><<<(unsigned)blocks, 256, 0, s>>>(p);
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

cudaError_t launch_act(int nb, const ActParams& p, cudaStream_t s) {
  if (p.n_mv == 0) return cudaSuccess;
  if (nb == 2) {
    switch (p.mode) {
      case 0: return launch_nb2_mode<0>(p, s);
      case 1: return launch_nb2_mode<1>(p, s);
      default: return launch_nb2_mode<2>(p, s);
    }
  }
  return nb == 4 ? launch_nb<4>(p, s) : launch_nb<8>(p, s);
}

}  // namespace cl
