// act_variants.cu -- standalone timing of activation-kernel variants at cfg2
// (B=64, C=64, P=4096, N_B=4, Linear). Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o act_variants act_variants.cu
// Prints, per variant, the best and median of 30 event-timed launches in TB/s
// (algorithmic bytes: read + write of the whole tensor), after a max-abs
// check against variant 0.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

struct P_ {
  const float* x; float* y; long long n_mv; long long P; int C; const float* w; const float* b;
  unsigned magP, shP, magC, shC;  // unsigned division by P and C (n < 2^31)
};

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_stream256(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ unsigned fdiv(unsigned n, unsigned mag, unsigned sh) {
  return (unsigned)(((unsigned long long)n * mag) >> sh);
}
__device__ __forceinline__ float4 gate4(float4 v, const float* __restrict__ w, float b) {
  float s = fmaf(v.x, __ldg(w), fmaf(v.y, __ldg(w + 1), fmaf(v.z, __ldg(w + 2), fmaf(v.w, __ldg(w + 3), b))));
  float g = 1.f / (1.f + __expf(-s));
  v.x *= g; v.y *= g; v.z *= g; v.w *= g;
  return v;
}

// V0: the library kernel (64-bit index, 64-bit division per multivector, U = 4)
__global__ void __launch_bounds__(256) v0(P_ p) {
  constexpr int U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float4* x = (const float4*)p.x; float4* y = (float4*)p.y;
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < p.n_mv; base += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long i = base + u * stride; if (i < p.n_mv) v[u] = ld_stream(x + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long i = base + u * stride;
      if (i < p.n_mv) {
        int c = (int)((i / p.P) % p.C);
        const float* w = p.w + c * 4;
        float s = 0.f;
        s = fmaf(v[u].x, __ldg(w), s); s = fmaf(v[u].y, __ldg(w + 1), s); s = fmaf(v[u].z, __ldg(w + 2), s); s = fmaf(v[u].w, __ldg(w + 3), s);
        s += __ldg(p.b + c);
        float g = 1.f / (1.f + expf(-s));
        float4 o = v[u]; o.x *= g; o.y *= g; o.z *= g; o.w *= g;
        st_stream(y + i, o);
      }
    }
  }
}

// V1/V2/V5: 32-bit index, magic division, U multivectors in flight
template <int U, bool L2P>
__global__ void __launch_bounds__(256) v1(P_ p) {
  const unsigned n = (unsigned)p.n_mv;
  const unsigned stride = gridDim.x * blockDim.x;
  const float4* x = (const float4*)p.x; float4* y = (float4*)p.y;
  for (unsigned base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { unsigned i = base + u * stride; if (i < n) v[u] = L2P ? ld_stream256(x + i) : ld_stream(x + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      unsigned i = base + u * stride;
      if (i < n) {
        unsigned bc = fdiv(i, p.magP, p.shP);
        unsigned c = bc - fdiv(bc, p.magC, p.shC) * (unsigned)p.C;
        st_stream(y + i, gate4(v[u], p.w + c * 4, __ldg(p.b + c)));
      }
    }
  }
}

// V3: one chunk of 256*U contiguous multivectors per block, no loop (many waves)
template <int U>
__global__ void __launch_bounds__(256) v3(P_ p) {
  const unsigned n = (unsigned)p.n_mv;
  const unsigned base = blockIdx.x * 256u * U + threadIdx.x;
  const float4* x = (const float4*)p.x; float4* y = (float4*)p.y;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { unsigned i = base + u * 256; if (i < n) v[u] = ld_stream(x + i); }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    unsigned i = base + u * 256;
    if (i < n) {
      unsigned bc = fdiv(i, p.magP, p.shP);
      unsigned c = bc - fdiv(bc, p.magC, p.shC) * (unsigned)p.C;
      st_stream(y + i, gate4(v[u], p.w + c * 4, __ldg(p.b + c)));
    }
  }
}

// V4: pure copy with the V1 structure (ceiling of this access pattern)
template <int U>
__global__ void __launch_bounds__(256) v4(P_ p) {
  const unsigned n = (unsigned)p.n_mv;
  const unsigned stride = gridDim.x * blockDim.x;
  const float4* x = (const float4*)p.x; float4* y = (float4*)p.y;
  for (unsigned base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { unsigned i = base + u * stride; if (i < n) v[u] = ld_stream(x + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) { unsigned i = base + u * stride; if (i < n) st_stream(y + i, v[u]); }
  }
}

// V6: TMA bulk pipeline. Persistent CTA (1 per SM... or 2), chunks of CH bytes,
// S stages; one thread issues cp.async.bulk global->smem, all threads gate in
// smem, one thread issues cp.async.bulk smem->global.
template <int CH, int S>
__global__ void __launch_bounds__(256) v6(P_ p) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long full[S];
  const long long nbytes = p.n_mv * 16;
  const long long nch = (nbytes + CH - 1) / CH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](long long ch, int s) {
    long long off = ch * CH; unsigned bytes = (unsigned)min((long long)CH, nbytes - off);
    unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
    unsigned dst = (unsigned)__cvta_generic_to_shared(sm + s * CH);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"((const char*)p.x + off), "r"(bytes), "r"(bar) : "memory");
  };
  int k = 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < S; ++s) { long long ch = blockIdx.x + (long long)s * gridDim.x; if (ch < nch) issue(ch, s); }
  unsigned phase[S] = {};
  (void)phase;
  unsigned ph = 0;
  for (long long ch = blockIdx.x; ch < nch; ch += gridDim.x, ++k) {
    const int s = k % S;
    if (k > 0 && s == 0) ph ^= 1;
    unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
    asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(bar), "r"(ph) : "memory");
    long long off = ch * CH; unsigned bytes = (unsigned)min((long long)CH, nbytes - off);
    float4* buf = (float4*)(sm + s * CH);
    const unsigned i0 = (unsigned)(off / 16);
    for (unsigned j = threadIdx.x; j < bytes / 16; j += 256) {
      unsigned i = i0 + j;
      unsigned bc = fdiv(i, p.magP, p.shP);
      unsigned c = bc - fdiv(bc, p.magC, p.shC) * (unsigned)p.C;
      buf[j] = gate4(buf[j], p.w + c * 4, __ldg(p.b + c));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)p.y + off), "r"((unsigned)__cvta_generic_to_shared(buf)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      long long nx = ch + (long long)S * gridDim.x;
      if (nx < nch) issue(nx, s);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static void magic(unsigned d, unsigned& m, unsigned& s) {
  // n < 2^31: p = 31 + ceil(log2 d), m = ceil(2^p / d) < 2^32 is exact (n * (m d - 2^p) < 2^p)
  unsigned l = 0; while ((1u << l) < d) ++l;
  s = 31 + l;
  m = (unsigned)(((1ull << s) + d - 1) / d);
}

int main() {
  const int B = 64, C = 64, P = 4096;
  const long long n = (long long)B * C * P;
  const size_t bytes = n * 16;
  float *x, *y, *y0, *w, *b;
  CK(cudaMalloc(&x, bytes)); CK(cudaMalloc(&y, bytes)); CK(cudaMalloc(&y0, bytes));
  CK(cudaMalloc(&w, C * 4 * 4)); CK(cudaMalloc(&b, C * 4));
  std::vector<float> hx(n * 4), hw(C * 4), hb(C);
  srand(1);
  for (auto& v : hx) v = (rand() / (float)RAND_MAX - 0.5f) * 4;
  for (auto& v : hw) v = rand() / (float)RAND_MAX - 0.5f;
  for (auto& v : hb) v = (rand() / (float)RAND_MAX - 0.5f) * 0.2f;
  CK(cudaMemcpy(x, hx.data(), bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(w, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
  P_ p{x, y0, n, P, C, w, b, 0, 0, 0, 0};
  magic(P, p.magP, p.shP); magic(C, p.magC, p.shC);
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  auto occ = [&](const void* k, int smem) { int nb = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, smem)); return nb; };
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto cap = [&](long long want, const void* k, int smem) { long long c = (long long)sms * occ(k, smem); return (unsigned)std::max(1LL, std::min(want, c)); };
  // reference output
  v0<<<cap((n + 1023) / 1024, (const void*)v0, 0), 256>>>(p);
  CK(cudaDeviceSynchronize());
  std::vector<float> r(n * 4), t(n * 4);
  CK(cudaMemcpy(r.data(), y0, bytes, cudaMemcpyDeviceToHost));
  p.y = y;
  auto run = [&](const char* name, auto launch) {
    CK(cudaMemset(y, 0, bytes));
    launch(); CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(t.data(), y, bytes, cudaMemcpyDeviceToHost));
    double md = 0; for (size_t i = 0; i < t.size(); ++i) md = std::max(md, (double)fabsf(t[i] - r[i]));
    std::vector<float> ms;
    for (int it = 0; it < 30; ++it) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float m; CK(cudaEventElapsedTime(&m, e0, e1)); ms.push_back(m);
    }
    std::sort(ms.begin(), ms.end());
    printf("%-34s best %7.2f us %5.2f TB/s  median %7.2f us %5.2f TB/s  maxdiff %.2e\n", name, ms[0] * 1e3,
           2.0 * bytes / ms[0] / 1e9, ms[15] * 1e3, 2.0 * bytes / ms[15] / 1e9, md);
  };
  run("v0 library (64b div, U4)", [&] { v0<<<cap((n + 1023) / 1024, (const void*)v0, 0), 256>>>(p); });
  run("v1 magic U4", [&] { v1<4, false><<<cap((n + 1023) / 1024, (const void*)v1<4, false>, 0), 256>>>(p); });
  run("v1 magic U8", [&] { v1<8, false><<<cap((n + 2047) / 2048, (const void*)v1<8, false>, 0), 256>>>(p); });
  run("v1 magic U2", [&] { v1<2, false><<<cap((n + 511) / 512, (const void*)v1<2, false>, 0), 256>>>(p); });
  run("v5 magic U4 L2::256B", [&] { v1<4, true><<<cap((n + 1023) / 1024, (const void*)v1<4, true>, 0), 256>>>(p); });
  run("v5 magic U8 L2::256B", [&] { v1<8, true><<<cap((n + 2047) / 2048, (const void*)v1<8, true>, 0), 256>>>(p); });
  run("v3 chunk U4 (waves)", [&] { v3<4><<<(unsigned)((n + 1023) / 1024), 256>>>(p); });
  run("v3 chunk U8 (waves)", [&] { v3<8><<<(unsigned)((n + 2047) / 2048), 256>>>(p); });
  run("v3 chunk U16 (waves)", [&] { v3<16><<<(unsigned)((n + 4095) / 4096), 256>>>(p); });
  run("v4 copy U4", [&] { v4<4><<<cap((n + 1023) / 1024, (const void*)v4<4>, 0), 256>>>(p); });
  run("v4 copy U8", [&] { v4<8><<<cap((n + 2047) / 2048, (const void*)v4<8>, 0), 256>>>(p); });
  CK(cudaFuncSetAttribute(v6<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 4));
  CK(cudaFuncSetAttribute(v6<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4));
  CK(cudaFuncSetAttribute(v6<16384, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 6));
  run("v6 bulk 16K x4", [&] { v6<16384, 4><<<cap(1 << 30, (const void*)v6<16384, 4>, 16384 * 4), 256, 16384 * 4>>>(p); });
  run("v6 bulk 16K x6", [&] { v6<16384, 6><<<cap(1 << 30, (const void*)v6<16384, 6>, 16384 * 6), 256, 16384 * 6>>>(p); });
  run("v6 bulk 32K x4", [&] { v6<32768, 4><<<cap(1 << 30, (const void*)v6<32768, 4>, 32768 * 4), 256, 32768 * 4>>>(p); });
  run("cudaMemcpy D2D", [&] { CK(cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice)); });
  return 0;
}
