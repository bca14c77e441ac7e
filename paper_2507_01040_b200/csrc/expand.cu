// expand.cu -- (1) on-device Clifford kernel construction.
//
// The real (C_out*N_B) x (C_in*N_B) x Q filter of conv.py:188-202 has entry
//   W[(co,t), (ci,j), q] = coeff(t^j, j) * f[t^j, ci, co, q],
// coeff from the blade-product table of the signature (algebra.py:87-99),
// including zero (degenerate) and negative metric values. Every entry is a
// single signed filter value, so construction is exact.
//
// Two outputs:
//  * the reference layout (for parity tests / export), and
//  * the tensor-core operand images used by conv_tc.cu, built ONCE per layer
//    at create time: per (N-tile, K-iteration) a contiguous block of K-major
//    SWIZZLE_NONE UMMA core matrices [image][k-step][2 x 16 B chunks][n_tile
//    rows][16 B], images = {hi, lo} for 3xTF32, {tf32}, {bf16} or the four
//    four int8 digits of the fp32-accurate mode (per-column power-of-two scale).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace cl {

Sig make_sig(const int* g, int k) {
  Sig sg{{0, 0, 0}, k};
  for (int i = 0; i < k; ++i) sg.g[i] = g[i];
  static const int flip = [] {
    const char* e = CL_ENV("CL_DBG_FLIP_COEFF");
    int i = 0, j = 0;
    return (e && sscanf(e, "%d,%d", &i, &j) == 2 && i >= 0 && i < 8 && j >= 0 && j < 8) ? 1 + i * 8 + j : 0;
  }();
  sg.flip = flip;
  return sg;
}

__global__ void expand_ref_kernel(Sig sg, const float* __restrict__ f, int C_in, int C_out, int Q,
                                  float* __restrict__ out) {
  const int nb = 1 << sg.k;
  const long long total = (long long)C_out * nb * C_in * nb * Q;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(idx % Q);
    long long r = idx / Q;
    const int j = (int)(r % nb); r /= nb;
    const int ci = (int)(r % C_in); r /= C_in;
    const int t = (int)(r % nb);
    const int co = (int)(r / nb);
    out[idx] = expanded_entry(sg, f, nb, C_in, C_out, Q, co, t, ci, j, q);
  }
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// One thread per (n_tile, k_iter, k_local, row); writes every image.
__global__ void expand_img_kernel(Sig sg, const float* __restrict__ f, int C_in, int C_out,
                                  ConvPlan pl, const float* __restrict__ w_scale, uint8_t* __restrict__ img) {
  const int nb = pl.nb;
  const int k_stage = pl.ks * 32 / pl.esize;  // K elements per stage
  const long long total = (long long)pl.n_ntiles * pl.k_iters * k_stage * pl.n_tile;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx % pl.n_tile);
    long long r = idx / pl.n_tile;
    const int kl = (int)(r % k_stage); r /= k_stage;
    const int kit = (int)(r % pl.k_iters);
    const int nt = (int)(r / pl.k_iters);
    const int q = kit / pl.n_gs, gsi = kit % pl.n_gs;
    const int n = nt * pl.n_tile + row;
    const int wd = pl.bs.on ? pl.bs.w : nb;  // components per channel in the operand basis
    const int co = n / wd, t = n % wd;
    const int ci = gsi * pl.cps + kl / wd, j = kl % wd;
    double wv = 0.0;
    if (co < C_out && ci < C_in)
      wv = pl.bs.on ? basis_entry(sg, pl.bs, f, C_in, C_out, pl.Q, co, t, ci, j, q)
                    : (double)expanded_entry(sg, f, nb, C_in, C_out, pl.Q, co, t, ci, j, q);
    const float w = (float)wv;
    // position inside the stage image
    const int byte_k = kl * pl.esize;
    const int s = byte_k >> 5, h = (byte_k >> 4) & 1, e = (byte_k & 15) / pl.esize;
    // 2-SM pair: the stage holds two contiguous column halves, one per CTA,
    // each laid out like a full stage of n_tile / 2 rows
    const int nrow = pl.pair ? pl.n_tile / 2 : pl.n_tile;
    const int half = row / nrow, rr = row % nrow;
    const size_t img_stride = pl.pair ? pl.b_img_bytes / 2 : pl.b_img_bytes;
    // halo plans: blocks ordered (N tile, channel group, CTA half, tap), so one
    // CTA's taps of a channel group are contiguous (one load per multi-tap
    // stage); otherwise (N tile, k_iter) with the two halves inside
    const size_t b_half = pl.pair ? pl.b_bytes / 2 : pl.b_bytes;
    uint8_t* base = pl.halo ? img + ((((size_t)nt * pl.n_gs + gsi) * (pl.pair ? 2 : 1) + half) * pl.Q + q) * b_half
                            : img + ((size_t)nt * pl.k_iters + kit) * pl.b_bytes + (size_t)half * b_half;
    const size_t off = (size_t)s * nrow * 32 + (size_t)h * nrow * 16 + (size_t)rr * 16 + (size_t)e * pl.esize;
    if (pl.prec == kPrecFp32) {
      int8_t d[kDigitsW];
      digits_b256_d<kDigitsW>(wv / (double)__ldg(w_scale + n), d);
#pragma unroll
      for (int k = 0; k < kDigitsW; ++k) *reinterpret_cast<int8_t*>(base + (size_t)k * img_stride + off) = d[k];
    } else if (pl.prec == kPrec3xTf32) {
      // hi = w rounded to tf32, lo = the remainder rounded to tf32: both
      // operands reach the tensor core exactly (it reads the top 19 bits)
      const float hi = tf32_rna(w);
      *reinterpret_cast<float*>(base + off) = hi;
      *reinterpret_cast<float*>(base + img_stride + off) = tf32_rna((float)(wv - (double)hi));
    } else if (pl.prec == kPrecTf32) {
      *reinterpret_cast<float*>(base + off) = tf32_rna(w);
    } else {
      *reinterpret_cast<__nv_bfloat16*>(base + off) = __float2bfloat16_rn(w);
    }
  }
}

static unsigned grid_for(long long total) {
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  return (unsigned)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_expand_ref(const int* g, int k, const float* f, int C_in, int C_out, int Q,
                              float* out, cudaStream_t s) {
  const Sig sg = make_sig(g, k);
  const int nb = 1 << k;
  const long long total = (long long)C_out * nb * C_in * nb * Q;
  expand_ref_kernel<<<grid_for(total), 256, 0, s>>>(sg, f, C_in, C_out, Q, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_expand_images(const int* g, const ConvPlan& pl, const float* f, int C_in,
                                 int C_out, const float* w_scale, uint8_t* img, cudaStream_t s) {
  const Sig sg = make_sig(g, pl.ka);
  const long long total =
      (long long)pl.n_ntiles * pl.k_iters * (pl.ks * 32 / pl.esize) * pl.n_tile;
  expand_img_kernel<<<grid_for(total), 256, 0, s>>>(sg, f, C_in, C_out, pl, w_scale, img);
  count_launch();
  return cudaGetLastError();
}

}  // namespace cl
