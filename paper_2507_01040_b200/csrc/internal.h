// internal.h -- host-side plan / parameter structs shared by the CUDA
// translation units of libclifford_b200.so (not part of the C-ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

// A/B timing switches and fault injection (CL_NO_PAIR, CL_NO_HALO, CL_TPS,
// CL_DBG_SKIP, CL_DBG_FLIP_COEFF, ...) are read ONLY by the diagnostic build
// libclifford_b200_ab.so (-DCL_AB_SWITCHES, see build.py). The production
// library never looks at the environment, so a stray variable cannot change
// its kernels or their results.
#ifdef CL_AB_SWITCHES
#define CL_ENV(name) getenv(name)
#else
#define CL_ENV(name) ((const char*)nullptr)
#endif

namespace cl {

// Arithmetic modes (values = the C-ABI cl_precision codes):
//   kPrecFp32    int8 digit slices (Ozaki scheme), exact s32 TMEM accumulation
//   kPrecTf32    one TF32 pass
//   kPrecBf16    BF16 operands
//   kPrec3xTf32  3xTF32 split (hi/lo), fp32 TMEM accumulation
enum Prec : int { kPrecFp32 = 0, kPrecTf32 = 1, kPrecBf16 = 2, kPrec3xTf32 = 3 };
constexpr int kDigitsA = 4;  // int8 digits per activation value in kPrecFp32 (31 bits)
constexpr int kDigitsW = 4;  // int8 digits per filter value (31 bits, per-column scale)
constexpr int kLevels = 4;   // digit-pair levels kept: i + j <= 3 (0-based)

constexpr int kTileM = 128;          // GEMM rows per tile (= TMEM lanes)
// exact mode: reduction length of one accumulation group. Level L sums
// (L + 1) <= 4 digit-pair products of |d_i w_j| <= 2^14 per K element, so
// |L| <= 4 * 2^14 * K < 2^31 for K <= 32000 (s32 TMEM accumulators).
constexpr int kMaxKGroup = 32000;
// 3xTF32: reduction elements per accumulation group. The tensor core's fp32
// accumulation truncates, so its error grows with the number of MMAs chained
// into one accumulator. Two measures keep max_rel_error(floor 1e-2) <= 1e-4
// at K = 13824 (profiles/r02_3xtf32_drain_study.txt):
//  * the cross terms A_lo*B_hi + A_hi*B_lo (2^-11 of the product) accumulate
//    over the whole tile in their OWN TMEM accumulator (the "lo" slot), so
//    their truncation is 2^-11 smaller and they never truncate the main sum;
//  * the A_hi*B_hi accumulator is drained every kX3GroupK elements
//    (kX3GroupK / 8 chained MMAs) into fp32 registers (round-to-nearest sums).
#ifndef CL_X3_GROUP_K
#define CL_X3_GROUP_K 192
#endif
constexpr int kX3GroupK = CL_X3_GROUP_K;
constexpr int kX3HiSlots = 3;  // rotating A_hi*B_hi slots; the 4th 128-column slot is the lo accumulator

// Change of basis (basis.cu): x' = T x splits the conv into ncol independent
// GEMMs sharing a w x w filter; T rows = (column, component), entries +-1/0,
// T T^T = 2 I.
struct Basis {
  int on;
  int ncol, w;
  int8_t T[64];   // row-major [s][blade], 8 x 8 (unused rows/cols zero)
  // every row of T and every column of T (blade) has exactly two +-1 entries:
  // x'[s] = sgn * x[fwd[s][0]] + sgn * x[fwd[s][1]], x[t] = (+-x'[inv[t][0]] +- x'[inv[t][1]]) / 2
  int8_t fwd[8][2], fwd_sgn[8][2];
  int8_t inv[8][2], inv_sgn[8][2];
};
bool find_basis(const int* g, int k, Basis* bs);

struct Sig {
  int g[3];
  int k;
  // fault injection (the reference's parity_report schedule_transform,
  // bench.py:566-576): 1 + i*8 + j negates the product-table coefficient of
  // (e_i, e_j) in kernel construction; 0 = off. Set only by CL_DBG_FLIP_COEFF="i,j".
  int flip = 0;
};
// Sig of a signature g (k values) with the CL_DBG_FLIP_COEFF fault applied.
Sig make_sig(const int* g, int k);

#if defined(__CUDACC__)
// W[(co,t),(ci,j),q] = coeff(t^j, j) f[t^j, ci, co, q]  (conv.py:188-202)
__device__ __forceinline__ float expanded_entry(const Sig& sg, const float* __restrict__ f, int nb, int C_in,
                                                int C_out, int Q, int co, int t, int ci, int j, int q) {
  const int i = t ^ j;
  int c = blade_coeff(i, j, sg.g, sg.k);
  if (sg.flip == 1 + i * 8 + j) c = -c;
  if (c == 0) return 0.f;
  const float v = __ldg(f + (((long long)i * C_in + ci) * C_out + co) * Q + q);
  return c > 0 ? v : -v;
}
// Filter in the changed basis: R(f)[r][m] = (T L_f T^T)[r][m] / 2 (first
// w x w block), L_f the expanded N_B x N_B block above; exact in fp64.
__device__ __forceinline__ double basis_entry(const Sig& sg, const Basis& bs, const float* __restrict__ f,
                                              int C_in, int C_out, int Q, int co, int r, int ci, int m, int q) {
  const int nb = 1 << sg.k;
  double s = 0.0;
  for (int a = 0; a < nb; ++a) {
    const int ta = bs.T[r * 8 + a];
    if (!ta) continue;
    for (int b = 0; b < nb; ++b) {
      const int tb = bs.T[m * 8 + b];
      if (!tb) continue;
      s += (double)(ta * tb) * (double)expanded_entry(sg, f, nb, C_in, C_out, Q, co, a, ci, b, q);
    }
  }
  return 0.5 * s;
}
#endif
constexpr int kConvThreads = 384;    // 12 warps, see conv_tc.cu
// 20 warps (four epilogue warp groups) for the int8 mode (one accumulator slot to drain) and the
// 2-D / 1-D fp32-accumulator modes (measured faster); 12 warps (two groups) for 3-D bf16 / tf32
// (their 3-D epilogue spills at 96 registers) and 3xTF32 (warps 8-11 split A)
// 3xTF32 (prec 3): 16 warps = two epilogue groups (they hold the drained
// partial sums in registers) + the splitter group
#ifndef CL_X3_EPI_GROUPS
#define CL_X3_EPI_GROUPS 2
#endif
constexpr int kX3EpiGroups = CL_X3_EPI_GROUPS;  // 3xTF32 epilogue warp groups (each drains 128 / groups columns)
constexpr int conv_threads(int prec, int nb) {
  return prec == 3 ? 128 * (2 + kX3EpiGroups) : ((prec == 0 || nb <= 4) ? 640 : kConvThreads);
}
constexpr int kMaxSmem = 232448;     // 227 KB opt-in dynamic shared memory per CTA

// Tiling plan of one conv layer, fixed at create time (conv.py:101-140 fixes
// its CPU kernel parameters at the same point).
struct ConvPlan {
  int k, nb;            // spatial rank, blades
  int ka;               // algebra rank (nb = 2^ka); differs from k for the linear layer
  Basis bs;             // change of basis (bs.on) for M2(R) / M2(C) signatures
  int prec;             // Prec
  int esize;            // operand element bytes (4 fp32/tf32, 2 bf16)
  int rb;               // bytes of one A row-group (16 or 32)
  int epg;              // operand elements per row-group (rb / esize)
  int merged_bc;        // tensor-map dim 4 = b*G + g (3-D) instead of separate (g, b) dims
  int packed;           // operand is a packed 16-byte-group copy (bf16, or fp32 in 1-D)
  int cpg;              // channels per row-group of the A operand
  int G;                // row-groups per sample in the A tensor (padded)
  int gs;               // row-groups per pipeline stage
  int ks;               // MMA K-steps (32 B of K per row) per stage
  int n_gs;             // stages per filter tap
  int Q, d_filter;      // taps
  int k_iters;          // Q * n_gs
  int cps;              // channels per stage = gs * epg / nb
  int N, n_tile, n_ntiles;
  int tx, ty, tz;       // output tile extents (tx*ty*tz == 128)
  uint32_t a_bytes, b_img_bytes, b_bytes, stage_bytes;
  int n_img;            // B images per stage (2 for 3xTF32 hi/lo, 4 int8 digits)
  int n_a;              // A tiles per stage (2 for 3xTF32 hi/lo, 4 int8 digits)
  int n_tma_a;          // A tensor loads per stage (4 for int8 digits, else 1)
  int levels;           // TMEM accumulators per tile (4 digit levels for kPrecFp32)
  int acc_slots;        // accumulator buffers (2 = epilogue overlaps next tile's MMA)
  // accumulation groups (exact mode, long reductions): the s32 level
  // accumulators are drained every `drain` pipeline stages -- each group's
  // reduction length stays <= kMaxKGroup -- and the groups are combined
  // exactly in int64 by the epilogue; drain = stages per tile (one group) otherwise
  int drain, n_groups, stages_per_tile;
  int stages;
  uint32_t tmem_cols;
  size_t smem_bytes;
  // halo mode: each channel group's input halo (hx x hy x hz pixels) is loaded
  // once and reused by every filter tap through descriptor offsets
  int halo, hx, hy, hz, hs;
  uint32_t halo_bytes, halo_slot, ring_off;
  int tps;  // halo mode: filter taps (B images) per pipeline stage
  // 2-SM MMA (cta_group::2): a CTA pair computes M = 256 rows; each CTA holds
  // its 128 A rows and half of the B columns (the filter images are laid out
  // as two contiguous column halves per stage)
  int pair;
};

struct ConvKParams {
  int B, k, nb;
  int d_in, d_out, pad;
  int tx, ty, tz, ntx, nty, ntz;
  int n_ntiles, n_tile, N, C_out;
  long long num_tiles;
  int d_filter, n_gs, gs, G, merged_bc, k_iters, ks;
  uint32_t a_bytes, b_bytes, b_img_bytes, stage_bytes, tmem_cols;
  int stages, n_a, n_tma_a, levels, acc_slots;
  int drain, n_groups;        // accumulation group = `drain` pipeline stages; n_groups per tile (see ConvPlan)
  long long* grp_scratch;     // n_groups > 1: per-(CTA, row, column) int64 partial sums of the exact mode
  int cs;                     // cluster size: 2 for a 2-SM (cta_group::2) pair, else 1
  int pair;                   // 2-SM MMA: M = 256 over the pair, B columns split between the two CTAs
  int halo, hx, hy, hz, hs;   // halo mode (see ConvPlan)
  int tps;                    // halo mode: filter taps per B stage
  int bcls;                   // int8 epilogue change-of-basis pattern class (see conv_tc.cu), 0 = generic
  int epx;                    // A tensor map with merged (pixel, row) inner dim: 8-byte elements per pixel, else 0
  uint32_t halo_bytes, halo_slot, ring_off;
  Basis bs;                   // change of basis: rows = (pixel, column), epilogue inverse transform
  long long num_m_tiles;      // real pixel tiles (tiles beyond are cluster padding)
  int dbg_skip;
  unsigned long long* dbg_acc;  // timing instrumentation (CL_DBG_CLK): cycle counters, else null               // timing experiments only: bit 0 skips A loads, bit 1 skips B loads (garbage results)
  const uint8_t* b_img;
  const float* a_scale;       // kPrecFp32: per-sample power-of-two scale of the A digits
  const float* w_scale;       // kPrecFp32: per-column power-of-two scale of the B digits
  const float* bias;          // (NB, C_out)
  const float* bias_t;        // (C_out, NB) copy: one vector load per (channel, lane)
  float* y;                   // fp32 protocol output (or null)
  __nv_bfloat16* y_bf16;      // bf16 A-ready output (or null)
  int ybf_groups;             // groups per sample of the packed bf16 output tensor (B, Gy, P, 16 B)
  const float* resid;         // residual source (protocol layout) or null
  int res_side, res_crop;     // residual spatial side and centre-crop offset
  int act_mode;               // -1 none, 0 Linear, 1 Sum, 2 Mean
  const float* act_w;         // (C_out, NB) blade-keyed weights / 0-1 mask
  const float* act_b;         // (C_out) Linear bias
  float act_K;                // K as float (Mean divisor)
  unsigned act_kmask;         // kernel blades of the gate (non-kernel blades are selected out, never * 0)
  unsigned* amax_out;         // int8 epilogue: per-sample atomicMax of finite |stored value| (float bits), or null
  unsigned* nf_out;           // int8 epilogue: per-sample flag, a stored value is Inf / NaN (with amax_out)
  unsigned long long* tile_ctr;  // dynamic tile scheduler: zeroed work counter (cluster tiles), or null = static order
};

struct ActParams {
  const float* x;
  float* y;
  long long n_mv;     // B * C * P multivectors
  long long P;
  int C;
  int mode;
  const float* w;     // (C, NB)
  const float* b;     // (C)
  float Kf;
  unsigned kmask;     // bit j set: blade j is a kernel blade (only those enter the gate)
  int K;              // kernel blades, in the caller's order ki[0..K)
  int ki[8];
  // exact unsigned division of n < 2^31 by P and by C: q = (n * mag) >> sh
  // (filled by launch_act)
  unsigned magP, shP, magC, shC;
};

// launchers (conv_tc.cu / expand.cu / activation.cu)
cudaError_t launch_conv(const ConvPlan& plan, const CUtensorMap& tmap, const CUtensorMap& bmap,
                        const ConvKParams& p, int grid, cudaStream_t s);
cudaError_t launch_expand_ref(const int* g, int k, const float* f, int C_in, int C_out, int Q,
                              float* out, cudaStream_t s);
cudaError_t launch_expand_images(const int* g, const ConvPlan& plan, const float* f, int C_in,
                                 int C_out, const float* w_scale, uint8_t* img, cudaStream_t s);
cudaError_t launch_transpose(const float* in, float* out, int rows, int cols, cudaStream_t s);
cudaError_t launch_pack_rows(const float* x, void* out, int nb, int esize, long long B, int C, long long P,
                             int G, const Basis& bs, cudaStream_t s);
cudaError_t launch_act(int nb, const ActParams& p, cudaStream_t s);
// gate_preactivation (s per multivector, written to p.y as (B, C, P)) and
// gather_vpack (the K kernel blades in ki order, p.y as (B, C, P, K))
cudaError_t launch_act_preact(int nb, const ActParams& p, cudaStream_t s);
cudaError_t launch_act_gather(int nb, const ActParams& p, cudaStream_t s);
// kPrecFp32 operand preparation (slice.cu): per-sample max over the finite
// values + a per-sample non-finite flag (zeroed by the launcher)
cudaError_t launch_sample_absmax(const float* x, long long B, long long per_sample, unsigned* amax, unsigned* flags,
                                 cudaStream_t s);
// small layers: per-sample absmax + slicing in one cluster launch (no amax
// buffer; flags[b] is written, not accumulated)
cudaError_t launch_absmax_slice(const float* x, int8_t* digits, float* scale, unsigned* flags, int nb, long long B,
                                int C, long long P, int G, const Basis& bs, cudaStream_t s);
// exact mode: NaN over the receptive fields of non-finite inputs (flagged samples only)
struct PoisonParams {
  const float* x;           // conv input (B, C_in, d_in^k, nb)
  float* y;                 // conv output (B, C_out, d_out^k, nb)
  const unsigned* flags;    // per-sample: input holds Inf / NaN
  unsigned* flags_out;      // optional: per-sample flags for the next conv (block)
  long long B, P_in, P_out;
  int C_in, C_out, nb, k, d_in, d_out, d_filter, pad;
};
cudaError_t launch_poison_nonfinite(const PoisonParams& p, cudaStream_t s);
cudaError_t launch_slice_input(const float* x, const unsigned* amax, int8_t* digits, float* scale,
                               int nb, long long B, int C, long long P, int G, const Basis& bs, cudaStream_t s);
cudaError_t launch_weight_colscale(const int* g, const ConvPlan& pl, const float* f, int C_in, int C_out,
                                   float* w_scale, cudaStream_t s);

int num_sms();
void count_launch(int n = 1);
// Host-side launch helpers, cached per (kernel, device): resident blocks per SM
// of a kernel (the occupancy calculator costs microseconds per call) and the
// dynamic shared-memory opt-in (cudaFuncSetAttribute once, not per launch).
int resident_blocks_per_sm(const void* kern, int threads, size_t smem);
cudaError_t ensure_smem_optin(const void* kern, int bytes);

}  // namespace cl
