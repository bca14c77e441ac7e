// conv_tc.cu -- (2) Clifford convolution as an implicit GEMM on tcgen05.
//
// GEMM view of conv.py:151-182:
//   M = output pixels of one sample tile (128 rows = TMEM lanes),
//   N = C_out * N_B  (n = co*N_B + t),
//   K = Q * C_in * N_B (k = (q, ci, j)),
//   A[m, k] = x[b, ci, p(m) + q, j]   -- never materialised: each pipeline
//             stage TMA-loads the shifted input box (j, x, y[, z], channels)
//             straight from the protocol layout (B, C, d^k, N_B); "same"
//             padding and tile overhang come from TMA out-of-bounds zero fill.
//   B[n, k] = expanded Clifford filter (subsystem (1), expand.cu), stored as
//             ready-to-copy UMMA K-major tiles, one bulk copy per stage.
//
// Warp roles (384 threads, 1 CTA per SM, persistent over tiles):
//   warp 0      TMA producer (one lane)
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::tf32 / kind::f16,
//               accumulator double-buffered in TMEM (2 x N_TILE fp32 columns)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld -> bias [-> activation] [-> residual]
//               -> coalesced stores in the protocol layout (thread = pixel
//               row, holds all N_B blades of each output channel)
//   warps 12-15 3xTF32 splitter: A -> (A_hi, A_lo) in shared memory (the
//               3xTF32 kernel has 512 threads: epilogue warps 4-11)
//
// 3xTF32: D = (A_lo*B_hi + A_hi*B_lo) + A_hi*B_hi with hi = x rounded to
// nearest tf32 and lo = x - hi rounded to tf32. The cross terms accumulate in
// their own TMEM accumulator over the whole tile; A_hi*B_hi in rotating
// group slots drained into fp32 registers (x3_drain_groups, kX3GroupK).
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace cl {

// Timing instrumentation (CL_DBG_CLK cycle counters, CL_DBG_SKIP work
// skipping) exists only in the diagnostic build; the production kernels
// compile it out.
#ifdef CL_AB_SWITCHES
constexpr bool kDbg = true;
#else
constexpr bool kDbg = false;
#endif
__device__ __forceinline__ int dbg_skip(const ConvKParams& p) { return kDbg ? p.dbg_skip : 0; }

// Gate of one multivector. Non-kernel blades are selected out (kmask), not
// weighted by zero: the reference never reads them (activation.py:142-162).
template <int NB>
__device__ __forceinline__ float act_gate(const float (&v)[NB], int mode, const float* __restrict__ w,
                                          float bias, float Kf, unsigned kmask) {
  float wv[NB];  // the channel's NB gate weights: vector loads (w = act_w + channel * NB is 8 / 16-byte aligned)
  if constexpr (NB == 2) {
    const float2 w2 = __ldg(reinterpret_cast<const float2*>(w));
    wv[0] = w2.x; wv[1] = w2.y;
  } else {
#pragma unroll
    for (int j = 0; j < NB / 4; ++j) {
      const float4 w4 = __ldg(reinterpret_cast<const float4*>(w) + j);
      wv[4 * j] = w4.x; wv[(4 * j + 1) % NB] = w4.y; wv[(4 * j + 2) % NB] = w4.z; wv[(4 * j + 3) % NB] = w4.w;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const float t = fmaf(v[j], wv[j], s);
    s = ((kmask >> j) & 1u) ? t : s;
  }
  if (mode == 0) s += bias;
  else if (mode == 2) s = s * (1.f / Kf);
  // fast exp / reciprocal (~1e-7 relative on the gate, far inside the block's bounds): the
  // precise forms' slow-path CALLs serialised the channels of an epilogue chunk
  return __frcp_rn(1.f + __expf(-s));
}

// MMA of the precision mode, 1-SM or 2-SM (pair leader).
template <int PREC, bool PAIR>
__device__ __forceinline__ void mma_mode(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (PREC == kPrecFp32) {
    if constexpr (PAIR) mma_i8_cg2(d, a, b, idesc, acc); else mma_i8(d, a, b, idesc, acc);
  } else if constexpr (PREC == kPrecBf16) {
    if constexpr (PAIR) mma_bf16_cg2(d, a, b, idesc, acc); else mma_bf16(d, a, b, idesc, acc);
  } else {
    if constexpr (PAIR) mma_tf32_cg2(d, a, b, idesc, acc); else mma_tf32(d, a, b, idesc, acc);
  }
}

template <int PREC, bool PAIR>
__device__ __forceinline__ void mma_mode_g(uint32_t issue, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t acc) {
  if constexpr (PREC == kPrecFp32) {
    if constexpr (PAIR) mma_i8_cg2_g(issue, d, a, b, idesc, acc); else mma_i8_g(issue, d, a, b, idesc, acc);
  } else if constexpr (PREC == kPrecBf16) {
    if constexpr (PAIR) mma_bf16_cg2_g(issue, d, a, b, idesc, acc); else mma_bf16_g(issue, d, a, b, idesc, acc);
  } else {
    if constexpr (PAIR) mma_tf32_cg2_g(issue, d, a, b, idesc, acc); else mma_tf32_g(issue, d, a, b, idesc, acc);
  }
}
template <int PREC, bool PAIR>
__device__ __forceinline__ void mma_mode_s(uint32_t issue, uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo,
                                           uint32_t bhi, uint32_t idesc, uint32_t acc) {
  if constexpr (PREC == kPrecFp32) {
    if constexpr (PAIR) mma_i8_cg2_s(issue, d, alo, ahi, blo, bhi, idesc, acc);
    else mma_i8_s(issue, d, alo, ahi, blo, bhi, idesc, acc);
  } else if constexpr (PREC == kPrecBf16) {
    if constexpr (PAIR) mma_bf16_cg2_s(issue, d, alo, ahi, blo, bhi, idesc, acc);
    else mma_bf16_s(issue, d, alo, ahi, blo, bhi, idesc, acc);
  } else {
    if constexpr (PAIR) mma_tf32_cg2_s(issue, d, alo, ahi, blo, bhi, idesc, acc);
    else mma_tf32_s(issue, d, alo, ahi, blo, bhi, idesc, acc);
  }
}
template <bool PAIR>
__device__ __forceinline__ void commit_g(uint32_t issue, uint64_t* bar) {
  if constexpr (PAIR) mma_commit_cg2_g(issue, bar); else mma_commit_g(issue, bar);
}
// The ks K steps of one stage (tf32 / bf16 modes) in one asm block (common.cuh
// mma_*_ks): strides in 16-byte descriptor units, acc0 = first MMA's accumulate.
template <int PREC, bool PAIR, int KS>
__device__ __forceinline__ void mma_stage_t(uint32_t issue, uint32_t d, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                            uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_st, uint32_t b_st) {
  if constexpr (PREC == kPrecBf16) {
    if constexpr (PAIR) mma_bf16_cg2_ks<KS>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st);
    else mma_bf16_ks<KS>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st);
  } else {
    if constexpr (PAIR) mma_tf32_cg2_ks<KS>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st);
    else mma_tf32_ks<KS>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st);
  }
}
template <int PREC, bool PAIR>
__device__ __forceinline__ void mma_stage(int ks, uint32_t issue, uint32_t d, uint32_t a_lo, uint32_t a_hi,
                                          uint32_t b_lo, uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_st,
                                          uint32_t b_st) {
  switch (ks) {
    case 1: mma_stage_t<PREC, PAIR, 1>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st); break;
    case 2: mma_stage_t<PREC, PAIR, 2>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st); break;
    case 4: mma_stage_t<PREC, PAIR, 4>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st); break;
    default: mma_stage_t<PREC, PAIR, 8>(issue, d, a_lo, a_hi, b_lo, b_hi, idesc, acc0, a_st, b_st); break;
  }
}

// A-operand TMA box at (x, c1, c2, c3). With a merged (pixel x row-bytes)
// inner dimension of 8-byte elements (p.epx per pixel; one TMA line per tile
// row instead of one per pixel) the coordinates shift left by one.
template <bool PAIR>
__device__ __forceinline__ void load_a_box(const ConvKParams& p, void* dst, const CUtensorMap* map, uint64_t* bar,
                                           int x, int c1, int c2, int c3) {
  if constexpr (PAIR) {  // bytes complete on the pair leader's barrier
    if (p.epx) tma_load_5d_cg2(dst, map, bar, x * p.epx, c1, c2, c3, 0);
    else tma_load_5d_cg2(dst, map, bar, 0, x, c1, c2, c3);
  } else {
    if (p.epx) tma_load_5d(dst, map, bar, x * p.epx, c1, c2, c3, 0);
    else tma_load_5d(dst, map, bar, 0, x, c1, c2, c3);
  }
}

// register-array picks with a runtime index (selects, no local memory)
template <int W>
__device__ __forceinline__ float pick_wf(const float (&a)[W], int i) {
  if constexpr (W == 1) return a[0];
  else if constexpr (W == 2) return i ? a[1] : a[0];
  else return (i & 2) ? ((i & 1) ? a[3] : a[2]) : ((i & 1) ? a[1] : a[0]);
}
template <int W>
__device__ __forceinline__ long long pick_w(const long long (&a)[W], int i) {
  if constexpr (W == 1) return a[0];
  else if constexpr (W == 2) return i ? a[1] : a[0];
  else return (i & 2) ? ((i & 1) ? a[3] : a[2]) : ((i & 1) ? a[1] : a[0]);
}

// Persistent tile order: CTAs of one cluster (consecutive blockIdx, rank r)
// take consecutive pixel tiles of the SAME N tile so they can share each B
// stage by multicast; N tiles of one pixel-tile group run back to back (A
// reuse in L2). Returns false for cluster padding tiles (no output).
__device__ __forceinline__ bool decode_tile(const ConvKParams& p, long long t, int crank, int& nt, int& tx,
                                            int& ty, int& tz, int& b) {
  const long long c = t / p.cs;
  nt = (int)(c % p.n_ntiles);
  long long m = (c / p.n_ntiles) * p.cs + crank;
  const bool real = m < p.num_m_tiles;
  if (!real) m = p.num_m_tiles - 1;
  if (p.k == 1) {  // 1-D: tile rows span (position x, sample): b = first sample of the tile
    tx = (int)(m % p.ntx);
    ty = (int)(m / p.ntx);
    tz = 0;
    b = ty * p.ty;
    return real;
  }
  tx = (int)(m % p.ntx); m /= p.ntx;
  ty = (int)(m % p.nty); m /= p.nty;
  tz = (int)(m % p.ntz);
  b = (int)(m / p.ntz);
  return real;
}

// An epilogue warp hands an accumulator slot back to the MMA warp: one
// arrival per warp (the barrier counts warps of both CTAs of a pair, on the
// leader) after every lane's TMEM loads are fenced. Per-thread arrivals had
// sent 256 remote arrives per slot and CTA over DSMEM.
template <bool PAIR>
__device__ __forceinline__ void release_acc(uint64_t* bar) {
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    if constexpr (PAIR) mbar_arrive_leader_relaxed(bar); else mbar_arrive(bar);
  }
}

// Exact mode with several accumulation groups per tile (reductions longer
// than kMaxKGroup): drain the first n_groups - 1 groups of this thread's TMEM
// row into its int64 partial sums, S = L0 2^24 + L1 2^16 + L2 2^8 + L3 per
// column (each group's s32 levels are exact, so the sum is exact); the last
// group is combined with them in the epilogue's phase 1. Only the GROUPS
// instantiation of the kernel contains it (the extra loop would cost the
// common epilogue registers).
template <bool PAIR>
__device__ __forceinline__ void drain_groups(const ConvKParams& p, uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                                          int ew, int row, int c_beg, int c_end, uint32_t slot_cols, int slots,
                                          int& acc, uint32_t& acc_phase) {
  long long* scr = p.grp_scratch + ((long long)blockIdx.x * kTileM + row) * p.n_tile;
  for (int grp = 0; grp + 1 < p.n_groups; ++grp) {
    mbar_wait_sleep(&tfull[acc], acc_phase, 64);
    tc_fence_after();
    const uint32_t ta = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)acc * slot_cols;
    for (int c0 = c_beg; c0 < c_end; c0 += 4) {
      uint32_t l0[4], l1[4], l2[4], l3[4];
      tmem_ldn<4>(ta + (uint32_t)c0, l0);
      tmem_ldn<4>(ta + (uint32_t)(p.n_tile + c0), l1);
      tmem_ldn<4>(ta + (uint32_t)(2 * p.n_tile + c0), l2);
      tmem_ldn<4>(ta + (uint32_t)(3 * p.n_tile + c0), l3);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        long long sv = ((long long)(int)l0[c] << 24) + ((long long)(int)l1[c] << 16) +
                       ((long long)(int)l2[c] << 8) + (long long)(int)l3[c];
        if (grp > 0) sv += scr[c0 + c];
        scr[c0 + c] = sv;
      }
    }
    release_acc<PAIR>(&tempty[acc]);
    if (++acc == slots) { acc = 0; acc_phase ^= 1; }
  }
}

// 3xTF32 accumulation groups: the MMA warp rotates `slots` TMEM slots, one
// group of kX3GroupK reduction elements of A_hi*B_hi each, and accumulates the
// cross terms of the whole tile in the lo accumulator behind them. This thread
// drains the first n_groups - 1 groups of its row (columns [c_beg, c_end))
// into fp32 registers with round-to-nearest adds, then adds the sums and the
// lo accumulator into the last group's slot in TMEM (tcgen05.st), hands the
// lo accumulator back and returns with that slot full, so the regular
// epilogue reads the complete accumulator. (The tensor core's fp32
// accumulation truncates; over K = 13824 its error reached 7e-3 under the
// reference metric, profiles/r02_3xtf32_drain_study.txt.)
template <bool PAIR>
__device__ __forceinline__ void x3_drain_groups(const ConvKParams& p, uint64_t* tfull, uint64_t* tempty,
                                                uint32_t tmem_base, int ew, int c_beg, int c_end, uint32_t slot_cols,
                                                int slots, int& acc, uint32_t& acc_phase) {
  constexpr int kCh = (128 / kX3EpiGroups + 15) / 16;  // 16-column chunks of this thread's share
  float sm[16 * kCh];
#pragma unroll
  for (int i = 0; i < 16 * kCh; ++i) sm[i] = 0.f;
  const uint32_t lane_base = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)c_beg;
  for (int grp = 0; grp < p.n_groups; ++grp) {
    mbar_wait_sleep(&tfull[acc], acc_phase, 20);
    tc_fence_after();
    const long long dbg_d0 = (kDbg && p.dbg_acc) ? clock64() : 0;
    const uint32_t ta = lane_base + (uint32_t)acc * slot_cols;
    const bool last = grp + 1 == p.n_groups;
#pragma unroll
    for (int j = 0; j < kCh; ++j) {
      if (c_beg + 16 * j >= c_end) break;
      uint32_t r[16];
      if (last) {  // the tile's cross terms first (one register buffer: two in flight spilled)
        tmem_ld16(lane_base + (uint32_t)kX3HiSlots * slot_cols + (uint32_t)(16 * j), r);
        tmem_ld_wait_dep16(r);
#pragma unroll
        for (int i = 0; i < 16; ++i) sm[16 * j + i] += __uint_as_float(r[i]);
      }
      tmem_ld16(ta + (uint32_t)(16 * j), r);
      tmem_ld_wait_dep16(r);
      if (!last) {
#pragma unroll
        for (int i = 0; i < 16; ++i) sm[16 * j + i] += __uint_as_float(r[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(sm[16 * j + i] + __uint_as_float(r[i]));
        tmem_st16(ta + (uint32_t)(16 * j), r);
      }
    }
    if (last) {
      release_acc<PAIR>(&tempty[kX3HiSlots]);  // lo accumulator read: the next tile may overwrite it
      tmem_st_wait();  // the regular epilogue reads this slot next (same thread, same lanes)
      return;
    }
    release_acc<PAIR>(&tempty[acc]);
    if (kDbg && p.dbg_acc && threadIdx.x == 128) {  // timing instrumentation: drain cycles per group
      atomicAdd(p.dbg_acc + 11, (unsigned long long)(clock64() - dbg_d0));
      atomicAdd(p.dbg_acc + 12, 1ull);
    }
    if (++acc == slots) { acc = 0; acc_phase ^= 1; }
  }
}

// BCLS: change-of-basis pattern class of the int8 epilogue. 1 = the M2(C)
// basis of the (1,1,1) family: each lane's blades use own rows {0,0,3,3} and
// partner rows {2,2,1,1} (compile-time picks, 2 shuffles per channel); 0 = any.
template <int NB, int PREC, bool PAIR, int BCLS = 0, bool GROUPS = false>
__global__ void __launch_bounds__(conv_threads(PREC, NB), 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap bmap,
                   const __grid_constant__ ConvKParams p) {
  constexpr bool kSplit = (PREC == kPrec3xTf32);
  constexpr bool kInt8 = (PREC == kPrecFp32);
  // 3xTF32 pairs (halo mode only): each CTA's A halo lands on its OWN barrier
  // for its splitter, whose "split done" arrivals go to the leader's barrier
  constexpr bool kAOwn = kSplit;
  // 2-D bf16 / tf32 layers never change basis (capi.cu use_basis): their
  // kernels carry no basis epilogue
  constexpr bool kBasisEpi = !(NB == 4 && (PREC == kPrecTf32 || PREC == kPrecBf16));
  // epilogue warp groups: warps 4-7, plus warps 8-11 when they are not the
  // 3xTF32 splitter (each group drains half of the accumulator columns)
  // (3xTF32: warps 4-11, the splitter is warps 12-15)
  constexpr int kEpiGroups = kSplit ? kX3EpiGroups : (conv_threads(PREC, NB) == 640 ? 4 : 2);
  // A row-group bytes: packed 16-byte groups for bf16 / int8 digits / 1-D,
  // otherwise one protocol multivector (16 B in 2-D, 32 B in 3-D)
  constexpr int RB = (PREC == kPrecBf16 || kInt8 || NB == 2) ? 16 : NB * 4;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const int HS = p.halo ? p.hs : 0;
  uint8_t* ring = smem + p.ring_off;  // pipeline stages (after the halo buffers in halo mode)
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)S * p.stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* lo_ready = empty + S;
  uint64_t* tfull = lo_ready + S;  // accumulator slots: 4 barriers each (3xTF32 rotates 4 slots)
  uint64_t* tempty = tfull + 4;
  uint64_t* hfull = tempty + 4;   // halo buffers: loaded
  uint64_t* hempty = hfull + 4;   //               consumed by the last tap's MMAs (up to 4 slots)
  uint64_t* hlo = hempty + 4;     //               3xTF32 split done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hlo + 4);
  constexpr int kSchedR = 8;       // tile-scheduler ring depth (> tiles the producer may lead the epilogue by)
  uint64_t* sfull = hlo + 5;       // ring slot published
  uint64_t* sempty = sfull + kSchedR;  // ring slot read by every consumer warp (on the leader)
  long long* sids = reinterpret_cast<long long*>(sempty + kSchedR);

  // warp index through a shuffle: ptxas then knows it is warp-uniform, so the
  // role branches below are uniform and each role's loop values can live on
  // the uniform datapath (with threadIdx.x >> 5 the MMA issue loop ran on
  // vector registers and R2UR'd every descriptor)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;

  const int cs = p.cs;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // one MMA commit (the pair leader's reaches both CTAs)
      mbar_init(&lo_ready[s], 128);
    }
    for (int a = 0; a < 4; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * kEpiGroups * (PAIR ? 2 : 1));  // one per epilogue warp of both CTAs, on the leader
    }
    for (int a = 0; a < 4; ++a) {
      mbar_init(&hfull[a], 1);
      mbar_init(&hempty[a], 1);
      mbar_init(&hlo[a], 128 * (PAIR ? 2 : 1));
    }
    // consumers of the tile ring: the MMA warp, the peer's producer, every
    // epilogue / splitter warp of both CTAs (all arrive on the leader's copy)
    const uint32_t n_sched = 1u + (PAIR ? 1u : 0u) + (uint32_t)(4 * kEpiGroups + (kSplit ? 4 : 0)) * (PAIR ? 2u : 1u);
    for (int r = 0; r < kSchedR; ++r) {
      mbar_init(&sfull[r], 1);
      mbar_init(&sempty[r], n_sched);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmap);
    if constexpr (PAIR) tma_prefetch_desc(&bmap);
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_cg2(tmem_slot, p.tmem_cols);
    else tmem_alloc(tmem_slot, p.tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // the pair's barriers and TMEM exist before any cross-CTA traffic
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform (see `warp`)
  const int crank = cs > 1 ? (int)cluster_ctarank() : 0;

  const long long num_tiles = p.num_tiles;
  const int nQ = p.k_iters / p.n_gs;  // filter taps
  const uint32_t a_total = p.a_bytes * (uint32_t)p.n_a;
  const int slots = p.acc_slots;
  const uint32_t slot_cols = (uint32_t)(p.levels * p.n_tile);

  // ---- tile scheduler ----
  // Cluster tile c covers the CTA tiles c*cs + rank (decode_tile). Static
  // order (p.tile_ctr null): c = cluster + it * clusters. Dynamic: the first
  // tile is the cluster's own, later ones come from an atomic counter that
  // the (leader's) producer bumps; it publishes each c through a kSchedR-deep
  // ring in shared memory (the peer's copy written over DSMEM), and every
  // consumer warp reads the same sequence. Keeps the CTAs' in-flight tiles a
  // compact window (halo neighbours meet in L2) and leaves no drift tail.
  const long long n_ct = num_tiles / cs, n_cl = (long long)gridDim.x / cs, c_first = (long long)blockIdx.x / cs;
  const bool dyn = p.tile_ctr != nullptr;
  auto sched_read = [&](int it, bool one_lane) -> long long {
    if (!dyn || it == 0) {  // the first tile is the cluster's own in both orders
      const long long c = c_first + (long long)it * n_cl;
      return c < n_ct ? c : -1;
    }
    const int slot = (it - 1) & (kSchedR - 1);  // ring entry j = it - 1 holds tile it
    const uint32_t ph = (uint32_t)((it - 1) / kSchedR) & 1u;
    if (PAIR && crank != 0) mbar_wait_cluster(&sfull[slot], ph);
    else mbar_wait(&sfull[slot], ph);
    const long long c = *reinterpret_cast<volatile long long*>(&sids[slot]);
    if (!one_lane) __syncwarp();
    if (one_lane || lane == 0) {  // CTA-scope arrive on the leader (a cluster release would
      if (PAIR && crank != 0) mbar_arrive_leader(&sempty[slot]);  // stall the MMA warp)
      else mbar_arrive(&sempty[slot]);
    }
    return c;
  };
  // The leader's producer publishes tile it+1 early in tile it (after the
  // tile's first A load, so the release / DSMEM store never delays it; the
  // peer's producer finds the id ready), and bumps the counter one tile
  // earlier still (the atomic's round trip overlaps a tile).
  unsigned long long ahead = 0;  // counter value requested during the previous tile
  long long c_next = -1;         // published id of the next tile
  auto sched_cur = [&](int it) -> long long {  // the (leader's) producer
    if (!dyn || it == 0) {
      const long long c = c_first + (long long)it * n_cl;
      return c < n_ct ? c : -1;
    }
    return c_next;
  };
  auto sched_pub = [&](int it) {  // once per tile it >= 0 of the leader's producer
    if (!dyn) return;
    if (it == 0) ahead = atomicAdd(p.tile_ctr, 1ull);
    long long n = n_cl + (long long)ahead;
    if (n >= n_ct) n = -1;
    else ahead = atomicAdd(p.tile_ctr, 1ull);
    const int slot = it & (kSchedR - 1);  // ring entry j = it holds tile it + 1
    const uint32_t ph = (uint32_t)(it / kSchedR) & 1u;
    mbar_wait(&sempty[slot], ph ^ 1u);
    sids[slot] = n;
    if constexpr (PAIR) st_remote_arrive(&sids[slot], n, &sfull[slot], 1);
    mbar_arrive(&sfull[slot]);
    c_next = n;
  };

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int hsl = 0;
      uint32_t hphase = 0;
      const int df = p.d_filter;
      // pair: each CTA loads its own A rows and its half of the B columns; the
      // leader alone arms its barriers for the bytes of both CTAs
      const bool arm = !PAIR || crank == 0;
      const uint32_t b_cta = PAIR ? p.b_bytes / 2 : p.b_bytes;
      const uint32_t tx_bytes = (PAIR ? 2u : 1u) * (p.halo ? b_cta : p.a_bytes * (uint32_t)p.n_tma_a + b_cta);
      auto load_b = [&](int nt, int kit, uint32_t sub = 0) {
        uint8_t* sB = ring + (size_t)stage * p.stage_bytes + (p.halo ? 0u : a_total) + sub;
        const size_t off = ((size_t)nt * p.k_iters + kit) * p.b_bytes;
        if constexpr (PAIR) tma_load_2d_cg2(sB, &bmap, &full[stage], 0, (int)((off + (size_t)crank * b_cta) >> 9));
        else bulk_load(sB, p.b_img + off, p.b_bytes, &full[stage]);
      };
      for (int it = 0;; ++it) {
        const bool leader = !PAIR || crank == 0;
        const long long c = leader ? sched_cur(it) : sched_read(it, true);
        if (c < 0) break;
        bool published = !leader;  // the leader publishes the next tile once per tile
        const long long t = c * cs;
        int nt, tx, ty, tz, b;
        decode_tile(p, t, crank, nt, tx, ty, tz, b);
        const int x0 = tx * p.tx - p.pad, y0 = ty * p.ty - p.pad, z0 = tz * p.tz - p.pad;
        if (p.halo) {
          // one halo box per channel group, then the B stage of every tap
          for (int gsi = 0; gsi < p.n_gs; ++gsi) {
            const int g0 = gsi * p.gs;
            const long long dbg_e0 = (kDbg && p.dbg_acc) ? clock64() : 0;
            mbar_wait(&hempty[hsl], hphase ^ 1);
            if (kDbg && p.dbg_acc) atomicAdd(p.dbg_acc + 10, (unsigned long long)(clock64() - dbg_e0));
            uint8_t* hA = smem + (size_t)hsl * p.halo_slot;
            if (kAOwn) mbar_arrive_expect_tx(&hfull[hsl], p.halo_bytes * (uint32_t)p.n_tma_a);
            else if (arm) mbar_arrive_expect_tx(&hfull[hsl], (PAIR ? 2u : 1u) * p.halo_bytes * (uint32_t)p.n_tma_a);
            for (int d = 0; d < p.n_tma_a; ++d) {  // int8: one halo per digit plane (planes stacked over the batch)
              const int bb = d * p.B + b;
              if (p.merged_bc)
                load_a_box<PAIR && !kAOwn>(p, hA + (size_t)d * p.a_bytes, &tmap, &hfull[hsl], x0, y0, z0, bb * p.G + g0);
              else
                load_a_box<PAIR && !kAOwn>(p, hA + (size_t)d * p.a_bytes, &tmap, &hfull[hsl], x0, y0, g0, bb);
            }
            if (++hsl == HS) { hsl = 0; hphase ^= 1; }
            if (!published) { sched_pub(it); published = true; }
            for (int q0 = 0; q0 < nQ; q0 += p.tps) {  // tps filter taps per B stage
              const int nq = min(p.tps, nQ - q0);
              const long long dbg_e1 = (kDbg && p.dbg_acc) ? clock64() : 0;
              mbar_wait(&empty[stage], phase ^ 1);
              if (kDbg && p.dbg_acc) atomicAdd(p.dbg_acc + 9, (unsigned long long)(clock64() - dbg_e1));
              if (dbg_skip(p) & 1) {  // timing experiment: no B loads (results garbage)
                if (arm) mbar_arrive(&full[stage]);
              } else {
                // halo plans store each (N tile, channel group, CTA half)'s taps
                // contiguously (expand.cu): the stage's taps arrive in ONE request
                // (each TMA request costs its issuing thread ~290 cycles,
                // tools/probe/tma_rate.cu). Pairs load a fixed box of tps taps
                // (a short last stage over-reads into the next block; unused).
                uint8_t* sB = ring + (size_t)stage * p.stage_bytes;
                const size_t blk = ((size_t)nt * p.n_gs + gsi) * (PAIR ? 2u : 1u) + (PAIR ? (size_t)crank : 0u);
                const size_t off = (blk * (size_t)nQ + (size_t)q0) * b_cta;
                if constexpr (PAIR) {
                  if (arm) mbar_arrive_expect_tx(&full[stage], tx_bytes * (uint32_t)p.tps);
                  tma_load_2d_cg2(sB, &bmap, &full[stage], 0, (int)(off >> 9));
                } else {
                  mbar_arrive_expect_tx(&full[stage], tx_bytes * (uint32_t)nq);
                  bulk_load(sB, p.b_img + off, b_cta * (uint32_t)nq, &full[stage]);
                }
              }
              if (++stage == S) { stage = 0; phase ^= 1; }
            }
          }
          if (!published) sched_pub(it);
          continue;
        }
        for (int kit = 0; kit < p.k_iters; ++kit) {
          const int q = kit / p.n_gs, g0 = (kit - q * p.n_gs) * p.gs;
          int qx, qy, qz;
          if (p.k == 3) { qz = q / (df * df); qy = (q / df) % df; qx = q % df; }
          else { qz = 0; qy = q / df; qx = q % df; }
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = ring + (size_t)stage * p.stage_bytes;
          if (arm) mbar_arrive_expect_tx(&full[stage], tx_bytes);
          for (int d = 0; d < p.n_tma_a; ++d) {
            const int bb = d * p.B + b;  // digit planes are stacked over the batch
            if (p.merged_bc)
              load_a_box<PAIR>(p, sA + d * p.a_bytes, &tmap, &full[stage], x0 + qx, y0 + qy, z0 + qz, bb * p.G + g0);
            else if (p.k == 1)  // dims (e, x, sample, group, plane)
              load_a_box<PAIR>(p, sA + d * p.a_bytes, &tmap, &full[stage], x0 + qx, b, g0, d);
            else
              load_a_box<PAIR>(p, sA + d * p.a_bytes, &tmap, &full[stage], x0 + qx, y0 + qy, g0, bb);
          }
          load_b(nt, kit);
          if (++stage == S) { stage = 0; phase ^= 1; }
          if (!published) { sched_pub(it); published = true; }
        }
        if (!published) sched_pub(it);
      }
    }
  } else if (warp == 1 && (!PAIR || crank == 0)) {
    // ===================== MMA issuer (the pair leader's in 2-SM mode) =====================
    // The warp runs the loop converged (all lanes wait on the barriers, all
    // values warp-uniform); one elected lane issues tcgen05.mma + commit.
    // Descriptors are template + (address >> 4): start address is the low
    // 14-bit field, and CTA-local shared addresses < 2^18 never carry out of it.
    const uint32_t issuer = elect_one();  // the lane whose guarded tcgen05 instructions issue
    constexpr uint32_t kM = PAIR ? 256u : 128u;
    const uint32_t idesc = kInt8 ? instr_desc_i8(kM, (uint32_t)p.n_tile)
                                 : instr_desc(PREC == kPrecBf16 ? 1u : 2u, kM, (uint32_t)p.n_tile);
    const uint32_t n_cta = PAIR ? (uint32_t)p.n_tile / 2u : (uint32_t)p.n_tile;  // B rows in this CTA
    // 32-byte swizzled protocol rows (3-D tf32 modes) unless a changed basis packs 16-byte rows
    const bool rb32 = (RB == 32) && !p.bs.on;
    const uint64_t a_tmpl = rb32 ? smem_desc(0, 16, 256, kSwizzle32B) : smem_desc(0, 2048, 128, kSwizzleNone);
    const uint64_t b_tmpl = smem_desc(0, n_cta * 16u, 128, kSwizzleNone);
    const uint32_t a_img4 = p.a_bytes >> 4, b_img4 = (PAIR ? p.b_img_bytes / 2 : p.b_img_bytes) >> 4;
    const uint32_t b_ks4 = (n_cta * 32u) >> 4;
    const uint32_t b_cta4 = (PAIR ? p.b_bytes / 2 : p.b_bytes) >> 4;  // one tap's B image in a multi-tap stage
    const uint32_t a_tot4 = a_total >> 4;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int hsl = 0;
    uint32_t hphase = 0;
    const int df = p.d_filter;
    const int ncol = p.bs.on ? p.bs.ncol : 1;
    // halo mode: K-major SWIZZLE_NONE, SBO = halo row pitch (the tile is one
    // 8-row core-matrix group wide), LBO = one channel-group plane of the halo
    const uint32_t h_plane = (uint32_t)(p.hx * p.hy * p.hz * ncol * 16);
    const uint64_t h_tmpl = smem_desc(0, h_plane, (uint32_t)(p.hx * ncol * 16), kSwizzleNone);
    const uint32_t h_img4 = p.a_bytes >> 4, h_plane4 = h_plane >> 4;  // digit / lo plane stride
    const uint64_t a_kstep = 2u * h_plane4;                                // next K step: 2 groups
    const uint32_t h_dx = (uint32_t)ncol;                                  // next tap along x
    const uint32_t h_wrap_x = (uint32_t)((p.hx - df) * ncol);              // x wrapped: next halo row
    const uint32_t h_wrap_y = (uint32_t)((p.hy - df) * p.hx * ncol);       // y wrapped: next halo plane
    // Accumulation groups: `p.drain` consecutive pipeline stages accumulate
    // into one TMEM slot (the first MMA of a group overwrites it); the last
    // stage of a group commits it to the epilogue, the next group waits for a
    // free slot. One group per tile except in the exact mode's long
    // reductions (ConvPlan::drain).
    uint32_t d_tmem = 0;
    int sg = 0;  // stage index inside the current group
    // 3xTF32: the tile-long accumulator of the cross terms (behind the hi slots)
    const uint32_t d_lo = tmem_base + (uint32_t)kX3HiSlots * slot_cols;
    uint32_t lo_phase = 0;
    auto group_begin = [&]() {
      const long long dbg_w0 = (kDbg && p.dbg_acc) ? clock64() : 0;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      if (kDbg && p.dbg_acc && lane == 0) {  // timing instrumentation: MMA warp's wait for the accumulator
        atomicAdd(p.dbg_acc + 2, (unsigned long long)(clock64() - dbg_w0));
        atomicAdd(p.dbg_acc + 3, 1ull);
      }
      d_tmem = tmem_base + (uint32_t)acc * slot_cols;
    };
    // after a stage (warp-uniform): close the group when it ended, open the next one
    auto stage_done = [&](bool gend, bool tile_last) {
      if (gend) {
        if (++acc == slots) { acc = 0; acc_phase ^= 1; }
        sg = 0;
        if (!tile_last) group_begin();
      } else {
        ++sg;
      }
    };
    for (int it = 0;; ++it) {
      // the exit test on a warp-uniform copy of the tile id (REDUX writes a
      // uniform register): a branch on the raw shared-memory load made ptxas
      // treat the whole issue loop as divergent, moving every descriptor,
      // stage and phase value to vector registers (R2UR before each MMA)
      if (__reduce_min_sync(0xffffffffu, sched_read(it, false) < 0 ? -1 : 0) < 0) break;
      group_begin();
      if constexpr (kSplit) {  // the previous tile's lo accumulator has been read by every epilogue warp
        mbar_wait(&tempty[kX3HiSlots], lo_phase ^ 1);
        tc_fence_after();
        lo_phase ^= 1;
      }
      if constexpr (!kInt8) {
        if (p.halo) {
          // bf16 / tf32 / 3xTF32 halo mode: lean warp-converged issue. All
          // lanes run the loop on warp-uniform values; elect.sync inside the
          // MMA / commit asm issues (bare UTC*MMA on uniform registers). The
          // per-stage MMA-warp cost had bounded the N = 128 stages of these
          // modes (cfg4 bf16: ~110 SASS instructions, ~650 cycles per 4-MMA
          // stage of 256 tensor cycles). Accumulation groups of p.drain
          // stages (3xTF32's periodic drains) rotate the TMEM slots.
          constexpr int CG = PAIR ? 2 : 1;
          const uint32_t a_hi = (uint32_t)(h_tmpl >> 32), b_hi = (uint32_t)(b_tmpl >> 32);
          const uint32_t stg4 = p.stage_bytes >> 4, hslot4 = p.halo_slot >> 4;
          const uint32_t h_base = (uint32_t)h_tmpl + ((smem_u32(smem) & 0x3FFFFu) >> 4);
          const uint32_t b_base = (uint32_t)b_tmpl + ((smem_u32(ring) & 0x3FFFFu) >> 4);
          const uint32_t a_ks = (uint32_t)a_kstep;
          const long long dbg_t0 = (kDbg && p.dbg_acc) ? clock64() : 0;
          // one filter tap's KS K steps at (a, b)
          auto tap_mmas = [&](auto ks_c, uint32_t a, uint32_t b, uint32_t accf, uint32_t accl) {
            constexpr int KS = decltype(ks_c)::value;
            if constexpr (kSplit)
              mma_stage_x3_e<CG, KS>(d_tmem, d_lo, a, a_hi, b, b_hi, idesc, accf, accl, a_ks, b_ks4, h_img4, b_img4);
            else
              mma_stage_e<PREC == kPrecBf16 ? 1 : 2, CG, KS>(d_tmem, a, a_hi, b, b_hi, idesc, accf, a_ks, b_ks4);
          };
          auto run = [&](auto ks_c, auto tps_c) {
            constexpr int TPS = decltype(tps_c)::value;  // 0: runtime p.tps
            const int tps = TPS ? TPS : p.tps;
            uint32_t accf = 0, accl = 0;  // accumulate flags: hi slot (per group), lo accumulator (per tile)
            uint32_t b_cur = b_base + (uint32_t)stage * stg4;
            for (int gsi = 0; gsi < p.n_gs; ++gsi) {
              const long long dbg_h0 = (kDbg && p.dbg_acc) ? clock64() : 0;
              mbar_wait(kSplit ? &hlo[hsl] : &hfull[hsl], hphase);  // 3xTF32: A_lo written
              if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 4, (unsigned long long)(clock64() - dbg_h0));
              tc_fence_after();
              uint32_t a_cur = h_base + (uint32_t)hsl * hslot4;
              int qx = 0, qy = 0;
              for (int q0 = 0; q0 < nQ; q0 += tps) {
                const int nq = TPS == 1 ? 1 : min(tps, nQ - q0);
                const long long dbg_s0 = (kDbg && p.dbg_acc) ? clock64() : 0;
                mbar_wait(&full[stage], phase);
                if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 5, (unsigned long long)(clock64() - dbg_s0));
                tc_fence_after();
                uint32_t b0 = b_cur;
                for (int i = 0; i < nq; ++i) {
                  tap_mmas(ks_c, a_cur, b0, accf, accl);
                  accf = 1u;
                  accl = 1u;
                  b0 += b_cta4;
                  a_cur += h_dx;
                  if (++qx == df) {
                    qx = 0;
                    a_cur += h_wrap_x;
                    if (++qy == df) { qy = 0; a_cur += h_wrap_y; }
                  }
                }
                commit_e<CG>(&empty[stage]);
                b_cur += stg4;
                if (++stage == S) { stage = 0; phase ^= 1; b_cur = b_base; }
                // accumulation group ended (not the tile's last stage): hand the
                // slot to the epilogues, open the next one
                if (++sg == p.drain && !(gsi == p.n_gs - 1 && q0 + nq >= nQ)) {
                  commit_e<CG>(&tfull[acc]);
                  if (++acc == slots) { acc = 0; acc_phase ^= 1; }
                  group_begin();
                  sg = 0;
                  accf = 0;
                }
              }
              commit_e<CG>(&hempty[hsl]);  // halo reusable once its last tap retires
              if (++hsl == HS) { hsl = 0; hphase ^= 1; }
            }
            commit_e<CG>(&tfull[acc]);
          };
          using I1 = std::integral_constant<int, 1>;
          using I0 = std::integral_constant<int, 0>;
          const bool t1 = p.tps == 1;
          switch (p.ks) {
            case 1: if (t1) run(I1{}, I1{}); else run(I1{}, I0{}); break;
            case 2: if (t1) run(std::integral_constant<int, 2>{}, I1{}); else run(std::integral_constant<int, 2>{}, I0{}); break;
            case 4: if (t1) run(std::integral_constant<int, 4>{}, I1{}); else run(std::integral_constant<int, 4>{}, I0{}); break;
            default: if (t1) run(std::integral_constant<int, 8>{}, I1{}); else run(std::integral_constant<int, 8>{}, I0{}); break;
          }
          if (++acc == slots) { acc = 0; acc_phase ^= 1; }
          sg = 0;
          if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 8, (unsigned long long)(clock64() - dbg_t0));
          continue;
        }
      }
      if (kInt8 && p.halo) {  // (the other modes took the lean path above)
        for (int gsi = 0; gsi < p.n_gs; ++gsi) {
          const long long dbg_h0 = (kDbg && p.dbg_acc) ? clock64() : 0;
          mbar_wait(&hfull[hsl], hphase);
          if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 4, (unsigned long long)(clock64() - dbg_h0));
          tc_fence_after();
          const uint32_t hA4 = (smem_u32(smem + (size_t)hsl * p.halo_slot) & 0x3FFFFu) >> 4;
          // tap (qx, qy, qz) -> halo offset in 16-byte rows, stepped without divisions
          uint32_t tap4 = 0;
          int qx = 0, qy = 0;
          if (p.tps == 1) {  // one tap per stage (kept separate: the multi-tap loop's codegen costs 20% here)
            for (int q = 0; q < nQ; ++q) {
              const long long dbg_s0 = (kDbg && p.dbg_acc) ? clock64() : 0;
              mbar_wait(&full[stage], phase);
              if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 5, (unsigned long long)(clock64() - dbg_s0));
              tc_fence_after();
              const uint32_t sB4 = (smem_u32(ring + (size_t)stage * p.stage_bytes) & 0x3FFFFu) >> 4;
              if (elect_one()) {
                const uint32_t a_hi = (uint32_t)(h_tmpl >> 32), b_hi = (uint32_t)(b_tmpl >> 32);
                uint32_t a0 = (uint32_t)h_tmpl + hA4 + tap4, b0 = (uint32_t)b_tmpl + sB4;
                #pragma unroll
                for (int s = 0; s < 8; ++s) {  // ks <= 8, unrolled: constant per-step offsets
                  if (s >= p.ks) break;
                  const uint32_t first = (sg == 0 && s == 0) ? 1u : 0u;
                  if constexpr (kInt8) {  // the K step's 10 digit-pair MMAs in one asm block
                    if constexpr (PAIR)
                      mma_i8_cg2_kstep(1u, d_tmem, a0, a_hi, b0, b_hi, idesc, first ? 0u : 1u, h_img4, b_img4,
                                       (uint32_t)p.n_tile);
                    else
                      mma_i8_kstep(1u, d_tmem, a0, a_hi, b0, b_hi, idesc, first ? 0u : 1u, h_img4, b_img4,
                                   (uint32_t)p.n_tile);
                  }
                  a0 += (uint32_t)a_kstep;
                  b0 += b_ks4;
                }
                const bool tile_last = q == nQ - 1 && gsi == p.n_gs - 1;
                if constexpr (PAIR) {
                  mma_commit_cg2(&empty[stage]);
                  if (q == nQ - 1) mma_commit_cg2(&hempty[hsl]);  // halo reusable once the last tap retires
                  if (sg == p.drain - 1 || tile_last) mma_commit_cg2(&tfull[acc]);
                } else {
                  mma_commit(&empty[stage]);
                  if (q == nQ - 1) mma_commit(&hempty[hsl]);
                  if (sg == p.drain - 1 || tile_last) mma_commit(&tfull[acc]);
                }
              }
              __syncwarp();
              if (++stage == S) { stage = 0; phase ^= 1; }
              {
                const bool tile_last = q == nQ - 1 && gsi == p.n_gs - 1;
                stage_done(sg == p.drain - 1 || tile_last, tile_last);
              }
              tap4 += h_dx;
              if (++qx == df) {
                qx = 0;
                tap4 += h_wrap_x;
                if (++qy == df) { qy = 0; tap4 += h_wrap_y; }
              }
            }
          } else {
            // several taps per stage (small int8 layers, e.g. cfg1): converged per-MMA issue
            for (int q0 = 0; q0 < nQ; q0 += p.tps) {  // tps filter taps per B stage
              const int nq = min(p.tps, nQ - q0);
              const long long dbg_s0 = (kDbg && p.dbg_acc) ? clock64() : 0;
              mbar_wait(&full[stage], phase);
              if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 5, (unsigned long long)(clock64() - dbg_s0));
              tc_fence_after();
              const uint32_t sB4 = (smem_u32(ring + (size_t)stage * p.stage_bytes) & 0x3FFFFu) >> 4;
              {
                // converged issue (every lane computes the warp-uniform descriptors,
                // one lane's guard is set); descriptors as 32-bit low halves + constant
                // high halves, so the per-MMA arithmetic is 32-bit uniform adds
                const uint32_t a_hi = (uint32_t)(h_tmpl >> 32), b_hi = (uint32_t)(b_tmpl >> 32);
                uint32_t a_tap = (uint32_t)h_tmpl + hA4 + tap4;
                uint32_t b_cur = (uint32_t)b_tmpl + sB4;
                const uint32_t a_ks = (uint32_t)a_kstep, b_ks = b_ks4, a_img = h_img4, b_img = b_img4;
                uint32_t accf = (sg == 0) ? 0u : 1u;
                int x = qx, y = qy;
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // taps of this stage (tps <= 4)
                  if (i >= nq) break;
                  uint32_t a0 = a_tap, b0 = b_cur;
                  #pragma unroll
                  for (int s = 0; s < 8; ++s) {  // ks <= 8, unrolled: constant per-step offsets
                    if (s >= p.ks) break;
                    if constexpr (kInt8) {
#pragma unroll
                      for (int L = 0; L < kLevels; ++L) {
                        const int i0 = L > kDigitsW - 1 ? L - (kDigitsW - 1) : 0;
#pragma unroll
                        for (int ii = i0; ii <= L && ii < kDigitsA; ++ii) {
                          const int j = L - ii;
                          mma_mode_s<PREC, PAIR>(issuer, d_tmem + (uint32_t)(L * p.n_tile), a0 + (uint32_t)ii * a_img,
                                                 a_hi, b0 + (uint32_t)j * b_img, b_hi, idesc, ii == i0 ? accf : 1u);
                        }
                      }
                    }
                    accf = 1u;
                    a0 += a_ks;
                    b0 += b_ks;
                  }
                  b_cur += b_cta4;
                  a_tap += h_dx;
                  if (++x == df) {
                    x = 0;
                    a_tap += h_wrap_x;
                    if (++y == df) { y = 0; a_tap += h_wrap_y; }
                  }
                }
                const bool last = q0 + nq == nQ;
                commit_g<PAIR>(issuer, &empty[stage]);
                if (last) commit_g<PAIR>(issuer, &hempty[hsl]);  // halo reusable once the last tap retires
                if (sg == p.drain - 1 || (last && gsi == p.n_gs - 1)) commit_g<PAIR>(issuer, &tfull[acc]);
              }
              __syncwarp();
              if (++stage == S) { stage = 0; phase ^= 1; }
              {
                const bool tile_last = q0 + nq == nQ && gsi == p.n_gs - 1;
                stage_done(sg == p.drain - 1 || tile_last, tile_last);
              }
              for (int i = 0; i < nq; ++i) {  // advance the warp-uniform tap state
                tap4 += h_dx;
                if (++qx == df) {
                  qx = 0;
                  tap4 += h_wrap_x;
                  if (++qy == df) { qy = 0; tap4 += h_wrap_y; }
                }
              }
            }
          }
          if (++hsl == HS) { hsl = 0; hphase ^= 1; }
        }
        continue;
      }
      for (int kit = 0; kit < p.k_iters; ++kit) {
        const long long dbg_s0 = (kDbg && p.dbg_acc) ? clock64() : 0;
        if (kSplit) mbar_wait(&lo_ready[stage], phase);
        else mbar_wait(&full[stage], phase);
        if (kDbg && p.dbg_acc && lane == 0) atomicAdd(p.dbg_acc + 5, (unsigned long long)(clock64() - dbg_s0));
        tc_fence_after();
        // (cluster launches return cluster-window shared addresses: keep the
        // CTA-local 18 bits so nothing carries past the 14-bit start field)
        const uint32_t sA4 = (smem_u32(ring + (size_t)stage * p.stage_bytes) & 0x3FFFFu) >> 4;
        const uint32_t sB4 = sA4 + a_tot4;
        if (elect_one()) {
          // descriptors as 32-bit low halves + constant high halves (the
          // per-MMA arithmetic is a 32-bit add on the uniform datapath), the
          // K steps unrolled with a uniform early exit
          const uint32_t a_hi = (uint32_t)(a_tmpl >> 32), b_hi = (uint32_t)(b_tmpl >> 32);
          uint32_t a0 = (uint32_t)a_tmpl + sA4, b0 = (uint32_t)b_tmpl + sB4;
          if constexpr (!kInt8 && !kSplit)
            mma_stage<PREC, PAIR>(p.ks, 1u, d_tmem, a0, a_hi, b0, b_hi, idesc, sg == 0 ? 0u : 1u, 256u, b_ks4);
#pragma unroll
          for (int s = 0; s < 8; ++s) {  // ks <= 8
            if (kInt8 || kSplit ? s >= p.ks : true) break;
            const uint32_t first = (sg == 0 && s == 0) ? 1u : 0u;
            if constexpr (kInt8) {
              // D_L += A_i * B_j over digit pairs with i + j = L <= 3 (Ozaki levels,
              // 4 digits each): 10 MMAs per K step, one asm block
              if constexpr (PAIR)
                mma_i8_cg2_kstep(1u, d_tmem, a0, a_hi, b0, b_hi, idesc, first ? 0u : 1u, a_img4, b_img4,
                                 (uint32_t)p.n_tile);
              else
                mma_i8_kstep(1u, d_tmem, a0, a_hi, b0, b_hi, idesc, first ? 0u : 1u, a_img4, b_img4,
                             (uint32_t)p.n_tile);
            } else if constexpr (kSplit) {
              const uint32_t lo_first = (kit == 0 && s == 0) ? 0u : 1u;  // the tile's first cross-term MMA overwrites
              mma_mode_s<kPrecTf32, PAIR>(1u, d_lo, a0 + a_img4, a_hi, b0, b_hi, idesc, lo_first);         // A_lo * B_hi
              mma_mode_s<kPrecTf32, PAIR>(1u, d_lo, a0, a_hi, b0 + b_img4, b_hi, idesc, 1u);               // A_hi * B_lo
              mma_mode_s<kPrecTf32, PAIR>(1u, d_tmem, a0, a_hi, b0, b_hi, idesc, first ? 0u : 1u);         // A_hi * B_hi
            } else {
              mma_mode_s<PREC, PAIR>(1u, d_tmem, a0, a_hi, b0, b_hi, idesc, first ? 0u : 1u);
            }
            a0 += 256u;
            b0 += b_ks4;
          }
          // smem slot free (in both CTAs of a pair) once these MMAs retire
          const bool gend = sg == p.drain - 1 || kit == p.k_iters - 1;
          if constexpr (PAIR) {
            mma_commit_cg2(&empty[stage]);
            if (gend) mma_commit_cg2(&tfull[acc]);  // accumulator (group) ready for the epilogues
          } else {
            mma_commit(&empty[stage]);
            if (gend) mma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
        stage_done(sg == p.drain - 1 || kit == p.k_iters - 1, kit == p.k_iters - 1);
      }
    }
  } else if (warp >= 4 && warp < 4 + 4 * kEpiGroups) {
    // ===================== epilogue =====================
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    const int eg = (warp - 4) >> 2;
    const int c_half = ((p.n_tile / kEpiGroups + 15) / 16) * 16;
    const int c_beg = eg * c_half, c_end = min(p.n_tile, c_beg + c_half);
    const int row = ew * 32 + lane;
    // with a change of basis a pixel owns ncol = 2 adjacent rows (lanes), one per matrix column
    // (2-D bf16 / tf32 kernels: compile-time false, see kBasisEpi)
    const bool bs_on = kBasisEpi && p.bs.on;
    const int bcol = bs_on ? (row & 1) : 0;
    const int prow = bs_on ? (row >> 1) : row;
    int inv_i0[NB], inv_i1[NB], inv_s0[NB], inv_s1[NB];  // two-term inverse transform (registers)
#pragma unroll
    for (int t2 = 0; t2 < NB; ++t2) {
      inv_i0[t2] = p.bs.inv[t2 % 8][0];
      inv_i1[t2] = p.bs.inv[t2 % 8][1];
      inv_s0[t2] = p.bs.inv_sgn[t2 % 8][0];
      inv_s1[t2] = p.bs.inv_sgn[t2 % 8][1];
    }
    // int8 epilogue: the two terms of each of this lane's blades, own column / partner column
    constexpr int WL = (NB >= 4) ? NB / 2 : 1;
    int inv_o[WL], inv_p[WL], inv_os[WL], inv_ps[WL];
#pragma unroll
    for (int j = 0; j < WL; ++j) {
      const int t = bcol * WL + j;
      const int a0 = p.bs.inv[t % 8][0], a1 = p.bs.inv[t % 8][1];
      const bool first_own = (a0 / WL) == bcol;
      inv_o[j] = (first_own ? a0 : a1) % WL;
      inv_p[j] = (first_own ? a1 : a0) % WL;
      inv_os[j] = first_own ? p.bs.inv_sgn[t % 8][0] : p.bs.inv_sgn[t % 8][1];
      inv_ps[j] = first_own ? p.bs.inv_sgn[t % 8][1] : p.bs.inv_sgn[t % 8][0];
    }
    // the same signs as +-1 multipliers (fp32-accumulator epilogue: one FMUL / FFMA per term)
    float sgn_o[WL], sgn_p[WL];
    const unsigned act_kml = (p.act_kmask >> (bcol * WL)) & ((1u << WL) - 1u);  // this lane's kernel blades
#pragma unroll
    for (int j = 0; j < WL; ++j) {
      sgn_o[j] = inv_os[j] > 0 ? 1.f : -1.f;
      sgn_p[j] = inv_ps[j] > 0 ? 1.f : -1.f;
    }
    const int lx = prow % p.tx, ly = (prow / p.tx) % p.ty, lz = prow / (p.tx * p.ty);
    const int d_out = p.d_out;
    const long long P_out = (p.k == 3) ? (long long)d_out * d_out * d_out
                                       : (p.k == 2 ? (long long)d_out * d_out : (long long)d_out);
    const long long P_res = (p.k == 3) ? (long long)p.res_side * p.res_side * p.res_side
                                       : (p.k == 2 ? (long long)p.res_side * p.res_side : (long long)p.res_side);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int it = 0;; ++it) {
      const long long c = sched_read(it, false);
      if (c < 0) break;
      const long long t = c * cs;
      int nt, tx, ty, tz, b;
      const bool real = decode_tile(p, t, crank, nt, tx, ty, tz, b);
      const int ox = tx * p.tx + lx, oy = ty * p.ty + ly, oz = tz * p.tz + lz;
      bool valid;
      long long pix, pres = 0;
      const int rs = p.res_side, cr = p.res_crop;
      if (p.k == 1) {  // row = (sample b + ly, position ox)
        b += ly;
        valid = real && ox < d_out && b < p.B;
        pix = ox;
        pres = ox + cr;
      } else {
        valid = real && ox < d_out && oy < d_out && oz < ((p.k == 3) ? d_out : 1);
        pix = (p.k == 3) ? ((long long)oz * d_out + oy) * d_out + ox : (long long)oy * d_out + ox;
        pres = (p.k == 3) ? ((long long)(oz + cr) * rs + (oy + cr)) * rs + (ox + cr)
                          : (long long)(oy + cr) * rs + (ox + cr);
      }
      double a_sc = 0.0;
      if constexpr (kInt8) if (valid) a_sc = (double)__ldg(p.a_scale + b) * (1.0 / 16384.0);  // 2^-14: two leading digits
      if constexpr (!kInt8) {
        // fused residual (block conv2): start this thread's residual lines towards
        // L2 now, while the tile's MMAs still run. The epilogue loads them chunk
        // by chunk right before use and had waited a DRAM round trip per chunk
        // (CL_DBG_CLK, cfg3 bf16 conv2: 28.5 K cycles per tile against 16.9 K for
        // conv1, and the MMA warp waited 12.4 K of its 18 K cycles per tile for a
        // free accumulator). The int8 mode adds the residual in its phase 2, off
        // the critical path.
        if (p.resid != nullptr && valid) {
          const int wv = bs_on ? NB / 2 : NB;  // floats of one channel in this lane
          const float* rbase = p.resid + ((long long)b * p.C_out * P_res + pres) * NB + (bs_on ? bcol * wv : 0);
          for (int c = c_beg; c < c_end; c += wv) {
            const int co = (nt * p.n_tile + c) / wv;
            if (co < p.C_out) prefetch_l2(rbase + (long long)co * P_res * NB);
          }
        }
      }
      if constexpr (kInt8 && GROUPS)  // exact mode, several accumulation groups per tile
        drain_groups<PAIR>(p, tfull, tempty, tmem_base, ew, row, c_beg, c_end, slot_cols, slots, acc, acc_phase);
      if constexpr (kSplit)  // returns with the last group's slot full and complete (lo accumulator added)
        x3_drain_groups<PAIR>(p, tfull, tempty, tmem_base, ew, c_beg, c_end, slot_cols, slots, acc, acc_phase);
      else
        mbar_wait_sleep(&tfull[acc], acc_phase, 64);  // off the critical path: poll gently
      tc_fence_after();
      const long long dbg_t0 = (kDbg && p.dbg_acc) ? clock64() : 0;
      const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)acc * slot_cols;
      if constexpr (kInt8) {
        // Two-phase epilogue: this mode has ONE accumulator slot (4 exact
        // levels x N_TILE fill TMEM), so the next tile's MMAs wait for it.
        // Phase 1 drains TMEM into registers (level combine, change-of-basis
        // inverse, bias, activation gate) and releases the slot; phase 2 adds
        // the residual and stores while the next tile's MMAs run.
        constexpr int kHold = 32;           // columns per thread: N_TILE <= 128 over 4 warp groups
        constexpr int CH = (NB == 8 && BCLS == 0) ? 8 : 4;  // columns per chunk: whole channels (BCLS > 0 implies the basis: 4)
        float hv[kHold];
#pragma unroll
        for (int ci = 0; ci < kHold / CH; ++ci) {
          const int c0 = c_beg + ci * CH;
          const int n0 = nt * p.n_tile + c0;
          if (c0 < c_end && n0 < p.N && !(dbg_skip(p) & 4)) {
            long long sv[CH];  // exact: S = L0 2^24 + L1 2^16 + L2 2^8 + L3 (|S| < 2^53 for K <= 32000)
            {
              uint32_t l0[CH], l1[CH], l2[CH], l3[CH];
              tmem_ldn<CH>(taddr + (uint32_t)c0, l0);
              tmem_ldn<CH>(taddr + (uint32_t)(p.n_tile + c0), l1);
              tmem_ldn<CH>(taddr + (uint32_t)(2 * p.n_tile + c0), l2);
              tmem_ldn<CH>(taddr + (uint32_t)(3 * p.n_tile + c0), l3);
              tmem_ld_wait();
#pragma unroll
              for (int c = 0; c < CH; ++c)
                sv[c] = ((long long)(int)l0[c] << 24) + ((long long)(int)l1[c] << 16) +
                        ((long long)(int)l2[c] << 8) + (long long)(int)l3[c];
              if constexpr (GROUPS) {  // the earlier accumulation groups of this tile (exact int64 sum)
                const long long* scr = p.grp_scratch + ((long long)blockIdx.x * kTileM + row) * p.n_tile + c0;
#pragma unroll
                for (int c = 0; c < CH; ++c) sv[c] += scr[c];
              }
            }
            if (bs_on) {
              if constexpr (NB >= 4) {
                // lane (column bcol) produces blades bcol*W + j: x = (s_o own[o_j] + s_p partner[p_j]) / 2,
                // combined exactly in int64 (one weight scale per channel), rounded once
                constexpr int W = NB / 2;
#pragma unroll
                for (int cc = 0; cc < CH / W; ++cc) {
                  const int co = n0 / W + cc;
                  const int cq = min(co, p.C_out - 1);
                  long long own[W], oth[W];
                  long long recvA = 0, recvB = 0;
                  if constexpr (BCLS == 2 && W == 4) {
                    // degenerate (1,-1,0) family: lane 0 sends rows 2, 3, lane 1 rows 0, 1
#pragma unroll
                    for (int r = 0; r < W; ++r) { own[r] = sv[cc * W + r]; oth[r] = 0; }
                    const long long sA = bcol ? own[0] : own[2], sB = bcol ? own[1] : own[3];
                    recvA = ((long long)__shfl_xor_sync(0xffffffffu, (int)(sA >> 32), 1) << 32) |
                            (long long)(unsigned)__shfl_xor_sync(0xffffffffu, (int)(sA & 0xffffffffll), 1);
                    recvB = ((long long)__shfl_xor_sync(0xffffffffu, (int)(sB >> 32), 1) << 32) |
                            (long long)(unsigned)__shfl_xor_sync(0xffffffffu, (int)(sB & 0xffffffffll), 1);
                  }
#pragma unroll
                  for (int r = 0; r < W; ++r) {
                    if constexpr (BCLS == 2) break;
                    own[r] = sv[cc * W + r];
                    oth[r] = 0;
                    // BCLS 1: the partner only needs rows 1 and 2
                    if (BCLS == 0 || r == 1 || r == 2) {
                      const int lo = __shfl_xor_sync(0xffffffffu, (int)(own[r] & 0xffffffffll), 1);
                      const int hi = __shfl_xor_sync(0xffffffffu, (int)(own[r] >> 32), 1);
                      oth[r] = ((long long)hi << 32) | (long long)(unsigned)lo;
                    }
                  }
                  const double sc = a_sc * (0.5 / 16777216.0) * (double)__ldg(p.w_scale + nt * p.n_tile + cc * W + c0);
                  // this lane's W biases: one vector load
                  float bw[W];
                  if constexpr (W == 4) {
                    const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias_t + cq * NB + bcol * W));
                    bw[0] = b4.x; bw[1 % W] = b4.y; bw[2 % W] = b4.z; bw[3 % W] = b4.w;
                  } else {
                    const float2 b2 = __ldg(reinterpret_cast<const float2*>(p.bias_t + cq * NB + bcol * W));
                    bw[0] = b2.x; bw[1 % W] = b2.y;
                  }
                  float v[W];
#pragma unroll
                  for (int j = 0; j < W; ++j) {
                    long long a, bq;
                    if constexpr (BCLS == 1 && W == 4) {
                      a = own[(j >> 1) * 3];        // rows 0, 0, 3, 3
                      bq = oth[2 - (j >> 1)];       // rows 2, 2, 1, 1
                    } else if constexpr (BCLS == 2 && W == 4) {
                      constexpr int kQ[4] = {0, 1, 1, 0};
                      a = bcol ? own[3 - kQ[j]] : own[kQ[j]];                 // rows 0,1,1,0 / 3,2,2,3
                      bq = (((j == 0) || (j == 3)) != (bcol != 0)) ? recvB : recvA;
                    } else {
                      a = pick_w<W>(own, inv_o[j]);
                      bq = pick_w<W>(oth, inv_p[j]);
                    }
                    const long long xs = (inv_os[j] > 0 ? a : -a) + (inv_ps[j] > 0 ? bq : -bq);
                    v[j] = (float)fma((double)xs, sc, (double)bw[j]);
                  }
#pragma unroll
                  for (int j = 0; j < W; ++j) hv[ci * CH + cc * W + j] = v[j];
                }
              }
            } else {
#pragma unroll
              for (int cc = 0; cc < CH / NB; ++cc) {
                const int co = n0 / NB + cc;
                const int cq = min(co, p.C_out - 1);
                float v[NB];
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                  const double sc = a_sc * (1.0 / 16777216.0) * (double)__ldg(p.w_scale + min(n0 + cc * NB + j, p.N - 1));
                  v[j] = (float)fma((double)sv[cc * NB + j], sc, (double)__ldg(p.bias + j * p.C_out + cq));
                }
                if (p.act_mode >= 0 && co < p.C_out) {
                  const float gte = act_gate<NB>(v, p.act_mode, p.act_w + co * NB,
                                                 p.act_mode == 0 ? __ldg(p.act_b + co) : 0.f, p.act_K, p.act_kmask);
#pragma unroll
                  for (int j = 0; j < NB; ++j) v[j] *= gte;
                }
#pragma unroll
                for (int j = 0; j < NB; ++j) hv[ci * CH + cc * NB + j] = v[j];
              }
            }
          }
        }
        release_acc<PAIR>(&tempty[acc]);
        if (kDbg && p.dbg_acc && threadIdx.x == 128) {  // timing instrumentation: phase-1 cycles per tile
          atomicAdd(p.dbg_acc, (unsigned long long)(clock64() - dbg_t0));
          atomicAdd(p.dbg_acc + 1, 1ull);
        }
        if (++acc == slots) { acc = 0; acc_phase ^= 1; }
        // The fused activation gate of the change-of-basis path (block conv1) runs
        // here, after the accumulator went back to the MMA warp: it only needs the
        // held values (CL_DBG_CLK: inside phase 1 it had cost 7 K of cfg3's 19.6 K
        // cycles per tile, all of them waited for by the next tile's MMAs). All
        // lanes take part (the partner-lane shuffle), valid or not.
        if (p.act_mode >= 0 && bs_on && !(dbg_skip(p) & 4)) {
          if constexpr (NB >= 4) {
            constexpr int W = NB / 2;
            const float inv_K = 1.f / p.act_K;
#pragma unroll
            for (int ci = 0; ci < kHold / CH; ++ci) {
              const int c0 = c_beg + ci * CH;
              const int n0 = nt * p.n_tile + c0;
              if (c0 < c_end && n0 < p.N) {
                float sg[CH / W];  // gate pre-activations, finished for the chunk's channels together (ILP)
#pragma unroll
                for (int cc = 0; cc < CH / W; ++cc) {
                  const int cq = min(n0 / W + cc, p.C_out - 1);
                  float aw[W];
                  if constexpr (W == 4) {
                    const float4 a4 = __ldg(reinterpret_cast<const float4*>(p.act_w + cq * NB + bcol * W));
                    aw[0] = a4.x; aw[1 % W] = a4.y; aw[2 % W] = a4.z; aw[3 % W] = a4.w;
                  } else {
                    const float2 a2 = __ldg(reinterpret_cast<const float2*>(p.act_w + cq * NB + bcol * W));
                    aw[0] = a2.x; aw[1 % W] = a2.y;
                  }
                  float part = 0.f;
#pragma unroll
                  for (int j = 0; j < W; ++j)
                    if ((p.act_kmask >> (bcol * W + j)) & 1u) part = fmaf(hv[ci * CH + cc * W + j], aw[j], part);
                  sg[cc] = part + __shfl_xor_sync(0xffffffffu, part, 1);
                }
#pragma unroll
                for (int cc = 0; cc < CH / W; ++cc) {
                  const int cq = min(n0 / W + cc, p.C_out - 1);
                  if (p.act_mode == 0) sg[cc] += __ldg(p.act_b + cq);
                  else if (p.act_mode == 2) sg[cc] = sg[cc] * inv_K;
                  // fast exp / reciprocal: ~1e-7 relative on the gate, far inside the block's 1e-4 bound
                  const float gte = __frcp_rn(1.f + __expf(-sg[cc]));
#pragma unroll
                  for (int j = 0; j < W; ++j) hv[ci * CH + cc * W + j] *= gte;
                }
              }
            }
          }
        }
        // fused absmax for the next conv: max finite |stored value| (float bits) and a
        // non-finite marker (NaN-sticky max of |value| bits), see finite_abs_bits
        unsigned ymax = 0, yany = 0;
        if (valid && !(dbg_skip(p) & 4))
#pragma unroll
        for (int ci = 0; ci < kHold / CH; ++ci) {
          const int c0 = c_beg + ci * CH;
          const int n0 = nt * p.n_tile + c0;
          if (c0 < c_end && n0 < p.N) {
            // W blades of one channel per store: the lane's half (change of basis) or all N_B
            constexpr int W = (NB >= 4) ? NB / 2 : NB;
            const int wv = bs_on ? W : NB;
#pragma unroll
            for (int cc = 0; cc < CH / W; ++cc) {
              if (cc * wv >= CH) break;
              const int co = n0 / wv + cc;
              if (co >= p.C_out) break;
              const long long off = bs_on ? (long long)bcol * W : 0;
              if (bs_on) {
                float h[W];
#pragma unroll
                for (int j = 0; j < W; ++j) h[j] = hv[ci * CH + cc * W + j];
                if (p.resid) {
                  const float* rp = p.resid + (((long long)b * p.C_out + co) * P_res + pres) * NB + off;
                  if constexpr (W == 2) {
                    const float2 q2 = __ldg(reinterpret_cast<const float2*>(rp));
                    h[0] += q2.x; h[1 % W] += q2.y;
                  } else {
                    const float4 q4 = __ldg(reinterpret_cast<const float4*>(rp));
                    h[0] += q4.x; h[1 % W] += q4.y; h[2 % W] += q4.z; h[3 % W] += q4.w;
                  }
                }
                if (p.y) {
                  float* yp = p.y + (((long long)b * p.C_out + co) * P_out + pix) * NB + off;
                  if constexpr (W == 2) *reinterpret_cast<float2*>(yp) = make_float2(h[0], h[1 % W]);
                  else *reinterpret_cast<float4*>(yp) = make_float4(h[0], h[1 % W], h[2 % W], h[3 % W]);
                }
#pragma unroll
                for (int j = 0; j < W; ++j) { ymax = max(ymax, finite_abs_bits(h[j])); yany = max(yany, abs_bits(h[j])); }
              } else {
                if (cc >= CH / NB) break;
                float v[NB];
#pragma unroll
                for (int j = 0; j < NB; ++j) v[j] = hv[ci * CH + cc * NB + j];
                if (p.resid) {
                  const float* rp = p.resid + (((long long)b * p.C_out + co) * P_res + pres) * NB;
                  if constexpr (NB == 2) {
                    const float2 q2 = __ldg(reinterpret_cast<const float2*>(rp));
                    v[0] += q2.x; v[1] += q2.y;
                  } else {
#pragma unroll
                    for (int j = 0; j < NB / 4; ++j) {
                      const float4 q4 = __ldg(reinterpret_cast<const float4*>(rp) + j);
                      v[4 * j] += q4.x; v[4 * j + 1] += q4.y; v[4 * j + 2] += q4.z; v[4 * j + 3] += q4.w;
                    }
                  }
                }
                if (p.y) {
                  float* yp = p.y + (((long long)b * p.C_out + co) * P_out + pix) * NB;
                  if constexpr (NB == 2) {
                    *reinterpret_cast<float2*>(yp) = make_float2(v[0], v[1]);
                  } else {
#pragma unroll
                    for (int j = 0; j < NB / 4; ++j)
                      reinterpret_cast<float4*>(yp)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                  }
                }
#pragma unroll
                for (int j = 0; j < NB; ++j) { ymax = max(ymax, finite_abs_bits(v[j])); yany = max(yany, abs_bits(v[j])); }
              }
            }
          }
        }
        if (p.amax_out) {
          if (p.k == 1) {  // 1-D: rows of one tile belong to different samples
            if (valid) {
              atomicMax(p.amax_out + b, ymax);
              if (yany >= 0x7f800000u) atomicOr(p.nf_out + b, 1u);
            }
          } else {  // one sample per tile: reduce over the warp first
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              ymax = max(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
              yany = max(yany, __shfl_xor_sync(0xffffffffu, yany, o));
            }
            if (lane == 0 && real) {
              atomicMax(p.amax_out + b, ymax);
              if (yany >= 0x7f800000u) atomicOr(p.nf_out + b, 1u);
            }
          }
        }
        continue;
      }
      // fp32-accumulator modes (tf32 / 3xTF32 / bf16): fp32 math, the next
      // chunk's TMEM load in flight while this one is processed
      const int c_stop = (dbg_skip(p) & 4) ? c_beg : c_end;
      uint32_t cur[16], nxt[16];
      bool have = c_beg < c_stop && nt * p.n_tile + c_beg < p.N;
      if (have) {
        tmem_ld16(taddr + (uint32_t)c_beg, cur);
        tmem_ld_wait_dep16(cur);
      }
      for (int c0 = c_beg; have; c0 += 16) {
        const int n0 = nt * p.n_tile + c0;
        const bool more = c0 + 16 < c_stop && n0 + 16 < p.N;
        if (more) tmem_ld16(taddr + (uint32_t)(c0 + 16), nxt);
        // the chunk's residual values (16 floats: the lane's share of every
        // channel of the chunk), loaded up front so their latencies overlap.
        // Channel cc of the chunk occupies floats [cc*wv, cc*wv + wv) of rq:
        // wv = 4 -> rq[cc]; wv = 2 (2-D under the change of basis, 8 channels
        // per chunk) -> rq[cc / 2].xy or .zw.
        float4 rq[4];
        const bool use_res = p.resid != nullptr && valid;
#pragma unroll
        for (int r = 0; r < 4; ++r) rq[r] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (use_res && (bs_on || NB == 4)) {  // NB = 8 / NB = 2 without a basis: loaded in place below
          const int wv = bs_on ? NB / 2 : NB;  // floats of one channel this lane adds
          const int nch = 16 / wv;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const int co = n0 / wv + cc;
            if (cc < nch && co < p.C_out) {
              const float* rp = p.resid + (((long long)b * p.C_out + co) * P_res + pres) * NB + (bs_on ? bcol * wv : 0);
              if (wv == 2) {
                const float2 q2 = __ldg(reinterpret_cast<const float2*>(rp));
                if (cc & 1) { rq[cc >> 1].z = q2.x; rq[cc >> 1].w = q2.y; }
                else { rq[cc >> 1].x = q2.x; rq[cc >> 1].y = q2.y; }
              } else if (cc < 4) {
                rq[cc] = __ldg(reinterpret_cast<const float4*>(rp));
              }
            }
          }
        }
        if (bs_on) {
          if constexpr (NB >= 4 && kBasisEpi) {
            // The chunk's biases, and its gate weights when no residual occupies rq
            // (block conv1), loaded for all channels up front like the residual: loaded
            // per channel right before use, each first use waited a full L1 round trip
            // (ncu, cfg3 3xTF32 conv1: long_sb 38 % of the epilogue's samples).
            constexpr int WB = NB / 2;
            float4 bq[4];
            const bool aw_in_rq = p.act_mode >= 0 && !use_res;
#pragma unroll
            for (int cc = 0; cc < 16 / WB; ++cc) {
              const int cq = min(n0 / WB + cc, p.C_out - 1);
              if constexpr (WB == 4) {
                bq[cc % 4] = __ldg(reinterpret_cast<const float4*>(p.bias_t + cq * NB + bcol * WB));
                if (aw_in_rq) rq[cc % 4] = __ldg(reinterpret_cast<const float4*>(p.act_w + cq * NB + bcol * WB));
              } else {
                const float2 b2 = __ldg(reinterpret_cast<const float2*>(p.bias_t + cq * NB + bcol * WB));
                if (cc & 1) { bq[(cc >> 1) % 4].z = b2.x; bq[(cc >> 1) % 4].w = b2.y; }
                else { bq[(cc >> 1) % 4].x = b2.x; bq[(cc >> 1) % 4].y = b2.y; }
                if (aw_in_rq) {
                  const float2 a2 = __ldg(reinterpret_cast<const float2*>(p.act_w + cq * NB + bcol * WB));
                  if (cc & 1) { rq[(cc >> 1) % 4].z = a2.x; rq[(cc >> 1) % 4].w = a2.y; }
                  else { rq[(cc >> 1) % 4].x = a2.x; rq[(cc >> 1) % 4].y = a2.y; }
                }
              }
            }
            // change of basis: lane (column bcol) produces blades bcol*W + j as
            // (s_o own[o_j] + s_p partner[p_j]) / 2; the gate sums over both lanes.
            // This loop had been instruction bound (ncu: ~640 issued instructions per
            // 16-column chunk and warp, 13.6 K cycles per cfg4 bf16 tile against 13.8 K
            // of MMAs): the signs are +-1 multipliers held in registers, bias and gate
            // weights one vector load per channel, the gate code sits behind one
            // warp-uniform branch, and the (1,1,1) / degenerate basis families take
            // compile-time picks (BCLS, as in the int8 epilogue).
            constexpr int W = NB / 2;
            const bool act = p.act_mode >= 0;
            const float act_inv_K = 1.f / p.act_K;
            // the chunk's first output address; channels step by one (P_out, N_B) plane
            float* const y_chunk = p.y ? p.y + (((long long)b * p.C_out + n0 / W) * P_out + pix) * NB + bcol * W : nullptr;
            const long long y_step = P_out * NB;
            // Linear gates: the chunk's gate biases up front, like the weights
            float ab[16 / W];
#pragma unroll
            for (int cc = 0; cc < 16 / W; ++cc)
              ab[cc] = p.act_mode == 0 ? __ldg(p.act_b + min(n0 / W + cc, p.C_out - 1)) : 0.f;
            // Three passes over the chunk's channels -- combine, gate, residual + store --
            // so that each warp-uniform condition (gate on? residual? output?) is tested
            // once per chunk instead of once per channel (ncu: 55 BRA, 133 ISETP and 73
            // LDC / LDCU of ~1000 issued instructions per 8-channel chunk).
            float hq[16];
#pragma unroll
            for (int cc = 0; cc < 16 / W; ++cc) {
              float own[W], oth[W];
              float recvA = 0.f, recvB = 0.f;
#pragma unroll
              for (int r = 0; r < W; ++r) {
                own[r] = __uint_as_float(cur[cc * W + r]);
                oth[r] = 0.f;
                if constexpr (BCLS == 2) continue;
                // BCLS 1: the partner only needs rows 1 and 2
                if (BCLS == 0 || r == 1 || r == 2) oth[r] = __shfl_xor_sync(0xffffffffu, own[r], 1);
              }
              if constexpr (BCLS == 2 && W == 4) {
                // degenerate (1,-1,0) family: lane 0 sends rows 2, 3, lane 1 rows 0, 1
                recvA = __shfl_xor_sync(0xffffffffu, bcol ? own[0] : own[2], 1);
                recvB = __shfl_xor_sync(0xffffffffu, bcol ? own[1] : own[3 % W], 1);
              }
              float bw[W];
              if constexpr (W == 4) {
                const float4 b4 = bq[cc % 4];
                bw[0] = b4.x; bw[1 % W] = b4.y; bw[2 % W] = b4.z; bw[3 % W] = b4.w;
              } else {
                const float4 b4 = bq[(cc >> 1) % 4];
                bw[0] = (cc & 1) ? b4.z : b4.x;
                bw[1 % W] = (cc & 1) ? b4.w : b4.y;
              }
#pragma unroll
              for (int j = 0; j < W; ++j) {
                float a, bq;
                if constexpr (BCLS == 1 && W == 4) {
                  a = own[(j >> 1) * 3];   // rows 0, 0, 3, 3
                  bq = oth[2 - (j >> 1)];  // rows 2, 2, 1, 1
                } else if constexpr (BCLS == 2 && W == 4) {
                  constexpr int kQ[4] = {0, 1, 1, 0};
                  a = bcol ? own[3 - kQ[j]] : own[kQ[j]];  // rows 0,1,1,0 / 3,2,2,3
                  bq = (((j == 0) || (j == 3)) != (bcol != 0)) ? recvB : recvA;
                } else {
                  a = pick_wf<W>(own, inv_o[j]);
                  bq = pick_wf<W>(oth, inv_p[j]);
                }
                // (+-a) + (+-bq) rounded once (the +-1 products are exact), then / 2 + bias
                hq[cc * W + j] = fmaf(fmaf(sgn_o[j], a, sgn_p[j] * bq), 0.5f, bw[j]);
              }
            }
            if (act) {
              float sg[16 / W];
#pragma unroll
              for (int cc = 0; cc < 16 / W; ++cc) {
                const int cq = min(n0 / W + cc, p.C_out - 1);
                float aw[W];
                if constexpr (W == 4) {
                  const float4 a4 = aw_in_rq ? rq[cc % 4]
                                             : __ldg(reinterpret_cast<const float4*>(p.act_w + cq * NB + bcol * W));
                  aw[0] = a4.x; aw[1 % W] = a4.y; aw[2 % W] = a4.z; aw[3 % W] = a4.w;
                } else {
                  float2 a2;
                  if (aw_in_rq) {
                    const float4 a4 = rq[(cc >> 1) % 4];
                    a2 = (cc & 1) ? make_float2(a4.z, a4.w) : make_float2(a4.x, a4.y);
                  } else {
                    a2 = __ldg(reinterpret_cast<const float2*>(p.act_w + cq * NB + bcol * W));
                  }
                  aw[0] = a2.x; aw[1 % W] = a2.y;
                }
                float part = 0.f;
#pragma unroll
                for (int j = 0; j < W; ++j)
                  if ((act_kml >> j) & 1u) part = fmaf(hq[cc * W + j], aw[j], part);
                sg[cc] = part + __shfl_xor_sync(0xffffffffu, part, 1);
              }
#pragma unroll
              for (int cc = 0; cc < 16 / W; ++cc) {
                if (p.act_mode == 0) sg[cc] += ab[cc];
                else if (p.act_mode == 2) sg[cc] = sg[cc] * act_inv_K;
                // fast exp / reciprocal, as in the int8 epilogue (~1e-7 relative on the gate)
                const float gte = __frcp_rn(1.f + __expf(-sg[cc]));
#pragma unroll
                for (int j = 0; j < W; ++j) hq[cc * W + j] *= gte;
              }
            }
            if (valid) {
              const int nch = min(16 / W, p.C_out - n0 / W);  // channels of this chunk that exist
              if (use_res) {  // (rq is zero for channels that do not exist)
#pragma unroll
                for (int cc = 0; cc < 16 / W; ++cc) {
                  if constexpr (W == 4) {
                    const float4 q4 = rq[cc % 4];
                    hq[cc * W] += q4.x; hq[cc * W + 1 % W] += q4.y; hq[cc * W + 2 % W] += q4.z; hq[cc * W + 3 % W] += q4.w;
                  } else {  // W == 2: channel cc is rq[cc / 2].xy (even) or .zw (odd)
                    const float4 q4 = rq[(cc >> 1) % 4];
                    hq[cc * W] += (cc & 1) ? q4.z : q4.x;
                    hq[cc * W + 1 % W] += (cc & 1) ? q4.w : q4.y;
                  }
                }
              }
              if (y_chunk) {
#pragma unroll
                for (int cc = 0; cc < 16 / W; ++cc) {
                  if (cc < nch) {
                    float* yp = y_chunk + cc * y_step;
                    if constexpr (W == 2) *reinterpret_cast<float2*>(yp) = make_float2(hq[cc * W], hq[cc * W + 1 % W]);
                    else *reinterpret_cast<float4*>(yp) = make_float4(hq[cc * W], hq[cc * W + 1 % W], hq[cc * W + 2 % W], hq[cc * W + 3 % W]);
                  }
                }
              }
            }
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < 16 / NB; ++cc) {
            const int co = n0 / NB + cc;
            const int cq = min(co, p.C_out - 1);
            float v[NB];
            {  // the channel's NB biases: vector loads from the (C_out, NB) copy
              float bw[NB];
              if constexpr (NB == 2) {
                const float2 b2 = __ldg(reinterpret_cast<const float2*>(p.bias_t + cq * NB));
                bw[0] = b2.x; bw[1] = b2.y;
              } else {
#pragma unroll
                for (int j = 0; j < NB / 4; ++j) {
                  const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias_t + cq * NB) + j);
                  bw[4 * j] = b4.x; bw[(4 * j + 1) % NB] = b4.y; bw[(4 * j + 2) % NB] = b4.z; bw[(4 * j + 3) % NB] = b4.w;
                }
              }
#pragma unroll
              for (int j = 0; j < NB; ++j) v[j] = __uint_as_float(cur[cc * NB + j]) + bw[j];
            }
            if (!valid || co >= p.C_out) continue;
            if (p.act_mode >= 0) {
              const float gte = act_gate<NB>(v, p.act_mode, p.act_w + co * NB,
                                             p.act_mode == 0 ? __ldg(p.act_b + co) : 0.f, p.act_K, p.act_kmask);
#pragma unroll
              for (int j = 0; j < NB; ++j) v[j] *= gte;
            }
            if (use_res) {
              if constexpr (NB == 4) {
                const float4 q4 = rq[cc % 4];
                v[0] += q4.x; v[1 % NB] += q4.y; v[2 % NB] += q4.z; v[3 % NB] += q4.w;
              } else if constexpr (NB == 2) {
                const float2 q2 = __ldg(reinterpret_cast<const float2*>(
                    p.resid + (((long long)b * p.C_out + co) * P_res + pres) * NB));
                v[0] += q2.x; v[1 % NB] += q2.y;
              } else {
                const float* rp = p.resid + (((long long)b * p.C_out + co) * P_res + pres) * NB;
#pragma unroll
                for (int j = 0; j < NB / 4; ++j) {
                  const float4 q4 = __ldg(reinterpret_cast<const float4*>(rp) + j);
                  v[4 * j] += q4.x; v[(4 * j + 1) % NB] += q4.y; v[(4 * j + 2) % NB] += q4.z; v[(4 * j + 3) % NB] += q4.w;
                }
              }
            }
            if (p.y) {
              float* yp = p.y + (((long long)b * p.C_out + co) * P_out + pix) * NB;
              if constexpr (NB == 2) {
                *reinterpret_cast<float2*>(yp) = make_float2(v[0], v[1]);
              } else {
#pragma unroll
                for (int j = 0; j < NB / 4; ++j)
                  reinterpret_cast<float4*>(yp)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              }
            }
            if (p.y_bf16) {
              // next conv's packed bf16 operand: (B, Gy, P, 16 B), cpg = 8 / NB channels per group
              constexpr int cpg = 8 / NB;
              __nv_bfloat16* yp = p.y_bf16 + (((long long)b * p.ybf_groups + co / cpg) * P_out + pix) * 8 + (co % cpg) * NB;
              uint32_t u[NB / 2];
#pragma unroll
              for (int j = 0; j < NB / 2; ++j) {
                __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
                u[j] = *reinterpret_cast<uint32_t*>(&hh);
              }
              if constexpr (NB == 2) *reinterpret_cast<uint32_t*>(yp) = u[0];
              else if constexpr (NB == 4) *reinterpret_cast<uint2*>(yp) = make_uint2(u[0], u[1]);
              else *reinterpret_cast<uint4*>(yp) = make_uint4(u[0], u[1 % (NB / 2)], u[2 % (NB / 2)], u[3 % (NB / 2)]);
            }
          }
        }
        have = more;
        if (more) {
          tmem_ld_wait_dep16(nxt);
#pragma unroll
          for (int c = 0; c < 16; ++c) cur[c] = nxt[c];
        }
      }
      release_acc<PAIR>(&tempty[acc]);
      if (kDbg && p.dbg_acc && threadIdx.x == 128) {  // timing instrumentation: epilogue cycles per tile
        atomicAdd(p.dbg_acc, (unsigned long long)(clock64() - dbg_t0));
        atomicAdd(p.dbg_acc + 1, 1ull);
      }
      if (++acc == slots) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4 + 4 * kEpiGroups) {
    // ===================== 3xTF32 splitter =====================
    if constexpr (kSplit) {
      const int tid = threadIdx.x - 32 * (4 + 4 * kEpiGroups);
      auto split = [&](uint8_t* buf, uint32_t bytes, uint32_t lo_off) {
        uint4* a = reinterpret_cast<uint4*>(buf);
        float4* lo = reinterpret_cast<float4*>(buf + lo_off);
        const int n4 = (int)(bytes / 16);
        for (int i = tid; i < n4; i += 128) {
          // hi = round-to-nearest tf32, lo = the remainder rounded to tf32
          // (both exact for the tensor core, which reads the top 19 bits; a
          // truncated hi left |lo| up to 2^-10 |x| and lo's own truncation
          // an error of 2^-20 |x|, 16x fp32's)
          uint4 v = a[i];
          uint4 h;
          h.x = tf32_rna_bits(v.x); h.y = tf32_rna_bits(v.y); h.z = tf32_rna_bits(v.z); h.w = tf32_rna_bits(v.w);
          float4 l;
          l.x = __uint_as_float(tf32_rna_bits(__float_as_uint(__uint_as_float(v.x) - __uint_as_float(h.x))));
          l.y = __uint_as_float(tf32_rna_bits(__float_as_uint(__uint_as_float(v.y) - __uint_as_float(h.y))));
          l.z = __uint_as_float(tf32_rna_bits(__float_as_uint(__uint_as_float(v.z) - __uint_as_float(h.z))));
          l.w = __uint_as_float(tf32_rna_bits(__float_as_uint(__uint_as_float(v.w) - __uint_as_float(h.w))));
          a[i] = h;
          lo[i] = l;
        }
        fence_proxy_async_smem();
      };
      int stage = 0;
      uint32_t phase = 0;
      int hsl = 0;
      uint32_t hphase = 0;
      for (int it = 0;; ++it) {
        if (sched_read(it, false) < 0) break;
        if (p.halo) {
          for (int gsi = 0; gsi < p.n_gs; ++gsi) {
            mbar_wait(&hfull[hsl], hphase);
            split(smem + (size_t)hsl * p.halo_slot, p.halo_bytes, p.a_bytes);
            if constexpr (PAIR) mbar_arrive_leader(&hlo[hsl]); else mbar_arrive(&hlo[hsl]);
            if (++hsl == HS) { hsl = 0; hphase ^= 1; }
          }
          continue;
        }
        for (int kit = 0; kit < p.k_iters; ++kit) {
          mbar_wait(&full[stage], phase);
          split(ring + (size_t)stage * p.stage_bytes, p.a_bytes, p.a_bytes);
          mbar_arrive(&lo_ready[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // no CTA leaves while its pair may still touch its smem / TMEM
  if (kDbg && p.dbg_acc && threadIdx.x == 0) {  // timing instrumentation: spread of the CTAs' finish times
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicMax(p.dbg_acc + 6, t_end);
    atomicMax(p.dbg_acc + 7, ~t_end);
  }
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_cg2(tmem_base, p.tmem_cols);
    else tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

template <int NB, int PREC, bool PAIR, int BCLS = 0, bool GROUPS = false>
static cudaError_t launch_t(const ConvPlan& plan, const CUtensorMap& tmap, const CUtensorMap& bmap,
                            const ConvKParams& p, int grid, cudaStream_t s) {
  auto kfn = conv_tc_kernel<NB, PREC, PAIR, BCLS, GROUPS>;
  cudaError_t e = ensure_smem_optin(reinterpret_cast<const void*>(kfn), (int)plan.smem_bytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(conv_threads(PREC, NB));
  cfg.dynamicSmemBytes = plan.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)p.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kfn, tmap, bmap, p);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int NB>
static cudaError_t launch_nb(const ConvPlan& plan, const CUtensorMap& tmap, const CUtensorMap& bmap,
                             const ConvKParams& p, int grid, cudaStream_t s) {
  if (plan.prec == kPrecFp32 && p.n_groups > 1) {  // long exact-mode reductions (generic basis picks)
    if (p.pair) return launch_t<NB, kPrecFp32, true, 0, true>(plan, tmap, bmap, p, grid, s);
    return launch_t<NB, kPrecFp32, false, 0, true>(plan, tmap, bmap, p, grid, s);
  }
  if (p.pair) {
    switch (plan.prec) {
      case kPrecFp32:
        if constexpr (NB == 8) {
          if (p.bcls == 1) return launch_t<NB, kPrecFp32, true, 1>(plan, tmap, bmap, p, grid, s);
          if (p.bcls == 2) return launch_t<NB, kPrecFp32, true, 2>(plan, tmap, bmap, p, grid, s);
        }
        return launch_t<NB, kPrecFp32, true>(plan, tmap, bmap, p, grid, s);
      case kPrecTf32:
        if constexpr (NB == 8) {
          if (p.bcls == 1) return launch_t<NB, kPrecTf32, true, 1>(plan, tmap, bmap, p, grid, s);
          if (p.bcls == 2) return launch_t<NB, kPrecTf32, true, 2>(plan, tmap, bmap, p, grid, s);
        }
        return launch_t<NB, kPrecTf32, true>(plan, tmap, bmap, p, grid, s);
      case kPrecBf16:
        if constexpr (NB == 8) {
          if (p.bcls == 1) return launch_t<NB, kPrecBf16, true, 1>(plan, tmap, bmap, p, grid, s);
          if (p.bcls == 2) return launch_t<NB, kPrecBf16, true, 2>(plan, tmap, bmap, p, grid, s);
        }
        return launch_t<NB, kPrecBf16, true>(plan, tmap, bmap, p, grid, s);
      default:
        if constexpr (NB == 8) {
          if (p.bcls == 1) return launch_t<NB, kPrec3xTf32, true, 1>(plan, tmap, bmap, p, grid, s);
          if (p.bcls == 2) return launch_t<NB, kPrec3xTf32, true, 2>(plan, tmap, bmap, p, grid, s);
        }
        return launch_t<NB, kPrec3xTf32, true>(plan, tmap, bmap, p, grid, s);
    }
  }
  switch (plan.prec) {
    case kPrecFp32: return launch_t<NB, kPrecFp32, false>(plan, tmap, bmap, p, grid, s);
    case kPrec3xTf32: return launch_t<NB, kPrec3xTf32, false>(plan, tmap, bmap, p, grid, s);
    case kPrecTf32: return launch_t<NB, kPrecTf32, false>(plan, tmap, bmap, p, grid, s);
    default: return launch_t<NB, kPrecBf16, false>(plan, tmap, bmap, p, grid, s);
  }
}

cudaError_t launch_conv(const ConvPlan& plan, const CUtensorMap& tmap, const CUtensorMap& bmap,
                        const ConvKParams& p, int grid, cudaStream_t s) {
#ifdef CL_PROBE_ONE  // SASS experiments only (nvcc -cubin -DCL_PROBE_ONE=<prec>): one instantiation
  return launch_t<8, CL_PROBE_ONE, true>(plan, tmap, bmap, p, grid, s);
#else
  if (plan.nb == 2) return launch_nb<2>(plan, tmap, bmap, p, grid, s);
  if (plan.nb == 4) return launch_nb<4>(plan, tmap, bmap, p, grid, s);
  return launch_nb<8>(plan, tmap, bmap, p, grid, s);
#endif
}

// fp32 protocol (B, C, P, NB) -> packed 16-byte row groups (B, G, P, [ncol x] 16 B):
// group g holds channels g*cpg .. g*cpg+cpg-1 (zero beyond C), w values each,
// as bf16 (esize 2) or fp32 (esize 4); cpg = 16 / (w * esize). Without a change
// of basis w = NB (the blades); with one, each pixel yields ncol rows of the
// transformed components x'[c*w + r] = sum_I T[c*w + r][I] x[I].
__global__ void transpose_kernel(const float* __restrict__ in, float* __restrict__ out, int rows, int cols) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * cols; i += gridDim.x * blockDim.x)
    out[(i % cols) * rows + i / cols] = in[i];
}
cudaError_t launch_transpose(const float* in, float* out, int rows, int cols, cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  transpose_kernel<<<(rows * cols + 255) / 256, 256, 0, s>>>(in, out, rows, cols);
  count_launch();
  return cudaGetLastError();
}

template <int NB, int ESIZE, bool BASIS>
__global__ void __launch_bounds__(256) pack_rows_kernel(const float* __restrict__ x, uint4* __restrict__ out,
                                                        long long B, int C, long long P, int G, Basis bs) {
  constexpr int NCOL = BASIS ? 2 : 1;
  constexpr int W = BASIS ? NB / 2 : NB;   // components per channel and row
  constexpr int NV = 16 / ESIZE;           // values per 16-byte row
  constexpr int CPG = NV / W;              // channels per row group
  float T[BASIS ? NB * NB : 1];            // x'[c*W + r] = sum_I T[c*W + r][I] x[I] (entries 0, +-1)
  if constexpr (BASIS) {
#pragma unroll
    for (int a = 0; a < NB; ++a)
#pragma unroll
      for (int I = 0; I < NB; ++I) T[a * NB + I] = (float)bs.T[a * 8 + I];
  }
  const long long total = B * G * P;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pp = i % P;
    const long long bg = i / P;
    const int g = (int)(bg % G);
    const long long b = bg / G;
    float v[NCOL][NV];
#pragma unroll
    for (int cl = 0; cl < CPG; ++cl) {
      const int c = g * CPG + cl;
      float m[NB];
      if (c < C) {
        const float* src = x + ((b * C + c) * P + pp) * NB;
        if constexpr (NB == 2) {
          const float2 q = __ldg(reinterpret_cast<const float2*>(src));
          m[0] = q.x; m[1] = q.y;
        } else {
#pragma unroll
          for (int h = 0; h < NB / 4; ++h) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(src) + h);
            m[4 * h] = q.x; m[4 * h + 1] = q.y; m[4 * h + 2] = q.z; m[4 * h + 3] = q.w;
          }
        }
      } else {
#pragma unroll
        for (int I = 0; I < NB; ++I) m[I] = 0.f;
      }
#pragma unroll
      for (int col = 0; col < NCOL; ++col)
#pragma unroll
        for (int r = 0; r < W; ++r) {
          float xv;
          if constexpr (BASIS) {
            xv = 0.f;
#pragma unroll
            for (int I = 0; I < NB; ++I) xv = fmaf(T[(col * W + r) * NB + I], m[I], xv);  // exact: +-1 / 0 terms
          } else {
            xv = m[r];
          }
          v[col][cl * W + r] = xv;
        }
    }
#pragma unroll
    for (int col = 0; col < NCOL; ++col) {
      uint4 u;
      if constexpr (ESIZE == 4) {
        u = make_uint4(__float_as_uint(v[col][0]), __float_as_uint(v[col][1]), __float_as_uint(v[col][2]),
                       __float_as_uint(v[col][3]));
      } else {
        __nv_bfloat162 h;
        h = __floats2bfloat162_rn(v[col][0], v[col][1]); u.x = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[col][2], v[col][3]); u.y = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[col][4 % NV], v[col][5 % NV]); u.z = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[col][6 % NV], v[col][7 % NV]); u.w = *reinterpret_cast<uint32_t*>(&h);
      }
      out[i * NCOL + col] = u;
    }
  }
}

template <int NB, int ESIZE, bool BASIS>
static void launch_pack_t(const float* x, void* out, long long B, int C, long long P, int G, const Basis& bs,
                          cudaStream_t s) {
  auto kern = pack_rows_kernel<NB, ESIZE, BASIS>;
  const int per_sm = resident_blocks_per_sm(reinterpret_cast<const void*>(kern), 256, 0);
  const long long total = B * G * P;
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)num_sms() * per_sm;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, 256, 0, s>>>(x, reinterpret_cast<uint4*>(out), B, C, P, G, bs);
}

cudaError_t launch_pack_rows(const float* x, void* out, int nb, int esize, long long B, int C, long long P, int G,
                             const Basis& bs, cudaStream_t s) {
  if (B * G * P == 0) return cudaSuccess;
  if (bs.on) {
    if (nb == 4) { if (esize == 2) launch_pack_t<4, 2, true>(x, out, B, C, P, G, bs, s); else launch_pack_t<4, 4, true>(x, out, B, C, P, G, bs, s); }
    else { if (esize == 2) launch_pack_t<8, 2, true>(x, out, B, C, P, G, bs, s); else launch_pack_t<8, 4, true>(x, out, B, C, P, G, bs, s); }
  } else if (nb == 2) {
    if (esize == 2) launch_pack_t<2, 2, false>(x, out, B, C, P, G, bs, s); else launch_pack_t<2, 4, false>(x, out, B, C, P, G, bs, s);
  } else if (nb == 4) {
    if (esize == 2) launch_pack_t<4, 2, false>(x, out, B, C, P, G, bs, s); else launch_pack_t<4, 4, false>(x, out, B, C, P, G, bs, s);
  } else {
    if (esize == 2) launch_pack_t<8, 2, false>(x, out, B, C, P, G, bs, s); else launch_pack_t<8, 4, false>(x, out, B, C, P, G, bs, s);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace cl
