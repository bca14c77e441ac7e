// common.cuh -- shared device/host helpers for the sm_100a Clifford path:
// integer Clifford algebra (host+device), and thin inline-PTX wrappers for
// mbarrier, TMA (cp.async.bulk[.tensor]), tcgen05 (alloc / mma / commit / ld)
// and the UMMA shared-memory / instruction descriptors.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define CL_HD __host__ __device__ __forceinline__

namespace cl {

// ---------------------------------------------------------------------------
// Clifford algebra on blade bitmasks (restated from algebra.py:73-99).
// e_I e_J = (-1)^swaps * prod_{b in I&J} g_b * e_{I^J}; swaps counts pairs
// (a in I, b in J) with a > b.
// ---------------------------------------------------------------------------
CL_HD int popc(unsigned v) {
#ifdef __CUDA_ARCH__
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}

CL_HD int reorder_sign(int i, int j) {
  int swaps = 0;
  for (int s = 1; s < 8; ++s) swaps += popc((unsigned)((i >> s) & j));
  return (swaps & 1) ? -1 : 1;
}

CL_HD int blade_coeff(int i, int j, const int* g, int k) {
  int c = reorder_sign(i, j);
  const int shared = i & j;
  for (int b = 0; b < k; ++b)
    if ((shared >> b) & 1) c *= g[b];
  return c;
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
#if defined(__CUDACC__)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Wait with cluster-scope acquire: for data a peer CTA wrote into this CTA's
// shared memory before its release-cluster arrive on `bar`.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Store a 64-bit value into CTA `rank`'s copy of a shared variable, then
// arrive (release, cluster scope) on that CTA's copy of `bar`.
__device__ __forceinline__ void st_remote_arrive(long long* var, long long v, uint64_t* bar, uint32_t rank) {
  uint32_t rv, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rv) : "r"(smem_u32(var)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(rv), "l"(v) : "memory");
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
}

// Wait with back-off for warps that are off the critical path (the epilogue
// waiting for an accumulator, the producer waiting for a free slot): a tight
// try_wait spin from many warps floods the MIO queue that tcgen05.mma issue
// shares, so sleep between polls.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t done;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}

// one lane of a converged warp (elect.sync): the MMA issuer idiom
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n}"
      : "=r"(pred));
  return pred;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA: 5-D tiled tensor load into this CTA's shared memory.
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(c4)
      : "memory");
}
// ---- 2-SM (cta_group::2) variants: a CTA pair shares one M=256 MMA ---------
// Shared::cluster address of the same object in the pair's leader (rank 0):
// cluster-window shared addresses carry the CTA rank in bit 24.
__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }
// TMA into this CTA's shared memory, completing bytes on the LEADER's barrier.
__device__ __forceinline__ void tma_load_5d_cg2(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_addr(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// Remote (or local) arrive on the leader's copy of a barrier.
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(bar)) : "memory");
}
// The same arrival without release semantics: for hand-offs that publish no
// memory (an epilogue warp returning a TMEM slot: its tcgen05.ld results are
// in registers after tcgen05.wait::ld, ordered by tcgen05.fence::before_thread_sync).
// The release form makes the thread wait for ALL its outstanding global stores
// first (ERRBAR / MEMBAR in the SASS) -- the previous tile's output, a DRAM
// write round trip per returned slot (ncu, cfg3 3xTF32 conv1: 15 % of the
// epilogue warps' samples sat on that fence).
__device__ __forceinline__ void mbar_arrive_leader_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(bar)) : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// Non-tensor bulk copy global -> shared (size multiple of 16 B).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Multicast bulk copy: the same bytes land at `dst` (and complete_tx on `bar`,
// same offsets) in every CTA of the cluster selected by cta_mask.
__device__ __forceinline__ void bulk_load_multicast(void* dst, const void* src, uint32_t bytes,
                                                    uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// load a float from the same shared-memory variable of CTA `rank` of this cluster (DSMEM)
__device__ __forceinline__ float ld_shared_cluster_f32(const float* local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// ---- tcgen05 ---------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::f16 (bf16 operands, fp32 accumulator)
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::i8 (s8 x s8 -> s32 accumulator: exact integer accumulation)
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// cta_group::2 MMAs (issued by the pair leader; A rows and B columns split
// between the two CTAs' shared memory at the same offsets, D in both TMEMs)
__device__ __forceinline__ void mma_tf32_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_i8_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-converged issue: every lane runs the issue loop on warp-uniform values
// (descriptors stay on the uniform datapath) and the instruction is guarded so
// only the lane with `issue` set performs it.
#define CL_MMA_GUARDED(NAME, KIND, GROUP)                                                                  \
  __device__ __forceinline__ void NAME(uint32_t issue, uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,   \
                                       uint32_t idesc, uint32_t accumulate) {                             \
    asm volatile(                                                                                         \
        "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"                 \
        "@q tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),        \
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(issue)                                   \
        : "memory");                                                                                      \
  }
CL_MMA_GUARDED(mma_tf32_g, "tf32", "1")
CL_MMA_GUARDED(mma_bf16_g, "f16", "1")
CL_MMA_GUARDED(mma_i8_g, "i8", "1")
CL_MMA_GUARDED(mma_tf32_cg2_g, "tf32", "2")
CL_MMA_GUARDED(mma_bf16_cg2_g, "f16", "2")
CL_MMA_GUARDED(mma_i8_cg2_g, "i8", "2")
#undef CL_MMA_GUARDED
__device__ __forceinline__ void mma_commit_g(uint32_t issue, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar)),
      "r"(issue)
      : "memory");
}
__device__ __forceinline__ void mma_commit_cg2_g(uint32_t issue, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %2;\n}" ::"r"(
          smem_u32(bar)),
      "r"(issue), "h"((uint16_t)3)
      : "memory");
}

// Split-descriptor variants: the 64-bit descriptors travel as (lo, hi) 32-bit
// halves and are joined inside the asm, so the per-MMA address arithmetic is
// 32-bit and stays on the uniform datapath (the high halves are loop constants).
#define CL_MMA_SPLIT(NAME, KIND, GROUP)                                                                    \
  __device__ __forceinline__ void NAME(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi,     \
                                       uint32_t b_lo, uint32_t b_hi, uint32_t idesc, uint32_t accumulate) { \
    asm volatile(                                                                                         \
        "{\n\t.reg .pred p, q;\n\t.reg .b64 da, db;\n\t"                                                  \
        "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"                                                 \
        "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\t"                                                 \
        "@q tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], da, db, %5, p;\n}" ::"r"(d_tmem),        \
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate), "r"(issue)                \
        : "memory");                                                                                      \
  }
CL_MMA_SPLIT(mma_tf32_s, "tf32", "1")
CL_MMA_SPLIT(mma_bf16_s, "f16", "1")
CL_MMA_SPLIT(mma_i8_s, "i8", "1")
CL_MMA_SPLIT(mma_tf32_cg2_s, "tf32", "2")
CL_MMA_SPLIT(mma_bf16_cg2_s, "f16", "2")
CL_MMA_SPLIT(mma_i8_cg2_s, "i8", "2")
#undef CL_MMA_SPLIT

// KS consecutive K steps of one pipeline stage in ONE asm block (tf32 / f16
// kinds): the 64-bit descriptors are joined once and advanced by 64-bit adds
// inside the block (straight-line), so per MMA the issue path is an add pair
// plus the MMA. Per-MMA asm calls cost ~16 SASS instructions each
// (R2UR.BROADCAST of every operand, VOTEU, UMOV), which left N = 128 stages
// MMA-issue bound (cfg4 bf16: tensor pipe 42 %). `issue` guards the MMAs
// (warp-converged issue); `acc0` is the first MMA's accumulate flag; the
// strides are in 16-byte descriptor units. (Generated: one body per KS.)
// One K step of the exact (int8) mode in ONE asm block: the 10 digit-pair
// MMAs D_L += A_i * B_j (i + j = L <= 3, 4 digits each; conv_tc.cu Ozaki
// levels), the 4 A-plane / 4 B-image descriptors and the 4 level columns
// formed once. acc0 = accumulate flag of each level's first MMA.
__device__ __forceinline__ void mma_i8_kstep(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                        uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_img, uint32_t b_img,
                                        uint32_t level_cols) {
  asm volatile(
        "{\n\t.reg .pred p, q, t;\n\t.reg .b64 a0, a1, a2, a3, b0, b1, b2, b3, sa, sb;\n\t.reg .b32 d1, d2, d3;\n\t"
        "mov.b64 a0, {%1, %2};\n\tmov.b64 b0, {%3, %4};\n\t"
        "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
        "add.s64 a1, a0, sa;\n\tadd.s64 a2, a1, sa;\n\tadd.s64 a3, a2, sa;\n\t"
        "add.s64 b1, b0, sb;\n\tadd.s64 b2, b1, sb;\n\tadd.s64 b3, b2, sb;\n\t"
        "add.u32 d1, %0, %10;\n\tadd.u32 d2, d1, %10;\n\tadd.u32 d3, d2, %10;\n\t"
        "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [%0], a0, b0, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d1], a0, b1, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d1], a1, b0, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d2], a0, b2, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d2], a1, b1, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d2], a2, b0, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d3], a0, b3, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d3], a1, b2, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d3], a2, b1, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::i8 [d3], a3, b0, %5, t;\n\t"
        "}"
        ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_img),
        "r"(b_img), "r"(level_cols)
      : "memory");
}
__device__ __forceinline__ void mma_i8_cg2_kstep(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                        uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_img, uint32_t b_img,
                                        uint32_t level_cols) {
  asm volatile(
        "{\n\t.reg .pred p, q, t;\n\t.reg .b64 a0, a1, a2, a3, b0, b1, b2, b3, sa, sb;\n\t.reg .b32 d1, d2, d3;\n\t"
        "mov.b64 a0, {%1, %2};\n\tmov.b64 b0, {%3, %4};\n\t"
        "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
        "add.s64 a1, a0, sa;\n\tadd.s64 a2, a1, sa;\n\tadd.s64 a3, a2, sa;\n\t"
        "add.s64 b1, b0, sb;\n\tadd.s64 b2, b1, sb;\n\tadd.s64 b3, b2, sb;\n\t"
        "add.u32 d1, %0, %10;\n\tadd.u32 d2, d1, %10;\n\tadd.u32 d3, d2, %10;\n\t"
        "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [%0], a0, b0, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d1], a0, b1, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d1], a1, b0, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d2], a0, b2, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d2], a1, b1, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d2], a2, b0, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d3], a0, b3, %5, p;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d3], a1, b2, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d3], a2, b1, %5, t;\n\t"
        "@q tcgen05.mma.cta_group::2.kind::i8 [d3], a3, b0, %5, t;\n\t"
        "}"
        ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_img),
        "r"(b_img), "r"(level_cols)
      : "memory");
}
template <int KS>
__device__ __forceinline__ void mma_tf32_ks(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                         uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_step, uint32_t b_step) {
  static_assert(KS == 1 || KS == 2 || KS == 4 || KS == 8, "K steps per stage");
  if constexpr (KS == 1) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 2) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 4) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 8) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
}
template <int KS>
__device__ __forceinline__ void mma_bf16_ks(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                         uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_step, uint32_t b_step) {
  static_assert(KS == 1 || KS == 2 || KS == 4 || KS == 8, "K steps per stage");
  if constexpr (KS == 1) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 2) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 4) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 8) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
}
template <int KS>
__device__ __forceinline__ void mma_tf32_cg2_ks(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                         uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_step, uint32_t b_step) {
  static_assert(KS == 1 || KS == 2 || KS == 4 || KS == 8, "K steps per stage");
  if constexpr (KS == 1) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 2) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 4) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 8) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
}
template <int KS>
__device__ __forceinline__ void mma_bf16_cg2_ks(uint32_t issue, uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                         uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_step, uint32_t b_step) {
  static_assert(KS == 1 || KS == 2 || KS == 4 || KS == 8, "K steps per stage");
  if constexpr (KS == 1) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 2) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 4) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
  else if constexpr (KS == 8) {
    asm volatile(
          "{\n\t.reg .pred p, q, t;\n\t.reg .b64 da, db, sa, sb;\n\t"
          "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
          "cvt.u64.u32 sa, %8;\n\tcvt.u64.u32 sb, %9;\n\t"
          "setp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %7, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "add.s64 da, da, sa;\n\tadd.s64 db, db, sb;\n\t"
          "@q tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, t;\n\t"
          "}"
          ::"r"(d_tmem), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(issue), "r"(a_step),
          "r"(b_step)
        : "memory");
  }
}

// KS MMAs of one stage issued by the whole (converged) warp: elect.sync inside
// the asm picks the issuing lane, so ptxas emits bare UTC*MMA instructions on
// uniform registers (no per-lane guard, no R2UR.BROADCAST / VOTEU). The
// descriptor low halves advance by 32-bit adds (start-address field; the
// high halves are loop constants). KIND: 1 = f16 (bf16), 2 = tf32. acc0 =
// accumulate flag of the first MMA. Must be called by all 32 lanes; the
// matching commit is commit_e (elect.sync picks the same lowest lane).
#define CL_MMA_E_HEAD                                                                                    \
  "{\n\t.reg .pred e, p;\n\t.reg .b32 al, bl;\n\t.reg .b64 da, db;\n\t"                                  \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\t"                                              \
  "mov.b32 al, %1;\n\tmov.b32 bl, %3;\n\tmov.b64 da, {al, %2};\n\tmov.b64 db, {bl, %4};\n\t"
#define CL_MMA_E_NEXT "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\tmov.b64 da, {al, %2};\n\tmov.b64 db, {bl, %4};\n\t"
#define CL_MMA_E_ARGS                                                                                    \
  ::"r"(d), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(a_step), "r"(b_step) \
      : "memory"
template <int KIND, int CG, int KS>
__device__ __forceinline__ void mma_stage_e(uint32_t d, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                            uint32_t idesc, uint32_t acc0, uint32_t a_step, uint32_t b_step) {
  static_assert(KIND == 1 || KIND == 2, "f16 / tf32 kinds");
  static_assert(CG == 1 || CG == 2, "cta_group");
  static_assert(KS == 1 || KS == 2 || KS == 4 || KS == 8, "K steps per stage");
  // (asm strings must be literals: one body per (KIND, CG, KS))
  if constexpr (CG == 2 && KIND == 1) {
    if constexpr (KS == 1) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 2) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 4) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
  } else if constexpr (CG == 2 && KIND == 2) {
    if constexpr (KS == 1) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 2) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 4) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
  } else if constexpr (CG == 1 && KIND == 1) {
    if constexpr (KS == 1) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 2) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 4) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
  } else {
    if constexpr (KS == 1) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 2) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else if constexpr (KS == 4) asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
    else asm volatile(CL_MMA_E_HEAD "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n\t" CL_MMA_E_NEXT "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, 1;\n}" CL_MMA_E_ARGS);
  }
}
// 3xTF32: KS K steps of 3 tf32 MMAs each: the cross terms A_lo*B_hi + A_hi*B_lo
// go to the tile-long lo accumulator d_lo, A_hi*B_hi to the group slot d
// (kX3GroupK, internal.h; the lo images sit a_img / b_img 16-byte units after
// the hi ones); same issue conventions as mma_stage_e. acc0 / acc_lo0 = the
// accumulate flags of the first hi / first lo MMA.
#define CL_X3_HEAD                                                                                       \
  "{\n\t.reg .pred e, p, q;\n\t.reg .b32 al, bl, t;\n\t.reg .b64 da, db, dl;\n\t"                        \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\tsetp.ne.b32 q, %12, 0;\n\t"                   \
  "mov.b32 al, %1;\n\tmov.b32 bl, %3;\n\t"
#define CL_X3_STEP(CGS, ACC, ACCL)                                                                       \
  "add.u32 t, al, %9;\n\tmov.b64 dl, {t, %2};\n\tmov.b64 db, {bl, %4};\n\t"                                \
  "@e tcgen05.mma.cta_group::" CGS ".kind::tf32 [%11], dl, db, %5, " ACCL ";\n\t"                          \
  "add.u32 t, bl, %10;\n\tmov.b64 da, {al, %2};\n\tmov.b64 dl, {t, %4};\n\t"                               \
  "@e tcgen05.mma.cta_group::" CGS ".kind::tf32 [%11], da, dl, %5, 1;\n\t"                                  \
  "@e tcgen05.mma.cta_group::" CGS ".kind::tf32 [%0], da, db, %5, " ACC ";\n\t"                             \
  "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\t"
#define CL_X3_ARGS                                                                                        \
  ::"r"(d), "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(a_step), "r"(b_step), \
      "r"(a_img), "r"(b_img), "r"(d_lo), "r"(acc_lo0)                                                      \
      : "memory"
template <int CG, int KS>
__device__ __forceinline__ void mma_stage_x3_e(uint32_t d, uint32_t d_lo, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                               uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t acc_lo0,
                                               uint32_t a_step, uint32_t b_step, uint32_t a_img, uint32_t b_img) {
  static_assert(KS == 1 || KS == 2 || KS == 4 || KS == 8, "K steps per stage");
  if constexpr (CG == 2) {
    if constexpr (KS == 1) asm volatile(CL_X3_HEAD CL_X3_STEP("2", "p", "q") "}" CL_X3_ARGS);
    else if constexpr (KS == 2) asm volatile(CL_X3_HEAD CL_X3_STEP("2", "p", "q") CL_X3_STEP("2", "1", "1") "}" CL_X3_ARGS);
    else if constexpr (KS == 4)
      asm volatile(CL_X3_HEAD CL_X3_STEP("2", "p", "q") CL_X3_STEP("2", "1", "1") CL_X3_STEP("2", "1", "1")
                       CL_X3_STEP("2", "1", "1") "}" CL_X3_ARGS);
    else
      asm volatile(CL_X3_HEAD CL_X3_STEP("2", "p", "q") CL_X3_STEP("2", "1", "1") CL_X3_STEP("2", "1", "1")
                       CL_X3_STEP("2", "1", "1") CL_X3_STEP("2", "1", "1") CL_X3_STEP("2", "1", "1")
                       CL_X3_STEP("2", "1", "1") CL_X3_STEP("2", "1", "1") "}" CL_X3_ARGS);
  } else {
    if constexpr (KS == 1) asm volatile(CL_X3_HEAD CL_X3_STEP("1", "p", "q") "}" CL_X3_ARGS);
    else if constexpr (KS == 2) asm volatile(CL_X3_HEAD CL_X3_STEP("1", "p", "q") CL_X3_STEP("1", "1", "1") "}" CL_X3_ARGS);
    else if constexpr (KS == 4)
      asm volatile(CL_X3_HEAD CL_X3_STEP("1", "p", "q") CL_X3_STEP("1", "1", "1") CL_X3_STEP("1", "1", "1")
                       CL_X3_STEP("1", "1", "1") "}" CL_X3_ARGS);
    else
      asm volatile(CL_X3_HEAD CL_X3_STEP("1", "p", "q") CL_X3_STEP("1", "1", "1") CL_X3_STEP("1", "1", "1")
                       CL_X3_STEP("1", "1", "1") CL_X3_STEP("1", "1", "1") CL_X3_STEP("1", "1", "1")
                       CL_X3_STEP("1", "1", "1") CL_X3_STEP("1", "1", "1") "}" CL_X3_ARGS);
  }
}
#undef CL_X3_HEAD
#undef CL_X3_STEP
#undef CL_X3_ARGS
#undef CL_MMA_E_HEAD
#undef CL_MMA_E_NEXT
#undef CL_MMA_E_ARGS
// Commit (whole converged warp; elect.sync picks the lane that issued the MMAs).
template <int CG>
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  if constexpr (CG == 2)
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}

// Commit the pair's MMAs to the barrier at the same offset in both CTAs.
__device__ __forceinline__ void mma_commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Commit arriving on the barrier at the same offset in every CTA of cta_mask.
__device__ __forceinline__ void mma_commit_multicast(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
// tcgen05.wait::ld that also ties the loaded registers to the wait, so the
// compiler cannot move their uses above it (for loads left in flight while
// other work runs).
// fp32 bits rounded to the nearest tf32 (ties away; cvt.rna.tf32.f32)
__device__ __forceinline__ uint32_t tf32_rna_bits(uint32_t u) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(__uint_as_float(u)));
  return r;
}
// Start the cache line of a global address towards L2 (no register, no wait).
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// 16 columns of this thread's TMEM lane (32x32b shape, like tmem_ld16)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_wait_dep16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 lanes x N consecutive 32-bit columns (N = 4 or 8).
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
  }
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

#endif  // __CUDACC__

// ---- int8 digit slicing (kPrecFp32, see slice.cu) --------------------------
// v = s * sum_i d_i 2^(-7-8(i-1)) with balanced base-256 digits d_i in [-128, 127]
// (two's-complement bytes of the rounded fixed-point value).
#if defined(__CUDACC__)
// power-of-two s with amax * 128/126 <= s: the leading digit stays in [-127, 127]
// |v| as float bits, for max-reductions as unsigned integers: NaN (> Inf >
// any finite) sticks, where fmaxf would drop it.
__device__ __forceinline__ unsigned abs_bits(float v) { return __float_as_uint(v) & 0x7fffffffu; }
// |v| as float bits, 0 for Inf / NaN: the exact mode's scales cover the FINITE
// values; non-finite inputs are sliced as 0 and their receptive fields are
// poisoned to NaN afterwards (slice.cu poison_nonfinite_kernel), as the
// reference's fp64 einsum turns them (0 * Inf = NaN, conv.py:168-176).
__device__ __forceinline__ unsigned finite_abs_bits(float v) {
  const unsigned a = __float_as_uint(v) & 0x7fffffffu;
  return a < 0x7f800000u ? a : 0u;
}
__device__ __forceinline__ bool non_finite(float v) { return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u; }
// Power-of-two scale above amax; NaN when amax is not finite, so a sample
// holding Inf / NaN comes out NaN in the exact mode instead of as digits of garbage.
__device__ __forceinline__ float pow2_scale_for(float amax) {
  if (!(amax <= 3.4028235e38f)) return __uint_as_float(0x7fc00000u);
  if (!(amax > 0.f)) return 1.f;
  int e;
  frexpf(amax * 1.016f, &e);
  return ldexpf(1.f, e);
}
// u (|u| <= 126/128) -> ND balanced base-256 digits, most significant first;
// |u - sum_i d_i 2^(-7-8(i-1))| <= 2^(-8 ND)
template <int ND>
__device__ __forceinline__ void digits_b256(float u, int8_t (&d)[ND]) {
  int X = __float2int_rn(ldexpf(u, 8 * ND - 1));  // exact scaling, one rounding
#pragma unroll
  for (int i = ND - 1; i > 0; --i) {
    const int lo = (int)(int8_t)(X & 0xFF);
    d[i] = (int8_t)lo;
    X = (X - lo) >> 8;
  }
  d[0] = (int8_t)X;
}
// double-precision input (transformed operands are exact sums of two fp32)
template <int ND>
__device__ __forceinline__ void digits_b256_d(double u, int8_t (&d)[ND]) {
  long long X = __double2ll_rn(ldexp(u, 8 * ND - 1));
#pragma unroll
  for (int i = ND - 1; i > 0; --i) {
    const long long lo = (long long)(int8_t)(X & 0xFF);
    d[i] = (int8_t)lo;
    X = (X - lo) >> 8;
  }
  d[0] = (int8_t)X;
}
#endif

// ---- UMMA descriptors (layouts: cute/arch/mma_sm100_desc.hpp conventions) ---
enum : uint32_t { kSwizzleNone = 0, kSwizzle32B = 6 };

CL_HD uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// Instruction descriptor for dense MMA with fp32 accumulator, K-major A and B.
// fmt: 1 = BF16, 2 = TF32 (kind::f16 / kind::tf32 operand format codes).
CL_HD uint32_t instr_desc(uint32_t fmt, uint32_t M, uint32_t N) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
// kind::i8: signed A and B (format 1), s32 accumulator (c_format 2).
CL_HD uint32_t instr_desc_i8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

}  // namespace cl
