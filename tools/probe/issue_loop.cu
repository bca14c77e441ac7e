// SASS probe (compile only: nvcc -cubin, then cuobjdump -sass): code shape of
// the MMA warp's per-stage loop for the bf16 halo path under three issue
// styles. VARIANT 1: elect block around the MMA asm; 2: warp-converged with a
// per-lane guard predicate; 3: elect.sync inside the asm.
#include <cstdint>
#include "../../paper_2507_01040_b200/csrc/common.cuh"
using namespace cl;

#ifndef VARIANT
#define VARIANT 1
#endif

template <int KS>
__device__ __forceinline__ void mma_ks_elect(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                             uint32_t b_hi, uint32_t idesc, uint32_t acc0, uint32_t a_step,
                                             uint32_t b_step) {
  // KS bf16 MMAs (cta_group::2), 32-bit descriptor low halves advanced in-asm
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 al, bl;\n\t.reg .b64 da, db;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b32 al, %1;\n\tmov.b32 bl, %3;\n\t"
      "mov.b64 da, {al, %2};\n\tmov.b64 db, {bl, %4};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t"
      "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\t"
      "mov.b64 da, {al, %2};\n\tmov.b64 db, {bl, %4};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t"
      "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\t"
      "mov.b64 da, {al, %2};\n\tmov.b64 db, {bl, %4};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t"
      "add.u32 al, al, %7;\n\tadd.u32 bl, bl, %8;\n\t"
      "mov.b64 da, {al, %2};\n\tmov.b64 db, {bl, %4};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, 1;\n\t"
      "}" ::"r"(d_tmem),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc0), "r"(a_step), "r"(b_step)
      : "memory");
}

__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

struct P {
  int nQ, S, df, hx, hy;
  uint32_t stage_bytes, a_kstep, b_ks, h_tmpl_lo, h_tmpl_hi, b_tmpl_lo, b_tmpl_hi, idesc;
};

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ P p, int tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 200000);
  uint64_t* empty = full + 8;
  uint64_t* tfull = empty + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 4);
  if (threadIdx.x >= 32) return;
  const uint32_t tmem = *tslot;
  const uint32_t issuer = elect_one();
  const uint32_t h_base = p.h_tmpl_lo + ((smem_u32(smem) & 0x3FFFFu) >> 4);
  const uint32_t b_base = p.b_tmpl_lo + ((smem_u32(smem + 65536) & 0x3FFFFu) >> 4);
  const uint32_t stg4 = p.stage_bytes >> 4;
  const uint32_t h_dx = 2, h_wrap_x = (uint32_t)((p.hx - p.df) * 2), h_wrap_y = (uint32_t)((p.hy - p.df) * p.hx * 2);
  int stage = 0;
  uint32_t phase = 0;
  for (int t = 0;; ++t) {
#ifdef SCHED
    long long c = *reinterpret_cast<volatile long long*>(smem + 8 * (t & 7));
#if SCHED == 2
    c = __shfl_sync(0xffffffffu, c, 0);
#endif
    if (c < 0) break;
#else
    if (t >= tiles) break;
#endif
    uint32_t tap4 = 0, accf = 0;
    int qx = 0, qy = 0;
    const uint32_t d = tmem + (uint32_t)(t & 1) * 128u;
    for (int q = 0; q < p.nQ; ++q) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      const uint32_t a0 = h_base + tap4, b0 = b_base + (uint32_t)stage * stg4;
#if VARIANT == 1
      if (elect_one()) {
        switch (p.nQ & 3) { case 0: mma_bf16_cg2_ks<4>(1u, d, a0, p.h_tmpl_hi, b0, p.b_tmpl_hi, p.idesc, accf, p.a_kstep, p.b_ks); break; case 1: mma_bf16_cg2_ks<2>(1u, d, a0, p.h_tmpl_hi, b0, p.b_tmpl_hi, p.idesc, accf, p.a_kstep, p.b_ks); break; default: mma_bf16_cg2_ks<8>(1u, d, a0, p.h_tmpl_hi, b0, p.b_tmpl_hi, p.idesc, accf, p.a_kstep, p.b_ks); }
        mma_commit_cg2(&empty[stage]);
        if (q == p.nQ - 1) mma_commit_cg2(&tfull[t & 1]);
      }
      __syncwarp();
#elif VARIANT == 2
      mma_bf16_cg2_ks<4>(issuer, d, a0, p.h_tmpl_hi, b0, p.b_tmpl_hi, p.idesc, accf, p.a_kstep, p.b_ks);
      mma_commit_cg2_g(issuer, &empty[stage]);
      if (q == p.nQ - 1) mma_commit_cg2_g(issuer, &tfull[t & 1]);
#else
      mma_ks_elect<4>(d, a0, p.h_tmpl_hi, b0, p.b_tmpl_hi, p.idesc, accf, p.a_kstep, p.b_ks);
      commit_elect(&empty[stage]);
      if (q == p.nQ - 1) commit_elect(&tfull[t & 1]);
#endif
      accf = 1;
      if (++stage == p.S) { stage = 0; phase ^= 1; }
      tap4 += h_dx;
      if (++qx == p.df) {
        qx = 0;
        tap4 += h_wrap_x;
        if (++qy == p.df) { qy = 0; tap4 += h_wrap_y; }
      }
    }
  }
  (void)issuer;
}
