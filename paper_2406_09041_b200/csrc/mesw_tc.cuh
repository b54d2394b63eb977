// tcgen05 / TMEM / mbarrier-cluster helpers and the 2-bit code expansion shared by the
// decode kernel (K2, mesw_linear.cu) and the prefill kernel (K3, mesw_prefill.cu).
#pragma once

#include "mesw_common.cuh"
#include "mesw_layout.cuh"

namespace mesw {

constexpr int kXRowGroupBytes = 2048;  // 8 token rows x 16 k-chunks x 16 B (one canonical 8-row group)

// Element index of x[t][k] in the canonical activation layout (see mesw.h): per 128-wide
// k-step, two halves h = (t/8)%2 (rows 0-7 / 8-15 of every 16-row window), each a
// [NP/16 windows][16 k-chunks][8 rows][8 elems] UMMA K-major tile -- the B-operand split
// of a cta_group::2 MMA (CTA h of the pair holds half h).
__device__ __forceinline__ size_t xc_index(int t, int k, int NP) {
  return (size_t)(k >> 7) * NP * 128 + (size_t)((t >> 3) & 1) * (NP / 2) * 128 + (size_t)(t >> 4) * 1024 +
         ((k & 127) >> 3) * 64 + (t & 7) * 8 + (k & 7);
}

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  // K-major, SWIZZLE_NONE canonical: LBO = 128 B (k-chunk stride), SBO = 2048 B (8-row group stride)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) |
         (1ull << 46);
}

__device__ __forceinline__ uint32_t idesc_bf16(int N) {
  // D f32, A/B bf16, both K-major, M = 128
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ uint32_t idesc_bf16_m256(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// cta_group::2 (M = 256 over a CTA pair) variants; only the leader CTA issues.
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// Whole-warp issue (all 32 lanes run the issuer loop with warp-uniform operands; one elected
// lane executes the tcgen05 op).  Issuing from a single divergent lane makes the compiler
// move every operand to uniform registers through an R2UR.BROADCAST loop per instruction,
// which doubles the issue cost (tools/micro/tc2_rate.cu: 730 -> 341 cycles per 8 MMAs).
__device__ __forceinline__ void mma2_ss_w(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma2_ts_w(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// One whole k-step (K = 128 = 8 x 16) of a cta_group::2 MMA chain in ONE asm block with one
// elect: the descriptor / TMEM-address increments are immediates inside the block, so ptxas
// keeps them in the uniform datapath (no per-instruction R2UR.BROADCAST round trip, which
// made every tcgen05.mma cost ~40 cycles of issue).  Callers pass warp-uniform operands
// (uni()): then the operands themselves need no broadcast either.
__device__ __forceinline__ uint32_t uni(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }
__device__ __forceinline__ uint64_t uni64(uint64_t v) {
  return ((uint64_t)uni((uint32_t)(v >> 32)) << 32) | uni((uint32_t)v);
}
#define MESW_SS_STEP(J)                                                   \
  "add.s64 ad, %1, " #J "*16;\nadd.s64 bd, %2, " #J "*16;\n"              \
  "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %3, 1;\n"
__device__ __forceinline__ void mma2_ss_k128(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b64 ad, bd;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      MESW_SS_STEP(1) MESW_SS_STEP(2) MESW_SS_STEP(3) MESW_SS_STEP(4) MESW_SS_STEP(5) MESW_SS_STEP(6)
      MESW_SS_STEP(7) "}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
#undef MESW_SS_STEP
#define MESW_TS_STEP(J)                                                   \
  "add.u32 at, %1, " #J "*8;\nadd.s64 bd, %2, " #J "*16;\n"               \
  "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [at], bd, %3, 1;\n"
__device__ __forceinline__ void mma2_ts_k128(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 at;\n.reg .b64 bd;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      MESW_TS_STEP(1) MESW_TS_STEP(2) MESW_TS_STEP(3) MESW_TS_STEP(4) MESW_TS_STEP(5) MESW_TS_STEP(6)
      MESW_TS_STEP(7) "}\n" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma2_ts_k64(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 at;\n.reg .b64 bd;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      MESW_TS_STEP(1) MESW_TS_STEP(2) MESW_TS_STEP(3) "}\n" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
#undef MESW_TS_STEP

__device__ __forceinline__ void tc2_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// Commit the issuing thread's MMAs to the same-offset mbarrier in both CTAs of the pair.
__device__ __forceinline__ void tc2_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* ptr, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(ptr), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mbarrier arrive on the same-offset barrier of CTA `rank` in the cluster (release.cluster).
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// Relaxed variant for "data already complete" signals (TMA complete_tx observed, or
// tcgen05.wait::st retired): orders nothing itself, avoids the cluster-scope release fence.
__device__ __forceinline__ void mbar_arrive_cta_relaxed(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// Wait with cluster-scope acquire (barriers that receive arrivals from the peer CTA).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}

__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#define MESW_R8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])
__device__ __forceinline__ void tmem_st64(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {"
      "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,"
      "%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,"
      "%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(taddr),
      MESW_R8(0), MESW_R8(8), MESW_R8(16), MESW_R8(24), MESW_R8(32), MESW_R8(40), MESW_R8(48), MESW_R8(56)
      : "memory");
}
#undef MESW_R8

#define MESW_R8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {"
      "%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      MESW_R8(0), MESW_R8(8), MESW_R8(16), MESW_R8(24)
      : "memory");
}
#undef MESW_R8

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 consecutive columns of this warp's 32 lanes (no wait: call tmem_ld_wait() before use)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- dequant
// 8*DB code bytes of one (kh, channel) chunk -> 32 bf16x2 registers (K pairs 0..31).
template <int DB>
__device__ __forceinline__ void dequant_chunk(const uint32_t* cw, uint32_t* r);

template <>
__device__ __forceinline__ void dequant_chunk<2>(const uint32_t* cw, uint32_t* r) {
  // word w: pair 8w+l, lo code at bit 2l, hi at 16+2l.  (mask | 0x4300) is the bf16
  // 128 + u*2^pos; one bf16x2 fma rescales and subtracts 128*2^-pos + Q_N (exact).
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t a = cw[w], b = a >> 6, c = a >> 12;
    uint32_t* o = r + 8 * w;
    o[0] = bf16x2_fma(lop3_and_or(a, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
    o[1] = bf16x2_fma(lop3_and_or(a, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);
    o[2] = bf16x2_fma(lop3_and_or(a, 0x00300030u, 0x43004300u), 0x3D803D80u, 0xC120C120u);
    o[3] = bf16x2_fma(lop3_and_or(b, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
    o[4] = bf16x2_fma(lop3_and_or(b, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);
    o[5] = bf16x2_fma(lop3_and_or(b, 0x00300030u, 0x43004300u), 0x3D803D80u, 0xC120C120u);
    o[6] = bf16x2_fma(lop3_and_or(c, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
    o[7] = bf16x2_fma(lop3_and_or(c, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);
  }
}

// 2-bit codes in offset form, one lop3 per bf16x2 word: the magic exponent is chosen per
// bit position so the result is the exact bf16 value c_l + u (c_l = 128, 32, 8 for code bits
// 0-1, 2-3, 4-5 of the mantissa) -- no rescaling fma.  The MMA accumulates
// sum_k (c_k + u_k) x_k = sum_k q_k x_k + sum_k (c_k + 2) x_k; the second term comes per
// (token, k-step) from the table the activation's producer wrote (mesw.h x_corr) and is
// subtracted in f32 in the epilogue.
__device__ __forceinline__ void dequant_chunk2_offset(const uint32_t* cw, uint32_t* r) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t a = cw[w], b = a >> 6, c = a >> 12;
    uint32_t* o = r + 8 * w;
    o[0] = lop3_and_or(a, 0x00030003u, 0x43004300u);
    o[1] = lop3_and_or(a, 0x000C000Cu, 0x42004200u);
    o[2] = lop3_and_or(a, 0x00300030u, 0x41004100u);
    o[3] = lop3_and_or(b, 0x00030003u, 0x43004300u);
    o[4] = lop3_and_or(b, 0x000C000Cu, 0x42004200u);
    o[5] = lop3_and_or(b, 0x00300030u, 0x41004100u);
    o[6] = lop3_and_or(c, 0x00030003u, 0x43004300u);
    o[7] = lop3_and_or(c, 0x000C000Cu, 0x42004200u);
  }
}

template <>
__device__ __forceinline__ void dequant_chunk<4>(const uint32_t* cw, uint32_t* r) {
  // word w: pair 4w+l, nibbles at bits 4l / 16+4l; d = q + 8 -> (128 + d) - 136
#pragma unroll
  for (int w = 0; w < 8; ++w)
#pragma unroll
    for (int l = 0; l < 4; ++l)
      r[4 * w + l] = bf16x2_fma(lop3_and_or(cw[w] >> (4 * l), 0x000F000Fu, 0x43004300u), 0x3F803F80u, 0xC308C308u);
}

template <>
__device__ __forceinline__ void dequant_chunk<8>(const uint32_t* cw, uint32_t* r) {
  // word w: pair 2w+l, bytes l / 2+l; d = q + 128
#pragma unroll
  for (int w = 0; w < 16; ++w)
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const float lo = __uint_as_float(0x4B000000u | ((cw[w] >> (8 * l)) & 0xFFu)) - 8388736.0f;
      const float hi = __uint_as_float(0x4B000000u | ((cw[w] >> (16 + 8 * l)) & 0xFFu)) - 8388736.0f;
      uint32_t d;
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
      r[2 * w + l] = d;
    }
}


}  // namespace mesw
