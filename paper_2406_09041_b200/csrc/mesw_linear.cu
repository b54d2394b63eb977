// K2: fused segmented multi-expert linear (sm_100a, tcgen05 + TMEM + TMA bulk copies).
//
//   y[t, j] = sum_i x[t,i] W[i,j]
//           + s_e[j] * sum_{i not in S_e} x[t,i] q_e[i,j] + sum_{i in S_e} x[t,i] half(R_e)[i,j]
//   with e = expert(t)   (Eq. 4; toylm.py:183-186)
//
// One persistent CTA per SM, warp-specialised (6 warps):
//   warp 0     producer: per unit (cg = 128 outputs, ks = 128 inputs) streams the base
//              weight tile (32 KiB, UMMA canonical layout) and each active expert's codes
//              with cp.async.bulk, and the activation rows with cp.async (16-byte chunks
//              scattered into the canonical K-major layout), into a ring of smem stages.
//   warp 1     MMA issuer (one thread): tcgen05.mma kind::f16, M=128 output channels,
//              N = tokens.  Base: A = W tile (smem descriptor), D_base in TMEM.  Delta:
//              A = dequantised codes IN TMEM, B = x rows of the expert's 16-token window,
//              D_delta in TMEM (one accumulator for all experts: windows are disjoint).
//   warps 2-5  dequant warpgroup: thread m owns output channel m; 2-bit codes -> exact
//              bf16 integers q in registers (lop3 magic-number trick) -> tcgen05.st into a
//              2-slot TMEM A ring; then the epilogue: tcgen05.ld of D_base / D_delta,
//              y = base + s_e[j]*delta + salient fp16 correction (+ residual, ReLU).
// Work split: units cg-major, CTA c owns [c*T/G, (c+1)*T/G) (stream-K); column groups cut
// by a range boundary are reduced in fixed k order by the last-arriving CTA.  Reduction
// order per (token, column) depends only on the shape, so results are bit-identical for
// any batch composition with the same padded row count.

#include <stdlib.h>

#include "mesw_common.cuh"
#include "mesw_host.h"
#include "mesw_layout.cuh"

namespace mesw {

constexpr int kDqGroups = 2;  // dequant warpgroups: group g expands k-half g of every job
constexpr int kProducerWarp = 0, kMmaWarp = 1, kDqWarp0 = 2, kEpiWarp0 = 2 + 4 * kDqGroups;
constexpr int kThreads = (kEpiWarp0 + 4) * 32;  // 14 warps
constexpr int kTmemCols = 512;
constexpr int kMaxASlots = 6;
constexpr int kAColsPerSlot = 64;
constexpr int kMaxRows = 192;  // padded token rows per launch (TMEM: 2 * rows <= 384)
constexpr int kMaxStages = 8;
constexpr int kXRowGroupBytes = 2048;  // 8 token rows x 16 k-chunks x 16 B
constexpr int kSalFast = 16;           // salient rows per column group handled from smem

// Element index of x[t][k] in the canonical activation layout (see mesw.h): per 128-wide
// k-step a [NP/8 row groups][16 k-chunks][8 rows][8 elems] tile of NP*128 bf16.
__device__ __forceinline__ size_t xc_index(int t, int k, int NP) {
  return (size_t)(k >> 7) * NP * 128 + (size_t)(t >> 3) * 1024 + ((k & 127) >> 3) * 64 + (t & 7) * 8 + (k & 7);
}

struct SegDesc {
  const uint8_t* codes;
  const float* steps;
  const int32_t* sal_off;
  const int32_t* sal_idx;
  const uint16_t* sal_rows;
  int begin, end, win0, winN;
};

struct LinearParams {
  const uint16_t* x;
  int B, NP, m, n;
  int n_cg, n_ks;
  const uint8_t* w;
  const mesw_expert_dev* table;
  int n_seg;
  int seg_begin[MESW_MAX_SEGMENTS];
  int seg_end[MESW_MAX_SEGMENTS];
  int seg_slot[MESW_MAX_SEGMENTS];
  void* y;
  int y_bf16, ldy;
  const uint16_t* residual;
  int ld_res;
  float* ws;
  int* counters;
  long long T;
  int G;
  int activation;
  // smem rings (byte offsets from the ring base): x tiles, base-weight tiles, code chunks
  int nx, xo, xbytes;
  int nw, wo;
  int nc, co, cbytes, segs_per_chunk, n_chunks;
  // tensor memory: n_acc accumulator buffers of 2*NP columns, A ring from a_col0
  int n_acc, n_aslots, a_col0;
  unsigned long long* tbuf;  // MESW_TIMING: per-CTA globaltimer stamps
  int dbg;  // perf experiments: bit0 skip dequant math, bit1 skip delta MMAs, bit2 skip tcgen05.st
};

struct Smem {
  uint64_t xfull[kMaxStages], xempty[kMaxStages];
  uint64_t wfull[kMaxStages], wempty[kMaxStages];
  uint64_t cfull[kMaxStages], cempty[kMaxStages];
  uint64_t aempty[kMaxASlots];
  uint64_t accfull[2], accempty[2];
  uint32_t tmem_base;
  int flag;
  int tok2seg[kMaxRows];
  SegDesc segs[MESW_MAX_SEGMENTS];
  float xsal[kMaxRows][16];  // x[t][salient idx r] of the current column group (k <= 16 fast path)
};

__host__ __device__ inline size_t ring_offset() { return (sizeof(Smem) + 1023) & ~size_t(1023); }

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

__device__ __forceinline__ int unit_owner(long long u, long long T, int G) {
  return (int)(((u + 1) * (long long)G - 1) / T);
}

// ---------------------------------------------------------------- epilogue
// Gather x[t][salient idx r] of column group cg for every row into smem (epilogue group,
// 128 threads, bar 1).  Runs BEFORE the accumulators are ready, so its global loads
// overlap the main loop.  Returns false if some segment has > kSalFast salient rows in
// cg (then the epilogue reads them from global memory).
__device__ __forceinline__ bool gather_salient_x(const LinearParams& p, Smem& S, int cg, int gtid) {
  bool fast = true;
  for (int q = 0; q < p.n_seg; ++q) {
    const SegDesc& sd = S.segs[q];
    if (sd.sal_off[cg + 1] - sd.sal_off[cg] > kSalFast) fast = false;
  }
  if (fast && p.n_seg > 0) {
    const int total = p.B * kSalFast;
    for (int i0 = gtid; i0 < total; i0 += 128 * 4) {
      float v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // issue the loads first (memory-level parallelism)
        const int i = i0 + 128 * k;
        v[k] = 0.f;
        if (i < total) {
          const int t = i / kSalFast, r = i % kSalFast;
          const int sg = S.tok2seg[t];
          if (sg >= 0) {
            const SegDesc& sd = S.segs[sg];
            const int r0 = sd.sal_off[cg];
            if (r < sd.sal_off[cg + 1] - r0) v[k] = bf16_to_f32(p.x[xc_index(t, sd.sal_idx[r0 + r], p.NP)]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + 128 * k;
        if (i < total) S.xsal[i / kSalFast][i % kSalFast] = v[k];
      }
    }
  }
  named_bar_sync(1, 128);
  return fast;
}

// Per-chunk epilogue operands that do not depend on the accumulators (prefetched one
// chunk ahead): the chunk's expert segment, its step s_e[j], salient rows R_e[r][j] and
// the residual.  A 16-row chunk holds rows of at most one segment (16-row aligned).
struct EpiPre {
  int sg;
  float sj;
  float R[kSalFast];
  float res[16];
};

__device__ __forceinline__ void epi_prefetch(const LinearParams& p, const Smem& S, int cg, int m, int t0,
                                             bool fast, EpiPre& e) {
  const int j = cg * kUnitN + m;
  e.sg = -1;
#pragma unroll
  for (int t = 0; t < 16; ++t)
    if (e.sg < 0 && t0 + t < p.B) e.sg = S.tok2seg[t0 + t];
  e.sj = 0.f;
#pragma unroll
  for (int r = 0; r < kSalFast; ++r) e.R[r] = 0.f;
  if (e.sg >= 0 && j < p.n) {
    const SegDesc& sd = S.segs[e.sg];
    e.sj = sd.steps[j];
    if (fast) {
      const int r0 = sd.sal_off[cg], k = sd.sal_off[cg + 1] - r0;
#pragma unroll
      for (int r = 0; r < kSalFast; ++r)
        if (r < k) e.R[r] = __half2float(__ushort_as_half(sd.sal_rows[(size_t)(r0 + r) * kUnitN + m]));
    }
  }
#pragma unroll
  for (int t = 0; t < 16; ++t)
    e.res[t] = (p.residual && t0 + t < p.B && j < p.n) ? bf16_to_f32(p.residual[(size_t)(t0 + t) * p.ld_res + j]) : 0.f;
}

// Thread owns output channel j = cg*128 + m; accumulators for the 16 rows [t0, t0+16).
__device__ __forceinline__ void epi_store16(const LinearParams& p, const Smem& S, int cg, int m, int t0,
                                            const float* vb, const float* vd, bool fast, const EpiPre& e) {
  const int j = cg * kUnitN + m;
  if (j >= p.n) return;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int tok = t0 + t;
    if (tok >= p.B) break;
    float v = vb[t];
    if (e.sg >= 0 && S.tok2seg[tok] == e.sg) {
      float d = e.sj * vd[t];
      if (fast) {
#pragma unroll
        for (int r = 0; r < kSalFast; ++r) d = fmaf(S.xsal[tok][r], e.R[r], d);
      } else {
        const SegDesc& sd = S.segs[e.sg];
        const int r0 = sd.sal_off[cg], k = sd.sal_off[cg + 1] - r0;
        for (int r = 0; r < k; ++r) {
          const float xv = bf16_to_f32(p.x[xc_index(tok, sd.sal_idx[r0 + r], p.NP)]);
          const float rv = __half2float(__ushort_as_half(sd.sal_rows[(size_t)(r0 + r) * kUnitN + m]));
          d = fmaf(xv, rv, d);
        }
      }
      v += d;
    }
    v += e.res[t];
    if (p.activation == 1) v = fmaxf(v, 0.f);
    if (p.y_bf16)
      reinterpret_cast<__nv_bfloat16*>(p.y)[(size_t)tok * p.ldy + j] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float*>(p.y)[(size_t)tok * p.ldy + j] = v;
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MESW_STAMP(i) \
  do { if (p.tbuf) p.tbuf[(size_t)blockIdx.x * 8 + (i)] = gtimer(); } while (0)

// ---------------------------------------------------------------- kernel
template <int DB>
__global__ void __launch_bounds__(kThreads, 1) me_linear_tc_kernel(const __grid_constant__ LinearParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Smem& S = *reinterpret_cast<Smem*>(smem);
  uint8_t* ring = smem + ring_offset();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const long long u0 = (long long)c * p.T / p.G, u1 = (long long)(c + 1) * p.T / p.G;
  constexpr int CB = kUnitN * kUnitK * DB / 8;  // code bytes per unit per expert
  constexpr int CHB = 8 * DB;                   // code bytes per (k-half, channel)
  const int NP = p.NP;

  const int n_issuers = 1 + (p.n_seg > 0 ? kDqGroups : 0);  // MMA warp + dequant groups
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.nx; ++i) { mbar_init(&S.xfull[i], 1); mbar_init(&S.xempty[i], n_issuers); }
    for (int i = 0; i < p.nw; ++i) { mbar_init(&S.wfull[i], 1); mbar_init(&S.wempty[i], 1); }
    for (int i = 0; i < p.nc; ++i) { mbar_init(&S.cfull[i], 1); mbar_init(&S.cempty[i], 128 * kDqGroups); }
    for (int i = 0; i < p.n_aslots; ++i) mbar_init(&S.aempty[i], 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&S.accfull[i], n_issuers); mbar_init(&S.accempty[i], 4); }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < kMaxRows; i += kThreads) S.tok2seg[i] = -1;
  __syncthreads();
  for (int q = threadIdx.x; q < p.n_seg; q += kThreads) {
    const mesw_expert_dev e = p.table[p.seg_slot[q]];
    SegDesc d;
    d.codes = reinterpret_cast<const uint8_t*>(e.codes);
    d.steps = e.steps;
    d.sal_off = e.sal_off;
    d.sal_idx = e.sal_idx;
    d.sal_rows = e.sal_rows;
    d.begin = p.seg_begin[q];
    d.end = p.seg_end[q];
    d.win0 = d.begin;                          // begin is a multiple of 16
    d.winN = ((d.end + 15) & ~15) - d.begin;   // 16-token window(s)
    S.segs[q] = d;
    for (int t = d.begin; t < d.end; ++t) S.tok2seg[t] = q;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  const bool has_w = p.w != nullptr;
  if (threadIdx.x == 0) MESW_STAMP(0);

  if (warp == kProducerWarp) {
    // ===================== producer: x tiles, weight tiles, code chunks =====================
    int sx = 0, sw = 0, sc = 0;
    uint32_t px = 0, pw = 0, pc = 0;
    bool fx = true, fw = true, fc = true;
    int ks = (int)(u0 % p.n_ks);
    for (long long u = u0; u < u1; ++u) {
      if (lane == 0) {
        if (!fx) mbar_wait(&S.xempty[sx], px ^ 1);
        mbar_arrive_expect_tx(&S.xfull[sx], (uint32_t)p.xbytes);
        bulk_g2s(ring + p.xo + (size_t)sx * p.xbytes, p.x + (size_t)ks * NP * kUnitK, p.xbytes, &S.xfull[sx]);
        if (++sx == p.nx) { sx = 0; px ^= 1; fx = false; }
        if (has_w) {
          if (!fw) mbar_wait(&S.wempty[sw], pw ^ 1);
          mbar_arrive_expect_tx(&S.wfull[sw], kUnitWBytes);
          bulk_g2s(ring + p.wo + (size_t)sw * kUnitWBytes, p.w + (size_t)u * kUnitWBytes, kUnitWBytes, &S.wfull[sw]);
          if (++sw == p.nw) { sw = 0; pw ^= 1; fw = false; }
        }
      }
      for (int ch = 0; ch < p.n_chunks; ++ch) {
        const int sg0 = ch * p.segs_per_chunk;
        const int sg1 = min(p.n_seg, sg0 + p.segs_per_chunk);
        if (lane == 0) {
          if (!fc) mbar_wait(&S.cempty[sc], pc ^ 1);
          mbar_arrive_expect_tx(&S.cfull[sc], (uint32_t)(sg1 - sg0) * CB);
        }
        __syncwarp();
        for (int q = sg0 + lane; q < sg1; q += 32)
          bulk_g2s(ring + p.co + (size_t)sc * p.cbytes + (size_t)(q - sg0) * CB, S.segs[q].codes + (size_t)u * CB,
                   CB, &S.cfull[sc]);
        __syncwarp();
        if (++sc == p.nc) { sc = 0; pc ^= 1; fc = false; }
      }
      if (++ks == p.n_ks) ks = 0;
    }
    if (lane == 0) MESW_STAMP(1);
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (one thread) =====================
    // The tensor pipe accepts one tcgen05.mma per ~45 cycles at these shapes, so the
    // issue loop is kept minimal: all smem descriptors are precomputed and advanced by
    // plain 64-bit adds (start address field += bytes/16), the k-loop is unrolled.
    if (lane == 0) {
      const uint64_t xdesc0 = smem_desc(smem_u32(ring + p.xo));
      const uint64_t wdesc0 = smem_desc(smem_u32(ring + p.wo));
      const uint32_t xstride = (uint32_t)p.xbytes >> 4, wstride = kUnitWBytes >> 4;
      const uint32_t id_base = idesc_bf16(NP);
      int sx = 0, sw = 0;
      uint32_t px = 0, pw = 0;
      int ab = 0;                 // accumulator buffer of the current piece
      int use0 = 0, use1 = 0;     // pieces already accumulated in buffers 0 / 1
      int ks = (int)(u0 % p.n_ks);
      for (long long u = u0; u < u1; ++u) {
        const bool piece_first = (u == u0 || ks == 0);
        const bool piece_last = (ks == p.n_ks - 1 || u == u1 - 1);
        const int use = ab ? use1 : use0;
        if (piece_first && use > 0) {
          mbar_wait(&S.accempty[ab], (uint32_t)((use - 1) & 1));  // epilogue drained it
          tc_fence_after();
        }
        const uint32_t d_base = tbase + (uint32_t)(ab * 2 * NP);
        const uint32_t f0 = piece_first ? 0u : 1u;  // accumulate flag of the first k-block
        mbar_wait(&S.xfull[sx], px);
        const uint64_t xd = xdesc0 + (uint64_t)(sx * xstride);
        if (has_w) {
          mbar_wait(&S.wfull[sw], pw);
          tc_fence_after();
          const uint64_t wd = wdesc0 + (uint64_t)(sw * wstride);
          mma_ss(d_base, wd, xd, id_base, f0);
#pragma unroll
          for (int j = 1; j < 8; ++j) mma_ss(d_base, wd + 16 * j, xd + 16 * j, id_base, 1u);
          tc_commit(&S.wempty[sw]);  // weight tile free once these MMAs complete
          if (++sw == p.nw) { sw = 0; pw ^= 1; }
        }
        tc_commit(&S.xempty[sx]);
        if (++sx == p.nx) { sx = 0; px ^= 1; }
        if (piece_last) {
          tc_commit(&S.accfull[ab]);
          if (ab) ++use1; else ++use0;
          if (p.n_acc == 2) ab ^= 1;
        }
        if (++ks == p.n_ks) ks = 0;
        if (u == u0) MESW_STAMP(2);
      }
      MESW_STAMP(3);
    }
  } else if (warp < kEpiWarp0) {
    // ===================== dequant groups: codes -> TMEM A -> delta MMAs =====================
    // Group g owns the jobs of experts q with q % 2 == g: its 128 threads (thread m =
    // output channel m) expand the job's codes for all 128 k into bf16 A rows in TMEM,
    // then one elected thread of the group issues the job's 8 tcgen05.mma (A from TMEM,
    // B = the x rows of the expert's 16-token window) and commits them.  No handshake
    // with the base-MMA warp: the groups and the MMA warp only meet at the x-tile release
    // and at the per-piece accumulator barriers.
    const int grp = (warp - kDqWarp0) >> 2;
    const int quarter = warp & 3;            // TMEM lanes [32*quarter, +32)
    const int mrow = quarter * 32 + lane;    // output channel within the column group
    const int gtid = ((warp - kDqWarp0) & 3) * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const int NAW = p.n_aslots / kDqGroups;  // A slots per group
    constexpr int WPJ = 2 * CHB / 4;         // code words per job per thread (both k-halves)
    constexpr int MJ = 32 / WPJ;             // own jobs per chunk held in registers (host agrees)
    const uint64_t xdesc0 = smem_desc(smem_u32(ring + p.xo));
    const uint32_t xstride = (uint32_t)p.xbytes >> 4;
    int sc = 0, sx = 0;
    uint32_t pc = 0, px = 0;
    long long job = 0;   // global job counter (jobs = (unit, segment) pairs)
    long long mine = 0;  // jobs handled by this group so far
    int ab = 0, use0 = 0, use1 = 0;
    int ks = (int)(u0 % p.n_ks);
    for (long long u = (p.n_seg > 0 ? u0 : u1); u < u1; ++u) {  // idle without experts
      const bool piece_first = (u == u0 || ks == 0);
      const bool piece_last = (ks == p.n_ks - 1 || u == u1 - 1);
      const uint32_t d_delta = tbase + (uint32_t)(ab * 2 * NP + NP);
      const uint32_t f0 = piece_first ? 0u : 1u;
      bool waited_acc = !(piece_first && (ab ? use1 : use0) > 0);
      bool waited_x = false;
      const uint64_t xd = xdesc0 + (uint64_t)(sx * xstride);
      for (int ch = 0; ch < p.n_chunks; ++ch) {
        const int sg0 = ch * p.segs_per_chunk;
        const int sg1 = min(p.n_seg, sg0 + p.segs_per_chunk);
        mbar_wait(&S.cfull[sc], pc);
        const uint8_t* cst = ring + p.co + (size_t)sc * p.cbytes;
        uint32_t cw[MJ][WPJ];
        int own[MJ];
        int nown = 0;
#pragma unroll
        for (int jq = 0; jq < MJ; ++jq) own[jq] = -1;
        for (int q = sg0; q < sg1; ++q) {
          if (q % kDqGroups != grp) continue;  // expert q always handled by group q % 2:
                                               // one issuing thread per accumulator window
                                               // keeps the k-order of its MMAs fixed
#pragma unroll
          for (int jq = 0; jq < MJ; ++jq)
            if (jq == nown) own[jq] = q;
          ++nown;
        }
#pragma unroll
        for (int jq = 0; jq < MJ; ++jq) {
          if (own[jq] >= 0) {
            const uint8_t* cb = cst + (size_t)(own[jq] - sg0) * CB;
#pragma unroll
            for (int kh = 0; kh < 2; ++kh)
#pragma unroll
              for (int v = 0; v < CHB / 16; ++v) {
                const uint4 t4 = lds128(cb + ((size_t)kh * 128 + mrow) * CHB + v * 16);
                const int w0 = kh * (CHB / 4) + 4 * v;
                cw[jq][w0] = t4.x; cw[jq][w0 + 1] = t4.y; cw[jq][w0 + 2] = t4.z; cw[jq][w0 + 3] = t4.w;
              }
          }
        }
        mbar_arrive(&S.cempty[sc]);  // every thread: release orders its own smem reads
        if (++sc == p.nc) { sc = 0; pc ^= 1; }
#pragma unroll
        for (int jq = 0; jq < MJ; ++jq) {
          if (own[jq] >= 0) {
            const int q = own[jq];
            const int aslot = grp * NAW + (int)(mine % NAW);
            const long long use = mine / NAW;
            if (use > 0) mbar_wait(&S.aempty[aslot], (uint32_t)((use - 1) & 1));
            const uint32_t a0 = tbase + (uint32_t)(p.a_col0 + aslot * kAColsPerSlot);
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {  // one k-half (32 columns) at a time
              uint32_t r[32];
              if (p.dbg & 1) {
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = cw[jq][i % WPJ];
              } else {
                dequant_chunk<DB>(&cw[jq][kh * (CHB / 4)], r);
              }
              if (!(p.dbg & 4)) tmem_st32(a0 + lane_addr + 32 * kh, r);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            named_bar_sync(2 + grp, 128);  // the job's A rows are all in TMEM
            if (gtid == 0) {
              if (!waited_acc) {  // previous piece in this buffer drained by the epilogue
                const int uacc = ab ? use1 : use0;
                mbar_wait(&S.accempty[ab], (uint32_t)((uacc - 1) & 1));
                waited_acc = true;
              }
              if (!waited_x) {
                mbar_wait(&S.xfull[sx], px);
                waited_x = true;
              }
              tc_fence_after();
              const SegDesc& sd = S.segs[q];
              const uint32_t id = idesc_bf16(sd.winN);
              const uint32_t dd = d_delta + (uint32_t)sd.win0;
              const uint64_t bd = xd + (uint64_t)((sd.win0 >> 3) * (kXRowGroupBytes >> 4));
              if (!(p.dbg & 2)) {
                mma_ts(dd, a0, bd, id, f0);
#pragma unroll
                for (int j = 1; j < 8; ++j) mma_ts(dd, a0 + 8 * j, bd + 16 * j, id, 1u);
              }
              tc_commit(&S.aempty[aslot]);
            }
            ++mine;
          }
        }
        job += sg1 - sg0;
      }
      if (gtid == 0) {
        if (!waited_acc) {
          const int uacc = ab ? use1 : use0;
          mbar_wait(&S.accempty[ab], (uint32_t)((uacc - 1) & 1));
        }
        if (!waited_x) mbar_wait(&S.xfull[sx], px);
        tc_commit(&S.xempty[sx]);  // this group's MMAs on the x tile are done
        if (piece_last) tc_commit(&S.accfull[ab]);
      }
      if (++sx == p.nx) { sx = 0; px ^= 1; }
      if (piece_last) {
        if (ab) ++use1; else ++use0;
        if (p.n_acc == 2) ab ^= 1;
      }
      if (++ks == p.n_ks) ks = 0;
    }
  } else {
    // ===================== epilogue warpgroup =====================
    const int quarter = warp & 3;
    const int mrow = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const int gtid = (warp - kEpiWarp0) * 32 + lane;  // 0..127
    const int cg_first = (int)(u0 / p.n_ks);
    int ab = 0;
    int acc_use[2] = {0, 0};
    long long u = u0;
    while (u < u1) {
      // the piece is the run of this CTA's units inside one column group
      const int cg = (int)(u / p.n_ks);
      const long long cg_end = (long long)(cg + 1) * p.n_ks;
      const long long piece_end = cg_end < u1 ? cg_end : u1;
      const bool whole = (u == (long long)cg * p.n_ks) && (piece_end == cg_end);
      // accumulator-independent operands first (overlaps the main loop)
      const bool fast = gather_salient_x(p, S, cg, gtid);
      EpiPre pre;
      epi_prefetch(p, S, cg, mrow, 0, fast, pre);
      mbar_wait(&S.accfull[ab], (uint32_t)(acc_use[ab] & 1));
      tc_fence_after();
      const uint32_t acc = tbase + lane_addr + (uint32_t)(ab * 2 * NP);
      if (p.dbg & 8) {
        // timing experiment: skip the epilogue
      } else if (whole) {
        for (int t0 = 0; t0 < NP; t0 += 16) {
          float vb[16], vd[16];
          if (has_w) {
            tmem_ld16(acc + (uint32_t)t0, vb);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) vb[i] = 0.f;  // delta-only: D_base never written
          }
          tmem_ld16(acc + (uint32_t)(NP + t0), vd);
          const EpiPre cur = pre;
          if (t0 + 16 < NP) epi_prefetch(p, S, cg, mrow, t0 + 16, fast, pre);
          epi_store16(p, S, cg, mrow, t0, vb, vd, fast, cur);
        }
      } else {
        const int slot = 2 * c + (cg == cg_first ? 0 : 1);
        const size_t slot_floats = (size_t)2 * NP * kUnitN;
        float* mine = p.ws + (size_t)slot * slot_floats;
        for (int t0 = 0; t0 < 2 * NP; t0 += 16) {
          float v[16];
          if (t0 < NP && !has_w) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          } else {
            tmem_ld16(acc + (uint32_t)t0, v);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcg(mine + (size_t)(t0 + i) * kUnitN + mrow, v[i]);
        }
      }
      // accumulators consumed -> the MMA warp may reuse this buffer
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.accempty[ab]);
      acc_use[ab]++;
      if (p.n_acc == 2) ab ^= 1;
      if (!whole && !(p.dbg & 8)) {
        __threadfence();
        named_bar_sync(1, 128);
        const long long first_u = (long long)cg * p.n_ks, last_u = first_u + p.n_ks - 1;
        const int c_first = unit_owner(first_u, p.T, p.G), c_last = unit_owner(last_u, p.T, p.G);
        if (gtid == 0) {
          const int prev = atomicAdd(&p.counters[cg], 1);
          S.flag = (prev == c_last - c_first) ? 1 : 0;
        }
        named_bar_sync(1, 128);
        if (S.flag) {
          __threadfence();
          const size_t slot_floats = (size_t)2 * NP * kUnitN;
          for (int t0 = 0; t0 < NP; t0 += 16) {
            float vb[16], vd[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) vb[i] = vd[i] = 0.f;
            for (int cc = c_first; cc <= c_last; ++cc) {
              const long long cu0 = (long long)cc * p.T / p.G;
              const int s2 = 2 * cc + ((int)(cu0 / p.n_ks) == cg ? 0 : 1);
              const float* src = p.ws + (size_t)s2 * slot_floats;
              float lb[16], ld[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {  // all loads of the slot in flight together
                lb[i] = __ldcg(src + (size_t)(t0 + i) * kUnitN + mrow);
                ld[i] = __ldcg(src + (size_t)(NP + t0 + i) * kUnitN + mrow);
              }
#pragma unroll
              for (int i = 0; i < 16; ++i) { vb[i] += lb[i]; vd[i] += ld[i]; }
            }
            const EpiPre cur = pre;
            if (t0 + 16 < NP) epi_prefetch(p, S, cg, mrow, t0 + 16, fast, pre);
            epi_store16(p, S, cg, mrow, t0, vb, vd, fast, cur);
          }
          if (gtid == 0) p.counters[cg] = 0;  // self-reset for the next launch
        }
      }
      named_bar_sync(1, 128);  // xsal / flag reuse by the next piece
      if (gtid == 0) MESW_STAMP(u == u0 ? 4 : 5);
      u = piece_end;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) MESW_STAMP(6);
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
  }
}

template <int DB>
int launch(const LinearParams& p, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(me_linear_tc_kernel<DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448);
    if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
    configured = true;
  }
  me_linear_tc_kernel<DB><<<p.G, kThreads, smem, stream>>>(p);
  return mesw_check_launch("me_linear");
}

}  // namespace mesw

using namespace mesw;

static int pad16(int v) { return (v + 15) & ~15; }

static unsigned long long* g_tbuf = nullptr;

// Debug: copy the last MESW_TIMING launch's per-CTA globaltimer stamps (8 per CTA).
extern "C" int mesw_debug_timing_copy(unsigned long long* h_out, int n_ctas) {
  if (!g_tbuf) return mesw_fail(MESW_ERR_VALUE, "no timing buffer (set MESW_TIMING)");
  cudaError_t e = cudaMemcpy(h_out, g_tbuf, (size_t)n_ctas * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? MESW_OK : mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" uint64_t mesw_linear_workspace_bytes(int32_t B, int32_t num_ctas) {
  const int np = pad16(B < 1 ? 1 : B);
  return (uint64_t)num_ctas * 2ull * 2ull * np * kUnitN * sizeof(float);
}

extern "C" int mesw_me_linear(const mesw_linear_args* a, void* stream) {
  if (!a) return mesw_fail(MESW_ERR_VALUE, "null args");
  if (a->B < 1 || a->B > kMaxRows)
    return mesw_fail(MESW_ERR_UNSUPPORTED, "fused linear supports 1 <= rows <= 192 per launch");
  if (a->m < 1 || a->n < 1) return mesw_fail(MESW_ERR_VALUE, "empty linear");
  const int m_pad = (a->m + kUnitK - 1) / kUnitK * kUnitK;
  const int n_pad = (a->n + kUnitN - 1) / kUnitN * kUnitN;
  if (a->x_layout != 0) return mesw_fail(MESW_ERR_VALUE, "x must be in the canonical tile layout (x_layout 0)");
  if (((uintptr_t)a->x) % 16 || ((uintptr_t)a->w) % 16) return mesw_fail(MESW_ERR_VALUE, "x / w must be 16-byte aligned");
  if (a->n_segments < 0 || a->n_segments > MESW_MAX_SEGMENTS) return mesw_fail(MESW_ERR_VALUE, "too many segments");
  if (a->n_segments > 0 && a->code_bits != 2 && a->code_bits != 4 && a->code_bits != 8)
    return mesw_fail(MESW_ERR_VALUE, "code_bits must be 2, 4 or 8");
  if (!a->w && a->n_segments == 0) return mesw_fail(MESW_ERR_VALUE, "nothing to compute (no base, no delta)");
  if (!a->y) return mesw_fail(MESW_ERR_VALUE, "null output");
  if (a->n_segments > 0 && !a->expert_table) return mesw_fail(MESW_ERR_VALUE, "null expert table");
  int prev_end = 0;
  for (int s = 0; s < a->n_segments; ++s) {
    if (a->seg_begin[s] < prev_end || a->seg_end[s] <= a->seg_begin[s] || a->seg_end[s] > a->B ||
        a->seg_slot[s] < 0)
      return mesw_fail(MESW_ERR_VALUE, "segments must be non-empty, ascending, disjoint and inside [0, B)");
    if (a->seg_begin[s] % 16)
      return mesw_fail(MESW_ERR_VALUE, "segment begins must be multiples of 16 rows (pad expert groups)");
    prev_end = a->seg_end[s];
  }
  int sms = mesw_device_sm_count();
  if (sms <= 0) return mesw_fail(MESW_ERR_CUDA, "no CUDA device");

  LinearParams p{};
  p.x = a->x; p.B = a->B; p.NP = pad16(a->B); p.m = a->m; p.n = a->n;
  p.n_cg = n_pad / kUnitN; p.n_ks = m_pad / kUnitK;
  p.w = reinterpret_cast<const uint8_t*>(a->w);
  p.table = a->expert_table;
  p.n_seg = a->n_segments;
  for (int s = 0; s < p.n_seg; ++s) {
    p.seg_begin[s] = a->seg_begin[s]; p.seg_end[s] = a->seg_end[s]; p.seg_slot[s] = a->seg_slot[s];
  }
  p.y = a->y; p.y_bf16 = a->y_bf16; p.ldy = a->ldy;
  p.residual = a->residual; p.ld_res = a->ld_res;
  p.ws = reinterpret_cast<float*>(a->workspace);
  p.counters = a->counters;
  p.T = (long long)p.n_cg * p.n_ks;
  p.activation = a->activation;
  {
    const char* e = getenv("MESW_DBG");
    p.dbg = e ? atoi(e) : 0;
    if (getenv("MESW_TIMING")) {
      if (!g_tbuf) cudaMalloc(&g_tbuf, 8 * 4096 * sizeof(unsigned long long));
      p.tbuf = g_tbuf;
    }
  }
  const int want = a->num_ctas > 0 ? a->num_ctas : sms;
  p.G = (int)((long long)want < p.T ? want : p.T);
  if (a->workspace_bytes < mesw_linear_workspace_bytes(a->B, p.G) || !a->workspace || !a->counters)
    return mesw_fail(MESW_ERR_VALUE, "workspace too small");

  // Shared-memory rings: x tiles (NP rows x 256 B), weight tiles (32 KiB), code chunks
  const int db = a->n_segments > 0 ? a->code_bits : 2;
  const int CB = kUnitN * kUnitK * db / 8;
  const int max_chunk = (db == 2 ? 4 : (db == 4 ? 2 : 1)) * kDqGroups;  // jobs per code chunk
  p.segs_per_chunk = p.n_seg == 0 ? 1 : (p.n_seg < max_chunk ? p.n_seg : max_chunk);
  p.n_chunks = p.n_seg == 0 ? 0 : (p.n_seg + p.segs_per_chunk - 1) / p.segs_per_chunk;
  p.xbytes = p.NP * kUnitK * 2;
  p.cbytes = p.segs_per_chunk * CB;
  const size_t budget = 232448 - ring_offset();
  // ring depths: prefer (x 3, codes 3, weights >= 3); shrink x/codes first when rows are many
  p.nx = 3;
  p.nc = p.n_chunks > 0 ? 3 : 0;
  for (;;) {
    const size_t used = (size_t)p.nx * p.xbytes + (size_t)p.nc * p.cbytes + 1024;
    p.nw = a->w ? (int)((budget > used ? budget - used : 0) / kUnitWBytes) : 0;
    if (p.nw > kMaxStages) p.nw = kMaxStages;
    if (!a->w || p.nw >= 3) break;
    if (p.nx > 2) { --p.nx; continue; }
    if (p.nc > 2) { --p.nc; continue; }
    if (p.nw >= 2) break;
    if (p.segs_per_chunk > kDqGroups) {  // smaller code chunks
      p.segs_per_chunk = (p.segs_per_chunk / 2 + kDqGroups - 1) / kDqGroups * kDqGroups;
      p.n_chunks = (p.n_seg + p.segs_per_chunk - 1) / p.segs_per_chunk;
      p.cbytes = p.segs_per_chunk * CB;
      continue;
    }
    return mesw_fail(MESW_ERR_UNSUPPORTED, "shared memory: fewer than 2 weight stages");
  }
  p.xo = 0;
  p.co = p.nx * p.xbytes;
  p.wo = (p.co + p.nc * p.cbytes + 1023) & ~1023;
  const size_t smem = ring_offset() + (size_t)p.wo + (size_t)p.nw * kUnitWBytes;
  if (smem > 232448) return mesw_fail(MESW_ERR_UNSUPPORTED, "shared memory overflow");
  // TMEM: n_acc buffers of [D_base NP | D_delta NP] columns, then the A ring (64-col slots)
  p.n_acc = (4 * p.NP + 2 * kAColsPerSlot <= kTmemCols) ? 2 : 1;
  int na = (kTmemCols - p.n_acc * 2 * p.NP) / kAColsPerSlot;
  if (na > kMaxASlots) na = kMaxASlots;
  na -= na % kDqGroups;
  if (na < kDqGroups) return mesw_fail(MESW_ERR_UNSUPPORTED, "tensor memory: too many rows for the A ring");
  p.n_aslots = na;
  p.a_col0 = kTmemCols - na * kAColsPerSlot;

  cudaStream_t s = (cudaStream_t)stream;
  switch (db) {
    case 2: return launch<2>(p, smem, s);
    case 4: return launch<4>(p, smem, s);
    default: return launch<8>(p, smem, s);
  }
}
