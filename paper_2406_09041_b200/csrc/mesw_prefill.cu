// K3: prefill / large-token-batch fused multi-expert linear (sm_100a: tcgen05 + TMEM,
// cta_group::2 CTA pairs, bulk-copy staging).
//
//   y[t, :] = x[t, :] . bf16(W + Dtilde_e)  (+ residual[t, :]),   e = expert of t's 128-token group
//   (Eq. 4: x.W + x.Dtilde_e; Dtilde = reconstruct(),
//    compress.py:115-121)
//
// At prefill every expert group holds >= 128 tokens, so the contraction is tensor-bound and
// the decode kernel's design point (a separate delta MMA chain on each expert's tokens) would
// double the tensor FLOPs.  Here the delta is folded into the A operand instead: per unit
// (128 output channels x 128 inputs) the merge warps read the bf16 base tile and the expert's
// 2-bit codes and form A = RN_bf16(W + s_j * q_ij) with one bf16x2 fma per input pair (q is an
// exact small integer, s_j rounded to bf16; salient inputs i in S_e get RN_bf16(W_ij +
// half(R_i)_j)), store A to TMEM, and the tensor pipe runs a single bf16 MMA chain per
// expert group -- the same FLOPs as the dense base GEMM.  The one extra rounding of W + Dtilde
// (|err| <= 2^-9 |W + Dtilde| per weight, the precision a bf16 fine-tuned weight would have)
// keeps layer outputs well inside the north-star tolerance (tests/test_gpu_prefill.py).
//
// Work: tiles (column-group pair, 256-token tile = two 128-token expert groups), persistent
// CTA pairs walk tiles cg-pair-major so the pairs running at the same time share W tiles in L2.
// Roles per CTA (24 warps at the default MESW_PF_GROUPS = 4):
//   warps 0, 2  producers (one thread each): W unit (32 KiB) + the two groups' code units
//               (4 KiB each); this CTA's half of the x tile (32 KiB: 2 groups x 8 windows x 2 KiB).
//   warp 1      leader: MMA issuer (M = 256 over the pair, N = 128 per group, K = 16);
//               peer: relays "x half landed" to the leader's barrier.
//   warps 4-19  four merge groups: group g owns k-slice g (32 inputs) of every unit, thread =
//               output row; LDS of W + codes, bf16x2 fma merge, tcgen05.st into the A slot.
//   warps 20-23 epilogue: tcgen05.ld of the 2 x 128-column accumulators, y stores; each
//               128-token group's accumulator is released as soon as it is drained.
// TMEM: accumulators [group 0 | group 1] x 128 columns, then 4 A slots of 64 columns.

#include <stdlib.h>

#include <algorithm>

#include "mesw_common.cuh"
#include "mesw_host.h"
#include "mesw_layout.cuh"
#include "mesw_tc.cuh"

namespace mesw {
namespace prefill {

#ifndef MESW_PF_GROUPS
#define MESW_PF_GROUPS 4
#endif
constexpr int kMergeGroups = MESW_PF_GROUPS;        // merge groups: group g owns k-slice g of every unit
constexpr int kSliceK = kUnitK / kMergeGroups;      // inputs per slice (32 at 4 groups)
constexpr int kSliceW = kSliceK / 2;                // bf16x2 words per slice (16)
constexpr int kMergeWarp0 = 4, kEpiWarp0 = kMergeWarp0 + 4 * kMergeGroups;
constexpr int kThreads = (kEpiWarp0 + 4) * 32;
constexpr int kTileTok = 256;      // tokens per tile (two 128-token groups)
constexpr int kGroupTok = 128;
constexpr int kASlots = 4;
constexpr int kACols = 64;
constexpr int kAccCols = 2 * kGroupTok;
#ifndef MESW_PF_NW
#define MESW_PF_NW 2
#endif
#ifndef MESW_PF_NX
#define MESW_PF_NX 4
#endif
// ring depths (W / x / codes): x is held until the MMAs finish; (3, 3) measured equal to (2, 4)
constexpr int kNW = MESW_PF_NW, kNX = MESW_PF_NX, kNC = 4;
constexpr int kXBytes = kTileTok / 2 * kUnitK * 2;  // this CTA's half of the x tile: 32 KiB
constexpr int kCBytes = 2 * 4096;                   // two groups' 2-bit code units
constexpr int kSmemBytes = 232448;

struct Params {
  const uint16_t* x;   // canonical layout, NP rows (multiple of 256)
  int NP, m, n, n_cg, n_ks;
  const uint8_t* w;    // canonical units
  const mesw_expert_dev* table;
  const int32_t* group_slot;  // [NP / 128]: expert-table slot of each 128-token group, -1 = base only
  void* y;
  int y_bf16, ldy, B;
  const uint16_t* residual;
  int ld_res;
  int n_tiles, n_tt, G;  // tiles, 256-token tiles, CTAs
  unsigned long long* prof;  // MESW_PF_PROF: leader issuer cycle counters per CTA pair (else null)
};

struct Smem {
  uint64_t wfull[kNW], wempty[kNW];
  uint64_t xfull[kNX], xempty[kNX];
  uint64_t cfull[kNC], cempty[kNC];
  uint64_t afull[kASlots], aempty[kASlots];
  uint64_t accfull, accempty[2];
  uint32_t tmem_base;
};

__host__ __device__ inline size_t ring_off() { return (sizeof(Smem) + 1023) & ~size_t(1023); }
constexpr size_t kWOff = 0, kXOff = kWOff + (size_t)kNW * kUnitWBytes, kCOff = kXOff + (size_t)kNX * kXBytes;
constexpr size_t kRingBytes = kCOff + (size_t)kNC * kCBytes;

__device__ __forceinline__ uint32_t idesc_m256(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

__device__ __forceinline__ uint32_t bf16x2_of(float v) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(d) : "f"(v));
  return d;
}

// merged A words of one k-slice: a[i] = RN_bf16x2(q_pair * s + w_pair) (single rounding).  cw:
// the slice's code words (8 pairs each: lo code at bit 2l, hi at 16 + 2l -- mesw_layout.cuh)
__device__ __forceinline__ void merge_slice(const uint32_t* wv, const uint32_t* cw, uint32_t s2, uint32_t* a) {
#pragma unroll
  for (int w = 0; w < kSliceW / 8; ++w) {
    const uint32_t c = cw[w], b = c >> 6, d = c >> 12;
    uint32_t q[8];  // exact bf16 q in {-2,-1,0,1} (dequant_chunk<2> magic-number form)
    q[0] = bf16x2_fma(lop3_and_or(c, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
    q[1] = bf16x2_fma(lop3_and_or(c, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);
    q[2] = bf16x2_fma(lop3_and_or(c, 0x00300030u, 0x43004300u), 0x3D803D80u, 0xC120C120u);
    q[3] = bf16x2_fma(lop3_and_or(b, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
    q[4] = bf16x2_fma(lop3_and_or(b, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);
    q[5] = bf16x2_fma(lop3_and_or(b, 0x00300030u, 0x43004300u), 0x3D803D80u, 0xC120C120u);
    q[6] = bf16x2_fma(lop3_and_or(d, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
    q[7] = bf16x2_fma(lop3_and_or(d, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[8 * w + i] = bf16x2_fma(q[i], s2, wv[8 * w + i]);
  }
}

#define MESW_R8(b) "r"(r[b + 0]), "r"(r[b + 1]), "r"(r[b + 2]), "r"(r[b + 3]), "r"(r[b + 4]), "r"(r[b + 5]), "r"(r[b + 6]), "r"(r[b + 7])
__device__ __forceinline__ void tmem_st_slice(uint32_t taddr, const uint32_t* r) {
  if constexpr (kSliceW == 16)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(taddr), MESW_R8(0), MESW_R8(8) : "memory");
  else
    tmem_st32(taddr, r);
}
#undef MESW_R8

__global__ void __launch_bounds__(kThreads, 1) me_linear_prefill_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Smem& S = *reinterpret_cast<Smem*>(smem);
  uint8_t* ring = smem + ring_off();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int c2 = blockIdx.x >> 1, G2 = p.G >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNW; ++i) { mbar_init(&S.wfull[i], 1); mbar_init(&S.wempty[i], 4 * kMergeGroups); }
    for (int i = 0; i < kNX; ++i) { mbar_init(&S.xfull[i], rank == 0 ? 2 : 1); mbar_init(&S.xempty[i], 1); }
    for (int i = 0; i < kNC; ++i) { mbar_init(&S.cfull[i], 1); mbar_init(&S.cempty[i], 4 * kMergeGroups); }
    for (int i = 0; i < kASlots; ++i) { mbar_init(&S.afull[i], 2 * 4 * kMergeGroups); mbar_init(&S.aempty[i], 1); }
    mbar_init(&S.accfull, 1);
    mbar_init(&S.accempty[0], 8);
    mbar_init(&S.accempty[1], 8);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  pdl_trigger();

  if (warp == 0 || warp == 2) {
    // ============================ producers ============================
    // warp 0: W units + code units (consumed by the merge warps, freed right after their LDS);
    // warp 2: x half-tiles (held until the k-step's MMAs complete).  Separate threads, so a
    // full x ring never holds back the weight stream.
    if (lane == 0) {
      uint64_t evict_first;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(evict_first));
      int s_ = 0;
      uint32_t ph = 0, pc2 = 0;
      int sc = 0;
      bool first = true, cfirst = true;
      if (warp == 2) pdl_wait();  // x is the previous kernel's output; W / codes are static
      for (int tile = c2; tile < p.n_tiles; tile += G2) {
        const int cgp = tile / p.n_tt, tt = tile % p.n_tt;
        const int cg = 2 * cgp + (int)rank;
        const int s0 = p.group_slot[2 * tt], s1 = p.group_slot[2 * tt + 1];
        const uint8_t* c0 = s0 >= 0 ? reinterpret_cast<const uint8_t*>(p.table[s0].codes) : nullptr;
        const uint8_t* c1 = s1 >= 0 ? reinterpret_cast<const uint8_t*>(p.table[s1].codes) : nullptr;
        for (int ks = 0; ks < p.n_ks; ++ks) {
          const size_t unit = (size_t)cg * p.n_ks + ks;
          if (warp == 0) {
            if (!first) mbar_wait(&S.wempty[s_], ph ^ 1);
            mbar_arrive_expect_tx(&S.wfull[s_], kUnitWBytes);
            bulk_g2s_hint(ring + kWOff + (size_t)s_ * kUnitWBytes, p.w + unit * kUnitWBytes, kUnitWBytes,
                          &S.wfull[s_], evict_first);
            if (++s_ == kNW) { s_ = 0; ph ^= 1; first = false; }
            if (!cfirst) mbar_wait(&S.cempty[sc], pc2 ^ 1);
            mbar_arrive_expect_tx(&S.cfull[sc], (c0 ? 4096u : 0u) + (c1 ? 4096u : 0u));
            uint8_t* cdst = ring + kCOff + (size_t)sc * kCBytes;
            if (c0) bulk_g2s_hint(cdst, c0 + unit * 4096, 4096, &S.cfull[sc], evict_first);
            if (c1) bulk_g2s_hint(cdst + 4096, c1 + unit * 4096, 4096, &S.cfull[sc], evict_first);
            if (++sc == kNC) { sc = 0; pc2 ^= 1; cfirst = false; }
          } else {
            if (!first) mbar_wait(&S.xempty[s_], ph ^ 1);
            mbar_arrive_expect_tx(&S.xfull[s_], kXBytes);
            // this CTA's half of 16 windows starting at window 16*tt of k-step ks
            const size_t xoff =
                (size_t)ks * p.NP * kUnitK + (size_t)rank * (p.NP / 2) * kUnitK + (size_t)tt * 16 * 1024;
            bulk_g2s(ring + kXOff + (size_t)s_ * kXBytes, p.x + xoff, kXBytes, &S.xfull[s_]);
            if (++s_ == kNX) { s_ = 0; ph ^= 1; first = false; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank != 0) {
      // ============================ peer: relay x-landed to the leader ============================
      if (lane == 0) {
        int sx = 0;
        uint32_t px = 0;
        for (int tile = c2; tile < p.n_tiles; tile += G2)
          for (int ks = 0; ks < p.n_ks; ++ks) {
            mbar_wait(&S.xfull[sx], px);
            mbar_arrive_cta_relaxed(&S.xfull[sx], 0);
            if (++sx == kNX) { sx = 0; px ^= 1; }
          }
      }
    } else {
      // ============================ leader: MMA issue ============================
      const uint64_t xdesc0 = smem_desc(smem_u32(ring + kXOff));
      const uint32_t id = idesc_m256(kGroupTok);
      int sx = 0;
      uint32_t px = 0;
      uint32_t job = 0;  // A-slot sequence: 2 per k-step
      int n_t = 0;
      long long pr[5] = {0, 0, 0, 0, 0};  // accempty, xfull, afull, issue, total (MESW_PF_PROF)
      const long long t_start = clock64();
      long long tq = 0;
      for (int tile = c2; tile < p.n_tiles; tile += G2, ++n_t) {

        for (int ks = 0; ks < p.n_ks; ++ks) {
          if (p.prof) tq = clock64();
          mbar_wait_cluster(&S.xfull[sx], px);
          if (p.prof) pr[1] += clock64() - tq;
          const uint64_t xd = xdesc0 + (uint64_t)(sx * (kXBytes >> 4));
#pragma unroll 1
          for (int g = 0; g < 2; ++g, ++job) {
            const int slot = (int)(job % kASlots);
            if (ks == 0 && n_t > 0) {  // group g's accumulator drained by the previous tile's epilogue
              if (p.prof) tq = clock64();
              mbar_wait_cluster(&S.accempty[g], (uint32_t)((n_t - 1) & 1));
              tc_fence_after();
              if (p.prof) pr[0] += clock64() - tq;
            }
            if (p.prof) tq = clock64();
            mbar_wait_cluster(&S.afull[slot], (job / kASlots) & 1);
            tc_fence_after();
            if (p.prof) { pr[2] += clock64() - tq; tq = clock64(); }
            const uint32_t d = tbase + (uint32_t)(g * kGroupTok);
            const uint32_t a = tbase + (uint32_t)(kAccCols + slot * kACols);
            // group g's 8 windows: 8 x 2 KiB into this CTA's half tile
            const uint64_t bd = xd + (uint64_t)(g * 8 * (kXRowGroupBytes >> 4));
            mma2_ts_k128(uni(d), uni(a), uni64(bd), uni(id), uni(ks > 0 ? 1u : 0u));
            tc2_commit_w(&S.aempty[slot]);
            if (p.prof) pr[3] += clock64() - tq;
          }
          tc2_commit_w(&S.xempty[sx]);
          if (++sx == kNX) { sx = 0; px ^= 1; }
        }
        tc2_commit_w(&S.accfull);
      }
      pr[4] = clock64() - t_start;
      if (p.prof && lane == 0)
        for (int i = 0; i < 5; ++i) p.prof[(size_t)c2 * 8 + i] = (unsigned long long)pr[i];
    }
  } else if (warp >= kMergeWarp0 && warp < kEpiWarp0) {
    // ============================ merge groups ============================
    const int g = (warp - kMergeWarp0) >> 2;  // k-slice of every unit
    const int quarter = warp & 3, mrow = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    int sw = 0, sc = 0;
    uint32_t pw = 0, pcp = 0;
    uint32_t job = 0;
    pdl_wait();
    for (int tile = c2; tile < p.n_tiles; tile += G2) {
      const int cgp = tile / p.n_tt, tt = tile % p.n_tt;
      const int cg = 2 * cgp + (int)rank;
      int slot_e[2];
      uint32_t s2[2];
      const int32_t* sal_idx[2];
      const uint16_t* sal_rows[2];
      int sal_r[2], sal_end[2], sal_next[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        slot_e[e] = p.group_slot[2 * tt + e];
        s2[e] = 0;
        sal_r[e] = sal_end[e] = 0;
        sal_next[e] = 1 << 30;
        sal_idx[e] = nullptr;
        sal_rows[e] = nullptr;
        if (slot_e[e] >= 0) {
          const mesw_expert_dev ex = p.table[slot_e[e]];
          s2[e] = bf16x2_of(ex.steps[(size_t)cg * kUnitN + mrow]);
          sal_r[e] = ex.sal_off[cg];
          sal_end[e] = ex.sal_off[cg + 1];
          sal_idx[e] = ex.sal_idx;
          sal_rows[e] = ex.sal_rows;
          if (sal_r[e] < sal_end[e]) sal_next[e] = sal_idx[e][sal_r[e]];  // one global read per hit, not per k-step
        }
      }
      for (int ks = 0; ks < p.n_ks; ++ks) {
        mbar_wait(&S.wfull[sw], pw);
        uint32_t wv[kSliceW];
        const uint8_t* wt = ring + kWOff + (size_t)sw * kUnitWBytes;
        constexpr int kChunks = kSliceK / 8;  // 16-byte k-chunks of the slice
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          const uint4 t4 = lds128(wt + (mrow >> 3) * 2048 + (kChunks * g + c) * 128 + (mrow & 7) * 16);
          wv[4 * c] = t4.x; wv[4 * c + 1] = t4.y; wv[4 * c + 2] = t4.z; wv[4 * c + 3] = t4.w;
        }
        mbar_wait(&S.cfull[sc], pcp);
        constexpr int kCW = kSliceW / 8;  // code words of the slice
        uint32_t cw[2][kCW];
        const uint8_t* ct = ring + kCOff + (size_t)sc * kCBytes;
        // slice g: k-half kh = (g * kSliceK) / 64, words from ((g * kSliceK) % 64) / 16
        const int kh = (g * kSliceK) >> 6, w0 = ((g * kSliceK) & 63) >> 4;
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int w = 0; w < kCW; ++w)
            cw[e][w] = *reinterpret_cast<const uint32_t*>(ct + (size_t)e * 4096 + ((size_t)kh * 128 + mrow) * 16 + (w0 + w) * 4);
        __syncwarp();
        if (lane == 0) { mbar_arrive(&S.wempty[sw]); mbar_arrive(&S.cempty[sc]); }
        if (++sw == kNW) { sw = 0; pw ^= 1; }
        if (++sc == kNC) { sc = 0; pcp ^= 1; }
        const int k0 = ks * kUnitK + g * kSliceK;  // first input channel of this k-slice
        int slots[2];
#pragma unroll
        for (int e = 0; e < 2; ++e, ++job) {
          const int slot = (int)(job % kASlots);
          slots[e] = slot;
          if (job >= kASlots) mbar_wait(&S.aempty[slot], ((job / kASlots) - 1) & 1);
          const uint32_t acol = tbase + lane_addr + (uint32_t)(kAccCols + slot * kACols + g * kSliceW);
          {
            uint32_t a[kSliceW];
            if (slot_e[e] >= 0) merge_slice(wv, cw[e], s2[e], a);
            else {
#pragma unroll
              for (int w = 0; w < kSliceW; ++w) a[w] = wv[w];  // base-only group
            }
            tmem_st_slice(acol, a);
          }
          // salient inputs of this k-half (their codes are q = 0): rewrite the pair word with
          // RN_bf16(W + half(R)) by a single-column store after the tile store (rare: k = 8 rows
          // per block)
          while (sal_next[e] < k0 + kSliceK) {
            const int i = sal_next[e] - k0;
            const float r0v = __half2float(__ushort_as_half(sal_rows[e][(size_t)sal_r[e] * kUnitN + mrow]));
            ++sal_r[e];
            sal_next[e] = sal_r[e] < sal_end[e] ? sal_idx[e][sal_r[e]] : (1 << 30);
            if (i < 0) continue;  // belongs to another group's k-slice
            const int pw = i >> 1;
            bool lo_s = (i & 1) == 0, hi_s = !lo_s;
            float r_lo = lo_s ? r0v : 0.f, r_hi = lo_s ? 0.f : r0v;
            if (lo_s && sal_next[e] == k0 + i + 1) {  // both halves of the pair salient
              hi_s = true;
              r_hi = __half2float(__ushort_as_half(sal_rows[e][(size_t)sal_r[e] * kUnitN + mrow]));
              ++sal_r[e];
              sal_next[e] = sal_r[e] < sal_end[e] ? sal_idx[e][sal_r[e]] : (1 << 30);
            }
            uint32_t ww = 0, cword = 0;
#pragma unroll
            for (int w = 0; w < kSliceW; ++w) ww = (w == pw) ? wv[w] : ww;
#pragma unroll
            for (int w = 0; w < kCW; ++w) cword = (w == (pw >> 3)) ? cw[e][w] : cword;
            const int sh = 2 * (pw & 7);
            const float sf = bf16_lo(s2[e]);
            const float qlo = (float)((int)((cword >> sh) & 3u) - 2), qhi = (float)((int)((cword >> (16 + sh)) & 3u) - 2);
            const float lo = lo_s ? bf16_lo(ww) + r_lo : fmaf(qlo, sf, bf16_lo(ww));
            const float hi = hi_s ? bf16_hi(ww) + r_hi : fmaf(qhi, sf, bf16_hi(ww));
            uint32_t v;
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(hi), "f"(lo));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // after the tile store
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(acol + (uint32_t)pw), "r"(v)
                         : "memory");
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (rank == 0) mbar_arrive(&S.afull[slots[e]]);
            else mbar_arrive_cta_relaxed(&S.afull[slots[e]], 0);
          }
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ============================ epilogue ============================
    const int quarter = warp & 3, mrow = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    pdl_wait();
    int n_t = 0;
    for (int tile = c2; tile < p.n_tiles; tile += G2, ++n_t) {
      const int cgp = tile / p.n_tt, tt = tile % p.n_tt;
      const int j = (2 * cgp + (int)rank) * kUnitN + mrow;
      const bool jok = j < p.n;
      mbar_wait_sleep(&S.accfull, (uint32_t)(n_t & 1));
      tc_fence_after();
      // Group e's 128 columns: [h = 0: CTA0's B rows = window rows 0-7 | h = 1: rows 8-15], each
      // 8 windows x 8 rows; 32 columns (4 windows) per tcgen05.ld.  Each group's accumulator is
      // released as soon as it is drained, so the next tile's first MMAs of group 0 overlap
      // the drain of group 1.
#pragma unroll 1
      for (int e = 0; e < 2; ++e) {
        const int t_e = tt * kTileTok + e * kGroupTok;  // first token of the group
        const bool fast = jok && p.y_bf16 && !p.residual && t_e + kGroupTok <= p.B;
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {  // (h, window quad)
          const int h = q >> 1, wq = q & 1;
          uint32_t r[32];
          tmem_ld32_nowait(tbase + lane_addr + (uint32_t)(e * kGroupTok + h * 64 + wq * 32), r);
          tmem_ld_wait();
          const int tq = t_e + 8 * h + wq * 4 * 16;  // token of column 0 of this load
          if (fast) {
            __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(p.y) + (size_t)tq * p.ldy + j;
            const size_t ld = (size_t)p.ldy;
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
              for (int rr = 0; rr < 8; ++rr)
                yp[(size_t)(w * 16 + rr) * ld] = __float2bfloat16_rn(__uint_as_float(r[w * 8 + rr]));
          } else if (jok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int t = tq + (i >> 3) * 16 + (i & 7);
              if (t >= p.B) continue;
              float yv = __uint_as_float(r[i]);
              if (p.residual) yv += bf16_to_f32(p.residual[(size_t)t * p.ld_res + j]);
              if (p.y_bf16)
                reinterpret_cast<__nv_bfloat16*>(p.y)[(size_t)t * p.ldy + j] = __float2bfloat16_rn(yv);
              else
                reinterpret_cast<float*>(p.y)[(size_t)t * p.ldy + j] = yv;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&S.accempty[e]);
          else mbar_arrive_cta(&S.accempty[e], 0);
        }
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(512));
  }
}

}  // namespace prefill
}  // namespace mesw

using namespace mesw;

static unsigned long long* g_pf_prof = nullptr;

// Debug (tools/pf_timing.py): copy the last MESW_PF_PROF launch's per-pair issuer counters
// [pair][8] = {wait accempty, wait x, wait A slots, MMA issue + commit, total} in SM cycles.
extern "C" int mesw_prefill_profile_copy(unsigned long long* h_out, int n) {
  if (!g_pf_prof) return mesw_fail(MESW_ERR_VALUE, "no profile buffer (set MESW_PF_PROF)");
  cudaError_t e = cudaMemcpy(h_out, g_pf_prof, (size_t)n * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? MESW_OK : mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int mesw_me_linear_prefill(const mesw_prefill_args* a, void* stream) {
  using namespace mesw::prefill;
  if (!a || !a->x || !a->w || !a->y || !a->group_slot) return mesw_fail(MESW_ERR_VALUE, "prefill: null argument");
  if (a->NP < kTileTok || a->NP % kTileTok) return mesw_fail(MESW_ERR_VALUE, "prefill: NP must be a multiple of 256");
  if (a->B < 1 || a->B > a->NP) return mesw_fail(MESW_ERR_VALUE, "prefill: 1 <= B <= NP");
  if (a->m < 1 || a->n < 1) return mesw_fail(MESW_ERR_VALUE, "prefill: empty linear");
  if (a->code_bits != 2) return mesw_fail(MESW_ERR_UNSUPPORTED, "prefill: 2-bit device codes only");
  if (((uintptr_t)a->x) % 16 || ((uintptr_t)a->w) % 16) return mesw_fail(MESW_ERR_VALUE, "x / w must be 16-byte aligned");
  const int m_pad = (a->m + kUnitK - 1) / kUnitK * kUnitK;
  const int n_pad = (a->n + kUnitN - 1) / kUnitN * kUnitN;
  const int sms = mesw_device_sm_count();
  if (sms <= 0) return mesw_fail(MESW_ERR_CUDA, "no CUDA device");
  Params p{};
  p.x = a->x; p.NP = a->NP; p.m = a->m; p.n = a->n;
  p.n_cg = ((n_pad + 2 * kUnitN - 1) / (2 * kUnitN)) * 2;
  p.n_ks = m_pad / kUnitK;
  p.w = reinterpret_cast<const uint8_t*>(a->w);
  p.table = a->expert_table;
  p.group_slot = a->group_slot;
  p.y = a->y; p.y_bf16 = a->y_bf16; p.ldy = a->ldy; p.B = a->B;
  p.residual = a->residual; p.ld_res = a->ld_res;
  p.n_tt = a->NP / kTileTok;
  p.n_tiles = (p.n_cg / 2) * p.n_tt;
  const int want = (a->num_ctas > 0 ? a->num_ctas : sms) / 2;
  p.G = 2 * std::max(1, std::min(want, p.n_tiles));
  static const bool prof = getenv("MESW_PF_PROF") != nullptr;
  if (prof) {
    if (!g_pf_prof) cudaMalloc(&g_pf_prof, 1024 * 8 * sizeof(unsigned long long));
    p.prof = g_pf_prof;
  }
  const size_t smem = ring_off() + kRingBytes;
  if (smem > (size_t)kSmemBytes) return mesw_fail(MESW_ERR_UNSUPPORTED, "prefill: shared memory overflow");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(me_linear_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = mesw_pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, me_linear_prefill_kernel, p);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("me_linear_prefill");
}
