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

#include <algorithm>

#include "mesw_common.cuh"
#include "mesw_host.h"
#include "mesw_layout.cuh"
#include "mesw_tc.cuh"

namespace mesw {

#ifndef MESW_DQ_GROUPS
#define MESW_DQ_GROUPS 2
#endif
#ifdef MESW_PROFILE
#define MESW_PROF(...) __VA_ARGS__
#else
#define MESW_PROF(...)
#endif
constexpr int kDqGroups = MESW_DQ_GROUPS;  // dequant warpgroups: group g fills the A slots s with s % kDqGroups == g
// warp roles: 0 producer (codes, weight tiles, activations), 1-3 MMA issuers, 4-11 two dequant groups, 12-15 epilogue (TMEM lane quarters = warp % 4)
constexpr int kProdWarp = 0, kMmaWarp = 1;
constexpr int kMaxIssuers = 3;  // warps 1..3
constexpr int kDqWarp0 = 4, kEpiWarp0 = kDqWarp0 + 4 * kDqGroups;
constexpr int kThreads = (kEpiWarp0 + 4) * 32;  // 16 warps
constexpr int kTmemCols = 512;
#ifndef MESW_HALF_JOBS
#define MESW_HALF_JOBS 0
#endif
#ifndef MESW_DQ_BATCH
#define MESW_DQ_BATCH 2
#endif
constexpr int kDqBatch = MESW_DQ_BATCH;  // jobs per TMEM-store completion wait (+2 % on C1 at 2)
// A job = one expert's dequantised A tile for one unit: 128 outputs x 128 k (64 TMEM columns).
// MESW_HALF_JOBS=1 makes each k-half (32 columns) its own job with its own slot (measured
// slower: the per-job handshake cost doubles, C1 45 -> 50 us).
constexpr int kJobHalves = MESW_HALF_JOBS ? 2 : 1;
constexpr int kMaxASlots = 16;
constexpr int kAColsPerSlot = 64 / kJobHalves;
constexpr int kMaxRows = 192;  // padded token rows per launch (TMEM: 2 * rows <= 384)
constexpr int kMaxStages = 8;
constexpr int kMaxCStages = 16;
#ifndef MESW_STAGE_MIN
#define MESW_STAGE_MIN 0
#endif
constexpr int kSalFast = 8;            // salient rows per column group handled from smem

struct SegDesc {
  const uint8_t* codes;
  const float* steps;
  const int32_t* sal_off;
  const int32_t* sal_idx;
  const uint16_t* sal_rows;
  int begin, end;
  int w0, nw;  // first 16-row window touched, windows touched (begins are multiples of 8 rows)
  int dcol;    // first column of the segment's delta accumulator (after the NP base columns)
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
  int seg_dcol[MESW_MAX_SEGMENTS];  // host-computed: prefix sums of 16 x windows touched
  int NPD;                          // delta accumulator columns (sum of 16 x windows touched)
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
  // A ring split per MMA issuer: issuer i owns slots [a_base[i], a_base[i] + a_na[i]) and
  // consumes its jobs in order; both dequant groups walk every job in the same order.  Every
  // slot is therefore filled and drained in one sequence, so the mbarrier parity waits on
  // it can never alias a phase two steps away.
  int a_base[3], a_na[3];
  int ring_bytes;  // dynamic shared memory past the Smem header
  const float* x_corr;  // offset-code bias table [t * x_corr_ld + ks] (OFF kernels)
  const int32_t* y_rows;  // optional output row map (mesw_linear_args.y_rows)
  int x_corr_ld;
  int n_iss;  // MMA issuer warps (a tcgen05.mma stream runs ~40 cycles/instr per issuer)
  int n_dq;   // delta issuers = active dequant groups (group g feeds delta issuer g)
  unsigned long long* tbuf;  // MESW_TIMING: per-CTA globaltimer stamps
  int dbg;  // reserved (MESW_DBG)
  // SwiGLU epilogue (mesw_linear_args.swiglu_I): columns [0, I) gate, [I, 2I) up
  int swiglu_I;
  uint16_t* act;
  int act_np;
  float* act_corr;
  int act_corr_ld;
};

struct Smem {
  uint64_t xfull[kMaxStages], xempty[kMaxStages];
  uint64_t wfull[kMaxStages], wempty[kMaxStages];
  uint64_t cfull[kMaxCStages], cempty[kMaxCStages];
  uint64_t afull[kMaxASlots], aempty[kMaxASlots];
  uint64_t accfull[2], accempty[2];
  uint64_t finbar;  // final-piece partials staged by bulk copy
  uint32_t tmem_base;
  int flag, sflag;
  struct { int on, cg, cgp, p_first, p_last, fast; } fin;  // final-piece reduction hand-off
  int tok2seg[kMaxRows];
  int half2seg[kMaxRows / 8];  // segment owning rows [8h, 8h + 8) (a segment begins on an 8-row half)
  int yrow[kMaxRows];  // output / residual row of launch row t (-1: not written)
  SegDesc segs[MESW_MAX_SEGMENTS];
  int sal_r0[MESW_MAX_SEGMENTS], sal_k[MESW_MAX_SEGMENTS];  // current column group's salient range
  float xsal[kMaxRows][kSalFast];  // x[t][salient idx r] of the current column group (fast path)
  float corr[kMaxRows];             // offset codes: per-token bias over the piece's k range
};

__host__ __device__ inline size_t ring_offset() { return (sizeof(Smem) + 1023) & ~size_t(1023); }

// Order in which a CTA walks its unit range [u0, u1): piece 0 = the run in the LAST
// column group, piece 1 = the run in the FIRST column group, then the middle column
// groups in order.  The two boundary pieces are the ones shared with neighbouring CTAs
// (stream-K), so their cross-CTA reductions happen early and overlap the main loop
// instead of forming a tail.
struct PieceOrder {
  long long u0, u1;
  int n_ks, cg_lo, cg_hi, np;
  __device__ __forceinline__ PieceOrder(long long a, long long b, int nks) : u0(a), u1(b), n_ks(nks) {
    cg_lo = (int)(a / nks);
    cg_hi = (int)((b - 1) / nks);
    np = b > a ? cg_hi - cg_lo + 1 : 0;
  }
  __device__ __forceinline__ int cg_of(int idx) const {
    return idx == 0 ? cg_hi : (idx == 1 ? cg_lo : cg_lo + idx - 1);
  }
  __device__ __forceinline__ void bounds(int idx, long long& a, long long& b) const {
    const long long c0 = (long long)cg_of(idx) * n_ks;
    a = c0 > u0 ? c0 : u0;
    b = c0 + n_ks < u1 ? c0 + n_ks : u1;
  }
};

// MMA issuer of expert segment q.  With a base weight, issuer 0 issues ONLY the base tile
// (so the weight stream never waits on the delta pipeline) and the segments go round-robin
// to issuers 1..n-1; without one (or with a single issuer) they go round-robin to all.
__host__ __device__ __forceinline__ int seg_issuer(int q, int n_iss, bool has_w) {
  return (has_w && n_iss > 1) ? 1 + q % (n_iss - 1) : q % n_iss;
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
  for (int q = gtid; q < p.n_seg; q += 128) {
    const SegDesc& sd = S.segs[q];
    const int r0 = sd.sal_off[cg];
    S.sal_r0[q] = r0;
    S.sal_k[q] = sd.sal_off[cg + 1] - r0;
  }
  named_bar_sync(1, 128);
  bool fast = true;
  for (int q = 0; q < p.n_seg; ++q)
    if (S.sal_k[q] > kSalFast) fast = false;
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
          if (sg >= 0 && r < S.sal_k[sg])
            v[k] = bf16_to_f32(p.x[xc_index(t, S.segs[sg].sal_idx[S.sal_r0[sg] + r], p.NP)]);
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

// Delta accumulators of the 16 rows [t0, t0 + 16) (one window w): rows 0-7 (the CTA0 half)
// from the segment owning half 2w, rows 8-15 from the owner of half 2w + 1.  A segment's
// delta range [dcol, dcol + 16 nw) holds its windows' CTA0 rows first, then the CTA1 rows.
template <bool HALF>
__device__ __forceinline__ void load_delta16(const Smem& S, uint32_t acc, int NP, int t0, float* vd) {
  const int w = t0 >> 4;
  if constexpr (!HALF) {  // every segment begins on a window: one owner for all 16 rows
    const int sg = S.half2seg[2 * w];
    if (sg >= 0) {
      const SegDesc& sd = S.segs[sg];
      const uint32_t c = acc + (uint32_t)(NP + sd.dcol + 8 * (w - sd.w0));
      tmem_ld8(c, vd);
      tmem_ld8(c + (uint32_t)(8 * sd.nw), vd + 8);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) vd[i] = 0.f;
    }
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int sg = S.half2seg[2 * w + h];
    if (sg >= 0) {
      const SegDesc& sd = S.segs[sg];
      tmem_ld8(acc + (uint32_t)(NP + sd.dcol + h * 8 * sd.nw + 8 * (w - sd.w0)), vd + 8 * h);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) vd[8 * h + i] = 0.f;
    }
  }
}

// Output / residual row of launch row t: the caller's row map (me_linear's device-side
// grouping), or t itself.  A kernel template parameter: launches without a map (the serving
// engine's) keep the plain row arithmetic in the latency-critical epilogue (a runtime branch
// there measured 5 % of the C2 step).
template <bool YMAP>
__device__ __forceinline__ int out_row(const LinearParams& p, const Smem& S, int t) {
  if constexpr (YMAP) return S.yrow[t];
  else return t;
}

// Per-chunk epilogue operands that do not depend on the accumulators (prefetched one
// chunk ahead): each 8-row half's expert segment, its step s_e[j], salient rows R_e[r][j],
// and the residual.  A half holds rows of at most one segment (segments begin on halves).
struct EpiPre {
  int sg[2];
  float sj[2];
  float R[kSalFast];   // salient rows of the first half's segment (or the second's if the first is empty)
  float R1[kSalFast];  // HALF: the second half's segment when it differs from the first
  float res[16];
};

__device__ __forceinline__ void load_sal_rows(const Smem& S, int sg, int m, float* R) {
  const SegDesc& sd = S.segs[sg];
  const int r0 = S.sal_r0[sg], k = S.sal_k[sg];  // smem: no dependent global round trip
#pragma unroll
  for (int r = 0; r < kSalFast; ++r)
    R[r] = r < k ? __half2float(__ushort_as_half(sd.sal_rows[(size_t)(r0 + r) * kUnitN + m])) : 0.f;
}

template <bool YMAP, bool HALF>
__device__ __forceinline__ void epi_prefetch(const LinearParams& p, const Smem& S, int cg, int m, int t0,
                                             bool fast, EpiPre& e, bool full = true) {
  const int j = cg * kUnitN + m;
  const int s0 = S.half2seg[t0 >> 3], s1 = HALF ? S.half2seg[(t0 >> 3) + 1] : s0;
  e.sg[0] = s0;
  e.sg[1] = s1;
  e.sj[0] = (s0 >= 0 && j < p.n) ? S.segs[s0].steps[j] : 0.f;
  e.sj[1] = s1 == s0 ? e.sj[0] : ((s1 >= 0 && j < p.n) ? S.segs[s1].steps[j] : 0.f);
  const int sr = e.sg[0] >= 0 ? e.sg[0] : e.sg[1];
#pragma unroll
  for (int r = 0; r < kSalFast; ++r) e.R[r] = 0.f;
  if (!full) return;  // stream-K partial pieces use only sg / sj (the final reducer reloads the rest)
  if (fast && sr >= 0 && j < p.n) load_sal_rows(S, sr, m, e.R);
  if (HALF) {
#pragma unroll
    for (int r = 0; r < kSalFast; ++r) e.R1[r] = 0.f;
    if (fast && s0 >= 0 && s1 >= 0 && s1 != s0 && j < p.n) load_sal_rows(S, s1, m, e.R1);
  }
#pragma unroll
  for (int t = 0; t < 16; ++t)
    e.res[t] = (p.residual && t0 + t < p.B && j < p.n && out_row<YMAP>(p, S, t0 + t) >= 0)
                   ? bf16_to_f32(p.residual[(size_t)out_row<YMAP>(p, S, t0 + t) * p.ld_res + j]) : 0.f;
}

// Thread owns output channel j = cg*128 + m; accumulators for the 16 rows [t0, t0+16).
// All 16 outputs are formed first and stored after: stores through the generic y pointer
// may alias shared memory, so interleaving them with the rows' smem reads serialised the
// rows (~300 cycles per row in the final stream-K reductions, measured).
template <bool YMAP, bool HALF>
__device__ __forceinline__ void epi_store16(const LinearParams& p, const Smem& S, int cg, int m, int t0,
                                            const float* vb, const float* vd, bool fast, const EpiPre& e,
                                            bool dry = false) {
  const int j = cg * kUnitN + m;
  if (j >= p.n) return;
  const bool two = HALF && e.sg[0] >= 0 && e.sg[1] >= 0 && e.sg[1] != e.sg[0];  // second half: other rows
  float out[16];
  if (fast) {
    // straight-line: no per-row branch, so the 16 rows' smem reads and fma chains overlap
    // (a data-dependent branch per row serialised them: ~170 cycles per row, measured)
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int tok = t0 + t;
      const int h = HALF ? (t >> 3) : 0;
      const bool match = tok < p.B && e.sg[h] >= 0 && S.tok2seg[tok] == e.sg[h];
      float d = e.sj[h] * vd[t];
#pragma unroll
      for (int r = 0; r < kSalFast; ++r) d = fmaf(S.xsal[tok][r], (h == 1 && two) ? e.R1[r] : e.R[r], d);
      float v = vb[t] + (match ? d : 0.f) + e.res[t];
      if (p.activation == 1) v = fmaxf(v, 0.f);
      out[t] = v;
    }
  } else {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int tok = t0 + t;
      float v = vb[t];
      const int h = HALF ? (t >> 3) : 0;
      if (tok < p.B && e.sg[h] >= 0 && S.tok2seg[tok] == e.sg[h]) {
        float d = e.sj[h] * vd[t];
        const SegDesc& sd = S.segs[e.sg[h]];
        const int r0 = sd.sal_off[cg], k = sd.sal_off[cg + 1] - r0;
        for (int r = 0; r < k; ++r) {
          const float xv = bf16_to_f32(p.x[xc_index(tok, sd.sal_idx[r0 + r], p.NP)]);
          const float rv = __half2float(__ushort_as_half(sd.sal_rows[(size_t)(r0 + r) * kUnitN + m]));
          d = fmaf(xv, rv, d);
        }
        v += d;
      }
      v += e.res[t];
      if (p.activation == 1) v = fmaxf(v, 0.f);
      out[t] = v;
    }
  }
  MESW_PROF(if (p.tbuf && threadIdx.x == 0) p.tbuf[4096 * 12 + (size_t)blockIdx.x * 8 + 2] = clock64();)
  if (dry) return;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int tok = t0 + t;
    if (tok >= p.B) break;
    const int orow = out_row<YMAP>(p, S, tok);
    if (orow < 0) continue;
    if (p.y_bf16)
      reinterpret_cast<__nv_bfloat16*>(p.y)[(size_t)orow * p.ldy + j] = __float2bfloat16_rn(out[t]);
    else
      reinterpret_cast<float*>(p.y)[(size_t)orow * p.ldy + j] = out[t];
  }
}

// Stream-K reduction + epilogue of one 16-row chunk of column group cg (thread owns
// column m): the contributors' partials are summed in fixed pair order (bit-identical for
// any launch geometry with the same row count), then stored through epi_store16.  The
// epilogue operands are fetched together with the partials: one L2 round trip per chunk.
// stage != nullptr: the contributors' slots were bulk-copied to shared memory (final piece).
template <bool YMAP, bool HALF>
__device__ __forceinline__ void reduce_chunk(const LinearParams& p, const Smem& S, int cg, int cgp, int rank, int m,
                                          int t0, int p_first, int p_last, bool fast, const EpiPre& pre,
                                          const float* stage, bool dry = false) {
  const int NP = p.NP;
  const long long T2 = p.T, G2 = p.G / 2;
  const size_t slot_floats = (size_t)NP * kUnitN;
  float vb[16], vd[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) vb[i] = vd[i] = 0.f;  // partials already hold base + s_j * delta
  for (int pp = p_first; pp <= p_last; ++pp) {
    float lb[16];
    if (stage) {
      const float* src = stage + (size_t)(pp - p_first) * slot_floats + (size_t)t0 * kUnitN + m;
#pragma unroll
      for (int i = 0; i < 16; ++i) lb[i] = src[(size_t)i * kUnitN];
    } else {
      const long long pu0 = (long long)pp * T2 / G2;
      const int s2 = 2 * (2 * pp + rank) + ((int)(pu0 / p.n_ks) == cgp ? 0 : 1);
      const float* src = p.ws + (size_t)s2 * slot_floats + (size_t)t0 * kUnitN + m;
#pragma unroll
      for (int i = 0; i < 16; ++i) lb[i] = __ldcg(src + (size_t)i * kUnitN);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) vb[i] += lb[i];
  }
  MESW_PROF(if (p.tbuf && threadIdx.x == 0) p.tbuf[4096 * 12 + (size_t)blockIdx.x * 8 + 1] = clock64();)
  epi_store16<YMAP, HALF>(p, S, cg, m, t0, vb, vd, fast, pre, dry);
}

// Offset-code bias weight of input k (mesw.h x_corr; same as mesw_glue.cu corr_w).
__device__ __forceinline__ float act_corr_w(int k) {
  const int l = ((k & 63) >> 1) & 7;
  const int m = l < 6 ? l % 3 : l - 6;
  return m == 0 ? 130.f : (m == 1 ? 34.f : 10.f);
}

// SwiGLU epilogue: called by the NT threads that just wrote the FINAL values of column group
// cg (tid in [0, NT)).  Gate block b = cg (cg < I/128) and up block b = cg - I/128 are final
// in two places of the launch; the second of them to finish computes act = silu(gate) * up
// for block b -- mesw_swiglu's arithmetic -- from y (L2) and writes the canonical input of
// the down projection plus its bias table (the SwiGLU launch disappears from the step).
template <int NT>
__device__ __forceinline__ void swiglu_final(const LinearParams& p, Smem& S, int cg, int tid) {
  const int nb = p.swiglu_I >> 7;
  const int blk = cg < nb ? cg : cg - nb;
  if (blk < 0 || blk >= nb) return;
  // the writers' y stores are ordered before thread 0's release by the barrier
  // (cumulativity): one device-scope fence per CTA, not one per thread
  if constexpr (NT == kThreads) __syncthreads(); else named_bar_sync(1, 128);
  if (tid == 0) {
    __threadfence();
    const int prev = atomicAdd(&p.counters[p.n_cg + blk], 1);
    S.sflag = prev == 1;
    if (prev == 1) p.counters[p.n_cg + blk] = 0;  // self-reset for the next launch
  }
  if constexpr (NT == kThreads) __syncthreads(); else named_bar_sync(1, 128);
  const bool second = S.sflag != 0;
  if (!second) return;  // (thread 0's fence + atomic acquired the other half; the barrier passes it on)
  const int I = p.swiglu_I, lane = tid & 31;
  const int i = blk * 128 + 4 * lane;  // this lane's 4 consecutive channels of the block
  for (int t = tid >> 5; t < p.B; t += NT / 32) {  // one warp per row
    const uint16_t* r = reinterpret_cast<const uint16_t*>(p.y) + (size_t)t * p.ldy;
    const uint2 g4 = __ldcg(reinterpret_cast<const uint2*>(r + i));
    const uint2 u4 = __ldcg(reinterpret_cast<const uint2*>(r + I + i));
    const uint32_t gg[2] = {g4.x, g4.y}, uu[2] = {u4.x, u4.y};
    uint32_t o[2];
    float c = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float g0 = bf16_lo(gg[h]), g1 = bf16_hi(gg[h]);
      const float s0 = g0 / (1.f + __expf(-g0)), s1 = g1 / (1.f + __expf(-g1));
      __nv_bfloat162 v = __floats2bfloat162_rn(s0 * bf16_lo(uu[h]), s1 * bf16_hi(uu[h]));
      o[h] = *reinterpret_cast<uint32_t*>(&v);
      c += act_corr_w(i + 2 * h) * (bf16_lo(o[h]) + bf16_hi(o[h]));
    }
    *reinterpret_cast<uint2*>(p.act + xc_index(t, i, p.act_np)) = make_uint2(o[0], o[1]);
    if (p.act_corr) {
#pragma unroll
      for (int q = 16; q; q >>= 1) c += __shfl_xor_sync(0xffffffffu, c, q);
      if (lane == 0) p.act_corr[(size_t)t * p.act_corr_ld + blk] = c;
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");  // not hoisted across barriers
  return t;
}
// Cycle-count profiling of the role loops (tools/ktiming.py): compiled in only with
// -DMESW_PROFILE (MESW_PROFILE=1 python build.py --force); zero cost otherwise.
#define MESW_STAMP(i) \
  do { if (p.tbuf) p.tbuf[(size_t)blockIdx.x * 8 + (i)] = gtimer(); } while (0)
// second stamp bank (tail phases, SM clock cycles: %globaltimer reads of different warps of
// one CTA were seen microseconds apart across a barrier), tools/ktiming.py
#define MESW_STAMP2(i) \
  do { if (p.tbuf) p.tbuf[4096 + (size_t)blockIdx.x * 8 + (i)] = (unsigned long long)clock64(); } while (0)

// ---------------------------------------------------------------- kernel
// A cluster of two CTAs ("pair") owns two adjacent column groups (256 output channels)
// and issues cta_group::2 MMAs with M = 256: every tcgen05.mma covers both column groups,
// halving the tensor-pipe instruction count (the bound at decode batch sizes).  Each CTA
// streams its own column group's weight tiles and codes, its own half of every 16-row
// activation window (B is split along N between the pair), dequantises its own A rows into
// its own TMEM, and drains its own accumulators; the leader (rank 0) issues all MMAs and
// commits them to both CTAs' barriers (multicast).  The peer relays its "tile landed"
// events to the leader's barriers.
template <int DB, bool OFF, bool YMAP, bool HALF>
__global__ void __launch_bounds__(kThreads, 1) me_linear_tc_kernel(const __grid_constant__ LinearParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Smem& S = *reinterpret_cast<Smem*>(smem);
  uint8_t* ring = smem + ring_offset();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int c = blockIdx.x;         // CTA index (stream-K slots)
  const int c2 = blockIdx.x >> 1;   // pair index
  const long long T2 = p.T, G2 = p.G / 2;
  const long long u0 = (long long)c2 * T2 / G2, u1 = (long long)(c2 + 1) * T2 / G2;  // pair units
  const PieceOrder po(u0, u1, p.n_ks);
  constexpr int CB = kUnitN * kUnitK * DB / 8;  // code bytes per unit per expert
  constexpr int CHB = 8 * DB;                   // code bytes per (k-half, channel)
  const int NP = p.NP, HP = NP / 2;             // rows per launch / per CTA half

  if (threadIdx.x == 0) {
    const uint32_t peer_relay = rank == 0 ? 2 : 1;  // leader: own tile + peer relay
    for (int i = 0; i < p.nx; ++i) { mbar_init(&S.xfull[i], peer_relay); mbar_init(&S.xempty[i], p.n_iss); }
    for (int i = 0; i < p.nw; ++i) { mbar_init(&S.wfull[i], peer_relay); mbar_init(&S.wempty[i], 1); }
    for (int i = 0; i < p.nc; ++i) { mbar_init(&S.cfull[i], 1); mbar_init(&S.cempty[i], 128 * p.n_dq); }
    for (int i = 0; i < p.n_aslots; ++i) { mbar_init(&S.afull[i], 8); mbar_init(&S.aempty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&S.accfull[i], p.n_iss); mbar_init(&S.accempty[i], 8); }
    mbar_init(&S.finbar, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  for (int i = threadIdx.x; i < kMaxRows; i += kThreads) {
    S.tok2seg[i] = -1;
    if (i < kMaxRows / 8) S.half2seg[i] = -1;
    S.yrow[i] = i < p.B ? (p.y_rows ? p.y_rows[i] : i) : -1;  // written by the host before launch
  }
  if (threadIdx.x == 0) S.fin.on = 0;
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
    d.w0 = d.begin >> 4;
    d.nw = ((d.end - 1) >> 4) - d.w0 + 1;
    d.dcol = p.seg_dcol[q];
    S.segs[q] = d;
    for (int t = d.begin; t < d.end; ++t) S.tok2seg[t] = q;
    for (int h = d.begin >> 3; h <= (d.end - 1) >> 3; ++h) S.half2seg[h] = q;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive
  tc_fence_after();
  const uint32_t tbase = S.tmem_base;
  const bool has_w = p.w != nullptr;
  if (threadIdx.x == 0) MESW_STAMP(0);
  pdl_trigger();

  if (warp == kProdWarp) {
    // ===================== producer (own column group / own x half), one thread =====================
    // per unit: code chunks, weight tile (both static: the first rings' worth is requested
    // before the PDL wait), activation half-tile (after it).
    if (lane == 0) {
      uint64_t evict_first;  // weights / codes are streamed once: do not let them evict partials
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(evict_first));
      int sw = 0, sx = 0, sc = 0;
      uint32_t pw = 0, px = 0, pc = 0;
      bool wfirst = true, xfirst = true, cfirst = true;
      auto issue_static = [&](int cg, int ks) {
        const long long unit = (long long)cg * p.n_ks + ks;  // this CTA's unit
        for (int ch = 0; ch < p.n_chunks; ++ch) {
          const int sg0 = ch * p.segs_per_chunk;
          const int sg1 = min(p.n_seg, sg0 + p.segs_per_chunk);
          if (!cfirst) mbar_wait(&S.cempty[sc], pc ^ 1);
          mbar_arrive_expect_tx(&S.cfull[sc], (uint32_t)(sg1 - sg0) * CB);
          for (int q = sg0; q < sg1; ++q)
            bulk_g2s_hint(ring + p.co + (size_t)sc * p.cbytes + (size_t)(q - sg0) * CB,
                          S.segs[q].codes + (size_t)unit * CB, CB, &S.cfull[sc], evict_first);
          if (++sc == p.nc) { sc = 0; pc ^= 1; cfirst = false; }
        }
        if (has_w) {
          if (!wfirst) mbar_wait(&S.wempty[sw], pw ^ 1);
          mbar_arrive_expect_tx(&S.wfull[sw], kUnitWBytes);
          bulk_g2s_hint(ring + p.wo + (size_t)sw * kUnitWBytes, p.w + (size_t)unit * kUnitWBytes, kUnitWBytes,
                        &S.wfull[sw], evict_first);
          if (++sw == p.nw) { sw = 0; pw ^= 1; wfirst = false; }
        }
      };
      int n_pre = 0;
      {
        int D = p.nx;
        if (has_w && p.nw < D) D = p.nw;
        if (p.n_chunks > 0 && p.nc / p.n_chunks < D) D = p.nc / p.n_chunks;
        for (int pi = 0; pi < po.np && n_pre < D; ++pi) {
          long long pa, pb;
          po.bounds(pi, pa, pb);
          const int cgp = po.cg_of(pi);
          for (long long u = pa; u < pb && n_pre < D; ++u, ++n_pre)
            issue_static(2 * cgp + (int)rank, (int)(u - (long long)cgp * p.n_ks));
        }
      }
      pdl_wait();
      int idx = 0;
      for (int pi = 0; pi < po.np; ++pi) {
        long long pa, pb;
        po.bounds(pi, pa, pb);
        const int cgp = po.cg_of(pi);
        const int cg = 2 * cgp + (int)rank;
        for (long long u = pa; u < pb; ++u, ++idx) {
          const int ks = (int)(u - (long long)cgp * p.n_ks);
          if (idx >= n_pre) issue_static(cg, ks);
          if (!xfirst) mbar_wait(&S.xempty[sx], px ^ 1);
          mbar_arrive_expect_tx(&S.xfull[sx], (uint32_t)p.xbytes);
          bulk_g2s(ring + p.xo + (size_t)sx * p.xbytes,
                   p.x + (size_t)ks * NP * kUnitK + (size_t)rank * HP * kUnitK, p.xbytes, &S.xfull[sx]);
          if (++sx == p.nx) { sx = 0; px ^= 1; xfirst = false; }
        }
      }
    }
  } else if (warp >= kMmaWarp && warp < kMmaWarp + kMaxIssuers) {
    const int role = warp - kMmaWarp;
    if (rank != 0) {
      // ===================== peer: relay "x / weight tile landed" to the leader =====================
      if (role == 0 && lane == 0) {
        int sx = 0, sw = 0;
        uint32_t px = 0, pw = 0;
        for (int pi = 0; pi < po.np; ++pi) {
          long long pa, pb;
          po.bounds(pi, pa, pb);
          for (long long u = pa; u < pb; ++u) {
            mbar_wait(&S.xfull[sx], px);
            mbar_arrive_cta_relaxed(&S.xfull[sx], 0);
            if (++sx == p.nx) { sx = 0; px ^= 1; }
            if (has_w) {
              mbar_wait(&S.wfull[sw], pw);
              mbar_arrive_cta_relaxed(&S.wfull[sw], 0);
              if (++sw == p.nw) { sw = 0; pw ^= 1; }
            }
          }
        }
      }
    } else if (role < p.n_iss) {
      // ===================== leader: issue the pair's MMAs (whole warp, elected lane) ========
      // Issuer 0 owns the base tile, segments go to seg_issuer().  Each accumulator range is
      // owned by exactly one issuer, so its k-ordered accumulate chain stays in one issue order.
      const bool do_base = has_w && role == 0;
      const uint64_t xdesc0 = smem_desc(smem_u32(ring + p.xo));
      const uint64_t wdesc0 = smem_desc(smem_u32(ring + p.wo));
      const uint32_t xstride = (uint32_t)p.xbytes >> 4, wstride = kUnitWBytes >> 4;
      const uint32_t id_base = idesc_bf16_m256(NP);
      const int na_own = p.a_na[role], abase_own = p.a_base[role];
      const int iss_first = (has_w && p.n_iss > 1) ? 1 : 0;  // seg_issuer(q) = iss_first + q % q_step
      const int q_step = p.n_iss - iss_first;
      const int q_own0 = role >= iss_first ? role - iss_first : p.n_seg;
      int sx = 0, sw = 0;
      uint32_t px = 0, pw = 0;
      int aslot = 0;  // index within this issuer's sub-ring
      uint32_t aph = 0;
      int ab = 0;
      int use0 = 0, use1 = 0;
      MESW_PROF(long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};)
      MESW_PROF(const long long tstart = clock64();)
      MESW_PROF(int ucount = 0;)
      MESW_PROF(if (p.tbuf && blockIdx.x == 0 && lane == 0) p.tbuf[4096 * 56 + 256 + role] = tstart;)
      MESW_PROF(long long tq;)
      for (int pi = 0; pi < po.np; ++pi) {
        long long pa, pb;
        po.bounds(pi, pa, pb);
        for (long long u = pa; u < pb; ++u) {
          MESW_PROF(const long long tu = clock64();)
          const bool piece_first = (u == pa);
          const bool piece_last = (u == pb - 1);
          const int use = ab ? use1 : use0;
          if (piece_first && use > 0) {
            MESW_PROF(tq = clock64();)
            mbar_wait_cluster(&S.accempty[ab], (uint32_t)((use - 1) & 1));  // both epilogues drained it
            tc_fence_after();
            MESW_PROF(prof[5] += clock64() - tq;)
          }
          const uint32_t d_base = tbase + (uint32_t)(ab * (NP + p.NPD));
          const uint32_t f0 = piece_first ? 0u : 1u;
          MESW_PROF(tq = clock64();)
          mbar_wait_cluster(&S.xfull[sx], px);
          MESW_PROF(prof[0] += clock64() - tq;)
          const uint64_t xd = xdesc0 + (uint64_t)(sx * xstride);
          if (do_base) {
            MESW_PROF(tq = clock64();)
            mbar_wait_cluster(&S.wfull[sw], pw);
            MESW_PROF(prof[1] += clock64() - tq;)
            MESW_PROF(tq = clock64();)
            tc_fence_after();
            const uint64_t wd = wdesc0 + (uint64_t)(sw * wstride);
            mma2_ss_k128(uni(d_base), uni64(wd), uni64(xd), uni(id_base), uni(f0));
            tc2_commit_w(&S.wempty[sw]);
            if (++sw == p.nw) { sw = 0; pw ^= 1; }
            MESW_PROF(prof[2] += clock64() - tq;)
          }
          // this issuer's segments: seg_issuer() is round-robin, so stride through them
          for (int q = q_own0; q < p.n_seg; q += q_step) {
#pragma unroll 1
            for (int kh = 0; kh < kJobHalves; ++kh) {
              MESW_PROF(tq = clock64();)
              mbar_wait_cluster(&S.afull[abase_own + aslot], aph);
              MESW_PROF(prof[3] += clock64() - tq;)
              MESW_PROF(if (p.tbuf && blockIdx.x == 0 && lane == 0 && prof[7] < 32) p.tbuf[4096 * 56 + 512 + role * 64 + 2 * prof[7]] = clock64();)
              MESW_PROF(tq = clock64();)
              tc_fence_after();
              // N = the windows the segment touches; rows of other segments in them (a half
              // window shared at a segment boundary) land in columns this segment never reads
              const uint32_t id = idesc_bf16_m256(16 * S.segs[q].nw);
              const uint32_t dd = d_base + (uint32_t)(NP + S.segs[q].dcol);
              const uint32_t a0 = tbase + (uint32_t)(p.a_col0 + (abase_own + aslot) * kAColsPerSlot);
              // B rows of the expert's windows: window w's half lives at w * 2048 B in each CTA
              const uint64_t bd = xd + (uint64_t)(S.segs[q].w0 * (kXRowGroupBytes >> 4)) + (uint64_t)(kh * 64);
#ifndef MESW_EXP_NOMMA
              if (kJobHalves == 2) mma2_ts_k64(uni(dd), uni(a0), uni64(bd), uni(id), uni(kh == 0 ? f0 : 1u));
              else mma2_ts_k128(uni(dd), uni(a0), uni64(bd), uni(id), uni(f0));
#endif
              tc2_commit_w(&S.aempty[abase_own + aslot]);
              if (++aslot == na_own) { aslot = 0; aph ^= 1; }
              MESW_PROF(prof[4] += clock64() - tq;)
              MESW_PROF(if (p.tbuf && blockIdx.x == 0 && lane == 0 && prof[7] < 32) p.tbuf[4096 * 56 + 512 + role * 64 + 2 * prof[7] + 1] = clock64();)
              MESW_PROF(prof[7]++;)
            }
          }
          tc2_commit_w(&S.xempty[sx]);
          if (++sx == p.nx) { sx = 0; px ^= 1; }
          if (piece_last) {
            tc2_commit_w(&S.accfull[ab]);
            if (ab) ++use1; else ++use0;
            if (p.n_acc == 2) ab ^= 1;
          }
          MESW_PROF(prof[5] += clock64() - tu;)
          MESW_PROF(if (p.tbuf && blockIdx.x == 0 && lane == 0 && ucount < 64) p.tbuf[4096 * 56 + role * 64 + ucount] = clock64();)
          MESW_PROF(++ucount;)
        }
      }
      if (role == 0 && lane == 0) MESW_STAMP(3);
      MESW_PROF(prof[6] = clock64() - tstart;)
      MESW_PROF(if (p.tbuf && lane == 0) for (int i = 0; i < 8; ++i) p.tbuf[(role < 2 ? 4096 * 8 + (size_t)blockIdx.x * 16 + role * 8 : 4096 * 48 + (size_t)blockIdx.x * 8) + i] = prof[i];)
    }
  } else if (warp < kEpiWarp0) {
    // ===================== dequant groups: own codes -> own TMEM A rows =====================
    // Issuer-affine groups: group g serves delta issuer g (segments q = g, g + n_dq, ...) and
    // walks that issuer's A sub-ring with two registers (position, laps).  No per-job issuer
    // lookup, no skipped jobs, no data-dependent branches in the loop: the profile of the
    // previous slot-affine form showed the dequant warps ~80 % busy on that bookkeeping
    // (branch_resolving / dependent-latency stalls), not on the expansion or the TMEM stores.
    const int grp = (warp - kDqWarp0) >> 2;
    const int quarter = warp & 3;
    const int mrow = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    constexpr int WPK = CHB / 4;  // code words per k-half of a channel
    const int n_dq = p.n_dq;
    const int dq_mask = n_dq - 1, dq_shift = n_dq - 1;  // n_dq in {1, 2} (kDqGroups == 2)
    static_assert(kDqGroups <= 2, "dequant bookkeeping assumes at most two groups");
    MESW_PROF(long long dprof[8] = {0, 0, 0, 0, 0, 0, 0, 0};)
    MESW_PROF(const long long dstart = clock64();)
    MESW_PROF(int dcount = 0;)
    MESW_PROF(long long dq;)
    if (grp < n_dq) {
      const int irole = grp + ((has_w && p.n_iss > 1) ? 1 : 0);  // the issuer warp this group feeds
      const int na = p.a_na[irole], ab = p.a_base[irole];
      int pos = 0, use = 0;
      int sc = 0;
      uint32_t pc = 0;
      for (int pi = 0; pi < po.np; ++pi) {
        long long pa, pb;
        po.bounds(pi, pa, pb);
        for (long long u = pa; u < pb; ++u) {
          for (int ch = 0; ch < p.n_chunks; ++ch) {
            const int sg0 = ch * p.segs_per_chunk;
            const int sg1 = min(p.n_seg, sg0 + p.segs_per_chunk);
            MESW_PROF(dq = clock64();)
            mbar_wait(&S.cfull[sc], pc);
            MESW_PROF(dprof[0] += clock64() - dq;)
            const uint8_t* cst = ring + p.co + (size_t)sc * p.cbytes;
            // this group's jobs in the chunk: (q, k-half) for q = q_first, q_first + n_dq, ...
            // Jobs go in batches of up to kDqBatch (distinct slots of the group's sub-ring): each
            // job is expanded and stored to TMEM, then ONE tcgen05.wait::st + fence covers the
            // batch before its slots are published -- the store-completion wait and the arrive
            // round trip were ~1/3 of a job's cycles when paid per job.
            // n_dq is 1 or 2: mask / shift, no integer division in the per-chunk bookkeeping
            const int q_first = sg0 + ((grp - (sg0 & dq_mask)) & dq_mask);
            const int n_jobs = (q_first < sg1 ? ((sg1 - 1 - q_first) >> dq_shift) + 1 : 0) * kJobHalves;
            for (int j0 = 0, nb = 0; j0 < n_jobs; j0 += nb) {
              nb = min(min(kDqBatch, n_jobs - j0), na);  // distinct slots only
              int slots[kDqBatch];
#pragma unroll
              for (int b = 0; b < kDqBatch; ++b) {
                if (b < nb) {
                  const int j = j0 + b;
                  const int q = q_first + (j / kJobHalves) * n_dq, jh = j % kJobHalves;
                  const int aslot = ab + pos;
                  slots[b] = aslot;
                  constexpr int KH = 2 / kJobHalves;  // k-halves per job
                  uint32_t cw[KH * WPK];
                  const uint8_t* cb = cst + (size_t)(q - sg0) * CB;
#pragma unroll
                  for (int kk = 0; kk < KH; ++kk)
#pragma unroll
                    for (int v = 0; v < CHB / 16; ++v) {
                      const uint4 t4 = lds128(cb + ((size_t)(jh * KH + kk) * 128 + mrow) * CHB + v * 16);
                      const int w0 = kk * WPK + 4 * v;
                      cw[w0] = t4.x; cw[w0 + 1] = t4.y; cw[w0 + 2] = t4.z; cw[w0 + 3] = t4.w;
                    }
                  MESW_PROF(const bool jst = p.tbuf && blockIdx.x == 0 && threadIdx.x == kDqWarp0 * 32 + grp * 128 && dprof[7] < 32;)
                  MESW_PROF(if (jst) p.tbuf[4096 * 56 + 512 + 256 + grp * 128 + 4 * dprof[7]] = clock64();)
                  MESW_PROF(dq = clock64();)
                  if (use > 0) mbar_wait(&S.aempty[aslot], (uint32_t)((use - 1) & 1));
                  MESW_PROF(if (jst) p.tbuf[4096 * 56 + 512 + 256 + grp * 128 + 4 * dprof[7] + 1] = clock64();)
                  MESW_PROF(dprof[1] += clock64() - dq;)
                  MESW_PROF(dq = clock64();)
                  const uint32_t a0 = tbase + (uint32_t)(p.a_col0 + aslot * kAColsPerSlot);
#ifndef MESW_EXP_NODQ
#pragma unroll
                  for (int kk = 0; kk < KH; ++kk) {
                    uint32_t r[32];
                    if (OFF) dequant_chunk2_offset(&cw[kk * WPK], r);
                    else dequant_chunk<DB>(&cw[kk * WPK], r);
                    tmem_st32(a0 + lane_addr + 32 * kk, r);
                  }
#endif
                  if (++pos == na) { pos = 0; ++use; }
                  MESW_PROF(dprof[2] += clock64() - dq;)
                  MESW_PROF(if (jst) p.tbuf[4096 * 56 + 512 + 256 + grp * 128 + 4 * dprof[7] + 2] = clock64();)
                  MESW_PROF(dprof[7]++;)
                }
              }
              MESW_PROF(dq = clock64();)
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {  // the group's 4 warps of each CTA -> leader's afull (8 arrivals per slot)
#pragma unroll
                for (int b = 0; b < kDqBatch; ++b)
                  if (b < nb) {
                    if (rank == 0) mbar_arrive(&S.afull[slots[b]]);
                    else mbar_arrive_cta_relaxed(&S.afull[slots[b]], 0);
                  }
              }
              MESW_PROF(dprof[3] += clock64() - dq;)
            }
            mbar_arrive(&S.cempty[sc]);  // every thread: release orders its own smem reads
            if (++sc == p.nc) { sc = 0; pc ^= 1; }
            MESW_PROF(if (p.tbuf && blockIdx.x == 0 && threadIdx.x == kDqWarp0 * 32 + grp * 128 && dcount < 64) p.tbuf[4096 * 56 + 128 + grp * 64 + dcount] = clock64();)
            MESW_PROF(++dcount;)
          }
        }
      }
    }
    MESW_PROF(dprof[6] = clock64() - dstart;)
    MESW_PROF(if (p.tbuf && quarter == 0 && lane == 0) for (int i = 0; i < 8; ++i) p.tbuf[4096 * 24 + (size_t)blockIdx.x * 16 + grp * 8 + i] = dprof[i];)
  } else {
    // ===================== epilogue warpgroup (own column group) =====================
    pdl_wait();  // reads x / residual, writes y / workspace: previous kernel must be complete
    const int quarter = warp & 3;
    const int mrow = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const int gtid = (warp - kEpiWarp0) * 32 + lane;  // 0..127
    const int cgp_first = (int)(u0 / p.n_ks);
    int ab = 0;
    int acc_use[2] = {0, 0};
    for (int pi = 0; pi < po.np; ++pi) {
      long long u, piece_end;
      po.bounds(pi, u, piece_end);
      const int cgp = po.cg_of(pi);
      const int cg = 2 * cgp + (int)rank;
      const long long cg_end = (long long)(cgp + 1) * p.n_ks;
#ifdef MESW_EXP_NORED
      const bool whole = true;  // experiment: no stream-K reduction (wrong sums; bounds the tail cost)
#else
      const bool whole = (u == (long long)cgp * p.n_ks) && (piece_end == cg_end);
#endif
      const bool fast = gather_salient_x(p, S, cg, gtid);
      if (OFF) {  // offset-code bias of each token over this piece's k-steps (table: 4 B / token / k-step)
        const int ks0 = (int)(u - (long long)cgp * p.n_ks), ks1 = (int)(piece_end - (long long)cgp * p.n_ks);
        for (int t = gtid; t < NP; t += 128) {
          const float* row = p.x_corr + (size_t)t * p.x_corr_ld;
          float acc = 0.f;
#pragma unroll 8
          for (int ks = ks0; ks < ks1; ++ks) acc += __ldg(row + ks);  // loads batched, adds in order
          S.corr[t] = acc;
        }
        named_bar_sync(1, 128);
      }
      EpiPre pre;
      epi_prefetch<YMAP, HALF>(p, S, cg, mrow, 0, fast, pre, whole);
      mbar_wait_sleep(&S.accfull[ab], (uint32_t)(acc_use[ab] & 1));
      tc_fence_after();
      if (gtid == 0 && pi == po.np - 1) MESW_STAMP(5);
      const uint32_t acc = tbase + lane_addr + (uint32_t)(ab * (NP + p.NPD));
      if (whole) {
        for (int t0 = 0; t0 < NP; t0 += 16) {
          float vb[16], vd[16];
          if (has_w) {
            tmem_ld8(acc + (uint32_t)(t0 / 2), vb);           // rows t0..t0+7 (first half)
            tmem_ld8(acc + (uint32_t)(HP + t0 / 2), vb + 8);  // rows t0+8..t0+15 (second half)
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) vb[i] = 0.f;  // delta-only: D_base never written
          }
          load_delta16<HALF>(S, acc, NP, t0, vd);
          if (OFF) {
#pragma unroll
            for (int i = 0; i < 16; ++i) vd[i] -= S.corr[t0 + i];  // offset-code bias (0 on padding rows)
          }
          epi_store16<YMAP, HALF>(p, S, cg, mrow, t0, vb, vd, fast, pre);
          if (t0 + 16 < NP) epi_prefetch<YMAP, HALF>(p, S, cg, mrow, t0 + 16, fast, pre);
        }
      } else {
        // stream-K partial: base + s_j * delta per row (natural row order, [NP][128] f32);
        // the salient term, residual and activation are applied once, by the final reducer
        const int slot = 2 * c + (cgp == cgp_first ? 0 : 1);
        const size_t slot_floats = (size_t)NP * kUnitN;
        float* mine = p.ws + (size_t)slot * slot_floats;
        for (int t0 = 0; t0 < NP; t0 += 16) {
          float vb[16], vd[16];
          if (has_w) {
            tmem_ld8(acc + (uint32_t)(t0 / 2), vb);
            tmem_ld8(acc + (uint32_t)(HP + t0 / 2), vb + 8);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) vb[i] = 0.f;
          }
          if (pre.sg[0] >= 0 || pre.sg[1] >= 0) {
            load_delta16<HALF>(S, acc, NP, t0, vd);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (pre.sg[i >> 3] >= 0 && S.tok2seg[t0 + i] == pre.sg[i >> 3])
                vb[i] = fmaf(pre.sj[i >> 3], OFF ? vd[i] - S.corr[t0 + i] : vd[i], vb[i]);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcg(mine + (size_t)(t0 + i) * kUnitN + mrow, vb[i]);
          if (t0 + 16 < NP) epi_prefetch<YMAP, HALF>(p, S, cg, mrow, t0 + 16, fast, pre, false);
        }
      }
      // accumulators consumed -> the leader may reuse this buffer
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&S.accempty[ab]);
        else mbar_arrive_cta(&S.accempty[ab], 0);
      }
      if (gtid == 0 && pi == po.np - 1) MESW_STAMP(6);
      acc_use[ab]++;
      if (p.n_acc == 2) ab ^= 1;
      if (whole && p.swiglu_I) swiglu_final<128>(p, S, cg, gtid);
      if (!whole) {
        named_bar_sync(1, 128);  // the partial stores above happen-before gtid 0's release
        // contributors to this column group: the pairs owning its first/last unit
        const long long first_u = (long long)cgp * p.n_ks, last_u = first_u + p.n_ks - 1;
        const int p_first = unit_owner(first_u, T2, (int)G2), p_last = unit_owner(last_u, T2, (int)G2);
        if (gtid == 0) {
          if (pi == po.np - 1) MESW_STAMP2(0);
          // acq_rel: releases this CTA's partials (ordered by the barrier) and, for the last
          // arriver, acquires every other contributor's (their release increments)
          const int prev = atom_add_acq_rel_gpu(&p.counters[cg], 1);
          if (pi == po.np - 1) MESW_STAMP2(1);
          S.flag = (prev == p_last - p_first) ? 1 : 0;
        }
        named_bar_sync(1, 128);
        if (S.flag) {
          if (pi == po.np - 1) {
            // final piece: handed to all 16 warps of the CTA after the role loops (their
            // chunks reduce in parallel: the tail of the launch is one L2 round trip deep)
            if (gtid == 0) {
              S.fin.cg = cg; S.fin.cgp = cgp; S.fin.p_first = p_first; S.fin.p_last = p_last;
              S.fin.fast = fast ? 1 : 0; S.fin.on = 1;
            }
          } else {
            for (int t0 = 0; t0 < NP; t0 += 16) {
              EpiPre pre;
              epi_prefetch<YMAP, HALF>(p, S, cg, mrow, t0, fast, pre);
              reduce_chunk<YMAP, HALF>(p, S, cg, cgp, (int)rank, mrow, t0, p_first, p_last, fast, pre, nullptr);
            }
            if (gtid == 0) p.counters[cg] = 0;  // self-reset for the next launch
            if (p.swiglu_I) swiglu_final<128>(p, S, cg, gtid);
          }
        }
      }
      named_bar_sync(1, 128);  // xsal / flag reuse by the next piece
      if (gtid == 0 && pi == po.np - 1) MESW_STAMP(7);
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) MESW_STAMP(1);
  if (threadIdx.x == kEpiWarp0 * 32) MESW_STAMP2(2);
  if (S.fin.on) {  // this CTA is the last contributor of its final column group (acquired above)
    if (threadIdx.x == 0) MESW_STAMP(2);
    const int fcg = S.fin.cg, fcgp = S.fin.cgp, pf = S.fin.p_first, pl = S.fin.p_last;
    const bool ffast = S.fin.fast != 0;
    const int fm = threadIdx.x % kUnitN;
    // Contributor slots are bulk-copied into the (now idle) smem ring in batches and summed,
    // in contributor order, into region 0 -- one L2 round trip per batch however many pairs
    // share the column group (small linears split a column group over many pairs).
    const size_t slot_floats = (size_t)NP * kUnitN, slot_bytes = slot_floats * sizeof(float);
    const int nC = pl - pf + 1;
    const int nbuf = (int)((size_t)p.ring_bytes / slot_bytes);
    // few contributors: every thread loads its 16 x nC partial values straight from L2 (one
    // round trip); many (small linears split a column group over many pairs): bulk-copy
    // batches into the idle smem ring
    const bool staged = nC > MESW_STAGE_MIN && (nbuf >= 2 || nC == 1);
    float* st = reinterpret_cast<float*>(ring);
    const int t_first = 16 * (threadIdx.x / kUnitN);
    EpiPre pre0;
    if (t_first < NP) epi_prefetch<YMAP, HALF>(p, S, fcg, fm, t_first, ffast, pre0);  // in flight with the copies
    MESW_PROF(long long fp[4] = {0, 0, 0, 0}; long long fq = clock64();)
    if (staged) {
      const long long T2 = p.T, G2 = p.G / 2;
      uint32_t ph = 0;
      for (int done = 0; done < nC;) {
        const int region0 = done == 0 ? 0 : 1;
        const int cnt = min(nC - done, nbuf - region0);
        if (threadIdx.x == 0) {
          // generic-proxy partials (global) and the smem the previous batch was read from ->
          // async-proxy (bulk copy) accesses
          asm volatile("fence.proxy.async.global;" ::: "memory");
          fence_proxy_async();
          mbar_arrive_expect_tx(&S.finbar, (uint32_t)(cnt * slot_bytes));
          for (int i = 0; i < cnt; ++i) {
            const int pp = pf + done + i;
            const long long pu0 = (long long)pp * T2 / G2;
            const int s2 = 2 * (2 * pp + (int)rank) + ((int)(pu0 / p.n_ks) == fcgp ? 0 : 1);
            bulk_g2s(ring + (size_t)(region0 + i) * slot_bytes, p.ws + (size_t)s2 * slot_floats, (uint32_t)slot_bytes,
                     &S.finbar);
          }
        }
        mbar_wait(&S.finbar, ph);
        if (threadIdx.x == 0 && done == 0) MESW_STAMP2(3);
        ph ^= 1;
        if (nC <= nbuf) break;  // all slots resident: summed in contributor order by reduce_chunk
        for (int i = 1; i < region0 + cnt; ++i)
          for (size_t e = threadIdx.x; e < slot_floats; e += kThreads) st[e] += st[(size_t)i * slot_floats + e];
        __syncthreads();
        done += cnt;
      }
    }
    MESW_PROF(fp[1] += clock64() - fq; fq = clock64();)
    if (threadIdx.x == 0) MESW_STAMP2(4);
#ifdef MESW_EXP_WARM
    for (int pass = 0; pass < 2; ++pass) {  // diagnostic: pass 0 runs the same code without stores
      const bool dry = pass == 0;
      if (pass == 1 && threadIdx.x == 0) MESW_STAMP2(7);
#else
    {
      const bool dry = false;
#endif
    for (int t0 = t_first; t0 < NP; t0 += 16 * (kThreads / kUnitN)) {
      EpiPre pre;
      if (t0 == t_first) pre = pre0;
      else epi_prefetch<YMAP, HALF>(p, S, fcg, fm, t0, ffast, pre);
      if (staged) reduce_chunk<YMAP, HALF>(p, S, fcg, fcgp, (int)rank, fm, t0, pf, nC <= nbuf ? pl : pf, ffast, pre, st, dry);
      else reduce_chunk<YMAP, HALF>(p, S, fcg, fcgp, (int)rank, fm, t0, pf, pl, ffast, pre, nullptr, dry);
      MESW_PROF(fp[2] += clock64() - fq; fq = clock64();)
    }
    }
    MESW_PROF(fp[3] = staged ? nC : -nC;)
    MESW_PROF(if (p.tbuf && threadIdx.x == 0) for (int i = 0; i < 4; ++i) p.tbuf[4096 * 40 + (size_t)blockIdx.x * 16 + i] = fp[i];)
    if (threadIdx.x == 0) p.counters[S.fin.cg] = 0;
    if (p.swiglu_I) swiglu_final<kThreads>(p, S, fcg, threadIdx.x);
    if (threadIdx.x == 0) MESW_STAMP(4);
  }
  if (threadIdx.x == 0) MESW_STAMP2(5);
  cluster_sync_all();  // the peer's MMAs / TMEM reads are complete before deallocation
  if (threadIdx.x == 0) MESW_STAMP2(6);
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
  }
}

template <int DB, bool OFF, bool YMAP, bool HALF>
int launch(const LinearParams& p, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(me_linear_tc_kernel<DB, OFF, YMAP, HALF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448);
    if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // CTA pairs for cta_group::2
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = mesw_pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, me_linear_tc_kernel<DB, OFF, YMAP, HALF>, p);
  if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
  return mesw_check_launch("me_linear");
}

}  // namespace mesw

using namespace mesw;

static int pad16(int v) { return (v + 15) & ~15; }

static unsigned long long* g_tbuf = nullptr;

// Debug: copy the last MESW_TIMING launch's per-CTA globaltimer stamps (8 per CTA).
extern "C" int mesw_debug_timing_copy(unsigned long long* h_out, int n_ctas) {
  if (!g_tbuf) return mesw_fail(MESW_ERR_VALUE, "no timing buffer (set MESW_TIMING)");
  cudaError_t e = cudaMemcpy(h_out, g_tbuf, (size_t)60 * 4096 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
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
    if (a->seg_begin[s] % 8)
      return mesw_fail(MESW_ERR_VALUE, "segment begins must be multiples of 8 rows (pad expert groups)");
    prev_end = a->seg_end[s];
  }
  int sms = mesw_device_sm_count();
  if (sms <= 0) return mesw_fail(MESW_ERR_CUDA, "no CUDA device");

  LinearParams p{};
  p.x = a->x; p.B = a->B; p.NP = pad16(a->B); p.m = a->m; p.n = a->n;
  p.n_cg = ((n_pad + 2 * kUnitN - 1) / (2 * kUnitN)) * 2; p.n_ks = m_pad / kUnitK;
  p.w = reinterpret_cast<const uint8_t*>(a->w);
  p.table = a->expert_table;
  p.n_seg = a->n_segments;
  p.NPD = 0;
  for (int s = 0; s < p.n_seg; ++s) {
    p.seg_begin[s] = a->seg_begin[s]; p.seg_end[s] = a->seg_end[s]; p.seg_slot[s] = a->seg_slot[s];
    p.seg_dcol[s] = p.NPD;
    p.NPD += 16 * (((a->seg_end[s] - 1) >> 4) - (a->seg_begin[s] >> 4) + 1);
  }
  p.y = a->y; p.y_bf16 = a->y_bf16; p.ldy = a->ldy;
  p.y_rows = a->y_rows;
  p.residual = a->residual; p.ld_res = a->ld_res;
  p.ws = reinterpret_cast<float*>(a->workspace);
  p.counters = a->counters;
  if (p.n_cg % 2) return mesw_fail(MESW_ERR_VALUE, "device buffers must cover an even number of 128-column groups");
  p.T = (long long)(p.n_cg / 2) * p.n_ks;  // pair units (2 column groups x 1 k-step)
  p.activation = a->activation;
  p.x_corr = (a->n_segments > 0 && a->code_bits == 2) ? a->x_corr : nullptr;
  p.x_corr_ld = a->x_corr_ld;
  p.swiglu_I = a->swiglu_I;
  if (p.swiglu_I) {
    if (p.swiglu_I < 0 || p.swiglu_I % kUnitN || 2 * p.swiglu_I != a->n || !a->y_bf16 || a->y_rows || !a->act ||
        a->act_np < p.NP || a->act_np % 16 || (a->act_corr && a->act_corr_ld < p.swiglu_I / kUnitN) ||
        a->residual || a->activation)
      return mesw_fail(MESW_ERR_VALUE, "swiglu epilogue: n = 2 I (I % 128 == 0), bf16 y without row map / "
                                       "residual / activation, act with >= canonical rows");
    p.act = a->act; p.act_np = a->act_np; p.act_corr = a->act_corr; p.act_corr_ld = a->act_corr_ld;
  }
  if (p.x_corr && p.x_corr_ld < p.n_ks)
    return mesw_fail(MESW_ERR_VALUE, "x_corr_ld must cover the k-steps of the linear");
  {
    static const char* e = getenv("MESW_DBG");  // experiment knobs: read once per process
    p.dbg = e ? atoi(e) : 0;
    static const bool timing = getenv("MESW_TIMING") != nullptr;
    if (timing) {
      if (!g_tbuf) cudaMalloc(&g_tbuf, 60 * 4096 * sizeof(unsigned long long)); cudaMemset(g_tbuf, 0, 60 * 4096 * 8);
      p.tbuf = g_tbuf;
    }
  }
  // n_cg here = column groups of the device buffers (a->n_alloc); pairs of CTAs (clusters of 2)
  const int want = (a->num_ctas > 0 ? a->num_ctas : sms) / 2;
  p.G = 2 * (int)((long long)(want > 0 ? want : 1) < p.T ? (want > 0 ? want : 1) : p.T);
  if (a->workspace_bytes < mesw_linear_workspace_bytes(a->B, p.G) || !a->workspace || !a->counters)
    return mesw_fail(MESW_ERR_VALUE, "workspace too small");

  // Shared-memory rings: x tiles (NP rows x 256 B), weight tiles (32 KiB), code chunks
  const int db = a->n_segments > 0 ? a->code_bits : 2;
  const int CB = kUnitN * kUnitK * db / 8;
  const int max_chunk = (db == 2 ? 4 : (db == 4 ? 2 : 1)) * kDqGroups;  // jobs per code chunk
  p.segs_per_chunk = p.n_seg == 0 ? 1 : (p.n_seg < max_chunk ? p.n_seg : max_chunk);
  p.n_chunks = p.n_seg == 0 ? 0 : (p.n_seg + p.segs_per_chunk - 1) / p.segs_per_chunk;
  p.xbytes = (p.NP / 2) * kUnitK * 2;  // this CTA's half of the activation tile
  p.cbytes = p.segs_per_chunk * CB;
  const size_t budget = 232448 - ring_offset();
  // ring depths: prefer (x 3, codes 3, weights >= 3); shrink x/codes first when rows are many
  // Ring depths: activations and codes 3 units ahead (their own producer thread), the
  // weight ring gets the rest of shared memory (its producer streams independently).
  // Ring depths: the producer walks all rings in unit order, so they share one lookahead D
  // (units), the largest that fits (<= kMaxStages, codes ring <= kMaxCStages chunks).
  for (;;) {
    const size_t per_unit = (a->w ? (size_t)kUnitWBytes : 0) + (size_t)p.xbytes + (size_t)p.n_chunks * p.cbytes;
    int D = (int)((budget - 1024) / per_unit);
    if (D > kMaxStages) D = kMaxStages;
    if (p.n_chunks > 0 && D * p.n_chunks > kMaxCStages) D = kMaxCStages / p.n_chunks;
    if (D >= 2) {
      p.nx = D;
      p.nw = a->w ? D : 0;
      p.nc = D * p.n_chunks;
      break;
    }
    {  // code-heavy launches: two units of weights / activations, the code ring gets the rest
      const size_t wx = 2 * ((a->w ? (size_t)kUnitWBytes : 0) + (size_t)p.xbytes) + 1024;
      const int nc = budget > wx ? (int)std::min<size_t>(kMaxCStages, (budget - wx) / p.cbytes) : 0;
      if (nc >= 2) {
        p.nx = 2;
        p.nw = a->w ? 2 : 0;
        p.nc = nc;
        break;
      }
    }
    if (p.segs_per_chunk <= kDqGroups) return mesw_fail(MESW_ERR_UNSUPPORTED, "shared memory: fewer than 2 stages");
    p.segs_per_chunk = (p.segs_per_chunk / 2 + kDqGroups - 1) / kDqGroups * kDqGroups;  // smaller chunks
    p.n_chunks = (p.n_seg + p.segs_per_chunk - 1) / p.segs_per_chunk;
    p.cbytes = p.segs_per_chunk * CB;
  }
  p.xo = 0;
  p.co = p.nx * p.xbytes;
  p.wo = (p.co + p.nc * p.cbytes + 1023) & ~1023;
  size_t smem = ring_offset() + (size_t)p.wo + (size_t)p.nw * kUnitWBytes;
  if (smem > 232448) return mesw_fail(MESW_ERR_UNSUPPORTED, "shared memory overflow");
  smem = 232448;  // one CTA per SM regardless: the slack stages the final stream-K reduction
  p.ring_bytes = (int)(smem - ring_offset());
  // TMEM: n_acc buffers of [D_base NP | D_delta NP] columns, then the A ring (64-col job slots).
  // Issuers: the base tile on warp role 0 (when there is a base), then n_dq <= 2 delta issuers;
  // segment q goes to delta issuer q % n_dq, fed by dequant group q % n_dq.  Each delta
  // issuer owns an A sub-ring of >= 1 slot (slots split by job count); prefer two
  // accumulator buffers, then more delta issuers.
  {
    static const int env_iss = getenv("MESW_ISS") ? atoi(getenv("MESW_ISS")) : 0;  // cap on delta issuers
    static const int nacc_max = getenv("MESW_NACC") ? atoi(getenv("MESW_NACC")) : 2;
    static const int env_maxslots = getenv("MESW_MAXSLOTS") ? atoi(getenv("MESW_MAXSLOTS")) : 0;
    int nd_max = std::min(p.n_seg, kDqGroups);
    if (env_iss > 0) nd_max = std::min(nd_max, env_iss);
    const int r0 = p.w ? 1 : 0;
    bool done = false;
    for (int n_acc = nacc_max; n_acc >= 1 && !done; --n_acc) {
      for (int nd = nd_max; nd >= (p.n_seg > 0 ? 1 : 0) && !done; --nd) {
        const int cols = kTmemCols - n_acc * (p.NP + p.NPD);
        int slots = cols / kAColsPerSlot;
        if (slots > kMaxASlots) slots = kMaxASlots;
        if (env_maxslots > 0 && slots > env_maxslots) slots = env_maxslots;
        if (cols < 0 || slots < nd) continue;
        for (int i = 0; i < 3; ++i) { p.a_base[i] = 0; p.a_na[i] = 0; }
        int jobs[2] = {0, 0};
        for (int q = 0; q < p.n_seg; ++q) jobs[q % nd]++;
        for (int g = 0; g < nd; ++g) p.a_na[r0 + g] = 1;
        for (int left = slots - nd; left > 0; --left) {  // next slot to the issuer with most jobs per slot
          int best = 0;
          for (int g = 1; g < nd; ++g)
            if (jobs[g] * p.a_na[r0 + best] > jobs[best] * p.a_na[r0 + g]) best = g;
          p.a_na[r0 + best]++;
        }
        int base = 0;
        for (int i = 0; i < 3; ++i) { p.a_base[i] = base; base += p.a_na[i]; }
        p.n_acc = n_acc;
        p.n_dq = nd;
        p.n_iss = std::max(1, r0 + nd);
        p.n_aslots = base;
        p.a_col0 = kTmemCols - base * kAColsPerSlot;
        done = true;
      }
    }
    if (!done) return mesw_fail(MESW_ERR_UNSUPPORTED, "tensor memory: too many rows for the A ring");
  }

  bool half = false;
  for (int q = 0; q < p.n_seg; ++q) half |= (p.seg_begin[q] % 16) != 0;
  cudaStream_t s = (cudaStream_t)stream;
  switch (db) {
    // (kernels with YMAP read the identity map when y_rows is NULL; HALF: a segment begins on
    // the second half of a window -- both are template parameters because the epilogue is the
    // latency-critical tail of every launch)
    case 2:
      if (p.x_corr) {
        if (p.y_rows) return half ? launch<2, true, true, true>(p, smem, s) : launch<2, true, true, false>(p, smem, s);
        return half ? launch<2, true, false, true>(p, smem, s) : launch<2, true, false, false>(p, smem, s);
      }
      return launch<2, false, true, true>(p, smem, s);
    case 4: return launch<4, false, true, true>(p, smem, s);
    default: return launch<8, false, true, true>(p, smem, s);
  }
}
