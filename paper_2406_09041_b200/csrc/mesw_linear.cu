// K2: fused segmented multi-expert linear for decode (sm_100a).
//
//   y[t, j] = sum_i x[t,i] W[i,j]
//           + s_e[j] * sum_{i not in S_e} x[t,i] q_e[i,j] + sum_{i in S_e} x[t,i] half(R_e)[i,j]
//   with e = expert(t)   (Eq. 4; toylm.py:183-186)
//
// Structure (one persistent CTA per SM, 8 consumer warps + 1 producer warp):
//  * Work is the list of units (column group cg of 128 outputs, k-step ks of 128
//    inputs), cg-major.  CTA c owns the contiguous range [c*T/G, (c+1)*T/G), so
//    every CTA streams the same number of bytes (stream-K); column groups cut by
//    a range boundary are reduced by the last-arriving CTA in fixed k order.
//  * The producer warp streams each unit's base-weight fragments (32 KiB), each
//    active expert's packed codes (4 KiB at 2 bits) and the x slab through a ring
//    of shared-memory stages with cp.async.bulk (TMA bulk engine) + mbarriers.
//  * Consumer warp w owns output tile w (16 columns) of the group.  Codes are
//    dequantised in registers (lop3 magic-number trick -> bf16 exact integers)
//    straight into mma.m16n8k16 A fragments; tokens are the N=8 dimension.
//    Base and delta accumulate in separate f32 fragments; the per-expert step,
//    salient fp16 correction, residual and dtype conversion are fused into the
//    epilogue.  Reduction order per (token, column) is fixed by the shape only,
//    so results are bit-identical under any batch composition.

#include "mesw_common.cuh"
#include "mesw_host.h"

namespace mesw {

constexpr int kXStride = kTileK + 8;  // bf16 elements per x row in smem (272 B, conflict-free)
constexpr int kMaxSegsPerStage = 16;

struct SegDesc {
  const uint8_t* codes;
  const float* steps;
  const int32_t* sal_off;
  const int32_t* sal_idx;
  const uint16_t* sal_rows;
  int begin, end;
};

struct LinearParams {
  const uint16_t* x;
  int B, m, n, ldx;
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
  int n_stages, stage_bytes, codes_off, x_off, segs_per_stage, n_chunks;
};

// ---------------------------------------------------------------- dequant
// Returns the 4 bf16x2 A-fragment registers of k-block kb holding q = d - OFF.
template <int DB>
__device__ __forceinline__ void dequant_kb(const uint32_t* cw, int kb, uint32_t* a);

template <>
__device__ __forceinline__ void dequant_kb<2>(const uint32_t* cw, int kb, uint32_t* a) {
  // pair p = kb*4+reg at bits 2*(p%8) (lo) / 16+2*(p%8) (hi) of word p/8.
  // (mask | 0x4300) is the bf16 128 + u*2^pos; fma rescales and subtracts 128*2^-pos + 2.
  const uint32_t w = (kb & 1) ? (cw[kb >> 1] >> 8) : cw[kb >> 1];
  a[0] = bf16x2_fma(lop3_and_or(w, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);   // x1  -130
  a[1] = bf16x2_fma(lop3_and_or(w, 0x000C000Cu, 0x43004300u), 0x3E803E80u, 0xC208C208u);   // x1/4 -34
  a[2] = bf16x2_fma(lop3_and_or(w, 0x00300030u, 0x43004300u), 0x3D803D80u, 0xC120C120u);   // x1/16 -10
  a[3] = bf16x2_fma(lop3_and_or(w >> 6, 0x00030003u, 0x43004300u), 0x3F803F80u, 0xC302C302u);
}

template <>
__device__ __forceinline__ void dequant_kb<4>(const uint32_t* cw, int kb, uint32_t* a) {
  // word kb, reg r: nibbles at bits 4r (lo) / 16+4r (hi); d = q + 8 -> 128+d - 136.
  const uint32_t w = cw[kb];
#pragma unroll
  for (int r = 0; r < 4; ++r)
    a[r] = bf16x2_fma(lop3_and_or(w >> (4 * r), 0x000F000Fu, 0x43004300u), 0x3F803F80u,
                      0xC308C308u);
}

template <>
__device__ __forceinline__ void dequant_kb<8>(const uint32_t* cw, int kb, uint32_t* a) {
  // words 2kb (regs 0,1) and 2kb+1 (regs 2,3); local r: bytes r (lo) / 2+r (hi); d = q + 128.
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t w = cw[2 * kb + (r >> 1)];
    const int sh = 8 * (r & 1);
    const float lo = __uint_as_float(0x4B000000u | ((w >> sh) & 0xFFu)) - 8388736.0f;
    const float hi = __uint_as_float(0x4B000000u | ((w >> (16 + sh)) & 0xFFu)) - 8388736.0f;
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    a[r] = d;
  }
}

// Owner CTA of unit u under the contiguous split [c*T/G, (c+1)*T/G).
__device__ __forceinline__ int unit_owner(long long u, long long T, int G) {
  return (int)(((u + 1) * (long long)G - 1) / T);
}

// ---------------------------------------------------------------- epilogue
template <int NT>
__device__ __forceinline__ void epilogue(const LinearParams& p, const SegDesc* segs,
                                         const int* tok2seg, int cg, int warp, int lane,
                                         const float (&accB)[NT][4], const float (&accD)[NT][4]) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int tok = nt * 8 + 2 * t + (i & 1);
      const int jl = warp * 16 + g + ((i & 2) ? 8 : 0);
      const int j = cg * kTileN + jl;
      if (tok >= p.B || j >= p.n) continue;
      float v = accB[nt][i];
      const int sg = tok2seg[tok];
      if (sg >= 0) {
        const SegDesc& sd = segs[sg];
        float d = sd.steps[j] * accD[nt][i];
        const int r0 = sd.sal_off[cg], r1 = sd.sal_off[cg + 1];
        const uint16_t* xrow = p.x + (size_t)tok * p.ldx;
        for (int r = r0; r < r1; ++r) {
          const float xv = bf16_to_f32(xrow[sd.sal_idx[r]]);
          const float rv = __half2float(__ushort_as_half(sd.sal_rows[(size_t)r * kTileN + jl]));
          d = fmaf(xv, rv, d);
        }
        v += d;
      }
      if (p.residual) v += bf16_to_f32(p.residual[(size_t)tok * p.ld_res + j]);
      if (p.activation == 1) v = fmaxf(v, 0.f);
      if (p.y_bf16)
        reinterpret_cast<__nv_bfloat16*>(p.y)[(size_t)tok * p.ldy + j] = __float2bfloat16_rn(v);
      else
        reinterpret_cast<float*>(p.y)[(size_t)tok * p.ldy + j] = v;
    }
  }
}

// ---------------------------------------------------------------- kernel
// NT: n-tiles of 8 tokens.  KSPLIT: consumer warps per 16-output tile (each takes
// 8/KSPLIT of the unit's 8 k-blocks); NACC: independent accumulator sets (k-block
// parity) to break the mma dependency chain when there is a single n-tile.
template <int NT>
struct Cfg {
  static constexpr int KSPLIT = NT <= 2 ? 2 : 1;
  static constexpr int NACC = NT == 1 ? 2 : 1;
  static constexpr int CW = kTilesPerCg * KSPLIT;  // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int KB2 = kKbPerKs / 2 / KSPLIT;  // k-block pairs per warp per unit
  static constexpr int XCHG = KSPLIT == 2 ? kTilesPerCg * NT * 32 * 8 * 4 : 0;
};

__host__ __device__ inline size_t header_bytes(int S, int NT, int xchg) {
  const size_t raw = (size_t)S * 16 + 16 + (size_t)NT * 8 * 4 + MESW_MAX_SEGMENTS * sizeof(SegDesc);
  return ((raw + 15) & ~size_t(15)) + xchg + 1023 & ~size_t(1023);
}

template <int NT>
__device__ __forceinline__ void load_x_frags(uint32_t (&b)[NT][4], const uint16_t* xl, int kb2) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
    ldmatrix_x4(b[nt][0], b[nt][1], b[nt][2], b[nt][3], xl + nt * 8 * kXStride + kb2 * 32);
}

template <int DB, int NT>
__global__ void __launch_bounds__(Cfg<NT>::THREADS, 1)
    me_linear_kernel(const __grid_constant__ LinearParams p) {
  using C = Cfg<NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int S = p.n_stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  int* flag = reinterpret_cast<int*>(empty + S);
  int* tok2seg = flag + 4;                                       // [NT*8]
  SegDesc* segs = reinterpret_cast<SegDesc*>(tok2seg + NT * 8);  // [n_seg]
  const size_t raw = (size_t)S * 16 + 16 + (size_t)NT * 8 * 4 + MESW_MAX_SEGMENTS * sizeof(SegDesc);
  float* xchg = reinterpret_cast<float*>(smem + ((raw + 15) & ~size_t(15)));
  uint8_t* ring = smem + header_bytes(S, NT, C::XCHG);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const long long u0 = (long long)c * p.T / p.G, u1 = (long long)(c + 1) * p.T / p.G;
  constexpr int CB = kTileN * kTileK * DB / 8;  // code bytes per (cg, ks)
  constexpr int CBL = 8 * DB;                   // code bytes per lane per ks
  constexpr int CBW = CBL / C::KSPLIT;          // ... per warp-lane share

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C::CW);
    }
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < NT * 8; i += C::THREADS) tok2seg[i] = -1;
  __syncthreads();
  for (int q = threadIdx.x; q < p.n_seg; q += C::THREADS) {
    const mesw_expert_dev e = p.table[p.seg_slot[q]];
    SegDesc d;
    d.codes = reinterpret_cast<const uint8_t*>(e.codes);
    d.steps = e.steps;
    d.sal_off = e.sal_off;
    d.sal_idx = e.sal_idx;
    d.sal_rows = e.sal_rows;
    d.begin = p.seg_begin[q];
    d.end = p.seg_end[q];
    segs[q] = d;
    for (int t = d.begin; t < d.end; ++t) tok2seg[t] = q;
  }
  __syncthreads();

  if (warp == C::CW) {
    // ===================== producer warp =====================
    int s = 0;
    uint32_t ph = 0;
    bool first_pass = true;
    int ks = (int)(u0 % p.n_ks);
    for (long long u = u0; u < u1; ++u) {
      for (int ch = 0; ch < p.n_chunks; ++ch) {
        if (!first_pass) mbar_wait(&empty[s], ph ^ 1);
        const bool do_w = (p.w != nullptr) && ch == 0;
        const int sg0 = ch * p.segs_per_stage;
        const int sg1 = min(p.n_seg, sg0 + p.segs_per_stage);
        const uint32_t bytes = (do_w ? kWBytesPerUnit : 0) + (uint32_t)(max(0, sg1 - sg0)) * CB +
                               (uint32_t)p.B * (kTileK * 2);
        uint8_t* st = ring + (size_t)s * p.stage_bytes;
        if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
        __syncwarp();
        if (do_w && lane == 0)
          bulk_g2s(st, p.w + (size_t)u * kWBytesPerUnit, kWBytesPerUnit, &full[s]);
        for (int q = sg0 + lane; q < sg1; q += 32)
          bulk_g2s(st + p.codes_off + (size_t)(q - sg0) * CB, segs[q].codes + (size_t)u * CB, CB,
                   &full[s]);
        for (int r = lane; r < p.B; r += 32)
          bulk_g2s(st + p.x_off + (size_t)r * kXStride * 2,
                   p.x + (size_t)r * p.ldx + (size_t)ks * kTileK, kTileK * 2, &full[s]);
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; first_pass = false; }
      }
      if (++ks == p.n_ks) ks = 0;
    }
    return;
  }

  // ===================== consumer warps =====================
  const int tile = warp & (kTilesPerCg - 1);
  const int kh = warp / kTilesPerCg;  // k-split index
  float accB[C::NACC][NT][4], accD[C::NACC][NT][4];
  const int cg_first = (int)(u0 / p.n_ks);
  int cg = cg_first, ks = (int)(u0 % p.n_ks);
  int s = 0;
  uint32_t ph = 0;
  long long piece_start = u0;
  for (long long u = u0; u < u1; ++u) {
    if (u == u0 || ks == 0) {
      piece_start = u;
#pragma unroll
      for (int a = 0; a < C::NACC; ++a)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) accB[a][nt][i] = accD[a][nt][i] = 0.f;
    }
    for (int ch = 0; ch < p.n_chunks; ++ch) {
      mbar_wait(&full[s], ph);
      const uint8_t* st = ring + (size_t)s * p.stage_bytes;
      const uint16_t* xs = reinterpret_cast<const uint16_t*>(st + p.x_off);
      // ldmatrix row address for this lane: token row (lane&7), k offset (lane>>3)*8
      const uint16_t* xl = xs + (lane & 7) * kXStride + (lane >> 3) * 8;
      const int kb2_0 = kh * C::KB2;

      // x fragments of this warp's k-blocks (hoisted when they fit in registers)
      uint32_t bx[C::KSPLIT == 2 ? C::KB2 : 1][NT][4];
      if constexpr (C::KSPLIT == 2) {
#pragma unroll
        for (int j = 0; j < C::KB2; ++j) load_x_frags<NT>(bx[j], xl, kb2_0 + j);
      }

      if (p.w != nullptr && ch == 0) {
        const uint4* Ws = reinterpret_cast<const uint4*>(st) + (tile * kKbPerKs) * 32 + lane;
#pragma unroll
        for (int j = 0; j < C::KB2; ++j) {
          uint32_t bl[NT][4];
          if constexpr (C::KSPLIT != 2) load_x_frags<NT>(bl, xl, kb2_0 + j);
          const uint4 w0 = Ws[(2 * (kb2_0 + j)) * 32];
          const uint4 w1 = Ws[(2 * (kb2_0 + j) + 1) * 32];
          const uint32_t a0[4] = {w0.x, w0.y, w0.z, w0.w};
          const uint32_t a1[4] = {w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt * 8 < p.B) {
              const uint32_t* bb = C::KSPLIT == 2 ? bx[C::KSPLIT == 2 ? j : 0][nt] : bl[nt];
              mma_bf16(accB[0][nt], a0, bb[0], bb[1]);
              mma_bf16(accB[C::NACC - 1][nt], a1, bb[2], bb[3]);
            }
          }
        }
      }

      const int sg0 = ch * p.segs_per_stage;
      const int sg1 = min(p.n_seg, sg0 + p.segs_per_stage);
      for (int q = sg0; q < sg1; ++q) {
        const int sb = segs[q].begin, se = segs[q].end;
        const int lo_nt = sb >> 3, hi_nt = (se - 1) >> 3;
        uint32_t cw[CBL / 4];  // full-unit word array; this warp reads its share only
        const uint8_t* cl = st + p.codes_off + (size_t)(q - sg0) * CB +
                            (size_t)(tile * 32 + lane) * CBL + kh * CBW;
        if constexpr (CBW == 8) {
          const uint2 t2 = *reinterpret_cast<const uint2*>(cl);
          cw[kh * 2 + 0] = t2.x; cw[kh * 2 + 1] = t2.y;
        } else {
#pragma unroll
          for (int v = 0; v < CBW / 16; ++v) {
            const uint4 t4 = lds128(cl + v * 16);
            const int w0 = kh * (CBW / 4) + 4 * v;
            cw[w0 + 0] = t4.x; cw[w0 + 1] = t4.y; cw[w0 + 2] = t4.z; cw[w0 + 3] = t4.w;
          }
        }
        // lane's B-fragment token for each n-tile, and whether it belongs to this segment
        bool mine[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int tok = nt * 8 + (lane >> 2);
          mine[nt] = tok >= sb && tok < se;
        }
#pragma unroll
        for (int j = 0; j < C::KB2; ++j) {
          uint32_t bm[NT][4];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt >= lo_nt && nt <= hi_nt) {
              if constexpr (C::KSPLIT == 2) {
#pragma unroll
                for (int r = 0; r < 4; ++r) bm[nt][r] = mine[nt] ? bx[C::KSPLIT == 2 ? j : 0][nt][r] : 0u;
              } else {
                ldmatrix_x4(bm[nt][0], bm[nt][1], bm[nt][2], bm[nt][3],
                            xl + nt * 8 * kXStride + (kb2_0 + j) * 32);
                if (!mine[nt]) bm[nt][0] = bm[nt][1] = bm[nt][2] = bm[nt][3] = 0u;
              }
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t a[4];
            dequant_kb<DB>(cw, 2 * (kb2_0 + j) + h, a);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              if (nt >= lo_nt && nt <= hi_nt)
                mma_bf16(accD[h % C::NACC][nt], a, bm[nt][2 * h], bm[nt][2 * h + 1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }

    // ---- end of a piece: full column group, or a range boundary ----
    if (ks == p.n_ks - 1 || u == u1 - 1) {
      // fold accumulator sets (fixed order), then the k-split halves through smem
      if constexpr (C::NACC == 2) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            accB[0][nt][i] += accB[1][nt][i];
            accD[0][nt][i] += accD[1][nt][i];
          }
      }
      if constexpr (C::KSPLIT == 2) {
        float* xw = xchg + ((size_t)tile * NT * 32 + lane) * 8;
        if (kh == 1) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float4* d = reinterpret_cast<float4*>(xw + (size_t)nt * 32 * 8);
            d[0] = make_float4(accB[0][nt][0], accB[0][nt][1], accB[0][nt][2], accB[0][nt][3]);
            d[1] = make_float4(accD[0][nt][0], accD[0][nt][1], accD[0][nt][2], accD[0][nt][3]);
          }
        }
        named_bar_sync(1, C::CW * 32);
        if (kh == 0) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const float4* d = reinterpret_cast<const float4*>(xw + (size_t)nt * 32 * 8);
            const float4 vb = d[0], vd = d[1];
            accB[0][nt][0] += vb.x; accB[0][nt][1] += vb.y; accB[0][nt][2] += vb.z; accB[0][nt][3] += vb.w;
            accD[0][nt][0] += vd.x; accD[0][nt][1] += vd.y; accD[0][nt][2] += vd.z; accD[0][nt][3] += vd.w;
          }
        }
        named_bar_sync(1, C::CW * 32);
      }
      if (kh == 0) {
        const bool whole = (piece_start == (long long)cg * p.n_ks) && (ks == p.n_ks - 1);
        if (whole) {
          epilogue<NT>(p, segs, tok2seg, cg, tile, lane, accB[0], accD[0]);
        } else {
          const int slot = 2 * c + (cg == cg_first ? 0 : 1);
          const size_t slot_floats = (size_t)kTilesPerCg * NT * 32 * 8;
          float* mine = p.ws + (size_t)slot * slot_floats + ((size_t)tile * NT * 32 + lane) * 8;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float4* dst = reinterpret_cast<float4*>(mine + (size_t)nt * 32 * 8);
            __stcg(dst, make_float4(accB[0][nt][0], accB[0][nt][1], accB[0][nt][2], accB[0][nt][3]));
            __stcg(dst + 1, make_float4(accD[0][nt][0], accD[0][nt][1], accD[0][nt][2], accD[0][nt][3]));
          }
          __threadfence();
          named_bar_sync(2, kTilesPerCg * 32);
          const long long first_u = (long long)cg * p.n_ks, last_u = first_u + p.n_ks - 1;
          const int c_first = unit_owner(first_u, p.T, p.G), c_last = unit_owner(last_u, p.T, p.G);
          if (threadIdx.x == 0) {
            const int prev = atomicAdd(&p.counters[cg], 1);
            *flag = (prev == c_last - c_first) ? 1 : 0;
          }
          named_bar_sync(2, kTilesPerCg * 32);
          if (*flag) {
            __threadfence();
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
              for (int i = 0; i < 4; ++i) accB[0][nt][i] = accD[0][nt][i] = 0.f;
            for (int cc = c_first; cc <= c_last; ++cc) {
              const long long cu0 = (long long)cc * p.T / p.G;
              const int s2 = 2 * cc + ((int)(cu0 / p.n_ks) == cg ? 0 : 1);
              const float* src = p.ws + (size_t)s2 * slot_floats + ((size_t)tile * NT * 32 + lane) * 8;
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                const float4* sp = reinterpret_cast<const float4*>(src + (size_t)nt * 32 * 8);
                const float4 vb = __ldcg(sp), vd = __ldcg(sp + 1);
                accB[0][nt][0] += vb.x; accB[0][nt][1] += vb.y; accB[0][nt][2] += vb.z; accB[0][nt][3] += vb.w;
                accD[0][nt][0] += vd.x; accD[0][nt][1] += vd.y; accD[0][nt][2] += vd.z; accD[0][nt][3] += vd.w;
              }
            }
            epilogue<NT>(p, segs, tok2seg, cg, tile, lane, accB[0], accD[0]);
            if (threadIdx.x == 0) p.counters[cg] = 0;  // self-reset for the next launch
          }
          named_bar_sync(2, kTilesPerCg * 32);
        }
      }
    }
    if (++ks == p.n_ks) { ks = 0; ++cg; }
  }
}

template <int DB, int NT>
int launch(const LinearParams& p, size_t smem, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(me_linear_kernel<DB, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return mesw_fail(MESW_ERR_CUDA, cudaGetErrorString(e));
    configured = true;
  }
  me_linear_kernel<DB, NT><<<p.G, Cfg<NT>::THREADS, smem, stream>>>(p);
  return mesw_check_launch("me_linear");
}

template <int DB>
int launch_nt(const LinearParams& p, int nt, size_t smem, cudaStream_t s) {
  switch (nt) {
    case 1: return launch<DB, 1>(p, smem, s);
    case 2: return launch<DB, 2>(p, smem, s);
    case 4: return launch<DB, 4>(p, smem, s);
    default: return launch<DB, 8>(p, smem, s);
  }
}

static int xchg_bytes(int nt) {
  switch (nt) {
    case 1: return Cfg<1>::XCHG;
    case 2: return Cfg<2>::XCHG;
    case 4: return Cfg<4>::XCHG;
    default: return Cfg<8>::XCHG;
  }
}

}  // namespace mesw

using namespace mesw;

static int round_nt(int B) {
  const int nt = (B + 7) / 8;
  return nt <= 1 ? 1 : nt <= 2 ? 2 : nt <= 4 ? 4 : 8;
}

extern "C" uint64_t mesw_linear_workspace_bytes(int32_t B, int32_t num_ctas) {
  const int nt = round_nt(B < 1 ? 1 : B);
  return (uint64_t)num_ctas * 2ull * kTilesPerCg * nt * 32 * 8 * sizeof(float);
}

extern "C" int mesw_me_linear(const mesw_linear_args* a, void* stream) {
  if (!a) return mesw_fail(MESW_ERR_VALUE, "null args");
  if (a->B < 1 || a->B > 64) return mesw_fail(MESW_ERR_UNSUPPORTED, "decode linear supports 1 <= B <= 64 tokens");
  if (a->m < 1 || a->n < 1) return mesw_fail(MESW_ERR_VALUE, "empty linear");
  const int m_pad = (a->m + kTileK - 1) / kTileK * kTileK;
  const int n_pad = (a->n + kTileN - 1) / kTileN * kTileN;
  if (a->ldx < m_pad || a->ldx % 8) return mesw_fail(MESW_ERR_VALUE, "ldx must be >= m_pad and a multiple of 8");
  if (((uintptr_t)a->x) % 16 || ((uintptr_t)a->w) % 16) return mesw_fail(MESW_ERR_VALUE, "x / w must be 16-byte aligned");
  if (a->n_segments < 0 || a->n_segments > MESW_MAX_SEGMENTS) return mesw_fail(MESW_ERR_VALUE, "too many segments");
  if (a->n_segments > 0 && a->code_bits != 2 && a->code_bits != 4 && a->code_bits != 8)
    return mesw_fail(MESW_ERR_VALUE, "code_bits must be 2, 4 or 8");
  if (!a->w && a->n_segments == 0) return mesw_fail(MESW_ERR_VALUE, "nothing to compute (no base, no delta)");
  if (!a->y) return mesw_fail(MESW_ERR_VALUE, "null output");
  if (a->n_segments > 0 && !a->expert_table) return mesw_fail(MESW_ERR_VALUE, "null expert table");
  int prev_end = 0;
  for (int s = 0; s < a->n_segments; ++s) {
    if (a->seg_begin[s] < prev_end || a->seg_end[s] <= a->seg_begin[s] || a->seg_end[s] > a->B || a->seg_slot[s] < 0)
      return mesw_fail(MESW_ERR_VALUE, "segments must be non-empty, ascending, disjoint and inside [0, B)");
    prev_end = a->seg_end[s];
  }
  int sms = mesw_device_sm_count();
  if (sms <= 0) return mesw_fail(MESW_ERR_CUDA, "no CUDA device");

  LinearParams p{};
  p.x = a->x; p.B = a->B; p.m = a->m; p.n = a->n; p.ldx = a->ldx;
  p.n_cg = n_pad / kTileN; p.n_ks = m_pad / kTileK;
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
  const int want = a->num_ctas > 0 ? a->num_ctas : sms;
  p.G = (int)((long long)want < p.T ? want : p.T);
  const int nt = round_nt(a->B);
  if (a->workspace_bytes < mesw_linear_workspace_bytes(a->B, p.G) || !a->workspace || !a->counters)
    return mesw_fail(MESW_ERR_VALUE, "workspace too small");

  // Stage layout: [W 32 KiB][codes segs_per_stage x CB][x slab NT*8 rows x 272 B]
  const int db = a->n_segments > 0 ? a->code_bits : 2;
  const int CB = kTileN * kTileK * db / 8;
  const int xbytes = nt * 8 * kXStride * 2;
  const int wbytes = a->w ? kWBytesPerUnit : 0;
  const size_t hdr = header_bytes(6, nt, xchg_bytes(nt));  // upper bound (S <= 6)
  const size_t budget = 232448 - hdr;
  int segs_per_stage = p.n_seg == 0 ? 0 : (p.n_seg < kMaxSegsPerStage ? p.n_seg : kMaxSegsPerStage);
  int stage = 0, S = 0;
  for (;;) {
    stage = (wbytes + segs_per_stage * CB + xbytes + 127) / 128 * 128;
    S = (int)(budget / stage);
    if (S > 6) S = 6;
    if (S >= 3 || segs_per_stage <= 1) break;
    segs_per_stage = (segs_per_stage + 1) / 2;
  }
  if (S < 2) return mesw_fail(MESW_ERR_UNSUPPORTED, "stage does not fit shared memory");
  p.n_stages = S;
  p.stage_bytes = stage;
  p.codes_off = wbytes;
  p.x_off = wbytes + segs_per_stage * CB;
  p.segs_per_stage = segs_per_stage > 0 ? segs_per_stage : 1;
  p.n_chunks = p.n_seg == 0 ? 1 : (p.n_seg + p.segs_per_stage - 1) / p.segs_per_stage;
  const size_t smem = header_bytes(S, nt, xchg_bytes(nt)) + (size_t)S * stage;
  if (smem > 232448) return mesw_fail(MESW_ERR_UNSUPPORTED, "shared memory overflow");

  cudaStream_t s = (cudaStream_t)stream;
  switch (db) {
    case 2: return launch_nt<2>(p, nt, smem, s);
    case 4: return launch_nt<4>(p, nt, smem, s);
    default: return launch_nt<8>(p, nt, smem, s);
  }
}
