/*
 * mesw.h -- C ABI of the B200-native ME-Switch multi-expert serving hot path.
 *
 * The reference (arXiv 2406.09041, /root/reference/pkg/src/meswitch) is pure
 * Python/numpy and has no FFI of its own.  This header is the boundary the
 * reference would bind (ctypes) to move its hot path to
 * the GPU.  Each entry point names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "d_" pointers are CUDA device pointers,
 *    "h_" pointers are host pointers.  `stream` is a cudaStream_t (NULL = legacy
 *    default stream).
 *  - Every function returns a mesw_status.  No C++ exception crosses the ABI;
 *    mesw_last_error() returns a thread-local message for the last failure.
 *  - Matrix orientation follows the reference (numerics.py:1-8): a delta /
 *    weight is [m x n] with rows = INPUT channels, columns = OUTPUT channels,
 *    y = x . W.
 *
 * Device layouts: a linear with m inputs
 * and n outputs is padded to m_pad = ceil(m/128)*128, n_pad = ceil(n/256)*256
 * (column groups come in pairs: one tcgen05 cta_group::2 MMA covers two) and cut
 * into column groups (cg, 128 outputs) x k-steps (ks, 128 inputs), stored cg-major.
 *  - base weight  : bf16, one 32 KiB unit per (cg, ks) in the UMMA K-major
 *                   SWIZZLE_NONE canonical layout (8 x 16 B core matrices, LBO 128 B,
 *                   SBO 2048 B): one bulk copy lands a ready tcgen05 A operand
 *  - delta codes  : DB-bit device codes d = q + OFF (DB=2: b=2, OFF=2; DB=4:
 *                   b in {1,3,4}, OFF=8; DB=8: b=8, OFF=128), same unit order,
 *                   2048*DB bytes per unit: per (k-half, output channel) 8*DB
 *                   contiguous bytes in bf16x2-pair order;
 *                   salient input rows forced to d = OFF (q = 0), which keeps the fused
 *                   result equal to CompressedDelta.reconstruct() (compress.py:115-121)
 *  - steps        : f32 [n_pad]
 *  - salient      : per column group: sal_off[n_cg+1] (int32), sal_idx[] (int32 input
 *                   channel), sal_rows[][128] (binary16 bits of R restricted to the cg)
 */
#ifndef MESW_H_
#define MESW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MESW_OK = 0,
  MESW_ERR_BAD_MAGIC = 1,           /* errors.BadMagicError          (errors.py:23) */
  MESW_ERR_UNSUPPORTED_VERSION = 2, /* errors.UnsupportedVersionError(errors.py:27) */
  MESW_ERR_TRUNCATED = 3,           /* errors.TruncatedArtifactError (errors.py:31) */
  MESW_ERR_VALUE = 4,               /* ValueError (shape / range / bits)            */
  MESW_ERR_CUDA = 5,                /* CUDA runtime failure                          */
  MESW_ERR_UNSUPPORTED = 6,         /* valid input this build does not handle        */
  MESW_ERR_INDEX = 7                /* IndexError (salient index >= input channels)  */
} mesw_status;

#define MESW_TILE_N 128 /* outputs per column group  */
#define MESW_TILE_K 128 /* inputs per k-step         */
#define MESW_MAX_SEGMENTS 64

/* ---------------------------------------------------------------- misc */
int mesw_abi_version(void);
const char* mesw_last_error(void);
/* Number of SMs of the current device (grid sizing), or -1. */
int mesw_device_sm_count(void);
/* Programmatic dependent launch for every kernel of this library (default on): a
 * launch may begin -- prologue, weight / code prefetch -- while the previous kernel
 * in the stream drains; each kernel waits (griddepcontrol.wait) before touching
 * data a previous kernel produces or consumes.  Returns the previous setting.   */
int mesw_set_pdl(int enable);

/* --------------------------------------------- MESW container (host side)
 * Replaces compress.deserialize_artifact (compress.py:513-549): validates the
 * magic, version, every layer block and the absence of trailing bytes, and
 * returns byte offsets of each block's fields into `buf` (no copies).       */
typedef struct {
  uint32_t m, n, bits, k;
  uint64_t idx_off;   /* k x u32 salient input channels, ascending            */
  uint64_t rows_off;  /* k x n x u16 binary16 salient rows                     */
  uint64_t steps_off; /* n x f32 step sizes                                    */
  uint64_t codes_off; /* packed codes, column-major LSB-first (quant.py:172-213) */
  uint64_t codes_len;
} mesw_layer_view;

/* Parse the container header: manifest JSON at [*manifest_off, +*manifest_len). */
int mesw_parse_header(const uint8_t* h_buf, uint64_t len, uint64_t* manifest_off,
                      uint32_t* manifest_len);
/* Walk `layer_count` layer blocks starting at `first_off`; fills `views`. */
int mesw_parse_layers(const uint8_t* h_buf, uint64_t len, uint64_t first_off,
                      uint32_t layer_count, mesw_layer_view* views);
/* quant.packed_nbytes (quant.py:190-192). */
uint64_t mesw_packed_nbytes(uint32_t rows, uint32_t cols, uint32_t bits);
/* compress.layer_block_nbytes(...).total (compress.py:589-597). */
uint64_t mesw_layer_block_nbytes(uint32_t m, uint32_t n, uint32_t bits, uint32_t k);

/* ------------------------------------------------ device geometry / loader */
/* Device code width for a MESW bit width: 2 -> 2, {1,3,4} -> 4, 8 -> 8 (0 if invalid). */
int mesw_device_code_bits(uint32_t bits);
/* Bytes of the device code buffer / base weight buffer for a padded linear. */
uint64_t mesw_codes_device_bytes(uint32_t m_pad, uint32_t n_pad, uint32_t code_bits);
uint64_t mesw_weight_device_bytes(uint32_t m_pad, uint32_t n_pad);

/* K1: repack one MESW layer block's packed codes (already on the device,
 * d_packed = the raw column-major run bytes) into the device code layout of
 * a (possibly fused) linear, at output-column offset col_base (multiple of
 * 128).  Salient rows (d_sal_idx, ascending, k entries) are forced to q = 0.
 * Replaces the consumer side of quant.unpack_codes (quant.py:216-236).       */
int mesw_repack_codes(const uint8_t* d_packed, uint32_t m, uint32_t n, uint32_t bits,
                      const int32_t* d_sal_idx, uint32_t k, uint8_t* d_codes,
                      uint32_t m_pad, uint32_t n_total_pad, uint32_t col_base,
                      void* stream);

/* Repack a bf16 base weight into the canonical tile layout.  If `transposed` == 0 the
 * source is [m][ld] (reference orientation, rows = inputs); otherwise [n][ld]
 * (torch nn.Linear weight, rows = outputs).  Written at column offset col_base. */
int mesw_repack_weight(const uint16_t* d_src, uint32_t m, uint32_t n, uint32_t ld,
                       int transposed, uint16_t* d_w, uint32_t m_pad,
                       uint32_t n_total_pad, uint32_t col_base, void* stream);

/* Host helper: build the per-column-group salient tables of a fused linear from
 * its blocks.  Block b covers output columns [col_base[b], col_base[b]+n[b]),
 * has k[b] salient input channels h_idx[b][...] and rows h_rows[b] (k x n
 * binary16).  Call once with the out pointers NULL to get *total, then again.
 * Indices must be strictly ascending and < m (input channels); otherwise
 * MESW_ERR_INDEX (the reference's reconstruct() raises IndexError, compress.py:119-120). */
int mesw_build_salient_tables(uint32_t m, uint32_t n_blocks, const uint32_t* col_base, const uint32_t* n,
                              const uint32_t* k, const uint32_t* const* h_idx,
                              const uint16_t* const* h_rows, uint32_t n_total_pad,
                              int32_t* h_sal_off, int32_t* h_sal_idx, uint16_t* h_sal_rows,
                              uint64_t* total);

/* K6 debug: device codes -> int8 codes [m][n] (row-major, reference
 * orientation) of the block at col_base; bit-exact with quant.unpack_codes
 * except salient rows, which read 0 (compress.py:205-214 writes them as 0). */
int mesw_unpack_codes_debug(const uint8_t* d_codes, uint32_t code_bits, uint32_t m,
                            uint32_t n, uint32_t m_pad, uint32_t n_total_pad,
                            uint32_t col_base, int8_t* d_out, void* stream);
/* K6 debug: dense f32 [m][n] reconstruction = CompressedDelta.reconstruct(). */
int mesw_dequant_debug(const uint8_t* d_codes, uint32_t code_bits, const float* d_steps,
                       const int32_t* d_sal_off, const int32_t* d_sal_idx,
                       const uint16_t* d_sal_rows, uint32_t m, uint32_t n, uint32_t m_pad,
                       uint32_t n_total_pad, uint32_t col_base, float* d_out, void* stream);
/* Debug: canonical-layout base weight -> bf16 [m][n] (reference orientation). */
int mesw_unpack_weight_debug(const uint16_t* d_w, uint32_t m, uint32_t n, uint32_t m_pad,
                             uint32_t n_total_pad, uint32_t col_base, uint16_t* d_out,
                             void* stream);

/* ------------------------------------------- K2: fused multi-expert linear
 * y[t, :] = x[t, :] . W  +  x[t, :] . Dtilde_{expert(t)}  (+ residual[t, :])
 * with Dtilde applied straight from the packed codes (Eq. 4
 * PAPER.md:123-130): s_j * sum_{i not in S} x_i q_ij + sum_{i in S} x_i half(R)_ij.
 * Tokens are grouped by expert: segment s covers rows [seg_begin[s], seg_end[s])
 * and uses expert-table slot seg_slot[s]; rows in no segment get no delta.  Segment
 * begins are multiples of 8 rows (a segment of <= 8 rows may take the second half of a
 * 16-row window); TMEM bounds a launch to NP + 16 x (windows touched, summed over the
 * segments) <= 384 columns.
 * Replaces toylm._apply_delta + provider (toylm.py:183-186) and SPEC
 * delta_matvec / batched_multi_model_forward's shared-base + delta stages.  */
typedef struct {
  const void* codes;        /* device code layout of this expert's linear     */
  const float* steps;       /* [n_pad]                                         */
  const int32_t* sal_off;   /* [n_cg + 1]                                      */
  const int32_t* sal_idx;   /* [sal_off[n_cg]]                                 */
  const uint16_t* sal_rows; /* [sal_off[n_cg]][128] binary16                   */
} mesw_expert_dev;

typedef struct {
  const uint16_t* x;  /* bf16 activations, canonical tile layout (mesw_pack_x)  */
  int32_t B, m, n;   /* n: output columns written; device buffers must cover
                         ceil(n/256)*256 columns (column groups come in pairs) */
  int32_t x_layout;   /* must be 0 (canonical)                                 */
  const uint16_t* w;  /* canonical-layout bf16 base, or NULL (delta only)     */
  const mesw_expert_dev* expert_table; /* DEVICE array indexed by slot        */
  int32_t code_bits;  /* 2, 4 or 8: shared by all experts of the launch       */
  int32_t n_segments; /* <= MESW_MAX_SEGMENTS                                 */
  int32_t seg_begin[MESW_MAX_SEGMENTS];
  int32_t seg_end[MESW_MAX_SEGMENTS];
  int32_t seg_slot[MESW_MAX_SEGMENTS];
  void* y;            /* [B][ldy] output                                       */
  int32_t y_bf16;     /* 1: bf16 output, 0: f32 output                         */
  int32_t ldy;
  const uint16_t* residual; /* optional bf16 [B][ld_res], added before rounding */
  int32_t ld_res;
  void* workspace;    /* scratch for split-K partials                          */
  uint64_t workspace_bytes;
  int32_t* counters;  /* >= n_pad/128 int32, zero before first use (self-resetting) */
  int32_t num_ctas;   /* 0 = one persistent CTA per SM                         */
  int32_t activation; /* 0: none, 1: ReLU (toylm.py:207), applied last         */
  /* Optional (2-bit codes): per-token offset-code bias table written by the producer of
   * x (mesw_pack_x / the decoder glue): x_corr[t * x_corr_ld + ks] = sum over the 128
   * inputs k of k-step ks of w_k * x[t][k], w_k = 130, 34, 10 for ((k % 64) / 2) % 8 in
   * {0,3,6}, {1,4,7}, {2,5} (rows t >= B: 0).  When given, codes expand with one
   * instruction per word (c + u offset form) and the bias is removed in f32 in the
   * epilogue (~1e-5 relative on the delta term); NULL: exact q expansion.          */
  const float* x_corr;
  int32_t x_corr_ld;
  /* Optional DEVICE int32 [B]: output (and residual) row of launch row t, -1 = not written.
   * Lets callers keep their own row order while the launch groups rows by expert
   * (mesw_pack_x_gather builds the grouped input).  NULL: row t -> row t. */
  const int32_t* y_rows;
  /* Optional SwiGLU epilogue (the decode engine's fused gate|up linear): swiglu_I > 0 means
   * columns [0, I) are gate and [I, 2I) up (n = 2I, I % 128 == 0, bf16 y, no row map /
   * residual / activation).  Besides y, the launch writes act = silu(gate) * up (mesw_swiglu's
   * arithmetic) in the canonical layout with act_np rows, and, when act_corr != NULL, its
   * offset-code bias table act_corr[t * act_corr_ld + k-step].  counters must then hold
   * n_pad/128 + I/128 entries (zero before first use, self-resetting). */
  int32_t swiglu_I;
  uint16_t* act;
  int32_t act_np;
  float* act_corr;
  int32_t act_corr_ld;
} mesw_linear_args;

/* ------------------------------------------- K3: prefill fused multi-expert linear
 * Large token batches (prefill, BASELINE config 4): tokens come in 128-token groups, group g
 * covering rows [128g, 128g+128) of the canonical x (NP rows, NP % 256 == 0) and using expert
 * slot group_slot[g] (DEVICE int32 array, -1 = base only).  y[t, :] = x[t, :] . bf16(W +
 * Dtilde_e) (+ residual): the delta is folded into the tensor-core A operand per unit
 * (RN_bf16(W + s_j q_ij), salient inputs RN_bf16(W + half(R))), so the tensor work equals
 * the dense base GEMM (Eq. 4; toylm.py:183-186 applies x.W + x.Dtilde).
 * 2-bit codes (code_bits 2).  Same expert table / weight layouts as mesw_me_linear. */
typedef struct {
  const uint16_t* x;     /* canonical layout of NP rows                               */
  int32_t NP, B, m, n;   /* NP: multiple of 256; rows >= B are not written            */
  const uint16_t* w;
  const mesw_expert_dev* expert_table;
  int32_t code_bits;
  const int32_t* group_slot; /* DEVICE [NP/128]                                       */
  void* y;
  int32_t y_bf16, ldy;
  const uint16_t* residual;
  int32_t ld_res;
  int32_t num_ctas;      /* 0 = all SMs (CTA pairs)                                   */
} mesw_prefill_args;

int mesw_me_linear_prefill(const mesw_prefill_args* a, void* stream);

/* mesw_pack_x with a row gather: canonical row t (< rows) = x row d_src[t], or zeros when
 * d_src[t] < 0 -- groups caller rows by expert on the device (no host round trip). */
int mesw_pack_x_gather(const uint16_t* d_x, int ldx, const int32_t* d_src, int rows, int m, uint16_t* d_xc,
                       float* d_corr, int corr_ld, void* stream);

/* Canonical activation layout consumed by mesw_me_linear: rows padded to
 * NP = ceil16(B); for each 128-wide k-step ks a tile of NP*128 bf16 split in two
 * halves h (rows 0-7 / 8-15 of every 16-row window -- the N split of a cta_group::2
 * MMA between the two CTAs of a pair), each [NP/16 windows][16 k-chunks][8 rows][8]
 * (the UMMA K-major SWIZZLE_NONE canonical B operand), so one bulk copy per CTA stages it:
 *   index(t, k) = (k/128)*NP*128 + ((t/8)%2)*(NP/2)*128 + (t/16)*1024
 *                 + ((k%128)/8)*64 + (t%8)*8 + k%8.
 * Rows >= B and columns >= m are written as 0.  d_corr (optional, NULL = none): also
 * write the offset-code bias table of mesw_linear_args.x_corr for all NP rows. */
int mesw_pack_x(const uint16_t* d_x, int B, int m, int ldx, uint16_t* d_xc, float* d_corr, int corr_ld,
                void* stream);
/* Inverse (debug / tests): canonical -> row-major [B][ldy]. */
int mesw_unpack_x(const uint16_t* d_xc, int B, int m, uint16_t* d_y, int ldy, void* stream);

/* Workspace bytes mesw_me_linear needs for a given B and CTA count. */
uint64_t mesw_linear_workspace_bytes(int32_t B, int32_t num_ctas);
int mesw_me_linear(const mesw_linear_args* args, void* stream);

/* Glue outputs: row-major with leading dimension ld, or -- when *_np > 0 -- the
 * canonical activation layout (see mesw_pack_x) with NP = *_np rows, ready to be
 * the x operand of the next fused linear.  d_corr (optional, NULL = none): also write
 * its offset-code bias table (mesw_linear_args.x_corr) with leading dimension corr_ld. */
/* ------------------------------------- K5: Mistral decoder glue (decode step)
 * The reference toy model has no attention (toylm.py:1-8); these are the
 * standard decoder pieces around the fused linears of the Mistral-shaped
 * serving stack.  bf16 storage, f32 arithmetic.              */
/* out[b, :] = table[ids[b], :]  (embedding gather; toylm.py:165 `embedding[ids]`) */
int mesw_embed(const int32_t* d_ids, int B, const uint16_t* d_table, int H, uint16_t* d_out,
               int ld_out, void* stream);
/* y = x * rsqrt(mean(x^2) + eps) * w */
int mesw_rmsnorm(const uint16_t* d_x, int ldx, const uint16_t* d_w, int B, int H, float eps,
                 uint16_t* d_y, int ldy, int y_np, float* d_corr, int corr_ld, void* stream);
/* RoPE (rotate-half) on the q and k heads of a fused qkv row, append k/v to the
 * caches [B][ctx_max][n_kv][head_dim] at position pos[b]. */
int mesw_rope_append(uint16_t* d_qkv, int ld_qkv, const int32_t* d_pos, int B, int n_heads,
                     int n_kv, int head_dim, float theta, uint16_t* d_kcache,
                     uint16_t* d_vcache, int ctx_max, void* stream);
/* GQA decode attention over len[b] cached positions; out [B][n_heads*head_dim].
 * Split over the context in 32-position blocks (partials in `workspace`, then merged);
 * workspace >= mesw_attention_workspace_bytes(B, n_heads, ctx_max). head_dim 128. */
uint64_t mesw_attention_workspace_bytes(int B, int n_heads, int ctx_max);
int mesw_attention_decode(const uint16_t* d_q, int ld_q, const uint16_t* d_kcache,
                          const uint16_t* d_vcache, const int32_t* d_len, int B, int n_heads,
                          int n_kv, int head_dim, int ctx_max, uint16_t* d_out, int ld_out,
                          int out_np, void* workspace, uint64_t workspace_bytes, float* d_corr,
                          int corr_ld, void* stream);
/* Fused decode form of mesw_rope_append + mesw_attention_decode: d_qkv holds the new
 * token's [q heads | k heads | v heads] row (not yet rotated), at position len[b] - 1
 * (callers keep len = pos + 1).  Rotates q per split, rotates k and appends k / v to the
 * caches from the split holding the new position, then attends as mesw_attention_decode.
 * Same results, bit for bit, as the two-call form; one launch fewer per layer.
 * Contract (the decode engine's): len[] and the cached rows [0, len[b] - 1) are read before
 * the kernel's PDL wait (only the new token's qkv row after it), so they must be complete
 * when the kernels between their writer and this launch start: written before a kernel
 * that does not trigger its dependents early (mesw_advance_positions, any non-libmesw
 * kernel, a memcpy) or before a graph launch. */
int mesw_attention_decode_rope(const uint16_t* d_qkv, int ld_qkv, uint16_t* d_kcache,
                               uint16_t* d_vcache, const int32_t* d_len, int B, int n_heads,
                               int n_kv, int head_dim, float theta, int ctx_max, uint16_t* d_out,
                               int ld_out, int out_np, void* workspace, uint64_t workspace_bytes,
                               float* d_corr, int corr_ld, void* stream);
/* out = silu(gate) * up for rows [gate(I) | up(I)]. */
int mesw_swiglu(const uint16_t* d_gu, int ld_gu, int B, int I, uint16_t* d_out, int ld_out,
                int out_np, float* d_corr, int corr_ld, void* stream);
/* Greedy next token: argmax with ties to the lowest id (toylm.py:247). */
int mesw_argmax(const void* d_logits, int is_bf16, int B, int V, int ld, int32_t* d_out,
                void* stream);
/* Decode bookkeeping: pos[b] += 1, len[b] = pos[b] + 1.  wrap_to >= 0 wraps a request that
 * reaches ctx_max back to wrap_to (benchmark steady state); wrap_to < 0 never wraps (serving:
 * the host checks the cache window before each step). */
int mesw_advance_positions(int32_t* d_pos, int32_t* d_len, int B, int ctx_max, int wrap_to,
                           void* stream);

/* ------------------------------------------------ f2: delta compression
 * Replaces compress.compress_layer (compress.py:178-215, metric "reconstruction"),
 * bit-exact: steps, salient indices, fp16 salient rows and packed codes equal the
 * reference's for the same f32 delta [m][n] (reference orientation: rows = input
 * channels) and f32 activation energies [m] (ActivationStats.energy).  Outputs:
 * d_steps f32[n], d_sal_idx int32[k] ascending, d_sal_rows binary16[k][n],
 * d_packed mesw_packed_nbytes(m, n, bits) bytes (column-major runs, LSB-first).  */
uint64_t mesw_compress_workspace_bytes(uint32_t m, uint32_t n);
int mesw_compress_layer(const float* d_delta, uint32_t m, uint32_t n, const float* d_energy,
                        uint32_t bits, uint32_t k, float* d_steps, int32_t* d_sal_idx,
                        uint16_t* d_sal_rows, uint8_t* d_packed, void* d_workspace,
                        uint64_t workspace_bytes, void* stream);

/* ------------------------------------------------ f3: step-size distillation
 * The per-layer pieces of compress.distill_step_sizes (compress.py:331-378); the model
 * forward / backward around them are plain f32 GEMMs (host side, distill.py).  Given the
 * same inputs each is bit-exact with the reference's numpy (f64 order kept, no FMA).
 * row_slot int32[m]: -1 for quantized rows, r >= 0 for salient row r (rows f32[k][n],
 * fp16-rounded values); NULL = no salient rows.
 * QuantizedLayerState.reconstruct (toylm.py:379-384), optionally fused with `w + d`
 * (toylm.py:422-424): out = (base ? base : 0) + reconstruction.                   */
int mesw_ste_reconstruct(const float* d_delta, uint32_t m, uint32_t n, const float* d_steps, uint32_t bits,
                         const int32_t* d_row_slot, const float* d_sal_rows, const float* d_base,
                         float* d_out, void* stream);
/* QuantizedLayerState.step_gradient -> quant.ste_step_gradient (toylm.py:386-391,
 * quant.py:142-169): grad f32[n] from upstream f32[m][n] (salient rows masked). */
int mesw_ste_step_grad(const float* d_delta, uint32_t m, uint32_t n, const float* d_steps, uint32_t bits,
                       const int32_t* d_row_slot, const float* d_upstream, float* d_grad, void* stream);
/* _Adam.step for one step vector (compress.py:288-302; f64 moments d_m/d_v, weight
 * decay 0) followed by the clamp max(steps, step_floor) (compress.py:375).
 * bias_corr1/2 = 1 - beta1**t, 1 - beta2**t (computed by the caller in f64). */
int mesw_adam_step(float* d_steps, double* d_m, double* d_v, const float* d_grad, uint32_t n, double lr,
                   double beta1, double beta2, double eps, double bias_corr1, double bias_corr2,
                   float step_floor, void* stream);
/* compress._repack (compress.py:325-335): codes of the unmasked rows re-derived from
 * the trained steps (salient_mask u8[m] != 0 -> code 0), packed like mesw_compress_layer. */
int mesw_quantize_pack(const float* d_delta, uint32_t m, uint32_t n, const float* d_steps, uint32_t bits,
                       const uint8_t* d_salient_mask, uint8_t* d_packed, void* stream);

/* ------------------------------------------------ K4: model-level router
 * Replaces SPEC router.classify for a batch of B queries:
 * multinomial Naive Bayes over FNV-1a-hashed character 2/3-grams (2^16 buckets),
 * hashing and f64 summation order as pinned in oracle/router.py.
 *   d_codepoints  int32 Unicode code points of all queries, concatenated
 *   d_offsets     int64[B+1]: query q = code points [off[q], off[q+1])
 *   d_loglik      f32[D][65536], d_logprior f32[D], 1 <= D <= 64 (two domains per warp lane)
 * Outputs: d_domain[B] (argmax, ties -> lowest id), d_conf[B] (softmax of the
 * winner), d_prior_only[B] (1 when the query has no n-gram; may be NULL).      */
int mesw_router_classify(const int32_t* d_codepoints, const int64_t* d_offsets, int B,
                         const float* d_loglik, const float* d_logprior, int D, int32_t* d_domain,
                         float* d_conf, int32_t* d_prior_only, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MESW_H_ */
