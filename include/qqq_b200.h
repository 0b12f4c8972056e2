/*
 * qqq_b200.h — C ABI of the B200-native (sm_100a) W4A8 hot path of QQQ
 * (arXiv 2406.09904). Plain pointers and sizes only; every device pointer is
 * caller-allocated (torch, or any CUDA allocator); every call is asynchronous
 * on the given stream and stateless ("pure functions").
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/qqq/<file>:<line>). Return value: QQQ_OK or one of
 * the QQQ_ERR_* codes, which the host layer maps to the reference's exception
 * classes (errors.py:4-33). Data-dependent errors the reference raises
 * (non-finite activations, out-of-range codes, bad padding, overflowing fused
 * scales) are reported through a caller-owned device int32 status word
 * (QQQ_STAT_* bits, atomically OR-ed) that the host checks after its sync.
 *
 * Library: paper_2406_09904_b200/lib/libqqq_b200.so (nvcc -gencode
 * arch=compute_100a,code=sm_100a). Weight-layout and kernel design: DESIGN.md.
 */
#ifndef QQQ_B200_H
#define QQQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* qqq_stream_t; /* == cudaStream_t */

enum {
  QQQ_OK = 0,
  QQQ_ERR_SHAPE = 1,       /* ShapeError */
  QQQ_ERR_DATA = 2,        /* DataError */
  QQQ_ERR_CONFIG = 3,      /* ConfigError */
  QQQ_ERR_CORRUPTION = 4,  /* CorruptionError */
  QQQ_ERR_CUDA = 5,        /* launch / driver failure */
  QQQ_ERR_UNSUPPORTED = 6  /* shape outside the kernel's contract (host re-lays out) */
};

enum {
  QQQ_STAT_NONFINITE = 1,   /* quantize.py:85-89 DataError */
  QQQ_STAT_CODE_RANGE = 2,  /* quantize.py:181-182 DataError */
  QQQ_STAT_PAD_NIBBLE = 4,  /* quantize.py:206-207 CorruptionError */
  QQQ_STAT_SCALE_INF = 8,   /* gemm.py:67-68 ConfigError */
  QQQ_STAT_NEED_CLAMP = 16, /* repack: FusedDequantQuant clamp needed -> I8 layout */
  QQQ_STAT_TINY_SCALE = 32  /* reserved */
};

enum { QQQ_MODE_PC = 0, QQQ_MODE_PG = 1, QQQ_MODE_I8 = 2 };

/* ---- activations -------------------------------------------------------- */

/* quant_act_per_token (quantize.py:92-100). x: M x K row-major (row stride ldx
 * elements), dtype 0=f16 1=f32 2=f64. q: int8 M x K (row stride ldq bytes),
 * s_a: f64[M]. Bit-exact with the reference (ties included). */
int qqq_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int8_t* q, int64_t ldq,
                  double* s_a, int32_t* status_dev, qqq_stream_t stream);
/* Same, also writing rowsum[M] = sum_k q[t, k] (int32), which the per-group
 * GEMM needs (its weights run as u8 = w8 + 128; acc = acc_u8 - 128*rowsum). */
int qqq_act_quant_ex(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int8_t* q, int64_t ldq,
                     double* s_a, int32_t* rowsum, int32_t* status_dev, qqq_stream_t stream);
/* apply_quant_linear's activation step (pipeline.py:146): quant_act_per_token
 * of x / smooth, smooth = the smoothing plan's f64[K] vector (smoothing.py:38-43),
 * divided in f64 inside the quantizer (replaces the numpy divide + quantize).
 * smooth_mask (optional, may be NULL): ceil(K/8) bytes, bit k set <=> smooth[k]
 * != 1.0 — channels outside the plan's `selected` set skip the f64 division
 * (and the load of smooth[k]); results are identical either way. */
int qqq_act_quant_smooth(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, const double* smooth,
                         const uint8_t* smooth_mask, int8_t* q, int64_t ldq, double* s_a, int32_t* rowsum,
                         int32_t* status_dev, qqq_stream_t stream);
/* Reciprocal table of a smoothing vector (once per layer): recip[k] = RN(1/smooth[k])
 * (IEEE division), NaN where |smooth[k]| is outside [2^-400, 2^400]. */
int qqq_smooth_reciprocal(const double* smooth, int64_t K, double* recip, qqq_stream_t stream);
/* qqq_act_quant_smooth with that table: each x / smooth[k] is computed as a
 * Markstein FMA sequence from recip[k] (the same correctly rounded quotient, so
 * codes and scales stay bit-identical to pipeline.py:146 + quantize.py:92-100);
 * NaN entries keep the IEEE division. The table is read for M <= 32 (decode
 * batches, where it measured faster); larger batches divide as
 * qqq_act_quant_smooth does. */
int qqq_act_quant_smooth_rcp(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, const double* smooth,
                             const double* smooth_recip, int8_t* q, int64_t ldq, double* s_a, int32_t* rowsum,
                             int32_t* status_dev, qqq_stream_t stream);
/* rowsum of existing int8 codes (activations not produced by qqq_act_quant_ex). */
int qqq_act_rowsum(const int8_t* q, int64_t M, int64_t K, int64_t ldq, int32_t* rowsum, qqq_stream_t stream);

/* K-split tensor parallelism (row-parallel linear): the reference scale uses
 * the FULL row (quantize.py:97-98), so each rank first computes its shard's
 * row absmax (f64[M]), the ranks all-reduce MAX it, and every rank quantizes
 * its shard with the global max. Identical codes to the unsplit reference. */
int qqq_act_absmax(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, double* row_max,
                   int32_t* status_dev, qqq_stream_t stream);
int qqq_act_quant_with_max(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, const double* row_max,
                           int8_t* q, int64_t ldq, double* s_a, int32_t* rowsum, int32_t* status_dev,
                           qqq_stream_t stream);

/* ---- offline weight preparation ----------------------------------------- */

/* quant_weight_per_channel (quantize.py:111-123) when group <= 0, else the
 * per-group code/scale step of quant_weight_per_group (quantize.py:126-149).
 * w: f64 K x N; codes: int8 K x N; scales: f64 [K/group or 1] x N. */
int qqq_quant_weight(const double* w, int64_t K, int64_t N, int64_t group, int8_t* codes, double* scales,
                     int32_t* status_dev, qqq_stream_t stream);

/* requant_scale (quantize.py:152-168): s_wc f64[N] from codes and s_wg [G x N]. */
int qqq_requant_scale(const int8_t* codes, const double* s_wg, int64_t K, int64_t N, int64_t G, double* s_wc,
                      qqq_stream_t stream);

/* pack_i4 / unpack_i4 (quantize.py:171-208). packed: uint8 ceil(K/2) x N. */
int qqq_pack_i4(const int8_t* codes, int64_t K, int64_t N, uint8_t* packed, int32_t* status_dev, qqq_stream_t stream);
int qqq_unpack_i4(const uint8_t* packed, int64_t rows, int64_t N, int8_t* codes, int32_t* status_dev,
                  qqq_stream_t stream);

/* FusedScales.from_quantized, per-group branch (gemm.py:65-69): s_star binary16
 * bits [G x N] = f16(s_wg / s_wc). (Per-channel s_w/16 is an exact host-side
 * tensor op.) */
int qqq_fused_scales_pg(const double* s_wg, const double* s_wc, int64_t G, int64_t N, uint16_t* s_star,
                        int32_t* status_dev, qqq_stream_t stream);

/* dequantize_ref (quantize.py:211-217): out f64 K x N = codes * scale
 * (group <= 0: per-channel scales[N]; else scales[(k/group), n]). */
int qqq_dequantize(const int8_t* codes, int64_t K, int64_t N, int64_t group, const double* scales, double* out,
                   qqq_stream_t stream);

/* ---- one-time repack into the tcgen05 kernel layout ---------------------- */

/* Bytes of the kernel-layout weight blob (layout: DESIGN.md / qqq_layout.cuh).
 * 0 if (mode, group) is not a kernel layout (per-group needs group in {32, 64}
 * or a multiple of 128; other group sizes use QQQ_MODE_I8). */
size_t qqq_repacked_weight_bytes(int mode, int64_t K, int64_t N, int64_t group);

/* QQQ_MODE_PC / QQQ_MODE_PG blob from the reference pack_i4 bytes (+ the fused
 * binary16 s_star [K/group x N] for PG). For PG, flags_dev gets
 * QQQ_STAT_NEED_CLAMP if, for the codes actually present, the clamp-free HFMA2
 * converter would differ from the reference's clamped FusedDequantQuant
 * (gemm.py:123-127); the caller then builds the QQQ_MODE_I8 blob instead. */
int qqq_repack_weights(const uint8_t* packed, const uint16_t* s_star, int64_t K, int64_t N, int mode, int64_t group,
                       void* out, int32_t* flags_dev, qqq_stream_t stream);

/* QQQ_MODE_I8 blob from an int8 K x N matrix (w8), or from pack_i4 bytes +
 * s_star via the reference's exact scalar FusedDequantQuant (gemm.py:110-127). */
int qqq_repack_weights_i8(const int8_t* w8, const uint8_t* packed, const uint16_t* s_star, int64_t group, int64_t K,
                          int64_t N, void* out, qqq_stream_t stream);

/* ---- the W4A8 GEMM ------------------------------------------------------- */

/* Caller-provided workspace, zero-initialised once; every launch leaves its
 * counter head zeroed again (launches sharing it must be stream-ordered). */
size_t qqq_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);

/* w4a8_gemm_per_channel (gemm.py:173-185): y f16 M x N = f16((acc*s_a)*s_w_folded),
 * acc = aq . (16*q). acc_opt (int32 M x N) is written when non-NULL. aq must be
 * 16-byte aligned with ldq % 16 == 0 and ldq >= round_up(K, 128) (bytes past K
 * in a row are read but multiply zero weights). */
int qqq_w4a8_gemm_pc(const int8_t* aq, int64_t ldq, const double* s_a, const void* w_repacked,
                     const double* s_w_folded, int64_t M, int64_t N, int64_t K, void* y, int64_t ldy, int32_t* acc_opt,
                     int64_t ldacc, void* workspace, size_t ws_bytes, qqq_stream_t stream);

/* w4a8_gemm_per_group (gemm.py:188-203): acc = aq . FusedDequantQuant(q, s*),
 * y = f16((acc*s_a)*s_wc); the blob carries s*. group in {32, 64} or k*128.
 * rowsum: sum of each token's int8 codes (qqq_act_quant_ex / qqq_act_rowsum). */
int qqq_w4a8_gemm_pg(const int8_t* aq, int64_t ldq, const double* s_a, const int32_t* rowsum,
                     const void* w_repacked, int64_t group, const double* s_wc, int64_t M, int64_t N, int64_t K,
                     void* y, int64_t ldy, int32_t* acc_opt, int64_t ldacc, void* workspace, size_t ws_bytes,
                     qqq_stream_t stream);

/* Generic form (mode PC/PG/I8) with an optional tile-plan override; I8 with
 * s_col == NULL is gemm_i8_i32 (gemm.py:145-154, acc only). */
typedef struct qqq_gemm_config {
  int ntok;  /* tokens per UMMA tile: 16/32/64/128/192/256/384, 0 = auto (192, 384: pair plans
             * only; 384 = two N=192 MMAs per K step, split 3 forced; 128 with
             * split 3: 128-token pair tiles) */
  int grid;  /* CTAs for stream-K, 0 = auto */
  int split; /* -1 auto, 0 whole tiles, 1 stream-K, 2 whole-tile waves + stream-K remainder,
              * 3 whole 256-channel pair tiles (2-CTA clusters, ntok 256, 192, 384 or 128), 4 cluster
              * split-K (one tile per cluster, DSMEM reduction: ntok 16/32 half-SM CTAs,
              * reduce-scatter by channel rows; ntok 128 whole-SM CTAs, by token range),
              * 5 stream-K over pair tiles, 6 pair-tile waves + stream-K remainder */
  int csplit; /* split 4 only: cluster size S (2..8 for ntok 16/32, 2 or 4 for ntok 128;
               * 0 = the planner's choice) */
  void* dbg; /* optional device buffer [grid][64] u64: per-CTA %globaltimer timeline (diagnostics) */
} qqq_gemm_config;

int qqq_w4a8_gemm_ex(int mode, const int8_t* aq, int64_t ldq, const double* s_a, const int32_t* rowsum,
                     const void* w_repacked, int64_t group, const double* s_col, int64_t M, int64_t N, int64_t K,
                     void* y, int64_t ldy, int32_t* acc_opt, int64_t ldacc, void* workspace, size_t ws_bytes,
                     const qqq_gemm_config* cfg, qqq_stream_t stream);

/* apply_quant_linear in one launch (replaces pipeline.py:144-152's
 * `quant_act_per_token(x / s)` + `w4a8_gemm_*` pair; mode PC or PG): the
 * epilogue warps of the GEMM's first-wave CTAs quantize x / smooth (fp16
 * [M, K], row pitch ldx; K, ldx multiples of 8, x / smooth / smooth_recip
 * 16-byte aligned) into q (row pitch ldq as for qqq_w4a8_gemm_ex), s_a and
 * rowsum -- bit-identical to qqq_act_quant_smooth(_rcp) -- while the weights
 * stream in; the MMAs start once every row is published. smooth_recip:
 * qqq_smooth_reciprocal's table or NULL. Non-finite quotients OR
 * QQQ_STAT_NONFINITE into *status_dev (DataError, quantize.py:85-89). The
 * workspace is qqq_w4a8_gemm_ex's (its head holds the row counter). */
int qqq_w4a8_gemm_smooth_fused(int mode, const void* x, int64_t ldx, const double* smooth,
                               const double* smooth_recip, int8_t* q, int64_t ldq, double* s_a, int32_t* rowsum,
                               int32_t* status_dev, const void* w_repacked, int64_t group, const double* s_col,
                               int64_t M, int64_t N, int64_t K, void* y, int64_t ldy, int32_t* acc_opt,
                               int64_t ldacc, void* workspace, size_t ws_bytes, const qqq_gemm_config* cfg,
                               qqq_stream_t stream);

/* The tile plan qqq_w4a8_gemm_ex would launch for (mode, M, N, K, cfg): the
 * planner's choice when cfg is NULL or all-auto, else the forced plan as the
 * launch resolves it (out->split is the effective split, out->csplit the
 * cluster size of split 4). Diagnostics and tests; no device work. */
int qqq_gemm_plan_info(int mode, int64_t M, int64_t N, int64_t K, const qqq_gemm_config* cfg,
                       qqq_gemm_config* out);

/* The dequant epilogue alone (gemm.py:182-184 / 200-202): y f16 M x N =
 * f16((acc*s_a)*s_col) in f64; used after an exact int32 all-reduce of K-split
 * partial accumulators (the GEMM with s_col == NULL returns acc only). */
int qqq_dequant_epilogue(const int32_t* acc, int64_t M, int64_t N, int64_t ldacc, const double* s_a,
                         const double* s_col, void* y, int64_t ldy, qqq_stream_t stream);

/* ---- conversion test hooks (the exact device functions the GEMM uses) ---- */

/* fused_dequant_quant (gemm.py:110-127): word_path=0 scalar reference branch
 * structure; word_path=1 the GEMM's HFMA2/PRMT converter (8 codes per s*). */
int qqq_test_fused_dequant_quant(const int8_t* q, const uint16_t* s_star, int8_t* out, int64_t n, int word_path,
                                 qqq_stream_t stream);
/* fast_i4_to_i8 (gemm.py:81-85) via the GEMM's per-channel shift converter. */
int qqq_test_pc_convert(const int8_t* q, int8_t* out, int64_t n, qqq_stream_t stream);
/* fast_f16_to_i8 (gemm.py:99-107). */
int qqq_test_fast_f16_to_i8(const uint16_t* bits, int8_t* out, int64_t n, qqq_stream_t stream);

/* ---- misc ---------------------------------------------------------------- */
/* Dense INT8 tensor-core peak probe (bench.py's roofline denominator): `grid`
 * CTAs (one per SM) each issue `iters` (multiple of 8) back-to-back
 * tcgen05.mma kind::i8 M=128 N=256 K=32 from shared memory; *ops_out = the
 * integer ops the launch performs. The caller times it with CUDA events. */
int qqq_probe_int8_peak(int grid, int iters, double* ops_out, qqq_stream_t stream);
int qqq_device_ok(void); /* QQQ_OK iff the current device is sm_100 */
const char* qqq_version(void);

/* ---- offline calibration ------------------------------------------
 * matmul_ref (numerics.py:94-109) on the GPU: C = A B in f64 with the reference's
 * rounding sequence (each product rounded, then added, in sequential k order;
 * no FMA), so smoothing_objective's error matrix (smoothing.py:108-113) is
 * bit-identical. A M x K, B K x N, C M x N, all row-major and contiguous. */
int qqq_matmul_ref_f64(const double* a, const double* b, double* c, int64_t M, int64_t K, int64_t N,
                       qqq_stream_t stream);
/* One block [i1, i2) of the GPTQ column sweep (gptq.py:161-181) over work (f64
 * K x N, row-major, updated in place), U = chol_inv (f64 K x K). gs = 0:
 * per-channel with the frozen scales scale_row[N]; gs > 0: per-group, s_wg
 * ((K/gs) x N) written at each group start (i1, i2 multiples of gs). Writes the
 * codes (int8 K x N, rows i1..i2) and the block's errors eb ((i2-i1) x N).
 * Bit-identical to the reference's block; the trailing update between blocks
 * (gptq.py:182-183) is a BLAS product left to the caller. */
int qqq_gptq_block(double* work, int64_t K, int64_t N, const double* u, int64_t i1, int64_t i2, int64_t gs,
                   double* scale_row, double* s_wg, int8_t* codes, double* eb, qqq_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* QQQ_B200_H */
