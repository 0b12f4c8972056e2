// B200 (sm_100a) W4A8 GEMM: per-channel and per-group QQQ dataflows on tcgen05.
//
// Reference semantics (pkg/src/qqq/gemm.py):
//   per-channel  (:173-185): w8 = 16*q ; acc = A_i8 . w8 (int32) ;
//                            y = f16((acc * s_a[t]) * s_w_folded[n])   (f64, one rounding)
//   per-group    (:188-203): w8 = FusedDequantQuant(q, s*[k/g, n]) ;
//                            acc = A_i8 . w8 ; y = f16((acc * s_a[t]) * s_wc[n])
//
// Design (weight-stationary, tokens on the MMA N axis):
//   * UMMA M = 128 output channels per tile, UMMA N = NTOK tokens (16..256),
//     int8 x int8 -> int32 accumulators in TMEM (tcgen05.mma kind::i8),
//     double-buffered so the epilogue of one tile overlaps the next tile's MMAs.
//   * Warp roles (512 threads). The SM sub-partition scheduler issues from the
//     highest warp id first, so latency-critical single-thread roles get the
//     high ids: w15 = MMA issuer, w14 = TMA/bulk producer, w12 = TMEM allocator,
//     w8-11 = epilogue (TMEM lane quadrant = warp % 4), w0-7 = INT4->INT8
//     converters (shift for PC, HFMA2 magic-number FusedDequantQuant for PG)
//     writing the canonical no-swizzle K-major operand into shared memory.
//   * Per k-block exactly two TMA ops: one cp.async.bulk of the contiguous
//     weight(+scale) super-slabs and one 3-D tensor TMA of the int8 activation
//     tile (SWIZZLE_128B, OOB token rows zero-filled).
//   * PDL: the first kStages k-blocks of weights are requested before
//     griddepcontrol.wait, overlapping the previous kernel's tail.
//   * Work split: stream-K over (tile, k-block) units across the SMs. A tile
//     split over several CTAs is reduced exactly: each segment stores its int32
//     partial to its own workspace slot, the last arriving CTA (atomic counter)
//     sums the slots (integer addition: order-free, bit-exact) and applies the
//     epilogue; counters are re-zeroed by that CTA.
//   * Epilogue: f64 (acc * s_a) * s_col then cvt.rn.f16.f64 -> bit-identical
//     to the reference's f64 epilogue with a single final rounding.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "act_quant_dev.cuh"
#include "qqq_common.cuh"
#include "qqq_layout.cuh"

namespace qqq {

#ifdef QQQ_TIMELINE
constexpr int kDbgSlots = 192;
#endif

// Big-CTA cluster split-K partial exchange: through DSMEM st.async (default), or
// through L2 (QQQ_CSB_L2=1: coalesced stores to per-(tile, destination, sender)
// workspace chunks, one gpu-scope fence + remote arrive per CTA, cluster-scope
// acquire). Measured: the L2 exchange is 0.4-0.9 us slower per GEMM on
// 4096x4096 / 11008x4096 at M = 32-256 (the fence and the L2 round trips cost
// more than DSMEM's ~20 B/clk), so DSMEM stays.
#ifndef QQQ_CSB_L2
#define QQQ_CSB_L2 0
#endif


struct GemmParams {
  const uint8_t* w;     // repacked weight blob (qqq_layout.cuh)
  const double* s_a;    // [M]
  const int32_t* rowsum;  // [M] sum of activation codes (per-group u8 x s8 correction)
  const double* s_col;  // [N] s_w_folded (PC) / s_wc (PG); nullptr -> acc only
  __half* y;
  int64_t ldy;
  int32_t* acc;  // optional
  int64_t ldacc;
  int32_t* ws;        // split-K accumulation slots [tiles][NTOK][128] int32, zero on entry and exit
  int32_t* counters;  // [tiles] arrival counters at the fixed head of the workspace; zero on entry and exit
  int M, N, K;
  int n_tiles, tok_tiles, kb_per_tile, ss_per_tile, ss_bytes, group, max_segs;
  int64_t units;
  int aligned_tiles;        // >0: CTA b owns whole tiles [b*aligned_tiles, ...)
  int dp_tiles;             // hybrid: CTA b first owns whole tiles [b*dp_tiles, (b+1)*dp_tiles), then
  int64_t sk_unit0;         //   its stream-K share of the units [sk_unit0, sk_unit0 + units)
  int y_tma;                // 1: y written by TMA stores from a shared-memory staging tile
  int pair;                 // 1: 2-CTA clusters (cta_group::2); tiles count 256-channel pair tiles
  int csplit;               // >1: cluster split-K (decode CTAs): cluster c = tile c, rank r = k-range r of csplit,
                            //     partials reduce-scattered over DSMEM (rank r finalizes channel rows r*128/csplit..)
  unsigned long long* dbg;  // optional per-CTA %globaltimer timeline, diagnostics only
  // Fused smoothed activation quantization (apply_quant_linear, pipeline.py:144-152), when xsrc
  // is set: the epilogue warps of CTAs [0, q_ctas) quantize x / smooth (fp16 [M, K], row pitch
  // ldx) into the activation operand (qdst, row pitch = the TMA map's), s_a and rowsum while the
  // weights stream in; the activation producers and the epilogue wait for all M rows (a counter
  // in the workspace head, zero on entry and exit).
  const __half* xsrc;
  int64_t ldx;
  const double* smooth;
  const double* srecip;  // qqq_smooth_reciprocal table or nullptr (IEEE division)
  int8_t* qdst;
  int64_t ldq;
  double* sa_dst;
  int32_t* rs_dst;
  int32_t* status;
  int q_ctas;
  // Always 0. A runtime zero the compiler cannot fold: the converters' stage
  // release is made data-dependent on their shared-memory loads through it
  // (`dep & zero`); with a literal `and 0` ptxas dropped the dependency.
  uint32_t zero;
};

// workspace-head slots of the fused quantization: rows published, CTAs done with them
constexpr int kQRowsSlot = 65536 - 2;
constexpr int kQDoneSlot = 65536 - 1;

template <int MODE, int NTOK, int BK, bool PAIR = false>
struct Cfg {
  static constexpr bool kConvert = MODE != kModeI8;
  // PAIR: a 2-CTA cluster computes a 256-channel x NTOK tile with
  // tcgen05.mma.cta_group::2 (UMMA M=256): each CTA converts its own 128
  // channels into its own TMEM, but loads only HALF of the activation tile
  // (NTOK/2 tokens; the pair's MMA reads B from both CTAs' shared memory), so
  // the per-SM activation traffic and staging halve — the NTOK=256 prefill
  // tile is otherwise starved of activation + weight bytes in flight.
  static constexpr bool kPair = PAIR;
  static constexpr int kTokLoad = PAIR ? NTOK / 2 : NTOK;  // activation rows this CTA loads per k-block
  // 384-token pair tiles: two MMAs of N = 192 per K step (UMMA N <= 256). Each CTA
  // loads two 96-row chunks, tokens [96r, 96r+96) and [192+96r, 192+96r+96) of the
  // tile, so accumulator column c is token c for both MMAs.
  static constexpr int kMmaSplit = NTOK > 256 ? 2 : 1;
  static constexpr int kMmaN = NTOK / kMmaSplit;
  // ---- CTA shape. Decode/mid tiles (NTOK <= 64) use a half-SM CTA: two per SM,
  // so a CTA's prologue / first-byte latency / epilogue tail overlaps the other
  // CTA's stream, and under PDL the next kernel's CTAs start (and prefetch
  // their weights) in the slots this kernel's CTAs free. Prefill tiles use the
  // whole SM (accumulators fill TMEM).
  static constexpr bool kSmall = NTOK <= 64 && MODE != kModeI8;  // (I8 stages are 2x larger)
  static constexpr int kCtasPerSm = kSmall ? 2 : 1;
#ifndef QQQ_BIG_CONV_WARPS
#define QQQ_BIG_CONV_WARPS 8
#endif
  // 2 per TMEM lane quadrant: each converter warp handles >= 2 slabs per
  // k-block so the per-k-block handshake cost (~80 instructions per warp) stays
  // well below the conversion work
  static constexpr int kNumConvWarps = kSmall ? 8 : QQQ_BIG_CONV_WARPS;
#ifndef QQQ_PAIR_CONV_GROUPS
#define QQQ_PAIR_CONV_GROUPS 2
#endif
  // k-block interleaving: converter group g (kNumConvWarps / kConvGroups warps,
  // covering all 128 rows and BK of k) takes the k-blocks it with it % groups ==
  // g, so each warp's fixed per-k-block latency (barrier waits, TMEM store
  // completion, arrive) overlaps the other group's k-block
#ifndef QQQ_BIG_CONV_GROUPS
#define QQQ_BIG_CONV_GROUPS 1
#endif
  static constexpr int kConvGroups = PAIR ? QQQ_PAIR_CONV_GROUPS : kSmall ? 1 : QQQ_BIG_CONV_GROUPS;
  static constexpr int kConvPerGroup = kNumConvWarps / kConvGroups;
  static_assert(kConvPerGroup % 4 == 0, "a converter group covers the 4 TMEM lane quadrants");
#ifndef QQQ_BIG_EPI_WARPS
#define QQQ_BIG_EPI_WARPS 12
#endif
  static constexpr int kNumEpiWarps = kSmall ? 4 : QQQ_BIG_EPI_WARPS;  // groups of 4 (one warp per lane quadrant)
  static constexpr int kEpiGroups = kNumEpiWarps / 4;
  static constexpr int kConvWarp0 = 0;
  static constexpr int kEpiWarp0 = kNumConvWarps;
  // big CTA: TMEM allocator, activation producer, weight producer and MMA warps;
  // small CTA: the MMA warp allocates TMEM, and ONE producer warp runs both
  // rings in k-block order (weights kWStages ahead, issued before the CTA
  // set-up barrier). A separate weight producer that keeps streaming through
  // the PDL wait (QQQ_SMALL_TWO_PRODUCERS, 15 warps at 64 registers) measured
  // 7% slower on 4096x4096 decode chains and equal elsewhere.
  static constexpr int kAllocWarp = kEpiWarp0 + kNumEpiWarps;
#ifndef QQQ_SMALL_TWO_PRODUCERS
  static constexpr int kActProducerWarp = kAllocWarp + 1;
  static constexpr int kWProducerWarp = kSmall ? kAllocWarp + 1 : kAllocWarp + 2;
#else
  static constexpr int kActProducerWarp = kAllocWarp + 1;
  static constexpr int kWProducerWarp = kAllocWarp + 2;
#endif
  static constexpr int kMmaWarp = kSmall ? kAllocWarp : kAllocWarp + 3;
  static constexpr int kNumThreads = ((kSmall ? kWProducerWarp : kMmaWarp) + 1) * 32;
  static constexpr int kSmemBudget = kSmall ? 111 * 1024 : 225 * 1024;
  static constexpr int kTmemBudget = kSmall ? 256 : 512;
  // split-K partial ring depth per epilogue group (2 when the shared memory allows)
  // (the NTOK=256 prefill tiles, mostly whole tiles, give it up for activation stages)
#ifndef QQQ_BIG_PARTBUFS
#define QQQ_BIG_PARTBUFS 2
#endif
  static constexpr int kPartBufs = (kEpiGroups > 2 && NTOK >= 256) ? 1 : kSmall ? 2 : QQQ_BIG_PARTBUFS;  // (part_full holds 2 per group)
  // y staging per epilogue warp: kYBufs x [16 tok][32 ch] fp16 (1 KiB each); the
  // whole-SM 128-token tile single-buffers it (the 12 KiB buy its activation
  // ring one more stage), the paired epilogue chunks of 256/384-token tiles
  // and the half-SM CTAs keep two
#ifndef QQQ_BIG128_YBUFS
#define QQQ_BIG128_YBUFS 1
#endif
  static constexpr int kYBufs = (!kSmall && !PAIR && NTOK == 128) ? QQQ_BIG128_YBUFS : 2;
  static constexpr int kYWarpBytes = kYBufs * 1024;
  static constexpr int kEpiSmem = kNumEpiWarps * kYWarpBytes + kEpiGroups * kPartBufs * 8192;  // y staging + partial ring
  // Two rings. Weights: their own TMA ring (released by the converters once
  // the packed bytes are consumed, or by the MMA in I8 mode). K-blocks: ring
  // slot s = activation stage s = TMEM A buffer s, guarded by ONE full barrier
  // (activation TMA bytes + one arrival per converter warp + the producer's
  // arrive) and ONE empty barrier (the MMA's commit), so the MMA warp pays one
  // wait and one commit per k-block (each ~130 cycles, scripts/mma_probe2.cu).
  static constexpr int kXBytes = kTokLoad * BK;
  static constexpr int kSSMax = MODE == kModeI8 ? 16384 : MODE == kModePC ? 8192 : 8192 + 256 * 4;
  static constexpr int kWBytes = (BK / 128) * kSSMax;  // worst case (PG, g = 32)
  // Converted int8 weights (the MMA A operand) live in TMEM, not shared memory:
  // kABufs buffers of BK/4 columns (128 lanes x 4 int8 per column). This keeps
  // the 1 B/weight operand off the shared-memory crossbar, which otherwise
  // bounds the decode stream (TMA write + STS + MMA read of every weight).
  static constexpr int kACols = BK / 4;
  static constexpr int kAccBufs = NTOK >= 256 ? 1 : 2;
  static constexpr int kAccCols = kAccBufs * NTOK;
  static constexpr int kABufsMax = kConvert ? (kTmemBudget - kAccCols) / kACols : 8;
  static constexpr int kRingBudget = kSmemBudget - 2048 - NTOK * 12 - kEpiSmem;
  // k-block ring depth: what is left after 3 weight stages, at most 4 and at
  // most the number of TMEM A buffers that fit beside the accumulators
  static constexpr int kXStagesRaw = (kRingBudget - 3 * kWBytes) / kXBytes;
#ifndef QQQ_PAIR_XCAP
#define QQQ_PAIR_XCAP 6
#endif
#ifndef QQQ_PAIR_WMAX
#define QQQ_PAIR_WMAX 12
#endif
#ifndef QQQ_SMALL_XCAP
#define QQQ_SMALL_XCAP 4
#endif
#ifndef QQQ_BIG_XCAP
#define QQQ_BIG_XCAP 4
#endif
  static constexpr int kXCapWanted = PAIR ? QQQ_PAIR_XCAP : kSmall ? QQQ_SMALL_XCAP : QQQ_BIG_XCAP;
  static constexpr int kXCap = kABufsMax < kXCapWanted ? kABufsMax : kXCapWanted;
  static constexpr int kXStages = kXStagesRaw < 2 ? 2 : (kXStagesRaw > kXCap ? kXCap : kXStagesRaw);
  // Whole-tile plans of the whole-SM (non-pair) CTA borrow the split-K partial
  // ring, idle when no tile is split, as one more activation stage (and TMEM A
  // buffer): the k-block pace of these tiles is bound by the activation
  // ring's latency, not by its bandwidth (runtime ring size: `nx` in the kernel).
  static constexpr int kPartBytes = kEpiGroups * kPartBufs * 8192;
#ifndef QQQ_XTRA_STAGE
#define QQQ_XTRA_STAGE 1
#endif
  static constexpr int kXStagesXtra =
      (QQQ_XTRA_STAGE && !kSmall && !PAIR && kConvert && kPartBytes >= kXBytes && kXStages + 1 <= kABufsMax) ? 1 : 0;
  static constexpr int kXStagesMax = kXStages + kXStagesXtra;
  static constexpr int kABufs = kConvert ? kXStagesMax : 0;
  static constexpr int kWStagesRaw = (kRingBudget - kXStages * kXBytes) / kWBytes;
  static_assert(kXStages <= kABufsMax || !kConvert, "TMEM A buffers");
  static constexpr int kWMax = PAIR ? QQQ_PAIR_WMAX : 12;
  static constexpr int kWStages = kWStagesRaw > kWMax ? kWMax : kWStagesRaw;
  static_assert(kWStages >= 2, "shared memory budget too small");
  static constexpr int kOffX = 0;  // 1024-aligned: NTOK*BK is a multiple of 2048
  static constexpr int kOffW = kOffX + kXStages * kXBytes;
  static constexpr int kOffBar = (kOffW + kWStages * kWBytes + 1023) / 1024 * 1024;
  static constexpr int kNumBars = 2 * kXStagesMax + 2 * kWStages + 4 + 2 * kEpiGroups;
  static constexpr int kOffSA = kOffBar + (kNumBars * 8 + 16 + 15) / 16 * 16;  // per-token scales of a tile (f64)
  static constexpr int kOffRS = kOffSA + NTOK * 8;                             // per-token code sums (int32)
  static constexpr int kOffY = (kOffRS + NTOK * 4 + 127) / 128 * 128;  // per epilogue warp: 2 x [16 tok][32 ch] fp16
  // per group: kPartBufs x 8 KiB split-K partial chunks (1024-aligned when it doubles as an activation stage)
  static constexpr int kOffPart = kXStagesXtra ? (kOffY + kNumEpiWarps * kYWarpBytes + 1023) / 1024 * 1024
                                               : kOffY + kNumEpiWarps * kYWarpBytes;
  static constexpr int kSmemBytes = kOffPart + kEpiGroups * kPartBufs * 8192 + 1024;  // +1024 alignment slack
  static_assert(kSmemBytes <= kSmemBudget + 1024 && kSmemBytes * kCtasPerSm <= 227 * 1024,
                "over the per-CTA shared memory budget");
  static constexpr int kTmemNeed = kAccCols + kABufs * kACols;
  static_assert(kTmemNeed <= kTmemBudget, "TMEM over-subscribed");
  static constexpr uint32_t kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128
                                        : kTmemNeed <= 256 ? 256 : 512;
  // per-group: the converter emits w8 + 128 (no XOR); the MMA runs u8 x s8 and
  // the epilogue subtracts 128 * rowsum(a) — exact in int32 (K <= 65536)
  static constexpr bool kU8 = MODE == kModePG;
  static constexpr uint32_t kIdesc = make_idesc_i8(PAIR ? 256 : 128, kMmaN, kU8);
  static_assert(kMmaN % 16 == 0 && kMmaN >= 16 && kMmaN <= 256 && (kMmaSplit == 1 || PAIR), "invalid UMMA N");
  static_assert(BK % 128 == 0, "BK must be a multiple of the 128-byte swizzle atom");
};

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
QQQ_DEVICE unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// In-kernel timeline stamps exist only in the developer build (-DQQQ_TIMELINE,
// libqqq_b200_tl.so); the product build carries no instrumentation code.
#ifdef QQQ_TIMELINE
#define QQQ_STAMP(slot)                                                   \
  do {                                                                    \
    if (p.dbg) p.dbg[(size_t)blockIdx.x * kDbgSlots + (slot)] = gtimer(); \
  } while (0)
#else
#define QQQ_STAMP(slot) \
  do {                  \
  } while (0)
#endif

// whole-SM weight producer: spins (a suspended try_wait woke measurably late
// behind the converters' release; 1-2% at mid/prefill M)
#ifndef QQQ_WPROD_SLEEP
#define wprod_wait mbar_wait
#else
#define wprod_wait mbar_wait_sleep
#endif
#ifdef QQQ_XPROD_SPIN
#define xprod_wait mbar_wait
#else
#define xprod_wait mbar_wait_sleep
#endif
#ifdef QQQ_CONV_SLEEP
#define conv_wait mbar_wait_sleep
#else
#define conv_wait mbar_wait
#endif
#ifdef QQQ_MMA_SPIN
#define mma_wait mbar_wait
#else
#define mma_wait mbar_wait_sleep
#endif

// Programmatic dependent launch (PDL). No-ops without the launch attribute.
QQQ_DEVICE void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
QQQ_DEVICE void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

QQQ_DEVICE void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

QQQ_DEVICE __half f64_to_f16_rn(double v) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(v));
  return __ushort_as_half(h);
}

// 16 bytes into another cluster CTA's shared memory, completing 16 transaction
// bytes on that CTA's mbarrier (both shared::cluster addresses)
QQQ_DEVICE void st_async_v4(uint32_t cl_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t cl_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cl_addr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(cl_bar)
               : "memory");
}

QQQ_DEVICE void red_add_s32(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// pair mode: this CTA's half of the activation tile lands in its own shared
// memory; the transaction bytes complete on the EVEN CTA's barrier (cl_bar, a
// shared::cluster address), which the pair MMA issuer waits on
QQQ_DEVICE void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                 uint32_t cl_bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(cl_bar)
      : "memory");
}

QQQ_DEVICE void tma_load_3d(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(smem_dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Exact int32 -> f64 without the (quarter-rate) I2F.F64 unit:
// 2^52 + 2^31 + a is exactly representable; one DADD removes the bias.
QQQ_DEVICE double i32_to_f64_exact(int32_t a) {
  return __hiloint2double(0x43300000, (int)((uint32_t)a ^ 0x80000000u)) - 4503601774854144.0;
}

// y = f16((acc * s_a[t]) * s_col) for 16 tokens of one channel, branch-free:
// f64 with one final RN rounding (cvt.rn.f16.f64), as gemm.py:182-184/200-202.
// (only the first nvalid tokens are converted: rows past M are never stored)
QQQ_DEVICE void dequant16(const uint32_t (&r)[16], const double* sa, double s_col, uint16_t (&h)[16],
                          int nvalid = 16) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
#ifdef QQQ_EXP_NO_DEQ
    h[i] = (uint16_t)r[i];
#else
    if (i < nvalid) {
      const double v = (i32_to_f64_exact((int32_t)r[i]) * sa[i]) * s_col;
      h[i] = __half_as_ushort(f64_to_f16_rn(v));
    } else {
      h[i] = 0;
    }
#endif
  }
}

// The same for all 16 tokens, unpredicated (TMA-stored chunks: rows past M
// are clipped by the store, so their values are never written). Phases of 8
// independent conversions / products: the predicated per-token form compiled
// to one dependent DADD -> DMUL -> DMUL -> F2F chain after another and ran at
// half the FP64 pipe's rate (scripts/epi_probe.cu: 10 values/clk/SM).
QQQ_DEVICE void dequant16_all(const uint32_t (&r)[16], const double* sa, double s_col, uint16_t (&h)[16]) {
#pragma unroll
  for (int g = 0; g < 16; g += 8) {
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = i32_to_f64_exact((int32_t)r[g + i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] *= sa[g + i];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] *= s_col;
#pragma unroll
    for (int i = 0; i < 8; ++i) h[g + i] = __half_as_ushort(f64_to_f16_rn(d[i]));
  }
}

// ---- fused smoothed activation quantization (GemmParams::xsrc) ----
// The M x K activation block is cut into work items (row, slice of kQSlice
// channels) spread over every epilogue group (128 threads) of the first-wave
// CTAs, so a row's quotients are computed by several SMs at once:
//   phase A (all of a group's items, no waiting): x / s_k for the slice
//     (Markstein with the reciprocal table, IEEE division without it or where
//     the table holds NaN), slice absmax -> atomicMax on the row's slot,
//     release-increment of the row's phase-A count;
//   phase B (per item): wait for the row's phase-A count to reach its slice
//     count, s = m / 127, codes rint(RN(xs / s)) by Markstein for the slice,
//     partial code sum -> the row's sum slot, acq_rel-increment of the row's
//     phase-B count; the last slice of a row writes s_a and rowsum, re-arms the
//     row's slots and counts the row as published.
// The arithmetic is act_quant_row_kernel<.., kSmooth = true>'s (act_quant.cu),
// so q / s_a / rowsum are bit-identical to quant_act_smoothed's (the max is
// order-independent, the code sum an exact integer sum). Phase A never waits,
// so no group waits on an item another group has not started (deadlock-free
// among co-resident CTAs). Per-row slots (workspace head, zero on entry and
// exit): m (u64 bits of a non-negative double), code sum, phase-A and phase-B
// counts.
constexpr int kQSlice = 2048;                 // channels per work item (2 x 8 per thread)
QQQ_DEVICE int32_t* qrow_slots(const GemmParams& p) { return p.counters + kQRowsSlot - 6 * p.M - 2; }

QQQ_DEVICE void smooth_vecs(const GemmParams& p, int row, int slice, int gt, double (&xs)[2][8], bool& bad,
                            double& m) {
  const uint4* xr = reinterpret_cast<const uint4*>(p.xsrc + (int64_t)row * p.ldx);
  const int64_t nv = p.K / 8;
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const int64_t i = (int64_t)slice * (kQSlice / 8) + v * 128 + gt;
    if (i < nv) {
      smooth8(__ldg(xr + i), p.smooth, p.srecip, i, xs[v]);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double a = fabs(xs[v][t]);
        bad |= is_bad(a);
        m = a > m ? a : m;
      }
    }
  }
}

// Returns the number of rows this group finished (published by the caller).
QQQ_DEVICE int quantize_rows_fused(const GemmParams& p, int grp, int ngroups, int gt, uint8_t* scratch, int bar_id) {
  if ((int)blockIdx.x >= p.q_ctas) return 0;
  const int wq = gt >> 5, lane = gt & 31;
  const int S = (p.K + kQSlice - 1) / kQSlice;  // slices per row
  const int items = p.M * S;
  const int G = p.q_ctas * ngroups, g = grp * p.q_ctas + (int)blockIdx.x;
  int32_t* slots = qrow_slots(p);  // [M] u64 m | [M] sum | [M] cntA | [M] cntB
  unsigned long long* mslot = reinterpret_cast<unsigned long long*>(slots);
  int32_t* sumslot = slots + 2 * p.M;
  int32_t* cnta = sumslot + p.M;
  int32_t* cntb = cnta + p.M;
  double* red = reinterpret_cast<double*>(scratch);  // [4] per-warp maxima
  int* ired = reinterpret_cast<int*>(scratch + 32);   // [4] per-warp code sums
  // ---- phase A
#pragma unroll 1
  for (int it = g; it < items; it += G) {
    const int row = it / S, slice = it % S;
    double xs[2][8];
    double m = 0.0;
    bool bad = false;
    smooth_vecs(p, row, slice, gt, xs, bad, m);
    if (bad) atomicOr(p.status, kStatNonFinite);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, m, o);
      m = t > m ? t : m;
    }
    if (lane == 0) red[wq] = m;
    named_bar_sync(bar_id, 128);
    if (gt == 0) {
#pragma unroll
      for (int w = 0; w < 4; ++w) m = red[w] > m ? red[w] : m;
      atomicMax(mslot + row, (unsigned long long)__double_as_longlong(m));
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnta + row) : "memory");
    }
    named_bar_sync(bar_id, 128);  // red[] reused by the next item
  }
  // ---- phase B
  if (gt == 0 && grp == 0) QQQ_STAMP(177);
  int rows = 0;
#pragma unroll 1
  for (int it = g; it < items; it += G) {
    const int row = it / S, slice = it % S;
    if (gt == 0) {
      unsigned long long t0 = 0;
#pragma unroll 1
      for (uint32_t n = 0;; ++n) {
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnta + row) : "memory");
        if (v >= S) break;
        __nanosleep(32);
#ifndef QQQ_NO_WATCHDOG
        if ((n & 1023) == 1023) {
          const unsigned long long t = gtimer();
          if (t0 == 0)
            t0 = t;
          else if (t - t0 > QQQ_WATCHDOG_NS)
            __trap();
        }
#endif
      }
    }
    named_bar_sync(bar_id, 128);
    unsigned long long mb;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(mb) : "l"(mslot + row) : "memory");
    const double m = __longlong_as_double((long long)mb);
    const double s = (m > 0.0) ? m / 127.0 : 1.0;
    const double rs = 1.0 / s;
    const bool ieee = !markstein_safe(s);
    double xs[2][8];
    double mm = 0.0;
    bool bad = false;
    smooth_vecs(p, row, slice, gt, xs, bad, mm);  // (recomputed: registers are not held across phase A)
    int8_t* qr = p.qdst + (int64_t)row * p.ldq;
    const int64_t nv = p.K / 8;
    int csum = 0;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int64_t i = (int64_t)slice * (kQSlice / 8) + v * 128 + gt;
      if (i < nv) {
        *reinterpret_cast<uint2*>(qr + i * 8) = codes8_f64(xs[v], s, rs, ieee, csum);
      }
    }
    // codes are read by other CTAs' tensor TMA (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if (lane == 0) ired[wq] = csum;
    named_bar_sync(bar_id, 128);
    if (gt == 0) {
      const int part = ired[0] + ired[1] + ired[2] + ired[3];
      atomicAdd(sumslot + row, part);
      int prev;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(cntb + row) : "memory");
      if (prev == S - 1) {  // the row's last slice: every slice's sum and codes are visible
        int total;
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(total) : "l"(sumslot + row) : "memory");
        p.sa_dst[row] = s;
        p.rs_dst[row] = total;
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(mslot + row), "l"(0ull) : "memory");
        asm volatile("st.relaxed.gpu.global.s32 [%0], 0;" ::"l"(sumslot + row) : "memory");
        asm volatile("st.relaxed.gpu.global.s32 [%0], 0;" ::"l"(cnta + row) : "memory");
        asm volatile("st.relaxed.gpu.global.s32 [%0], 0;" ::"l"(cntb + row) : "memory");
        ++rows;
      }
    }
    named_bar_sync(bar_id, 128);  // ired[] reused by the next item
  }
  return rows;  // (meaningful in thread gt == 0)
}

// Publish the rows this group finished: one gpu-scope release of the count
// (the finishing thread acquired every slice of those rows).
QQQ_DEVICE void publish_rows_fused(const GemmParams& p, int rows, int gt, int bar_id) {
  (void)bar_id;
  if (gt == 0 && rows > 0)
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p.counters + kQRowsSlot), "r"(rows) : "memory");
}

// Wait until all M rows are published (acquire), then order this thread's
// later async-proxy (TMA) reads after it. Co-residency: only CTAs of the first
// wave quantize and they wait on nothing before publishing.
QQQ_DEVICE void wait_rows_fused(const GemmParams& p) {
  const int32_t* c = p.counters + kQRowsSlot;
  unsigned long long t0 = 0;
#pragma unroll 1
  for (uint32_t n = 0;; ++n) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (v >= p.M) break;
    __nanosleep(32);
#ifndef QQQ_NO_WATCHDOG
    if ((n & 1023) == 1023) {
      const unsigned long long t = gtimer();
      if (t0 == 0)
        t0 = t;
      else if (t - t0 > QQQ_WATCHDOG_NS)
        __trap();
    }
#endif
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Dequant epilogue for up to 16 consecutive tokens of one output channel n:
// y = f16((acc * s_a[t]) * s_col[n]) in f64 with one final RN rounding
// (gemm.py:182-184 / 200-202); acc written as-is when requested.
// Direct (per-element) stores: used for the optional int32 acc output and for
// y when its row pitch does not allow a TMA store.
QQQ_DEVICE void store_outputs(const GemmParams& p, const uint32_t (&r)[16], const double* sa, int t0, int nvalid,
                              int n, bool n_ok, double s_col) {
  if (!n_ok) return;
  if (p.acc) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nvalid) p.acc[(int64_t)(t0 + i) * p.ldacc + n] = (int32_t)r[i];
  }
  if (p.s_col && !p.y_tma) {
    uint16_t h[16];
    dequant16_all(r, sa, s_col, h);  // (entries past nvalid are computed but not stored)
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nvalid) reinterpret_cast<uint16_t*>(p.y)[(int64_t)(t0 + i) * p.ldy + n] = h[i];
  }
}

QQQ_DEVICE void tma_store_2d(const CUtensorMap* map, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
// bulk reduction of a shared-memory block into global memory (int32 add, done
// in L2 at bulk bandwidth; replaces per-element atomics for split-K partials)
QQQ_DEVICE void bulk_reduce_add_s32(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.s32 [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
QQQ_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
QQQ_DEVICE void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
QQQ_DEVICE void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Segment iterator: the CTA's contiguous (tile, k-block) unit range split at tile borders.
// A CTA's work: up to two contiguous (tile, k-block) unit ranges, iterated in
// order and split at tile borders: [u, u1) then [v, v1) (hybrid plans: whole
// data-parallel tiles first, then the stream-K share).
// (32-bit unit indices: units = tiles x k-blocks < 65536 x 512. Every warp
// role keeps an iterator live across its whole loop; 64-bit state was spilled
// to local memory, and a spill reload after a long barrier wait missed L1 and
// cost an L2 round trip on the decode critical path.)
struct SegIter {
  int u, u1, v, v1;
  int kbt;
  QQQ_DEVICE int total() const { return (u1 - u) + (v1 - v); }
  QQQ_DEVICE bool next(int& tile, int& kb0, int& kb1) {
    if (u >= u1) {
      if (v >= v1) return false;
      u = v;
      u1 = v1;
      v = v1;
    }
    tile = u / kbt;
    kb0 = u - tile * kbt;
    const int rem = u1 - u;
    kb1 = (kbt - kb0) < rem ? kbt : kb0 + rem;
    u += kb1 - kb0;
    return true;
  }
};

QQQ_DEVICE SegIter make_iter(const GemmParams& p) {
  SegIter it;
  it.kbt = p.kb_per_tile;
  it.v = it.v1 = 0;
  if (p.csplit > 1) {  // cluster split-K: one tile per cluster, an even k-range per rank
    const int c = blockIdx.x / p.csplit, r = blockIdx.x % p.csplit;
    it.u = c * p.kb_per_tile + r * p.kb_per_tile / p.csplit;
    it.u1 = c * p.kb_per_tile + (r + 1) * p.kb_per_tile / p.csplit;
    return it;
  }
  if (p.aligned_tiles > 0) {
    // pair plans: the CTA pair (2b, 2b+1) owns 256-channel pair tiles
    const int64_t tiles = (int64_t)(p.pair ? (p.n_tiles + 1) / 2 : p.n_tiles) * p.tok_tiles;
    int64_t t0 = (int64_t)(p.pair ? blockIdx.x >> 1 : blockIdx.x) * p.aligned_tiles;
    int64_t t1 = t0 + p.aligned_tiles < tiles ? t0 + p.aligned_tiles : tiles;
    if (t0 > tiles) t0 = tiles;
    if (t1 < t0) t1 = t0;
    it.u = (int)(t0 * p.kb_per_tile);
    it.u1 = (int)(t1 * p.kb_per_tile);
  } else {
    // (pair plans: the stream-K "CTA" is the CTA pair; both CTAs take the same units)
    const int64_t b = p.pair ? blockIdx.x >> 1 : blockIdx.x, G = p.pair ? gridDim.x >> 1 : gridDim.x;
    it.u = (int)(p.sk_unit0 + b * p.units / G);
    it.u1 = (int)(p.sk_unit0 + (b + 1) * p.units / G);
    if (p.dp_tiles > 0) {
      it.v = it.u;
      it.v1 = it.u1;
      it.u = (int)(b * p.dp_tiles * p.kb_per_tile);
      it.u1 = it.u + p.dp_tiles * p.kb_per_tile;
    }
  }
  return it;
}

// stream-K: the CTA whose stream-K range contains unit u (start(b) = sk_unit0 + floor(b*U/G))
QQQ_DEVICE int cta_of_unit(int64_t u, const GemmParams& p, int grid) {
  return (int)(((u - p.sk_unit0 + 1) * grid - 1) / p.units);
}

// Incremental (n_tile, token tile, k-block) cursor over consecutive units of a
// stream-K range: one division at construction, none per step.
struct UnitCursor {
  int n_tile, tt, kb;
  QQQ_DEVICE UnitCursor(const GemmParams& p, int64_t u) {
    const int tile = (int)(u / p.kb_per_tile);
    n_tile = tile / p.tok_tiles;
    tt = tile % p.tok_tiles;
    kb = (int)(u % p.kb_per_tile);
  }
  QQQ_DEVICE void adv(const GemmParams& p) {
    if (++kb == p.kb_per_tile) {
      kb = 0;
      if (++tt == p.tok_tiles) {
        tt = 0;
        ++n_tile;
      }
    }
  }
};

// one weight k-block (BK/128 super-slabs of one 128-channel tile) -> ring stage
template <int BK>
QQQ_DEVICE void issue_weight_kblock(const GemmParams& p, const UnitCursor& c, uint8_t* dst, uint64_t* bar) {
  const int nss = min(BK / 128, p.ss_per_tile - c.kb * (BK / 128));
  const uint32_t wbytes = (uint32_t)(nss * p.ss_bytes);
  const int64_t ss0 = (int64_t)c.n_tile * p.ss_per_tile + (int64_t)c.kb * (BK / 128);
  mbar_arrive_expect_tx(bar, wbytes);
  bulk_g2s(dst, p.w + ss0 * p.ss_bytes, wbytes, bar);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int MODE, int NTOK, int BK, bool PAIR>
__global__ void __launch_bounds__(Cfg<MODE, NTOK, BK, PAIR>::kNumThreads, Cfg<MODE, NTOK, BK, PAIR>::kCtasPerSm)
    w4a8_gemm_kernel(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap y_map,
                     const GemmParams p) {
  using C = Cfg<MODE, NTOK, BK, PAIR>;
  static_assert(!PAIR || (C::kConvert && !C::kSmall), "pair mode: prefill convert tiles");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kb_full = bars;                   // [kXStages] activations landed + A buffer converted
  uint64_t* kb_empty = kb_full + C::kXStagesMax;  // [kXStages] MMA done with activation stage / A buffer
  uint64_t* w_full = kb_empty + C::kXStagesMax;
  uint64_t* w_empty = w_full + C::kWStages;
  uint64_t* acc_full = w_empty + C::kWStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* part_full = acc_empty + 2;  // [group][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::kNumBars);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Pair mode: CTA rank 0 of the cluster ("even" CTA) issues the pair MMAs and
  // owns the barriers they wait on (k-block full: both CTAs' activation bytes
  // and converter arrivals; accumulator empty: both CTAs' epilogues); the
  // MMA commits arrive on the barrier copies of both CTAs.
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  // output-channel tile of a (pair) tile index
  auto ntile_of = [&](int tile) -> int {
    return PAIR ? (tile / p.tok_tiles) * 2 + (int)crank : tile / p.tok_tiles;
  };

  if (threadIdx.x == 0) {
    QQQ_STAMP(0);
#ifdef QQQ_TIMELINE
    if (p.dbg) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.dbg[(size_t)blockIdx.x * kDbgSlots + 191] = smid;
    }
#endif
    griddep_launch_dependents();
    for (int s = 0; s < C::kXStagesMax; ++s) {
      mbar_init(&kb_full[s], C::kConvert ? (PAIR ? 2 : 1) * C::kConvPerGroup + 1 : 1);
      mbar_init(&kb_empty[s], 1);
    }
    if (!C::kSmall) {  // small CTAs: the producer warp owns (and initialises) its weight ring
      for (int s = 0; s < C::kWStages; ++s) {
        mbar_init(&w_full[s], 1);
        mbar_init(&w_empty[s], C::kConvert ? C::kConvPerGroup : 1);
      }
    }
    for (int j = 0; j < C::kAccBufs; ++j) {
      mbar_init(&acc_full[j], 1);
      mbar_init(&acc_empty[j], (PAIR ? 2 : 1) * C::kNumEpiWarps);
    }
    for (int i = 0; i < 2 * C::kEpiGroups; ++i)  // (big-CTA cluster split-K, L2 exchange: part_full[1] counts the S-1 peers)
      mbar_init(&part_full[i], (QQQ_CSB_L2 && i == 1 && !C::kSmall && !PAIR && NTOK == 128 && p.csplit > 1) ? p.csplit - 1 : 1);
    mbar_fence_init();
  }
  if (warp == C::kActProducerWarp && lane == 0) tma_prefetch_desc(&act_map);
  if (warp == C::kAllocWarp) {
    if constexpr (PAIR)
      tmem_alloc_pair(tmem_slot, C::kTmemCols);
    else
      tmem_alloc(tmem_slot, C::kTmemCols);
  }
  if (C::kSmall && warp == C::kWProducerWarp) {
    // The first weight copies do not wait for the CTA set-up (TMEM allocation,
    // other barriers): the decode critical path starts with this HBM latency.
    if (lane == 0) {
      for (int s = 0; s < C::kWStages; ++s) {
        mbar_init(&w_full[s], 1);
        mbar_init(&w_empty[s], C::kNumConvWarps);
      }
      mbar_fence_init();
    }
    __syncwarp();
    SegIter si0 = make_iter(p);
    const int total = (int)si0.total();
    UnitCursor c(p, si0.u);
    for (int i = 0; i < C::kWStages && i < total; ++i) {
      if (elect_one()) issue_weight_kblock<BK>(p, c, smem + C::kOffW + i * C::kWBytes, &w_full[i]);
      __syncwarp();
      c.adv(p);
    }
  }
  tc_fence_before();
  // The TMEM base address (written to shared memory by tcgen05.alloc) and the
  // barrier inits are published to the CTA by bar.sync. The cluster barrier
  // below uses a RELAXED arrive (a .release arrive is a per-thread MEMBAR.GPU),
  // which orders nothing: with it alone, warps of cluster CTAs read a stale
  // tmem_slot now and then (left by the SM's previous CTA) and converted into
  // another CTA's TMEM columns.
  __syncthreads();
  if (PAIR || p.csplit > 1)
    cluster_sync_all();  // every cluster CTA's barriers initialised before any remote arrive / store
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // activation ring / TMEM A ring size of this launch (see Cfg::kXStagesXtra)
  const int nx = (C::kXStagesXtra && p.aligned_tiles > 0 && p.csplit <= 1) ? C::kXStagesMax : C::kXStages;
  auto xstage = [&](int st) -> uint8_t* {
    return st < C::kXStages ? smem + C::kOffX + st * C::kXBytes : smem + C::kOffPart;
  };
  // the even CTA's k-block-full and accumulator-empty barriers (pair mode)
  const uint32_t kb_full_cl = PAIR ? mapa_shared(kb_full, 0) : 0u;
  const uint32_t acc_empty_cl = PAIR ? mapa_shared(acc_empty, 0) : 0u;

  // The single-issuer roles (producers, MMA) run their loops with the whole
  // warp converged and elect one lane per async instruction: the operands are
  // then warp-uniform and live in uniform registers. Issuing tcgen05.mma from
  // a divergent single lane costs ~150 cycles per MMA (R2UR waterfall,
  // scripts/mma_probe.cu) against a 16-cycle issue floor at N = 16.
#ifndef QQQ_SMALL_TWO_PRODUCERS
  if (C::kSmall && warp == C::kWProducerWarp) {
    // ========== producer warp (small CTA): weight + activation rings ==========
    // One in-order loop over this CTA's k-blocks i = 0..total-1: the weight
    // stage of k-block i is refilled (k-block i + kWStages) once the
    // converters released it, the activation slot of k-block i once its MMAs
    // retired. The weight prologue is issued before the PDL wait (weights
    // never depend on the previous kernel).
    SegIter si = make_iter(p);
    const int total = (int)si.total();  // small CTAs: a single stream-K range (no data-parallel part)
    UnitCursor wc(p, si.u), xc = wc;
    uint32_t wi = 0, xi = 0;  // ring slots of the next copies
    auto issue_w = [&]() {
      if (elect_one()) issue_weight_kblock<BK>(p, wc, smem + C::kOffW + wi * C::kWBytes, &w_full[wi]);
      __syncwarp();
      wc.adv(p);
      if (++wi == C::kWStages) wi = 0;
    };
    auto issue_x = [&]() {
      if (elect_one()) {
        mbar_arrive_expect_tx(&kb_full[xi], C::kXBytes);
        tma_load_3d(smem + C::kOffX + xi * C::kXBytes, &act_map, 0, xc.tt * NTOK, xc.kb * (BK / 128), &kb_full[xi]);
      }
      __syncwarp();
      xc.adv(p);
      if (++xi == C::kXStages) xi = 0;
    };
    // the weight prologue was issued before the set-up barrier: advance past it
    for (int i = 0; i < C::kWStages && i < total; ++i) {
      wc.adv(p);
      if (++wi == C::kWStages) wi = 0;
    }
    griddep_wait();  // the int8 activations come from the previous kernel
    if (lane == 0) QQQ_STAMP(3);
    if (p.xsrc) {  // ... or from this kernel's fused quantization
      if (lane == 0) wait_rows_fused(p);
      __syncwarp();
      if (lane == 0) QQQ_STAMP(180);
    }
    for (int i = 0; i < C::kXStages && i < total; ++i) issue_x();
    if (lane == 0) QQQ_STAMP(181);
    uint32_t ws = 0, wph = 0, xs = 0, xph = 0;
#pragma unroll 1
    for (int i = 0; i < total; ++i) {
      if (i + C::kWStages < total) {
        mbar_wait_sleep(&w_empty[ws], wph);
        issue_w();
      }
      if (++ws == C::kWStages) {
        ws = 0;
        wph ^= 1;
      }
      if (i + C::kXStages < total) {
        mbar_wait_sleep(&kb_empty[xs], xph);
        issue_x();
        if (lane == 0 && i < 16) QQQ_STAMP(112 + i);
      }
      if (++xs == C::kXStages) {
        xs = 0;
        xph ^= 1;
      }
    }
  } else
#endif
  if (warp == C::kWProducerWarp) {
    // ===================== weight producer (bulk copies) =====================
    // Weights never depend on the previous kernel in the stream: no PDL wait,
    // so under PDL they stream in while the previous kernel drains. (Small
    // CTAs issued the first kWStages k-blocks before the set-up barrier.)
    if (lane == 0) QQQ_STAMP(1);
    SegIter si = make_iter(p);
    int tile, kb0, kb1;
    uint32_t s = 0, ph = 0;
    int i = 0;
    const int pre = C::kSmall ? (si.total() < C::kWStages ? si.total() : C::kWStages) : 0;
    while (si.next(tile, kb0, kb1)) {
      // (pair mode, odd channel-tile count: the missing last tile converts a copy of
      //  a real one; its rows are never stored)
      const int n_tile = min(ntile_of(tile), p.n_tiles - 1);
#pragma unroll 1
      for (int kb = kb0; kb < kb1; ++kb, ++i) {
        if (i >= pre) {
          wprod_wait(&w_empty[s], ph ^ 1);
          if (elect_one()) {
            // the last k-block of a tile may hold fewer super-slabs (K_pad % BK != 0):
            // the stale rest of the stage meets zero-filled (OOB) activations
            const int nss = min(BK / 128, p.ss_per_tile - kb * (BK / 128));
            const uint32_t wbytes = (uint32_t)(nss * p.ss_bytes);
            mbar_arrive_expect_tx(&w_full[s], wbytes);
            if (i < 16) QQQ_STAMP(155 + i);
            const int64_t ss0 = (int64_t)n_tile * p.ss_per_tile + (int64_t)kb * (BK / 128);
            bulk_g2s(smem + C::kOffW + s * C::kWBytes, p.w + ss0 * p.ss_bytes, wbytes, &w_full[s]);
          }
          __syncwarp();
        }
        if (++s == C::kWStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    if (lane == 0) QQQ_STAMP(2);
  } else if (warp == C::kActProducerWarp) {
    // ================== activation producer (3-D tensor TMA) ==================
    griddep_wait();  // the int8 activations come from the previous kernel
    if (p.xsrc) {  // ... or from this kernel's fused quantization
      if (lane == 0) wait_rows_fused(p);
      __syncwarp();
      if (lane == 0) QQQ_STAMP(180);
    }
    if (lane == 0) QQQ_STAMP(3);
    SegIter si = make_iter(p);
    int tile, kb0, kb1;
    uint32_t s = 0, ph = 0, xit = 0;
    while (si.next(tile, kb0, kb1)) {
      const int tok0 = (tile % p.tok_tiles) * NTOK;
#pragma unroll 1
      for (int kb = kb0; kb < kb1; ++kb, ++xit) {
        xprod_wait(&kb_empty[s], ph ^ 1);
        if (lane == 0 && xit < 16) QQQ_STAMP(112 + xit);
        if (elect_one()) {
          if constexpr (PAIR) {
            // each CTA loads its half of the tokens; the bytes of both count on the even CTA's barrier
            if (crank == 0) mbar_arrive_expect_tx(&kb_full[s], 2 * C::kXBytes);
            if constexpr (C::kMmaSplit == 2) {
              constexpr int kHalf = C::kTokLoad / 2;  // 96 rows per chunk
              tma_load_3d_pair(xstage(s), &act_map, 0, tok0 + (int)crank * kHalf,
                               kb * (BK / 128), kb_full_cl + s * 8);
              tma_load_3d_pair(xstage(s) + kHalf * 128, &act_map, 0,
                               tok0 + NTOK / 2 + (int)crank * kHalf, kb * (BK / 128), kb_full_cl + s * 8);
            } else {
              tma_load_3d_pair(xstage(s), &act_map, 0, tok0 + (int)crank * C::kTokLoad,
                               kb * (BK / 128), kb_full_cl + s * 8);
            }
          } else {
#ifdef QQQ_EXP_HALF_X
            mbar_arrive_expect_tx(&kb_full[s], NTOK >= 128 ? C::kXBytes / 2 : C::kXBytes);
#else
            mbar_arrive_expect_tx(&kb_full[s], C::kXBytes);
#endif
            tma_load_3d(xstage(s), &act_map, 0, tok0, kb * (BK / 128), &kb_full[s]);
          }
        }
        __syncwarp();
        if (++s == nx) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == C::kMmaWarp && crank == 0) {
    // ============================ MMA issuer ============================
    // (pair mode: the even CTA issues for both; the odd CTA's MMA warp idles)
    SegIter si = make_iter(p);
    int tile, kb0, kb1;
    uint32_t it = 0, seg = 0;
    uint32_t xs = 0, xph = 0, ws = 0, wph = 0, j = 0, jph = 0;
    while (si.next(tile, kb0, kb1)) {
      if constexpr (PAIR)
        mbar_wait_cluster(&acc_empty[j], jph ^ 1);
      else
        mbar_wait_sleep(&acc_empty[j], jph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + j * NTOK;
#pragma unroll 1
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        if constexpr (PAIR)
          mbar_wait_cluster(&kb_full[xs], xph);
        else
          mma_wait(&kb_full[xs], xph);  // activations landed and (convert modes) the A buffer is converted
        if (lane == 0 && it < 16) QQQ_STAMP(96 + it);
        if constexpr (!C::kConvert) mma_wait(&w_full[ws], wph);
        tc_fence_after();
        const uint32_t act_addr = smem_u32(xstage(xs));
        const uint64_t b_desc0 = make_smem_desc(act_addr, 16, 1024, 2);
        const uint32_t a_tmem = tmem_base + C::kAccCols + xs * C::kACols;  // TMEM column address (convert modes)
        const uint32_t a_smem = smem_u32(smem + C::kOffW + ws * C::kWBytes);  // I8 mode
        const uint32_t acc0 = kb > kb0 ? 1u : 0u;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk) {
            // B: SWIZZLE_128B [k-atom][NTOK rows][128 B]; 32 B K-steps inside the atom
            const uint64_t b_desc = b_desc0 + (uint64_t)(((kk / 4) * (C::kTokLoad * 128) + (kk % 4) * 32) >> 4);
            const uint32_t acc = kk > 0 ? 1u : acc0;
            if constexpr (PAIR && C::kMmaSplit == 2) {
              static_assert(BK == 128, "384-token tiles: one 128-byte swizzle atom per k-block");
              mma_i8_ts_pair(d_tmem, a_tmem + kk * 8, b_desc, C::kIdesc, acc);
              mma_i8_ts_pair(d_tmem + C::kMmaN, a_tmem + kk * 8, b_desc + (uint64_t)((C::kTokLoad / 2 * 128) >> 4),
                             C::kIdesc, acc);
            } else if constexpr (PAIR) {
              mma_i8_ts_pair(d_tmem, a_tmem + kk * 8, b_desc, C::kIdesc, acc);
            } else if constexpr (C::kConvert) {
              mma_i8_ts(d_tmem, a_tmem + kk * 8, b_desc, C::kIdesc, acc);  // A: 8 TMEM columns per K=32
            } else {
              // A: canonical K-major, no swizzle: [k16 chunk][128 rows][16 B]
              mma_i8_ss(d_tmem, make_smem_desc(a_smem + kk * 2 * 2048, 2048, 128, 0), b_desc, C::kIdesc, acc);
            }
          }
          if constexpr (PAIR)
            mma_commit_pair(&kb_empty[xs], 0x3);
          else
            mma_commit(&kb_empty[xs]);
          if constexpr (!C::kConvert) mma_commit(&w_empty[ws]);
        }
        __syncwarp();
        if (lane == 0 && it < 16) QQQ_STAMP(20 + it);
        if (++xs == nx) {
          xs = 0;
          xph ^= 1;
        }
        if constexpr (!C::kConvert) {
          if (++ws == C::kWStages) {
            ws = 0;
            wph ^= 1;
          }
        }
      }
      if (elect_one()) {
        if constexpr (PAIR)
          mma_commit_pair(&acc_full[j], 0x3);
        else
          mma_commit(&acc_full[j]);
      }
      __syncwarp();
      if (++j == C::kAccBufs) {
        j = 0;
        jph ^= 1;
      }
      ++seg;
    }
  } else if (warp >= C::kConvWarp0 && warp < C::kConvWarp0 + C::kNumConvWarps) {
    // ====================== INT4 -> INT8 converters ======================
    // Warp w owns TMEM lane quadrant q = w % 4 (rows 32q..32q+31) and every
    // other 32-k slab (parity w / 4): thread = one output channel.
    if constexpr (C::kConvert) {
#ifdef QQQ_EXP_CONV_AFTER_WAIT
      griddep_wait();  // experiment: no conversion while the previous kernel runs
#endif
      constexpr int kPhases = C::kConvPerGroup / 4;
      const int q = warp & 3, h = (warp >> 2) % kPhases;  // quadrant, slab phase (0..kPhases-1)
      const int grp = (warp >> 2) / kPhases;               // k-block interleaving group
      const bool stamp_warp = warp % C::kConvPerGroup == 0;
      const int row = q * 32 + lane;
      constexpr int kSlabs = BK / 32 / kPhases;  // slabs per warp per k-block
      uint32_t magic;
      asm("mov.b32 %0, 0x64006400;" : "=r"(magic));  // a register operand for the fused and-or lop3
      // loop-invariant shared-memory offsets (inside a weight stage) of this
      // thread's packed slabs and group scales, and its TMEM column offsets
      uint32_t voff[kSlabs], soff[kSlabs];
      {
        const int geff = p.group < 128 ? p.group : 128;
#pragma unroll
        for (int i = 0; i < kSlabs; ++i) {
          const int c = h + kPhases * i;
          voff[i] = (uint32_t)((c >> 2) * p.ss_bytes + ((c & 3) * 128 + row) * 16);
          soff[i] = (uint32_t)((c >> 2) * p.ss_bytes + 8192 + ((((c & 3) * 32) / geff) * 128 + row) * 2);
        }
      }
      const uint32_t a_lane = tmem_base + ((uint32_t)(q * 32) << 16) + C::kAccCols + h * 8;
      const uint32_t wst0 = smem_u32(smem + C::kOffW);
      SegIter si = make_iter(p);
      int tile, kb0, kb1;
      uint32_t ws = 0, wph = 0, ab = 0, aph = 0, it = 0;
      while (si.next(tile, kb0, kb1)) {
#pragma unroll 1
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          if (C::kConvGroups > 1 && (int)(it % C::kConvGroups) != grp) {  // the other group's k-block
            if (++ws == C::kWStages) {
              ws = 0;
              wph ^= 1;
            }
            if (++ab == nx) {
              ab = 0;
              aph ^= 1;
            }
            continue;
          }
          conv_wait(&w_full[ws], wph);
          if (stamp_warp && lane == 0 && it < 16) QQQ_STAMP(4 + it);
          const uint32_t wst = wst0 + ws * C::kWBytes;
          uint4 v[kSlabs];
          uint32_t s1[kSlabs];
#pragma unroll
          for (int i = 0; i < kSlabs; ++i) {  // all shared loads first (ILP)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w)
                         : "r"(wst + voff[i]));
            if constexpr (MODE == kModePG) {
              uint16_t sv;
              asm volatile("ld.shared.u16 %0, [%1];" : "=h"(sv) : "r"(wst + soff[i]));
              s1[i] = sv;
            }
          }
          // Release the packed stage as soon as its bytes are in registers (before
          // the conversion), so the producer refills it one conversion earlier.
          // The arrive must not issue before the loads have RETURNED (LDS is
          // asynchronous: an arrive without a data dependency lets the producer's
          // next copy overwrite the stage under loads still in flight, which
          // corrupted one TMEM lane quadrant's A rows now and then): fold the last
          // word of every slab (and the scales) into a zero offset of the barrier
          // address. The zero must be opaque to ptxas (p.zero): it folded a
          // literal `and 0` and issued the arrive right behind the loads.
          {
            uint32_t dep = 0;
#pragma unroll
            for (int i = 0; i < kSlabs; ++i) {
              dep ^= v[i].w;
              if constexpr (MODE == kModePG) dep ^= s1[i];
            }
#ifdef QQQ_EXP_NODEP
            asm volatile("" ::"r"(dep));
            dep = 0;
#else
            asm volatile("and.b32 %0, %0, %1;" : "+r"(dep) : "r"(p.zero));
#endif
            // one arrive per warp (the loads are one instruction per slab for the
            // whole warp, so lane 0's data dependency covers every lane).
            // (Per-lane arrives with a 32x arrival count were measured to complete
            // the phase early — stages refilled under the readers — so the
            // warp-level release stays.)
            // a per-warp named barrier (ids 8-15) rather than __syncwarp: the same
            // ordering, in a form compute-sanitizer racecheck follows (measured
            // perf-neutral)
            named_bar_sync(8 + (warp & 7), 32);
            if (lane == 0) mbar_arrive_addr(smem_u32(&w_empty[ws]) + dep);
          }
          if (++ws == C::kWStages) {
            ws = 0;
            wph ^= 1;
          }
          uint32_t o[kSlabs][8];
#pragma unroll
          for (int i = 0; i < kSlabs; ++i) {
#ifdef QQQ_EXP_NO_CONV
            o[i][0] = v[i].x; o[i][1] = v[i].y; o[i][2] = v[i].z; o[i][3] = v[i].w;
            o[i][4] = v[i].x ^ s1[i]; o[i][5] = v[i].y; o[i][6] = v[i].z; o[i][7] = v[i].w;
            continue;
#endif
            if constexpr (MODE == kModePC) {
              pc_convert_word(v[i].x, o[i][0], o[i][4]);
              pc_convert_word(v[i].y, o[i][1], o[i][5]);
              pc_convert_word(v[i].z, o[i][2], o[i][6]);
              pc_convert_word(v[i].w, o[i][3], o[i][7]);
            } else {
              const __half2 s2 = u32_as_h2(s1[i] | (s1[i] << 16));
              const __half2 s16 = __hmul2(s2, u32_as_h2(0x2C002C00u));  // * 1/16
              pg_convert_word<false, true>(v[i].x, s2, s16, magic, o[i][0], o[i][1]);
              pg_convert_word<false, true>(v[i].y, s2, s16, magic, o[i][2], o[i][3]);
              pg_convert_word<false, true>(v[i].z, s2, s16, magic, o[i][4], o[i][5]);
              pg_convert_word<false, true>(v[i].w, s2, s16, magic, o[i][6], o[i][7]);
            }
          }
          conv_wait(&kb_empty[ab], aph ^ 1);
          // the wait loop exits per lane: reconverge before the .sync.aligned
          // tcgen05.st / wait::st
#ifndef QQQ_EXP_NOSYNC
          __syncwarp();
#endif
          tc_fence_after();
          if (stamp_warp && lane == 0 && it < 16) QQQ_STAMP(64 + it);
          const uint32_t abase = a_lane + ab * C::kACols;
#ifndef QQQ_EXP_NO_STTM
#pragma unroll
          for (int i = 0; i < kSlabs; ++i) tmem_st8(abase + kPhases * i * 8, o[i]);
          tmem_wait_st();
          // keep the source registers of the asynchronous stores live (unreused)
          // until tcgen05.wait::st has returned
#ifndef QQQ_EXP_NOKEEP
#pragma unroll
          for (int i = 0; i < kSlabs; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) asm volatile("" ::"r"(o[i][j]));
#endif
#else
          if (o[0][0] == 0x12345678u && o[kSlabs - 1][7] == 0x9abcdef0u) tmem_st8(abase, o[0]);
#endif
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR)
              mbar_arrive_cluster(kb_full_cl + ab * 8);
            else
              mbar_arrive(&kb_full[ab]);
          }
          if (++ab == nx) {
            ab = 0;
            aph ^= 1;
          }
          if (stamp_warp && lane == 0 && it < 16) QQQ_STAMP(80 + it);
        }
      }
    }
  } else if (warp >= C::kEpiWarp0 && warp < C::kEpiWarp0 + C::kNumEpiWarps) {
    // ============================== epilogue ==============================
    // Whole tiles go straight from TMEM to y. A tile split over CTAs
    // b_first..b_last (stream-K) is finished by its OWNER b_first, for which it
    // is the last segment of its range; the other CTAs handle it first in
    // theirs, store their int32 partial to a workspace slot and release an
    // arrival counter. The owner acquires the counter, adds the partials to its
    // own TMEM accumulator (exact integer sum) and applies the dequant. All
    // CTAs of the grid are co-resident (grid <= #SMs), so the wait cannot
    // deadlock, and it is normally already satisfied.
    // two halves of 4 warps (each covering all 128 TMEM lanes) take alternate
    // 16-token chunks: half the per-thread work, same TMEM/partial/y protocol
    constexpr int H = C::kEpiGroups;
    const int eh = (warp - C::kEpiWarp0) >> 2;
    const int q = warp & 3;  // TMEM lane quadrant accessible to this warp
    const int row = q * 32 + lane;
    // The first segment's column scale is weight metadata (never written by the
    // previous kernel, like the weights): load it before the PDL wait so the
    // decode epilogue does not pay a cold HBM round trip after the MMAs.
    int n_first = -1;
    double s_col_first = 0.0;
    {
      SegIter pk = make_iter(p);
      int t_, a_, b_;
      if (pk.next(t_, a_, b_)) {
        n_first = ntile_of(t_) * 128 + row;
#ifndef QQQ_EXP_NOSCOL
        if (n_first < p.N && p.s_col)
          asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(s_col_first) : "l"(p.s_col + n_first));
#else
        n_first = -1;
#endif
      }
    }
    griddep_wait();  // y / acc / workspace / counters / s_a may belong to the previous kernel
    if (p.xsrc) {
      // fused smoothed quantization: this group's token rows, then wait for all of them
      const int gq = warp - C::kEpiWarp0;
      const int grp = gq >> 2, gt = (gq & 3) * 32 + lane;
      if (threadIdx.x == C::kEpiWarp0 * 32) QQQ_STAMP(176);
      const int rows = quantize_rows_fused(p, grp, C::kEpiGroups, gt, smem + C::kOffY + (grp * 4) * C::kYWarpBytes, 2 + grp);
      if (threadIdx.x == C::kEpiWarp0 * 32) QQQ_STAMP(178);
      publish_rows_fused(p, rows, gt, 2 + grp);
      if (threadIdx.x == C::kEpiWarp0 * 32) wait_rows_fused(p);
      if (threadIdx.x == C::kEpiWarp0 * 32) QQQ_STAMP(179);
      named_bar_sync(1, C::kNumEpiWarps * 32);
    }
    const int et = threadIdx.x - C::kEpiWarp0 * 32;  // 0..kAll-1
    const bool lead = et == 0;                    // segment-level lead (counters)
    const bool hlead = (et & 127) == 0;           // half lead (TMA stores, partial prefetch)
    const int kBarAll = 1, kBarHalf = 2 + eh;
    constexpr int kAll = C::kNumEpiWarps * 32, kHalf = kAll / H;
    double* sa_smem = reinterpret_cast<double*>(smem + C::kOffSA);
    int32_t* rs_smem = reinterpret_cast<int32_t*>(smem + C::kOffRS);
    uint8_t* ystage = smem + C::kOffY + (warp - C::kEpiWarp0) * C::kYWarpBytes;  // per warp: kYBufs x [16 tok][32 ch] fp16
    constexpr int PB = C::kPartBufs;
    uint8_t* pstage = smem + C::kOffPart + eh * (PB * 8192);
    uint64_t* pfull = part_full + 2 * eh;
    uint32_t ych = 0;     // y staging chunks issued by this half
    uint32_t pchunk = 0;  // partial-sum chunks consumed by this half (part_full parity)
    uint32_t pcon = 0;    // contributor chunks staged by this half (ring buffer alternation)
    SegIter si = make_iter(p);
    int tile, kb0, kb1;
    uint32_t seg = 0;
    while (si.next(tile, kb0, kb1)) {
      const int n_tile = ntile_of(tile);
      const int tok0 = (tile % p.tok_tiles) * NTOK;
      const int tvalid = (p.M - tok0) < NTOK ? (p.M - tok0) : NTOK;
      // stage this tile's per-token scales (and code sums) while the MMAs run
      named_bar_sync(kBarAll, kAll);  // previous segment done reading sa_smem / rs_smem
      for (int t = et; t < tvalid; t += kAll) {
        // (L2-coherent loads: with the fused quantization these are written in this
        // launch by other CTAs; a const-pointer load may compile to the
        // non-coherent path and be hoisted above the acquire)
        sa_smem[t] = __ldcg(p.s_a + tok0 + t);
        if constexpr (C::kU8) rs_smem[t] = 128 * __ldcg(p.rowsum + tok0 + t);
      }
      named_bar_sync(kBarAll, kAll);
      const int n = n_tile * 128 + row;
      const bool n_ok = n < p.N;
      const bool cs = C::kSmall && p.csplit > 1;  // cluster split-K: DSMEM reduce-scatter below
      // big-CTA cluster split-K (128-token tiles): reduce-scatter by TOKEN range
      const bool csb = !C::kSmall && !PAIR && NTOK == 128 && p.csplit > 1;
#ifdef QQQ_EXP_NO_FIXUP
      const bool whole = true;  // experiment: every segment stores its own partial (wrong results)
#else
      const bool whole = cs || csb || (kb0 == 0 && kb1 == p.kb_per_tile);
#endif
      const double s_col = n == n_first ? s_col_first : (n_ok && p.s_col) ? p.s_col[n] : 0.0;
      int seg_idx = 0, nsegs = 1;
      int32_t* slots = nullptr;
      // pair plans: segments are counted in CTA pairs; each CTA of a pair reduces its
      // own 128 channels in its own slot / counter (index tile * 2 + rank)
      const int slot_id = PAIR ? tile * 2 + (int)crank : tile;
      if (!whole) {
        const int64_t u_first = (int64_t)tile * p.kb_per_tile;
        const int G = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
        const int b_first = cta_of_unit(u_first, p, G);
        const int b_last = cta_of_unit(u_first + p.kb_per_tile - 1, p, G);
        seg_idx = (PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x) - b_first;
        nsegs = b_last - b_first + 1;
        slots = p.ws + (int64_t)slot_id * NTOK * 128;  // one zero-initialised accumulation slot per tile
      }
      const bool owner = whole || seg_idx == 0;
      const int j = seg % C::kAccBufs;
      if (cs && lead) {
        // this CTA finalizes channel rows [ceil(me*128/S), ceil((me+1)*128/S)): the
        // other S-1 ranks each send those rows' NTOK int32 partials
        const int S = p.csplit, me = (int)cluster_ctarank();
        const int mine = ((me + 1) * 128 + S - 1) / S - (me * 128 + S - 1) / S;
        mbar_arrive_expect_tx(&part_full[0], (uint32_t)((S - 1) * mine * NTOK * 4));
      }
      if (!QQQ_CSB_L2 && csb && lead) {
        // this CTA finalizes tokens [me*T, (me+1)*T) of all 128 channels (T = NTOK/S):
        // the other S-1 ranks each send those tokens' int32 partials, 16-token chunk
        // by chunk (only chunks holding valid tokens)
        const int S = p.csplit, me = (int)cluster_ctarank(), T = NTOK / S;
        int nvc = 0;
        for (int c0 = me * T; c0 < (me + 1) * T; c0 += 16) nvc += c0 < tvalid ? 1 : 0;
        if (nvc) mbar_arrive_expect_tx(&part_full[0], (uint32_t)((S - 1) * nvc * 16 * 128 * 4));
        else mbar_arrive(&part_full[0]);
      }
      // ONE warp polls the accumulator barrier (backoff), the others block in a
      // named barrier: with every epilogue warp polling, the polls were ~40% of
      // all instructions issued in a prefill kernel (ncu), taken from the converters
#ifdef QQQ_EPI_ALLPOLL
      mbar_wait_backoff(&acc_full[j], (seg / C::kAccBufs) & 1);
#else
      if (warp == C::kEpiWarp0) mbar_wait_backoff(&acc_full[j], (seg / C::kAccBufs) & 1);
      named_bar_sync(kBarAll, kAll);
#endif
      tc_fence_after();
      if (lead && seg < 4) QQQ_STAMP(36 + 2 * seg);
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + j * NTOK;
      const int nchunks = (tvalid + 15) / 16;
      const int nmine = (nchunks - eh + H - 1) / H;  // chunks c = eh, eh + H, ...
      if (cs) {
        if constexpr (NTOK <= 32) {
        // ---- cluster split-K: reduce-scatter the int32 partials over DSMEM. The
        // thread of channel row `row` sends its NTOK partials to the rank that
        // finalizes the row (st.async, completing bytes on that rank's barrier);
        // the finalizing rank adds the S-1 received partials to its own, applies
        // the dequant and stores y directly (a few rows per CTA).
        const int S = p.csplit, me = (int)cluster_ctarank();
        const int dest = row * S / 128;
        const int rows_per = (128 + S - 1) / S;
        const int drow0 = (dest * 128 + S - 1) / S;
        int32_t* recv = reinterpret_cast<int32_t*>(pstage);  // [S][rows_per][NTOK]
        uint32_t own[NTOK];
#pragma unroll
        for (int c0 = 0; c0 < NTOK; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);  // (includes tcgen05.wait::ld)
#pragma unroll
          for (int i = 0; i < 16; ++i) own[c0 + i] = r[i];
        }
#ifdef QQQ_DBG_PARTIALS
        if (p.dbg) {  // debug build: every CTA's own partial [cta][128 rows][NTOK], and a re-read 4 us later
          int32_t* d = reinterpret_cast<int32_t*>(p.dbg) + ((size_t)blockIdx.x * 128 + row) * NTOK;
#pragma unroll
          for (int i = 0; i < NTOK; ++i) d[i] = (int32_t)own[i];
          const unsigned long long t0 = gtimer();
          while (gtimer() - t0 < 4000) __nanosleep(200);
          int32_t* d2 = d + (size_t)gridDim.x * 128 * NTOK;
#pragma unroll
          for (int c0 = 0; c0 < NTOK; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(taddr + c0, r);
#pragma unroll
            for (int i = 0; i < 16; ++i) d2[c0 + i] = (int32_t)r[i];
          }
        }
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[j]);
        if (lead) QQQ_STAMP(150);
        if (dest != me) {
          const uint32_t dst = mapa_shared(recv + (me * rows_per + (row - drow0)) * NTOK, (uint32_t)dest);
          const uint32_t dbar = mapa_shared(&part_full[0], (uint32_t)dest);
#pragma unroll
          for (int i = 0; i < NTOK; i += 4) st_async_v4(dst + i * 4, own[i], own[i + 1], own[i + 2], own[i + 3], dbar);
        } else {
          mbar_wait(&part_full[0], seg & 1);
          if (lead) QQQ_STAMP(151);
          const int lr = row - drow0;
#pragma unroll 1
          for (int sg = 0; sg < S; ++sg) {
            if (sg == me) continue;
            const int32_t* src = recv + (sg * rows_per + lr) * NTOK;
#pragma unroll
            for (int i = 0; i < NTOK; ++i) own[i] += (uint32_t)src[i];
          }
          if (lead) QQQ_STAMP(152);
          if (n_ok) {
#pragma unroll
            for (int c0 = 0; c0 < NTOK; c0 += 16) {
              if (c0 >= tvalid) break;
              uint32_t r[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                r[i] = own[c0 + i];
                if constexpr (C::kU8) r[i] -= (uint32_t)rs_smem[c0 + i];  // u8 weights carried +128
              }
              if (p.acc) {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                  if (c0 + i < tvalid) p.acc[(int64_t)(tok0 + c0 + i) * p.ldacc + n] = (int32_t)r[i];
              }
              if (p.s_col) {
                uint16_t h[16];
                dequant16(r, sa_smem + c0, s_col, h, tvalid - c0);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                  if (c0 + i < tvalid) reinterpret_cast<uint16_t*>(p.y)[(int64_t)(tok0 + c0 + i) * p.ldy + n] = h[i];
              }
            }
          }
        }
        }  // NTOK <= 32
        if (lead) QQQ_STAMP(153);
        if (lead && seg < 4) QQQ_STAMP(37 + 2 * seg);
        ++seg;
        continue;
      }
      if constexpr (!C::kSmall && !PAIR && NTOK == 128) {
        if (csb) {
          // ---- big-CTA cluster split-K: reduce-scatter the int32 partials over
          // DSMEM by token range. Rank me finalizes tokens [me*T, (me+1)*T) for all
          // 128 channel rows, so every epilogue warp (each TMEM lane quadrant) takes
          // part. Receive layout (one slot per peer, in rank order without me):
          // [slot][chunk of 16 tokens][4 token quads][128 rows][4 int32]: one
          // st.async.v4 of a warp writes 512 contiguous bytes.
          const int S = p.csplit, me = (int)cluster_ctarank(), T = NTOK / S, CPR = T / 16;
          int32_t* recv = reinterpret_cast<int32_t*>(smem + C::kOffPart);
          const uint32_t recv_cl0 = smem_u32(recv);
          const uint32_t pbar = smem_u32(&part_full[0]);
          // phase 1: send every valid chunk owned by another rank (this group's chunks)
#if QQQ_CSB_L2
          // workspace chunk (tile, dest d, sender slot j, chunk cc): [4 token quads][128 rows][4 int32]
          auto ws_chunk = [&](int d, int jslot, int cc) -> int4* {
            return reinterpret_cast<int4*>(p.ws + ((((size_t)tile * S + d) * (S - 1) + jslot) * CPR + cc) * 2048);
          };
#pragma unroll 1
          for (int li = 0; li < nmine; ++li) {
            const int c = eh + H * li, c0 = c * 16;
            const int d = c0 / T;
            if (d == me) continue;
            uint32_t r[16];
            tmem_ld16(taddr + c0, r);  // (includes tcgen05.wait::ld)
            int4* dst = ws_chunk(d, me < d ? me : me - 1, c - d * CPR) + row;
#pragma unroll
            for (int t4 = 0; t4 < 4; ++t4)
              __stcg(dst + t4 * 128, make_int4((int)r[4 * t4], (int)r[4 * t4 + 1], (int)r[4 * t4 + 2], (int)r[4 * t4 + 3]));
          }
          // publish: every epilogue thread's stores, then ONE gpu-scope fence and a
          // remote arrive on each peer's part_full[1] (count S-1)
          named_bar_sync(kBarAll, kAll);
          if (lead) {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int d = 0; d < S; ++d)
              if (d != me) mbar_arrive_cluster(mapa_shared(&part_full[1], (uint32_t)d));
          }
#else
#pragma unroll 1
          for (int li = 0; li < nmine; ++li) {
            const int c = eh + H * li, c0 = c * 16;
            const int d = c0 / T;
            if (d == me) continue;
            uint32_t r[16];
            tmem_ld16(taddr + c0, r);  // (includes tcgen05.wait::ld)
            const int slot = me < d ? me : me - 1;
            const uint32_t off = (uint32_t)((((slot * CPR + (c - d * CPR)) * 4) * 128 + row) * 16);
            const uint32_t dst = mapa_shared_u32(recv_cl0 + off, (uint32_t)d);
            const uint32_t dbar = mapa_shared_u32(pbar, (uint32_t)d);
#pragma unroll
            for (int t4 = 0; t4 < 4; ++t4)
              st_async_v4(dst + t4 * 128 * 16, r[4 * t4], r[4 * t4 + 1], r[4 * t4 + 2], r[4 * t4 + 3], dbar);
          }
#endif
          if (lead) QQQ_STAMP(150);
          // phase 2: own token range: own partial (TMEM) + the S-1 received ones
          bool waited = false;
#pragma unroll 1
          for (int li = 0; li < nmine; ++li) {
            const int c = eh + H * li, c0 = c * 16;
            if (c0 / T != me) continue;
            if (!waited) {
#if QQQ_CSB_L2
              mbar_wait_acq_cluster(&part_full[1], seg & 1);
#else
              mbar_wait(&part_full[0], seg & 1);
#endif
              waited = true;
              if (lead) QQQ_STAMP(151);
            }
            uint32_t r[16];
            tmem_ld16(taddr + c0, r);
#pragma unroll 1
            for (int slot = 0; slot < S - 1; ++slot) {
#if QQQ_CSB_L2
              const int4* src = ws_chunk(me, slot, c - me * CPR) + row;
#else
              const int4* src = reinterpret_cast<const int4*>(recv) + ((slot * CPR + (c - me * CPR)) * 4) * 128 + row;
#endif
#pragma unroll
              for (int t4 = 0; t4 < 4; ++t4) {
#if QQQ_CSB_L2
                const int4 v = __ldcg(src + t4 * 128);
#else
                const int4 v = src[t4 * 128];
#endif
                r[4 * t4] += (uint32_t)v.x;
                r[4 * t4 + 1] += (uint32_t)v.y;
                r[4 * t4 + 2] += (uint32_t)v.z;
                r[4 * t4 + 3] += (uint32_t)v.w;
              }
            }
            if constexpr (C::kU8) {
#pragma unroll
              for (int i = 0; i < 16; ++i) r[i] -= (uint32_t)rs_smem[c0 + i];  // u8 weights carried +128
            }
            store_outputs(p, r, sa_smem + c0, tok0 + c0, tvalid - c0, n, n_ok, s_col);
            if (p.y_tma) {
              uint16_t* stg = reinterpret_cast<uint16_t*>(ystage) + (C::kYBufs == 2 ? (ych & 1) * 512 : 0);
              uint16_t h[16];
              dequant16_all(r, sa_smem + c0, s_col, h);
              if (lane == 0) {
                if constexpr (C::kYBufs == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
              }
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 16; ++i) stg[i * 32 + lane] = h[i];
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&y_map, stg, n_tile * 128 + q * 32, tok0 + c0);
                bulk_commit();
              }
              ++ych;
            }
          }
#if !QQQ_CSB_L2
          if (!waited && lead) mbar_wait(&part_full[0], seg & 1);  // (keep the barrier phase in step)
#endif
          if (lead) QQQ_STAMP(153);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[j]);
          ++seg;
          continue;
        }
      }
      if (!owner) {
        // ---- contributor: add the partial into the tile's slot, release the counter.
        // Chunks with few valid tokens use per-element red.add; fuller chunks are
        // staged in shared memory and reduced with ONE bulk cp.reduce (L2-side
        // int32 add at bulk bandwidth; per-lane atomics run at ~1 lane/clk/SM).
#pragma unroll 1
        for (int li = 0; li < nmine; ++li) {
          const int c0 = (eh + H * li) * 16;
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);  // (includes tcgen05.wait::ld)
          if (tvalid - c0 < 4) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < tvalid) red_add_s32(slots + (c0 + i) * 128 + row, (int32_t)r[i]);
          } else {
            // rows past tvalid hold zeros (their activations were zero-filled)
            int32_t* stg = reinterpret_cast<int32_t*>(pstage + (pcon % PB) * 8192);
            if (hlead) bulk_wait_read<PB - 1>();  // the reduce that used this buffer PB chunks ago has read it
            named_bar_sync(kBarHalf, kHalf);
#pragma unroll
            for (int i = 0; i < 16; ++i) stg[i * 128 + row] = (int32_t)r[i];
            fence_proxy_async_smem();
            named_bar_sync(kBarHalf, kHalf);
            if (hlead) {
              bulk_reduce_add_s32(slots + c0 * 128, stg, 8192);
              bulk_commit();
            }
            ++pcon;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR)
            mbar_arrive_cluster(acc_empty_cl + j * 8);
          else
            mbar_arrive(&acc_empty[j]);
        }
        // publish: the group leads wait for their bulk reductions to complete, then
        // CTA barrier and ONE gpu-scope release by the lead (cumulative over the
        // red.adds / completed bulk reductions ordered before it by the barrier)
        if (hlead) {
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        named_bar_sync(kBarAll, kAll);
        if (lead) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.counters + slot_id) : "memory");
        if (lead) QQQ_STAMP(61);
      } else {
        if (!whole) {
          // ---- owner of a split tile: wait for the other nsegs-1 contributions
          if (lead) {
            int32_t* cnt = p.counters + slot_id;
            int v;
            unsigned long long t0 = 0;
#pragma unroll 1
            for (uint32_t n = 0;; ++n) {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
              if (v >= nsegs - 1) break;
#ifndef QQQ_NO_WATCHDOG
              // a contributor that never arrives (not co-resident, corrupted
              // counters) traps the launch after ~4 s instead of hanging the GPU
              if ((n & 1023) == 1023) {
                const unsigned long long t = gtimer();
                if (t0 == 0)
                  t0 = t;
                else if (t - t0 > QQQ_WATCHDOG_NS)
                  __trap();
              }
#endif
            }
            *cnt = 0;  // re-arm for the next launch (every contributor has arrived)
            QQQ_STAMP(60);
          }
          named_bar_sync(kBarAll, kAll);
        }
        // reduced partial chunks [16 tok][128 rows] int32 (8 KiB, contiguous in the
        // slot) are bulk-copied into this half's PB-deep smem ring, PB chunks ahead
        auto part_issue = [&](int li) {
          const uint32_t pc = pchunk + li;
          mbar_arrive_expect_tx(&pfull[pc % PB], 8192);
          bulk_g2s(pstage + (pc % PB) * 8192, slots + (int64_t)(eh + H * li) * 16 * 128, 8192, &pfull[pc % PB]);
        };
        if (!whole && hlead) {
          bulk_wait_read<0>();  // earlier contributor reductions have read the shared ring
          for (int li = 0; li < PB && li < nmine; ++li) part_issue(li);
        }
        int li0 = 0;
#ifndef QQQ_EPI_NO_PAIRS
        // (single-buffered 256/384-token accumulators only, where the epilogue is
        // serial with the next tile's MMAs; elsewhere it is overlapped and the
        // extra registers cost more than the pairs save)
#ifndef QQQ_EPI_PAIRS_MIN_NTOK
#define QQQ_EPI_PAIRS_MIN_NTOK 256
#endif
        if (NTOK >= QQQ_EPI_PAIRS_MIN_NTOK && C::kYBufs == 2 && whole && p.y_tma && !p.acc &&
            (!PAIR || n_tile < p.n_tiles)) {
          // Whole tile, TMA-stored y: this warp's chunks two at a time (one TMEM
          // load wait, one staging fence and bulk group per pair; the two 1 KiB
          // staging buffers hold the pair, the previous pair's stores must have
          // read them). Per-chunk latency steps were ~0.45 us of each ~0.8 us chunk.
          uint16_t* stg0 = reinterpret_cast<uint16_t*>(ystage);
#pragma unroll 1
          for (; li0 + 1 < nmine; li0 += 2) {
            const int c0a = (eh + H * li0) * 16, c0b = (eh + H * (li0 + 1)) * 16;
            uint32_t ra[16], rb[16];
            tmem_ld16x2(taddr + c0a, taddr + c0b, ra, rb);
            if constexpr (C::kU8) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                ra[i] -= (uint32_t)rs_smem[c0a + i];  // u8 weights carried +128
                rb[i] -= (uint32_t)rs_smem[c0b + i];
              }
            }
            {  // (one chunk's halves live at a time: the kernel is at its register cap)
              uint16_t h[16];
              dequant16_all(ra, sa_smem + c0a, s_col, h);
              if (lane == 0) bulk_wait_read<0>();  // the previous pair's stores have read the staging
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 16; ++i) stg0[i * 32 + lane] = h[i];
              dequant16_all(rb, sa_smem + c0b, s_col, h);
#pragma unroll
              for (int i = 0; i < 16; ++i) stg0[512 + i * 32 + lane] = h[i];
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&y_map, stg0, n_tile * 128 + q * 32, tok0 + c0a);
              tma_store_2d(&y_map, stg0 + 512, n_tile * 128 + q * 32, tok0 + c0b);
              bulk_commit();
            }
          }
          if (li0 > 0) {
            if (lane == 0) bulk_wait_read<0>();  // (the per-chunk loop alternates the buffers by ych)
            __syncwarp();
          }
        }
#endif
#pragma unroll 1
        for (int li = li0; li < nmine; ++li) {
          const int c0 = (eh + H * li) * 16;
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);  // (includes tcgen05.wait::ld)
          if (lead && seg == 0 && li < 16) QQQ_STAMP(44 + li);
          if (!whole) {
            const uint32_t pc = pchunk + li;
            mbar_wait(&pfull[pc % PB], (pc / PB) & 1);
            if (lead && li == 0) QQQ_STAMP(62);
            const int32_t* part = reinterpret_cast<const int32_t*>(pstage + (pc % PB) * 8192);
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] += (uint32_t)part[i * 128 + row];
            // return the slot to zero for the next launch (entries past tvalid were never touched)
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < tvalid) __stcg(slots + (c0 + i) * 128 + row, 0);
            named_bar_sync(kBarHalf, kHalf);  // this half has read the buffer
            if (hlead && li + PB < nmine) part_issue(li + PB);
          }
          if constexpr (C::kU8) {
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] -= (uint32_t)rs_smem[c0 + i];  // u8 weights carried +128
          }
          store_outputs(p, r, sa_smem + c0, tok0 + c0, tvalid - c0, n, n_ok, s_col);
          if (p.y_tma && (!PAIR || n_tile < p.n_tiles)) {
            // y chunk -> this warp's staging [16 tok][32 ch] fp16 -> its own TMA store
            // (OOB rows/cols clipped): no cross-warp barrier on the store path
            uint16_t* stg = reinterpret_cast<uint16_t*>(ystage) + (C::kYBufs == 2 ? (ych & 1) * 512 : 0);
            uint16_t h[16];
            dequant16_all(r, sa_smem + c0, s_col, h);
            if (lead && seg == 0 && li < 4) QQQ_STAMP(128 + li);
            if (lane == 0) {  // the store that used this buffer (two chunks ago; one with a single buffer) has read it
              if constexpr (C::kYBufs == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
            }
            __syncwarp();
            if (lead && seg == 0 && li < 4) QQQ_STAMP(132 + li);
#pragma unroll
            for (int i = 0; i < 16; ++i) stg[i * 32 + lane] = h[i];
            fence_proxy_async_smem();
            __syncwarp();
            if (lead && seg == 0 && li < 4) QQQ_STAMP(136 + li);
            if (lane == 0) {
              tma_store_2d(&y_map, stg, n_tile * 128 + q * 32, tok0 + c0);
              bulk_commit();
            }
            if (lead && seg == 0 && li < 4) QQQ_STAMP(140 + li);
            ++ych;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR)
            mbar_arrive_cluster(acc_empty_cl + j * 8);
          else
            mbar_arrive(&acc_empty[j]);
        }
        if (!whole) pchunk += nmine;
      }
      if (lead && seg < 4) QQQ_STAMP(37 + 2 * seg);
      ++seg;
    }
    if (lead) QQQ_STAMP(154);
    if (lane == 0) bulk_wait_read<0>();  // y stores have read their staging before the CTA retires
    if (lead) QQQ_STAMP(63);
  }

  if (PAIR || p.csplit > 1) {
    // no CTA of the cluster retires while another may still signal its barriers,
    // store into its shared memory or (pair) read its shared memory / TMEM
    tc_fence_before();
    __syncthreads();  // (CTA-scope ordering of the TMEM reads before the dealloc; the relaxed cluster barrier has none)
    cluster_sync_all();
  } else {
    tc_fence_before();
    __syncthreads();
  }
  if (threadIdx.x == 0) QQQ_STAMP(42);
  if (p.xsrc && threadIdx.x == 0) {
    // the last CTA done with the fused-quantization counter re-arms it
    int prev;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p.counters + kQDoneSlot) : "memory");
    if (prev == (int)gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.s32 [%0], 0;" ::"l"(p.counters + kQRowsSlot) : "memory");
      asm volatile("st.relaxed.gpu.global.s32 [%0], 0;" ::"l"(p.counters + kQDoneSlot) : "memory");
    }
  }
  if (warp == C::kAllocWarp) {
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc_pair(tmem_base, C::kTmemCols);
    else
      tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// Per-device host caches (SM counts, co-resident pair clusters, kernel
// attributes): the C ABI runs on the calling thread's current device, which
// the caller sets to the stream's device (the Python layer does).
constexpr int kMaxDevices = 64;

static int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}

static int num_sms() {
  static int n[kMaxDevices] = {};
  const int dev = cur_device();
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

struct LaunchPlan {
  int ntok, bk, grid, aligned_tiles, tok_tiles, n_tiles, kb_per_tile, tiles, max_segs, dp_tiles, pair, csplit;
  int64_t units, sk_unit0;
};

// k-block depth per token tile: 256 for the half-SM decode CTAs (8 converter
// warps x 4 slabs, 64-column TMEM A buffers), 128 for prefill (small
// activation stages beside 256-column accumulators)
#ifndef QQQ_BIG_BK
#define QQQ_BIG_BK 256
#endif
#ifndef QQQ_SMALL_BK
#define QQQ_SMALL_BK 256
#endif
static constexpr int bk_for(int mode, int ntok) { return ntok <= 64 ? QQQ_SMALL_BK : mode == kModeI8 ? 128 : QQQ_BIG_BK; }
static constexpr int ctas_per_sm(int mode, int ntok) { return ntok <= 64 && mode != kModeI8 ? 2 : 1; }
#ifndef QQQ_PAIR_BK
#define QQQ_PAIR_BK 128
#endif
static constexpr int kPairBk = QQQ_PAIR_BK;

template <int MODE, int NTOK, int BK, bool PAIR>
__global__ void w4a8_gemm_kernel(const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                                 const GemmParams);

// 2-CTA clusters of the pair kernel that fit on the GPU at once (a GPC with an
// odd number of free SMs strands one): the stream-K pair plans never exceed it
static int pair_slots(int mode) {
  static int slots[kMaxDevices][2] = {};
  int* n = slots[cur_device()];
  const int i = mode == kModePC ? 0 : 1;
  if (n[i] == 0) {
    using C = Cfg<kModePG, 256, kPairBk, true>;
    auto kern = mode == kModePC ? w4a8_gemm_kernel<kModePC, 256, kPairBk, true>
                                : w4a8_gemm_kernel<kModePG, 256, kPairBk, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(2 * (unsigned)num_sms());
    lc.blockDim = dim3(C::kNumThreads);
    lc.dynamicSmemBytes = C::kSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, (void*)kern, &lc) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / 2 - 4;  // conservative
    }
    n[i] = std::min(c, num_sms() / 2);
  }
  return n[i];
}

// split: 0 = whole tiles (data-parallel), 1 = stream-K over all units,
//        2 = hybrid: full waves of whole tiles, the remainder stream-K'd over all CTAs,
//        3 = whole 256-channel pair tiles on 2-CTA clusters (NTOK = 256, PC/PG)
static LaunchPlan plan_for(int mode, int64_t M, int64_t N, int64_t K, int ntok, int split, int force_grid,
                           int force_cs = 0) {
  LaunchPlan lp{};
  // cluster split-K: decode tiles only (NTOK 16/32, 2 CTAs per SM). (A 128-token
  // prefill variant — 64 KiB partials over DSMEM — measured slower than stream-K:
  // the exchange ran at ~7 B/clk per SM.)
  if (split == 4 && ntok == 128 && mode != kModeI8) {
    // big-CTA cluster split-K (128-token tiles): one tile per cluster of S in {2, 4}
    // whole-SM CTAs, partials reduce-scattered by token range over DSMEM (the
    // receive buffer, (S-1) x 128/S tokens x 128 rows x 4 B, is the 48 KiB partial
    // ring). For mid M on few channel tiles (4096x4096: 32 tiles for 148 SMs).
    lp.ntok = ntok;
    lp.bk = bk_for(mode, ntok);
    lp.tok_tiles = (int)((M + ntok - 1) / ntok);
    lp.n_tiles = (int)(round_up(N, kTileN) / kTileN);
    lp.kb_per_tile = (int)((round_up(K, kKPadTo) + lp.bk - 1) / lp.bk);
    lp.tiles = lp.n_tiles * lp.tok_tiles;
    lp.units = (int64_t)lp.tiles * lp.kb_per_tile;
    lp.max_segs = 1;
    const int slots = force_grid > 0 ? std::min(force_grid, num_sms()) : num_sms();
    int S = 1;
    if ((force_cs == 2 || force_cs == 4) && force_cs <= lp.kb_per_tile) {
      S = force_cs;
    } else {
      for (int c : {4, 2})
        if ((int64_t)lp.tiles * c <= slots && c <= lp.kb_per_tile) {
          S = c;
          break;
        }
    }
    if (S == 1) return plan_for(mode, M, N, K, ntok, 1, force_grid);
    lp.csplit = S;
    lp.grid = lp.tiles * S;
    return lp;
  }
  if (split == 4 && (ntok > 32 || ctas_per_sm(mode, ntok) != 2)) split = 1;
  if (split == 4) {
    // cluster split-K: one tile per cluster of S decode CTAs: the largest S that
    // fits the CTA slots and leaves every rank >= 1 k-block
    lp.ntok = ntok;
    lp.bk = bk_for(mode, ntok);
    lp.tok_tiles = (int)((M + ntok - 1) / ntok);
    lp.n_tiles = (int)(round_up(N, kTileN) / kTileN);
    lp.kb_per_tile = (int)((round_up(K, kKPadTo) + lp.bk - 1) / lp.bk);
    lp.tiles = lp.n_tiles * lp.tok_tiles;
    lp.units = (int64_t)lp.tiles * lp.kb_per_tile;
    lp.max_segs = 1;
    // 32-token clusters run two CTAs per SM again. They had been capped to one
    // after stress runs saw one TMEM lane quadrant of one CTA's partial corrupted
    // in 1-10% of the launches; the cause was the converters' weight-stage
    // release racing their own shared-memory loads (see the converter loop),
    // which the co-resident CTA's timing exposed. 6000 stress launches clean
    // since the fix; QQQ_NT32_ONE_PER_SM=1 restores the cap.
#ifndef QQQ_NT32_ONE_PER_SM
#define QQQ_NT32_ONE_PER_SM 0
#endif
    static const bool allow32 = !QQQ_NT32_ONE_PER_SM || getenv("QQQ_EXP_NTOK32_TWO_PER_SM") != nullptr;
    const int slots = (force_grid > 0 ? std::min(force_grid, num_sms()) : num_sms()) *
                      ((ntok == 32 && !allow32) ? 1 : ctas_per_sm(mode, ntok));
    // Cluster size S <= 8 (portable), receive buffer [S][ceil(128/S)][NTOK] int32
    // within the 16 KiB partial ring (every S for NTOK=16, divisors of 128 for
    // 32). Measured (profiles/r01_csplit_size_sweep.txt): the fastest S is the
    // smallest that keeps >= 0.8 CTAs per SM pulling weights and <= 8 k-blocks per
    // CTA — more, shorter CTAs lose to SM sharing and per-CTA fixed costs (4096x4096:
    // S=4 5.6 us vs S=8 7.9 us), fewer, longer ones to the per-CTA stream rate.
    auto fits = [&](int c) {
      const int rows_per = (128 + c - 1) / c;
      return (int64_t)lp.tiles * c <= slots && c <= lp.kb_per_tile && c * rows_per * ntok * 4 <= 16384;
    };
    int S = 1;
    if (force_cs >= 2 && force_cs <= 8 && fits(force_cs)) {
      S = force_cs;  // caller's cluster size (tests of every S the rule below can pick)
    } else {
      for (int c = 2; c <= 8; ++c) {
        if (!fits(c)) continue;
        S = c;  // the largest fitting S, unless a smaller one meets both targets below
        if (lp.tiles * c * 5 >= num_sms() * 4 && (lp.kb_per_tile + c - 1) / c <= 8) break;
      }
    }
    if (S == 1) return plan_for(mode, M, N, K, ntok, 1, force_grid);
    lp.csplit = S;
    lp.grid = lp.tiles * S;
    return lp;
  }
  const bool pair_plan = split == 3 || split == 5 || split == 6;
  if (pair_plan && ((ntok != 256 && ntok != 192 && ntok != 384 && ntok != 128) || mode == kModeI8))
    split = split == 3 ? 0 : split == 5 ? 1 : 2;
  if (ntok == 384 && (split == 0 || split == 1 || split == 2 || split == 5 || split == 6))
    split = 3;  // (384-token tiles: whole pair tiles only)
  if (split == 3 || split == 5 || split == 6) {
    // pair tiles: 3 = whole pair tiles, 5 = stream-K over (pair tile, k-block) units
    // across the CTA pairs, 6 = whole-tile waves + the remainder stream-K'd
    lp.ntok = ntok;
    lp.bk = kPairBk;
    lp.pair = 1;
    lp.tok_tiles = (int)((M + ntok - 1) / ntok);
    lp.n_tiles = (int)(round_up(N, kTileN) / kTileN);
    lp.kb_per_tile = (int)((round_up(K, kKPadTo) + lp.bk - 1) / lp.bk);
    lp.tiles = ((lp.n_tiles + 1) / 2) * lp.tok_tiles;  // pair tiles
    lp.units = (int64_t)lp.tiles * lp.kb_per_tile;
    lp.max_segs = 1;
    // co-resident 2-CTA clusters (a split tile's owner waits for its contributors)
    const int pairs = force_grid > 0 ? std::max(1, std::min(force_grid / 2, pair_slots(mode))) : pair_slots(mode);
    if (split == 6) {
      const int waves = lp.tiles / pairs, rem = lp.tiles % pairs;
      if (waves >= 1 && rem > 0) {
        lp.grid = 2 * pairs;
        lp.dp_tiles = waves;
        lp.sk_unit0 = (int64_t)waves * pairs * lp.kb_per_tile;
        lp.units = (int64_t)rem * lp.kb_per_tile;
        const int64_t per = std::max<int64_t>(1, lp.units / pairs);
        lp.max_segs = (int)std::min<int64_t>((lp.kb_per_tile + per - 1) / per + 1, pairs);
        return lp;
      }
      split = waves >= 1 ? 3 : 5;
    }
    if (split == 5) {
      const int g = (int)std::min<int64_t>(lp.units, pairs);
      lp.grid = 2 * g;
      const int64_t per = lp.units / g;
      lp.max_segs = (int)std::min<int64_t>((lp.kb_per_tile + per - 1) / per + 1, g);
      return lp;
    }
    const int per = (lp.tiles + pairs - 1) / pairs;
    lp.aligned_tiles = per;
    lp.grid = 2 * ((lp.tiles + per - 1) / per);
    return lp;
  }
  lp.ntok = ntok;
  lp.bk = bk_for(mode, ntok);
  lp.tok_tiles = (int)((M + ntok - 1) / ntok);
  lp.n_tiles = (int)(round_up(N, kTileN) / kTileN);
  lp.kb_per_tile = (int)((round_up(K, kKPadTo) + lp.bk - 1) / lp.bk);  // last k-block may be partial
  lp.tiles = lp.n_tiles * lp.tok_tiles;
  lp.units = (int64_t)lp.tiles * lp.kb_per_tile;
  const int sms = num_sms() * ctas_per_sm(mode, ntok);  // CTA slots
  lp.max_segs = 1;
  if (split == 2 && ctas_per_sm(mode, ntok) == 2) split = 1;  // small CTAs: a single stream-K range
  if (split == 2) {
    const int g = force_grid > 0 ? std::min(force_grid, sms) : sms;
    const int waves = lp.tiles / g, rem = lp.tiles % g;
    if (waves >= 1 && rem > 0) {
      lp.aligned_tiles = 0;
      lp.grid = g;
      lp.dp_tiles = waves;
      lp.sk_unit0 = (int64_t)waves * g * lp.kb_per_tile;
      lp.units = (int64_t)rem * lp.kb_per_tile;
      const int64_t per = std::max<int64_t>(1, lp.units / g);
      lp.max_segs = (int)std::min<int64_t>((lp.kb_per_tile + per - 1) / per + 1, g);
      return lp;
    }
    split = waves >= 1 ? 0 : 1;  // exact waves: data-parallel; under one wave: stream-K
  }
  if (split == 1) {
    lp.aligned_tiles = 0;
    // Split tiles are finished by an owner CTA that waits for its contributors,
    // so every CTA must be co-resident: never more CTAs than CTA slots.
    int g = force_grid > 0 ? std::min(force_grid, sms) : sms;
    lp.grid = (int)(lp.units < g ? lp.units : g);
    const int64_t per = lp.units / lp.grid;  // >= 1: most CTAs overlapping one tile
    lp.max_segs = (int)((lp.kb_per_tile + per - 1) / per + 1);
    if (lp.max_segs > lp.grid) lp.max_segs = lp.grid;
  } else {
    const int per = (lp.tiles + sms - 1) / sms;
    lp.aligned_tiles = per;
    lp.grid = (lp.tiles + per - 1) / per;
  }
  return lp;
}

// Tile-plan cost model (us), fitted (log least squares, scripts/fit_planner.py)
// to the B200 tile-plan sweeps profiles/r01_tileplan_sweep_v2.jsonl (decode /
// mid M) and profiles/r01_pair_sweep.jsonl (prefill, incl. pair tiles) of this
// kernel (1.2% regret against the best measured plan over both sweeps):
//   per-k-block time u = max(weight bytes / per-CTA HBM share, conversion, MMA)
//   whole tiles: T = T0 + units_per_CTA * u + waves * epilogue
//   stream-K:    T = T0 + units_per_CTA * u + fix-up + epilogue
static double plan_cost_us(const LaunchPlan& lp, int64_t M) {
  const double T0 = 1.087, kBsm = 26.03e3, kBtot = 5379e3, kConv = 14.24e-6, kMma = 1.719, kF0 = 5.248,
               kF1 = 0.3505, kE0 = 0.512, kE1 = 0.1027;
  const double clk = 1900.0;  // MHz
  const int cps = lp.ntok <= 64 ? 2 : 1;
  const int64_t ucta = lp.aligned_tiles > 0 ? (int64_t)lp.aligned_tiles * lp.kb_per_tile
                                            : (int64_t)lp.dp_tiles * lp.kb_per_tile + (lp.units + lp.grid - 1) / lp.grid;
  const double bw = std::min(kBsm, kBtot / lp.grid);  // bytes/us per CTA
  const double wkb = lp.bk * 64.0 * (1.0 + 1.0 / 32);
  const double mma = (lp.bk / 32.0) * (lp.ntok / 2.0) / clk * kMma;
  const double conv = lp.bk * 128.0 * kConv * cps;
  const double u = std::max(std::max(wkb / bw, conv), mma);
  const double mt = (double)std::min<int64_t>(lp.ntok, M) / 16.0;
  const double epi = kE0 + kE1 * mt;
  if (lp.csplit > 1 && lp.ntok == 128) {
    // big-CTA cluster split-K: linear fit (0.3 us rms, 0.6 us max) to 14 measured
    // points on 4096x4096 / 11008x4096, M = 32..256, S = 2 / 4 (graph-timed, cold
    // weights): per-CTA k-blocks, the DSMEM exchange share (S-1)/S, the valid
    // 16-token chunks, and a second token tile
    const double ucta_cs = (double)((lp.kb_per_tile + lp.csplit - 1) / lp.csplit);
    const double mtc = (double)std::min<int64_t>(M, 128) / 16.0;
    return -0.173 + 0.558 * ucta_cs + 7.826 * (lp.csplit - 1.0) / lp.csplit + 0.225 * mtc +
           (lp.tok_tiles > 1 ? 1.386 : 0.0);
  }
  if (lp.csplit > 1) {
    // cluster split-K (linear fit to profiles/r01_csplit_sweep.jsonl, 7% rms): a
    // fixed cost, the per-CTA k-blocks, a penalty for the k-blocks of CTAs that
    // share an SM, +2.2 us for the 32-token tile (2 weight stages)
    const int ucta_cs = (lp.kb_per_tile + lp.csplit - 1) / lp.csplit;
    const double shared = std::max(0, lp.grid - num_sms()) / (double)num_sms();
    // (+2 us on 32-token clusters: the round-1 fit underestimates them, e.g.
    //  11008x4096 M=32 S=4 measured 14.6 us against 12.1; with +2 the planner
    //  takes them where they win, 4096x11008 M=17-32: 13.9 -> 12.0-12.4 us)
#ifndef QQQ_NT32_PENALTY
#define QQQ_NT32_PENALTY 2.0
#endif
    return 4.813 + 0.456 * ucta_cs + 0.671 * shared * ucta_cs + (lp.ntok == 32 ? QQQ_NT32_PENALTY : 0.0) + 0.012 * mt;
  }
  if (lp.pair) {
    // 2-CTA pair tiles: ~0.41 us per 128-deep k-block of a 256x256 pair tile; the
    // 192-token pair tile double-buffers its accumulator, so only the last tile's
    // epilogue is exposed (per-k-block time scaled by the MMA width, 192/256)
    // (x kPairF: the paired epilogue chunks took 5-8% off the 256/384-token pair
    //  tiles after the fit; e.g. 4096x22016 M=256: pair tiles 30.6 us against the
    //  33.0 of the stream-K plan the unscaled model preferred)
#ifndef QQQ_PAIR_COST_F
#define QQQ_PAIR_COST_F 0.93
#endif
    const double kT0p = 1.41, kUp = 0.4133, kPairF = QQQ_PAIR_COST_F;
    const double tiles_pp = lp.aligned_tiles > 0 ? (double)lp.aligned_tiles : (double)lp.units / lp.kb_per_tile / (lp.grid / 2);
    if (lp.ntok == 192) return kT0p + tiles_pp * lp.kb_per_tile * kUp * 0.78 + epi;
    return kPairF * (kT0p + tiles_pp * lp.kb_per_tile * kUp + tiles_pp * epi);
  }
  if (lp.aligned_tiles > 0) return T0 + ucta * u + lp.aligned_tiles * epi;
  return T0 + ucta * u + kF0 + kF1 * mt + epi;
}

static LaunchPlan make_plan(int mode, int64_t M, int64_t N, int64_t K, int force_ntok, int force_grid,
                            int force_split, int force_cs = 0) {
  if (force_ntok > 0 || force_split >= 0 || force_grid > 0) {
    const int nt = force_ntok > 0 ? force_ntok : (M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256);
    const int sk = force_split >= 0 ? force_split : (nt <= 64 ? 1 : 2);
    return plan_for(mode, M, N, K, nt, sk, force_grid, force_cs);
  }
  LaunchPlan best{};
  double best_t = 1e30;
  // NTOK=64 stays available by config but is not auto-selected: as a half-SM
  // CTA it only fits 2 weight + 2 activation stages, and the NTOK=128 plan
  // measured faster at every M it would cover (r01_tileplan_sweep_v2)
  for (int nt : {16, 32, 128, 192, 256}) {
    // a smaller tile already covers every token (but the 128-token cluster plan
    // spreads a few channel tiles over more SMs from M = 17 on)
    if (nt > 32 && nt / 4 >= M && !(nt == 128 && M > 16)) break;
    if (nt == 192) {
      // 192-token pair tiles (double-buffered accumulators) stay a forced-plan option:
      // measured slower than the 256-token pair tile wherever it would be picked
      // (4096x11008 M=1024 54.3 vs 51.8 us, 11008x4096 66.3 vs 38.3 us): prefill is
      // co-bound by the INT4->INT8 conversion, which a 192-token tile repeats for
      // 6 instead of 4 token tiles at M = 1024, more than the hidden epilogue saves.
      // One regime where it measured faster: two 256-token tiles per channel pair
      // would fill between one and 1.6 waves of CTA pairs (4096x11008 M=512: 30.6
      // vs 33.8 us); three 192-token tiles fill the pairs more evenly and hide their
      // epilogues.
      if (mode == kModeI8) continue;
      const LaunchPlan lp256 = plan_for(mode, M, N, K, 256, 3, 0);
      const double waves256 = (double)lp256.tiles / std::max(1, pair_slots(mode));
      const bool regime = M > 448 && M <= 576 && waves256 > 1.0 && waves256 < 1.6;
      if (!regime && !getenv("QQQ_EXP_AUTO_192")) continue;
      const LaunchPlan lp = plan_for(mode, M, N, K, nt, 3, 0);
      const double t = regime ? 0.0 : plan_cost_us(lp, M);
      if (lp.tiles <= 65536 && t < best_t) {
        best_t = t;
        best = lp;
      }
      continue;
    }
    // whole tiles / stream-K / pair tiles / cluster split-K (the hybrid never won a sweep point)
    for (int sk = 0; sk < 5; ++sk) {
      if (sk == 2 || (sk == 3 && (nt != 256 || mode == kModeI8)) ||
          (sk == 4 && ((nt > 32 && nt != 128) || mode == kModeI8)))
        continue;
      if (nt == 128 && nt / 4 >= M && sk != 4) continue;  // (only the cluster plan at M <= 32)
      const LaunchPlan lp = plan_for(mode, M, N, K, nt, sk, 0);
      if (lp.tiles > 65536) continue;
      const double t = plan_cost_us(lp, M);
      if (t < best_t) {
        best_t = t;
        best = lp;
      }
    }
  }
  // 384-token pair tiles (two N=192 MMAs per K step, each weight tile converted
  // for 384 tokens): taken over the 256-token pair tile when they need fewer
  // waves of CTA pairs after a 15% longer tile (measured: 8192x8192 M=768 51.0 ->
  // 40.7 us, 28672x8192 M=768 165 -> 121, 4096x11008 M=1024 52.1 -> 46.9,
  // 8192x28672 M=1024 222 -> 196; slower wherever the wave count does not drop)
  if (best.ntok == 256 && M >= 640 && mode != kModeI8) {
    const LaunchPlan lp256 = plan_for(mode, M, N, K, 256, 3, 0);
    const LaunchPlan lp384 = plan_for(mode, M, N, K, 384, 3, 0);
    const double pairs = std::max(1, pair_slots(mode));
    const double w256 = std::ceil(lp256.tiles / pairs), w384 = std::ceil(lp384.tiles / pairs);
    if (lp384.pair && w384 * 1.15 < w256) best = lp384;
  }
  return best;
}

// Workspace = [kMaxTiles int32 counters (fixed head, zero between launches)]
//             [split-K partial slots of the current plan (never need zeroing)].
constexpr int kMaxTiles = 65536;
constexpr size_t kCounterBytes = (size_t)kMaxTiles * 4;

static size_t plan_ws_bytes(const LaunchPlan& lp) {
  if (QQQ_CSB_L2 && lp.csplit > 1 && lp.ntok == 128)  // (S-1) received partials per tile, 64 KiB each
    return kCounterBytes + (size_t)lp.tiles * (lp.csplit - 1) * lp.ntok * 128 * 4;
  if (lp.aligned_tiles > 0 || lp.csplit > 1) return kCounterBytes;
  if (lp.pair) return kCounterBytes + (size_t)lp.tiles * 2 * lp.ntok * 128 * 4;  // a slot per (pair tile, CTA)
  return kCounterBytes + (size_t)lp.tiles * lp.ntok * 128 * 4;
}

template <int MODE, int NTOK, int BK, bool PAIR = false>
static int launch_t(const CUtensorMap& map, const CUtensorMap& ymap, const GemmParams& p, int grid,
                    cudaStream_t stream) {
  using C = Cfg<MODE, NTOK, BK, PAIR>;
  auto kern = w4a8_gemm_kernel<MODE, NTOK, BK, PAIR>;
  static bool attr_set[kMaxDevices] = {};  // per instantiation and device
  const int dev = cur_device();
  static const int one_per_sm = getenv("QQQ_EXP_ONE_CTA_PER_SM") ? 1 : 0;  // developer A/B switch
  const int smem_bytes = (one_per_sm && C::kSmall) ? 150 * 1024 : C::kSmemBytes;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
      return kErrCuda;
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(C::kNumThreads);
  lc.dynamicSmemBytes = smem_bytes;
  lc.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const int pdl = getenv("QQQ_NO_PDL") ? 0 : 1;  // developer A/B switch
  attr[0].val.programmaticStreamSerializationAllowed = pdl;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = PAIR ? 2 : (p.csplit > 1 ? p.csplit : 1);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = (PAIR || p.csplit > 1) ? 2 : 1;
  return cudaLaunchKernelEx(&lc, kern, map, ymap, p) == cudaSuccess ? kOk : kErrCuda;
}

template <int MODE>
static int launch_mode(int ntok, const CUtensorMap& map, const CUtensorMap& ymap, const GemmParams& p, int grid,
                       cudaStream_t st) {
  switch (ntok) {
    case 16: return launch_t<MODE, 16, bk_for(MODE, 16)>(map, ymap, p, grid, st);
    case 32: return launch_t<MODE, 32, bk_for(MODE, 32)>(map, ymap, p, grid, st);
    case 64: return launch_t<MODE, 64, bk_for(MODE, 64)>(map, ymap, p, grid, st);
    case 128: return launch_t<MODE, 128, bk_for(MODE, 128)>(map, ymap, p, grid, st);
    case 256: return launch_t<MODE, 256, bk_for(MODE, 256)>(map, ymap, p, grid, st);
    default: return kErrConfig;
  }
}

template <int MODE>
static int launch_pair(int ntok, const CUtensorMap& map, const CUtensorMap& ymap, const GemmParams& p, int grid,
                       cudaStream_t st) {
  if constexpr (MODE == kModeI8)
    return kErrConfig;
  else if (ntok == 192)  // double-buffered accumulators (2 x 192 + 4 A buffers of 32 TMEM columns)
    return launch_t<MODE, 192, kPairBk, true>(map, ymap, p, grid, st);
  else if (ntok == 384)  // 384-token tiles: each weight tile converted for more tokens
    return launch_t<MODE, 384, kPairBk, true>(map, ymap, p, grid, st);
  else if (ntok == 128)  // 128-token pair tiles: half the activation bytes per SM of a 128-token tile
    return launch_t<MODE, 128, kPairBk, true>(map, ymap, p, grid, st);
  else
    return launch_t<MODE, 256, kPairBk, true>(map, ymap, p, grid, st);
}

}  // namespace qqq

using namespace qqq;

extern "C" size_t qqq_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  size_t best = 0;  // any plan a caller may force or the cost model may pick
  for (int nt : {16, 32, 64, 128, 256}) {
    LaunchPlan lp = plan_for(kModePG, M, N, K, nt, 1, 0);  // slots do not change the slot bytes
    size_t b = plan_ws_bytes(lp);
    if (b > best) best = b;
  }
  for (int nt : {192, 256}) {
    LaunchPlan lp = plan_for(kModePG, M, N, K, nt, 5, 0);  // pair stream-K: a slot per (pair tile, CTA)
    best = std::max(best, plan_ws_bytes(lp));
  }
  for (int cs : {2, 4}) {  // 128-token clusters (partials exchanged through the workspace)
    LaunchPlan lp = plan_for(kModePG, M, N, K, 128, 4, 0, cs);
    best = std::max(best, plan_ws_bytes(lp));
  }
  return best;
}

// The tile plan a launch with these arguments would use (the planner's pick,
// or the forced plan resolved the way the launch resolves it).
extern "C" int qqq_gemm_plan_info(int mode, int64_t M, int64_t N, int64_t K, const qqq_gemm_config* cfg,
                                  qqq_gemm_config* out) {
  if (M <= 0 || N <= 0 || K <= 0 || !out) return kErrShape;
  const LaunchPlan lp = make_plan(mode, M, N, K, cfg ? cfg->ntok : 0, cfg ? cfg->grid : 0, cfg ? cfg->split : -1,
                                  cfg ? cfg->csplit : 0);
  out->ntok = lp.ntok;
  out->grid = lp.grid;
  out->csplit = lp.csplit;
  out->dbg = nullptr;
  if (lp.csplit > 1)
    out->split = 4;
  else if (lp.pair)
    out->split = lp.aligned_tiles > 0 ? 3 : lp.dp_tiles > 0 ? 6 : 5;
  else
    out->split = lp.aligned_tiles > 0 ? 0 : lp.dp_tiles > 0 ? 2 : 1;
  return kOk;
}

// Generic entry: mode 0 = per-channel (PC), 1 = per-group (PG), 2 = pre-converted int8 (I8).
namespace qqq {
// fused smoothed quantization inputs (qqq_w4a8_gemm_smooth_fused)
struct FusedQuantArgs {
  const void* x;
  int64_t ldx;
  const double* smooth;
  const double* recip;
  int32_t* status;
};

static int gemm_launch(int mode, const int8_t* aq, int64_t ldq, const double* s_a, const int32_t* rowsum,
                       const void* w_repacked, int64_t group, const double* s_col, int64_t M, int64_t N, int64_t K,
                       void* y, int64_t ldy, int32_t* acc_opt, int64_t ldacc, void* workspace, size_t ws_bytes,
                       const qqq_gemm_config* cfg, cudaStream_t stream, const FusedQuantArgs* fq) {
  if (M < 0 || N <= 0 || K <= 0) return kErrShape;
  if (K > (1 << 16)) return kErrShape;  // gemm.py:49,151
  if (M == 0) return kOk;
  if (mode == kModePG && !pg_group_ok(group)) return kErrUnsupported;
  if (mode == kModePG && !rowsum) return kErrConfig;
  // 3-D activation view {128, M, ceil(K/128)}: rows must hold round_up(K, 128) bytes
  if ((ldq % 16) != 0 || ldq < round_up(K, 128) || (reinterpret_cast<uintptr_t>(aq) & 15) != 0)
    return kErrUnsupported;
  if (s_col && (!y || ldy < N)) return kErrShape;
  if (!s_col && !acc_opt) return kErrConfig;
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return kErrCuda;

  LaunchPlan lp = make_plan(mode, M, N, K, cfg ? cfg->ntok : 0, cfg ? cfg->grid : 0, cfg ? cfg->split : -1,
                            cfg ? cfg->csplit : 0);
  // (the fused quantization keeps 6 int32 slots per token row below its row counter)
  if (lp.tiles * (lp.pair ? 2 : 1) > (fq ? kQRowsSlot - 6 * M - 2 : (int64_t)kMaxTiles) || lp.units > 0x7fffffff)
    return kErrUnsupported;
  if (ws_bytes < plan_ws_bytes(lp)) return kErrConfig;

  CUtensorMap map;
  const int64_t katoms = (K + 127) / 128;
  cuuint64_t dims[3] = {128u, (cuuint64_t)M, (cuuint64_t)katoms};
  cuuint64_t strides[2] = {(cuuint64_t)ldq, 128u};
#ifdef QQQ_EXP_HALF_X
  cuuint32_t box[3] = {128u, (cuuint32_t)(lp.ntok >= 128 ? lp.ntok / 2 : lp.ntok), (cuuint32_t)(lp.bk / 128)};
#else
  // (pair CTAs load half the tile's tokens; 384-token tiles in two 96-row chunks)
  cuuint32_t box[3] = {128u, (cuuint32_t)(lp.ntok == 384 ? 96 : lp.pair ? lp.ntok / 2 : lp.ntok),
                       (cuuint32_t)(lp.bk / 128)};
#endif
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)aq, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return kErrCuda;

  // y: fp16 [M, N] (row pitch ldy elements); TMA store box = 128 channels x 16 tokens
  CUtensorMap ymap;
  memset(&ymap, 0, sizeof(ymap));
  int y_tma = 0;
  static const bool no_ytma = getenv("QQQ_EXP_NO_YTMA") != nullptr;
  if (s_col && y && !no_ytma && (ldy * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
    cuuint64_t ydims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t ystr[1] = {(cuuint64_t)(ldy * 2)};
    cuuint32_t ybox[2] = {32u, 16u};  // one epilogue warp's [16 tok][32 ch] chunk
    cuuint32_t yes[2] = {1u, 1u};
    if (enc(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, y, ydims, ystr, ybox, yes, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      y_tma = 1;
  }

  GemmParams p{};
  p.y_tma = y_tma;
  p.w = (const uint8_t*)w_repacked;
  p.s_a = s_a;
  p.rowsum = rowsum;
  p.s_col = s_col;
  p.y = (__half*)y;
  p.ldy = ldy;
  p.acc = acc_opt;
  p.ldacc = ldacc;
  p.counters = (int32_t*)workspace;
  p.ws = (int32_t*)((uint8_t*)workspace + kCounterBytes);
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.n_tiles = lp.n_tiles;
  p.tok_tiles = lp.tok_tiles;
  p.kb_per_tile = lp.kb_per_tile;
  p.ss_per_tile = (int)(round_up(K, kKPadTo) / kSuperK);
  p.ss_bytes = (int)ss_bytes(mode, group);
  p.group = (int)group;
  p.max_segs = lp.max_segs;
  p.units = lp.units;
  p.aligned_tiles = lp.aligned_tiles;
  p.dp_tiles = lp.dp_tiles;
  p.sk_unit0 = lp.sk_unit0;
  p.pair = lp.pair;
  p.csplit = lp.csplit;
  p.dbg = cfg ? (unsigned long long*)cfg->dbg : nullptr;
  if (fq) {
    p.xsrc = (const __half*)fq->x;
    p.ldx = fq->ldx;
    p.smooth = fq->smooth;
    p.srecip = fq->recip;
    p.qdst = const_cast<int8_t*>(aq);
    p.ldq = ldq;
    p.sa_dst = const_cast<double*>(s_a);
    p.rs_dst = const_cast<int32_t*>(rowsum);
    p.status = fq->status;
    p.q_ctas = std::min(lp.grid, num_sms());  // CTAs of the first wave (co-resident)
  }

  if (lp.pair) {
    switch (mode) {
      case kModePC: return launch_pair<kModePC>(lp.ntok, map, ymap, p, lp.grid, stream);
      case kModePG: return launch_pair<kModePG>(lp.ntok, map, ymap, p, lp.grid, stream);
      default: return kErrConfig;
    }
  }
  switch (mode) {
    case kModePC: return launch_mode<kModePC>(lp.ntok, map, ymap, p, lp.grid, stream);
    case kModePG: return launch_mode<kModePG>(lp.ntok, map, ymap, p, lp.grid, stream);
    case kModeI8: return launch_mode<kModeI8>(lp.ntok, map, ymap, p, lp.grid, stream);
    default: return kErrConfig;
  }
}

}  // namespace qqq

extern "C" int qqq_w4a8_gemm_ex(int mode, const int8_t* aq, int64_t ldq, const double* s_a, const int32_t* rowsum,
                                const void* w_repacked, int64_t group, const double* s_col, int64_t M, int64_t N,
                                int64_t K, void* y, int64_t ldy, int32_t* acc_opt, int64_t ldacc, void* workspace,
                                size_t ws_bytes, const qqq_gemm_config* cfg, cudaStream_t stream) {
  return gemm_launch(mode, aq, ldq, s_a, rowsum, w_repacked, group, s_col, M, N, K, y, ldy, acc_opt, ldacc, workspace,
                     ws_bytes, cfg, stream, nullptr);
}

// apply_quant_linear's activation step fused into the GEMM (pipeline.py:144-152):
// quantize x / smooth (fp16 [M, K]) into (q, s_a, rowsum) exactly as
// qqq_act_quant_smooth(_rcp) does, inside the GEMM launch, then the GEMM on them.
extern "C" int qqq_w4a8_gemm_smooth_fused(int mode, const void* x, int64_t ldx, const double* smooth,
                                          const double* smooth_recip, int8_t* q, int64_t ldq, double* s_a,
                                          int32_t* rowsum, int32_t* status_dev, const void* w_repacked, int64_t group,
                                          const double* s_col, int64_t M, int64_t N, int64_t K, void* y, int64_t ldy,
                                          int32_t* acc_opt, int64_t ldacc, void* workspace, size_t ws_bytes,
                                          const qqq_gemm_config* cfg, cudaStream_t stream) {
  if (mode != kModePC && mode != kModePG) return kErrConfig;
  if (!x || !smooth || !q || !s_a || !rowsum || !status_dev) return kErrConfig;
  if (M > 0 && (K % 8 != 0 || ldx % 8 != 0 || ldx < K || (reinterpret_cast<uintptr_t>(x) & 15) != 0 ||
                (reinterpret_cast<uintptr_t>(smooth) & 15) != 0 ||
                (smooth_recip && (reinterpret_cast<uintptr_t>(smooth_recip) & 15) != 0)))
    return kErrUnsupported;
  const FusedQuantArgs fq{x, ldx, smooth, smooth_recip, status_dev};
  return gemm_launch(mode, q, ldq, s_a, rowsum, w_repacked, group, s_col, M, N, K, y, ldy, acc_opt, ldacc, workspace,
                     ws_bytes, cfg, stream, &fq);
}

extern "C" int qqq_w4a8_gemm_pc(const int8_t* aq, int64_t ldq, const double* s_a, const void* w_repacked,
                                const double* s_w_folded, int64_t M, int64_t N, int64_t K, void* y, int64_t ldy,
                                int32_t* acc_opt, int64_t ldacc, void* workspace, size_t ws_bytes, cudaStream_t stream) {
  return qqq_w4a8_gemm_ex(kModePC, aq, ldq, s_a, nullptr, w_repacked, 0, s_w_folded, M, N, K, y, ldy, acc_opt, ldacc,
                          workspace, ws_bytes, nullptr, stream);
}

extern "C" int qqq_w4a8_gemm_pg(const int8_t* aq, int64_t ldq, const double* s_a, const int32_t* rowsum,
                                const void* w_repacked, int64_t group, const double* s_wc, int64_t M, int64_t N,
                                int64_t K, void* y, int64_t ldy, int32_t* acc_opt, int64_t ldacc, void* workspace,
                                size_t ws_bytes, cudaStream_t stream) {
  return qqq_w4a8_gemm_ex(kModePG, aq, ldq, s_a, rowsum, w_repacked, group, s_wc, M, N, K, y, ldy, acc_opt, ldacc,
                          workspace, ws_bytes, nullptr, stream);
}
