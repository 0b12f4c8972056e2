// Shared device helpers for the B200 (sm_100a) W4A8 path: PTX wrappers for
// mbarrier / TMA / tcgen05, and the bit-exact INT4 -> INT8 conversions of the
// QQQ dataflows (reference: pkg/src/qqq/gemm.py:81-142).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "qqq_b200.h"  // the C ABI these kernels implement

#define QQQ_DEVICE __device__ __forceinline__

// Watchdog of the spin waits (ns): a wait that never completes traps the launch
// instead of hanging the GPU. Sanitizer builds raise it (tools serialise CTAs).
#ifndef QQQ_WATCHDOG_NS
#define QQQ_WATCHDOG_NS 4000000000ull
#endif
#ifndef QQQ_WATCHDOG_ITERS
#define QQQ_WATCHDOG_ITERS (1u << 24)
#endif

namespace qqq {

// ----------------------------------------------------------------------------
// Status codes shared with include/qqq_b200.h
// ----------------------------------------------------------------------------
enum : int {
  kOk = 0,
  kErrShape = 1,
  kErrData = 2,
  kErrConfig = 3,
  kErrCorruption = 4,
  kErrCuda = 5,
  kErrUnsupported = 6,
};

// device-side status bits (written with atomicOr into a caller-owned int32)
enum : int {
  kStatNonFinite = 1,     // quant_act_per_token / weight quantizers: DataError
  kStatCodeRange = 2,     // pack_i4: code outside [-8, 7]: DataError
  kStatPadNibble = 4,     // unpack_i4: nonzero odd-K padding: CorruptionError
  kStatScaleInf = 8,      // FusedScales.from_quantized: s* overflows binary16
  kStatNeedClamp = 16,    // repack: some s* needs the FusedDequantQuant clamp
  kStatTinyScale = 32,    // repack: some s* < 2^-10 (s*/16 inexact)
};

// ----------------------------------------------------------------------------
// Generic small helpers
// ----------------------------------------------------------------------------
QQQ_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

QQQ_DEVICE uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

QQQ_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ----------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------
QQQ_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

QQQ_DEVICE void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

QQQ_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

QQQ_DEVICE void mbar_arrive_addr(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

QQQ_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Parity wait. A watchdog turns a pipeline deadlock into a trapped launch
// (cudaErrorLaunchFailure) after ~2^24 polls (seconds) instead of hanging the GPU.
QQQ_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
#pragma unroll 1
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
#ifndef QQQ_NO_WATCHDOG
    if (n > QQQ_WATCHDOG_ITERS) __trap();
#endif
  }
}

// Parity wait for roles that idle for long stretches (epilogue, producers):
// the try_wait carries a suspend-time hint, so the warp sleeps in hardware
// until the phase completes instead of re-issuing the poll loop at high warp
// priority and stealing issue slots from the converter warps.
QQQ_DEVICE void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  unsigned long long t0 = 0;
#pragma unroll 1
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(0x100000u)
        : "memory");
    if (done) return;
#ifndef QQQ_NO_WATCHDOG
    // a suspended poll may last up to the hint: bound the wait in time (~4 s)
    if ((n & 255) == 255) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > QQQ_WATCHDOG_NS) __trap();
    }
#endif
  }
}

// ---- 2-CTA cluster (cta_group::2) helpers ----
QQQ_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of `p` (a shared::cta variable) in CTA `rank` of the cluster
QQQ_DEVICE uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
QQQ_DEVICE uint32_t mapa_shared_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on a barrier of another CTA of the cluster. Default (.release.cta)
// semantics: a .cluster-scope release compiles to MEMBAR.ALL.GPU, which under a
// streaming HBM load costs ~0.9 us per arrive (measured); the data it guards
// is tcgen05/async-proxy traffic, ordered by the tcgen05 fences and the
// mbarrier itself.
QQQ_DEVICE void mbar_arrive_cluster(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
// parity wait with an explicit cluster-scope ACQUIRE: data published by peer
// CTAs (global-memory stores, fence.acq_rel.gpu, remote arrive) is visible after it
QQQ_DEVICE void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  unsigned long long t0 = 0;
#pragma unroll 1
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(0x100000u)
        : "memory");
    if (done) return;
#ifndef QQQ_NO_WATCHDOG
    if ((n & 255) == 255) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > QQQ_WATCHDOG_NS) __trap();
    }
#endif
  }
}
// parity wait with cluster-scope acquire (arrivals come from the peer CTA too)
QQQ_DEVICE void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  unsigned long long t0 = 0;
#pragma unroll 1
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(0x100000u)
        : "memory");
    if (done) return;
#ifndef QQQ_NO_WATCHDOG
    if ((n & 255) == 255) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > QQQ_WATCHDOG_NS) __trap();
    }
#endif
  }
}
// Cluster-wide barrier, relaxed arrive: what it publishes (mbarrier inits) is
// made visible by fence.mbarrier_init.release.cluster, and the end-of-kernel use
// only orders completed DSMEM traffic; a .release arrive costs a MEMBAR.GPU per
// thread (~1 us under a streaming HBM load).
QQQ_DEVICE void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

// Parity wait for a role that idles for most of the kernel (the epilogue
// waiting for its accumulator): exponential __nanosleep backoff capped at
// 256 ns. A NANOSLEEP.SYNCS wait is woken by every mbarrier event in the CTA
// and re-polls ~1M times per decode kernel (30% extra issue pressure on the
// converters' sub-partitions, measured with ncu); this polls ~100 times.
QQQ_DEVICE void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0, ns = 32;
#pragma unroll 1
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
#ifndef QQQ_NO_WATCHDOG
    if (n > QQQ_WATCHDOG_ITERS) __trap();
#endif
  }
}

// ----------------------------------------------------------------------------
// TMA / bulk copies (async proxy)
// ----------------------------------------------------------------------------
QQQ_DEVICE void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

QQQ_DEVICE void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem_dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

QQQ_DEVICE void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

QQQ_DEVICE void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ----------------------------------------------------------------------------
// tcgen05 (5th-gen tensor core, TMEM accumulators)
// ----------------------------------------------------------------------------
QQQ_DEVICE void tmem_alloc(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

QQQ_DEVICE void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// pair (cta_group::2) TMEM allocation: the warp with the same id in both CTAs
// of the pair executes it; both CTAs get the same column range
QQQ_DEVICE void tmem_alloc_pair(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
QQQ_DEVICE void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// pair MMA (issued by the even CTA): D (M = 256 rows, 128 per CTA's TMEM) (+)=
// A[tmem, 128 rows per CTA] * B[smem, N/2 rows per CTA]^T
QQQ_DEVICE void mma_i8_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit of the pair's MMAs, arriving on the barrier at the same offset in every CTA of `mask`
QQQ_DEVICE void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

QQQ_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
QQQ_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32 (kind::i8)
QQQ_DEVICE void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, int8 x int8 -> int32 (A K-major in TMEM:
// lane = row, each 32-bit column packs 4 consecutive k; one K=32 step = 8 columns)
QQQ_DEVICE void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32-bit, 8 consecutive columns per thread (thread i -> lane base + i)
QQQ_DEVICE void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

QQQ_DEVICE void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

QQQ_DEVICE void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

QQQ_DEVICE void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32-bit, 16 consecutive columns per thread, and the wait for the
// load in the SAME asm statement. tcgen05.ld writes its destination registers
// asynchronously (they are valid only after tcgen05.wait::ld); as two asm
// statements the compiler may copy or spill the outputs between them — it did
// once register pressure rose (64-register half-SM CTAs), storing garbage for
// the 32-token cluster split-K partials.
QQQ_DEVICE void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
#ifndef QQQ_EXP_SPLITLD
      "tcgen05.wait::ld.sync.aligned;"
#endif
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#ifdef QQQ_EXP_SPLITLD
  tmem_wait_ld();
#endif
}

// Two 16-column TMEM loads (columns at taddr_a and taddr_b) and ONE wait:
// the epilogue's paired chunks pay the tcgen05.ld latency once.
QQQ_DEVICE void tmem_ld16x2(uint32_t taddr_a, uint32_t taddr_b, uint32_t (&a)[16], uint32_t (&b)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
        "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]),
        "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
        "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15])
      : "r"(taddr_a), "r"(taddr_b)
      : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "version 1" format).
//   layout: 0 = SWIZZLE_NONE (canonical interleaved core matrices), 2 = SWIZZLE_128B
QQQ_DEVICE uint64_t make_smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  d |= (uint64_t)(layout & 0x7) << 61;
  return d;
}

// Instruction descriptor for kind::i8: (s8|u8) x s8 -> s32, both operands K-major.
__host__ __device__ constexpr uint32_t make_idesc_i8(uint32_t M, uint32_t N, bool a_unsigned = false) {
  return (2u << 4)                      // c_format = S32
         | ((a_unsigned ? 0u : 1u) << 7)  // a_format: 0 = unsigned, 1 = signed int8
         | (1u << 10)         // b_format = signed int8
         | ((N >> 3) << 17)   // n_dim
         | ((M >> 4) << 24);  // m_dim
}

// ----------------------------------------------------------------------------
// QQQ conversions (bit-exact with gemm.py)
// ----------------------------------------------------------------------------

// Per-channel FastINT4toINT8 (gemm.py:81-85, applied as `codes*16` at :180):
// one 32-bit word of the per-channel kernel layout holds 8 biased nibbles u=q+8;
// byte j's low nibble is k=4i+j and its high nibble is k=16+4i+j. Returns the
// two int8x4 words 16*q (low nibbles) and 16*q (high nibbles):
//   (u << 4) ^ 0x80  ==  16*(u-8) as a two's-complement byte.
QQQ_DEVICE void pc_convert_word(uint32_t w, uint32_t& lo, uint32_t& hi) {
  lo = ((w << 4) & 0xF0F0F0F0u) ^ 0x80808080u;
  hi = (w & 0xF0F0F0F0u) ^ 0x80808080u;
}

QQQ_DEVICE uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
QQQ_DEVICE __half2 u32_as_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// Per-group FusedDequantQuant (gemm.py:110-142) on one word of the per-group
// kernel layout. Nibble p sits at bits 4p; pairs (p, p+4) form half2 lanes and
// cover k = (0,1) p=0, (2,3) p=1, (4,5) p=2, (6,7) p=3 of this word's 8 k's.
//   FastINT4toFP16: half(0x6400|u) = 1024+u ; minus 1032 -> q exactly
//   odd pairs use the nibble in place (1024+16u), minus 1152 -> 16q, and are
//   multiplied by s*/16 (exact when s* >= 2^-10, checked at repack time) so the
//   single-rounding FMA q*s* + 1152 is computed identically.
//   FastFP16toINT8: low byte of the fp16 bits, XOR 0x80.
// kClamp reproduces the reference's out-of-range clamp to [-127, 127]; the
// repack proves it unnecessary for the weights it accepts on the fast path.
// (a & MASK) | c in ONE lop3 (the magic constant is kept in a register so the
// single-immediate LOP3 encoding can take the mask)
template <uint32_t MASK>
QQQ_DEVICE uint32_t and_or(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(MASK), "r"(c));
  return d;
}

// kUnsigned: emit w8 + 128 as an unsigned byte (skip the XOR 0x80); the GEMM
// then runs a u8 x s8 MMA and subtracts 128 * rowsum(activation codes).
template <bool kClamp, bool kUnsigned = false>
QQQ_DEVICE void pg_convert_word(uint32_t w, __half2 s2, __half2 s2_16, uint32_t magic, uint32_t& out_lo,
                                uint32_t& out_hi) {
  const __half2 k1032 = u32_as_h2(0xE408E408u);  // -1032.0
  const __half2 k1152 = u32_as_h2(0xE480E480u);  // -1152.0
  const __half2 kAdd = u32_as_h2(0x64806480u);   // +1152.0
  uint32_t a = and_or<0x000F000Fu>(w, magic);
  uint32_t b = and_or<0x00F000F0u>(w, magic);
  uint32_t w8 = w >> 8;
  uint32_t c = and_or<0x000F000Fu>(w8, magic);
  uint32_t d = and_or<0x00F000F0u>(w8, magic);
  __half2 ra = __hfma2(__hadd2(u32_as_h2(a), k1032), s2, kAdd);
  __half2 rb = __hfma2(__hadd2(u32_as_h2(b), k1152), s2_16, kAdd);
  __half2 rc = __hfma2(__hadd2(u32_as_h2(c), k1032), s2, kAdd);
  __half2 rd = __hfma2(__hadd2(u32_as_h2(d), k1152), s2_16, kAdd);
  if (kClamp) {
    const __half2 lo = u32_as_h2(0x64016401u);  // 1025
    const __half2 hi = u32_as_h2(0x64FF64FFu);  // 1279
    ra = __hmin2(__hmax2(ra, lo), hi);
    rb = __hmin2(__hmax2(rb, lo), hi);
    rc = __hmin2(__hmax2(rc, lo), hi);
    rd = __hmin2(__hmax2(rd, lo), hi);
  }
  out_lo = __byte_perm(h2_as_u32(ra), h2_as_u32(rb), 0x6420);
  out_hi = __byte_perm(h2_as_u32(rc), h2_as_u32(rd), 0x6420);
  if (!kUnsigned) {
    out_lo ^= 0x80808080u;
    out_hi ^= 0x80808080u;
  }
}

// Scalar FusedDequantQuant with the reference's full branch structure
// (gemm.py:110-127 / vectorized :130-142): fma(q, s*, 1152) in binary16 with a
// single rounding, then the aligned-window test on the bit pattern.
QQQ_DEVICE int8_t fused_dequant_quant_scalar(int q, __half s_star) {
  __half r = __hfma(__int2half_rn(q), s_star, __float2half_rn(1152.0f));
  uint16_t bits = __half_as_ushort(r);
  if (bits >= 0x6400 && bits < 0x6500) {
    int b = (bits & 0xFF) ^ 0x80;
    int v = b >= 128 ? b - 256 : b;
    return (int8_t)(v < -127 ? -127 : v);
  }
  // prod = q*s* is exact; its sign decides the saturation side
  float prod = (float)q * __half2float(s_star);
  return (int8_t)(prod > 0.0f ? 127 : -127);
}

// FastFP16toINT8 (gemm.py:99-107): fma with multiplicand 1.0, low byte ^ 0x80
QQQ_DEVICE int8_t fast_f16_to_i8(__half x) {
  __half r = __hadd(x, __float2half_rn(1152.0f));
  int b = (__half_as_ushort(r) & 0xFF) ^ 0x80;
  return (int8_t)(b >= 128 ? b - 256 : b);
}

}  // namespace qqq
