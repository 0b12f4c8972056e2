// Per-token symmetric INT8 activation quantization on B200.
//
// Reference: pkg/src/qqq/quantize.py:92-100 (quant_act_per_token)
//   m = max_k |x[t,k]| ; s = m/127 (f64) or 1.0 if m == 0
//   q = clip(rint(x / s), -127, 127)       (f64 divide, half-even rint)
//   non-finite input -> DataError (quantize.py:85-89)
//
// One CTA per token row: a vectorised 16-byte absmax pass (warp shuffles +
// shared-memory block reduce) followed by a quantize pass that re-reads the
// row from L1/L2 and writes 16-byte int8 vectors.
//
// Bit-exactness for fp16 input: the fast path
// computes t = x * RN(127/m) in fp32 (|t - x*127/m| <= 2*127*2^-24 < 2e-5).
// Whenever t is within 1e-3 of a half-integer we recompute the reference
// formula rint(x / (m/127.0)) in f64 verbatim, so the result equals the
// reference on every input, ties included (the reference is not half-even on
// exact ties because of its double rounding). f32/f64 inputs always take the
// verbatim f64 formula.
#include <type_traits>

#include "act_quant_dev.cuh"
#include "qqq_common.cuh"

namespace qqq {

template <int kThreads, typename Acc>
QQQ_DEVICE Acc block_max(Acc v, Acc* red) {
  for (int o = 16; o > 0; o >>= 1) { Acc t = __shfl_xor_sync(0xffffffffu, v, o); v = t > v ? t : v; }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < kThreads / 32) ? red[l] : Acc(0);
    for (int o = 16; o > 0; o >>= 1) { Acc t = __shfl_xor_sync(0xffffffffu, v, o); v = t > v ? t : v; }
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// kSmooth: the reference's apply_quant_linear (pipeline.py:144-152) quantizes
// x / s with the smoothing vector s (f64, per input channel) divided in f64
// first: every element is then an f64 value, so absmax and codes use the
// verbatim f64 formula (IEEE division, as numpy).
template <typename T, int kThreads, bool kSmooth = false>
__global__ void __launch_bounds__(kThreads) act_quant_kernel(const T* __restrict__ x, int64_t K, int64_t ldx,
                                                              int8_t* __restrict__ q, int64_t ldq,
                                                              double* __restrict__ s_out, int32_t* status,
                                                              const double* __restrict__ row_max_in,
                                                              double* __restrict__ row_max_out,
                                                              int32_t* __restrict__ rowsum_out,
                                                              const double* __restrict__ smooth = nullptr) {
  using Acc = typename std::conditional<sizeof(T) == 8 || kSmooth, double, float>::type;
  __shared__ Acc red[32];
  // PDL: let the GEMM that consumes q start its prologue / weight prefetch now,
  // and wait for whatever produced x before reading it.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t row = blockIdx.x;
  const T* xr = x + row * ldx;
  int8_t* qr = q + row * ldq;

  // ---- pass 1: absmax + finiteness -------------------------------------------------
  Acc m = Acc(0);
  bool bad = false;
  constexpr int kVec = 16 / sizeof(T);
  const bool vec_ok = (K % kVec == 0) && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
  if (vec_ok) {
    const int64_t nv = K / kVec;
    const uint4* xv = reinterpret_cast<const uint4*>(xr);
    for (int64_t i = threadIdx.x; i < nv; i += kThreads) {
      uint4 pk = __ldg(xv + i);
      const T* e = reinterpret_cast<const T*>(&pk);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        Acc a;
        if constexpr (kSmooth) {
          a = fabs(smooth_div(to_f64<T>(e[j]), smooth[i * kVec + j]));
        } else {
          a = absval(e[j]);
        }
        bad |= is_bad(a);  // inf or NaN
        m = a > m ? a : m;
      }
    }
  } else {
    for (int64_t i = threadIdx.x; i < K; i += kThreads) {
      Acc a;
      if constexpr (kSmooth) {
        a = fabs(smooth_div(to_f64<T>(xr[i]), smooth[i]));
      } else {
        a = absval(xr[i]);
      }
      bad |= is_bad(a);
      m = a > m ? a : m;
    }
  }
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) atomicOr(status, kStatNonFinite);
  }
  m = block_max<kThreads, Acc>(m, red);
  if (row_max_out) {  // absmax-only pass (K-split tensor parallelism: all-reduce MAX follows)
    if (threadIdx.x == 0) row_max_out[row] = (double)m;
    return;
  }
  if (row_max_in) m = (Acc)row_max_in[row];  // the full-row max from the all-reduce (exact: fp16/fp32 values)
  const double s = (m > Acc(0)) ? (double)m / 127.0 : 1.0;
  if (threadIdx.x == 0) s_out[row] = s;

  // ---- pass 2: codes ----------------------------------------------------------------
  const bool zero_row = !(m > Acc(0));
  const float inv = zero_row ? 0.0f : 127.0f / (float)m;  // fp16 path only
  const double inv64 = 1.0 / s;                            // smoothed (f64) path
  auto code = [&](T v, int64_t k) -> int8_t {
    if (zero_row) return 0;
    if constexpr (kSmooth) {
      return quant_code_f64(smooth_div(to_f64<T>(v), smooth[k]), inv64, s);
    } else if constexpr (sizeof(T) == 2) {
      return quant_code_f16(__half2float(v), inv, s);
    } else {
      return quant_code_exact(to_f64<T>(v), s);
    }
  };
  const bool qvec_ok = vec_ok && (K % 16 == 0) && ((reinterpret_cast<uintptr_t>(qr) & 15) == 0);
  int csum = 0;  // sum of this thread's codes (for the u8 x s8 per-group GEMM correction)
  if (qvec_ok) {
    // 16 codes per thread-iteration: 16 * sizeof(T) bytes in, 16 bytes out
    const int64_t n16 = K / 16;
    for (int64_t i = threadIdx.x; i < n16; i += kThreads) {
      alignas(16) int8_t out[16];
#pragma unroll
      for (int h = 0; h < (int)sizeof(T); ++h) {
        uint4 pk = __ldg(reinterpret_cast<const uint4*>(xr + i * 16) + h);
        const T* e = reinterpret_cast<const T*>(&pk);
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          out[h * kVec + j] = code(e[j], i * 16 + h * kVec + j);
          csum += out[h * kVec + j];
        }
      }
      *reinterpret_cast<uint4*>(qr + i * 16) = *reinterpret_cast<const uint4*>(out);
    }
  } else {
    for (int64_t i = threadIdx.x; i < K; i += kThreads) {
      const int8_t c = code(xr[i], i);
      qr[i] = c;
      csum += c;
    }
  }
  if (rowsum_out) {
    __shared__ int isum[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if ((threadIdx.x & 31) == 0) isum[threadIdx.x >> 5] = csum;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int i = 0; i < kThreads / 32; ++i) t += isum[i];
      rowsum_out[row] = t;
    }
  }
}

// Register-resident variant for rows that fit in one CTA's registers (fp16
// input, K <= kThreads * kVPT * 8): every thread issues its kVPT 16-byte loads
// up front (one HBM/L2 round trip per row instead of one per loop trip), the
// row max is one warp-shuffle + shared-memory reduction, and the codes are
// computed from the registers (no second pass over x). Same arithmetic as
// act_quant_kernel, so the same bit-exactness argument holds.
template <int kThreads, int kVPT, bool kSmooth>
__global__ void __launch_bounds__(kThreads) act_quant_row_kernel(const __half* __restrict__ x, int64_t K, int64_t ldx,
                                                                  int8_t* __restrict__ q, int64_t ldq,
                                                                  double* __restrict__ s_out, int32_t* status,
                                                                  int32_t* __restrict__ rowsum_out,
                                                                  const double* __restrict__ smooth,
                                                                  const uint8_t* __restrict__ smooth_mask,
                                                                  const double* __restrict__ recip) {
  using Acc = typename std::conditional<kSmooth, double, float>::type;
  __shared__ Acc red[32];
  __shared__ int isum[kThreads / 32];
  // x / s_k for the 8 channels of vector i: s_k is read only for smoothed
  // channels (mask bit set), the rest divide by 1.0 exactly (= x)
  auto sdiv = [&](double xv, int64_t i, int t, uint32_t mbits) -> double {
    if (smooth_mask == nullptr) return smooth_div(xv, smooth[i * 8 + t]);
    return ((mbits >> t) & 1u) ? xv / smooth[i * 8 + t] : xv;
  };
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t row = blockIdx.x;
  const uint4* xv = reinterpret_cast<const uint4*>(x + row * ldx);
  const int64_t nv = K / 8;  // 16-byte vectors in the row
  uint4 v[kVPT];
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int64_t i = threadIdx.x + (int64_t)j * kThreads;
    v[j] = i < nv ? __ldg(xv + i) : make_uint4(0, 0, 0, 0);
  }
  uint32_t mb[kVPT];
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int64_t i = threadIdx.x + (int64_t)j * kThreads;
    mb[j] = (kSmooth && smooth_mask != nullptr && i < nv) ? (uint32_t)__ldg(smooth_mask + i) : 0u;
    // the smoothing values are consumed vector by vector below: start all their
    // fetches now (no registers held) so those loads hit L1
    if (kSmooth && smooth_mask == nullptr && i < nv) asm volatile("prefetch.global.L1 [%0];" ::"l"(smooth + i * 8));
  }
  Acc m = Acc(0);
  bool bad = false;
  // smoothed rows: the quotients x / s_k (IEEE f64 division, once per element,
  // unconditionally — x / 1.0 == x, and a per-lane `s_k == 1` branch diverges in
  // nearly every warp anyway) stay in registers for the code pass; s_k is read
  // as 16-byte pairs
  double xs[kSmooth ? kVPT : 1][8];
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int64_t i = threadIdx.x + (int64_t)j * kThreads;
    if (i < nv) {
      const __half* e = reinterpret_cast<const __half*>(&v[j]);
      if constexpr (kSmooth) {
        if (recip != nullptr) {  // Markstein division with the reciprocal table
          smooth8(v[j], smooth, recip, i, xs[j]);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const Acc a = fabs(xs[j][t]);
            bad |= is_bad(a);
            m = a > m ? a : m;
          }
          continue;
        }
        double sk[8];
        if (smooth_mask == nullptr) {
          const double2* sv = reinterpret_cast<const double2*>(smooth + i * 8);  // 64 B per vector
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double2 d = __ldg(sv + h);
            sk[2 * h] = d.x;
            sk[2 * h + 1] = d.y;
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double xv = (double)__half2float(e[t]);
          xs[j][t] = smooth_mask == nullptr ? xv / sk[t] : sdiv(xv, i, t, mb[j]);
          const Acc a = fabs(xs[j][t]);
          bad |= is_bad(a);
          m = a > m ? a : m;
        }
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const Acc a = absval(e[t]);
          bad |= is_bad(a);
          m = a > m ? a : m;
        }
      }
    }
  }
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) atomicOr(status, kStatNonFinite);
  }
  m = block_max<kThreads, Acc>(m, red);
  const double s = (m > Acc(0)) ? (double)m / 127.0 : 1.0;
  if (threadIdx.x == 0) s_out[row] = s;
  const bool zero_row = !(m > Acc(0));
  const float inv = zero_row ? 0.0f : 127.0f / (float)m;
  const double rs = 1.0 / s;
  const bool ieee = !markstein_safe(s);
  int8_t* qr = q + row * ldq;
  int csum = 0;
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int64_t i = threadIdx.x + (int64_t)j * kThreads;
    if (i < nv) {
      uint2 o;
      if constexpr (kSmooth)
        o = codes8_f64(xs[j], s, rs, ieee, csum);
      else
        o = codes8_f16(v[j], inv, s, rs, csum);
      *reinterpret_cast<uint2*>(qr + i * 8) = o;
    }
  }
  if (rowsum_out) {
    for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if ((threadIdx.x & 31) == 0) isum[threadIdx.x >> 5] = csum;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < kThreads / 32; ++w) t += isum[w];
      rowsum_out[row] = t;
    }
  }
}

QQQ_DEVICE uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
QQQ_DEVICE void st_async_b64(uint32_t cl_addr, uint64_t v, uint32_t cl_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(cl_addr), "l"(v),
               "r"(cl_bar)
               : "memory");
}
QQQ_DEVICE void st_async_b32(uint32_t cl_addr, uint32_t v, uint32_t cl_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(cl_addr), "r"(v),
               "r"(cl_bar)
               : "memory");
}

// Small-M variant (decode batches): a token row is split over a cluster of G =
// ceil(K/8 / kThreads) CTAs, one 16-byte vector per thread, so the per-thread
// dependent work is one vector instead of up to 4 (the row kernel's latency is
// instruction-bound: ~135 instructions per element with the smoothing
// division). The CTAs exchange their partial absmax (st.async into every
// peer's shared memory, completing on its mbarrier) and their code sums (into
// rank 0, which writes s_a and rowsum). Same arithmetic as the row kernel.
template <int kThreads, bool kSmooth, int kVPT = 1>
#ifndef QQQ_QCLUSTER_MINB
#define QQQ_QCLUSTER_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, QQQ_QCLUSTER_MINB) act_quant_cluster_kernel(const __half* __restrict__ x, int64_t K,
                                                                      int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                                      double* __restrict__ s_out, int32_t* status,
                                                                      int32_t* __restrict__ rowsum_out,
                                                                      const double* __restrict__ smooth,
                                                                      const double* __restrict__ recip) {
  using Acc = typename std::conditional<kSmooth, double, float>::type;
  __shared__ uint64_t bar[2];       // [0] peer maxima landed, [1] (rank 0) peer code sums landed
  __shared__ double peer_max[8];
  __shared__ int32_t peer_sum[8];
  __shared__ Acc red[32];
  __shared__ int isum[kThreads / 32];
  const uint32_t G = cluster_nctarank(), rank = cluster_ctarank();
  const int64_t row = blockIdx.x / G;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  cluster_sync_all();  // every CTA's barriers initialised before any st.async targets them
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t nv = K / 8;
  const int64_t v0 = rank * nv / G, v1 = (rank + 1) * nv / G;
  // kVPT 16-byte vectors per thread: v0 + threadIdx.x + j * kThreads (all loads first)
  uint4 v[kVPT];
  bool has[kVPT];
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int64_t i = v0 + threadIdx.x + (int64_t)j * kThreads;
    has[j] = i < v1;
    v[j] = has[j] ? __ldg(reinterpret_cast<const uint4*>(x + row * ldx) + i) : make_uint4(0, 0, 0, 0);
  }
  double xs[kSmooth ? kVPT : 1][8];
  Acc m = Acc(0);
  bool bad = false;
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int64_t i = v0 + threadIdx.x + (int64_t)j * kThreads;
    const __half* e = reinterpret_cast<const __half*>(&v[j]);
    if constexpr (kSmooth) {
      if (has[j]) {
        smooth8(v[j], smooth, recip, i, xs[j]);
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) xs[j][t] = 0.0;
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const Acc a = kSmooth ? (Acc)fabs(xs[kSmooth ? j : 0][t]) : (Acc)fabsf(__half2float(e[t]));
      bad |= is_bad(a);
      m = a > m ? a : m;
    }
  }
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) atomicOr(status, kStatNonFinite);
  }
  m = block_max<kThreads, Acc>(m, red);
  if (threadIdx.x == 0) {
    const double md = (double)m;
    peer_max[rank] = md;
    if (G > 1) {
      mbar_arrive_expect_tx(&bar[0], (G - 1) * 8);
      for (uint32_t d = 0; d < G; ++d)
        if (d != rank)
          st_async_b64(mapa_shared(&peer_max[rank], d), __double_as_longlong(md), mapa_shared(&bar[0], d));
      mbar_wait(&bar[0], 0);
    }
  }
  __syncthreads();
  Acc mr = Acc(0);
  for (uint32_t d = 0; d < G; ++d) mr = (Acc)peer_max[d] > mr ? (Acc)peer_max[d] : mr;
  const double s = (mr > Acc(0)) ? (double)mr / 127.0 : 1.0;
  const bool zero_row = !(mr > Acc(0));
  const float inv = zero_row ? 0.0f : 127.0f / (float)mr;
  const double rs = 1.0 / s;
  int csum = 0;
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    if (has[j]) {
      const int64_t i = v0 + threadIdx.x + (int64_t)j * kThreads;
      uint2 o;
      if constexpr (kSmooth)
        o = codes8_f64(xs[j], s, rs, !markstein_safe(s), csum);
      else
        o = codes8_f16(v[j], inv, s, rs, csum);
      *reinterpret_cast<uint2*>(q + row * ldq + i * 8) = o;
    }
  }
  for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  if ((threadIdx.x & 31) == 0) isum[threadIdx.x >> 5] = csum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += isum[w];
    if (rank != 0) {
      st_async_b32(mapa_shared(&peer_sum[rank], 0), (uint32_t)t, mapa_shared(&bar[1], 0));
    } else {
      if (G > 1) {
        mbar_arrive_expect_tx(&bar[1], (G - 1) * 4);
        mbar_wait(&bar[1], 0);
        for (uint32_t d = 1; d < G; ++d) t += peer_sum[d];
      }
      s_out[row] = s;
      if (rowsum_out) rowsum_out[row] = t;
    }
  }
}

// rowsum of existing int8 codes (activations built outside quant_act_per_token)
__global__ void rowsum_kernel(const int8_t* __restrict__ q, int64_t K, int64_t ldq, int32_t* __restrict__ out) {
  const int8_t* qr = q + (int64_t)blockIdx.x * ldq;
  int s = 0;
  for (int64_t i = threadIdx.x; i < K; i += blockDim.x) s += qr[i];
  __shared__ int red[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) t += red[i];
    out[blockIdx.x] = t;
  }
}

}  // namespace qqq

using namespace qqq;

static int act_quant_launch(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int8_t* q, int64_t ldq,
                            double* s_a, int32_t* status_dev, const double* row_max_in, double* row_max_out,
                            int32_t* rowsum, cudaStream_t stream, const double* smooth = nullptr,
                            const uint8_t* smooth_mask = nullptr, const double* recip = nullptr) {
  if (M < 0 || K <= 0 || ldx < K || (!row_max_out && ldq < K)) return kErrShape;
  if (M == 0) return kOk;
  constexpr int kT = 256;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)M);
  lc.blockDim = dim3(kT);
  lc.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaError_t e;
  // M <= 256 (decode and mid batches), smoothed fp16 rows up to 8 x 256 vectors: row split over
  // a cluster (measured: 4.7 vs 5.2 us per smoothed M=1 quantizer in the C4 chain; the
  // plain quantizer's ~35 instructions per element gain nothing from it)
#ifndef QQQ_QCLUSTER_CT
#define QQQ_QCLUSTER_CT 256
#endif
#ifndef QQQ_QCLUSTER_VPT
#define QQQ_QCLUSTER_VPT 1
#endif
  constexpr int kCT = QQQ_QCLUSTER_CT, kCV = QQQ_QCLUSTER_VPT;
  // The reciprocal table replaces the per-element division routine by 5 FMA-pipe
  // ops but adds a 64-byte table read per 8 channels: a win for decode batches
  // (C4 stack quantizers 16.5 -> 14.7 us at M = 1..16), a loss from M ~ 64 on
  // (33.0 -> 36.9 us at M = 256), where the kernel waits on loads, not issue.
#ifndef QQQ_RECIP_MAXM
#define QQQ_RECIP_MAXM 32
#endif
  constexpr int64_t kRecipMaxM = QQQ_RECIP_MAXM;
#ifndef QQQ_QCLUSTER_MAXM
#define QQQ_QCLUSTER_MAXM 256
#endif
  if (smooth && x_dtype == 0 && !row_max_in && !row_max_out && !smooth_mask && M <= QQQ_QCLUSTER_MAXM && K % 8 == 0 &&
      K <= (int64_t)8 * kCT * kCV * 8 && ldx % 8 == 0 && ldq % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(q) & 7) == 0 && (reinterpret_cast<uintptr_t>(smooth) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(recip) & 15) == 0) {
    const int G = (int)((K / 8 + kCT * kCV - 1) / (kCT * kCV));
    cudaLaunchAttribute ca[2];
    ca[0] = attr[0];
    ca[1].id = cudaLaunchAttributeClusterDimension;
    ca[1].val.clusterDim.x = G;
    ca[1].val.clusterDim.y = 1;
    ca[1].val.clusterDim.z = 1;
    cudaLaunchConfig_t cc = lc;
    cc.gridDim = dim3((unsigned)(M * G));
    cc.blockDim = dim3(kCT);
    cc.attrs = ca;
    cc.numAttrs = 2;
    e = cudaLaunchKernelEx(&cc, act_quant_cluster_kernel<kCT, true, kCV>, (const __half*)x, K, ldx, q, ldq, s_a,
                           status_dev, rowsum, smooth, M <= kRecipMaxM ? recip : nullptr);
    return e == cudaSuccess ? kOk : kErrCuda;
  }
  // fp16 rows that fit one CTA's registers: the single-round-trip kernel
  constexpr int kRT = 512, kRV = 4;
  if (x_dtype == 0 && !row_max_in && !row_max_out && K % 8 == 0 &&
      K <= (int64_t)kRT * kRV * 8 && ldx % 8 == 0 &&
      ldq % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(q) & 7) == 0 &&
      (reinterpret_cast<uintptr_t>(smooth) & 15) == 0 &&  // (smoothing vector read as 16-byte pairs)
      (reinterpret_cast<uintptr_t>(recip) & 15) == 0) {
    lc.blockDim = dim3(kRT);
    if (smooth)
      e = cudaLaunchKernelEx(&lc, act_quant_row_kernel<kRT, kRV, true>, (const __half*)x, K, ldx, q, ldq, s_a,
                             status_dev, rowsum, smooth, smooth_mask, M <= kRecipMaxM ? recip : nullptr);
    else
      e = cudaLaunchKernelEx(&lc, act_quant_row_kernel<kRT, kRV, false>, (const __half*)x, K, ldx, q, ldq, s_a,
                             status_dev, rowsum, smooth, smooth_mask, (const double*)nullptr);
    return e == cudaSuccess ? kOk : kErrCuda;
  }
  if (smooth) {
    if (row_max_in || row_max_out) return kErrConfig;
    switch (x_dtype) {
      case 0:
        e = cudaLaunchKernelEx(&lc, act_quant_kernel<__half, kT, true>, (const __half*)x, K, ldx, q, ldq, s_a,
                               status_dev, row_max_in, row_max_out, rowsum, smooth);
        break;
      case 1:
        e = cudaLaunchKernelEx(&lc, act_quant_kernel<float, kT, true>, (const float*)x, K, ldx, q, ldq, s_a,
                               status_dev, row_max_in, row_max_out, rowsum, smooth);
        break;
      case 2:
        e = cudaLaunchKernelEx(&lc, act_quant_kernel<double, kT, true>, (const double*)x, K, ldx, q, ldq, s_a,
                               status_dev, row_max_in, row_max_out, rowsum, smooth);
        break;
      default:
        return kErrConfig;
    }
    return e == cudaSuccess ? kOk : kErrCuda;
  }
  switch (x_dtype) {
    case 0:
      e = cudaLaunchKernelEx(&lc, act_quant_kernel<__half, kT>, (const __half*)x, K, ldx, q, ldq, s_a, status_dev,
                             row_max_in, row_max_out, rowsum, nullptr);
      break;
    case 1:
      e = cudaLaunchKernelEx(&lc, act_quant_kernel<float, kT>, (const float*)x, K, ldx, q, ldq, s_a, status_dev,
                             row_max_in, row_max_out, rowsum, nullptr);
      break;
    case 2:
      e = cudaLaunchKernelEx(&lc, act_quant_kernel<double, kT>, (const double*)x, K, ldx, q, ldq, s_a, status_dev,
                             row_max_in, row_max_out, rowsum, nullptr);
      break;
    default:
      return kErrConfig;
  }
  return e == cudaSuccess ? kOk : kErrCuda;
}

extern "C" int qqq_act_quant(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int8_t* q, int64_t ldq,
                             double* s_a, int32_t* status_dev, cudaStream_t stream) {
  return act_quant_launch(x, x_dtype, M, K, ldx, q, ldq, s_a, status_dev, nullptr, nullptr, nullptr, stream);
}

extern "C" int qqq_act_quant_ex(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, int8_t* q,
                                int64_t ldq, double* s_a, int32_t* rowsum, int32_t* status_dev, cudaStream_t stream) {
  return act_quant_launch(x, x_dtype, M, K, ldx, q, ldq, s_a, status_dev, nullptr, nullptr, rowsum, stream);
}

extern "C" int qqq_act_rowsum(const int8_t* q, int64_t M, int64_t K, int64_t ldq, int32_t* rowsum,
                              cudaStream_t stream) {
  if (M < 0 || K <= 0 || ldq < K) return kErrShape;
  if (M == 0) return kOk;
  rowsum_kernel<<<(unsigned)M, 256, 0, stream>>>(q, K, ldq, rowsum);
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

extern "C" int qqq_act_absmax(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx, double* row_max,
                              int32_t* status_dev, cudaStream_t stream) {
  return act_quant_launch(x, x_dtype, M, K, ldx, nullptr, 0, nullptr, status_dev, nullptr, row_max, nullptr, stream);
}

extern "C" int qqq_act_quant_with_max(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx,
                                      const double* row_max, int8_t* q, int64_t ldq, double* s_a, int32_t* rowsum,
                                      int32_t* status_dev, cudaStream_t stream) {
  if (!row_max) return kErrConfig;
  return act_quant_launch(x, x_dtype, M, K, ldx, q, ldq, s_a, status_dev, row_max, nullptr, rowsum, stream);
}

// apply_quant_linear's activation step (pipeline.py:146): quant_act_per_token
// of x / s, the f64 division fused into the quantizer (one pass over x).
extern "C" int qqq_act_quant_smooth(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx,
                                    const double* smooth, const uint8_t* smooth_mask, int8_t* q, int64_t ldq,
                                    double* s_a, int32_t* rowsum, int32_t* status_dev, cudaStream_t stream) {
  if (!smooth) return kErrConfig;
  return act_quant_launch(x, x_dtype, M, K, ldx, q, ldq, s_a, status_dev, nullptr, nullptr, rowsum, stream, smooth,
                          smooth_mask);
}

// Reciprocal table of a smoothing vector for qqq_act_quant_smooth_rcp:
// recip[k] = RN(1/s_k) (IEEE division), or NaN where 2^-400 <= |s_k| <= 2^400
// does not hold (those channels keep the IEEE division of x / s_k).
__global__ void smooth_recip_kernel(const double* __restrict__ smooth, int64_t K, double* __restrict__ recip) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < K) {
    const double b = smooth[k];
    recip[k] = markstein_safe(b) ? 1.0 / b : __longlong_as_double(0x7ff8000000000000LL);
  }
}

extern "C" int qqq_smooth_reciprocal(const double* smooth, int64_t K, double* recip, cudaStream_t stream) {
  if (!smooth || !recip) return kErrConfig;
  if (K <= 0) return kErrShape;
  smooth_recip_kernel<<<(unsigned)((K + 255) / 256), 256, 0, stream>>>(smooth, K, recip);
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

// qqq_act_quant_smooth with the smoothing vector's reciprocal table: the x / s_k
// divisions become Markstein FMA sequences (same IEEE quotients, bit-identical
// codes and scales), the form a layer uses once its table is cached.
extern "C" int qqq_act_quant_smooth_rcp(const void* x, int x_dtype, int64_t M, int64_t K, int64_t ldx,
                                        const double* smooth, const double* smooth_recip, int8_t* q, int64_t ldq,
                                        double* s_a, int32_t* rowsum, int32_t* status_dev, cudaStream_t stream) {
  if (!smooth || !smooth_recip) return kErrConfig;
  return act_quant_launch(x, x_dtype, M, K, ldx, q, ldq, s_a, status_dev, nullptr, nullptr, rowsum, stream, smooth,
                          nullptr, smooth_recip);
}
