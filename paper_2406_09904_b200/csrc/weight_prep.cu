// Offline weight preparation on the GPU (the "weight packing" half of the
// drop-in API) plus the one-time repack into the tcgen05 kernel layout.
//
// Reference (pkg/src/qqq/quantize.py, gemm.py):
//   quant_weight_per_channel  quantize.py:103-123   s = max|col|/7 (or 1), q = clip(rint(w/s), -8, 7)
//   quant_weight_per_group    quantize.py:126-149   per (group, col) scale, then requant_scale
//   requant_scale             quantize.py:152-168   s_wc = max_k |f16(q*s_wg)| / 127 (or 1)
//   pack_i4 / unpack_i4       quantize.py:171-208   byte(k2,n) = u[2k2,n] | u[2k2+1,n] << 4, u = q+8
//   dequantize_ref            quantize.py:211-217
//   FusedScales.from_quantized gemm.py:61-69        s* = f16(s_wg / s_wc) (ConfigError on overflow)
// All arithmetic is IEEE f64 with half-even rint and a single RN rounding to
// binary16 (cvt.rn.f16.f64), matching numpy bit for bit.
#include "qqq_common.cuh"
#include "qqq_layout.cuh"

namespace qqq {

QQQ_DEVICE uint16_t f64_to_f16_bits(double v) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(v));
  return h;
}
QQQ_DEVICE double f16_bits_to_f64(uint16_t b) { return (double)__half2float(__ushort_as_half(b)); }

QQQ_DEVICE bool finite64(double v) { return fabs(v) <= 1.7976931348623157e308; }

// One thread per (group, column): scale = max|w|/7 over the group's rows.
__global__ void quant_w_kernel(const double* __restrict__ w, int64_t K, int64_t N, int64_t gs, int8_t* __restrict__ codes,
                               double* __restrict__ scales, int32_t* status) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t g = blockIdx.y;
  if (n >= N) return;
  const int64_t k0 = g * gs;
  double m = 0.0;
  bool bad = false;
  for (int64_t k = k0; k < k0 + gs; ++k) {
    double a = fabs(w[k * N + n]);
    bad |= !finite64(a);
    m = fmax(m, a);
  }
  if (bad) atomicOr(status, kStatNonFinite);
  const double s = (m > 0.0) ? m / 7.0 : 1.0;
  scales[g * N + n] = s;
  for (int64_t k = k0; k < k0 + gs; ++k) {
    double r = rint(w[k * N + n] / s);
    r = fmin(fmax(r, -8.0), 7.0);
    codes[k * N + n] = (int8_t)(int)r;
  }
}

// Per-channel scales (quantize.py:111-123) for tall groups: the column max is
// split over kRqRows thread rows (coalesced loads) and reduced in shared
// memory, then codes are produced one element per thread (quant_codes_kernel).
constexpr int kRqRows = 8;
__global__ void __launch_bounds__(32 * kRqRows) colmax_scale_kernel(const double* __restrict__ w, int64_t K, int64_t N,
                                                                    double* __restrict__ scales, int32_t* status) {
  __shared__ double red[kRqRows][32];
  __shared__ int bad_s;
  if (threadIdx.x == 0 && threadIdx.y == 0) bad_s = 0;
  __syncthreads();
  const int64_t n = blockIdx.x * 32 + threadIdx.x;
  double m = 0.0;
  bool bad = false;
  if (n < N) {
    for (int64_t k = threadIdx.y; k < K; k += kRqRows) {
      const double a = fabs(w[k * N + n]);
      bad |= !finite64(a);
      m = fmax(m, a);
    }
  }
  if (bad) bad_s = 1;
  red[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
#pragma unroll
    for (int r = 1; r < kRqRows; ++r) m = fmax(m, red[r][threadIdx.x]);
    scales[n] = (m > 0.0) ? m / 7.0 : 1.0;
  }
  if (threadIdx.x == 0 && threadIdx.y == 0 && bad_s) atomicOr(status, kStatNonFinite);
}

__global__ void quant_codes_kernel(const double* __restrict__ w, int64_t K, int64_t N, const double* __restrict__ scales,
                                   int8_t* __restrict__ codes) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= K * N) return;
  double r = rint(w[idx] / scales[idx % N]);
  r = fmin(fmax(r, -8.0), 7.0);
  codes[idx] = (int8_t)(int)r;
}

// s_wc[n] = max_k |f16(q[k,n] * s_wg[k/gs, n])| / 127, or 1.0 (quantize.py:152-168)
// Block = 32 columns x kRows k-lanes: the K loop is split over kRows rows of
// threads (coalesced 32-byte code loads per warp) and max-reduced in shared
// memory (max is exact and order-free). Was one thread per column (2.4 ms per
// 4096x4096 matrix on a quarter of the SMs).
__global__ void __launch_bounds__(32 * kRqRows) requant_kernel(const int8_t* __restrict__ codes,
                                                               const double* __restrict__ s_wg, int64_t K, int64_t N,
                                                               int64_t gs, double* __restrict__ s_wc) {
  __shared__ double red[kRqRows][32];
  const int64_t n = blockIdx.x * 32 + threadIdx.x;
  double m = 0.0;
  if (n < N) {
    for (int64_t k = threadIdx.y; k < K; k += kRqRows) {
      const double prod = (double)codes[k * N + n] * s_wg[(k / gs) * N + n];
      const double d = f16_bits_to_f64(f64_to_f16_bits(prod));
      m = fmax(m, fabs(d));
    }
  }
  red[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
#pragma unroll
    for (int r = 1; r < kRqRows; ++r) m = fmax(m, red[r][threadIdx.x]);
    s_wc[n] = (m > 0.0) ? m / 127.0 : 1.0;
  }
}

__global__ void pack_kernel(const int8_t* __restrict__ codes, int64_t K, int64_t N, uint8_t* __restrict__ packed,
                            int32_t* status) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t K2 = (K + 1) / 2;
  if (idx >= K2 * N) return;
  const int64_t k2 = idx / N, n = idx % N;
  const int q0 = codes[(2 * k2) * N + n];
  const int q1 = (2 * k2 + 1 < K) ? codes[(2 * k2 + 1) * N + n] : 0;
  if (q0 < -8 || q0 > 7 || q1 < -8 || q1 > 7) atomicOr(status, kStatCodeRange);
  packed[idx] = (uint8_t)(((q0 + 8) & 0xF) | (((q1 + 8) & 0xF) << 4));
}

__global__ void unpack_kernel(const uint8_t* __restrict__ packed, int64_t rows, int64_t N, int8_t* __restrict__ codes,
                              int32_t* status) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t K2 = (rows + 1) / 2;
  if (idx >= K2 * N) return;
  const int64_t k2 = idx / N, n = idx % N;
  const uint8_t b = packed[idx];
  codes[(2 * k2) * N + n] = (int8_t)((int)(b & 0xF) - 8);
  if (2 * k2 + 1 < rows) {
    codes[(2 * k2 + 1) * N + n] = (int8_t)((int)(b >> 4) - 8);
  } else if ((b >> 4) != 8) {
    atomicOr(status, kStatPadNibble);
  }
}

__global__ void fused_scales_kernel(const double* __restrict__ s_wg, const double* __restrict__ s_wc, int64_t G,
                                    int64_t N, uint16_t* __restrict__ s_star, int32_t* status) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= G * N) return;
  const uint16_t h = f64_to_f16_bits(s_wg[idx] / s_wc[idx % N]);
  if ((h & 0x7C00) == 0x7C00) atomicOr(status, kStatScaleInf);
  s_star[idx] = h;
}

__global__ void dequant_kernel(const int8_t* __restrict__ codes, int64_t K, int64_t N, int64_t gs,
                               const double* __restrict__ scales, double* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= K * N) return;
  const int64_t k = idx / N, n = idx % N;
  const double s = gs > 0 ? scales[(k / gs) * N + n] : scales[n];
  out[idx] = (double)codes[idx] * s;
}

// --- repack into the tcgen05 kernel layout (qqq_layout.cuh) -----------------

QQQ_DEVICE int ref_nibble(const uint8_t* packed, int64_t K, int64_t N, int64_t k, int64_t n) {
  if (k >= K || n >= N) return 8;  // zero code
  const uint8_t b = packed[(k >> 1) * N + n];
  return (k & 1) ? (b >> 4) : (b & 0xF);
}

// One thread per (n_pad, slab): 32 nibbles of one channel -> 16 B of the PC/PG blob.
__global__ void repack4_kernel(const uint8_t* __restrict__ packed, int64_t K, int64_t N, int64_t N_pad, int64_t slabs,
                               int mode, int64_t ssb, uint8_t* __restrict__ out) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t slab = blockIdx.y;
  if (n >= N_pad) return;
  int u[32];
  // Padding k >= K: per-channel/I8 use the zero code (signed MMA). Per-group runs
  // the MMA on u8 = w8 + 128, so padding must be u8 0: code q = -8 with the
  // padding scale s* = 16 gives RN(-8*16 + 1152) = 1024 -> byte 0 exactly.
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int64_t k = slab * 32 + e;
    u[e] = (mode == kModePG && k >= K) ? 0 : ref_nibble(packed, K, N, k, n);
  }
  uint32_t wd[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t v = 0;
    if (mode == kModePC) {
#pragma unroll
      for (int j = 0; j < 4; ++j) v |= (uint32_t)(u[4 * i + j] | (u[16 + 4 * i + j] << 4)) << (8 * j);
    } else {
#pragma unroll
      for (int pp = 0; pp < 8; ++pp) v |= (uint32_t)u[8 * i + 2 * (pp % 4) + pp / 4] << (4 * pp);
    }
    wd[i] = v;
  }
  const int64_t n_tile = n / kTileN, row = n % kTileN;
  const int64_t ss = (n_tile * (slabs / 4) + slab / 4);
  uint4* dst = reinterpret_cast<uint4*>(out + ss * ssb + ((slab % 4) * kTileN + row) * 16);
  *dst = make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

// One thread per (n_pad, super-slab, local group): the s* of that group chunk
// into the PG blob, plus the fast-path admissibility test. The HFMA2 converter
// omits the reference's clamp (gemm.py:123-127); that is exact iff every code q
// present gives RN(q*s* + 1152) in [1025, 1279], and by monotonicity in q it
// suffices to test the chunk's min and max code. Weights from requant_scale
// always pass (test_gemm.py:273-280). A tiny s* is harmless: |q*s*| < 1/2, so
// both RN(q*s* + 1152) and the s*/16 form give exactly 1152.
__global__ void repack_scales_kernel(const uint16_t* __restrict__ s_star, const uint8_t* __restrict__ packed,
                                     int64_t K, int64_t N, int64_t N_pad, int64_t group, int64_t ssb,
                                     int64_t ss_per_tile, uint8_t* __restrict__ out, int32_t* flags) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int ngs = pg_groups_per_ss(group);
  const int64_t ss = blockIdx.y / ngs;
  const int gl = blockIdx.y % ngs;
  if (n >= N_pad) return;
  const int64_t geff = group < 128 ? group : 128;
  const int64_t k0 = ss * 128 + gl * geff;  // first k of this chunk
  uint16_t h = k0 >= K ? (uint16_t)0x4C00 : (uint16_t)0;  // K padding: s* = 16 (see repack4_kernel)
  if (k0 < K && n < N) {
    h = s_star[(k0 / group) * N + n];
    int qmin = 7, qmax = -8;
    for (int64_t k = k0; k < k0 + geff && k < K; ++k) {
      const int q = ref_nibble(packed, K, N, k, n) - 8;
      qmin = min(qmin, q);
      qmax = max(qmax, q);
    }
    const __half s = __ushort_as_half(h);
    const __half add = __float2half_rn(1152.0f);
    const float r_a = __half2float(__hfma(__int2half_rn(qmin), s, add));
    const float r_b = __half2float(__hfma(__int2half_rn(qmax), s, add));
    const float lo = fminf(r_a, r_b), hi = fmaxf(r_a, r_b);
    if (!(lo >= 1025.0f && hi <= 1279.0f)) atomicOr(flags, kStatNeedClamp);  // NaN fails too
  }
  const int64_t n_tile = n / kTileN, row = n % kTileN;
  uint16_t* dst = reinterpret_cast<uint16_t*>(out + (n_tile * ss_per_tile + ss) * ssb + 8192);
  dst[gl * kTileN + row] = h;
}

// One thread per (n_pad, slab, chunk): 16 int8 of the I8 blob. src is either
// a K x N int8 matrix (w8) or the reference packed bytes + s* (per-group,
// exact scalar FusedDequantQuant including the reference's clamp).
__global__ void repack8_kernel(const int8_t* __restrict__ w8, const uint8_t* __restrict__ packed,
                               const uint16_t* __restrict__ s_star, int64_t group, int64_t K, int64_t N, int64_t N_pad,
                               int64_t slabs, uint8_t* __restrict__ out) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t slab = blockIdx.y / 2, chunk = blockIdx.y % 2;
  if (n >= N_pad) return;
  alignas(16) int8_t v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int64_t k = slab * 32 + chunk * 16 + e;
    int8_t r = 0;
    if (k < K && n < N) {
      if (w8) {
        r = w8[k * N + n];
      } else {
        const int q = ref_nibble(packed, K, N, k, n) - 8;
        r = fused_dequant_quant_scalar(q, __ushort_as_half(s_star[(k / group) * N + n]));
      }
    }
    v[e] = r;
  }
  const int64_t n_tile = n / kTileN, row = n % kTileN;
  // I8 blob: per tile, consecutive slabs of [2 chunks][128 rows][16 B] (== [k16 chunk][row][16 B])
  *reinterpret_cast<uint4*>(out + (((n_tile * slabs + slab) * 2 + chunk) * kTileN + row) * 16) =
      *reinterpret_cast<const uint4*>(v);
}

// y = f16((acc * s_a[t]) * s_col[n]) in f64 (gemm.py:182-184 / 200-202): the
// epilogue applied after an exact int32 all-reduce of K-split partials.
__global__ void dequant_epilogue_kernel(const int32_t* __restrict__ acc, int64_t M, int64_t N, int64_t ldacc,
                                        const double* __restrict__ s_a, const double* __restrict__ s_col,
                                        uint16_t* __restrict__ y, int64_t ldy) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const int64_t t = idx / N, n = idx % N;
  y[t * ldy + n] = f64_to_f16_bits(((double)acc[t * ldacc + n] * s_a[t]) * s_col[n]);
}

// --- exhaustive-test hooks for the device conversion functions --------------

__global__ void fdq_scalar_kernel(const int8_t* q, const uint16_t* s, int8_t* out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fused_dequant_quant_scalar(q[i], __ushort_as_half(s[i]));
}

// 8 codes sharing one s* per word: exercises exactly the GEMM's converter path.
__global__ void fdq_word_kernel(const int8_t* q, const uint16_t* s, int8_t* out, int64_t nwords) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nwords) return;
  uint32_t w = 0;
  for (int pp = 0; pp < 8; ++pp) w |= (uint32_t)((q[8 * i + 2 * (pp % 4) + pp / 4] + 8) & 0xF) << (4 * pp);
  const __half s1 = __ushort_as_half(s[i]);
  const __half2 s2 = __halves2half2(s1, s1);
  const __half2 s16 = __hmul2(s2, u32_as_h2(0x2C002C00u));
  uint32_t lo, hi;
  pg_convert_word<false>(w, s2, s16, 0x64006400u, lo, hi);
  reinterpret_cast<uint32_t*>(out)[2 * i] = lo;
  reinterpret_cast<uint32_t*>(out)[2 * i + 1] = hi;
}

__global__ void pc_word_kernel(const int8_t* q, int8_t* out, int64_t nwords) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nwords) return;
  // word i holds k = 4j (low nibble of byte j) and k = 4 + j (high nibble) of its 8 codes
  uint32_t w = 0;
  for (int j = 0; j < 4; ++j) w |= (uint32_t)(((q[8 * i + j] + 8) & 0xF) | (((q[8 * i + 4 + j] + 8) & 0xF) << 4)) << (8 * j);
  uint32_t lo, hi;
  pc_convert_word(w, lo, hi);
  reinterpret_cast<uint32_t*>(out)[2 * i] = lo;
  reinterpret_cast<uint32_t*>(out)[2 * i + 1] = hi;
}

__global__ void f16_to_i8_kernel(const uint16_t* bits, int8_t* out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fast_f16_to_i8(__ushort_as_half(bits[i]));
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
static inline int ok() { return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda; }

}  // namespace qqq

using namespace qqq;

extern "C" int qqq_quant_weight(const double* w, int64_t K, int64_t N, int64_t group, int8_t* codes, double* scales,
                                int32_t* status_dev, cudaStream_t st) {
  if (K <= 0 || N <= 0) return kErrShape;
  const int64_t gs = group > 0 ? group : K;
  if (K % gs != 0) return kErrConfig;
  if (gs > 256) {  // tall groups (per-channel): split the column max over K, then one thread per code
    colmax_scale_kernel<<<(unsigned)((N + 31) / 32), dim3(32, kRqRows), 0, st>>>(w, K, N, scales, status_dev);
    quant_codes_kernel<<<nblk(K * N, 256), 256, 0, st>>>(w, K, N, scales, codes);
    return ok();
  }
  dim3 grid(nblk(N, 128), (unsigned)(K / gs));
  quant_w_kernel<<<grid, 128, 0, st>>>(w, K, N, gs, codes, scales, status_dev);
  return ok();
}

extern "C" int qqq_requant_scale(const int8_t* codes, const double* s_wg, int64_t K, int64_t N, int64_t G,
                                 double* s_wc, cudaStream_t st) {
  if (K <= 0 || N <= 0 || G <= 0) return kErrShape;
  if (K % G != 0) return kErrShape;  // quantize.py:165-166
  requant_kernel<<<(unsigned)((N + 31) / 32), dim3(32, kRqRows), 0, st>>>(codes, s_wg, K, N, K / G, s_wc);
  return ok();
}

extern "C" int qqq_pack_i4(const int8_t* codes, int64_t K, int64_t N, uint8_t* packed, int32_t* status_dev,
                           cudaStream_t st) {
  if (K <= 0 || N <= 0) return kErrShape;
  pack_kernel<<<nblk(((K + 1) / 2) * N, 256), 256, 0, st>>>(codes, K, N, packed, status_dev);
  return ok();
}

extern "C" int qqq_unpack_i4(const uint8_t* packed, int64_t rows, int64_t N, int8_t* codes, int32_t* status_dev,
                             cudaStream_t st) {
  if (rows <= 0 || N <= 0) return kErrShape;
  unpack_kernel<<<nblk(((rows + 1) / 2) * N, 256), 256, 0, st>>>(packed, rows, N, codes, status_dev);
  return ok();
}

extern "C" int qqq_fused_scales_pg(const double* s_wg, const double* s_wc, int64_t G, int64_t N, uint16_t* s_star,
                                   int32_t* status_dev, cudaStream_t st) {
  if (G <= 0 || N <= 0) return kErrShape;
  fused_scales_kernel<<<nblk(G * N, 256), 256, 0, st>>>(s_wg, s_wc, G, N, s_star, status_dev);
  return ok();
}

extern "C" int qqq_dequantize(const int8_t* codes, int64_t K, int64_t N, int64_t group, const double* scales,
                              double* out, cudaStream_t st) {
  if (K <= 0 || N <= 0) return kErrShape;
  dequant_kernel<<<nblk(K * N, 256), 256, 0, st>>>(codes, K, N, group, scales, out);
  return ok();
}

extern "C" size_t qqq_repacked_weight_bytes(int mode, int64_t K, int64_t N, int64_t group) {
  if (K <= 0 || N <= 0) return 0;
  if (mode == kModePG && !pg_group_ok(group)) return 0;
  const int64_t kp = round_up(K, kKPadTo), np = round_up(N, kTileN);
  return (size_t)((np / kTileN) * (kp / kSuperK) * ss_bytes(mode, group));
}

// PC / PG blob from the reference pack_i4 bytes (+ s* for PG). For PG,
// flags_dev gets QQQ_STAT_NEED_CLAMP if the clamp-free converter would not be
// bit-exact for these weights (the caller then uses the I8 blob instead).
extern "C" int qqq_repack_weights(const uint8_t* packed, const uint16_t* s_star, int64_t K, int64_t N, int mode,
                                  int64_t group, void* out, int32_t* flags_dev, cudaStream_t st) {
  if (K <= 0 || N <= 0) return kErrShape;
  if (mode != kModePC && mode != kModePG) return kErrConfig;
  if (mode == kModePG && (!pg_group_ok(group) || !s_star || !flags_dev || K % group != 0)) return kErrConfig;
  const int64_t np = round_up(N, kTileN), kp = round_up(K, kKPadTo);
  const int64_t slabs = kp / kSlabK, sspt = kp / kSuperK;
  const int64_t ssb = ss_bytes(mode, group);
  dim3 grid(nblk(np, 128), (unsigned)slabs);
  repack4_kernel<<<grid, 128, 0, st>>>(packed, K, N, np, slabs, mode, ssb, (uint8_t*)out);
  if (mode == kModePG) {
    dim3 g2(nblk(np, 128), (unsigned)(sspt * pg_groups_per_ss(group)));
    repack_scales_kernel<<<g2, 128, 0, st>>>(s_star, packed, K, N, np, group, ssb, sspt, (uint8_t*)out, flags_dev);
  }
  return ok();
}

// I8 blob from an int8 K x N matrix (w8 != NULL) or from packed + s* (per-group,
// exact scalar conversion incl. the clamp).
extern "C" int qqq_repack_weights_i8(const int8_t* w8, const uint8_t* packed, const uint16_t* s_star, int64_t group,
                                     int64_t K, int64_t N, void* out, cudaStream_t st) {
  if (K <= 0 || N <= 0) return kErrShape;
  if (!w8 && (!packed || !s_star || group <= 0)) return kErrConfig;
  const int64_t np = round_up(N, kTileN), slabs = round_up(K, kKPadTo) / kSlabK;
  dim3 grid(nblk(np, 128), (unsigned)(slabs * 2));
  repack8_kernel<<<grid, 128, 0, st>>>(w8, packed, s_star, group, K, N, np, slabs, (uint8_t*)out);
  return ok();
}

extern "C" int qqq_test_fused_dequant_quant(const int8_t* q, const uint16_t* s_star, int8_t* out, int64_t n,
                                            int word_path, cudaStream_t st) {
  if (n <= 0) return kErrShape;
  if (word_path) {
    if (n % 8) return kErrShape;
    fdq_word_kernel<<<nblk(n / 8, 256), 256, 0, st>>>(q, s_star, out, n / 8);
  } else {
    fdq_scalar_kernel<<<nblk(n, 256), 256, 0, st>>>(q, s_star, out, n);
  }
  return ok();
}

extern "C" int qqq_test_pc_convert(const int8_t* q, int8_t* out, int64_t n, cudaStream_t st) {
  if (n <= 0 || n % 8) return kErrShape;
  pc_word_kernel<<<nblk(n / 8, 256), 256, 0, st>>>(q, out, n / 8);
  return ok();
}

extern "C" int qqq_test_fast_f16_to_i8(const uint16_t* bits, int8_t* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return kErrShape;
  f16_to_i8_kernel<<<nblk(n, 256), 256, 0, st>>>(bits, out, n);
  return ok();
}

extern "C" int qqq_dequant_epilogue(const int32_t* acc, int64_t M, int64_t N, int64_t ldacc, const double* s_a,
                                    const double* s_col, void* y, int64_t ldy, cudaStream_t st) {
  if (M < 0 || N <= 0 || ldacc < N || ldy < N) return kErrShape;
  if (M == 0) return kOk;
  dequant_epilogue_kernel<<<nblk(M * N, 256), 256, 0, st>>>(acc, M, N, ldacc, s_a, s_col, (uint16_t*)y, ldy);
  return ok();
}

extern "C" int qqq_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kErrCuda;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? kOk : kErrUnsupported;
}

extern "C" const char* qqq_version(void) { return "qqq-b200 0.1.0 sm_100a"; }
