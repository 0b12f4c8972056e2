// Device helpers of the per-token activation quantizer (quantize.py:92-100,
// pipeline.py:146), shared by the standalone quantizer kernels (act_quant.cu)
// and the GEMM's fused smoothed-quantization prologue (w4a8_gemm.cu).
#pragma once
#include "qqq_common.cuh"

namespace qqq {

template <typename T>
QQQ_DEVICE double to_f64(T v);
QQQ_DEVICE float absval(__half v) { return fabsf(__half2float(v)); }
QQQ_DEVICE float absval(float v) { return fabsf(v); }
QQQ_DEVICE double absval(double v) { return fabs(v); }
QQQ_DEVICE bool is_bad(float a) { return !(a <= 3.4028234663852886e38f); }
QQQ_DEVICE bool is_bad(double a) { return !(a <= 1.7976931348623157e308); }
template <>
QQQ_DEVICE double to_f64<__half>(__half v) { return (double)__half2float(v); }
template <>
QQQ_DEVICE double to_f64<float>(float v) { return (double)v; }
template <>
QQQ_DEVICE double to_f64<double>(double v) { return v; }

QQQ_DEVICE int8_t quant_code_exact(double x, double s) {
  double r = rint(x / s);
  r = fmin(fmax(r, -127.0), 127.0);
  return (int8_t)(int)r;
}

// Same result as quant_code_exact without the f64 division on the common path:
// inv = RN(1/s); |x*inv - x/s| <= 2^-51 * 127, so rint agrees unless x/s is
// within 1e-9 of a half-integer, where the verbatim division decides.
QQQ_DEVICE int8_t quant_code_f64(double x, double inv, double s) {
  const double u = x * inv;
  const double r = rint(u);
  if (fabs(fabs(u - r) - 0.5) < 1e-9) return quant_code_exact(x, s);
  return (int8_t)(int)fmin(fmax(r, -127.0), 127.0);
}

// the smoothed activation x / s_k (pipeline.py:146, f64 IEEE division); most
// channels are not smoothed (s_k == 1.0, x / 1.0 == x exactly)
QQQ_DEVICE double smooth_div(double x, double sk) { return sk == 1.0 ? x : x / sk; }

// RN(a / b) without the division routine (Markstein): y = RN(1/b); q0 =
// RN(a*y) can be ~1.3 ulp off, so one FMA correction q1 = RN(q0 + RN(a - b*q0)*y)
// brings it within one ulp; then r1 = a - b*q1 is exact in one FMA and
// RN(q1 + r1*y) is the correctly rounded quotient (Markstein's theorem, y within
// half an ulp of 1/b), i.e. the IEEE division numpy performs. The callers keep
// |b| and the quotients inside the normal range (qqq_smooth_reciprocal). b == 1
// gives a exactly (y = 1, residuals 0). Checked in exact rational arithmetic by
// tests/test_pipeline.py::test_markstein_division_is_ieee.
QQQ_DEVICE double div_markstein(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double q1 = __fma_rn(__fma_rn(-q0, b, a), y, q0);
  return __fma_rn(__fma_rn(-q1, b, a), y, q1);
}

// 8 int8 codes (low byte of each word) -> 8 packed bytes; csum += their sum
QQQ_DEVICE uint2 pack8(const uint32_t (&b)[8], int& csum) {
  uint2 o;
  o.x = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
  o.y = __byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
  csum = __dp4a((int)o.x, 0x01010101, csum);
  csum = __dp4a((int)o.y, 0x01010101, csum);
  return o;
}

// Codes of 8 fp16 values (quantize.py:99 rint(x / s), clip): t = x * RN(127/m)
// in fp32, rounded half-even by adding 1.5*2^23 (the code is then the low byte
// of the sum's bits; |t| <= 127 < 2^22). One batched test per 8 values: if any
// t lies within 2^-14 of a half-integer, all 8 take the reference formula in
// f64. The band: inv = 127/m (1 + d1), t = x*inv (1 + d2), |d1|, |d2| <= 2^-24,
// so |t - x*127/m| <= 127 * 2.01 * 2^-24 < 1.6e-5 < 2^-14 = 6.1e-5 (and the
// reference quotient is within 2^-44 of x*127/m). A wider band (1e-3, as in
// quant_code_f16) sent ~40% of the warps of a K=11008 row into the f64 path.
QQQ_DEVICE uint2 codes8_f16(const uint4& v, float inv, double s, double rs, int& csum) {
  constexpr float kMagic = 12582912.0f;
  const __half* e = reinterpret_cast<const __half*>(&v);
  uint32_t b[8];
  float emax = 0.0f;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const float tt = __fmul_rn(__half2float(e[t]), inv);
    const float w = __fadd_rn(tt, kMagic);
    emax = fmaxf(emax, fabsf(__fsub_rn(tt, __fsub_rn(w, kMagic))));
    b[t] = __float_as_uint(w);
  }
  if (emax > 0.5f - 0x1p-14f) {
#pragma unroll
    for (int t = 0; t < 8; ++t)  // rint(RN(x / s)) exactly (s = m/127 with m an fp16 value: Markstein-safe)
      b[t] = (uint32_t)__double2loint(__dadd_rn(div_markstein((double)__half2float(e[t]), s, rs), 6755399441055744.0));
  }
  return pack8(b, csum);
}

// Codes of 8 smoothed f64 values: u = RN(x / s) by Markstein (rs = RN(1/s)),
// rint(u) half-even by adding 1.5*2^52 (|u| <= 127, no clip needed since
// |x| <= m). Bit-identical to the reference, no near-tie fallback. `ieee`:
// s outside the range where the FMA residual stays normal -> IEEE division.
QQQ_DEVICE uint2 codes8_f64(const double (&xs)[8], double s, double rs, bool ieee, int& csum) {
  constexpr double kMagic = 6755399441055744.0;
  uint32_t b[8];
  if (ieee) {
#pragma unroll
    for (int t = 0; t < 8; ++t) b[t] = (uint32_t)(int)quant_code_exact(xs[t], s);
  } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) b[t] = (uint32_t)__double2loint(__dadd_rn(div_markstein(xs[t], s, rs), kMagic));
  }
  return pack8(b, csum);
}

// x / s_k for the 8 channels of one vector (pipeline.py:146): with the
// reciprocal table y (qqq_smooth_reciprocal; NaN marks a channel whose s_k is
// outside the safe range) by Markstein, else IEEE division
QQQ_DEVICE void smooth8(const uint4& v, const double* __restrict__ smooth, const double* __restrict__ recip,
                        int64_t i, double (&xs)[8]) {
  const __half* e = reinterpret_cast<const __half*>(&v);
  const double2* sv = reinterpret_cast<const double2*>(smooth + i * 8);
  double sk[8];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const double2 d = __ldg(sv + h);
    sk[2 * h] = d.x;
    sk[2 * h + 1] = d.y;
  }
  bool slow = recip == nullptr;
  if (!slow) {
    const double2* yv = reinterpret_cast<const double2*>(recip + i * 8);
    double y[8];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double2 d = __ldg(yv + h);
      y[2 * h] = d.x;
      y[2 * h + 1] = d.y;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      xs[t] = div_markstein((double)__half2float(e[t]), sk[t], y[t]);
      slow |= y[t] != y[t];
    }
  }
  if (slow) {
#pragma unroll
    for (int t = 0; t < 8; ++t) xs[t] = (double)__half2float(e[t]) / sk[t];
  }
}

// Markstein is exact while the quotients and FMA residuals stay normal
QQQ_DEVICE bool markstein_safe(double b) { return fabs(b) >= 0x1p-400 && fabs(b) <= 0x1p400; }

// fp16 fast path; inv = RN(127/m) in fp32 (m = row absmax > 0), s the f64
// scale. |x*inv - x*127/m| <= 2*127*2^-24 < 2e-5, far inside the 1e-3 band.
QQQ_DEVICE int8_t quant_code_f16(float x, float inv, double s) {
  float t = x * inv;
  float r = rintf(t);
  float d = fabsf(fabsf(t - r) - 0.5f);
  if (d < 1e-3f) return quant_code_exact((double)x, s);
  r = fminf(fmaxf(r, -127.0f), 127.0f);
  return (int8_t)(int)r;
}

}  // namespace qqq
