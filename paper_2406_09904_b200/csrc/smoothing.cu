// Offline calibration on the GPU: the f64 products of the
// smoothing-threshold search.
//
// Reference: pkg/src/qqq/numerics.py:94-109 (matmul_ref)
//   out = 0; for k in 0..K-1: out += a[:, k] * b[k, :]
// numpy rounds each product and then each sum (no fused multiply-add), in
// sequential k order. smoothing.py:108-113 compares the quantized product with
// the exact one through this function, so reproducing its rounding sequence
// makes every candidate's error matrix bit-identical to the reference's.
//
// One CTA computes a 64 x 64 output tile, 4 x 4 outputs per thread; A and B
// k-slabs of 16 are staged through shared memory. Each output keeps its own
// sequential k order (DMUL then DADD, __dmul_rn / __dadd_rn so nvcc cannot
// contract them into DFMA). The f64 pipe bounds it: 2MNK flops at ~half the
// FP64 peak (no FMA), fine for calibration-sized matrices.
#include "qqq_common.cuh"

namespace qqq {

constexpr int kMT = 64, kNT = 64, kKT = 16;

__global__ void __launch_bounds__(256) matmul_seq_f64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                             double* __restrict__ c, int64_t M, int64_t K, int64_t N) {
  __shared__ double as[kKT][kMT + 1];
  __shared__ double bs[kKT][kNT];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.y * kMT, n0 = (int64_t)blockIdx.x * kNT;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = 0; k0 < K; k0 += kKT) {
    for (int e = threadIdx.x; e < kMT * kKT; e += 256) {
      const int mm = e / kKT, kk = e % kKT;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      as[kk][mm] = (gm < M && gk < K) ? a[gm * K + gk] : 0.0;
    }
    for (int e = threadIdx.x; e < kKT * kNT; e += 256) {
      const int kk = e / kNT, nn = e % kNT;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      bs[kk][nn] = (gk < K && gn < N) ? b[gk * N + gn] : 0.0;
    }
    __syncthreads();
    const int kn = K - k0 < kKT ? (int)(K - k0) : kKT;
    for (int kk = 0; kk < kn; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = as[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(av[i], bv[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx + 16 * j;
      if (gn < N) c[gm * N + gn] = acc[i][j];
    }
  }
}

}  // namespace qqq

using namespace qqq;

extern "C" int qqq_matmul_ref_f64(const double* a, const double* b, double* c, int64_t M, int64_t K, int64_t N,
                                  cudaStream_t stream) {
  if (M < 0 || K < 0 || N < 0) return kErrShape;
  if (M == 0 || N == 0) return kOk;
  if (!c) return kErrConfig;
  if (K == 0)  // empty sum: zeros, as numpy's np.zeros start value
    return cudaMemsetAsync(c, 0, (size_t)(M * N) * sizeof(double), stream) == cudaSuccess ? kOk : kErrCuda;
  if (!a || !b) return kErrConfig;
  if ((N + kNT - 1) / kNT > 0x7fffffff || (M + kMT - 1) / kMT > 65535) return kErrShape;
  const dim3 grid((unsigned)((N + kNT - 1) / kNT), (unsigned)((M + kMT - 1) / kMT));
  matmul_seq_f64_kernel<<<grid, 256, 0, stream>>>(a, b, c, M, K, N);
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}
