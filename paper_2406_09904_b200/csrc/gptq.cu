// Offline calibration on the GPU: the GPTQ column sweep.
//
// Reference: pkg/src/qqq/gptq.py:161-183 (gptq_sweep, inner loop of one block)
//   for i in [i1, i2):                       (j = i - i1)
//     per-group, i % g == 0: scale_row = max|wb[j:j+g, :]| / 7 (1.0 if 0) -> s_wg[i/g]
//     q = clip(rint(wb[j] / scale_row), -8, 7); deq = q * scale_row
//     err = (wb[j] - deq) / U[i, i]
//     wb[j+1:, :] -= outer(U[i, i+1:i2], err);  eb[j] = err
// Every output column n is independent (the scale, the code, the error and the
// rank-1 update of column n touch column n only), so one thread owns one
// column and runs the block's i loop sequentially; the CTA stages its 32
// columns x B rows of the block in shared memory. The operations and their
// rounding sequence are numpy's (IEEE division, product then difference, no
// FMA), so one block is bit-identical to the reference. The trailing update
// work[i2:] -= U[i1:i2, i2:]^T @ eb is a BLAS product in both implementations
// (gptq.py:182-183), done by the host between blocks.
#include <cstdint>

#include "qqq_common.cuh"

namespace qqq {

constexpr int kGCols = 32;

// kSmem: the block's rows of the CTA's columns live in shared memory (blocks of
// up to 800 rows); larger blocks update `work` in place in global memory
// (coalesced: consecutive threads own consecutive columns).
template <bool kSmem>
__global__ void __launch_bounds__(kGCols) gptq_block_kernel(double* __restrict__ work, int64_t N,
                                                            const double* __restrict__ u, int64_t K, int64_t i1,
                                                            int64_t i2, int64_t gs, double* __restrict__ scale_row,
                                                            double* __restrict__ s_wg, int8_t* __restrict__ codes,
                                                            double* __restrict__ eb) {
  extern __shared__ double smem_wb[];  // [B][kGCols]
  const int64_t B = i2 - i1;
  const int t = threadIdx.x;
  const int64_t n = (int64_t)blockIdx.x * kGCols + t;
  const bool valid = n < N;
  if (!kSmem && !valid) return;  // (global mode: no block-wide barrier below)
  double* const wb = kSmem ? smem_wb : work + i1 * N + n - t;  // wb[r * ld + t]
  const int64_t ld = kSmem ? kGCols : N;
  if (kSmem)
    for (int64_t r = 0; r < B; ++r) wb[r * ld + t] = valid ? work[(i1 + r) * N + n] : 0.0;
  double scale = (valid && gs == 0) ? scale_row[n] : 1.0;
  for (int64_t j = 0; j < B; ++j) {
    const int64_t i = i1 + j;
    if (gs > 0 && i % gs == 0) {  // group boundary: scale from the compensated rows of the group
      double gm = 0.0;
      for (int64_t r = j; r < j + gs && r < B; ++r) gm = fmax(gm, fabs(wb[r * ld + t]));
      scale = gm > 0.0 ? gm / 7.0 : 1.0;
      if (valid) s_wg[(i / gs) * N + n] = scale;
    }
    const double row = wb[j * ld + t];
    const double q = fmin(fmax(rint(row / scale), -8.0), 7.0);
    const double deq = __dmul_rn(q, scale);
    const double err = __dsub_rn(row, deq) / u[i * K + i];
    if (valid) {
      codes[i * N + n] = (int8_t)(int)q;
      eb[j * N + n] = err;
    }
    const double* ur = u + i * K + i1;  // U[i, i1 + r]
    for (int64_t r = j + 1; r < B; ++r) wb[r * ld + t] = __dsub_rn(wb[r * ld + t], __dmul_rn(ur[r], err));
  }
  if (kSmem && valid)  // the block's compensated rows (gptq.py:181: work[i1:i2] = wb)
    for (int64_t r = 0; r < B; ++r) work[(i1 + r) * N + n] = wb[r * ld + t];
}

}  // namespace qqq

using namespace qqq;

extern "C" int qqq_gptq_block(double* work, int64_t K, int64_t N, const double* u, int64_t i1, int64_t i2, int64_t gs,
                              double* scale_row, double* s_wg, int8_t* codes, double* eb, cudaStream_t stream) {
  if (K <= 0 || N <= 0 || i1 < 0 || i2 <= i1 || i2 > K) return kErrShape;
  if (!work || !u || !codes || !eb || (gs == 0 && !scale_row) || (gs > 0 && !s_wg)) return kErrConfig;
  if (gs < 0 || (gs > 0 && (i1 % gs != 0 || (i2 - i1) % gs != 0))) return kErrConfig;
  const size_t smem = (size_t)(i2 - i1) * kGCols * sizeof(double);
  const unsigned grid = (unsigned)((N + kGCols - 1) / kGCols);
  if (smem > 200 * 1024) {
    gptq_block_kernel<false><<<grid, kGCols, 0, stream>>>(work, N, u, K, i1, i2, gs, scale_row, s_wg, codes, eb);
  } else {
    if (smem > 48 * 1024 && cudaFuncSetAttribute(gptq_block_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem) != cudaSuccess)
      return kErrCuda;
    gptq_block_kernel<true><<<grid, kGCols, smem, stream>>>(work, N, u, K, i1, i2, gs, scale_row, s_wg, codes, eb);
  }
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}
