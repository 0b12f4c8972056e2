// Dense INT8 tensor-core peak of this GPU, measured (diagnostics for bench.py's
// roofline): every SM issues back-to-back tcgen05.mma.cta_group::1.kind::i8
// M=128 N=256 K=32 from shared memory into two TMEM accumulators (the largest
// single-CTA UMMA shape, the one the GEMM's prefill tiles use), with no memory
// traffic. ops = grid * iters * 2*128*256*32; the caller times the launch with
// CUDA events at the clocks it records.
#include "qqq_common.cuh"

namespace qqq {

__global__ void __launch_bounds__(128, 1) int8_peak_kernel(int iters) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    constexpr uint32_t idesc = make_idesc_i8(128, 256, false);
    // operands: whatever the shared memory holds (throughput does not depend on values)
    const uint64_t a_desc = make_smem_desc(smem_u32(smem), 16, 1024, 2);          // 128 rows x 32 B
    const uint64_t b_desc = make_smem_desc(smem_u32(smem + 16384), 16, 1024, 2);  // 256 rows x 32 B
#pragma unroll 1
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (elect_one())
          mma_i8_ss(tbase + (uint32_t)((j & 1) * 256), a_desc + (uint64_t)(j & 3) * 2, b_desc + (uint64_t)(j & 3) * 2,
                    idesc, (i + j) >= 2 ? 1u : 0u);
        __syncwarp();
      }
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace qqq

using namespace qqq;

extern "C" int qqq_probe_int8_peak(int grid, int iters, double* ops_out, cudaStream_t stream) {
  if (grid <= 0 || iters <= 0 || (iters % 8) != 0) return kErrConfig;
  constexpr int kSmem = 48 * 1024 + 1024;
  if (cudaFuncSetAttribute(int8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess)
    return kErrCuda;
  int8_peak_kernel<<<grid, 128, kSmem, stream>>>(iters);
  if (ops_out) *ops_out = (double)grid * iters * 2.0 * 128 * 256 * 32;
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}
