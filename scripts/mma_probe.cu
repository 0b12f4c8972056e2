// tcgen05 kind::i8 issue-rate probe (developer tool, not part of the library):
// cycles per MMA for M=128, N in {16..256}, K=32, A from TMEM (ts) or shared
// memory (ss), accumulating into 1..8 independent TMEM accumulators round-robin.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2406_09904_b200/csrc \
//        -o scripts/mma_probe scripts/mma_probe.cu
#include <cstdio>

#include "qqq_common.cuh"

using namespace qqq;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(int iters, int nacc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
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
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_i8(128, N, false);
    const uint32_t a_tmem = tbase + 256;  // A: 8 columns per K=32 step (cols 256..263)
    const uint32_t b_addr = smem_u32(smem);
    const uint64_t b_desc = make_smem_desc(b_addr, 16, 1024, 2);
    const uint64_t a_desc = make_smem_desc(smem_u32(smem + 65536), 2048, 128, 0);
    const int acc_cols = N;  // accumulators at 0, N, 2N, ... (< 256 columns)
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tbase + (uint32_t)((i % nacc) * acc_cols);
      if (TS)
        mma_i8_ts(d, a_tmem, b_desc, idesc, i >= nacc ? 1u : 0u);
      else
        mma_i8_ss(d, a_desc, b_desc, idesc, i >= nacc ? 1u : 0u);
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = (unsigned long long)(t2 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// warp-converged issue (whole warp runs the loop, one elected lane issues),
// compile-time accumulator rotation, no divisions in the loop
template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) probe_uni(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
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
    constexpr uint32_t idesc = make_idesc_i8(128, N, false);
    const uint32_t a_tmem = tbase + 256;
    const uint64_t b_desc = make_smem_desc(smem_u32(smem), 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t d = tbase + (uint32_t)((j % NACC) * N);
        if (elect_one()) mma_i8_ts(d, a_tmem + (j & 3) * 8, b_desc + (uint64_t)(j & 3) * 2, idesc, (i + j) >= NACC ? 1u : 0u);
        __syncwarp();
      }
    }
    long long t1 = clock64();
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = (unsigned long long)(t1 - t0);
      out[1] = (unsigned long long)(t2 - t0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int N, int NACC>
void run_uni(unsigned long long* d_out) {
  auto k = probe_uni<N, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  const int iters = 4096;
  k<<<1, 128, 150 * 1024>>>(iters, d_out);
  k<<<1, 128, 150 * 1024>>>(iters, d_out);
  unsigned long long h[2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("UNI N=%3d nacc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d)\n", N, NACC, (double)h[0] / iters,
         (double)h[1] / iters, 128 * N / 256);
}

template <int N, bool TS>
void run(unsigned long long* d_out) {
  auto k = probe<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  for (int nacc : {1, 2, 4, 8}) {
    if (nacc * N > 256) continue;
    const int iters = 4096;
    k<<<1, 128, 150 * 1024>>>(iters, nacc, d_out);  // warm
    k<<<1, 128, 150 * 1024>>>(iters, nacc, d_out);
    unsigned long long h[2];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=%3d %s nacc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d)\n", N, TS ? "ts" : "ss", nacc,
           (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256);
  }
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 64);
  run_uni<16, 1>(d_out);
  run_uni<16, 2>(d_out);
  run_uni<16, 4>(d_out);
  run_uni<32, 1>(d_out);
  run_uni<64, 1>(d_out);
  run_uni<128, 1>(d_out);
  run_uni<256, 1>(d_out);
  run<16, true>(d_out);
  run<16, false>(d_out);
  run<32, true>(d_out);
  run<64, true>(d_out);
  run<128, true>(d_out);
  run<256, true>(d_out);
  run<256, false>(d_out);
  run<128, false>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
