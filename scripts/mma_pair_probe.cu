// tcgen05 kind::i8 issue-rate probe for the 2-CTA pair MMA (developer tool):
// cycles per MMA for cta_group::2 M=256 x N x K=32 (A in TMEM, B in shared
// memory of both CTAs) against cta_group::1 M=128 on one CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2406_09904_b200/csrc \
//        -o scripts/mma_pair_probe scripts/mma_pair_probe.cu
#include <cstdio>

#include "qqq_common.cuh"

using namespace qqq;

template <int N, bool PAIR>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    if (PAIR)
      tmem_alloc_pair(&tslot, 512);
    else
      tmem_alloc(&tslot, 512);
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0 && rank == 0) {
    constexpr uint32_t idesc = make_idesc_i8(PAIR ? 256 : 128, N, false);
    const uint32_t a_tmem = tbase + 256;
    const uint64_t b_desc = make_smem_desc(smem_u32(smem), 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (elect_one()) {
          if (PAIR)
            mma_i8_ts_pair(tbase, a_tmem + (j & 3) * 8, b_desc + (uint64_t)(j & 3) * 2, idesc, (i + j) > 0);
          else
            mma_i8_ts(tbase, a_tmem + (j & 3) * 8, b_desc + (uint64_t)(j & 3) * 2, idesc, (i + j) > 0);
        }
        __syncwarp();
      }
    }
    long long t1 = clock64();
    if (elect_one()) {
      if (PAIR)
        mma_commit_pair(&bar, 0x3);
      else
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = (unsigned long long)(t1 - t0);
      out[1] = (unsigned long long)(t2 - t0);
    }
  } else if (PAIR && warp == 0) {
    mbar_wait(&bar, 0);  // the multicast commit
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (PAIR)
      tmem_dealloc_pair(tbase, 512);
    else
      tmem_dealloc(tbase, 512);
  }
}

template <int N, bool PAIR>
void run(unsigned long long* d_out) {
  auto k = probe<N, PAIR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(PAIR ? 2 : 1);
  lc.blockDim = dim3(128);
  lc.dynamicSmemBytes = 100 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&lc, k, iters, d_out);
  unsigned long long h[2];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (per-SM floor %d)  err=%s\n",
         PAIR ? "PAIR M=256" : "ONE  M=128", N, (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 64);
  run<128, false>(d_out);
  run<256, false>(d_out);
  run<128, true>(d_out);
  run<256, true>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
