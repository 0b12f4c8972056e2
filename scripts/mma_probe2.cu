// Kernel-faithful tcgen05 kind::i8 pacing probe (developer tool): k-blocks of
// BK/32 MMAs (M=128, N=NTOK, A from TMEM buffers, B from a ring of SW128
// activation stages), one commit per k-block, waiting on the commit of the
// k-block kABufs back (the converters' a_empty handshake).
#include <cstdio>
#include "qqq_common.cuh"
using namespace qqq;

template <int NTOK, int BK, bool U8, int VAR>
__global__ void __launch_bounds__(128, 1) pace(int kblocks, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tslot;
  constexpr int kXBytes = NTOK * BK, kXStages = 4, kABufs = 4, kACols = BK / 4;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    constexpr uint32_t idesc = make_idesc_i8(128, NTOK, U8);
    long long t0 = clock64();
    uint32_t b = 0, bph = 0;
    for (int it = 0; it < kblocks; ++it) {
      if (it >= kABufs && VAR != 2 && VAR != 4) mbar_wait(&bars[b], bph ^ 1);  // a_empty of this buffer
      tc_fence_after();
      const uint32_t a_addr = tbase + (NTOK == 256 ? 256 : 2 * NTOK) + b * kACols;
      const uint32_t act = smem_u32(smem + (it % kXStages) * kXBytes);
      if (VAR == 0) {
#pragma unroll
        for (int kk = 0; kk < BK / 32; ++kk) {
          const uint32_t b_addr = act + (kk / 4) * (NTOK * 128) + (kk % 4) * 32;
          const uint64_t b_desc = make_smem_desc(b_addr, 16, 1024, 2);
          if (elect_one()) mma_i8_ts(tbase + (NTOK == 256 ? 0 : (it & 1) * NTOK), a_addr + kk * 8, b_desc, idesc, kk > 0 ? 1u : 0u);
          __syncwarp();
        }
      } else {
        const uint64_t d0 = make_smem_desc(act, 16, 1024, 2);
        const uint32_t dt = tbase + (NTOK == 256 ? 0 : (it & 1) * NTOK);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8_ts(dt, a_addr + kk * 8, d0 + (uint64_t)(((kk / 4) * (NTOK * 128) + (kk % 4) * 32) >> 4), idesc,
                      kk > 0 ? 1u : 0u);
        }
        __syncwarp();
      }
      if (VAR < 3 || it >= kblocks - kABufs) {
        if (elect_one()) mma_commit(&bars[b]);
        __syncwarp();
      }
      if (++b == kABufs) { b = 0; bph ^= 1; }
    }
    long long t1 = clock64();
    for (int i = 0; i < kABufs; ++i) { mbar_wait(&bars[b], bph ^ 1); if (++b == kABufs) { b = 0; bph ^= 1; } }
    long long t2 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int NTOK, int BK, bool U8, int VAR = 0>
void run(unsigned long long* d) {
  auto k = pace<NTOK, BK, U8, VAR>;
  const int smem = 4 * NTOK * BK;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kb = 512;
  k<<<1, 128, smem>>>(kb, d);
  k<<<1, 128, smem>>>(kb, d);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("VAR=%d NTOK=%3d BK=%d %s: %.1f cyc/kblock issue, %.1f cyc/kblock total (%d MMAs/kblock, floor %d)\n", VAR, NTOK, BK,
         U8 ? "u8" : "s8", (double)h[0] / kb, (double)h[1] / kb, BK / 32, (BK / 32) * 128 * NTOK / 256);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  run<256, 128, true, 0>(d);
  run<256, 128, true, 1>(d);
  run<256, 128, true, 2>(d);
  run<128, 128, true, 1>(d);
  run<128, 128, true, 2>(d);

  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
