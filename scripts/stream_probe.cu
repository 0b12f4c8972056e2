// Streaming-bandwidth probe for the decode (HBM-bound) regime: how fast can
// 148 SMs pull a read-only buffer into shared memory with cp.async.bulk
// (TMA 1-D) vs plain 16-byte LDG? Developer tool (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe scripts/stream_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_stream(const uint8_t* src, size_t per_cta, int chunk, int stages, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[32];
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  int nchunks = (int)(per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long acc = 0;
  for (int i = 0; i < nchunks + stages; ++i) {
    if (i >= stages) {  // consume chunk i - stages
      int j = i - stages, s = j % stages;
      uint32_t ph = (j / stages) & 1, done = 0;
      while (!done) {
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0,1,0,p;}"
                     : "=r"(done) : "r"(su32(&full[s])), "r"(ph) : "memory");
      }
      acc += sm[s * chunk];
    }
    if (i < nchunks) {
      int s = i % stages;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + (size_t)s * chunk)),
                   "l"(base + (size_t)i * chunk), "r"(chunk), "r"(su32(&full[s]))
                   : "memory");
    }
  }
  sink[blockIdx.x] = acc;
}

template <int U>
__global__ void ldg_stream(const uint4* src, size_t n16_per_cta, unsigned long long* sink) {
  const uint4* base = src + (size_t)blockIdx.x * n16_per_cta;
  uint32_t x = 0;
  for (size_t i = threadIdx.x; i < n16_per_cta; i += (size_t)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t idx = i + (size_t)u * blockDim.x;
      v[u] = idx < n16_per_cta ? __ldg(base + idx) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (x == 0x12345678) sink[blockIdx.x] = x;
}

int main() {
  const size_t total = (size_t)1 << 30;  // 1 GiB, far larger than L2
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int chunks[] = {4096, 8192, 16384, 32768};
  const int stagess[] = {2, 4, 6, 8, 12};
  for (int mult : {1, 2}) {
    int ctas = sms * mult;
    for (int chunk : chunks)
      for (int st : stagess) {
        if ((size_t)chunk * st > (mult == 1 ? 196608u : 98304u)) continue;
        size_t per = total / ctas / chunk * chunk;
        for (int r = 0; r < 2; ++r) {
          cudaEventRecord(a);
          bulk_stream<<<ctas, 32, chunk * st>>>(buf, per, chunk, st, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("bulk ctas=%d chunk=%6d stages=%2d inflight=%7d B/SM: %7.1f GB/s\n", ctas, chunk, st,
               chunk * st * mult, per * ctas / ms / 1e6);
      }
  }
  for (int threads : {256, 512, 1024})
    for (int ctas : {148, 296}) {
      size_t n16 = total / 16 / ctas;
      for (int r = 0; r < 2; ++r) {
        cudaEventRecord(a);
        ldg_stream<8><<<ctas, threads>>>((const uint4*)buf, n16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("ldg  ctas=%d threads=%4d unroll=8: %7.1f GB/s\n", ctas, threads, n16 * 16 * ctas / ms / 1e6);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
