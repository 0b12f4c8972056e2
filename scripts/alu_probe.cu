// Per-SM throughput of the conversion instruction classes (developer tool):
// 8 independent chains per thread, 16 warps per CTA, one CTA per SM.
#include <cstdio>
#include <cuda_fp16.h>
#include <stdint.h>

template <int OP>
__global__ void __launch_bounds__(512) k(uint32_t* out, int iters, uint32_t seed) {
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = seed * (threadIdx.x + 7 * i + 1);
  uint32_t m = seed ^ 0x64006400u, s = seed | 0x3c003c00u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) asm volatile("lop3.b32 %0, %0, 0x000F000F, %1, 0xEA;" : "+r"(r[i]) : "r"(m));
        if (OP == 1) asm volatile("prmt.b32 %0, %0, %1, 0x6420;" : "+r"(r[i]) : "r"(m));
        if (OP == 2) asm volatile("{.reg .b32 c; mov.b32 c, 0xE408E408; add.rn.f16x2 %0, %0, c;}" : "+r"(r[i]));
        if (OP == 3) asm volatile("{.reg .b32 c; mov.b32 c, 0x64806480; fma.rn.f16x2 %0, %0, %1, c;}" : "+r"(r[i]) : "r"(s));
        if (OP == 4) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(s), "r"(m));
        if (OP == 5) asm volatile("shr.b32 %0, %0, 8;" : "+r"(r[i]));
        if (OP == 6) asm volatile("xor.b32 %0, %0, %1;" : "+r"(r[i]) : "r"(m));
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= r[i];
  if (x == 0x1234567u) out[0] = x;
}

template <int OP>
void run(const char* name, uint32_t* d) {
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<OP><<<148, 512>>>(d, iters, 3);
  cudaEventRecord(a);
  k<OP><<<148, 512>>>(d, iters, 3);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double instr_per_sm = (double)iters * 64 * 16;  // warp-instructions per SM
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-28s %.2f warp-instr/cycle/SM (%.2f per SMSP) [max-clock est.]\n", name, instr_per_sm / cycles,
         instr_per_sm / cycles / 4);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 64);
  run<0>("LOP3 (and-or, reg c)", d);
  run<1>("PRMT", d);
  run<2>("HADD2 (imm)", d);
  run<3>("HFMA2 (R,R,imm)", d);
  run<4>("HFMA2 (R,R,R)", d);
  run<5>("SHF.R", d);
  run<6>("LOP3 xor reg", d);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
