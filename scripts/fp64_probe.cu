// Throughput probe for the epilogue's FP64 / conversion instructions on this
// part (developer tool). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>

template <int OP>
__global__ void k(double* out, int iters, double seed) {
  double a = seed + threadIdx.x, b = 1.0000001, acc = 0;
  int ia = threadIdx.x;
  unsigned short h = 0;
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) {  // DMUL, 4 independent chains
      x0 *= b; x1 *= b; x2 *= b; x3 *= b;
    } else if (OP == 1) {  // I2F.F64
      x0 += (double)(ia + i); x1 += (double)(ia - i); x2 += (double)(ia ^ i); x3 += (double)(ia | i);
    } else if (OP == 2) {  // F2F.F16.F64
      unsigned short t0, t1, t2, t3;
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t0) : "d"(x0 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t1) : "d"(x1 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t2) : "d"(x2 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t3) : "d"(x3 + i));
      h ^= t0 ^ t1 ^ t2 ^ t3;
    } else if (OP == 3) {  // FFMA reference
      float f0 = (float)x0, f1 = (float)x1;
      for (int j = 0; j < 4; ++j) { f0 = f0 * 1.0001f + 0.5f; f1 = f1 * 1.0001f + 0.5f; }
      x0 = f0; x1 = f1;
    }
  }
  acc = x0 + x1 + x2 + x3 + h;
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"DMUL", "I2F.F64", "F2F.F16.F64", "FFMA(+2 F2F)"};
  int iters = 4096;
  for (int op = 0; op < 4; ++op) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 1) k<1><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 2) k<2><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 3) k<3><<<148 * 4, 256>>>(out, iters, 1.0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double ops = 148.0 * 4 * 256 * iters * 4;
    printf("%-14s %8.3f ms  %10.1f Gop/s  %6.1f op/clk/SM @1.9GHz\n", names[op], ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
