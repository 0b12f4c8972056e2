// Throughput of the f64 -> f32 and f32 -> f16 conversions (developer probe):
// can RN16(RN32(v)) with a midpoint check replace cvt.rn.f16.f64 (12/clk/SM)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/cvt2_probe scripts/cvt2_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>

template <int OP>
__global__ void k(unsigned* out, int iters, double seed) {
  double x0 = seed + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float f0 = (float)x0, f1 = (float)x1, f2 = (float)x2, f3 = (float)x3;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) {  // cvt.rn.f16.f64
      unsigned short t0, t1, t2, t3;
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t0) : "d"(x0 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t1) : "d"(x1 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t2) : "d"(x2 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(t3) : "d"(x3 + i));
      acc ^= t0 ^ t1 ^ t2 ^ t3;
    } else if (OP == 1) {  // cvt.rn.f32.f64
      float t0, t1, t2, t3;
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(t0) : "d"(x0 + i));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(t1) : "d"(x1 + i));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(t2) : "d"(x2 + i));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(t3) : "d"(x3 + i));
      acc ^= __float_as_uint(t0) ^ __float_as_uint(t1) ^ __float_as_uint(t2) ^ __float_as_uint(t3);
    } else if (OP == 2) {  // cvt.rn.f16.f32
      unsigned short t0, t1, t2, t3;
      asm volatile("cvt.rn.f16.f32 %0, %1;" : "=h"(t0) : "f"(f0 + i));
      asm volatile("cvt.rn.f16.f32 %0, %1;" : "=h"(t1) : "f"(f1 + i));
      asm volatile("cvt.rn.f16.f32 %0, %1;" : "=h"(t2) : "f"(f2 + i));
      asm volatile("cvt.rn.f16.f32 %0, %1;" : "=h"(t3) : "f"(f3 + i));
      acc ^= t0 ^ t1 ^ t2 ^ t3;
    } else if (OP == 3) {  // cvt.rn.f16x2.f32 (two values per instruction)
      unsigned t0, t1;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(t0) : "f"(f0 + i), "f"(f1 + i));
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(t1) : "f"(f2 + i), "f"(f3 + i));
      acc ^= t0 ^ t1;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"cvt.rn.f16.f64", "cvt.rn.f32.f64", "cvt.rn.f16.f32", "cvt.rn.f16x2.f32(x2)"};
  int iters = 4096;
  for (int op = 0; op < 4; ++op) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 1) k<1><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 2) k<2><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 3) k<3><<<148 * 4, 256>>>(out, iters, 1.0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    double ops = 148.0 * 4 * 256 * iters * 4;  // conversions (values)
    printf("%-22s %8.3f ms  %6.1f values/clk/SM @1.9GHz\n", names[op], ms, ops / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
