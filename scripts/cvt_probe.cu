// Conversion-instruction throughput on this part (developer tool).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
template <int OP>
__global__ void k(uint32_t* out, int iters, double seed) {
  double d0 = seed + threadIdx.x, d1 = d0 + 1, d2 = d0 + 2, d3 = d0 + 3;
  float f0 = (float)d0, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
  int i0 = threadIdx.x, i1 = i0 + 1, i2 = i0 + 2, i3 = i0 + 3;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) {  // cvt.rn.f32.f64
      float a, b, c, e;
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(a) : "d"(d0 + i));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(b) : "d"(d1 + i));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(c) : "d"(d2 + i));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(e) : "d"(d3 + i));
      acc ^= __float_as_uint(a) ^ __float_as_uint(b) ^ __float_as_uint(c) ^ __float_as_uint(e);
    } else if (OP == 1) {  // cvt.rn.f32.s32
      float a, b, c, e;
      asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a) : "r"(i0 + i));
      asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(b) : "r"(i1 + i));
      asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(c) : "r"(i2 + i));
      asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(e) : "r"(i3 + i));
      acc ^= __float_as_uint(a) ^ __float_as_uint(b) ^ __float_as_uint(c) ^ __float_as_uint(e);
    } else if (OP == 2) {  // cvt.rn.f16x2.f32 (2 outputs each)
      uint32_t a, b;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(a) : "f"(f0 + i), "f"(f1 + i));
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(b) : "f"(f2 + i), "f"(f3 + i));
      acc ^= a ^ b;
    } else if (OP == 3) {  // cvt.rn.f16.f64
      unsigned short a, b, c, e;
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(a) : "d"(d0 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(b) : "d"(d1 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(c) : "d"(d2 + i));
      asm volatile("cvt.rn.f16.f64 %0, %1;" : "=h"(e) : "d"(d3 + i));
      acc ^= a ^ b ^ c ^ e;
    } else if (OP == 4) {  // cvt.rz.f32.f64
      float a, b, c, e;
      asm volatile("cvt.rz.f32.f64 %0, %1;" : "=f"(a) : "d"(d0 + i));
      asm volatile("cvt.rz.f32.f64 %0, %1;" : "=f"(b) : "d"(d1 + i));
      asm volatile("cvt.rz.f32.f64 %0, %1;" : "=f"(c) : "d"(d2 + i));
      asm volatile("cvt.rz.f32.f64 %0, %1;" : "=f"(e) : "d"(d3 + i));
      acc ^= __float_as_uint(a) ^ __float_as_uint(b) ^ __float_as_uint(c) ^ __float_as_uint(e);
    }
  }
  if (acc == 0x12345u) out[0] = acc;
}
int main() {
  uint32_t* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"F2F.F32.F64 (rn)", "I2F.F32.S32", "F2FP.F16.F32 x2", "F2F.F16.F64", "F2F.F32.F64 (rz)"};
  int iters = 4096;
  for (int op = 0; op < 5; ++op) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 1) k<1><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 2) k<2><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 3) k<3><<<148 * 4, 256>>>(out, iters, 1.0);
      if (op == 4) k<4><<<148 * 4, 256>>>(out, iters, 1.0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double ops = 148.0 * 4 * 256 * iters * 4;  // outputs
    printf("%-20s %8.3f ms  %6.1f outputs/clk/SM @1.9GHz\n", names[op], ms, ops / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
