/*
 * A plain C caller of the C ABI (include/qqq_b200.h): what a reference-side
 * FFI binding does for one per-group W4A8 linear, with nothing but the header,
 * libqqq_b200.so and the CUDA runtime.
 *
 *   gemm_caller <dir> <M> <K> <N> <group>
 *
 * Reads <dir>/x.f16 (M x K binary16), <dir>/packed.u8 (ceil(K/2) x N pack_i4
 * bytes), <dir>/s_star.f16 (K/group x N), <dir>/s_wc.f64 (N); runs
 * qqq_act_quant_ex -> qqq_repack_weights -> qqq_w4a8_gemm_pg on one stream and
 * writes <dir>/y.f16 (M x N) and <dir>/acc.i32 (M x N). Exit status: 0 on
 * success, 10 + the QQQ_ERR_* code of the failing call, 2 on I/O errors.
 * (tests/test_c_abi.py builds it with gcc and checks y / acc against the oracle.)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "qqq_b200.h"

static void* read_file(const char* dir, const char* name, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  void* buf = malloc(bytes ? bytes : 1);
  size_t got = fread(buf, 1, bytes, f);
  fclose(f);
  if (got != bytes) {
    free(buf);
    return NULL;
  }
  return buf;
}

static int write_file(const char* dir, const char* name, const void* data, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f) return -1;
  size_t put = fwrite(data, 1, bytes, f);
  fclose(f);
  return put == bytes ? 0 : -1;
}

static void* to_device(const void* host, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 16) != cudaSuccess) return NULL;
  if (bytes && cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
  return d;
}

#define CHECK_QQQ(call)                                     \
  do {                                                      \
    int rc_ = (call);                                       \
    if (rc_ != QQQ_OK) {                                    \
      fprintf(stderr, "%s failed: status %d\n", #call, rc_); \
      return 10 + rc_;                                      \
    }                                                       \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 6) {
    fprintf(stderr, "usage: %s <dir> <M> <K> <N> <group>\n", argv[0]);
    return 2;
  }
  const char* dir = argv[1];
  const int64_t M = atoll(argv[2]), K = atoll(argv[3]), N = atoll(argv[4]), G = atoll(argv[5]);
  const int64_t Kp = (K + 127) / 128 * 128; /* int8 code rows: 128-byte aligned pitch */
  const size_t x_b = (size_t)(M * K * 2), p_b = (size_t)((K + 1) / 2 * N), s_b = (size_t)(K / G * N * 2);
  void* hx = read_file(dir, "x.f16", x_b);
  void* hp = read_file(dir, "packed.u8", p_b);
  void* hs = read_file(dir, "s_star.f16", s_b);
  void* hc = read_file(dir, "s_wc.f64", (size_t)N * 8);
  if (!hx || !hp || !hs || !hc) return 2;
  if (qqq_device_ok() != QQQ_OK) {
    fprintf(stderr, "not an sm_100 device\n");
    return 10 + QQQ_ERR_CUDA;
  }

  cudaStream_t stream;
  cudaStreamCreate(&stream);
  qqq_stream_t st = (qqq_stream_t)stream;
  void* dx = to_device(hx, x_b);
  void* dp = to_device(hp, p_b);
  void* ds = to_device(hs, s_b);
  void* dc = to_device(hc, (size_t)N * 8);
  int8_t* dq = NULL;
  double* dsa = NULL;
  int32_t *drs = NULL, *dstat = NULL, *dacc = NULL;
  void *dy = NULL, *dw = NULL, *dws = NULL;
  cudaMalloc((void**)&dq, (size_t)(M * Kp));
  cudaMemset(dq, 0, (size_t)(M * Kp));
  cudaMalloc((void**)&dsa, (size_t)M * 8);
  cudaMalloc((void**)&drs, (size_t)M * 4);
  cudaMalloc((void**)&dstat, 4);
  cudaMemset(dstat, 0, 4);
  cudaMalloc(&dy, (size_t)(M * N * 2));
  cudaMalloc((void**)&dacc, (size_t)(M * N * 4));

  /* quant_act_per_token (quantize.py:92-100) + the per-row code sums */
  CHECK_QQQ(qqq_act_quant_ex(dx, 0, M, K, K, dq, Kp, dsa, drs, dstat, st));

  /* FusedScales are given (s_star, s_wc); one-time repack into the kernel layout */
  const size_t wb = qqq_repacked_weight_bytes(QQQ_MODE_PG, K, N, G);
  if (wb == 0) return 10 + QQQ_ERR_UNSUPPORTED;
  cudaMalloc(&dw, wb);
  CHECK_QQQ(qqq_repack_weights((const uint8_t*)dp, (const uint16_t*)ds, K, N, QQQ_MODE_PG, G, dw, dstat, st));

  /* caller-owned split-K workspace, zeroed once */
  const size_t wsb = qqq_gemm_workspace_bytes(M, N, K);
  cudaMalloc(&dws, wsb);
  cudaMemset(dws, 0, wsb);

  /* w4a8_gemm_per_group (gemm.py:188-203): the 17-parameter entry point */
  CHECK_QQQ(qqq_w4a8_gemm_pg(dq, Kp, dsa, drs, dw, G, (const double*)dc, M, N, K, dy, N, dacc, N, dws, wsb, st));
  if (cudaStreamSynchronize(stream) != cudaSuccess) return 10 + QQQ_ERR_CUDA;

  int32_t stat = 0;
  cudaMemcpy(&stat, dstat, 4, cudaMemcpyDeviceToHost);
  if (stat & QQQ_STAT_NONFINITE) return 10 + QQQ_ERR_DATA;
  if (stat & QQQ_STAT_NEED_CLAMP) return 10 + QQQ_ERR_UNSUPPORTED; /* caller would build the I8 blob */

  void* hy = malloc((size_t)(M * N * 2));
  void* ha = malloc((size_t)(M * N * 4));
  cudaMemcpy(hy, dy, (size_t)(M * N * 2), cudaMemcpyDeviceToHost);
  cudaMemcpy(ha, dacc, (size_t)(M * N * 4), cudaMemcpyDeviceToHost);
  if (write_file(dir, "y.f16", hy, (size_t)(M * N * 2)) || write_file(dir, "acc.i32", ha, (size_t)(M * N * 4)))
    return 2;
  printf("ok %s\n", qqq_version());
  return 0;
}
