// Kernel-side weight layout of the B200 W4A8 path (produced once, offline, by
// qqq_repack_weights from the reference's `pack_i4` bytes, quantize.py:171-189).
//
//   tile        = 128 output channels (the UMMA M of the weight-stationary GEMM)
//   slab        = 32 consecutive k of a tile (one int8 MMA K-step)
//   super-slab  = 128 consecutive k of a tile (4 slabs) = the unit of the blob
//   K_pad = round_up(K, 256), N_pad = round_up(N, 128)
//
// The blob is [n_tile][super-slab][SSB bytes]; a k-block of BK k's of one tile
// is BK/128 consecutive super-slabs, i.e. ONE contiguous cp.async.bulk (TMA
// op count, not bytes, bounds a decode-sized copy stream: probe in
// scripts/stream_probe.cu, 4 KiB ops cap at 2.1 TB/s, 16 KiB ops reach 6.9 TB/s).
//
// Super-slab contents by mode:
//   PC (per-channel): 4 x [128 rows][16 B] nibbles                   SSB = 8192
//   PG (per-group):   4 x [128 rows][16 B] nibbles, then the super-slab's
//                     group scales s* as [ngs][128 rows] binary16,
//                     ngs = 128 / min(g, 128)                      SSB = 8192 + 256*ngs
//   I8 (int8):        8 x [128 rows][16 B] int8 (k16-chunk major)     SSB = 16384
//                     == the canonical no-swizzle K-major UMMA operand, bulk
//                     copied straight into the MMA's A buffer.
// Nibble order inside a row's 16 B (4 little-endian words w_i, i = 0..3):
//   PC: word i byte j = u[4i+j] | u[16+4i+j] << 4        (pc_convert_word)
//   PG: word i nibble p (bits 4p) = u[8i + 2*(p%4) + p/4] (pg_convert_word)
// u = q + 8 (the reference's biased storage); padding codes are u = 8 (q = 0),
// padding scales are 0.
#pragma once

#include <stdint.h>

namespace qqq {

constexpr int kTileN = 128;
constexpr int kSlabK = 32;
constexpr int kSuperK = 128;
constexpr int kKPadTo = 256;

enum WeightMode : int { kModePC = 0, kModePG = 1, kModeI8 = 2 };

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// per-group fast path: groups never straddle a 32-k slab nor a 128-k super-slab
__host__ __device__ inline bool pg_group_ok(int64_t g) {
  return g > 0 && ((g % 32 == 0 && 128 % g == 0) || g % 128 == 0);
}
__host__ __device__ inline int pg_groups_per_ss(int64_t g) { return (int)(128 / (g < 128 ? g : 128)); }

__host__ __device__ inline int64_t ss_bytes(int mode, int64_t g) {
  return mode == kModeI8 ? 16384 : mode == kModePC ? 8192 : 8192 + 256 * pg_groups_per_ss(g);
}

}  // namespace qqq
