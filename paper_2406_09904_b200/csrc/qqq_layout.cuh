// Kernel-side weight layout of the B200 W4A8 path (produced once, offline, by
// qqq_repack_weights from the reference's `pack_i4` bytes, quantize.py:171-189).
//
//   tile   = 128 output channels (the UMMA M of the weight-stationary GEMM)
//   slab   = 32 consecutive k of one tile (one int8 MMA K-step)
//   K_pad  = round_up(K, 256), N_pad = round_up(N, 128)
//
// 4-bit layouts (per-channel "PC" and per-group "PG"):
//   byte offset(n_tile, slab, row, b) = ((n_tile * slabs + slab) * 128 + row) * 16 + b
//   i.e. every (tile, slab) is 2 KiB: 128 rows x 16 B (32 nibbles); a k-block of
//   BK k's of one tile is BK*64 contiguous bytes -> one cp.async.bulk.
//   Nibble order inside a row's 16 B (4 little-endian words w_i, i = 0..3):
//     PC: word i byte j = u[4i+j] | u[16+4i+j] << 4        (pc_convert_word)
//     PG: word i nibble p (bits 4p) = u[8i + 2*(p%4) + p/4] (pg_convert_word)
//   u = q + 8 (the reference's biased storage); padding codes are u = 8 (q = 0).
//
// 8-bit layout ("I8": pre-converted int8 weights, used for gemm_i8_i32 and for
// per-group weights outside the fast path's proven range):
//   offset(n_tile, slab, chunk, row, b) = (((n_tile * slabs + slab) * 2 + chunk) * 128 + row) * 16 + b
//   chunk = (k % 32) / 16, b = k % 16 — exactly the canonical no-swizzle K-major
//   UMMA operand layout, so it is bulk-copied straight into the A operand.
//
// PG scales: s*[n_tile][G_pad][128] binary16 (G_pad = ceil(K_pad / g)), zero padded.
#pragma once

namespace qqq {

constexpr int kTileN = 128;
constexpr int kSlabK = 32;
constexpr int kKPadTo = 256;

enum WeightMode : int { kModePC = 0, kModePG = 1, kModeI8 = 2 };

__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace qqq
