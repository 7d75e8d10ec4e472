// dequant.cuh — R5 dequantisation arithmetic shared by the dequantiser
// (dequant_rows_kernel, elementwise.cu) and the opt-in fused producer of the
// reconstruction GEMM (gemm.cu).  Payload layout: DESIGN.md §4 (tile = params
// section, then per group a token-major code block).
#pragma once

#include "internal.h"

namespace kvtc {

// R5: D^ = fp16(x^) with x^ = v * scale + shift, v the integer level (int2 /
// int4) or the E4M3 value (fp8).  v, scale and shift are exact in fp16, so
// fma.rn.f16x2 rounds the exact x^ once: the oracle's fp16(fp64 x^).
__device__ __forceinline__ uint32_t hfma2_u(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t hsub2_u(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t prmt_u(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t mask, uint32_t bits) {   // (a & mask) | bits
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(mask), "r"(bits));
  return d;
}
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint32_t two_bytes) {
  uint32_t d;
  const unsigned short in = static_cast<unsigned short>(two_bytes & 0xFFFF);
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(d) : "h"(in));
  return d;
}
__device__ __forceinline__ uint32_t ld_u32_any(const uint8_t *p) {
  if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) return *reinterpret_cast<const uint32_t *>(p);
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}
// The codes of 8 consecutive elements of one token (8 * b bits, byte aligned).
__device__ __forceinline__ void load_codes8(const uint8_t *p, int b, uint32_t &lo, uint32_t &hi) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  hi = 0;
  if (b == 2) {
    lo = (a & 1) == 0 ? uint32_t(*reinterpret_cast<const uint16_t *>(p)) : uint32_t(p[0]) | (uint32_t(p[1]) << 8);
  } else if (b == 4) {
    lo = ld_u32_any(p);
  } else if ((a & 7) == 0) {
    const uint2 v = *reinterpret_cast<const uint2 *>(p);
    lo = v.x;
    hi = v.y;
  } else {
    lo = ld_u32_any(p);
    hi = ld_u32_any(p + 4);
  }
}
// 8 elements -> 8 fp16 (one 16-byte chunk of an A row).  Integer levels become
// fp16 through the 1024 + c bit trick (exact), pairs (c_k, c_k+4) per word,
// reordered with prmt after the fma.
__device__ __forceinline__ uint4 dq8(int type, uint32_t lo, uint32_t hi, uint32_t params) {
  const uint32_t sh = params & 0xFFFFu, sc = params >> 16;
  const uint32_t sh2 = sh | (sh << 16), sc2 = sc | (sc << 16);
  uint4 o;
  if (type == KVTC_T_FP8) {
    o.x = hfma2_u(e4m3x2_to_f16x2(lo), sc2, sh2);
    o.y = hfma2_u(e4m3x2_to_f16x2(lo >> 16), sc2, sh2);
    o.z = hfma2_u(e4m3x2_to_f16x2(hi), sc2, sh2);
    o.w = hfma2_u(e4m3x2_to_f16x2(hi >> 16), sc2, sh2);
    return o;
  }
  // int4: nibble k at bits 4k; int2: spread the two code bytes to bytes 0 and 2
  const bool i4 = type == KVTC_T_INT4;
  const uint32_t x = i4 ? lo : prmt_u(lo, 0u, 0x4140u);
  const uint32_t mask = i4 ? 0x000F000Fu : 0x00030003u;
  const int step = i4 ? 4 : 2;
  uint32_t y[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    y[k] = hfma2_u(hsub2_u(and_or(x >> (k * step), mask, 0x64006400u), 0x64006400u), sc2, sh2);   // (c_k, c_k+4)
  o.x = prmt_u(y[0], y[1], 0x5410u);
  o.y = prmt_u(y[2], y[3], 0x5410u);
  o.z = prmt_u(y[0], y[1], 0x7632u);
  o.w = prmt_u(y[2], y[3], 0x7632u);
  return o;
}
// One element of any group (columns that are not whole aligned 8-chunks of one
// group: size-1 groups, misaligned starts).
__device__ __forceinline__ uint16_t dq1(const uint8_t *tile, const int64_t *coff, int ntok, int row, const DqCol &d) {
  if (!d.type) return 0;
  const uint32_t pr = ld_u32_any(tile + 4 * (int64_t(d.gidx) * ntok + row));
  const int b = bits_of(d.type);
  const int64_t bit = (int64_t(row) * d.size + d.j) * b;
  const uint32_t code = (uint32_t(tile[coff[d.gidx] + (bit >> 3)]) >> (bit & 7)) & ((1u << b) - 1);
  const uint32_t v = d.type == KVTC_T_FP8 ? e4m3x2_to_f16x2(code) : uint32_t(__half_as_ushort(__uint2half_rn(code)));
  return uint16_t(hfma2_u(v, pr >> 16, pr & 0xFFFFu) & 0xFFFFu);
}
// Element-by-element chunk (partial tiles only): out of line, so the unrolled
// per-stage loops stay small (the inlined copies overflowed the instruction cache).
static __device__ __noinline__ uint4 dq_generic8(const DqCol *cols, int col0, const uint8_t *tile, const int64_t *coff,
                                          int ntok, int row) {
  uint16_t h[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) h[k] = dq1(tile, coff, ntok, row, cols[col0 + k]);
  return make_uint4(uint32_t(h[0]) | (uint32_t(h[1]) << 16), uint32_t(h[2]) | (uint32_t(h[3]) << 16),
                    uint32_t(h[4]) | (uint32_t(h[5]) << 16), uint32_t(h[6]) | (uint32_t(h[7]) << 16));
}

// One block of D^: rows [32 by, 32 by + 32) x chunks [32 bx, 32 bx + 32), by
// kWarps warps (lane, wy).  Chunks that are 8 aligned elements of one group of a
// full tile (DqChunk ok = 1): lane = chunk, a warp writes 512 contiguous bytes of
// a row, 4 rows' loads issued before any is consumed; each reads its token's fp16
// factors (4 B) and 8 codes (2 / 4 / 8 B, aligned) and converts with dq8.  Every
// other chunk (size-1 runs, misaligned starts, the partial last tile) goes one
// warp per chunk with lane = row, so the per-(group, token) factor and code loads
// of a warp are consecutive in the payload (token-major group blocks).  Columns
// past r_nz in the last chunk are written as 0 (the GEMM's tensor map never reads
// them).  Plain loads: the fused kernel reads payload bytes written in the same
// launch (after a gpu-scope acquire), which the non-coherent path may not see.
template <int kWarps>
__device__ __forceinline__ void dequant_block(const DqArgs &a, int64_t by, int64_t bx, int lane, int wy) {
  constexpr int kRows = 32 / kWarps;                 // rows per thread, in batches of 4
  const int64_t t = (by * 32) / kTileM;              // tile (32 | 128)
  const int ntok = int(a.m - t * kTileM < kTileM ? a.m - t * kTileM : kTileM);
  const bool full = ntok == kTileM;
  const int rbase = int(by * 32 - t * kTileM);        // first row of the block inside the tile
  const uint8_t *tile = a.payload + t * a.tile_bytes;
  __half *drow = a.Dh + (t * kTileM + rbase) * a.ld;
  const int k = int(bx) * 32 + lane;
  const DqChunk d = k < a.nch8 ? a.chunks[k] : DqChunk{0, 0, 0, 0, 0, -1};
  const bool dense = full && k < a.nch8 && d.ok == 1;
  if (dense) {
    const int b = bits_of(d.type);
#pragma unroll
    for (int r0 = 0; r0 < kRows; r0 += 4) {
      uint32_t pr[4], lo[4], hi[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = rbase + wy + kWarps * (r0 + r);
        pr[r] = *reinterpret_cast<const uint32_t *>(tile + d.par_base + 4 * row);
        load_codes8(tile + d.code_base + row * int32_t(d.stride), b, lo[r], hi[r]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        *reinterpret_cast<uint4 *>(drow + (wy + kWarps * (r0 + r)) * a.ld + 8 * int64_t(k)) =
            dq8(d.type, lo[r], hi[r], pr[r]);
    }
  }
  uint32_t other = __ballot_sync(0xFFFFFFFFu, k < a.nch8 && !dense);
  const int64_t *coff = full ? a.codes_off_full : a.codes_off_last;
  const int row = rbase + lane;
  for (int j = 0; other; ++j, other >>= 1) {
    if (!(other & 1u) || (j % kWarps) != wy) continue;
    const int kk = int(bx) * 32 + j;
    const DqChunk e = a.chunks[kk];
    if (row >= ntok) continue;
    uint4 v;
    if (full && e.run_code >= 0) {
      // 8 size-1 groups of one type: factors 512 B apart, code blocks run_stride apart
      const int b = bits_of(e.type);
      uint32_t pr[8], cd[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        pr[q] = *reinterpret_cast<const uint32_t *>(tile + e.par_base + q * 4 * kTileM + 4 * row);
        const int bit = row * b;
        cd[q] = (uint32_t(tile[e.run_code + q * int32_t(e.stride) + (bit >> 3)]) >> (bit & 7)) & ((1u << b) - 1);
      }
      uint32_t hv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t x =
            e.type == KVTC_T_FP8 ? e4m3x2_to_f16x2(cd[q]) : uint32_t(__half_as_ushort(__uint2half_rn(cd[q])));
        hv[q] = hfma2_u(x, pr[q] >> 16, pr[q] & 0xFFFFu) & 0xFFFFu;
      }
      v = make_uint4(hv[0] | (hv[1] << 16), hv[2] | (hv[3] << 16), hv[4] | (hv[5] << 16), hv[6] | (hv[7] << 16));
    } else {
      v = dq_generic8(a.cols, 8 * kk, tile, coff, ntok, row);
    }
    *reinterpret_cast<uint4 *>(drow + lane * a.ld + 8 * int64_t(kk)) = v;
  }
}
}  // namespace kvtc
