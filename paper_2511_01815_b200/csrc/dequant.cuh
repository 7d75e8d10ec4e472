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
}  // namespace kvtc
