// quant.cuh — the per-(token, group) quantiser of the compress epilogue, shared
// by the fused tcgen05 epilogue (gemm.cu) and the SIMT reference kernel
// (elementwise.cu).  Readings Q2/Q3/Q5 with fp16 shift/scale (R3) and RNE codes
// (R4), evaluated in fp32 from the fp32 accumulator.
#pragma once
#include "common.cuh"

namespace kvtc {

__device__ __forceinline__ void store_u32_any(uint8_t *p, uint32_t v, bool aligned) {
  if (aligned) {
    *reinterpret_cast<uint32_t *>(p) = v;
  } else {
    p[0] = v & 0xFF; p[1] = (v >> 8) & 0xFF; p[2] = (v >> 16) & 0xFF; p[3] = v >> 24;
  }
}

// ---------------------------------------------------------------- epilogues
// Quantise one (token, group piece) whose fp32 coefficients are x[0..size).
// Implements Q2/Q3/Q5 in fp32 with fp16 shift/scale (R3, R4).
__device__ __forceinline__ void group_factors(int type, float mn, float mx, uint16_t &sh, uint16_t &sc) {
  if (type == KVTC_T_FP8) {
    sh = f16_bits_f32(__fmul_rn(__fadd_rn(mx, mn), 0.5f));
    sc = f16_bits_f32(__fdiv_rn(__fmul_rn(__fsub_rn(mx, mn), 0.5f), 448.0f));
  } else {
    const float L = type == KVTC_T_INT2 ? 3.0f : 15.0f;
    sh = f16_bits_f32(mn);
    sc = f16_bits_f32(__fdiv_rn(__fsub_rn(mx, mn), L));
  }
}
// Q4: a 16-bit factor that is not finite (exponent field all ones: inf or NaN)
// means the coefficient range overflowed binary16 -> KVTC_E_NUMERIC.
__device__ __forceinline__ bool factor_overflow(uint16_t sh, uint16_t sc) {
  return (sh & 0x7C00u) == 0x7C00u || (sc & 0x7C00u) == 0x7C00u;
}
__device__ __forceinline__ uint32_t encode_one(int type, float x, float shift, float scale) {
  if (scale == 0.0f) return 0u;
  const float y = __fdiv_rn(__fsub_rn(x, shift), scale);
  if (type == KVTC_T_FP8) return e4m3_from_f32(y);
  const float L = type == KVTC_T_INT2 ? 3.0f : 15.0f;
  return static_cast<uint32_t>(fminf(fmaxf(rintf(y), 0.0f), L));
}

// Writes the codes of `size` coefficients (byte-aligned per token) to dst.
__device__ __forceinline__ void write_codes_aligned(uint8_t *dst, const float *x, int size, int type, float shift,
                                                    float scale, bool aligned4) {
  const int b = bits_of(type);
  const int per_word = 32 / b;
  for (int c0 = 0; c0 < size; c0 += per_word) {
    uint32_t w = 0;
    const int n = min(per_word, size - c0);
    for (int j = 0; j < n; ++j) w |= encode_one(type, x[c0 + j], shift, scale) << (j * b);
    const int nbytes = (n * b + 7) / 8;
    uint8_t *p = dst + (c0 * b) / 8;
    if (nbytes == 4) {
      store_u32_any(p, w, aligned4);
    } else {
      for (int k = 0; k < nbytes; ++k) p[k] = (w >> (8 * k)) & 0xFF;
    }
  }
}

// The codes of 16 coefficients (byte-aligned), fully unrolled so x stays in registers.
__device__ __forceinline__ void write_codes16(uint8_t *dst, const float *x, int type, float shift, float scale,
                                              bool aligned4) {
  uint32_t c[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) c[j] = encode_one(type, x[j], shift, scale);
  const int b = bits_of(type);
  const int per = 32 / b;                       // codes per 32-bit word: 16 / 8 / 4
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    if (w * per >= 16) break;
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j >= w * per && j < (w + 1) * per) v |= c[j] << ((j - w * per) * b);
    store_u32_any(dst + 4 * w, v, aligned4);
  }
}

// Emit shift/scale (part 0 only) and the codes of one (token, group piece).
//   x: the piece's fp32 coefficients (D - mu V_c), mn/mx: the row min/max over
//   the WHOLE group; row: token index inside the tile; warp_tok0: first token of
//   this warp; tile_base: payload tile; cb: the group's code block in this tile.
// Sub-byte tokens (size*bits < 8) are packed by an OR-reduction over the warp,
// so all 32 lanes of the warp must call this together (valid = row < ntok).
__device__ __forceinline__ void emit_group(const float *x, int size, int full_size, int part, int type, int gidx,
                                           float mn, float mx, bool valid, int row, int lane, int warp_tok0,
                                           int ntok, bool last, uint8_t *tile_base, uint8_t *cb) {
  uint16_t sh, sc;
  group_factors(type, mn, mx, sh, sc);
  const float shift = f16_val(sh), scale = f16_val(sc);
  if (valid && part == 0)
    store_u32_any(tile_base + 4 * (int64_t(gidx) * ntok + row), uint32_t(sh) | (uint32_t(sc) << 16), !last);
  const int b = bits_of(type);
  const int tok_bits = full_size * b;
  if ((tok_bits & 7) == 0) {
    if (valid)
      write_codes_aligned(cb + int64_t(row) * (tok_bits / 8) + part * (size * b / 8), x, size, type, shift, scale,
                          !last);
    return;
  }
  uint32_t bits_v = 0;
  for (int c = 0; c < size; ++c) bits_v |= (valid ? encode_one(type, x[c], shift, scale) : 0u) << (c * b);
  const int nb = tok_bits;
  const int bitpos = lane * nb;
  const int64_t blk_len = (int64_t(ntok) * nb + 7) / 8;
  const int64_t warp_byte0 = int64_t(warp_tok0) * nb / 8;
  for (int w = 0; w < nb; ++w) {                 // 32 lanes * nb bits = nb words
    uint32_t mine = 0;
    if ((bitpos >> 5) == w) mine = bits_v << (bitpos & 31);
    if (((bitpos + nb - 1) >> 5) == w && (bitpos >> 5) != w) mine = bits_v >> (32 - (bitpos & 31));
    const uint32_t word = __reduce_or_sync(0xffffffffu, mine);
    if (lane == w) {
      const int64_t off = warp_byte0 + 4 * w;
      if (!last) {
        *reinterpret_cast<uint32_t *>(cb + off) = word;
      } else {
        for (int k = 0; k < 4; ++k)
          if (off + k < blk_len) cb[off + k] = (word >> (8 * k)) & 0xFF;
      }
    }
  }
}

}  // namespace kvtc
