// elementwise.cu — the HBM-bound kernels around the GEMMs:
//   K1   gather + un-RoPE: cache view -> X [m x p] bf16, features (layer, head,
//        dim); keys rotated by -theta with reading R1.
//   rope_table  (cos, sin)(theta), theta = fp32(pos) * inv_freq (fp32), evaluated
//        in fp64 and rounded to fp32 (R1/R7 tables).
//   quant_pack_simt  the §4 quantiser/packer from an fp32 D (test reference for
//        the fused epilogue: same device functions, no tensor cores).
//   dequant  payload -> D^ fp16 (R5).
//   raw token copies for sinks / window.
#include "internal.h"
#include "quant.cuh"
#include "dequant.cuh"

namespace kvtc {

// ------------------------------------------------------------- RoPE tables
__global__ void rope_table_kernel(const float *invf, int half, int64_t pos_first, int64_t n, float2 *cs) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n * half) return;
  const int64_t r = i / half;
  const int j = int(i % half);
  const float pos = float(pos_first + r);
  const float theta = __fmul_rn(pos, invf[j]);
  double s, c;
  sincos(double(theta), &s, &c);
  cs[i] = make_float2(__double2float_rn(c), __double2float_rn(s));
}

kvtc_status launch_rope_table(const float *invf_dev, int32_t half, int64_t pos_first, int64_t n, float2 *cs,
                              cudaStream_t st) {
  const int64_t total = n * half;
  if (total == 0) return KVTC_OK;
  rope_table_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, st>>>(invf_dev, half, pos_first, n, cs);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

// R1: x1' = fp32(fp32(x1 c) + fp32(x2 s)), x2' = fp32(fp32(x2 c) - fp32(x1 s)), then bf16.
__device__ __forceinline__ void unrope_pair(float x1, float x2, float2 t, __nv_bfloat16 &o1, __nv_bfloat16 &o2) {
  o1 = __float2bfloat16_rn(__fadd_rn(__fmul_rn(x1, t.x), __fmul_rn(x2, t.y)));
  o2 = __float2bfloat16_rn(__fsub_rn(__fmul_rn(x2, t.x), __fmul_rn(x1, t.y)));
}

__device__ __forceinline__ int64_t view_slot(int layout, int page_tokens, const int32_t *block_table, int64_t tok) {
  if (layout == KVTC_LAYOUT_PAGED) return int64_t(block_table[tok / page_tokens]) * page_tokens + tok % page_tokens;
  return tok;
}

// ---------------------------------------------------------------- K1 gather
// One thread = 8 consecutive elements of the low half of a head (+ their
// partners in the high half for half-split pairing), one (token, layer, head).
struct GatherArgs {
  __nv_bfloat16 *const *bases;
  int32_t layout, page_tokens;
  const int32_t *block_table;
  int32_t layers, heads, d, pairing;
  int64_t tok_begin, ntok;
  const float2 *cs;  // [ntok x d/2] or null (values)
  __nv_bfloat16 *X;
  int64_t ldx;       // row stride of X (elements, >= layers * heads * d)
};

__device__ __forceinline__ void gather_unit(const GatherArgs &a, const int64_t r, const int layer, const int head,
                                            const int v) {
  const int64_t tok = a.tok_begin + r;
  const int64_t slot = view_slot(a.layout, a.page_tokens, a.block_table, tok);
  const int hd = a.heads * a.d;
  const __nv_bfloat16 *src = a.bases[layer] + slot * hd + head * a.d;
  __nv_bfloat16 *dst = a.X + r * a.ldx + int64_t(layer) * hd + head * a.d;
  if (a.pairing == 0) {
    const int j0 = v * 8;  // low-half offset
    uint4 lo = *reinterpret_cast<const uint4 *>(src + j0);
    uint4 hi = *reinterpret_cast<const uint4 *>(src + a.d / 2 + j0);
    if (a.cs) {
      const __nv_bfloat16 *l = reinterpret_cast<const __nv_bfloat16 *>(&lo);
      const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&hi);
      __align__(16) __nv_bfloat16 ol[8], oh[8];
      const float2 *t = a.cs + r * (a.d / 2) + j0;
#pragma unroll
      for (int k = 0; k < 8; ++k) unrope_pair(__bfloat162float(l[k]), __bfloat162float(h[k]), t[k], ol[k], oh[k]);
      lo = *reinterpret_cast<uint4 *>(ol);
      hi = *reinterpret_cast<uint4 *>(oh);
    }
    *reinterpret_cast<uint4 *>(dst + j0) = lo;
    *reinterpret_cast<uint4 *>(dst + a.d / 2 + j0) = hi;
  } else {
    // interleaved pairs (2j, 2j+1): this thread owns elements [16v, 16v+16)
    const int j0 = v * 16;
    uint4 w0 = *reinterpret_cast<const uint4 *>(src + j0);
    uint4 w1 = *reinterpret_cast<const uint4 *>(src + j0 + 8);
    if (a.cs) {
      __align__(16) __nv_bfloat16 in[16], out[16];
      *reinterpret_cast<uint4 *>(in) = w0;
      *reinterpret_cast<uint4 *>(in + 8) = w1;
      const float2 *t = a.cs + r * (a.d / 2) + j0 / 2;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        unrope_pair(__bfloat162float(in[2 * k]), __bfloat162float(in[2 * k + 1]), t[k], out[2 * k], out[2 * k + 1]);
      w0 = *reinterpret_cast<uint4 *>(out);
      w1 = *reinterpret_cast<uint4 *>(out + 8);
    }
    *reinterpret_cast<uint4 *>(dst + j0) = w0;
    *reinterpret_cast<uint4 *>(dst + j0 + 8) = w1;
  }
}

// Grid-stride over (token, layer, head, 16-element piece) units; a bounded grid
// when it overlaps a persistent GEMM (codec.cu).  32-bit index math (the launcher
// falls back to 64-bit only past 2^32 units).
template <typename Idx>
__global__ void __launch_bounds__(256) gather_kernel(GatherArgs a, Idx total) {
  const Idx vph = Idx(a.d / 16);                      // threads per head (8 lo + 8 hi elements each)
  const Idx per_layer = Idx(a.heads) * vph;
  const Idx per_tok = Idx(a.layers) * per_layer;
  for (Idx i = Idx(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += Idx(gridDim.x) * blockDim.x) {
    const Idx r = i / per_tok;
    Idx rem = i - r * per_tok;
    const Idx layer = rem / per_layer;
    rem -= layer * per_layer;
    const Idx head = rem / vph;
    gather_unit(a, int64_t(r), int(layer), int(head), int(rem - head * vph));
  }
}

kvtc_status launch_gather(const kvtc_kv_view &v, __nv_bfloat16 *const *layer_base_dev, int64_t tok_begin,
                          int64_t ntok, const float2 *cs, int32_t pairing, __nv_bfloat16 *X, cudaStream_t st,
                          int32_t max_ctas, int64_t ldx) {
  GatherArgs a;
  a.bases = layer_base_dev;
  a.layout = v.layout;
  a.page_tokens = v.page_tokens;
  a.block_table = v.block_table;
  a.layers = v.shape.layers;
  a.heads = v.shape.kv_heads;
  a.d = v.shape.head_dim;
  a.pairing = pairing;
  a.tok_begin = tok_begin;
  a.ntok = ntok;
  a.cs = cs;
  a.X = X;
  a.ldx = ldx > 0 ? ldx : int64_t(v.shape.layers) * v.shape.kv_heads * v.shape.head_dim;
  const int64_t total = ntok * v.shape.layers * v.shape.kv_heads * (v.shape.head_dim / 16);
  if (total == 0) return KVTC_OK;
  int64_t grid = ceil_div(total, 256);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  grid = std::min<int64_t>(grid, int64_t(1) << 30);
  if (total < (int64_t(1) << 32) - int64_t(grid) * 256) {
    KVTC_MAX_CARVEOUT(gather_kernel<uint32_t>);
    gather_kernel<uint32_t><<<unsigned(grid), 256, 0, st>>>(a, uint32_t(total));
  } else {
    KVTC_MAX_CARVEOUT(gather_kernel<uint64_t>);
    gather_kernel<uint64_t><<<unsigned(grid), 256, 0, st>>>(a, uint64_t(total));
  }
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

// Calibration gather: rows (seq, tok) from several views, un-RoPE computed inline.
struct SeqInfo {
  int64_t pos0;
  int32_t layout, page_tokens;
  const int32_t *block_table;
  __nv_bfloat16 *const *bases;  // device array [layers]
};

// cos/sin of every sampled row's absolute position (R1 table, one entry per (row, j))
__global__ void rows_rope_table_kernel(const SeqInfo *seqs, const int64_t *rows, int64_t n, int half,
                                       const float *invf, float2 *cs) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n * half) return;
  const int64_t r = i / half;
  const int j = int(i % half);
  const float pos = float(seqs[rows[2 * r]].pos0 + rows[2 * r + 1]);
  const float theta = __fmul_rn(pos, invf[j]);
  double s, c;
  sincos(double(theta), &s, &c);
  cs[i] = make_float2(__double2float_rn(c), __double2float_rn(s));
}

// one thread = one rotation pair (or two plain elements) of one sampled row
__global__ void gather_rows_kernel(const SeqInfo *seqs, const int64_t *rows, int64_t n, int layers, int heads, int d,
                                   const float2 *cs, int pairing, int64_t ld, __nv_bfloat16 *X) {
  const int64_t p = int64_t(layers) * heads * d;
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n * (p / 2)) return;
  const int64_t r = i / (p / 2);
  const int64_t q = i % (p / 2);
  const int layer = int(q / (heads * (d / 2)));
  const int head = int((q / (d / 2)) % heads);
  const int j = int(q % (d / 2));
  const SeqInfo s = seqs[rows[2 * r]];
  const int64_t tok = rows[2 * r + 1];
  const int64_t slot = view_slot(s.layout, s.page_tokens, s.block_table, tok);
  const __nv_bfloat16 *src = s.bases[layer] + slot * (int64_t(heads) * d) + head * d;
  const int i1 = pairing == 0 ? j : 2 * j;
  const int i2 = pairing == 0 ? j + d / 2 : 2 * j + 1;
  __nv_bfloat16 o1 = src[i1], o2 = src[i2];
  if (cs) unrope_pair(__bfloat162float(o1), __bfloat162float(o2), cs[r * (d / 2) + j], o1, o2);
  __nv_bfloat16 *dst = X + r * ld + int64_t(layer) * heads * d + head * d;
  dst[i1] = o1;
  dst[i2] = o2;
}

kvtc_status launch_gather_rows(const kvtc_kv_view *seqs, int32_t nseq, __nv_bfloat16 *const *bases_dev,
                               const int64_t *rows_dev, int64_t n, const float *invf_dev, int32_t unrope,
                               int32_t pairing, int64_t ld, __nv_bfloat16 *X, cudaStream_t st) {
  // bases_dev: device array [nseq * layers]
  std::vector<SeqInfo> h(nseq);
  const int L = seqs[0].shape.layers;
  for (int i = 0; i < nseq; ++i) {
    h[i].pos0 = seqs[i].pos0;
    h[i].layout = seqs[i].layout;
    h[i].page_tokens = seqs[i].page_tokens;
    h[i].block_table = seqs[i].block_table;
    h[i].bases = bases_dev + int64_t(i) * L;
  }
  const kvtc_shape &sh = seqs[0].shape;
  const int half = sh.head_dim / 2;
  SeqInfo *d_info = nullptr;
  float2 *cs = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&d_info, sizeof(SeqInfo) * nseq, st));
  // pageable -> device: returns once the source has been staged, so h may go out of scope
  KVTC_CUDA_TRY(cudaMemcpyAsync(d_info, h.data(), sizeof(SeqInfo) * nseq, cudaMemcpyHostToDevice, st));
  if (unrope && n > 0) {
    KVTC_CUDA_TRY(cudaMallocAsync(&cs, sizeof(float2) * n * half, st));
    rows_rope_table_kernel<<<unsigned(ceil_div(n * half, 256)), 256, 0, st>>>(d_info, rows_dev, n, half, invf_dev, cs);
    KVTC_LAUNCH_CHECK();
  }
  const int64_t total = n * (int64_t(sh.layers) * sh.kv_heads * sh.head_dim / 2);
  if (total > 0) {
    gather_rows_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, st>>>(d_info, rows_dev, n, sh.layers, sh.kv_heads,
                                                                        sh.head_dim, cs, pairing, ld, X);
    KVTC_LAUNCH_CHECK();
  }
  if (cs) cudaFreeAsync(cs, st);
  cudaFreeAsync(d_info, st);
  return KVTC_OK;
}

// ------------------------------------------------------- SIMT quantise + pack
// Block = one payload tile (128 tokens) x one segment; thread = token row.
__global__ void __launch_bounds__(128) quant_pack_simt_kernel(const SegDesc *segs, const GroupDesc *groups,
                                                              const float *D, int64_t ldd, int64_t m,
                                                              int64_t tile_bytes, const int64_t *codes_off_last,
                                                              uint8_t *payload) {
  const SegDesc sd = segs[blockIdx.x];
  const int row = threadIdx.x;
  const int lane = row & 31;
  const int64_t m0 = int64_t(blockIdx.y) * kTileM;
  const int64_t tok = m0 + row;
  const bool valid = tok < m;
  const int ntok = int(m - m0 < kTileM ? m - m0 : kTileM);
  const bool last = ntok < kTileM;
  uint8_t *tile_base = payload + blockIdx.y * tile_bytes;
  const float *xr = D + (valid ? tok : 0) * ldd + sd.col0;
  for (int gi = sd.g_begin; gi < sd.g_end; ++gi) {
    const GroupDesc gd = groups[gi];
    const float *xg = xr + gd.col - gd.part * gd.size;
    float mn = xg[0], mx = xg[0];
    for (int c = 1; c < gd.full_size; ++c) {
      mn = fminf(mn, xg[c]);
      mx = fmaxf(mx, xg[c]);
    }
    uint8_t *cb = tile_base + (last ? codes_off_last[gd.gidx] : gd.codes_off);
    emit_group(xr + gd.col, gd.size, gd.full_size, gd.part, gd.type, gd.gidx, mn, mx, valid, row, lane, row & ~31,
               ntok, last, tile_base, cb);
  }
}

// ------------------------------------------------- wide groups (size k*256)
// Block = one payload tile x one wide group; warp per token row: coalesced
// float4 reads of the row's fp32 coefficients, warp min/max, then lane j packs
// code words j, j+32, ... (Q2/Q3/Q5, R3/R4 via quant.cuh).
__device__ __forceinline__ float4 load4(const float *p, bool vec) {
  return vec ? *reinterpret_cast<const float4 *>(p) : make_float4(p[0], p[1], p[2], p[3]);
}

__global__ void __launch_bounds__(128) quant_wide_kernel(const WideDesc *wide, const float *D, int64_t ldd,
                                                         int use_wcol, int64_t m, int64_t tile_bytes,
                                                         const int64_t *codes_off_last, uint8_t *payload,
                                                         const TileRef *tiles, int32_t *status) {
  const WideDesc wd = wide[blockIdx.x];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t m0 = int64_t(blockIdx.y) * kTileM;
  const TileRef *tref = tiles ? tiles + blockIdx.y : nullptr;
  const int ntok = tref ? tref->ntok : int(m - m0 < kTileM ? m - m0 : kTileM);
  const bool last = ntok < kTileM;
  uint8_t *tile_base = tref ? tref->payload : payload + blockIdx.y * tile_bytes;
  uint8_t *cb = tile_base + (last ? (tref ? tref->codes_off : codes_off_last)[wd.gidx] : wd.codes_off);
  const int b = bits_of(wd.type);
  const int per_word = 32 / b;
  const int words = wd.size * b / 32;
  const int64_t tok_bytes = int64_t(wd.size) * b / 8;
  for (int r = warp; r < ntok; r += 4) {
    const float *x = D + (m0 + r) * ldd + (use_wcol ? wd.wcol : wd.col);
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    float mn = INFINITY, mx = -INFINITY;
    for (int c = 4 * lane; c < wd.size; c += 128) {
      const float4 v = load4(x + c, vec);
      mn = fminf(fminf(mn, v.x), fminf(fminf(v.y, v.z), v.w));
      mx = fmaxf(fmaxf(mx, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    uint16_t sh, sc;
    group_factors(wd.type, mn, mx, sh, sc);
    const float shift = f16_val(sh), scale = f16_val(sc);
    if (lane == 0) {
      uint8_t *pp = tile_base + 4 * (int64_t(wd.gidx) * ntok + r);
      store_u32_any(pp, uint32_t(sh) | (uint32_t(sc) << 16), (reinterpret_cast<uintptr_t>(pp) & 3) == 0);
      int32_t *stw = tref ? tref->status : status;
      if (stw && factor_overflow(sh, sc)) atomicOr(stw, 1);
    }
    uint8_t *dst = cb + int64_t(r) * tok_bytes;
    const bool al = (reinterpret_cast<uintptr_t>(dst) & 3) == 0;
    for (int w = lane; w < words; w += 32) {
      uint32_t word = 0;
      for (int j = 0; j < per_word; j += 4) {
        const float4 v = load4(x + w * per_word + j, vec);
        word |= encode_one(wd.type, v.x, shift, scale) << (j * b);
        word |= encode_one(wd.type, v.y, shift, scale) << ((j + 1) * b);
        word |= encode_one(wd.type, v.z, shift, scale) << ((j + 2) * b);
        word |= encode_one(wd.type, v.w, shift, scale) << ((j + 3) * b);
      }
      store_u32_any(dst + 4 * w, word, al);
    }
  }
}

kvtc_status launch_quant_wide(const WideDesc *wide, int32_t nwide, const float *D, int64_t ldd, int use_wcol,
                              int64_t m, int64_t tile_bytes, const int64_t *codes_off_last, uint8_t *payload,
                              cudaStream_t st, const TileRef *tiles, int32_t *status) {
  if (nwide == 0 || m == 0) return KVTC_OK;
  dim3 grid(unsigned(nwide), unsigned(ceil_div(m, kTileM)));
  KVTC_MAX_CARVEOUT(quant_wide_kernel);             // may run beside a GEMM (values' wide groups)
  quant_wide_kernel<<<grid, 128, 0, st>>>(wide, D, ldd, use_wcol, m, tile_bytes, codes_off_last, payload, tiles,
                                          status);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_quant_pack_simt(const SegDesc *segs, const GroupDesc *groups, int32_t nsegs, int32_t G,
                                   const float *D, int64_t ldd, int64_t m, int64_t tile_bytes,
                                   const int64_t *codes_off_last, uint8_t *payload, cudaStream_t st) {
  (void)G;
  if (nsegs == 0 || m == 0) return KVTC_OK;
  dim3 grid(unsigned(nsegs), unsigned(ceil_div(m, kTileM)));
  quant_pack_simt_kernel<<<grid, 128, 0, st>>>(segs, groups, D, ldd, m, tile_bytes, codes_off_last, payload);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

// ---------------------------------------------------------------- dequant
// D2 (R5): D^ [m][ld] fp16 from the payload, 32 rows x 32 8-column chunks per
// block of 8 warps (dequant_block, dequant.cuh: dq8's 1024 + c bit trick and
// fma.rn.f16x2 round the exact x^ once).  Grid-stride over blocks (bounded grid
// beside a GEMM).  The decompression path itself runs the same blocks inside the
// inflater (inflate_dequant_kernel, deflate.cu); this kernel serves the stage
// API, layer-streamed and batched decompression.
__global__ void __launch_bounds__(256) dequant_rows_kernel(const DqChunk *chunks, const DqCol *cols, int32_t nch8,
                                                           const int64_t *codes_off_full,
                                                           const int64_t *codes_off_last, int64_t tile_bytes,
                                                           const uint8_t *payload, int64_t m, __half *Dh, int64_t ld) {
  const int64_t nbx = (nch8 + 31) / 32, nby = (m + 31) / 32;
  const DqArgs a{chunks, cols, nch8, codes_off_full, codes_off_last, tile_bytes, payload, m, Dh, ld};
  for (int64_t blk = blockIdx.x; blk < nbx * nby; blk += gridDim.x) {
    const int64_t by = blk / nbx;
    dequant_block<8>(a, by, blk - by * nbx, threadIdx.x, threadIdx.y);
  }
}

kvtc_status launch_dequant(const DqChunk *chunks, const DqCol *cols, int32_t r_nz, const int64_t *codes_off_full,
                           const int64_t *codes_off_last, int64_t tile_bytes, const uint8_t *payload, int64_t m,
                           __half *Dh, int64_t ld, cudaStream_t st, int32_t max_ctas) {
  if (r_nz == 0 || m == 0) return KVTC_OK;
  KVTC_CHECK_ARG(ld % 8 == 0 && ld >= (r_nz + 7) / 8 * 8, "D^ leading dimension");
  KVTC_CHECK_ARG((reinterpret_cast<uintptr_t>(Dh) & 15) == 0, "D^ must be 16-byte aligned");
  const int32_t nch8 = (r_nz + 7) / 8;
  int64_t grid = ceil_div(nch8, 32) * ceil_div(m, 32);
  if (max_ctas > 0) grid = std::min<int64_t>(grid, max_ctas);
  grid = std::min<int64_t>(grid, int64_t(1) << 30);
  KVTC_MAX_CARVEOUT(dequant_rows_kernel);
  dequant_rows_kernel<<<unsigned(grid), dim3(32, 8), 0, st>>>(chunks, cols, nch8, codes_off_full, codes_off_last,
                                                              tile_bytes, payload, m, Dh, ld);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

// ------------------------------------------------------------ raw tokens
// flat buffer [layers][ntok][h*d] <-> view tokens
__global__ void raw_copy_kernel(__nv_bfloat16 *const *bases, int32_t layout, int32_t page_tokens,
                                const int32_t *block_table, int64_t view_tok0, __nv_bfloat16 *flat,
                                int64_t flat_ntok, int64_t flat_tok0, int64_t ntok, int32_t layer0, int32_t nlayers,
                                int32_t hd, int32_t to_flat) {
  const int vec = hd / 8;
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= int64_t(nlayers) * ntok * vec) return;
  const int v = int(i % vec);
  const int64_t r = (i / vec) % ntok;
  const int layer = layer0 + int(i / (int64_t(vec) * ntok));
  const int64_t slot = view_slot(layout, page_tokens, block_table, view_tok0 + r);
  uint4 *vp = reinterpret_cast<uint4 *>(bases[layer] + slot * hd) + v;
  uint4 *fp = reinterpret_cast<uint4 *>(flat + (int64_t(layer) * flat_ntok + flat_tok0 + r) * hd) + v;
  if (to_flat) *fp = *vp;
  else *vp = *fp;
}

kvtc_status launch_pack_raw(const kvtc_kv_view &src, __nv_bfloat16 *const *bases, int64_t tok, int64_t ntok,
                            __nv_bfloat16 *dst, int64_t flat_ntok, int64_t flat_tok0, cudaStream_t st) {
  const int hd = src.shape.kv_heads * src.shape.head_dim;
  const int64_t total = int64_t(src.shape.layers) * ntok * (hd / 8);
  if (total == 0) return KVTC_OK;
  raw_copy_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, st>>>(bases, src.layout, src.page_tokens, src.block_table,
                                                                   tok, dst, flat_ntok, flat_tok0, ntok, 0,
                                                                   src.shape.layers, hd, 1);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_unpack_raw(const __nv_bfloat16 *src, int64_t ntok_total, int64_t src_tok0, int64_t ntok,
                              const kvtc_kv_view &dst, __nv_bfloat16 *const *bases, int64_t dst_tok,
                              int32_t layer_begin, int32_t layer_end, cudaStream_t st) {
  const int hd = dst.shape.kv_heads * dst.shape.head_dim;
  const int64_t total = int64_t(layer_end - layer_begin) * ntok * (hd / 8);
  if (total == 0) return KVTC_OK;
  raw_copy_kernel<<<unsigned(ceil_div(total, 256)), 256, 0, st>>>(
      bases, dst.layout, dst.page_tokens, dst.block_table, dst_tok, const_cast<__nv_bfloat16 *>(src), ntok_total,
      src_tok0, ntok, layer_begin, layer_end - layer_begin, hd, 0);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

}  // namespace kvtc
