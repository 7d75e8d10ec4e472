// internal.h — host-side objects and kernel launchers shared by the library's
// translation units (not part of the ABI).
#pragma once

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace kvtc {

// One non-None group of a plan (PC order).  `col` is the column in the
// compacted operand space (non-None PCs only, in order).
struct PlanGroup {
  int32_t start, size, type, col;
};

// Device descriptor of one piece of a group handled by one GEMM tile.
struct GroupDesc {
  int32_t col;        // first column inside the tile (0..255)
  int32_t size;       // columns of this piece (<= 256)
  int32_t full_size;  // group size (pieces of a split group: size * parts)
  int32_t type;       // kvtc_type
  int32_t gidx;       // index of the group among non-None groups (params slot)
  int32_t part;       // piece index inside a split group
  int64_t codes_off;  // byte offset of the group's code block in a FULL tile
};
struct SegDesc {
  int32_t col0;       // first compacted column of the tile
  int32_t width;      // columns used
  int32_t g_begin, g_end;  // GroupDesc range
  int32_t f32_col;    // >= 0: a 256-column piece of a wide group; the epilogue
                      // stores D - mu V_c (fp32) at this column of the wide scratch
  int32_t wide;       // wide pieces: index of the group in the plan's WideDesc table, else -1
};
// A group wider than one tile (size = k * 256).  Each of its k pieces is a GEMM
// tile whose epilogue stores fp32 coefficients + the row min/max of the piece to
// a scratch; the epilogue of the piece that completes last (an arrival counter
// per (M-block, group)) quantises and packs the whole group (SIMT reference:
// quant_wide_kernel).
struct WideDesc {
  int32_t gidx;       // index among non-None groups (params slot)
  int32_t size, type;
  int32_t col;        // compacted column (D [m x r_nz])
  int32_t wcol;       // column in the wide scratch [m x wide_cols]
  int32_t pad;
  int64_t codes_off;  // code block offset in a FULL tile
};

// One column of the decompress GEMM's A operand (a compacted non-None PC) for the
// dequantising producer of the fused inverse path (D2 inside K5):
// the producer warps read codes + fp16 factors from the payload and write the
// fp16 A tile straight into shared memory.
struct DqCol {
  uint16_t gidx;      // group among non-None groups (params slot / code block)
  uint8_t type;       // kvtc_type; 0 = padding column past r_nz (A = 0)
  uint8_t chunk;      // 1: columns [c, c + 8) are elements j .. j + 7 (j % 8 == 0) of this group
  uint16_t j;         // element index inside the group
  uint16_t size;      // group size
  int32_t off_full;   // byte offset of the group's code block in a FULL tile
  int32_t pad;
};

// One 16-byte chunk (8 columns) of D^ (dequantiser, and per pipeline position
// the fused producer's shared-memory table): ok = 1 when the 8 columns are
// elements j .. j+7 (j % 8 == 0) of one group (byte offsets of a FULL tile); ok = 3
// for the other chunks with columns (code_base = 16 * its index in the fused
// producer's tail buffer).  run_code >= 0 marks an ok = 3 chunk whose columns are
// 8 consecutive size-1 groups of one type (the DP's per-PC groups): group q's
// code block starts at run_code + q * run_stride, its factors at par_base + q * 512.
struct DqChunk {
  int32_t code_base;  // group code block + j * bits / 8
  int32_t par_base;   // 4 * gidx * 128 (params of token 0)
  uint16_t stride;    // ok = 1: code bytes per token (size * bits / 8); runs: run_stride (16 * bits)
  uint8_t type;       // kvtc_type of the chunk's group (0: padding)
  uint8_t ok;
  int32_t run_code;   // -1, or the first code block of a size-1 run (FULL tile)
};
constexpr int kDqTabMaxBytes = 32 * 1024;   // shared-memory budget of the chunk table (16384 columns)

// Batched codec (kvtc_compress_batch / kvtc_decompress_batch): ONE GEMM over the
// concatenated rows of several conversations, each padded to whole 128-token
// tiles; tile mb of the GEMM refers to one tile of one conversation.
struct TileRef {
  uint8_t *payload;                 // this tile's payload bytes (compress: written; decompress: read by K5)
  const int64_t *codes_off;         // code-block offsets (full or partial tile)
  __nv_bfloat16 *const *bases;      // decompress: the conversation's device layer-base array
  const int32_t *block_table;       // decompress: paged layout
  int64_t tok0;                     // decompress: cache token of the tile's first row
  int32_t ntok;                     // valid rows (<= 128)
  int32_t layout, page_tokens;      // decompress: output view layout
  int32_t pad;
  int32_t *status;                  // compress: the item's status word (Q4 overflow bit), nullable
};

// Operands of a (basis, plan) pair, compacted to the plan's non-None PCs.
struct Operands {
  int32_t r_nz = 0, r_nz_pad = 0;
  __nv_bfloat16 *VcT = nullptr;  // [r_nz x (p + kXPad)]  rows = PCs (compress B operand, K-major)
  float *bias = nullptr;         // [r_nz] mu V_c (fp32)
  __half *Vd = nullptr;          // [p x r_nz_pad] (decompress B operand, K-major)
  CUtensorMap tm_VcT, tm_Vd;
  bool ready = false;
};

struct kvtc_basis_impl;
struct kvtc_plan_impl;

// CUDA driver entry point for cuTensorMapEncodeTiled (no libcuda link needed)
kvtc_status make_tmap_2d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                         uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer);
// 3-D map {d0, d1, d2} (strides of dims 1, 2 in bytes), box {box0, box1, 1}:
// the per-layer contiguous cache [layers][tokens][h*d] read in place.
kvtc_status make_tmap_3d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, uint64_t d0, uint64_t d1,
                         uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1);

// ------------------------------------------------------------------ launchers
// Scratch of the wide groups of a compress GEMM over m rows: fp32 coefficients
// [m x wide_cols], per-piece row min/max [m x wide_cols/256] float2, arrival
// counters [ceil(m/128) x nwide] int32.
inline size_t wide_scratch_bytes(int64_t m, int32_t wide_cols, int32_t nwide) {
  if (!nwide || !m) return 0;
  return size_t(m) * wide_cols * 4 + size_t(m) * (wide_cols / kMaxTileN) * 8 + size_t(ceil_div(m, kTileM)) * nwide * 4 +
         256;
}

struct GemmCompressArgs {
  const CUtensorMap *tmA;  // X [m x p] bf16, box {64, 128}
  const CUtensorMap *tmB;  // VcT [r_nz x p] bf16, box {64, 128}
  int32_t K;               // p
  int64_t m;
  const float *bias;       // [r_nz]
  // mode F32: D [m x ldd]; mode quantise: the wide-group scratch [m x ldd]
  float *D;
  int64_t ldd;
  // mode quantise
  uint8_t *payload;
  const SegDesc *segs;
  const GroupDesc *groups;
  int32_t nsegs;
  int32_t G;               // number of non-None groups
  int64_t tile_bytes;      // bytes of a full tile
  const int64_t *codes_off_last;  // [G] code-block offsets of the last partial tile
  // a_hd > 0: tmA is the 3-D map {hd, tokens, layers} of a contiguous cache and
  // row r of X is token a_row0 + r (k-block kb = layer kb*64/hd, column kb*64%hd)
  int32_t a_hd;
  int64_t a_row0;
  int64_t a_layer_rows;    // a_hd > 0 and a_layer_rows > 0: tmA is a 2-D map over [layers * tokens][h*d]
  const TileRef *tiles;    // non-null: batched rows (tile mb -> tiles[mb]); payload / m unused
  int32_t *status;         // nullable: bit 0 set when an fp16 shift / scale overflowed (Q4)
  // wide groups (quantised in the epilogue of their last piece): D is the scratch
  // of wide_scratch_bytes(m, ldd, nwide) bytes
  const WideDesc *wide;
  int32_t nwide;
};
kvtc_status launch_gemm_project_f32(const GemmCompressArgs &a, int32_t ncols, cudaStream_t st);
kvtc_status launch_gemm_project_quant(const GemmCompressArgs &a, cudaStream_t st);

struct GemmDecompressArgs {
  const CUtensorMap *tmA;  // D^ [m x r_nz_pad] fp16, box {64, 128}
  const CUtensorMap *tmB;  // Vd [p x r_nz_pad] fp16, box {64, 128}
  int32_t K;               // r_nz_pad
  int64_t m;
  int32_t n_begin, n_end;  // feature range (multiple of 256)
  const float *mu;         // [p]
  const float2 *cs;        // [m x d/2] cos/sin (keys) or nullptr
  int32_t layers, heads, head_dim, pairing;
  // output view
  int32_t layout, page_tokens;
  __nv_bfloat16 *const *layer_base;  // device array [layers]
  const int32_t *block_table;
  int64_t tok_begin;                 // cache token index of row 0
  int32_t tile_n;                    // N tile (<= 256, divides heads*head_dim)
  const TileRef *tiles;              // non-null: batched rows; the output view comes from tiles[mb]
  // fused inverse path (payload != nullptr or tiles != nullptr with dqcols): A = D^ is
  // dequantised from the payload inside the GEMM (tmA unused)
  const uint8_t *payload;            // m rows of 128-token payload tiles
  const int64_t *codes_off_full, *codes_off_last;
  int64_t tile_bytes;
  const DqCol *dqcols;               // [ceil(K / 128) * 128]; non-null selects the fused path
  const DqChunk *dqchunks;           // [ceil(K / 128) * 16]
  const int32_t *tail_cols;          // [n_tail] first column of each ok = 3 chunk
  int32_t n_tail;
  uint8_t *dq_tail;                  // [ceil(m / 128) * 128][n_tail * 16 B] pre-pass output
};
// Bytes of the fused path's tail buffer for m rows.
inline size_t dq_tail_bytes(int64_t m, int32_t n_tail) { return size_t(ceil_div(m, kTileM)) * kTileM * n_tail * 16; }
kvtc_status launch_gemm_reconstruct(const GemmDecompressArgs &a, cudaStream_t st);

// XtX accumulation: S[p x p] += C^T C for a chunk Ct [p x nk] (K-major);
// tmA and tmB: box {64, 128} over the same Ct.
kvtc_status launch_gemm_xtx(const CUtensorMap *tmA, const CUtensorMap *tmB, int32_t p, int32_t nk, float *S,
                            cudaStream_t st);

// elementwise.cu
kvtc_status launch_rope_table(const float *invf_dev, int32_t half, int64_t pos_first, int64_t n, float2 *cs,
                              cudaStream_t st);
kvtc_status launch_gather(const kvtc_kv_view &v, __nv_bfloat16 *const *layer_base_dev, int64_t tok_begin,
                          int64_t ntok, const float2 *cs, int32_t pairing, __nv_bfloat16 *X, cudaStream_t st,
                          int32_t max_ctas = 0, int64_t ldx = 0);   // ldx 0: dense rows (p)
kvtc_status launch_gather_rows(const kvtc_kv_view *seqs, int32_t nseq, __nv_bfloat16 *const *bases_dev,
                               const int64_t *rows_dev, int64_t n, const float *invf_dev, int32_t unrope,
                               int32_t pairing, int64_t ld, __nv_bfloat16 *X, cudaStream_t st);
// Wide groups: D [m x ldd] fp32; column of group w = use_wcol ? wcol : col.
kvtc_status launch_quant_wide(const WideDesc *wide, int32_t nwide, const float *D, int64_t ldd, int use_wcol, int64_t m,
                              int64_t tile_bytes, const int64_t *codes_off_last, uint8_t *payload, cudaStream_t st,
                              const TileRef *tiles = nullptr, int32_t *status = nullptr);
kvtc_status launch_quant_pack_simt(const SegDesc *segs, const GroupDesc *groups, int32_t nsegs, int32_t G,
                                   const float *D, int64_t ldd, int64_t m, int64_t tile_bytes,
                                   const int64_t *codes_off_last, uint8_t *payload, cudaStream_t st);
kvtc_status launch_codes_off_last(const int32_t *gsize, const int32_t *gbits, int32_t G, int32_t ntok,
                                  int64_t *out, cudaStream_t st);
// D2 operands of one stream (dequant_rows_kernel, inflate_dequant_kernel).
struct DqArgs {
  const DqChunk *chunks;
  const DqCol *cols;
  int32_t nch8;                         // 8-column chunks of D^ (ceil(r_nz / 8))
  const int64_t *codes_off_full, *codes_off_last;
  int64_t tile_bytes;
  const uint8_t *payload;
  int64_t m;
  __half *Dh;
  int64_t ld;
};

// Fused inverse front end (inflate_dequant_kernel, deflate.cu): one launch
// inflates the chunks of both sections and dequantises each 32-row block of D^
// as soon as every chunk of its tile is inflated (per-tile arrival counters).
struct InflateDqStream {
  const uint8_t *sec;
  uint64_t sec_len, n_out;
  uint32_t nch;
  uint8_t *out;                          // the inflated payload
  DqArgs dq;                             // dq.payload == out
  uint32_t ndq, nbx;                     // dequant items (tiles x nbx; 0: inflate only), 32-chunk blocks
  uint32_t *tile_done;                   // [ceil(m / 128)] inflated chunks per tile (zeroed)
};
struct InflateDqArgs {
  InflateDqStream s[2];
  uint32_t cb_shift;                     // log2 of the chunk bytes (16 / 32 / 64 KiB)
  uint32_t *ctr;                         // [0] next chunk item, [1] next dequant item (zeroed)
  int32_t *err;
};
kvtc_status launch_inflate_dequant(const InflateDqArgs &a, cudaStream_t st);

// D2: D^ [m x ld] fp16 (ld % 8 == 0, >= r_nz rounded up to 8; 16-byte aligned)
// from m tokens of payload, with the plan's chunk / column tables (api.cu).
kvtc_status launch_dequant(const DqChunk *chunks, const DqCol *cols, int32_t r_nz, const int64_t *codes_off_full,
                           const int64_t *codes_off_last, int64_t tile_bytes, const uint8_t *payload, int64_t m,
                           __half *Dh, int64_t ld, cudaStream_t st, int32_t max_ctas = 0);
kvtc_status launch_copy_tokens(const kvtc_kv_view &src, __nv_bfloat16 *const *src_bases, int64_t src_tok,
                               const kvtc_kv_view &dst, __nv_bfloat16 *const *dst_bases, int64_t dst_tok,
                               int64_t ntok, int32_t layer_begin, int32_t layer_end, cudaStream_t st);
// raw token rows packed as [layers][ntok][h*d] in a flat buffer
kvtc_status launch_pack_raw(const kvtc_kv_view &src, __nv_bfloat16 *const *bases, int64_t tok, int64_t ntok,
                            __nv_bfloat16 *dst, int64_t flat_ntok, int64_t flat_tok0, cudaStream_t st);
kvtc_status launch_unpack_raw(const __nv_bfloat16 *src, int64_t ntok_total, int64_t src_tok0, int64_t ntok,
                              const kvtc_kv_view &dst, __nv_bfloat16 *const *bases, int64_t dst_tok,
                              int32_t layer_begin, int32_t layer_end, cudaStream_t st);

// deflate.cu
size_t deflate_section_bound(size_t n, int32_t chunk);
size_t deflate_workspace(size_t n, int32_t chunk);
// Writes the section (header, chunk table, index, data) to out; sizes on device;
// *section_len_dev receives the section length (device uint64).
// The section is written at out + (off_dev ? *off_dev : 0) (device offset).
kvtc_status launch_deflate(const uint8_t *in, size_t n, int32_t chunk, uint8_t *out, const uint64_t *off_dev,
                           uint64_t *section_len_dev, void *ws, size_t ws_bytes, cudaStream_t st);
// Two phases of launch_deflate: chunk encoder into the workspace slots (max_ctas
// > 0 bounds the grid so the kernel can run beside a persistent GEMM), then the
// section layout + copy to out (workspace untouched in between).
kvtc_status launch_deflate_encode(const uint8_t *in, size_t n, int32_t chunk, void *ws, size_t ws_bytes,
                                  int32_t max_ctas, cudaStream_t st, uint32_t c_begin = 0,
                                  uint32_t c_end = 0xFFFFFFFFu);   // chunk range [c_begin, c_end)
kvtc_status launch_deflate_assemble(size_t n, int32_t chunk, const void *ws, uint8_t *out, const uint64_t *off_dev,
                                    uint64_t *section_len_dev, cudaStream_t st);
// Batched codec: one payload's DEFLATE job (its own workspace of
// deflate_workspace(n) bytes; chunk0 = first global chunk, ascending).
struct EncodeJob {
  const uint8_t *in;
  uint64_t n;
  void *ws;
  uint32_t chunk0, pad;
};
kvtc_status launch_deflate_encode_batch(const EncodeJob *jobs_dev, int32_t njobs, uint32_t total_chunks,
                                        int32_t chunk, cudaStream_t st, int32_t max_ctas = 0);
// SM count x per_sm: the bounded grid of a side-stream kernel overlapping a GEMM.
int corun_ctas(int per_sm);
// Kernels that share an SM must run under the same shared-memory carveout: the
// persistent GEMMs (196 KB) and every kernel that overlaps them on the side
// stream request the maximum (228 KB), which leaves 32 KB next to a GEMM CTA.
// (Without it ncu shows 196 / 32 / 228 KB configs and the side kernels wait for
// the GEMM to finish.)
#define KVTC_MAX_CARVEOUT(kernel)                                                                     \
  do {                                                                                              \
    static const bool kvtc_carveout_set_ = (cudaFuncSetAttribute(reinterpret_cast<const void *>(kernel), \
                                                                 cudaFuncAttributePreferredSharedMemoryCarveout, \
                                                                 int(cudaSharedmemCarveoutMaxShared)),  \
                                            true);                                                  \
    (void)kvtc_carveout_set_;                                                                       \
  } while (0)
// Inflate one section (sec: device pointer, len: bytes the section may occupy;
// every read stays inside [sec, sec + len)); *err != 0 afterwards = corrupt.
kvtc_status launch_inflate_section(const uint8_t *sec, uint64_t len, uint64_t n_out, uint32_t nchunks, uint8_t *out,
                                   int32_t *err, cudaStream_t st, int32_t max_ctas = 0);
kvtc_status check_section_header(const void *hdr_host, size_t len, size_t n_out, uint32_t *nchunks);
// Both streams' sections in one launch (two warps per chunk).
kvtc_status launch_inflate_sections(const uint8_t *sec0, uint64_t len0, uint64_t n0, uint32_t nch0, uint8_t *out0,
                                    const uint8_t *sec1, uint64_t len1, uint64_t n1, uint32_t nch1, uint8_t *out1,
                                    int32_t *err, cudaStream_t st, int32_t max_ctas = 0);
constexpr size_t kSectionHeaderBytes = 64;
// One section of a batched inflate (device table, chunk0 ascending).
struct InflateJob {
  const uint8_t *section;
  uint64_t sec_len;                // bytes the section may occupy
  uint64_t n_out;
  uint32_t nch, chunk0;
  uint8_t *out;
  int32_t *err;                    // this job's error word (nullable: the launch's)
};
kvtc_status launch_inflate_batch(const InflateJob *jobs_dev, int32_t njobs, uint32_t total_chunks, int32_t *err,
                                 cudaStream_t st);
kvtc_status launch_inflate_raw(const uint8_t *in, const int64_t *in_off, const int64_t *in_len, int32_t n,
                               uint8_t *out, const int64_t *out_off, const int64_t *out_len, int32_t *status,
                               cudaStream_t st);

// rans.cu: the static-model interleaved rANS back-end (reading Q24).  Encode
// writes a section at out + (*off_dev) like launch_deflate; decode needs
// rans_decode_workspace(nclasses) bytes of device scratch (the decoder tables).
size_t rans_section_bound(size_t n, int32_t chunk, int64_t tile_bytes);
size_t rans_workspace(size_t n, int32_t chunk, int64_t tile_bytes);
kvtc_status launch_rans_encode(const uint8_t *in, size_t n, int32_t chunk, int64_t tile_bytes, uint8_t *out,
                               const uint64_t *off_dev, uint64_t *section_len_dev, void *ws, size_t ws_bytes,
                               cudaStream_t st);
kvtc_status check_rans_header(const void *hdr_host, size_t len, size_t n_out, uint32_t *nchunks, uint32_t *nclasses);
size_t rans_decode_workspace(uint32_t nclasses);
kvtc_status launch_rans_decode(const uint8_t *sec, uint64_t len, uint64_t n_out, uint32_t nchunks, uint32_t nclasses,
                               uint8_t *out, void *ws, int32_t *err, cudaStream_t st);
constexpr size_t kRansHeaderBytes = 64;
constexpr uint32_t kRansMaxClasses = 64;          // span_log2 is chosen so a tile has <= 64 classes

// integrity.cu: 64-bit container checksums (see the file header).  launch_hash
// ADDS the checksum of [p, p + n) (p 16-byte aligned) to *out (zero it first);
// launch_hash_check ORs `bit` into *status when *got != expect.
constexpr uint64_t kSeedPayload = 0x4B5654432D504159ull, kSeedRaw = 0x4B5654432D524157ull,
                   kSeedHeader = 0x4B5654432D484452ull;
uint64_t host_hash(const void *data, size_t n, uint64_t seed);
kvtc_status launch_hash(const void *p, uint64_t n, uint64_t seed, uint64_t *out, cudaStream_t st,
                        int32_t max_ctas = 0);
kvtc_status launch_hash_check(const uint64_t *got, uint64_t expect, int32_t bit, int32_t *status, cudaStream_t st);
// Batched: job j adds the checksum of [p, p + n) to *out (device table).
struct HashJob {
  const uint8_t *p;
  uint64_t n, seed;
  uint64_t *out;
};
kvtc_status launch_hash_batch(const HashJob *jobs_dev, int32_t njobs, uint64_t max_n, cudaStream_t st,
                              int32_t max_ctas = 0);
// status[j / per] |= bit_of(j % per) for every j with got[j] != expect[j] (device arrays).
kvtc_status launch_hash_check_batch(const uint64_t *got, const uint64_t *expect, int32_t njobs, int32_t per,
                                   int32_t *status, cudaStream_t st);

// Stage timing (kvtc_profile_*): records an event pair around a scope when enabled.
struct ProfScope {
  int slot = -1;
  cudaStream_t st;
  ProfScope(const char *name, cudaStream_t s);
  ~ProfScope();
};

}  // namespace kvtc
