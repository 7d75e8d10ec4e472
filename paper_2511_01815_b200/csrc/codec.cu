// codec.cu — stage entry points and the compress / decompress orchestration
// with the container format of DESIGN.md §4.
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "api_internal.h"

using namespace kvtc;

namespace {

constexpr uint32_t kContainerMagic = 0x4354564Bu;  // "KVTC"
constexpr uint32_t kContainerVersion = 2;
constexpr uint32_t kFlagNumeric = 1u;              // an fp16 shift / scale overflowed (Q4)
constexpr uint32_t kFlagRans = 2u;                 // sections are rANS (Q24), not DEFLATE

// DESIGN.md §4.  Integrity (integrity.cu): payload_hash = checksum of each
// stream's payload before DEFLATE, raw_hash = of the raw sink / window section,
// header_hash = of bytes [0, 248) of this header.
struct ContainerHeader {
  uint32_t magic, version;
  int32_t layers, kv_heads, head_dim, sinks, window, chunk_bytes;
  int64_t tokens, pos0, m;
  uint64_t total_bytes, raw_bytes;
  uint64_t payload_bytes[2], entropy_bytes[2];
  uint64_t basis_fp[2], plan_fp[2];
  uint64_t raw_off, section_off[2];
  uint32_t flags, reserved;
  uint64_t payload_hash[2], raw_hash;
  uint8_t pad[248 - 192];
  uint64_t header_hash;
};
static_assert(sizeof(ContainerHeader) == KVTC_HEADER_BYTES, "container header size");
static_assert(offsetof(ContainerHeader, header_hash) == 248, "header hash last");

// Device scratch words of one container written by compress (zeroed first):
// [0..1] section lengths K/V, [2..3] section offsets K/V (the values' section
// comes first: its DEFLATE finishes beside the keys' GEMM, so it is assembled
// there; the keys' section follows it), [4] status bits,
// [5..6] payload checksums K/V, [7] raw-section checksum.
constexpr int kCompressWords = 8;

// lens: nullable (passthrough container); aux = lens (see kCompressWords).
__global__ void header_kernel(ContainerHeader h, uint8_t *out, const uint64_t *lens, const uint64_t *w) {
  if (lens) {
    h.entropy_bytes[0] = lens[0];
    h.entropy_bytes[1] = lens[1];
    h.section_off[0] = lens[2];
    h.section_off[1] = lens[3];
    h.total_bytes = lens[2] + lens[0];
    h.payload_hash[0] = w[5];
    h.payload_hash[1] = w[6];
  }
  h.flags = (h.flags & kFlagRans) | ((w[4] & 1) ? kFlagNumeric : 0u);   // the coder flag comes from the host
  h.raw_hash = w[7];
  h.header_hash = hash_words(reinterpret_cast<const uint64_t *>(&h), 31, kSeedHeader);
  *reinterpret_cast<ContainerHeader *>(out) = h;
}
// next = 16-aligned end of the K section; the alignment gap is zeroed so the
// container bytes are a function of the input alone.
__global__ void offset_after_kernel(const uint64_t *off, const uint64_t *len, uint64_t *next, uint8_t *out) {
  const uint64_t end = *off + *len, aligned = *off + ((*len + 15) & ~15ull);
  for (uint64_t i = end; i < aligned; ++i) out[i] = 0;
  *next = aligned;
}
// The decompress status word: 0, or KVTC_E_CORRUPT when the inflater or a
// checksum flagged the container.
__global__ void status_kernel(const int32_t *err, int32_t nerr, int32_t *status_out) {
  int32_t bad = 0;
  for (int i = 0; i < nerr; ++i) bad |= err[i];
  *status_out = bad ? int32_t(KVTC_E_CORRUPT) : 0;
}

inline uint64_t align16(uint64_t x) { return (x + 15) & ~15ull; }

// R1/R7 cos/sin table for tokens [tok_begin, tok_begin + m) of a view.
kvtc_status rope_table_for(const kvtc_basis *b, int64_t pos_first, int64_t m, float2 *cs, cudaStream_t st) {
  return launch_rope_table(b->d_invf, b->shape.head_dim / 2, pos_first, m, cs, st);
}

kvtc_status tmap_X(CUtensorMap *m, const void *X, int64_t rows, int64_t p, int64_t ld = 0) {
  return make_tmap_2d(m, X, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, uint64_t(p), uint64_t(rows), uint64_t(ld ? ld : p) * 2,
                      kBlockK, kTileM);
}

// A contiguous cache whose layers sit at a constant positive stride can be read
// by the GEMM in place through a 3-D tensor map (no gathered copy of X): rows
// are tokens, the K axis walks layer by layer.  Returns false if not eligible.
bool direct_view_map(const kvtc_kv_view &v, int64_t tok0, CUtensorMap *m, int64_t *layer_rows) {
  *layer_rows = 0;
  const int64_t hd = int64_t(v.shape.kv_heads) * v.shape.head_dim;
  if (v.layout != KVTC_LAYOUT_CONTIGUOUS || hd % kBlockK || v.tokens > INT32_MAX / 2 || tok0 < 0) return false;
  const auto base = reinterpret_cast<uintptr_t>(v.layer_base_host[0]);
  if (base % 16) return false;
  uint64_t stride = uint64_t(v.tokens) * hd * 2;
  if (v.shape.layers > 1) {
    const auto b1 = reinterpret_cast<uintptr_t>(v.layer_base_host[1]);
    if (b1 <= base || (b1 - base) % 16) return false;
    stride = b1 - base;
    for (int l = 2; l < v.shape.layers; ++l)
      if (reinterpret_cast<uintptr_t>(v.layer_base_host[l]) != base + l * stride) return false;
  }
  // layers packed back to back (one [layers][tokens][h*d] tensor): KVTC_DIRECT_2D=1
  // reads it through a 2-D map over [layers * tokens][h*d] instead
  const char *e2 = getenv("KVTC_DIRECT_2D");
  if (e2 && e2[0] == '1' && stride == uint64_t(v.tokens) * hd * 2 && v.tokens * v.shape.layers < INT32_MAX / 2) {
    *layer_rows = v.tokens;
    return make_tmap_2d(m, v.layer_base_host[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, uint64_t(hd),
                        uint64_t(v.tokens) * v.shape.layers, uint64_t(hd) * 2, kBlockK, kTileM) == KVTC_OK;
  }
  return make_tmap_3d(m, v.layer_base_host[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, uint64_t(hd), uint64_t(v.tokens),
                      uint64_t(v.shape.layers), uint64_t(hd) * 2, stride, kBlockK, kTileM) == KVTC_OK;
}

// X: the gathered rows [m x p], or nullptr with `direct` = the 3-D map of the
// cache itself (rows = tokens tok0 ..).  wide: scratch of wide_scratch_bytes(m,
// wide_cols, nwide) bytes for the plan's wide groups (nullptr if it has none);
// they are quantised inside the GEMM's epilogue.
kvtc_status run_project_quant(const kvtc_basis *b, kvtc_plan *pl, const Operands *op, const void *X, int64_t m,
                              uint8_t *payload, float *wide, cudaStream_t st, const CUtensorMap *direct = nullptr,
                              int64_t tok0 = 0, int64_t ldx = 0, const TileRef *tiles = nullptr,
                              int64_t layer_rows = 0, int32_t *status = nullptr) {
  if (m == 0 || pl->G == 0) return KVTC_OK;
  KVTC_CHECK_ARG(pl->nwide == 0 || wide, "wide-group scratch");
  CUtensorMap tA;
  kvtc_status s = KVTC_OK;
  if (!direct && (s = tmap_X(&tA, X, m, b->p, ldx))) return s;
  GemmCompressArgs a = {};
  a.tmA = direct ? direct : &tA;
  if (direct) {
    a.a_hd = b->shape.kv_heads * b->shape.head_dim;
    a.a_row0 = tok0;
    a.a_layer_rows = layer_rows;
  }
  a.tmB = &op->tm_VcT;
  a.K = b->p;
  a.m = m;
  a.bias = op->bias;
  a.payload = payload;
  a.G = pl->G;
  a.tile_bytes = pl->tile_bytes;
  a.codes_off_last = plan_codes_off_last(pl, m % kTileM);
  a.groups = pl->d_gdesc;
  a.segs = pl->d_segs;
  a.nsegs = pl->nsegs;
  a.D = wide;
  a.ldd = pl->wide_cols;
  a.tiles = tiles;
  a.status = status;
  a.wide = pl->d_wide;
  a.nwide = pl->nwide;
  if ((s = launch_gemm_project_quant(a, st))) return s;
  // KVTC_WIDE_DEFER=1 (A/B measurement only): the wide groups quantised by the
  // separate SIMT pass over the fp32 scratch instead of the epilogue fixup
  const char *wd = getenv("KVTC_WIDE_DEFER");
  if (pl->nwide && wd && wd[0] == '1')
    return launch_quant_wide(pl->d_wide, pl->nwide, wide, pl->wide_cols, 1, m, pl->tile_bytes, a.codes_off_last,
                             payload, st, tiles, status);
  return KVTC_OK;
}

// The inverse path's A operand.  Default: the SIMT kernel dequantises into D^
// (HBM, fp16) and the reconstruction GEMM reads it through TMA.  KVTC_DQ_FUSED=1:
// the GEMM's producer warps dequantise straight into the shared-memory stages
// (D^ never reaches HBM; bitwise equal output), for plans whose A-chunk table
// fits in shared memory.  Measured 7-8x slower on the bench shape (48 ms vs
// 6.3 ms per launch): A is consumed by all p / 256 column tiles,
// so the producers dequantise every element 128 times, and their shared-memory
// stores compete with the tensor core's operand reads; so it stays opt-in.
bool dq_fused_env() {
  const char *e = getenv("KVTC_DQ_FUSED");
  return e && e[0] == '1';
}
bool dq_fits(const kvtc_plan *pl) { return int64_t(pl->dq_cols_n) / 8 * int64_t(sizeof(DqChunk)) <= kDqTabMaxBytes; }
bool dq_fused(const kvtc_plan *kp, const kvtc_plan *vp) { return dq_fused_env() && dq_fits(kp) && dq_fits(vp); }

// The reconstruction GEMM (K5).  payload != nullptr (or tiles carrying payload
// pointers, `fused`): A = D^ is dequantised from the payload inside the GEMM;
// otherwise A is the fp16 D^ [m x ld] in HBM.
kvtc_status run_reconstruct(const kvtc_basis *b, kvtc_plan *pl, const Operands *op, const __half *Dh,
                            int64_t ld, int64_t m, int64_t tok_begin, int32_t lb, int32_t le, const kvtc_kv_view *out,
                            __nv_bfloat16 *const *bases_dev, const float2 *cs, cudaStream_t st,
                            const TileRef *tiles = nullptr, const uint8_t *payload = nullptr, bool fused = false,
                            uint8_t *dq_tail = nullptr) {
  const int hd = b->shape.kv_heads * b->shape.head_dim;
  if (m == 0 || lb >= le) return KVTC_OK;
  GemmDecompressArgs a = {};
  CUtensorMap tA;
  // with an empty plan D^ has no columns: use a 1-column zero view (K = 0 -> only mu)
  const int64_t kcols = std::max<int64_t>(pl->r_nz, 1);
  kvtc_status s = make_tmap_2d(&tA, fused ? static_cast<const void *>(b->d_mu) : Dh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                               uint64_t(kcols), uint64_t(fused ? 1 : m), fused ? uint64_t((kcols * 2 + 15) / 16 * 16)
                                                                          : uint64_t(ld) * 2,
                               kBlockK, kTileM);
  if (s) return s;
  if (fused) {
    a.payload = payload;
    a.codes_off_full = pl->d_codes_off_full;
    a.codes_off_last = plan_codes_off_last(pl, m % kTileM);
    a.tile_bytes = pl->tile_bytes;
    a.dqcols = pl->d_dqcols;
    a.dqchunks = pl->d_dqchunks;
    a.tail_cols = pl->d_tail_cols;
    a.n_tail = pl->n_tail;
    a.dq_tail = dq_tail;
  }
  a.tmA = &tA;
  a.tmB = pl->r_nz ? &op->tm_Vd : &tA;
  a.K = pl->r_nz;
  a.m = m;
  a.n_begin = lb * hd;
  a.n_end = le * hd;
  a.mu = b->d_mu;
  a.cs = b->has_rope ? cs : nullptr;
  a.layers = b->shape.layers;
  a.heads = b->shape.kv_heads;
  a.head_dim = b->shape.head_dim;
  a.pairing = b->pairing;
  a.layout = out->layout;
  a.page_tokens = out->page_tokens;
  a.layer_base = bases_dev;
  a.block_table = out->block_table;
  a.tok_begin = tok_begin;
  int tile = kMaxTileN;
  while (hd % tile) tile /= 2;
  a.tile_n = tile;
  a.tiles = tiles;
  return launch_gemm_reconstruct(a, st);
}

// Library-internal side stream (one per device) used to overlap the integer
// codec kernels (DEFLATE / inflate / dequantise) with the tensor-core GEMMs of
// the other stream: a persistent GEMM CTA (196 KB smem, 256 threads) leaves 32 KB
// on every SM, room for two codec CTAs of a bounded grid (corun_ctas(2)).
// Fork/join with events on the caller's stream.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};
SideStream *side_stream() {
  // per host thread and device: concurrent callers never share the fork/join events
  static thread_local SideStream per_dev[16];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream &S = per_dev[dev & 15];
  if (!S.s) {
    cudaStreamCreateWithFlags(&S.s, cudaStreamNonBlocking);
    for (auto &e : S.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return &S;
}

// Per-SM CTAs of a side-stream kernel beside a GEMM (tuning: KVTC_CORUN_<KIND>).
int corun_per_sm(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? std::max(1, atoi(e)) : dflt;
}

bool env_flag(const char *name, bool dflt) {
  const char *e = getenv(name);
  return e ? e[0] == '1' : dflt;
}

// The integer codec kernels run on the library's side stream beside the GEMMs by
// default; KVTC_NO_OVERLAP=1 (or KVTC_OVERLAP=0) runs every kernel on the caller's
// stream.  Re-measured after the round-2 codec rewrites (in-process interleaved
// sweep, profiles/r02j_sweep_overlap.log): 32.42 ms per step overlapped vs 32.55 ms
// serial -- the co-runners cost the GEMMs ~2.1 ms, about what the codec kernels
// take on their own, so the two schedules are within noise.
bool overlap_off() {
  const char *e = getenv("KVTC_NO_OVERLAP");
  if (e) return e[0] == '1';
  const char *o = getenv("KVTC_OVERLAP");
  return o && o[0] == '0';
}

// KVTC_NO_DIRECT=1 forces the gathered path (tests compare the two).
bool direct_off() {
  const char *e = getenv("KVTC_NO_DIRECT");
  return e && e[0] == '1';
}

bool same_shape(const kvtc_shape &a, const kvtc_shape &b) {
  return a.layers == b.layers && a.kv_heads == b.kv_heads && a.head_dim == b.head_dim;
}

}  // namespace

// ============================================================ stage entry points
extern "C" kvtc_status kvtc_stage_project(const kvtc_basis *b, const kvtc_plan *plan, const void *X, int64_t m,
                                          float *D, void *stream) {
  KVTC_CHECK_ARG(b && X && D && m >= 0, "project arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (m == 0) return KVTC_OK;
  CUtensorMap tA, tB;
  kvtc_status s = tmap_X(&tA, X, m, b->p);
  if (s) return s;
  GemmCompressArgs a = {};
  a.tmA = &tA;
  a.K = b->p;
  a.m = m;
  a.D = D;
  int32_t ncols;
  if (plan) {
    const Operands *op;
    if ((s = plan_operands(b, const_cast<kvtc_plan *>(plan), &op))) return s;
    if (op->r_nz == 0) return KVTC_OK;
    a.tmB = &op->tm_VcT;
    a.bias = op->bias;
    ncols = op->r_nz;
  } else {
    if ((s = make_tmap_2d(&tB, b->d_VcT, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, b->p, b->r, uint64_t(b->p) * 2, kBlockK,
                          kMaxTileN / 2)))
      return s;
    a.tmB = &tB;
    a.bias = b->d_bias;
    ncols = b->r;
  }
  a.ldd = ncols;
  return launch_gemm_project_f32(a, ncols, st);
}

// Joint cross-shard compression: the partial
// projection of one layer shard, D_g = X_g V_c[f0:f1, plan PCs] (- mu V_c when
// add_bias), fp32 [m x r_nz].  The shards' partials sum to kvtc_stage_project's
// D of the joint features.
extern "C" kvtc_status kvtc_stage_project_partial(const kvtc_basis *b, const kvtc_plan *plan, const void *X, int64_t m,
                                                  int32_t feat_begin, int32_t feat_end, int32_t add_bias, float *D,
                                                  void *stream) {
  KVTC_CHECK_ARG(b && plan && X && D && m >= 0, "project_partial arguments");
  KVTC_CHECK_ARG(0 <= feat_begin && feat_begin < feat_end && feat_end <= b->p && feat_begin % 8 == 0 &&
                     (feat_end - feat_begin) % 8 == 0,
                 "project_partial: feature range (multiples of 8 inside the basis)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (m == 0) return KVTC_OK;
  const Operands *op;
  kvtc_status s = plan_operands(b, const_cast<kvtc_plan *>(plan), &op);
  if (s) return s;
  if (op->r_nz == 0) return KVTC_OK;
  const int32_t pg = feat_end - feat_begin;
  CUtensorMap tA, tB;
  if ((s = tmap_X(&tA, X, m, pg))) return s;
  if ((s = make_tmap_2d(&tB, op->VcT + feat_begin, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, uint64_t(pg), uint64_t(op->r_nz),
                        uint64_t(b->p + kXPad) * 2, kBlockK, kMaxTileN / 2)))
    return s;
  float *zero = nullptr;
  if (!add_bias) {
    KVTC_CUDA_TRY(cudaMallocAsync(&zero, size_t(op->r_nz) * 4, st));
    KVTC_CUDA_TRY(cudaMemsetAsync(zero, 0, size_t(op->r_nz) * 4, st));
  }
  GemmCompressArgs a = {};
  a.tmA = &tA;
  a.tmB = &tB;
  a.K = pg;
  a.m = m;
  a.D = D;
  a.ldd = op->r_nz;
  a.bias = add_bias ? op->bias : zero;
  s = launch_gemm_project_f32(a, op->r_nz, st);
  if (zero) cudaFreeAsync(zero, st);
  return s;
}

extern "C" kvtc_status kvtc_stage_quantize_pack(const kvtc_plan *plan, const float *D, int64_t m, uint8_t *payload,
                                                void *stream) {
  KVTC_CHECK_ARG(plan && D && payload && m >= 0, "quantize_pack arguments");
  auto *pl = const_cast<kvtc_plan *>(plan);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t *col = plan_codes_off_last(pl, m % kTileM);
  kvtc_status s = launch_quant_pack_simt(pl->d_segs, pl->d_gdesc, pl->nsegs, pl->G, D, pl->r_nz, m, pl->tile_bytes,
                                         col, payload, st);
  if (s) return s;
  return launch_quant_wide(pl->d_wide, pl->nwide, D, pl->r_nz, 0, m, pl->tile_bytes, col, payload, st);
}

extern "C" kvtc_status kvtc_stage_project_quantize(const kvtc_basis *b, const kvtc_plan *plan, const void *X,
                                                   int64_t m, uint8_t *payload, void *stream) {
  KVTC_CHECK_ARG(b && plan && X && payload && m >= 0, "project_quantize arguments");
  auto *pl = const_cast<kvtc_plan *>(plan);
  const Operands *op;
  kvtc_status s = plan_operands(b, pl, &op);
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float *wide = nullptr;      // stream-ordered scratch for the wide groups
  if (pl->nwide && m) KVTC_CUDA_TRY(cudaMallocAsync(&wide, wide_scratch_bytes(m, pl->wide_cols, pl->nwide), st));
  s = run_project_quant(b, pl, op, X, m, payload, wide, st);
  if (wide) cudaFreeAsync(wide, st);
  return s;
}

extern "C" size_t kvtc_deflate_bound(size_t n, int32_t chunk_bytes) { return deflate_section_bound(n, chunk_bytes); }
extern "C" size_t kvtc_deflate_workspace_bytes(size_t n, int32_t chunk_bytes) {
  return deflate_workspace(n, chunk_bytes) + 256;
}

extern "C" kvtc_status kvtc_stage_deflate(const uint8_t *in, size_t n, int32_t chunk_bytes, uint8_t *out,
                                          size_t out_cap, size_t *out_len_host, void *workspace,
                                          size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(in && out && workspace, "deflate arguments");
  KVTC_CHECK_ARG(out_cap >= deflate_section_bound(n, chunk_bytes), "deflate output capacity");
  KVTC_CHECK_ARG(workspace_bytes >= kvtc_deflate_workspace_bytes(n, chunk_bytes), "deflate workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Bump ws(workspace, workspace_bytes);
  uint64_t *len = ws.take<uint64_t>(1);
  void *rest = ws.take<uint8_t>(deflate_workspace(n, chunk_bytes));
  kvtc_status s = launch_deflate(in, n, chunk_bytes, out, nullptr, len, rest, deflate_workspace(n, chunk_bytes), st);
  if (s) return s;
  if (out_len_host) {
    uint64_t h = 0;
    KVTC_CUDA_TRY(cudaMemcpyAsync(&h, len, 8, cudaMemcpyDeviceToHost, st));
    KVTC_CUDA_TRY(cudaStreamSynchronize(st));
    *out_len_host = size_t(h);
  }
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_stage_inflate(const uint8_t *section, size_t len, uint8_t *out, size_t n_out,
                                          void *stream) {
  KVTC_CHECK_ARG(section && out && len >= kSectionHeaderBytes, "inflate arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t hdr[kSectionHeaderBytes];
  KVTC_CUDA_TRY(cudaMemcpyAsync(hdr, section, sizeof(hdr), cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  uint32_t nch = 0;
  kvtc_status s = check_section_header(hdr, len, n_out, &nch);
  if (s) return s;
  int32_t *err = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&err, 4, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
  s = launch_inflate_section(section, len, n_out, nch, out, err, st);
  int32_t herr = 0;
  KVTC_CUDA_TRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(err, st);
  if (s) return s;
  if (herr) {
    set_error("corrupt DEFLATE stream (code %d)", herr);
    return KVTC_E_CORRUPT;
  }
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_stage_inflate_raw(const uint8_t *in, const int64_t *in_off, const int64_t *in_len,
                                              int32_t nstreams, uint8_t *out, const int64_t *out_off,
                                              const int64_t *out_len, int32_t *status_dev, void *stream) {
  KVTC_CHECK_ARG(nstreams >= 0 && (nstreams == 0 || (in && in_off && in_len && out && out_off && out_len && status_dev)),
                 "inflate_raw arguments");
  return launch_inflate_raw(in, in_off, in_len, nstreams, out, out_off, out_len, status_dev,
                            static_cast<cudaStream_t>(stream));
}

// rANS back-end stage entries (reading Q24).
extern "C" size_t kvtc_rans_bound(size_t n, int32_t chunk_bytes, int64_t tile_bytes) {
  return rans_section_bound(n, chunk_bytes, tile_bytes);
}
extern "C" size_t kvtc_rans_workspace_bytes(size_t n, int32_t chunk_bytes, int64_t tile_bytes) {
  return rans_workspace(n, chunk_bytes, tile_bytes);
}
extern "C" kvtc_status kvtc_stage_rans_encode(const uint8_t *in, size_t n, int32_t chunk_bytes, int64_t tile_bytes,
                                              uint8_t *out, size_t out_cap, size_t *out_len_host, void *workspace,
                                              size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(in && out && out_len_host, "rans_encode arguments");
  KVTC_CHECK_ARG(chunk_bytes >= 1024 && chunk_bytes <= (1 << 20) && chunk_bytes % 32 == 0, "rans chunk_bytes");
  KVTC_CHECK_ARG(out_cap >= rans_section_bound(n, chunk_bytes, tile_bytes), "rans output capacity");
  KVTC_CHECK_ARG((reinterpret_cast<uintptr_t>(out) & 15) == 0, "rans output must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t *len_dev = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&len_dev, 8, st));
  kvtc_status s = launch_rans_encode(in, n, chunk_bytes, tile_bytes, out, nullptr, len_dev, workspace,
                                     workspace_bytes, st);
  if (s) return s;
  uint64_t len = 0;
  KVTC_CUDA_TRY(cudaMemcpyAsync(&len, len_dev, 8, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(len_dev, st);
  *out_len_host = size_t(len);
  return KVTC_OK;
}
extern "C" kvtc_status kvtc_stage_rans_decode(const uint8_t *section, size_t len, uint8_t *out, size_t n_out,
                                              void *stream) {
  KVTC_CHECK_ARG(section && out && len >= kRansHeaderBytes, "rans_decode arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t hdr[kRansHeaderBytes];
  KVTC_CUDA_TRY(cudaMemcpyAsync(hdr, section, sizeof(hdr), cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  uint32_t nch = 0, ncls = 0;
  kvtc_status s = check_rans_header(hdr, len, n_out, &nch, &ncls);
  if (s) return s;
  void *ws = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&ws, rans_decode_workspace(ncls) + 16, st));
  int32_t *err = reinterpret_cast<int32_t *>(static_cast<uint8_t *>(ws) + rans_decode_workspace(ncls));
  KVTC_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
  if ((s = launch_rans_decode(section, len, n_out, nch, ncls, out, ws, err, st))) return s;
  int32_t e = 0;
  KVTC_CUDA_TRY(cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(ws, st);
  if (e) {
    set_error("corrupt rANS section (%d)", e);
    return KVTC_E_CORRUPT;
  }
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_stage_dequantize(const kvtc_plan *plan, const uint8_t *payload, int64_t m, uint16_t *Dh,
                                             int64_t ld, void *stream) {
  KVTC_CHECK_ARG(plan && payload && Dh && ld >= plan->r_nz && m >= 0, "dequantize arguments");
  auto *pl = const_cast<kvtc_plan *>(plan);
  return launch_dequant(pl->d_dqchunks, pl->d_dqcols, pl->r_nz, pl->d_codes_off_full, plan_codes_off_last(pl, m % kTileM),
                        pl->tile_bytes, payload, m, reinterpret_cast<__half *>(Dh), ld,
                        static_cast<cudaStream_t>(stream));
}

namespace {
kvtc_status stage_reconstruct(const kvtc_basis *b, const kvtc_plan *plan, const uint16_t *Dh, const uint8_t *payload,
                              int64_t ld, int64_t m, int64_t tok_begin, int32_t layer_begin, int32_t layer_end,
                              const kvtc_kv_view *out, void *stream) {
  kvtc_status s = check_view(out);
  if (s) return s;
  KVTC_CHECK_ARG(b && plan && (Dh || payload) && same_shape(out->shape, b->shape), "reconstruct arguments");
  KVTC_CHECK_ARG(payload || (ld % 8 == 0 && ld >= plan->r_nz), "ld must be a multiple of 8 and >= plan columns");
  KVTC_CHECK_ARG(0 <= layer_begin && layer_begin <= layer_end && layer_end <= b->shape.layers, "layer range");
  KVTC_CHECK_ARG(tok_begin >= 0 && tok_begin + m <= out->tokens, "token range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto *pl = const_cast<kvtc_plan *>(plan);
  const Operands *op;
  if ((s = plan_operands(b, pl, &op))) return s;
  const int half = b->shape.head_dim / 2;
  Bump need;
  need.take<void *>(b->shape.layers);
  need.take<float2>(m * half);
  need.take<uint8_t>(payload ? dq_tail_bytes(m, pl->n_tail) : 0);
  void *scratch = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&scratch, need.used, st));
  Bump ws(scratch, need.used);
  auto *bases = ws.take<__nv_bfloat16 *>(b->shape.layers);
  float2 *cs = ws.take<float2>(m * half);
  uint8_t *tail = ws.take<uint8_t>(payload ? dq_tail_bytes(m, pl->n_tail) : 0);
  if ((s = upload_bases(out, bases, st))) return s;
  if (b->has_rope && (s = rope_table_for(b, out->pos0 + tok_begin, m, cs, st))) return s;
  s = run_reconstruct(b, pl, op, reinterpret_cast<const __half *>(Dh), ld, m, tok_begin, layer_begin, layer_end, out,
                      bases, cs, st, nullptr, payload, payload != nullptr, tail);
  cudaFreeAsync(scratch, st);
  return s;
}
}  // namespace

extern "C" kvtc_status kvtc_stage_reconstruct(const kvtc_basis *b, const kvtc_plan *plan, const uint16_t *Dh,
                                              int64_t ld, int64_t m, int64_t tok_begin, int32_t layer_begin,
                                              int32_t layer_end, const kvtc_kv_view *out, void *stream) {
  return stage_reconstruct(b, plan, Dh, nullptr, ld, m, tok_begin, layer_begin, layer_end, out, stream);
}

extern "C" kvtc_status kvtc_stage_reconstruct_payload(const kvtc_basis *b, const kvtc_plan *plan,
                                                      const uint8_t *payload, int64_t m, int64_t tok_begin,
                                                      int32_t layer_begin, int32_t layer_end, const kvtc_kv_view *out,
                                                      void *stream) {
  KVTC_CHECK_ARG(payload, "reconstruct_payload: null payload");
  return stage_reconstruct(b, plan, nullptr, payload, 0, m, tok_begin, layer_begin, layer_end, out, stream);
}

// ================================================================== codec
namespace {
struct CompressLayout {
  int64_t m, nraw, raw_bytes;
  uint64_t pay[2];
  uint64_t sec_bound[2];
  uint64_t k_off;
  uint64_t bound;
};
CompressLayout compress_layout(const kvtc_plan *kp, const kvtc_plan *vp, const kvtc_kv_view *k,
                               const kvtc_policy *pol) {
  CompressLayout L{};
  const int64_t t = k->tokens;
  const int64_t sw = int64_t(pol->sinks) + pol->window;
  L.m = t > sw ? t - sw : 0;
  L.nraw = L.m ? sw : t;
  const int64_t hd = int64_t(k->shape.kv_heads) * k->shape.head_dim;
  L.raw_bytes = 2 * int64_t(k->shape.layers) * L.nraw * hd * 2;
  L.pay[0] = kvtc_payload_bytes(kp, L.m);
  L.pay[1] = kvtc_payload_bytes(vp, L.m);
  for (int s = 0; s < 2; ++s)
    L.sec_bound[s] = pol->coder == KVTC_CODER_RANS
                         ? rans_section_bound(L.pay[s], pol->chunk_bytes, (s ? vp : kp)->tile_bytes)
                         : deflate_section_bound(L.pay[s], pol->chunk_bytes);
  L.k_off = align16(KVTC_HEADER_BYTES + L.raw_bytes);
  L.bound = L.k_off + align16(L.sec_bound[0]) + align16(L.sec_bound[1]) + 64;
  return L;
}
}  // namespace

// Entropy-coder workspace of one stream (the chosen back-end).
size_t entropy_workspace(const kvtc_policy *pol, uint64_t n, const kvtc_plan *pl) {
  return pol->coder == KVTC_CODER_RANS ? rans_workspace(n, pol->chunk_bytes, pl->tile_bytes)
                                       : deflate_workspace(n, pol->chunk_bytes);
}

extern "C" size_t kvtc_compress_bound(const kvtc_plan *kp, const kvtc_plan *vp, const kvtc_kv_view *k,
                                      const kvtc_policy *pol) {
  if (!kp || !vp || !k || !pol) return 0;
  return size_t(compress_layout(kp, vp, k, pol).bound);
}

extern "C" size_t kvtc_compress_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                                const kvtc_plan *vp, const kvtc_kv_view *k, const kvtc_policy *pol) {
  if (!kb || !kp || !vb || !vp || !k || !pol) return 0;
  const CompressLayout L = compress_layout(kp, vp, k, pol);
  Bump b;
  b.take<void *>(k->shape.layers);
  b.take<void *>(k->shape.layers);
  b.take<uint64_t>(8);
  b.take<__nv_bfloat16>(L.m * (kb->p + kXPad));
  b.take<float2>(L.m * (kb->shape.head_dim / 2));
  b.take<uint8_t>(L.pay[0] + 16);
  b.take<uint8_t>(L.pay[1] + 16);
  b.take<uint8_t>(entropy_workspace(pol, L.pay[0], kp));
  b.take<uint8_t>(entropy_workspace(pol, L.pay[1], vp));
  b.take<uint8_t>(wide_scratch_bytes(L.m, std::max(kp->wide_cols, vp->wide_cols), std::max(kp->nwide, vp->nwide)));
  return b.used + 256;
}

extern "C" kvtc_status kvtc_compress(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                     const kvtc_plan *vp, const kvtc_kv_view *k, const kvtc_kv_view *v,
                                     const kvtc_policy *pol, void *out, size_t out_cap, size_t *out_len_host,
                                     void *workspace, size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && k && v && pol && out, "compress arguments");
  kvtc_status s;
  if ((s = check_view(k)) || (s = check_view(v))) return s;
  KVTC_CHECK_ARG(same_shape(k->shape, v->shape) && k->tokens == v->tokens && k->pos0 == v->pos0,
                 "key and value views differ");
  KVTC_CHECK_ARG(same_shape(k->shape, kb->shape) && same_shape(v->shape, vb->shape), "basis shape mismatch");
  KVTC_CHECK_ARG(kb->which == KVTC_KEYS && vb->which == KVTC_VALUES, "basis streams");
  KVTC_CHECK_ARG(pol->sinks >= 0 && pol->window >= 0, "policy");
  KVTC_CHECK_ARG(pol->chunk_bytes == 16384 || pol->chunk_bytes == 32768 || pol->chunk_bytes == 65536, "chunk_bytes");
  KVTC_CHECK_ARG(pol->coder == KVTC_CODER_DEFLATE || pol->coder == KVTC_CODER_RANS, "policy coder");
  const bool rans = pol->coder == KVTC_CODER_RANS;
  const CompressLayout L = compress_layout(kp, vp, k, pol);
  if (out_cap < L.bound) {
    set_error("output capacity %zu < bound %llu", out_cap, (unsigned long long)L.bound);
    return KVTC_E_CAPACITY;
  }
  const size_t need = kvtc_compress_workspace_bytes(kb, kp, vb, vp, k, pol);
  if (workspace_bytes < need || !workspace) {
    set_error("workspace %zu < %zu", workspace_bytes, need);
    return KVTC_E_CAPACITY;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto *kpl = const_cast<kvtc_plan *>(kp);
  auto *vpl = const_cast<kvtc_plan *>(vp);
  const Operands *kop, *vop;
  if ((s = plan_operands(kb, kpl, &kop)) || (s = plan_operands(vb, vpl, &vop))) return s;

  Bump ws(workspace, workspace_bytes);
  auto *kbases = ws.take<__nv_bfloat16 *>(k->shape.layers);
  auto *vbases = ws.take<__nv_bfloat16 *>(k->shape.layers);
  uint64_t *lens = ws.take<uint64_t>(kCompressWords);     // see kCompressWords
  int32_t *cstatus = reinterpret_cast<int32_t *>(lens + 4);
  const int64_t ldx = kb->p + kXPad;
  auto *X = ws.take<__nv_bfloat16>(L.m * ldx);
  float2 *cs = ws.take<float2>(L.m * (kb->shape.head_dim / 2));
  uint8_t *payload_k = ws.take<uint8_t>(L.pay[0] + 16);
  uint8_t *payload_v = ws.take<uint8_t>(L.pay[1] + 16);
  const size_t dws[2] = {entropy_workspace(pol, L.pay[0], kp), entropy_workspace(pol, L.pay[1], vp)};
  void *dwsp[2];
  dwsp[0] = ws.take<uint8_t>(dws[0]);
  dwsp[1] = ws.take<uint8_t>(dws[1]);
  // one scratch for both streams' wide groups (their GEMMs run one after the other on st)
  float *wide = reinterpret_cast<float *>(
      ws.take<uint8_t>(wide_scratch_bytes(L.m, std::max(kp->wide_cols, vp->wide_cols), std::max(kp->nwide, vp->nwide))));
  if ((s = upload_bases(k, kbases, st)) || (s = upload_bases(v, vbases, st))) return s;
  KVTC_CUDA_TRY(cudaMemsetAsync(lens, 0, kCompressWords * 8, st));

  uint8_t *o = static_cast<uint8_t *>(out);
  ContainerHeader h = {};
  h.magic = kContainerMagic;
  h.version = kContainerVersion;
  h.layers = k->shape.layers;
  h.kv_heads = k->shape.kv_heads;
  h.head_dim = k->shape.head_dim;
  h.sinks = pol->sinks;
  h.window = pol->window;
  h.chunk_bytes = pol->chunk_bytes;
  h.flags = rans && L.m ? kFlagRans : 0u;
  h.tokens = k->tokens;
  h.pos0 = k->pos0;
  h.m = L.m;
  h.raw_bytes = L.raw_bytes;
  h.payload_bytes[0] = L.pay[0];
  h.payload_bytes[1] = L.pay[1];
  h.basis_fp[0] = kb->fp;
  h.basis_fp[1] = vb->fp;
  h.plan_fp[0] = kp->fp;
  h.plan_fp[1] = vp->fp;
  h.raw_off = KVTC_HEADER_BYTES;
  h.section_off[1] = L.k_off;                  // first section: the values' (see kCompressWords)

  // raw sinks + window, K then V: [layers][nraw][h*d] each
  const int64_t hd = int64_t(k->shape.kv_heads) * k->shape.head_dim;
  auto *rawk = reinterpret_cast<__nv_bfloat16 *>(o + KVTC_HEADER_BYTES);
  auto *rawv = rawk + int64_t(k->shape.layers) * L.nraw * hd;
  const int64_t t = k->tokens;
  // raw sinks + window of the middle-token case: packed (and hashed) on the side
  // stream after the fork below, beside the values' GEMM
  auto pack_raw = [&](cudaStream_t q, bool side) -> kvtc_status {
    ProfScope ps_raw(side ? "c.raw_tokens_overlapped" : "c.raw_tokens", q);
    kvtc_status r;
    for (int sv = 0; sv < 2; ++sv) {
      const kvtc_kv_view *vw = sv ? v : k;
      __nv_bfloat16 *const *bs = sv ? vbases : kbases;
      __nv_bfloat16 *dst = sv ? rawv : rawk;
      if ((r = launch_pack_raw(*vw, bs, 0, pol->sinks, dst, L.nraw, 0, q))) return r;
      if ((r = launch_pack_raw(*vw, bs, t - pol->window, pol->window, dst, L.nraw, pol->sinks, q))) return r;
    }
    return launch_hash(rawk, L.raw_bytes, kSeedRaw, lens + 7, q);
  };
  if (!L.m) {
    if ((s = launch_pack_raw(*k, kbases, 0, t, rawk, L.nraw, 0, st))) return s;
    if ((s = launch_pack_raw(*v, vbases, 0, t, rawv, L.nraw, 0, st))) return s;
    if ((s = launch_hash(rawk, L.raw_bytes, kSeedRaw, lens + 7, st))) return s;
    header_kernel<<<1, 1, 0, st>>>(h, o, nullptr, lens);
    KVTC_LAUNCH_CHECK();
    if (out_len_host) {
      KVTC_CUDA_TRY(cudaStreamSynchronize(st));
      *out_len_host = size_t(h.raw_off + L.raw_bytes);
    }
    return KVTC_NOTHING_TO_COMPRESS;
  }
  KVTC_CUDA_TRY(cudaMemcpyAsync(lens + 3, &h.section_off[1], 8, cudaMemcpyHostToDevice, st));
  // Schedule: the tensor-core GEMMs run back to back on the
  // caller's stream; the HBM/integer kernels of the OTHER stream run beside them
  // on the side stream with bounded grids (2 CTAs per SM next to the persistent
  // GEMM CTA).  With a contiguous value cache read in place by the GEMM:
  //   st : V GEMM --------------------------> K GEMM -> K DEFLATE -> assemble
  //   aux: K un-RoPE gather -> (after V GEMM)  V DEFLATE ------------^
  // Otherwise X is shared: K gather -> K GEMM -> V gather -> V GEMM -> V DEFLATE,
  // with the keys' DEFLATE beside the values' gather/GEMM.  Each stream's
  // encoder writes its own slots; the sections are assembled at the end (K first).
  SideStream *ss = side_stream();
  const bool ovl = !overlap_off();
  cudaStream_t aux = ovl ? ss->s : st;
  const int side_ctas = ovl ? corun_ctas(corun_per_sm("KVTC_CORUN_DEFLATE", 2)) : 0;
  CUtensorMap tV;
  int64_t v_layer_rows = 0;
  const bool v_direct = !direct_off() && direct_view_map(*v, pol->sinks, &tV, &v_layer_rows);
  auto gather_keys = [&](cudaStream_t q, int ctas, const char *tag) -> kvtc_status {
    ProfScope ps(tag, q);
    kvtc_status r = rope_table_for(kb, k->pos0 + pol->sinks, L.m, cs, q);
    if (r) return r;
    return launch_gather(*k, kbases, pol->sinks, L.m, cs, kb->pairing, X, q, ctas, ldx);
  };
  // rows [r0, r1) of a stream (r0 a multiple of the 128-token tile): payload tiles
  // are addressed from r0; the wide-group scratch is per launch (launches on st
  // run one after the other)
  auto gemm = [&](int sv, bool direct, int64_t r0 = 0, int64_t r1 = -1) -> kvtc_status {
    ProfScope ps("c.project_quant_gemm", st);
    if (r1 < 0) r1 = L.m;
    const kvtc_plan *pl = sv ? vpl : kpl;
    uint8_t *pay = (sv ? payload_v : payload_k) + (r0 / kTileM) * pl->tile_bytes;
    return sv ? run_project_quant(vb, vpl, vop, X, r1 - r0, pay, wide, st, direct ? &tV : nullptr, pol->sinks + r0,
                                  ldx, nullptr, v_layer_rows, cstatus)
              : run_project_quant(kb, kpl, kop, X + r0 * ldx, r1 - r0, pay, wide, st, nullptr, 0, ldx, nullptr, 0,
                                  cstatus);
  };
  // the payload checksum is taken on the encoder's stream right before the call
  // that encodes the last chunk range: the whole payload is complete there
  auto encode = [&](int sv, cudaStream_t q, int ctas, const char *tag, uint32_t c0 = 0,
                    uint32_t c1 = 0xFFFFFFFFu) -> kvtc_status {
    // stage names: the rANS back-end encodes the values here (keys at the assembly point)
    ProfScope ps(!rans ? tag : (sv == 0 ? "c.rans_hash_k" : (q == st ? "c.rans_values" : "c.rans_values_overlapped")), q);
    kvtc_status r;
    if (c1 == 0xFFFFFFFFu && (r = launch_hash(sv ? payload_v : payload_k, L.pay[sv], kSeedPayload, lens + 5 + sv, q, ctas)))
      return r;
    if (rans) {
      // rANS back-end (Q24): histogram, tables, encode and the section in one call.
      // The values' section goes first (offset lens[3]); the keys' is encoded at the
      // assembly point below, once its offset (lens[2]) is known.
      if (sv == 0) return KVTC_OK;
      if ((r = launch_rans_encode(payload_v, L.pay[1], pol->chunk_bytes, vpl->tile_bytes, o, lens + 3, lens + 1,
                                  dwsp[1], dws[1], q)))
        return r;
      offset_after_kernel<<<1, 1, 0, q>>>(lens + 3, lens + 1, lens + 2, o);
      KVTC_LAUNCH_CHECK();
      return KVTC_OK;
    }
    if ((r = launch_deflate_encode(sv ? payload_v : payload_k, L.pay[sv], pol->chunk_bytes, dwsp[sv], dws[sv], ctas,
                                   q, c0, c1)))
      return r;
    if (sv == 1) {
      // the values' section goes first in the container: assembled right away on
      // the encoder's stream (beside the keys' GEMM when that is the side stream);
      // the keys' section starts at the 16-aligned end of it
      ProfScope pa("c.assemble_v", q);
      if ((r = launch_deflate_assemble(L.pay[1], pol->chunk_bytes, dwsp[1], o, lens + 3, lens + 1, q))) return r;
      offset_after_kernel<<<1, 1, 0, q>>>(lens + 3, lens + 1, lens + 2, o);
      KVTC_LAUNCH_CHECK();
    }
    return KVTC_OK;
  };
  KVTC_CUDA_TRY(cudaEventRecord(ss->ev[0], st));                 // fork point: bases, tables uploaded
  KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[0], 0));
  if ((s = pack_raw(aux, ovl))) return s;                         // joined before the assembly (ev[3])
  if (v_direct) {
    // tuning knobs (scripts/sweep_env.py): KVTC_C_GATHER_SIDE=0 runs the keys'
    // gather before the values' GEMM instead of beside it; KVTC_C_DEFLATE_SIDE=0
    // runs both encoders after the GEMMs instead of the values' beside the keys' GEMM
    const bool gather_side = ovl && env_flag("KVTC_C_GATHER_SIDE", true);
    const bool deflate_side = ovl && env_flag("KVTC_C_DEFLATE_SIDE", true);
    if (!gather_side && (s = gather_keys(st, 0, "c.gather_unrope"))) return s;
    if ((s = gemm(1, true))) return s;
    KVTC_CUDA_TRY(cudaEventRecord(ss->ev[2], st));               // V payload ready
    if (gather_side) {
      KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[0], 0));
      if ((s = gather_keys(aux, corun_ctas(corun_per_sm("KVTC_CORUN_GATHER", 3)), "c.gather_unrope_overlapped")))
        return s;
      KVTC_CUDA_TRY(cudaEventRecord(ss->ev[1], aux));            // X (keys) ready
      KVTC_CUDA_TRY(cudaStreamWaitEvent(st, ss->ev[1], 0));
    }
    // keys' GEMM in two row halves when KVTC_C_SPLIT=1 (measured slower: the encoder
    // beside the GEMM halves costs more GEMM time than the shorter tail saves): the chunks of
    // the first half are encoded beside the second half, so only the second
    // half's encoder is left after the last GEMM
    const int64_t tiles = (L.m + kTileM - 1) / kTileM;
    const int64_t half = (tiles / 2) * kTileM;
    const uint32_t c_half = uint32_t(uint64_t(half / kTileM) * kpl->tile_bytes / uint64_t(pol->chunk_bytes));
    const bool split = deflate_side && !rans && env_flag("KVTC_C_SPLIT", false) && half > 0 && c_half > 0;
    if (deflate_side) KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[2], 0));
    if (split) {
      if ((s = gemm(0, false, 0, half))) return s;
      KVTC_CUDA_TRY(cudaEventRecord(ss->ev[1], st));             // first half of the keys' payload ready
      if ((s = gemm(0, false, half, L.m))) return s;
    } else if ((s = gemm(0, false))) {
      return s;
    }
    if (deflate_side) {
      if ((s = encode(1, aux, side_ctas, "c.deflate_overlapped"))) return s;
      if (split) {
        KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[1], 0));
        if ((s = encode(0, aux, side_ctas, "c.deflate_overlapped", 0, c_half))) return s;
      }
    } else if ((s = encode(1, st, 0, "c.deflate"))) {
      return s;
    }
    if ((s = encode(0, st, 0, "c.deflate", split ? c_half : 0))) return s;
  } else {
    if ((s = gather_keys(st, 0, "c.gather_unrope"))) return s;
    if ((s = gemm(0, false))) return s;
    KVTC_CUDA_TRY(cudaEventRecord(ss->ev[2], st));               // K payload ready
    {
      ProfScope ps("c.gather", st);
      if ((s = launch_gather(*v, vbases, pol->sinks, L.m, nullptr, 0, X, st, 0, ldx))) return s;
    }
    if ((s = gemm(1, false))) return s;
    KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[2], 0));
    if ((s = encode(0, aux, side_ctas, ovl ? "c.deflate_overlapped" : "c.deflate"))) return s;
    if ((s = encode(1, st, 0, "c.deflate"))) return s;
  }
  KVTC_CUDA_TRY(cudaEventRecord(ss->ev[3], aux));
  KVTC_CUDA_TRY(cudaStreamWaitEvent(st, ss->ev[3], 0));          // join: both streams encoded
  {
    ProfScope ps(rans ? "c.rans_keys" : "c.assemble", st);
    if (rans) {
      if ((s = launch_rans_encode(payload_k, L.pay[0], pol->chunk_bytes, kpl->tile_bytes, o, lens + 2, lens + 0,
                                  dwsp[0], dws[0], st)))
        return s;
    } else if ((s = launch_deflate_assemble(L.pay[0], pol->chunk_bytes, dwsp[0], o, lens + 2, lens + 0, st))) {
      return s;
    }
  }
  header_kernel<<<1, 1, 0, st>>>(h, o, lens, lens);
  KVTC_LAUNCH_CHECK();
  if (out_len_host) {
    uint64_t l4[kCompressWords];
    KVTC_CUDA_TRY(cudaMemcpyAsync(l4, lens, sizeof(l4), cudaMemcpyDeviceToHost, st));
    KVTC_CUDA_TRY(cudaStreamSynchronize(st));
    *out_len_host = size_t(l4[2] + l4[0]);      // K section offset + K section length (the last section)
    if (l4[4] & 1) {
      set_error("a 16-bit shift/scale overflowed (container flagged)");
      return KVTC_E_NUMERIC;
    }
  }
  return KVTC_OK;
}

namespace {
// Internal consistency of a container header (host copy): its checksum, its
// flags, and every size / offset the decompressor uses, re-derived from the
// shape — so a damaged or crafted header can make no read outside the container
// and no write outside the caller's views.
kvtc_status validate_header(const ContainerHeader &h) {
  auto bad = [](const char *what) {
    set_error("corrupt container: %s", what);
    return KVTC_E_CORRUPT;
  };
  if (h.magic != kContainerMagic || h.version != kContainerVersion) {
    set_error("not a KVTC container (magic %08x version %u)", h.magic, h.version);
    return KVTC_E_CORRUPT;
  }
  if (hash_words(reinterpret_cast<const uint64_t *>(&h), 31, kSeedHeader) != h.header_hash)
    return bad("header checksum");
  if (h.layers <= 0 || h.layers > 65536 || h.kv_heads <= 0 || h.kv_heads > 65536 || h.head_dim <= 0 ||
      h.head_dim > 4096 || h.head_dim % 32 || h.sinks < 0 || h.window < 0 || h.tokens < 0 ||
      h.tokens > (int64_t(1) << 40) || (h.chunk_bytes != 16384 && h.chunk_bytes != 32768 && h.chunk_bytes != 65536))
    return bad("shape / policy fields");
  const int64_t sw = int64_t(h.sinks) + h.window;
  const int64_t m = h.tokens > sw ? h.tokens - sw : 0;
  if (h.m != m) return bad("m != tokens - sinks - window");
  const int64_t nraw = m ? sw : h.tokens;
  const uint64_t raw = 2ull * uint64_t(h.layers) * uint64_t(nraw) * uint64_t(h.kv_heads) * uint64_t(h.head_dim) * 2;
  if (h.raw_off != KVTC_HEADER_BYTES || h.raw_bytes != raw) return bad("raw section size / offset");
  if (m) {
    const uint64_t first = align16(KVTC_HEADER_BYTES + raw);      // values' section, then keys'
    if (h.section_off[1] != first || h.section_off[0] != first + align16(h.entropy_bytes[1]) ||
        h.entropy_bytes[0] < kSectionHeaderBytes || h.entropy_bytes[1] < kSectionHeaderBytes ||
        h.entropy_bytes[0] > (uint64_t(1) << 50) || h.entropy_bytes[1] > (uint64_t(1) << 50) ||
        h.total_bytes != h.section_off[0] + h.entropy_bytes[0])
      return bad("section offsets / lengths");
  }
  if (h.flags & ~(kFlagNumeric | kFlagRans)) return bad("unknown flags");
  if (h.flags & kFlagNumeric) {
    set_error("container flagged at compression: a 16-bit shift/scale overflowed (Q4)");
    return KVTC_E_NUMERIC;
  }
  return KVTC_OK;
}
}  // namespace

extern "C" kvtc_status kvtc_container_parse(const void *header_host, kvtc_container_info *info) {
  KVTC_CHECK_ARG(header_host && info, "container_parse arguments");
  ContainerHeader h;
  memcpy(&h, header_host, sizeof(h));
  *info = kvtc_container_info{};
  info->magic = h.magic;
  info->version = h.version;
  info->layers = h.layers;
  info->kv_heads = h.kv_heads;
  info->head_dim = h.head_dim;
  info->sinks = h.sinks;
  info->window = h.window;
  info->chunk_bytes = h.chunk_bytes;
  info->tokens = h.tokens;
  info->pos0 = h.pos0;
  info->m = h.m;
  info->total_bytes = h.m ? h.total_bytes : h.raw_off + h.raw_bytes;
  info->raw_bytes = h.raw_bytes;
  for (int s = 0; s < 2; ++s) {
    info->payload_bytes[s] = h.payload_bytes[s];
    info->entropy_bytes[s] = h.entropy_bytes[s];
    info->basis_fp[s] = h.basis_fp[s];
    info->plan_fp[s] = h.plan_fp[s];
    info->payload_hash[s] = h.payload_hash[s];
  }
  info->flags = h.flags;
  info->raw_hash = h.raw_hash;
  return validate_header(h);
}

namespace {
// Header (host copy) checked against the container rules and the caller's
// bases / plans; in_len > 0 also bounds the container length.
kvtc_status read_checked_header(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb, const kvtc_plan *vp,
                                const void *header_host, size_t in_len, ContainerHeader *out) {
  ContainerHeader h;
  memcpy(&h, header_host, sizeof(h));
  kvtc_container_info info;
  kvtc_status s = kvtc_container_parse(&h, &info);
  if (s) return s;
  const kvtc_shape shp{h.layers, h.kv_heads, h.head_dim};
  if (!same_shape(shp, kb->shape) || !same_shape(shp, vb->shape)) {
    set_error("container shape does not match the bases");
    return KVTC_E_MISMATCH;
  }
  if (h.basis_fp[0] != kb->fp || h.basis_fp[1] != vb->fp || h.plan_fp[0] != kp->fp || h.plan_fp[1] != vp->fp) {
    set_error("container was written with a different basis or plan");
    return KVTC_E_MISMATCH;
  }
  if (in_len && info.total_bytes > in_len) {
    set_error("container length %llu > buffer %zu", (unsigned long long)info.total_bytes, in_len);
    return KVTC_E_CORRUPT;
  }
  if (h.m && (h.payload_bytes[0] != kvtc_payload_bytes(kp, h.m) || h.payload_bytes[1] != kvtc_payload_bytes(vp, h.m))) {
    set_error("corrupt container: payload sizes do not match the plans");
    return KVTC_E_CORRUPT;
  }
  *out = h;
  return KVTC_OK;
}

// Workspace of one decompression (kvtc_decompress_workspace_bytes).
struct DecompWs {
  __nv_bfloat16 **kbases, **vbases;
  int32_t *err;          // [0] inflater, [1] checksum mismatch bits, [2] status word, [3] unused
  uint64_t *hsum;        // checksums of the inflated payloads K/V and of the raw section
  uint8_t *payloads[2];
  __half *Dh[2];
  float2 *cs;
  uint8_t *tail;         // fused path: the pre-pass columns (shared by K and V, one GEMM at a time)
  uint8_t *rans_ws[2];   // rANS containers: the decoder tables of each stream
  uint32_t *ictr;        // fused inflate + dequantise: [2] item counters, [2][ntiles] tile arrivals
  int64_t ld;
};
inline int64_t ictr_words(int64_t m) { return 2 + 2 * ceil_div(m, kTileM); }
DecompWs carve_decomp(const kvtc_plan *kp, const kvtc_plan *vp, const ContainerHeader &h, void *workspace,
                      size_t workspace_bytes) {
  Bump ws(workspace, workspace_bytes);
  DecompWs w;
  w.kbases = ws.take<__nv_bfloat16 *>(h.layers);
  w.vbases = ws.take<__nv_bfloat16 *>(h.layers);
  w.err = ws.take<int32_t>(4);
  w.hsum = ws.take<uint64_t>(4);
  w.payloads[0] = ws.take<uint8_t>(h.payload_bytes[0] + 16);
  w.payloads[1] = ws.take<uint8_t>(h.payload_bytes[1] + 16);
  w.ld = std::max(std::max(kp->r_nz_pad, vp->r_nz_pad), 8);
  // D^ only exists in HBM on the unfused (measurement) path
  const int64_t dh_rows = dq_fused(kp, vp) ? 0 : h.m;
  w.Dh[0] = ws.take<__half>(dh_rows * w.ld);
  w.Dh[1] = ws.take<__half>(dh_rows * w.ld);
  w.cs = ws.take<float2>(h.m * (h.head_dim / 2));
  w.tail = ws.take<uint8_t>(dq_fused(kp, vp) ? dq_tail_bytes(h.m, std::max(kp->n_tail, vp->n_tail)) : 0);
  const size_t rw = (h.flags & kFlagRans) ? rans_decode_workspace(kRansMaxClasses) : 0;
  w.rans_ws[0] = ws.take<uint8_t>(rw);
  w.rans_ws[1] = ws.take<uint8_t>(rw);
  w.ictr = ws.take<uint32_t>(ictr_words(h.m));
  return w;
}

// Both sections through ONE inflate launch (the inflater is latency-bound: as a
// bounded side-stream grid it ran 3-5x slower and delayed the values' GEMM).
// Every read is bounded by the section lengths of the validated header.
kvtc_status enqueue_inflate(const uint8_t *ib, const ContainerHeader &h, const DecompWs &w, cudaStream_t st) {
  uint32_t nch[2];
  for (int sv = 0; sv < 2; ++sv) nch[sv] = uint32_t((h.payload_bytes[sv] + h.chunk_bytes - 1) / h.chunk_bytes);
  if (h.flags & kFlagRans) {
    // rANS sections (Q24): tables + decode per stream; a bad section sets w.err
    ProfScope ps("d.rans_decode", st);
    for (int sv = 0; sv < 2; ++sv) {
      kvtc_status s = launch_rans_decode(ib + h.section_off[sv], h.entropy_bytes[sv], h.payload_bytes[sv], nch[sv],
                                         kRansMaxClasses, w.payloads[sv], w.rans_ws[sv], w.err, st);
      if (s) return s;
    }
    return KVTC_OK;
  }
  ProfScope ps("d.inflate", st);
  return launch_inflate_sections(ib + h.section_off[0], h.entropy_bytes[0], h.payload_bytes[0], nch[0], w.payloads[0],
                                 ib + h.section_off[1], h.entropy_bytes[1], h.payload_bytes[1], nch[1], w.payloads[1],
                                 w.err, st);
}
// Both sections inflated AND dequantised by one launch (inflate_dequant_kernel):
// each 32-row block of D^ is expanded as soon as its tile's chunks are inflated.
kvtc_status enqueue_inflate_dequant(const uint8_t *ib, const ContainerHeader &h, const DecompWs &w,
                                    const kvtc_plan *kp, const kvtc_plan *vp, cudaStream_t st) {
  ProfScope ps("d.inflate_dequant", st);
  KVTC_CUDA_TRY(cudaMemsetAsync(w.ictr, 0, size_t(ictr_words(h.m)) * 4, st));
  InflateDqArgs a{};
  const int64_t ntiles = ceil_div(h.m, kTileM);
  for (int sv = 0; sv < 2; ++sv) {
    kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
    InflateDqStream &x = a.s[sv];
    x.sec = ib + h.section_off[sv];
    x.sec_len = h.entropy_bytes[sv];
    x.n_out = h.payload_bytes[sv];
    x.nch = uint32_t((h.payload_bytes[sv] + h.chunk_bytes - 1) / h.chunk_bytes);
    x.out = w.payloads[sv];
    x.dq = DqArgs{pl->d_dqchunks, pl->d_dqcols, int32_t((pl->r_nz + 7) / 8), pl->d_codes_off_full,
                  plan_codes_off_last(pl, h.m % kTileM), pl->tile_bytes, w.payloads[sv], h.m, w.Dh[sv], w.ld};
    x.nbx = uint32_t(ceil_div(x.dq.nch8, 32));
    x.ndq = pl->r_nz ? uint32_t(x.nbx * ntiles) : 0u;
    x.tile_done = w.ictr + 2 + sv * ntiles;
    if (!pl->r_nz) KVTC_CUDA_TRY(cudaMemsetAsync(w.Dh[sv], 0, h.m * w.ld * 2, st));
  }
  KVTC_CHECK_ARG(h.chunk_bytes == 16384 || h.chunk_bytes == 32768 || h.chunk_bytes == 65536, "chunk bytes");
  a.cb_shift = h.chunk_bytes == 16384 ? 14 : (h.chunk_bytes == 32768 ? 15 : 16);
  a.ctr = w.ictr;
  a.err = w.err;
  return launch_inflate_dequant(a, st);
}
// Checksums of the inflated payloads and of the raw section against the header
// (integrity.cu): mismatch bits 1 / 2 (payload K / V), 4 (raw section).
kvtc_status enqueue_checks(const uint8_t *ib, const ContainerHeader &h, const DecompWs &w, cudaStream_t q,
                           int32_t ctas) {
  kvtc_status s;
  if (h.m)
    for (int sv = 0; sv < 2; ++sv)
      if ((s = launch_hash(w.payloads[sv], h.payload_bytes[sv], kSeedPayload, w.hsum + sv, q, ctas)) ||
          (s = launch_hash_check(w.hsum + sv, h.payload_hash[sv], 1 << sv, w.err + 1, q)))
        return s;
  if ((s = launch_hash(ib + h.raw_off, h.raw_bytes, kSeedRaw, w.hsum + 2, q, ctas)) ||
      (s = launch_hash_check(w.hsum + 2, h.raw_hash, 4, w.err + 1, q)))
    return s;
  return KVTC_OK;
}
kvtc_status enqueue_status(const DecompWs &w, int32_t *status_dev, cudaStream_t st) {
  status_kernel<<<1, 1, 0, st>>>(w.err, 2, status_dev ? status_dev : w.err + 2);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}
kvtc_status read_status(const DecompWs &w, cudaStream_t st) {
  int32_t v = 0;
  KVTC_CUDA_TRY(cudaMemcpyAsync(&v, w.err + 2, 4, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  if (v) {
    set_error("corrupt container: DEFLATE stream or checksum mismatch");
    return KVTC_E_CORRUPT;
  }
  return KVTC_OK;
}

// The whole decompression of a validated header, enqueued without host
// synchronisation.  Schedule: keys: dequantise -> GEMM on the caller's stream;
// values: dequantise + the checksums on the side stream (bounded grid, beside the
// keys' GEMM) -> GEMM; then the raw sinks / window and the status word.
kvtc_status decompress_enqueue(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb, const kvtc_plan *vp,
                               const uint8_t *ib, const ContainerHeader &h, int32_t layer_begin, int32_t layer_end,
                               const kvtc_kv_view *k_out, const kvtc_kv_view *v_out, int32_t *status_dev,
                               void *workspace, size_t workspace_bytes, cudaStream_t st) {
  kvtc_status s;
  if ((s = check_view(k_out)) || (s = check_view(v_out))) return s;
  const kvtc_shape shp{h.layers, h.kv_heads, h.head_dim};
  if (!same_shape(shp, k_out->shape) || !same_shape(shp, v_out->shape) || k_out->tokens != h.tokens ||
      v_out->tokens != h.tokens) {
    set_error("container shape does not match the output views");
    return KVTC_E_MISMATCH;
  }
  KVTC_CHECK_ARG(0 <= layer_begin && layer_begin <= layer_end && layer_end <= h.layers, "layer range");
  KVTC_CHECK_ARG((reinterpret_cast<uintptr_t>(ib) & 15) == 0, "container must be 16-byte aligned");
  const size_t need = kvtc_decompress_workspace_bytes(kb, kp, vb, vp, &h);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu < %zu", workspace_bytes, need);
    return KVTC_E_CAPACITY;
  }
  DecompWs w = carve_decomp(kp, vp, h, workspace, workspace_bytes);
  if ((s = upload_bases(k_out, w.kbases, st)) || (s = upload_bases(v_out, w.vbases, st))) return s;
  KVTC_CUDA_TRY(cudaMemsetAsync(w.err, 0, 16, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(w.hsum, 0, 32, st));
  const int64_t t = h.tokens;
  const int64_t nraw = h.m ? int64_t(h.sinks) + h.window : t;
  const int64_t hd = int64_t(h.kv_heads) * h.head_dim;
  const auto *rawk = reinterpret_cast<const __nv_bfloat16 *>(ib + h.raw_off);
  const auto *rawv = rawk + int64_t(h.layers) * nraw * hd;
  if (!h.m) {
    if ((s = enqueue_checks(ib, h, w, st, 0))) return s;
    if ((s = launch_unpack_raw(rawk, nraw, 0, t, *k_out, w.kbases, 0, layer_begin, layer_end, st))) return s;
    if ((s = launch_unpack_raw(rawv, nraw, 0, t, *v_out, w.vbases, 0, layer_begin, layer_end, st))) return s;
    return enqueue_status(w, status_dev, st);
  }
  if (kb->has_rope && (s = rope_table_for(kb, h.pos0 + h.sinks, h.m, w.cs, st))) return s;
  SideStream *ss = side_stream();
  const bool ovl = !overlap_off();
  cudaStream_t aux = ovl ? ss->s : st;
  // Only the keys' section is inflated up front; the values' is inflated on the side
  // stream (bounded grid) beside the keys' GEMM.  With the round-2 inflater this is
  // 0.2-0.4 ms per step faster than one two-stream launch up front (in-process
  // interleaved sweeps, profiles/r02k_sweep_inflate_side.log); KVTC_D_INFLATE_SIDE=0
  // restores the single launch.
  const bool inflate_side = ovl && !(h.flags & kFlagRans) && env_flag("KVTC_D_INFLATE_SIDE", true);
  // KVTC_D_INFLATE_DQ=1: one launch inflates and dequantises both streams
  // (inflate_dequant_kernel; measured slower than the split path: 1.25-1.32 vs
  // 0.79 ms in the step); default: the inflater, then the
  // dequantiser per stream -- keys here, values beside the keys' GEMM
  const bool front = !inflate_side && !(h.flags & kFlagRans) && !dq_fused(kp, vp) &&
                     env_flag("KVTC_D_INFLATE_DQ", false);
  if (front) {
    if ((s = enqueue_inflate_dequant(ib, h, w, kp, vp, st))) return s;
  } else if (inflate_side) {
    ProfScope ps("d.inflate_k", st);
    const uint32_t nk = uint32_t((h.payload_bytes[0] + h.chunk_bytes - 1) / h.chunk_bytes);
    if ((s = launch_inflate_section(ib + h.section_off[0], h.entropy_bytes[0], h.payload_bytes[0], nk,
                                    w.payloads[0], w.err, st)))
      return s;
  } else if ((s = enqueue_inflate(ib, h, w, st))) {
    return s;
  }
  const bool fused = dq_fused(kp, vp);
  auto expand = [&](int sv, cudaStream_t q, int ctas) -> kvtc_status {
    if (fused || front) return KVTC_OK;           // dequantised inside the GEMM / the inflater
    kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
    kvtc_status r;
    ProfScope ps(sv && ovl ? "d.dequant_overlapped" : "d.dequant", q);
    if ((r = launch_dequant(pl->d_dqchunks, pl->d_dqcols, pl->r_nz, pl->d_codes_off_full, plan_codes_off_last(pl, h.m % kTileM),
                            pl->tile_bytes, w.payloads[sv], h.m, w.Dh[sv], w.ld, q, ctas)))
      return r;
    if (pl->r_nz == 0) KVTC_CUDA_TRY(cudaMemsetAsync(w.Dh[sv], 0, h.m * w.ld * 2, q));
    return KVTC_OK;
  };
  if ((s = expand(0, st, 0))) return s;
  KVTC_CUDA_TRY(cudaEventRecord(ss->ev[2], st));                 // inflated, keys expanded
  for (int sv = 0; sv < 2; ++sv) {
    const kvtc_basis *b = sv ? vb : kb;
    kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
    const kvtc_kv_view *vw = sv ? v_out : k_out;
    __nv_bfloat16 *const *bs = sv ? w.vbases : w.kbases;
    const Operands *op;
    if ((s = plan_operands(b, pl, &op))) return s;
    if (sv == 1) KVTC_CUDA_TRY(cudaStreamWaitEvent(st, ss->ev[3], 0));   // join: values expanded, checks done
    {
      ProfScope ps("d.reconstruct_gemm", st);
      if ((s = run_reconstruct(b, pl, op, w.Dh[sv], w.ld, h.m, h.sinks, layer_begin, layer_end, vw, bs, w.cs, st,
                               nullptr, w.payloads[sv], fused, w.tail)))
        return s;
    }
    if (sv == 0) {
      KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[2], 0));
      const int ctas = ovl ? corun_ctas(corun_per_sm("KVTC_CORUN_DEQUANT", 2)) : 0;
      if (inflate_side) {
        ProfScope ps("d.inflate_v_overlapped", aux);
        const uint32_t nv = uint32_t((h.payload_bytes[1] + h.chunk_bytes - 1) / h.chunk_bytes);
        if ((s = launch_inflate_section(ib + h.section_off[1], h.entropy_bytes[1], h.payload_bytes[1], nv,
                                        w.payloads[1], w.err, aux, corun_ctas(corun_per_sm("KVTC_CORUN_INFLATE", 4)))))
          return s;
      }
      if ((s = expand(1, aux, ctas))) return s;
      {
        ProfScope ps(ovl ? "d.checksum_overlapped" : "d.checksum", aux);
        if ((s = enqueue_checks(ib, h, w, aux, ctas))) return s;
      }
      {
        // raw sinks + window of both streams (token rows the GEMMs never write)
        ProfScope ps(ovl ? "d.raw_tokens_overlapped" : "d.raw_tokens", aux);
        for (int rv = 0; rv < 2; ++rv) {
          const __nv_bfloat16 *raw = rv ? rawv : rawk;
          const kvtc_kv_view *ow = rv ? v_out : k_out;
          __nv_bfloat16 *const *obs = rv ? w.vbases : w.kbases;
          if ((s = launch_unpack_raw(raw, nraw, 0, h.sinks, *ow, obs, 0, layer_begin, layer_end, aux))) return s;
          if ((s = launch_unpack_raw(raw, nraw, h.sinks, h.window, *ow, obs, t - h.window, layer_begin, layer_end,
                                     aux)))
            return s;
        }
      }
      KVTC_CUDA_TRY(cudaEventRecord(ss->ev[3], aux));
    }
  }
  return enqueue_status(w, status_dev, st);
}
}  // namespace

extern "C" size_t kvtc_decompress_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                                  const kvtc_plan *vp, const void *in_header_host) {
  if (!kb || !kp || !vb || !vp || !in_header_host) return 0;
  ContainerHeader h;
  memcpy(&h, in_header_host, sizeof(h));
  if (validate_header(h) != KVTC_OK) return 0;     // the call itself reports why
  Bump b;
  b.take<void *>(h.layers);
  b.take<void *>(h.layers);
  b.take<int32_t>(4);
  b.take<uint64_t>(4);
  b.take<uint8_t>(h.payload_bytes[0] + 16);
  b.take<uint8_t>(h.payload_bytes[1] + 16);
  const int64_t dh_rows = dq_fused(kp, vp) ? 0 : h.m;
  b.take<__half>(dh_rows * std::max(std::max(kp->r_nz_pad, vp->r_nz_pad), 8));
  b.take<__half>(dh_rows * std::max(std::max(kp->r_nz_pad, vp->r_nz_pad), 8));
  b.take<float2>(h.m * (kb->shape.head_dim / 2));
  b.take<uint8_t>(dq_fused(kp, vp) ? dq_tail_bytes(h.m, std::max(kp->n_tail, vp->n_tail)) : 0);
  b.take<uint8_t>((h.flags & kFlagRans) ? rans_decode_workspace(kRansMaxClasses) : 0);
  b.take<uint8_t>((h.flags & kFlagRans) ? rans_decode_workspace(kRansMaxClasses) : 0);
  b.take<uint32_t>(2 + 2 * ((h.m + kTileM - 1) / kTileM));
  return b.used + 256;
}

extern "C" kvtc_status kvtc_decompress(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                       const kvtc_plan *vp, const void *in, size_t in_len, int32_t layer_begin,
                                       int32_t layer_end, const kvtc_kv_view *k_out, const kvtc_kv_view *v_out,
                                       void *workspace, size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && in && k_out && v_out, "decompress arguments");
  KVTC_CHECK_ARG(in_len >= KVTC_HEADER_BYTES, "container too short");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ContainerHeader hh, h;
  KVTC_CUDA_TRY(cudaMemcpyAsync(&hh, in, sizeof(hh), cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  kvtc_status s = read_checked_header(kb, kp, vb, vp, &hh, in_len, &h);
  if (s) return s;
  if ((s = decompress_enqueue(kb, kp, vb, vp, static_cast<const uint8_t *>(in), h, layer_begin, layer_end, k_out,
                              v_out, nullptr, workspace, workspace_bytes, st)))
    return s;
  return read_status(carve_decomp(kp, vp, h, workspace, workspace_bytes), st);
}

extern "C" kvtc_status kvtc_decompress_async(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                             const kvtc_plan *vp, const void *in, size_t in_len,
                                             const void *header_host, int32_t layer_begin, int32_t layer_end,
                                             const kvtc_kv_view *k_out, const kvtc_kv_view *v_out,
                                             int32_t *status_dev, void *workspace, size_t workspace_bytes,
                                             void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && in && header_host && k_out && v_out, "decompress_async arguments");
  KVTC_CHECK_ARG(in_len >= KVTC_HEADER_BYTES, "container too short");
  ContainerHeader h;
  kvtc_status s = read_checked_header(kb, kp, vb, vp, header_host, in_len, &h);
  if (s) return s;
  return decompress_enqueue(kb, kp, vb, vp, static_cast<const uint8_t *>(in), h, layer_begin, layer_end, k_out, v_out,
                            status_dev, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

// ============================================== layer-streamed decompression
// "the inverse projection ... can be performed layer-by-layer using
// sub-matrices of V^T, allowing generation to begin early".  The coefficients D^
// mix all layers, so inflate + dequantise run ONCE (kvtc_decompress_begin, into
// the caller's workspace, which also verifies the checksums); each
// kvtc_decompress_layers call then runs only the reconstruction GEMMs over its
// layers' h*d columns of V_d^T (and copies those layers' raw tokens), so a
// consumer can start on layer 0 while later layers are still being rebuilt.
// Workspace layout = kvtc_decompress's.
extern "C" kvtc_status kvtc_decompress_begin(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                             const kvtc_plan *vp, const void *in, size_t in_len, void *workspace,
                                             size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && in && in_len >= KVTC_HEADER_BYTES, "decompress_begin arguments");
  KVTC_CHECK_ARG((reinterpret_cast<uintptr_t>(in) & 15) == 0, "container must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ContainerHeader hh;
  KVTC_CUDA_TRY(cudaMemcpyAsync(&hh, in, sizeof(hh), cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  ContainerHeader h;
  kvtc_status s = read_checked_header(kb, kp, vb, vp, &hh, in_len, &h);
  if (s) return s;
  const size_t need = kvtc_decompress_workspace_bytes(kb, kp, vb, vp, &h);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu < %zu", workspace_bytes, need);
    return KVTC_E_CAPACITY;
  }
  DecompWs w = carve_decomp(kp, vp, h, workspace, workspace_bytes);
  const uint8_t *ib = static_cast<const uint8_t *>(in);
  KVTC_CUDA_TRY(cudaMemsetAsync(w.err, 0, 16, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(w.hsum, 0, 32, st));
  if (h.m && !(h.flags & kFlagRans) && !dq_fused(kp, vp) && env_flag("KVTC_D_INFLATE_DQ", false)) {
    if ((s = enqueue_inflate_dequant(ib, h, w, kp, vp, st))) return s;
    if (kb->has_rope && (s = rope_table_for(kb, h.pos0 + h.sinks, h.m, w.cs, st))) return s;
  } else if (h.m) {
    if ((s = enqueue_inflate(ib, h, w, st))) return s;
    ProfScope ps("d.dequant", st);
    for (int sv = 0; sv < 2 && !dq_fused(kp, vp); ++sv) {
      kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
      if ((s = launch_dequant(pl->d_dqchunks, pl->d_dqcols, pl->r_nz, pl->d_codes_off_full, plan_codes_off_last(pl, h.m % kTileM),
                              pl->tile_bytes, w.payloads[sv], h.m, w.Dh[sv], w.ld, st)))
        return s;
      if (pl->r_nz == 0) KVTC_CUDA_TRY(cudaMemsetAsync(w.Dh[sv], 0, h.m * w.ld * 2, st));
    }
    if (kb->has_rope && (s = rope_table_for(kb, h.pos0 + h.sinks, h.m, w.cs, st))) return s;
  }
  if ((s = enqueue_checks(ib, h, w, st, 0)) || (s = enqueue_status(w, nullptr, st))) return s;
  return read_status(w, st);
}

extern "C" kvtc_status kvtc_decompress_layers(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                              const kvtc_plan *vp, const void *in, const void *header_host,
                                              int32_t layer_begin, int32_t layer_end, const kvtc_kv_view *k_out,
                                              const kvtc_kv_view *v_out, void *workspace, size_t workspace_bytes,
                                              void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && in && header_host && k_out && v_out, "decompress_layers arguments");
  kvtc_status s;
  if ((s = check_view(k_out)) || (s = check_view(v_out))) return s;
  ContainerHeader h;
  if ((s = read_checked_header(kb, kp, vb, vp, header_host, 0, &h))) return s;
  const kvtc_shape shp{h.layers, h.kv_heads, h.head_dim};
  if (!same_shape(shp, k_out->shape) || !same_shape(shp, v_out->shape) || k_out->tokens != h.tokens ||
      v_out->tokens != h.tokens) {
    set_error("container shape does not match the output views");
    return KVTC_E_MISMATCH;
  }
  KVTC_CHECK_ARG(0 <= layer_begin && layer_begin <= layer_end && layer_end <= h.layers, "layer range");
  const size_t need = kvtc_decompress_workspace_bytes(kb, kp, vb, vp, &h);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu < %zu", workspace_bytes, need);
    return KVTC_E_CAPACITY;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DecompWs w = carve_decomp(kp, vp, h, workspace, workspace_bytes);
  if ((s = upload_bases(k_out, w.kbases, st)) || (s = upload_bases(v_out, w.vbases, st))) return s;
  const uint8_t *ib = static_cast<const uint8_t *>(in);
  const int64_t t = h.tokens;
  const int64_t nraw = h.m ? int64_t(h.sinks) + h.window : t;
  const int64_t hd = int64_t(h.kv_heads) * h.head_dim;
  const auto *rawk = reinterpret_cast<const __nv_bfloat16 *>(ib + h.raw_off);
  const auto *rawv = rawk + int64_t(h.layers) * nraw * hd;
  for (int sv = 0; sv < 2; ++sv) {
    const kvtc_basis *b = sv ? vb : kb;
    kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
    const kvtc_kv_view *vw = sv ? v_out : k_out;
    __nv_bfloat16 *const *bs = sv ? w.vbases : w.kbases;
    const __nv_bfloat16 *raw = sv ? rawv : rawk;
    if (!h.m) {
      if ((s = launch_unpack_raw(raw, nraw, 0, t, *vw, bs, 0, layer_begin, layer_end, st))) return s;
      continue;
    }
    const Operands *op;
    if ((s = plan_operands(b, pl, &op))) return s;
    {
      ProfScope ps("d.reconstruct_gemm", st);
      if ((s = run_reconstruct(b, pl, op, w.Dh[sv], w.ld, h.m, h.sinks, layer_begin, layer_end, vw, bs, w.cs, st,
                               nullptr, w.payloads[sv], dq_fused(kp, vp), w.tail)))
        return s;
    }
    if ((s = launch_unpack_raw(raw, nraw, 0, h.sinks, *vw, bs, 0, layer_begin, layer_end, st))) return s;
    if ((s = launch_unpack_raw(raw, nraw, h.sinks, h.window, *vw, bs, t - h.window, layer_begin, layer_end, st)))
      return s;
  }
  return KVTC_OK;
}

// ================================================================ batched codec
// Several conversations (or token ranges of conversations) in one call: their
// middle tokens are concatenated, each padded to whole 128-token tiles, so both
// projection GEMMs (and both reconstruction GEMMs) run ONCE over all rows; a
// per-tile table (TileRef) sends each tile's epilogue to its own conversation's
// payload (compress) or cache view (decompress).  Rows are independent under the
// per-token quantisation reading (Q1), so every output is byte-identical to the
// single-conversation call; the DEFLATE encoder and the inflater also run once
// over all chunks of all payloads.  Serving with many short requests and the
// incremental compression of c = 16 tokens per turn need exactly this.
namespace {
struct BatchItem {
  CompressLayout L;
  int64_t row0 = 0;      // first GEMM row (tile-aligned)
  int64_t tiles = 0;
};
int64_t batch_rows(const std::vector<BatchItem> &it) {
  int64_t r = 0;
  for (auto &b : it) r += b.tiles * kTileM;
  return r;
}
}  // namespace

extern "C" size_t kvtc_compress_batch_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                                      const kvtc_plan *vp, const kvtc_kv_view *k, int32_t n,
                                                      const kvtc_policy *pol) {
  if (!kb || !kp || !vb || !vp || !k || n <= 0 || !pol) return 0;
  Bump b;
  int64_t rows = 0;
  for (int i = 0; i < n; ++i) {
    const CompressLayout L = compress_layout(kp, vp, &k[i], pol);
    rows += (L.m + kTileM - 1) / kTileM * kTileM;
    b.take<void *>(k[i].shape.layers);
    b.take<void *>(k[i].shape.layers);
    b.take<uint8_t>(L.pay[0] + 16);
    b.take<uint8_t>(L.pay[1] + 16);
    b.take<uint8_t>(deflate_workspace(L.pay[0], pol->chunk_bytes));
    b.take<uint8_t>(deflate_workspace(L.pay[1], pol->chunk_bytes));
  }
  b.take<uint64_t>(kCompressWords * int64_t(n));
  b.take<__nv_bfloat16>(rows * (kb->p + kXPad));
  b.take<__nv_bfloat16>(rows * (kb->p + kXPad));
  b.take<float2>(rows * (kb->shape.head_dim / 2));
  b.take<uint8_t>(wide_scratch_bytes(rows, std::max(kp->wide_cols, vp->wide_cols), std::max(kp->nwide, vp->nwide)));
  b.take<TileRef>(2 * (rows / kTileM));
  b.take<EncodeJob>(2 * int64_t(n));
  b.take<HashJob>(3 * int64_t(n));
  return b.used + 256;
}

extern "C" kvtc_status kvtc_compress_batch(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                           const kvtc_plan *vp, const kvtc_kv_view *k, const kvtc_kv_view *v,
                                           int32_t n, const kvtc_policy *pol, void *const *out_host,
                                           const size_t *out_cap_host, size_t *out_len_host, void *workspace,
                                           size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && k && v && pol && out_host && out_cap_host && n > 0, "compress_batch arguments");
  KVTC_CHECK_ARG(kb->which == KVTC_KEYS && vb->which == KVTC_VALUES, "basis streams");
  KVTC_CHECK_ARG(pol->sinks >= 0 && pol->window >= 0, "policy");
  KVTC_CHECK_ARG(pol->chunk_bytes == 16384 || pol->chunk_bytes == 32768 || pol->chunk_bytes == 65536, "chunk_bytes");
  KVTC_CHECK_ARG(pol->coder == KVTC_CODER_DEFLATE, "batched compression writes DEFLATE sections (coder 0)");
  kvtc_status s;
  std::vector<BatchItem> it(n);
  int64_t row = 0;
  for (int i = 0; i < n; ++i) {
    if ((s = check_view(&k[i])) || (s = check_view(&v[i]))) return s;
    KVTC_CHECK_ARG(same_shape(k[i].shape, v[i].shape) && k[i].tokens == v[i].tokens && k[i].pos0 == v[i].pos0,
                   "key and value views differ");
    KVTC_CHECK_ARG(same_shape(k[i].shape, kb->shape) && same_shape(v[i].shape, vb->shape), "basis shape mismatch");
    it[i].L = compress_layout(kp, vp, &k[i], pol);
    if (out_cap_host[i] < it[i].L.bound) {
      set_error("batch item %d: output capacity %zu < bound %llu", i, out_cap_host[i],
                (unsigned long long)it[i].L.bound);
      return KVTC_E_CAPACITY;
    }
    it[i].row0 = row;
    it[i].tiles = (it[i].L.m + kTileM - 1) / kTileM;
    row += it[i].tiles * kTileM;
  }
  const size_t need = kvtc_compress_batch_workspace_bytes(kb, kp, vb, vp, k, n, pol);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu < %zu", workspace_bytes, need);
    return KVTC_E_CAPACITY;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto *kpl = const_cast<kvtc_plan *>(kp);
  auto *vpl = const_cast<kvtc_plan *>(vp);
  const Operands *kop, *vop;
  if ((s = plan_operands(kb, kpl, &kop)) || (s = plan_operands(vb, vpl, &vop))) return s;
  const int64_t rows = row, ntiles = rows / kTileM;
  const int half = kb->shape.head_dim / 2;
  const int64_t ldx = kb->p + kXPad;
  Bump ws(workspace, workspace_bytes);
  std::vector<__nv_bfloat16 **> kbases(n), vbases(n);
  std::vector<uint8_t *> pay_k(n), pay_v(n);
  std::vector<void *> dws_k(n), dws_v(n);
  for (int i = 0; i < n; ++i) {
    kbases[i] = ws.take<__nv_bfloat16 *>(k[i].shape.layers);
    vbases[i] = ws.take<__nv_bfloat16 *>(k[i].shape.layers);
    pay_k[i] = ws.take<uint8_t>(it[i].L.pay[0] + 16);
    pay_v[i] = ws.take<uint8_t>(it[i].L.pay[1] + 16);
    dws_k[i] = ws.take<uint8_t>(deflate_workspace(it[i].L.pay[0], pol->chunk_bytes));
    dws_v[i] = ws.take<uint8_t>(deflate_workspace(it[i].L.pay[1], pol->chunk_bytes));
  }
  uint64_t *lens = ws.take<uint64_t>(kCompressWords * int64_t(n));   // per item: see kCompressWords
  auto *X = ws.take<__nv_bfloat16>(rows * ldx);
  auto *X2 = ws.take<__nv_bfloat16>(rows * ldx);          // the values' rows (gathered beside the keys' GEMM)
  float2 *cs = ws.take<float2>(rows * half);
  float *wide = reinterpret_cast<float *>(
      ws.take<uint8_t>(wide_scratch_bytes(rows, std::max(kp->wide_cols, vp->wide_cols), std::max(kp->nwide, vp->nwide))));
  TileRef *d_tiles = ws.take<TileRef>(2 * ntiles);
  EncodeJob *d_jobs = ws.take<EncodeJob>(2 * int64_t(n));
  HashJob *d_hjobs = ws.take<HashJob>(3 * int64_t(n));            // raw sections, K payloads, V payloads

  // raw tokens, headers' host part, section offsets
  std::vector<ContainerHeader> hdr(n);
  std::vector<uint64_t> offs(kCompressWords * int64_t(n), 0);
  std::vector<HashJob> hjobs(3 * int64_t(n));
  uint64_t max_raw = 0, max_pay[2] = {0, 0};
  for (int i = 0; i < n; ++i) {
    if ((s = upload_bases(&k[i], kbases[i], st)) || (s = upload_bases(&v[i], vbases[i], st))) return s;
    const CompressLayout &L = it[i].L;
    ContainerHeader &h = hdr[i];
    h = ContainerHeader{};
    h.magic = kContainerMagic;
    h.version = kContainerVersion;
    h.layers = k[i].shape.layers;
    h.kv_heads = k[i].shape.kv_heads;
    h.head_dim = k[i].shape.head_dim;
    h.sinks = pol->sinks;
    h.window = pol->window;
    h.chunk_bytes = pol->chunk_bytes;
    h.tokens = k[i].tokens;
    h.pos0 = k[i].pos0;
    h.m = L.m;
    h.raw_bytes = L.raw_bytes;
    h.payload_bytes[0] = L.pay[0];
    h.payload_bytes[1] = L.pay[1];
    h.basis_fp[0] = kb->fp;
    h.basis_fp[1] = vb->fp;
    h.plan_fp[0] = kp->fp;
    h.plan_fp[1] = vp->fp;
    h.raw_off = KVTC_HEADER_BYTES;
    h.section_off[1] = L.k_off;                // the values' section first
    offs[kCompressWords * i + 3] = L.k_off;
    uint8_t *o = static_cast<uint8_t *>(out_host[i]);
    const int64_t hd = int64_t(k[i].shape.kv_heads) * k[i].shape.head_dim;
    auto *rawk = reinterpret_cast<__nv_bfloat16 *>(o + KVTC_HEADER_BYTES);
    auto *rawv = rawk + int64_t(k[i].shape.layers) * L.nraw * hd;
    const int64_t t = k[i].tokens;
    if (L.m) {
      for (int sv = 0; sv < 2; ++sv) {
        const kvtc_kv_view *vw = sv ? &v[i] : &k[i];
        __nv_bfloat16 *const *bs = sv ? vbases[i] : kbases[i];
        __nv_bfloat16 *dst = sv ? rawv : rawk;
        if ((s = launch_pack_raw(*vw, bs, 0, pol->sinks, dst, L.nraw, 0, st))) return s;
        if ((s = launch_pack_raw(*vw, bs, t - pol->window, pol->window, dst, L.nraw, pol->sinks, st))) return s;
      }
    } else {
      if ((s = launch_pack_raw(k[i], kbases[i], 0, t, rawk, L.nraw, 0, st))) return s;
      if ((s = launch_pack_raw(v[i], vbases[i], 0, t, rawv, L.nraw, 0, st))) return s;
    }
    uint64_t *li = lens + kCompressWords * i;
    hjobs[i] = HashJob{reinterpret_cast<const uint8_t *>(rawk), uint64_t(L.raw_bytes), kSeedRaw, li + 7};
    for (int sv = 0; sv < 2; ++sv)
      hjobs[(1 + sv) * int64_t(n) + i] = HashJob{sv ? pay_v[i] : pay_k[i], L.pay[sv], kSeedPayload, li + 5 + sv};
    max_raw = std::max<uint64_t>(max_raw, L.raw_bytes);
    for (int sv = 0; sv < 2; ++sv) max_pay[sv] = std::max<uint64_t>(max_pay[sv], L.m ? L.pay[sv] : 0);
  }
  KVTC_CUDA_TRY(cudaMemcpyAsync(lens, offs.data(), offs.size() * 8, cudaMemcpyHostToDevice, st));
  KVTC_CUDA_TRY(cudaMemcpyAsync(d_hjobs, hjobs.data(), hjobs.size() * sizeof(HashJob), cudaMemcpyHostToDevice, st));
  if ((s = launch_hash_batch(d_hjobs, n, max_raw, st))) return s;
  // tile tables: keys [0, ntiles), values [ntiles, 2 ntiles)
  std::vector<TileRef> tref(2 * ntiles);
  for (int i = 0; i < n; ++i) {
    for (int64_t j = 0; j < it[i].tiles; ++j) {
      const int ntok = int(std::min<int64_t>(kTileM, it[i].L.m - j * kTileM));
      for (int sv = 0; sv < 2; ++sv) {
        kvtc_plan *pl = sv ? vpl : kpl;
        TileRef &r = tref[sv * ntiles + it[i].row0 / kTileM + j];
        r = TileRef{};
        r.payload = (sv ? pay_v[i] : pay_k[i]) + j * pl->tile_bytes;
        r.codes_off = plan_codes_off_last(pl, ntok);
        r.ntok = ntok;
        r.status = reinterpret_cast<int32_t *>(lens + kCompressWords * i + 4);
        if (!r.codes_off) {
          set_error("code offsets: allocation failed");
          return KVTC_E_NOMEM;
        }
      }
    }
  }
  if (ntiles)
    KVTC_CUDA_TRY(cudaMemcpyAsync(d_tiles, tref.data(), tref.size() * sizeof(TileRef), cudaMemcpyHostToDevice, st));
  // Schedule (as kvtc_compress): st: keys' gathers -> keys' GEMM ->
  // values' GEMM -> values' DEFLATE -> assemble; aux (bounded grids beside the
  // GEMMs): values' gathers into X2, then the keys' DEFLATE.
  SideStream *ss = side_stream();
  const bool ovl = !overlap_off();
  cudaStream_t aux = ovl ? ss->s : st;
  KVTC_CUDA_TRY(cudaEventRecord(ss->ev[0], st));                 // bases, raw tokens, tables uploaded
  std::vector<EncodeJob> jobs[2];
  uint32_t nchunks[2] = {0, 0};
  for (int sv = 0; sv < 2; ++sv)
    for (int i = 0; i < n; ++i) {
      const uint64_t pb = it[i].L.pay[sv];
      if (!it[i].L.m || pb == 0) continue;
      EncodeJob j{};
      j.in = sv ? pay_v[i] : pay_k[i];
      j.n = pb;
      j.ws = sv ? dws_v[i] : dws_k[i];
      j.chunk0 = nchunks[sv];
      nchunks[sv] += uint32_t((pb + pol->chunk_bytes - 1) / pol->chunk_bytes);
      jobs[sv].push_back(j);
    }
  for (int sv = 0; sv < 2; ++sv)
    if (!jobs[sv].empty())
      KVTC_CUDA_TRY(cudaMemcpyAsync(d_jobs + sv * n, jobs[sv].data(), jobs[sv].size() * sizeof(EncodeJob),
                                    cudaMemcpyHostToDevice, st));
  if (ntiles) {
    {
      ProfScope ps("cb.gather_unrope", st);
      for (int i = 0; i < n; ++i) {
        if (!it[i].L.m) continue;
        if ((s = rope_table_for(kb, k[i].pos0 + pol->sinks, it[i].L.m, cs + it[i].row0 * half, st))) return s;
        if ((s = launch_gather(k[i], kbases[i], pol->sinks, it[i].L.m, cs + it[i].row0 * half, kb->pairing,
                               X + it[i].row0 * ldx, st, 0, ldx)))
          return s;
      }
    }
    {
      ProfScope ps("cb.project_quant_gemm", st);
      if ((s = run_project_quant(kb, kpl, kop, X, rows, nullptr, wide, st, nullptr, 0, ldx, d_tiles))) return s;
    }
    KVTC_CUDA_TRY(cudaEventRecord(ss->ev[2], st));               // keys' payloads ready
    KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[0], 0));
    {
      ProfScope ps(ovl ? "cb.gather_overlapped" : "cb.gather", aux);
      for (int i = 0; i < n; ++i) {
        if (!it[i].L.m) continue;
        if ((s = launch_gather(v[i], vbases[i], pol->sinks, it[i].L.m, nullptr, 0, X2 + it[i].row0 * ldx, aux,
                               ovl ? corun_ctas(3) : 0, ldx)))
          return s;
      }
    }
    KVTC_CUDA_TRY(cudaEventRecord(ss->ev[1], aux));              // values gathered
    KVTC_CUDA_TRY(cudaStreamWaitEvent(st, ss->ev[1], 0));
    {
      ProfScope ps("cb.project_quant_gemm", st);
      if ((s = run_project_quant(vb, vpl, vop, X2, rows, nullptr, wide, st, nullptr, 0, ldx, d_tiles + ntiles)))
        return s;
    }
    KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[2], 0));
    {
      ProfScope ps(ovl ? "cb.deflate_overlapped" : "cb.deflate", aux);
      if ((s = launch_hash_batch(d_hjobs + n, n, max_pay[0], aux, ovl ? corun_ctas(2) : 0))) return s;
      if (!jobs[0].empty() &&
          (s = launch_deflate_encode_batch(d_jobs, int32_t(jobs[0].size()), nchunks[0], pol->chunk_bytes, aux,
                                           ovl ? corun_ctas(2) : 0)))
        return s;
    }
    {
      ProfScope ps("cb.deflate", st);
      if ((s = launch_hash_batch(d_hjobs + 2 * int64_t(n), n, max_pay[1], st))) return s;
      if (!jobs[1].empty() &&
          (s = launch_deflate_encode_batch(d_jobs + n, int32_t(jobs[1].size()), nchunks[1], pol->chunk_bytes, st)))
        return s;
    }
  }
  KVTC_CUDA_TRY(cudaEventRecord(ss->ev[3], aux));
  KVTC_CUDA_TRY(cudaStreamWaitEvent(st, ss->ev[3], 0));          // join
  {
    ProfScope ps("cb.assemble", st);
    for (int i = 0; i < n; ++i) {
      uint8_t *o = static_cast<uint8_t *>(out_host[i]);
      uint64_t *li = lens + kCompressWords * i;
      if (!it[i].L.m) {
        header_kernel<<<1, 1, 0, st>>>(hdr[i], o, nullptr, li);
        KVTC_LAUNCH_CHECK();
        continue;
      }
      if ((s = launch_deflate_assemble(it[i].L.pay[1], pol->chunk_bytes, dws_v[i], o, li + 3, li + 1, st))) return s;
      offset_after_kernel<<<1, 1, 0, st>>>(li + 3, li + 1, li + 2, o);
      KVTC_LAUNCH_CHECK();
      if ((s = launch_deflate_assemble(it[i].L.pay[0], pol->chunk_bytes, dws_k[i], o, li + 2, li + 0, st))) return s;
      header_kernel<<<1, 1, 0, st>>>(hdr[i], o, li, li);
      KVTC_LAUNCH_CHECK();
    }
  }
  if (out_len_host) {
    std::vector<uint64_t> l(kCompressWords * int64_t(n));
    KVTC_CUDA_TRY(cudaMemcpyAsync(l.data(), lens, l.size() * 8, cudaMemcpyDeviceToHost, st));
    KVTC_CUDA_TRY(cudaStreamSynchronize(st));
    int bad = -1;
    for (int i = 0; i < n; ++i) {
      const uint64_t *li = l.data() + kCompressWords * i;
      out_len_host[i] = it[i].L.m ? size_t(li[2] + li[0]) : size_t(KVTC_HEADER_BYTES + it[i].L.raw_bytes);
      if ((li[4] & 1) && bad < 0) bad = i;
    }
    if (bad >= 0) {
      set_error("batch item %d: a 16-bit shift/scale overflowed (container flagged)", bad);
      return KVTC_E_NUMERIC;
    }
  }
  return KVTC_OK;
}

extern "C" size_t kvtc_decompress_batch_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                                        const kvtc_plan *vp, const void *const *in_header_host,
                                                        int32_t n) {
  if (!kb || !kp || !vb || !vp || !in_header_host || n <= 0) return 0;
  Bump b;
  int64_t rows = 0;
  for (int i = 0; i < n; ++i) {
    ContainerHeader h;
    memcpy(&h, in_header_host[i], sizeof(h));
    if (validate_header(h) != KVTC_OK) return 0;   // the call itself reports why
    rows += (h.m + kTileM - 1) / kTileM * kTileM;
    b.take<void *>(h.layers);
    b.take<void *>(h.layers);
    b.take<uint8_t>(h.payload_bytes[0] + 16);
    b.take<uint8_t>(h.payload_bytes[1] + 16);
  }
  const int64_t ld = std::max(std::max(kp->r_nz_pad, vp->r_nz_pad), 8);
  const int64_t dh_rows = dq_fused(kp, vp) ? 0 : rows;
  b.take<int32_t>(4);
  b.take<__half>(dh_rows * ld);
  b.take<__half>(dh_rows * ld);
  b.take<float2>(rows * (kb->shape.head_dim / 2));
  b.take<uint8_t>(dq_fused(kp, vp) ? dq_tail_bytes(rows, std::max(kp->n_tail, vp->n_tail)) : 0);
  b.take<TileRef>(2 * (rows / kTileM));
  b.take<InflateJob>(2 * int64_t(n));
  b.take<int32_t>(n);
  b.take<uint64_t>(3 * int64_t(n));
  b.take<uint64_t>(3 * int64_t(n));
  b.take<HashJob>(3 * int64_t(n));
  return b.used + 256;
}

namespace {
__global__ void batch_status_kernel(const int32_t *ierr, int32_t n, int32_t *status_out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    status_out[i] = ierr[i] ? int32_t(KVTC_E_CORRUPT) : 0;
}

// The batched decompression of host header copies `hdr` (validated here);
// status_dev (nullable): per-item verdicts written on the stream; otherwise the
// caller synchronises and reads *ierr_out (the per-item error words).
kvtc_status decompress_batch_core(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb, const kvtc_plan *vp,
                                  const void *const *in_host, const size_t *in_len_host, int32_t n,
                                  const kvtc_kv_view *k_out, const kvtc_kv_view *v_out,
                                  std::vector<ContainerHeader> &hdr, int32_t *status_dev, void *workspace,
                                  size_t workspace_bytes, cudaStream_t st, int32_t **ierr_out) {
  kvtc_status s;
  std::vector<BatchItem> it(n);
  std::vector<const void *> hptr(n);
  int64_t row = 0;
  for (int i = 0; i < n; ++i) {
    ContainerHeader h;
    if ((s = read_checked_header(kb, kp, vb, vp, &hdr[i], in_len_host[i], &h))) {
      const std::string msg = kvtc_last_error();
      set_error("batch item %d: %s", i, msg.c_str());
      return s;
    }
    if (h.flags & kFlagRans) {
      set_error("batch item %d: batched decompression reads DEFLATE containers (rANS: kvtc_decompress)", i);
      return KVTC_E_INVALID;
    }
    KVTC_CHECK_ARG((reinterpret_cast<uintptr_t>(in_host[i]) & 15) == 0, "containers must be 16-byte aligned");
    if ((s = check_view(&k_out[i])) || (s = check_view(&v_out[i]))) return s;
    const kvtc_shape shp{h.layers, h.kv_heads, h.head_dim};
    if (!same_shape(shp, k_out[i].shape) || !same_shape(shp, v_out[i].shape) || k_out[i].tokens != h.tokens ||
        v_out[i].tokens != h.tokens) {
      set_error("batch item %d: container shape does not match the output views", i);
      return KVTC_E_MISMATCH;
    }
    it[i].row0 = row;
    it[i].tiles = (h.m + kTileM - 1) / kTileM;
    row += it[i].tiles * kTileM;
    hptr[i] = &hdr[i];
  }
  const size_t need = kvtc_decompress_batch_workspace_bytes(kb, kp, vb, vp, hptr.data(), n);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu < %zu", workspace_bytes, need);
    return KVTC_E_CAPACITY;
  }
  const int64_t rows = row, ntiles = rows / kTileM;
  const int half = kb->shape.head_dim / 2;
  const int64_t ld = std::max(std::max(kp->r_nz_pad, vp->r_nz_pad), 8);
  Bump ws(workspace, workspace_bytes);
  std::vector<__nv_bfloat16 **> kbases(n), vbases(n);
  std::vector<uint8_t *> pay_k(n), pay_v(n);
  for (int i = 0; i < n; ++i) {
    kbases[i] = ws.take<__nv_bfloat16 *>(hdr[i].layers);
    vbases[i] = ws.take<__nv_bfloat16 *>(hdr[i].layers);
    pay_k[i] = ws.take<uint8_t>(hdr[i].payload_bytes[0] + 16);
    pay_v[i] = ws.take<uint8_t>(hdr[i].payload_bytes[1] + 16);
  }
  const bool fused = dq_fused(kp, vp);
  int32_t *err = ws.take<int32_t>(4);
  __half *Dh = ws.take<__half>((fused ? 0 : rows) * ld);
  __half *Dh_v = ws.take<__half>((fused ? 0 : rows) * ld);
  float2 *cs = ws.take<float2>(rows * half);
  uint8_t *dtail = ws.take<uint8_t>(fused ? dq_tail_bytes(rows, std::max(kp->n_tail, vp->n_tail)) : 0);
  TileRef *d_tiles = ws.take<TileRef>(2 * ntiles);
  InflateJob *d_jobs = ws.take<InflateJob>(2 * int64_t(n));
  int32_t *ierr = ws.take<int32_t>(n);                             // per item: inflate error / checksum bits
  *ierr_out = ierr;
  uint64_t *hsum = ws.take<uint64_t>(3 * int64_t(n));              // [raw | K payload | V payload] per item
  uint64_t *hexp = ws.take<uint64_t>(3 * int64_t(n));
  HashJob *d_hj = ws.take<HashJob>(3 * int64_t(n));
  KVTC_CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(ierr, 0, 4 * size_t(n), st));
  KVTC_CUDA_TRY(cudaMemsetAsync(hsum, 0, 24 * size_t(n), st));
  {
    // checksum jobs, item-major: j = 3 i + {0 raw, 1 K payload, 2 V payload}; items
    // without middle tokens compare their (empty) payloads against themselves
    std::vector<HashJob> hj(3 * int64_t(n));
    std::vector<uint64_t> ex(3 * int64_t(n));
    for (int i = 0; i < n; ++i) {
      const ContainerHeader &h = hdr[i];
      const uint8_t *ib = static_cast<const uint8_t *>(in_host[i]);
      hj[3 * i] = HashJob{ib + h.raw_off, h.raw_bytes, kSeedRaw, hsum + 3 * i};
      ex[3 * i] = h.raw_hash;
      for (int sv = 0; sv < 2; ++sv) {
        hj[3 * i + 1 + sv] = HashJob{sv ? pay_v[i] : pay_k[i], h.m ? h.payload_bytes[sv] : 0, kSeedPayload,
                                     hsum + 3 * i + 1 + sv};
        ex[3 * i + 1 + sv] = h.m ? h.payload_hash[sv] : host_hash(nullptr, 0, kSeedPayload);
      }
    }
    KVTC_CUDA_TRY(cudaMemcpyAsync(d_hj, hj.data(), hj.size() * sizeof(HashJob), cudaMemcpyHostToDevice, st));
    KVTC_CUDA_TRY(cudaMemcpyAsync(hexp, ex.data(), ex.size() * 8, cudaMemcpyHostToDevice, st));
  }
  for (int i = 0; i < n; ++i)
    if ((s = upload_bases(&k_out[i], kbases[i], st)) || (s = upload_bases(&v_out[i], vbases[i], st))) return s;
  // every section of every item: one inflate launch
  {
    ProfScope ps("db.inflate", st);
    std::vector<InflateJob> jobs;
    uint32_t c0 = 0;
    for (int i = 0; i < n; ++i)
      for (int sv = 0; sv < 2; ++sv) {
        const ContainerHeader &h = hdr[i];
        if (!h.m || h.payload_bytes[sv] == 0) continue;
        InflateJob j{};
        j.section = static_cast<const uint8_t *>(in_host[i]) + h.section_off[sv];
        j.sec_len = h.entropy_bytes[sv];
        j.n_out = h.payload_bytes[sv];
        j.nch = uint32_t((h.payload_bytes[sv] + h.chunk_bytes - 1) / h.chunk_bytes);
        j.chunk0 = c0;
        j.out = sv ? pay_v[i] : pay_k[i];
        j.err = ierr + i;
        c0 += j.nch;
        jobs.push_back(j);
      }
    if (!jobs.empty()) {
      KVTC_CUDA_TRY(cudaMemcpyAsync(d_jobs, jobs.data(), jobs.size() * sizeof(InflateJob), cudaMemcpyHostToDevice, st));
      if ((s = launch_inflate_batch(d_jobs, int32_t(jobs.size()), c0, err, st))) return s;
    }
  }
  // dequantise into each item's rows (keys on st, values on aux beside the keys'
  // GEMM), RoPE tables, tile tables
  SideStream *ss = side_stream();
  const bool ovl = !overlap_off();
  cudaStream_t aux = ovl ? ss->s : st;
  std::vector<TileRef> tref(2 * ntiles);
  for (int i = 0; i < n; ++i) {
    const ContainerHeader &h = hdr[i];
    for (int64_t j = 0; j < it[i].tiles; ++j)
      for (int sv = 0; sv < 2; ++sv) {
        const kvtc_kv_view &vw = sv ? v_out[i] : k_out[i];
        TileRef &r = tref[sv * ntiles + it[i].row0 / kTileM + j];
        r = TileRef{};
        r.bases = sv ? vbases[i] : kbases[i];
        r.block_table = vw.block_table;
        r.layout = vw.layout;
        r.page_tokens = vw.page_tokens;
        r.tok0 = h.sinks + j * kTileM;
        r.ntok = int(std::min<int64_t>(kTileM, h.m - j * kTileM));
        // the fused inverse path reads this tile's payload bytes
        kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
        r.payload = (sv ? pay_v[i] : pay_k[i]) + j * pl->tile_bytes;
        r.codes_off = r.ntok < kTileM ? plan_codes_off_last(pl, r.ntok) : pl->d_codes_off_full;
      }
  }
  if (ntiles)
    KVTC_CUDA_TRY(cudaMemcpyAsync(d_tiles, tref.data(), tref.size() * sizeof(TileRef), cudaMemcpyHostToDevice, st));
  uint64_t max_n = 0;
  for (int i = 0; i < n; ++i)
    max_n = std::max<uint64_t>(max_n, std::max(hdr[i].raw_bytes, std::max(hdr[i].payload_bytes[0], hdr[i].payload_bytes[1])));
  auto run_checks = [&](cudaStream_t q, int ctas) -> kvtc_status {
    kvtc_status r = launch_hash_batch(d_hj, 3 * n, max_n, q, ctas);
    if (r) return r;
    return launch_hash_check_batch(hsum, hexp, 3 * n, 3, ierr, q);
  };
  auto dequant_all = [&](int sv, cudaStream_t q, int ctas) -> kvtc_status {
    if (fused) return KVTC_OK;                    // dequantised inside the reconstruction GEMM
    kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
    for (int i = 0; i < n; ++i) {
      const ContainerHeader &h = hdr[i];
      if (!h.m) continue;
      __half *D = (sv ? Dh_v : Dh) + it[i].row0 * ld;
      kvtc_status r = launch_dequant(pl->d_dqchunks, pl->d_dqcols, pl->r_nz, pl->d_codes_off_full, plan_codes_off_last(pl, h.m % kTileM),
                                     pl->tile_bytes, sv ? pay_v[i] : pay_k[i], h.m, D, ld, q, ctas);
      if (r) return r;
      if (pl->r_nz == 0) KVTC_CUDA_TRY(cudaMemsetAsync(D, 0, h.m * ld * 2, q));
    }
    return KVTC_OK;
  };
  {
    ProfScope ps("db.dequant", st);
    if ((s = dequant_all(0, st, 0))) return s;
    for (int i = 0; i < n; ++i)
      if (hdr[i].m && kb->has_rope &&
          (s = rope_table_for(kb, hdr[i].pos0 + hdr[i].sinks, hdr[i].m, cs + it[i].row0 * half, st)))
        return s;
  }
  KVTC_CUDA_TRY(cudaEventRecord(ss->ev[2], st));                 // payloads inflated, keys expanded
  for (int sv = 0; sv < 2 && ntiles; ++sv) {
    const kvtc_basis *b = sv ? vb : kb;
    kvtc_plan *pl = const_cast<kvtc_plan *>(sv ? vp : kp);
    const Operands *op;
    if ((s = plan_operands(b, pl, &op))) return s;
    if (sv == 1) KVTC_CUDA_TRY(cudaStreamWaitEvent(st, ss->ev[3], 0));
    {
      ProfScope ps("db.reconstruct_gemm", st);
      // the view arguments only carry the shape here: every tile's output comes from its TileRef
      if ((s = run_reconstruct(b, pl, op, sv ? Dh_v : Dh, ld, rows, 0, 0, b->shape.layers, sv ? &v_out[0] : &k_out[0],
                               sv ? vbases[0] : kbases[0], cs, st, d_tiles + sv * ntiles, nullptr, fused, dtail)))
        return s;
    }
    if (sv == 0) {
      KVTC_CUDA_TRY(cudaStreamWaitEvent(aux, ss->ev[2], 0));
      {
        ProfScope ps(ovl ? "db.dequant_overlapped" : "db.dequant", aux);
        if ((s = dequant_all(1, aux, ovl ? corun_ctas(2) : 0))) return s;
      }
      {
        ProfScope ps(ovl ? "db.checksum_overlapped" : "db.checksum", aux);
        if ((s = run_checks(aux, ovl ? corun_ctas(2) : 0))) return s;
      }
      KVTC_CUDA_TRY(cudaEventRecord(ss->ev[3], aux));
    }
  }
  if (!ntiles && (s = run_checks(st, 0))) return s;
  {
    ProfScope ps("db.raw_tokens", st);
    for (int i = 0; i < n; ++i) {
      const ContainerHeader &h = hdr[i];
      const uint8_t *ib = static_cast<const uint8_t *>(in_host[i]);
      const int64_t t = h.tokens;
      const int64_t nraw = h.m ? int64_t(h.sinks) + h.window : t;
      const int64_t hd = int64_t(h.kv_heads) * h.head_dim;
      const auto *rawk = reinterpret_cast<const __nv_bfloat16 *>(ib + h.raw_off);
      const auto *rawv = rawk + int64_t(h.layers) * nraw * hd;
      for (int sv = 0; sv < 2; ++sv) {
        const kvtc_kv_view &vw = sv ? v_out[i] : k_out[i];
        __nv_bfloat16 *const *bs = sv ? vbases[i] : kbases[i];
        const __nv_bfloat16 *raw = sv ? rawv : rawk;
        if (!h.m) {
          if ((s = launch_unpack_raw(raw, nraw, 0, t, vw, bs, 0, 0, h.layers, st))) return s;
          continue;
        }
        if ((s = launch_unpack_raw(raw, nraw, 0, h.sinks, vw, bs, 0, 0, h.layers, st))) return s;
        if ((s = launch_unpack_raw(raw, nraw, h.sinks, h.window, vw, bs, t - h.window, 0, h.layers, st))) return s;
      }
    }
  }
  (void)err;
  if (status_dev) {
    batch_status_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(ierr, n, status_dev);
    KVTC_LAUNCH_CHECK();
  }
  return KVTC_OK;
}
}  // namespace

extern "C" kvtc_status kvtc_decompress_batch(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                             const kvtc_plan *vp, const void *const *in_host, const size_t *in_len_host,
                                             int32_t n, const kvtc_kv_view *k_out, const kvtc_kv_view *v_out,
                                             void *workspace, size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && in_host && in_len_host && k_out && v_out && n > 0,
                 "decompress_batch arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // all headers in one device-to-host round trip
  std::vector<ContainerHeader> hdr(n);
  for (int i = 0; i < n; ++i) {
    KVTC_CHECK_ARG(in_len_host[i] >= KVTC_HEADER_BYTES, "container too short");
    KVTC_CUDA_TRY(cudaMemcpyAsync(&hdr[i], in_host[i], sizeof(ContainerHeader), cudaMemcpyDeviceToHost, st));
  }
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  int32_t *ierr = nullptr;
  kvtc_status s = decompress_batch_core(kb, kp, vb, vp, in_host, in_len_host, n, k_out, v_out, hdr, nullptr, workspace,
                                        workspace_bytes, st, &ierr);
  if (s) return s;
  // one synchronisation: every item's inflate / checksum status
  std::vector<int32_t> st_host(n);
  KVTC_CUDA_TRY(cudaMemcpyAsync(st_host.data(), ierr, 4 * size_t(n), cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i)
    if (st_host[i]) {
      set_error("batch item %d: corrupt container (inflate / checksum status %d)", i, st_host[i]);
      return KVTC_E_CORRUPT;
    }
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_decompress_batch_async(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                                   const kvtc_plan *vp, const void *const *in_host,
                                                   const size_t *in_len_host, const void *const *in_header_host,
                                                   int32_t n, const kvtc_kv_view *k_out, const kvtc_kv_view *v_out,
                                                   int32_t *status_dev, void *workspace, size_t workspace_bytes,
                                                   void *stream) {
  KVTC_CHECK_ARG(kb && kp && vb && vp && in_host && in_len_host && in_header_host && k_out && v_out && n > 0 &&
                     status_dev,
                 "decompress_batch_async arguments");
  std::vector<ContainerHeader> hdr(n);
  for (int i = 0; i < n; ++i) {
    KVTC_CHECK_ARG(in_len_host[i] >= KVTC_HEADER_BYTES && in_header_host[i], "container too short / no header");
    memcpy(&hdr[i], in_header_host[i], sizeof(ContainerHeader));
  }
  int32_t *ierr = nullptr;
  return decompress_batch_core(kb, kp, vb, vp, in_host, in_len_host, n, k_out, v_out, hdr, status_dev, workspace,
                               workspace_bytes, static_cast<cudaStream_t>(stream), &ierr);
}

// ------------------------------------------------- calibration / allocation
// (implemented in calib.cu / dp.cu)

