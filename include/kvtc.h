/*
 * kvtc.h — C ABI of the B200-native KVTC codec (arXiv 2511.01815, "KV cache
 * Transform Coding").  Plain pointers and sizes only; no C++ or torch types.
 *
 * Citation keys: P:Lnnn = /root/reference/PAPER.md line nnn (the paper is the
 * authority on what is computed); Qk / Rk = reading k in DESIGN.md §3; §n =
 * DESIGN.md section n.
 *
 * Conventions shared by every entry point
 *  - Pointers named *_host are host memory; every other data pointer is DEVICE
 *    memory of the current CUDA device.  `stream` is a cudaStream_t (NULL =
 *    legacy default stream).  Work is enqueued asynchronously on `stream`;
 *    validation errors are returned before anything is enqueued; asynchronous
 *    kernel faults surface as KVTC_E_CUDA from the next call that synchronises.
 *  - Ownership: the caller owns every buffer it passes (inputs, outputs,
 *    workspaces).  The library owns the opaque kvtc_basis / kvtc_plan handles
 *    (created by kvtc_*_create / kvtc_calibrate / kvtc_allocate_bits*, released
 *    by kvtc_*_destroy).  Handles are immutable after creation and may be shared
 *    across threads and streams.
 *  - No exception crosses the ABI.  On failure a status < 0 is returned and
 *    kvtc_last_error() gives a thread-local message.
 *  - There is no CPU fallback: every compute step runs in the library's sm_100a
 *    kernels; on a device that is not sm_100 the calls return KVTC_E_UNSUPPORTED.
 */
#ifndef KVTC_H_
#define KVTC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVTC_ABI_VERSION 2

typedef enum {
  KVTC_OK = 0,
  KVTC_NOTHING_TO_COMPRESS = 1, /* t <= s + w: container holds raw tokens only (Q17)   */
  KVTC_E_INVALID = -1,          /* bad argument / shape                                */
  KVTC_E_NUMERIC = -2,          /* a 16-bit shift/scale overflowed (Q4)                */
  KVTC_E_CORRUPT = -3,          /* malformed container / DEFLATE stream / checksum     */
  KVTC_E_MISMATCH = -4,         /* basis / plan / shape fingerprint mismatch           */
  KVTC_E_CAPACITY = -5,         /* output or workspace buffer too small                */
  KVTC_E_CUDA = -6,             /* CUDA runtime / driver error                         */
  KVTC_E_NOMEM = -8,            /* device or host allocation failed                    */
  KVTC_E_UNSUPPORTED = -9       /* device is not sm_100 / feature not built            */
} kvtc_status;

typedef enum { KVTC_KEYS = 0, KVTC_VALUES = 1 } kvtc_stream;

/* Element types in the order of the paper's pseudocode, types = [None, int2,
 * int4, fp8].  Cost per token of a group of `size` PCs: 0 for None,
 * size*{2,4,8} + 32 otherwise (16-bit shift + 16-bit scale, Q1). */
typedef enum { KVTC_T_NONE = 0, KVTC_T_INT2 = 1, KVTC_T_INT4 = 2, KVTC_T_FP8 = 3 } kvtc_type;

typedef enum { KVTC_LAYOUT_CONTIGUOUS = 0, KVTC_LAYOUT_PAGED = 1 } kvtc_layout;

/* p = layers * kv_heads * head_dim features per token and stream. */
typedef struct {
  int32_t layers, kv_heads, head_dim;
} kvtc_shape;

/* RoPE description (Q10; the paper only says to undo it).
 * inv_freq_host: [head_dim/2] fp32 frequencies; pairing 0 = half-split
 * (j, j+d/2) (HF Llama/Mistral), 1 = interleaved (2j, 2j+1). */
typedef struct {
  const float *inv_freq_host;
  int32_t pairing;
} kvtc_rope;

/* A view of one conversation's cache for ONE stream (keys or values), bf16.
 *  layout CONTIGUOUS: layer_base_host[l] -> [tokens][kv_heads][head_dim]
 *  layout PAGED:      layer_base_host[l] -> [num_pages][page_tokens][kv_heads][head_dim];
 *                     token tau lives in page block_table[tau / page_tokens],
 *                     slot tau % page_tokens (block_table is DEVICE int32).
 * pos0 = absolute position of token 0 (RoPE angles use pos0 + tau).
 * keys_rotated: 1 if the cache holds post-RoPE keys (the usual case). */
typedef struct {
  kvtc_shape shape;
  int64_t tokens;
  int64_t pos0;
  int32_t layout;
  int32_t page_tokens;
  void *const *layer_base_host;
  const int32_t *block_table;
  int32_t keys_rotated;
  int32_t reserved;
} kvtc_kv_view;

/* Tokens kept raw: the first `sinks` (attention sinks, s = 4) and the last
 * `window` (w = 128).  chunk_bytes: entropy-coder chunk (Q15, 65536).
 * coder: the lossless back-end, KVTC_CODER_DEFLATE (default) or
 * KVTC_CODER_RANS (the static-model rANS of reading Q24, SURVEY §8(f)4;
 * single-conversation calls only). */
typedef enum { KVTC_CODER_DEFLATE = 0, KVTC_CODER_RANS = 1 } kvtc_coder;
typedef struct {
  int32_t sinks, window, chunk_bytes;
  int32_t coder;
} kvtc_policy;

/* DP configuration.  Budget B = floor(feature_bits * p / target_cr)
 * bits per token (Q6).  sizes_host: allowed group sizes (default {1,16,64,256,
 * 1024}); type_mask: bit t set = type t allowed (None always allowed);
 * dp_row_cap: DP rows used, the first 32768 (Q8). */
typedef struct {
  double target_cr;
  int32_t feature_bits;
  int32_t nsizes;
  const int32_t *sizes_host;
  uint32_t type_mask;
  int64_t dp_row_cap;
} kvtc_dp_config;

typedef struct kvtc_basis kvtc_basis; /* mu, V (fp32 master + bf16/fp16 operands), sigma, rope */
typedef struct kvtc_plan kvtc_plan;   /* groups, bits/token, r_eff, expected error              */

/* ------------------------------------------------------------------ misc */
int32_t kvtc_abi_version(void);
const char *kvtc_last_error(void);
/* Returns KVTC_OK when the current device is an sm_100 part the kernels run on. */
kvtc_status kvtc_device_check(void);

/* ----------------------------------------------------------------- basis
 * The calibrated transform of one stream: C - mu = U Sigma V^T.
 * kvtc_basis_create builds a basis from a host master: mu_host [p] fp32,
 * V_host [p x rank] fp32 row-major (column j = j-th principal direction,
 * sigma descending), sigma_host [rank] (nullable).  The library derives the
 * GEMM operands by RNE from the master (V_c = bf16(V), V_d = fp16(V); R2, R6)
 * and mu V_c in fp64 -> fp32.  rope may be NULL for values. */
kvtc_status kvtc_basis_create(const kvtc_shape *shape, kvtc_stream which, const kvtc_rope *rope,
                              int32_t rank, const float *mu_host, const float *V_host,
                              const float *sigma_host, kvtc_basis **out);
kvtc_status kvtc_basis_destroy(kvtc_basis *b);
/* Copies out p, rank and (each nullable) mu [p], V [p x rank] row-major, sigma [rank]. */
kvtc_status kvtc_basis_get(const kvtc_basis *b, int32_t *p, int32_t *rank, float *mu_host,
                           float *V_host, float *sigma_host);

/* ------------------------------------------------------------ calibration
 * P:L222-229.  samples_host: [n][2] int64 (sequence index, token index) — the
 * random draw is an input (sinks must already be excluded by the caller,
 * P:L223).  Keys are un-RoPE'd (R1) at pos0 + token.
 * kvtc_calibrate_accumulate ADDS sum_x (fp64 [p]) and xtx (fp32 [p x p],
 * row-major, upper and lower triangle) of the gathered bf16 rows into the
 * caller's device buffers — these are what a multi-GPU caller all-reduces
 * (NCCL sum) before kvtc_calibrate_finalize.  workspace: device scratch of
 * kvtc_calibrate_workspace_bytes(p) bytes.
 * kvtc_calibrate_finalize: Sigma = xtx - n mu mu^T (fp64), symmetric
 * eigendecomposition, descending order, canonical sign (Q13), rank =
 * min(rank_cap, n-1, p) (Q12).  Synchronises `stream`. */
size_t kvtc_calibrate_workspace_bytes(const kvtc_shape *shape);
kvtc_status kvtc_calibrate_accumulate(const kvtc_kv_view *seqs, int32_t nseq, const int64_t *samples_host,
                                      int64_t n, kvtc_stream which, const kvtc_rope *rope,
                                      double *sum_x, float *xtx, void *workspace, size_t workspace_bytes,
                                      void *stream);
kvtc_status kvtc_calibrate_finalize(const kvtc_shape *shape, kvtc_stream which, const kvtc_rope *rope,
                                    const double *sum_x, const float *xtx, int64_t n, int32_t rank_cap,
                                    void *stream, kvtc_basis **out);
/* Single-process convenience: accumulate + finalize (allocates its own scratch). */
kvtc_status kvtc_calibrate(const kvtc_kv_view *seqs, int32_t nseq, const int64_t *samples_host, int64_t n,
                           kvtc_stream which, const kvtc_rope *rope, int32_t rank_cap, void *stream,
                           kvtc_basis **out);

/* ------------------------------------------------------------ allocation
 * The DP of P:L1541-1603 on the GPU, bit-exact with the literal loop (§6):
 * canonical fp64 summation order (Q9), the loop's tie semantics as a scan (Q7),
 * budget axis at stride 2 (exact: every cost is even).
 * kvtc_allocate_bits_from_coeffs: P [n x r] fp32 row-major (device) are the
 * projected calibration rows, columns sorted by descending variance.
 * kvtc_allocate_bits: gathers the first dp_row_cap sample rows, projects them
 * with the basis (P = X V_c - mu V_c, the compress GEMM with fp32 output), then
 * runs the DP.  Both synchronise `stream`. */
kvtc_status kvtc_allocate_bits_from_coeffs(const float *P, int64_t n, int32_t r, int32_t p_original,
                                           const kvtc_dp_config *cfg, void *stream, kvtc_plan **out);
kvtc_status kvtc_allocate_bits(const kvtc_basis *b, const kvtc_kv_view *seqs, int32_t nseq,
                               const int64_t *samples_host, int64_t n, const kvtc_dp_config *cfg,
                               void *stream, kvtc_plan **out);
/* Plans for several target CRs (crs_host[ncr]; cfg->target_cr ignored) from ONE
 * DP table computed at the largest budget: column b of the DP does not depend on
 * how many columns were computed, so each plan equals the single-CR plan
 * bit for bit ("backtracking can use the tables"; the paper's CR sweeps,
 * P:L333).  out[ncr] receives one plan handle per CR. */
kvtc_status kvtc_allocate_bits_multi(const kvtc_basis *b, const kvtc_kv_view *seqs, int32_t nseq,
                                     const int64_t *samples_host, int64_t n, const kvtc_dp_config *cfg,
                                     const double *crs_host, int32_t ncr, void *stream, kvtc_plan **out);
kvtc_status kvtc_allocate_bits_from_coeffs_multi(const float *P, int64_t n, int32_t r, int32_t p_original,
                                                 const kvtc_dp_config *cfg, const double *crs_host, int32_t ncr,
                                                 void *stream, kvtc_plan **out);
/* DP tables for parity tests: best_error at even budgets, [(r+1) x (B/2+1)]
 * fp64 row-major (device, caller-allocated). */
kvtc_status kvtc_dp_best_table(const float *P, int64_t n, int32_t r, int64_t budget,
                               const kvtc_dp_config *cfg, double *best_even, void *stream);
/* Explicit plan: ngroups non-None groups (start_host, size_host, type_host),
 * non-overlapping, increasing start, within [0, r).  Group sizes the kernels
 * support (KVTC_E_INVALID otherwise): 1..256 with size*bits a multiple of 8 or
 * below 32 (sub-byte tokens are packed within one 32-bit word), and multiples
 * of 256 above that.  The paper's sizes {1, 16, 64, 256, 1024} all
 * qualify; the same rule applies to kvtc_dp_config.sizes_host. */
kvtc_status kvtc_plan_create(int32_t r, int32_t ngroups, const int32_t *start_host, const int32_t *size_host,
                             const int32_t *type_host, kvtc_plan **out);
kvtc_status kvtc_plan_destroy(kvtc_plan *p);
/* Copies the plan out; arrays may be NULL; *ngroups is always written.
 * expected_error: the DP table value best_error[r][B] (NaN for explicit plans). */
kvtc_status kvtc_plan_get(const kvtc_plan *p, int32_t *r, int32_t *ngroups, int32_t *start_host,
                          int32_t *size_host, int32_t *type_host, int64_t *bits_per_token,
                          int32_t *r_eff, double *expected_error, int64_t *budget);

/* ------------------------------------------------------------------ codec
 * Compress: tokens [0,s) and [t-w,t) are stored raw; the m =
 * t - s - w middle tokens of each stream go through un-RoPE (keys, R1) ->
 * D = X V_c - mu V_c (tcgen05 GEMM) -> per-(token, group) shift/scale/codes ->
 * bit-pack (§4 layout) -> chunked DEFLATE; everything in one container
 * written to out (device, 16-byte aligned).  Output layout: DESIGN.md §4.
 * A non-finite 16-bit shift or scale (Q4) flags the container: compress returns
 * KVTC_E_NUMERIC when it synchronises (out_len_host != NULL), and decompressing
 * a flagged container returns KVTC_E_NUMERIC.
 * kvtc_compress_bound: capacity that always suffices (stored-block worst case).
 * kvtc_compress_workspace_bytes: device scratch needed for the call.
 * *out_len_host (nullable) receives the container length (synchronises). */
size_t kvtc_compress_bound(const kvtc_plan *kp, const kvtc_plan *vp, const kvtc_kv_view *k,
                           const kvtc_policy *pol);
size_t kvtc_compress_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                     const kvtc_plan *vp, const kvtc_kv_view *k, const kvtc_policy *pol);
kvtc_status kvtc_compress(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb, const kvtc_plan *vp,
                          const kvtc_kv_view *k, const kvtc_kv_view *v, const kvtc_policy *pol, void *out,
                          size_t out_cap, size_t *out_len_host, void *workspace, size_t workspace_bytes,
                          void *stream);
/* Decompress: inflate -> unpack/dequantise (fp16, R5) ->
 * X^ = D^ V_d^T + mu (tcgen05 GEMM, R6) -> keys re-rotated (R7) -> bf16 written
 * into k_out / v_out (contiguous or paged views of the same shape and tokens).
 * Only layers [layer_begin, layer_end) are reconstructed ("layer-by-layer using
 * sub-matrices of V^T"); sinks/window of those layers are restored
 * byte-identical.  in: device container of in_len bytes, 16-byte aligned.
 *
 * Integrity ("This step is lossless"): the result is either exactly what
 * kvtc_compress encoded, or an error.  The header is validated on the host (its
 * checksum, every size and offset re-derived from the shape; reads never leave
 * [in, in + in_len)); the inflater checks every stream against the section's
 * side index; the inflated payloads and the raw sink/window section are checked
 * against the container's 64-bit checksums.  Any failure ->
 * KVTC_E_CORRUPT (the views may then hold partial output).  A container whose
 * compression flagged a 16-bit factor overflow -> KVTC_E_NUMERIC.
 *
 * kvtc_decompress reads the header (one device-to-host copy + synchronisation)
 * and synchronises again at the end to report the verdict.
 * kvtc_decompress_async never synchronises: header_host is the container's first
 * KVTC_HEADER_BYTES bytes (as returned by compress, or copied once), and the
 * verdict is written asynchronously to *status_dev (device int32: 0 = intact,
 * KVTC_E_CORRUPT otherwise) on `stream`; header / argument errors are returned
 * immediately. */
/* Workspace of a decompression of the container whose header is given (host
 * copy of its first KVTC_HEADER_BYTES bytes); 0 for a header that does not
 * validate (the decompress call then reports why). */
size_t kvtc_decompress_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                       const kvtc_plan *vp, const void *in_header_host);
kvtc_status kvtc_decompress(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb, const kvtc_plan *vp,
                            const void *in, size_t in_len, int32_t layer_begin, int32_t layer_end,
                            const kvtc_kv_view *k_out, const kvtc_kv_view *v_out, void *workspace,
                            size_t workspace_bytes, void *stream);
kvtc_status kvtc_decompress_async(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                  const kvtc_plan *vp, const void *in, size_t in_len, const void *header_host,
                                  int32_t layer_begin, int32_t layer_end, const kvtc_kv_view *k_out,
                                  const kvtc_kv_view *v_out, int32_t *status_dev, void *workspace,
                                  size_t workspace_bytes, void *stream);
/* ------------------------------------------- layer-streamed decompression
 * the inverse projection "can be performed layer-by-layer using
 * sub-matrices of V^T, allowing generation to begin early".  The PCA
 * coefficients mix all layers, so kvtc_decompress_begin inflates and
 * dequantises the container ONCE into `workspace` (kvtc_decompress_workspace_bytes
 * of it; one synchronisation to read the header); each kvtc_decompress_layers
 * call then rebuilds layers [layer_begin, layer_end) only (their h*d columns of
 * V^T, plus those layers' raw sink / window tokens), reading the coefficients from
 * the same workspace.  header_host: the container's first KVTC_HEADER_BYTES
 * bytes on the host.  The workspace must not be reused in between.  Results equal
 * kvtc_decompress bit for bit. */
kvtc_status kvtc_decompress_begin(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                  const kvtc_plan *vp, const void *in, size_t in_len, void *workspace,
                                  size_t workspace_bytes, void *stream);
kvtc_status kvtc_decompress_layers(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                   const kvtc_plan *vp, const void *in, const void *header_host, int32_t layer_begin,
                                   int32_t layer_end, const kvtc_kv_view *k_out, const kvtc_kv_view *v_out,
                                   void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------- batched codec
 * n conversations (or token ranges of conversations: a view whose layer bases
 * are offset by a tokens and pos0 += a) in one call.  Their middle tokens are
 * concatenated, each padded to whole 128-token tiles, so each projection GEMM,
 * each reconstruction GEMM, the DEFLATE encoder and the inflater run ONCE for
 * the whole batch (rows are independent, Q1).  Every container is byte-identical
 * to the one kvtc_compress writes for the same item.  Serving many short
 * requests, and compressing the c = 16 tokens that leave the window each turn
 * (P:L281), need this.
 *  k[i], v[i]: item i's views; out_host[i]: DEVICE pointer of its container
 *  buffer (out_cap_host[i] >= kvtc_compress_bound for that item);
 *  out_len_host[i] (nullable; forces one synchronisation): container lengths.
 *  Errors as kvtc_compress; the first failing item's index is in the message. */
size_t kvtc_compress_batch_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                           const kvtc_plan *vp, const kvtc_kv_view *k, int32_t n,
                                           const kvtc_policy *policy);
kvtc_status kvtc_compress_batch(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb, const kvtc_plan *vp,
                                const kvtc_kv_view *k, const kvtc_kv_view *v, int32_t n, const kvtc_policy *policy,
                                void *const *out_host, const size_t *out_cap_host, size_t *out_len_host,
                                void *workspace, size_t workspace_bytes, void *stream);
/* in_host[i]: DEVICE pointer of container i (length in_len_host[i]); all layers
 * are restored into k_out[i] / v_out[i].  in_header_host[i]: host copies of the
 * first KVTC_HEADER_BYTES bytes of each container.  One synchronisation (the
 * headers). */
size_t kvtc_decompress_batch_workspace_bytes(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                             const kvtc_plan *vp, const void *const *in_header_host, int32_t n);
kvtc_status kvtc_decompress_batch(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                  const kvtc_plan *vp, const void *const *in_host, const size_t *in_len_host,
                                  int32_t n, const kvtc_kv_view *k_out, const kvtc_kv_view *v_out, void *workspace,
                                  size_t workspace_bytes, void *stream);
/* As kvtc_decompress_batch without any host synchronisation: in_header_host[i]
 * are host copies of the containers' headers; status_dev [n] (device int32)
 * receives each item's integrity verdict (0 or KVTC_E_CORRUPT) on `stream`. */
kvtc_status kvtc_decompress_batch_async(const kvtc_basis *kb, const kvtc_plan *kp, const kvtc_basis *vb,
                                        const kvtc_plan *vp, const void *const *in_host, const size_t *in_len_host,
                                        const void *const *in_header_host, int32_t n, const kvtc_kv_view *k_out,
                                        const kvtc_kv_view *v_out, int32_t *status_dev, void *workspace,
                                        size_t workspace_bytes, void *stream);

/* Parse a container header (first KVTC_HEADER_BYTES bytes, copied to host).
 * info is filled in any case; the status is the header validation (KVTC_OK,
 * KVTC_E_CORRUPT for a damaged / inconsistent header, KVTC_E_NUMERIC for a
 * container flagged at compression). */
#define KVTC_HEADER_BYTES 256
typedef struct {
  uint32_t magic, version;
  int32_t layers, kv_heads, head_dim, sinks, window, chunk_bytes;
  int64_t tokens, pos0, m;
  uint64_t total_bytes;           /* container length                                  */
  uint64_t raw_bytes;             /* raw sink + window section (K and V)               */
  uint64_t payload_bytes[2];      /* pre-DEFLATE payload per stream                    */
  uint64_t entropy_bytes[2];      /* DEFLATE streams + chunk tables + indices          */
  uint64_t basis_fp[2], plan_fp[2];
  uint32_t flags;                 /* bit 0: a 16-bit shift/scale overflowed (Q4)        */
  uint32_t reserved;
  uint64_t payload_hash[2];       /* 64-bit checksums                    */
  uint64_t raw_hash;
} kvtc_container_info;
kvtc_status kvtc_container_parse(const void *header_host, kvtc_container_info *info);

/* --------------------------------------------------------- stage entry points
 * The individual kernels of the path, for parity tests and profiling.  Same
 * conventions; they never allocate. */
/* K1: rows tau in [tok_begin, tok_begin+ntok) of a view -> X [ntok x p] bf16
 * token-major, features (layer, head, dim); keys un-RoPE'd (R1). */
kvtc_status kvtc_stage_gather(const kvtc_kv_view *v, int64_t tok_begin, int64_t ntok, int32_t unrope,
                              const kvtc_rope *rope, void *X, void *stream);
/* GEMM with fp32 output: D [m x ncols] = X V_c[:, cols] - mu V_c[:, cols];
 * cols = the plan's non-None PCs in order (plan != NULL) or all rank PCs. */
kvtc_status kvtc_stage_project(const kvtc_basis *b, const kvtc_plan *plan, const void *X, int64_t m, float *D,
                               void *stream);
/* Payload bytes for m tokens (§4). */
size_t kvtc_payload_bytes(const kvtc_plan *plan, int64_t m);
/* Quantise + pack from a given fp32 D [m x ncols(plan)] (SIMT reference kernel). */
kvtc_status kvtc_stage_quantize_pack(const kvtc_plan *plan, const float *D, int64_t m, uint8_t *payload,
                                     void *stream);
/* Joint cross-shard compression ("chunks could be compressed jointly";
 * SURVEY §8(f)2): one basis over the features of all layer shards.  Shard g holds
 * the gathered rows X [m x (feat_end - feat_begin)] bf16 of its features
 * [feat_begin, feat_end) of the basis (multiples of 8); writes its partial
 * projection D [m x ncols(plan)] fp32 = X V_c[feat_begin:feat_end, plan PCs], minus
 * mu V_c when add_bias (exactly one shard).  The partials summed over the shards
 * (a reduce-scatter over token rows) are kvtc_stage_project's D of the joint
 * features, up to fp32 summation order.  Device pointers, caller-owned. */
kvtc_status kvtc_stage_project_partial(const kvtc_basis *b, const kvtc_plan *plan, const void *X, int64_t m,
                                       int32_t feat_begin, int32_t feat_end, int32_t add_bias, float *D,
                                       void *stream);
/* K2: fused tcgen05 projection + quantise + pack straight from TMEM. */
kvtc_status kvtc_stage_project_quantize(const kvtc_basis *b, const kvtc_plan *plan, const void *X, int64_t m,
                                        uint8_t *payload, void *stream);
/* K3: chunked DEFLATE of n bytes -> an entropy section (§4) at out; *out_len_host set. */
size_t kvtc_deflate_bound(size_t n, int32_t chunk_bytes);
size_t kvtc_deflate_workspace_bytes(size_t n, int32_t chunk_bytes);
kvtc_status kvtc_stage_deflate(const uint8_t *in, size_t n, int32_t chunk_bytes, uint8_t *out, size_t out_cap,
                               size_t *out_len_host, void *workspace, size_t workspace_bytes, void *stream);
/* K4: inflate an entropy section produced by kvtc_stage_deflate into out [n_out]. */
kvtc_status kvtc_stage_inflate(const uint8_t *section, size_t len, uint8_t *out, size_t n_out, void *stream);
/* K4 (generic): inflate nstreams independent raw RFC-1951 streams (e.g. zlib's,
 * wbits=-15): stream i = in[in_off[i] .. in_off[i]+in_len[i]) -> out[out_off[i] ..
 * +out_len[i]).  Offset arrays are device int64.  status_dev[i] = 0 ok, else
 * error (device int32 [nstreams]). */
kvtc_status kvtc_stage_inflate_raw(const uint8_t *in, const int64_t *in_off, const int64_t *in_len,
                                   int32_t nstreams, uint8_t *out, const int64_t *out_off,
                                   const int64_t *out_len, int32_t *status_dev, void *stream);
/* Alternative lossless back-end (ANS is in the paper's ablation,
 * P:L1305-1317): static-model interleaved rANS, one order-0 table per payload
 * tile-offset class (reading Q24; oracle/rans.py).  tile_bytes: the
 * payload's tile period (kvtc_payload_bytes of 128 tokens), 0 = none.  The
 * section is written at out (16-byte aligned, >= kvtc_rans_bound bytes);
 * *out_len_host receives its length (synchronising).  Decode returns
 * KVTC_E_CORRUPT for a malformed section or stream. */
size_t kvtc_rans_bound(size_t n, int32_t chunk_bytes, int64_t tile_bytes);
size_t kvtc_rans_workspace_bytes(size_t n, int32_t chunk_bytes, int64_t tile_bytes);
kvtc_status kvtc_stage_rans_encode(const uint8_t *in, size_t n, int32_t chunk_bytes, int64_t tile_bytes, uint8_t *out,
                                   size_t out_cap, size_t *out_len_host, void *workspace, size_t workspace_bytes,
                                   void *stream);
kvtc_status kvtc_stage_rans_decode(const uint8_t *section, size_t len, uint8_t *out, size_t n_out, void *stream);
/* Unpack + dequantise: payload -> D^ [m x ld] fp16 (ld a multiple of 8 and >=
 * ncols(plan) rounded up to 8, Dh 16-byte aligned, else KVTC_E_INVALID);
 * D^ = fp16(code * scale + shift) rounded once (R5).  Columns from
 * ncols to the next multiple of 8 are written as 0. */
kvtc_status kvtc_stage_dequantize(const kvtc_plan *plan, const uint8_t *payload, int64_t m, uint16_t *Dh,
                                  int64_t ld, void *stream);
/* K5: X^ = D^ V_d^T + mu for layers [layer_begin, layer_end), keys re-rotated
 * (R7), bf16 into the view at tokens [tok_begin, tok_begin + m). */
kvtc_status kvtc_stage_reconstruct(const kvtc_basis *b, const kvtc_plan *plan, const uint16_t *Dh, int64_t ld,
                                   int64_t m, int64_t tok_begin, int32_t layer_begin, int32_t layer_end,
                                   const kvtc_kv_view *out, void *stream);
/* D2 + K5 fused (kvtc_decompress takes this path only with
 * KVTC_DQ_FUSED=1, it is measured 7-8x slower: DESIGN.md §11): the same
 * reconstruction with A = D^ dequantised from the payload (m tokens of 128-token
 * tiles, as kvtc_stage_project_quantize writes it) by the GEMM's producer warps,
 * never written to HBM.  Bitwise equal to kvtc_stage_dequantize followed by
 * kvtc_stage_reconstruct. */
kvtc_status kvtc_stage_reconstruct_payload(const kvtc_basis *b, const kvtc_plan *plan, const uint8_t *payload,
                                           int64_t m, int64_t tok_begin, int32_t layer_begin, int32_t layer_end,
                                           const kvtc_kv_view *out, void *stream);

/* ------------------------------------------------------------- diagnostics
 * Per-stage device timing with CUDA events recorded on the caller's stream
 * around each stage of kvtc_compress / kvtc_decompress (off by default; enabling
 * resets).  kvtc_profile_read synchronises the recorded events and returns the
 * number of distinct stages (<= cap): names are written NUL-separated into
 * names_host (capacity names_cap bytes), total milliseconds and call counts into
 * ms_host / calls_host.  kvtc_launch_count: kernels this library launched since
 * the last reset (all entry points). */
void kvtc_profile_enable(int32_t on);
int32_t kvtc_profile_read(char *names_host, size_t names_cap, double *ms_host, int32_t *calls_host, int32_t cap);
int64_t kvtc_launch_count(void);
void kvtc_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* KVTC_H_ */
