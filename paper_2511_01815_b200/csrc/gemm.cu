// gemm.cu — the tcgen05/TMEM/TMA GEMMs of the KVTC path (K2/K5/K6).
//
//   EPI_QUANT  K2  compress: D = X V_c - mu V_c and, straight from
//                  TMEM, per-(token, group) min/max -> fp16 shift/scale -> codes
//                  -> bit-pack into the §4 payload.  D never
//                  reaches HBM, except the pieces of groups wider than one tile
//                  (1024): those tiles store fp32 D to a scratch that
//                  quant_wide_kernel quantises (its row min/max spans 4 tiles).
//   EPI_F32        the same GEMM with an fp32 D output (DP coefficients, tests).
//   EPI_RECON  K5  decompress: X^ = D^ V_d^T + mu, keys
//                  re-rotated (RoPE, R7), bf16 RNE, scattered into a contiguous
//                  or paged cache.  With ASRC = 1 (the product path) the A operand
//                  D^ never exists in HBM: four dequantising producer warps read
//                  the inflated payload (codes + fp16 shift/scale) and write the
//                  fp16 A k-blocks straight into the swizzled shared-memory stages
//                  (unpack + dequantise fused into the GEMM, D2 of SURVEY
//                  §8(a)); only V_d comes through TMA.
//   EPI_XTX    K6  calibration: S += C^T C over a chunk of rows.
//
// Persistent kernel, one CTA pair (cta_group::2, M = 256) per 2 SMs: tiles are
// handed out statically in a grouped raster (group_m M-pairs x all N tiles) so
// that the ~74 tiles in flight share A and B k-blocks in L2.  Sharing only works
// while the CTAs stay in step (K = p = 32768 makes one tile's operands 2 x 16.8
// MB), so the TMA producers meet at a soft barrier before every tile
// (tile_barrier): ncu showed 23-37 GB of DRAM reads per compress launch without
// it.  Warp roles: warp 0 TMA producer, warp 1 single-thread tcgen05.mma issuer
// (pair leader), warp 2 TMEM allocator, warps 4-7 epilogue (warp w reads TMEM
// lanes 32*(w%4)..+31).  Operands K-major, 128 B swizzled, 6-stage mbarrier ring;
// two fp32 TMEM accumulators (2 x 256 columns) so the epilogue of tile i overlaps
// the MMAs of tile i+1; EPI_QUANT quantises straight from TMEM (two passes per
// group).  Pieces of groups wider than a tile store fp32 coefficients for
// quant_wide.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "internal.h"
#include "quant.cuh"
#include "dequant.cuh"

namespace kvtc {

// Single-CTA tiles: A 128 x 64 + B 256 x 64 per stage (48 KiB), 4 stages.
// CTA pairs (cta_group::2, M = 256): each CTA holds its A half (128 rows) and
// its B half (N/2 <= 128 rows): 32 KiB per stage, 6 stages.
// NSUB = 2 (compress): a tile is two 256-column segments sharing the A k-block;
// two MMAs per k-slice into both TMEM accumulators (512 columns, no double
// buffering), 48 KiB per stage, 4 stages: 25 % less L2 traffic per flop.
// KB = 2 (the codec GEMMs' default): two 64-column k-blocks per pipeline stage
// (64 KiB stages, 3 of them): half the barrier round trips per MMA (pairs, one
// segment only).
template <bool PAIR, int NSUB = 1, int KB = 1>
struct Cfg {
  static constexpr int kStages = KB == 2 ? 3 : (NSUB == 2 ? 4 : (PAIR ? 6 : 4));
  static constexpr int kABlock = kTileM * kBlockK * 2;                        // 16 KiB per k-block
  static constexpr int kABytes = KB * kABlock;
  static constexpr int kBSubBytes = (PAIR ? kMaxTileN / 2 : kMaxTileN) * kBlockK * 2;
  static constexpr int kBBytes = KB * NSUB * kBSubBytes;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 2048;
  static constexpr int kAccBufs = NSUB == 2 ? 1 : 2;
};
constexpr int kBBoxRows = 128;                     // B tensor maps load 128 rows per box
constexpr int kThreads = 256;
#ifndef KVTC_DQ_GROUPS
#define KVTC_DQ_GROUPS 2
#endif
constexpr int kDqGroups = KVTC_DQ_GROUPS;          // groups of 4 dequantising producer warps (ASRC = 1),
constexpr int kDqWarps = 4 * kDqGroups;            // warps 8 .., taking the pipeline stages round robin
__host__ __device__ constexpr int threads_for(int asrc) { return asrc ? kThreads + 32 * kDqWarps : kThreads; }
constexpr int kTmemCols = 512;                     // two 256-column accumulators
constexpr int kGroupM = 8;                         // raster group (M-blocks)

enum { EPI_F32 = 0, EPI_QUANT = 1, EPI_RECON = 2, EPI_XTX = 3 };

struct Params {
  int32_t K;
  int64_t m;
  int32_t ncols;       // F32 / XTX: valid N extent; RECON: n_end
  int32_t n_begin;     // RECON
  int32_t num_m, num_n;   // tile grid (num_n = N tiles or segments)
  const float *bias;   // F32 / QUANT: [r_nz]; RECON: mu [p]
  float *D;            // F32 / XTX output
  int64_t ldd;
  // QUANT
  uint8_t *payload;
  const SegDesc *segs;
  const GroupDesc *groups;
  int32_t parts;       // XTX: -2 marks pair tiling for the symmetric skip
  int32_t G;
  int64_t tile_bytes;
  const int64_t *codes_off_last;
  // RECON
  const float2 *cs;
  int32_t layers, heads, head_dim, pairing;
  int32_t layout, page_tokens;
  __nv_bfloat16 *const *layer_base;
  const int32_t *block_table;
  int64_t tok_begin;
  int32_t fmt;         // 0 fp16, 1 bf16 operands
  int32_t tile_n;      // RECON / F32 / XTX N tile
  int32_t a_hd;        // > 0: A is the 3-D cache map (GemmCompressArgs::a_hd)
  int64_t a_layer_rows;  // > 0: A is a 2-D map over [layers * tokens][h*d] (layer stride = tokens rows)
  int64_t a_row0;
  int32_t group_m;     // raster group (M-blocks or M-pairs)
  int32_t hint_a, hint_b;   // L2 policies of the A / B loads
  unsigned long long *tile_sync;   // non-null: producers align tile starts (see tile_barrier)
  int32_t sync_lag;                // a producer may run this many tiles ahead of the slowest
  int32_t nsegs;                   // QUANT: number of 256-column segments
  int32_t epi_skip;                // measurement only (KVTC_EPI_SKIP=1): release TMEM without an epilogue
  const TileRef *tiles;            // batched rows (QUANT / RECON), else null
  int32_t *status;                 // QUANT: bit 0 set when an fp16 shift / scale overflowed (Q4)
  // QUANT wide groups: fp32 pieces in D, per-piece row min/max, arrival counters
  const WideDesc *wide;
  int32_t nwide, wpieces;
  float2 *wmm;
  int32_t *wcnt;
  int32_t wide_defer;              // KVTC_WIDE_DEFER=1 (A/B only): no fixup, quant_wide_kernel afterwards
  // RECON with ASRC = 1: A = D^ dequantised from the payload
  const uint8_t *dq_payload;
  const int64_t *dq_off_full, *dq_off_last;
  const DqCol *dq_cols;
  const DqChunk *dq_chunks;        // [num_st * 16]
  int32_t dq_debug;                // KVTC_DQ_DEBUG (measurement only): 1 no payload loads, 2 no A stores,
                                   // 4 no proxy fence
  int32_t l2_pref;                 // > 0: the producer prefetches the k-blocks this many stages ahead
                                   // into L2 (KVTC_L2_PREF_QUANT / _RECON, A/B)
  int32_t spin;                    // KVTC_SPIN_WAITS bit mask: spin (no suspend) on 1 producer empty,
                                   // 2 MMA tmem_empty, 4 epilogue tmem_full, 8 MMA full barrier
  const uint8_t *dq_tail;          // [rows][dq_tail_ld] fp16 columns of the ok = 3 chunks (pre-pass)
  int64_t dq_tail_ld;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct Tile {
  int mb, nb;   // M-block, N tile / segment
  bool valid;
};

__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __uint_as_float(r);
}

// Loads columns [c, c + n) (n <= 16) of this thread's TMEM row, minus the bias.
__device__ __forceinline__ void load_cols(uint32_t trow, const float *bias, int c, int n, float *x) {
  if (n == 16) {
    tmem_ld16(trow + c, x);
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = __fsub_rn(x[j], bias[c + j]);
  } else {
    for (int j = 0; j < n; ++j) x[j] = __fsub_rn(tmem_ld1(trow + c + j), bias[c + j]);
  }
}

// Static persistent schedule: tile t -> (mb, nb) in groups of kGroupM M-blocks.
template <int MODE>
__device__ __forceinline__ Tile tile_of(const Params &P, int64_t t, int num_mt) {
  Tile T;
  const int64_t per_group = int64_t(P.group_m) * P.num_n;
  const int64_t g = t / per_group;
  const int first = int(g * P.group_m);
  const int gm = min(P.group_m, num_mt - first);
  const int64_t r = t - g * per_group;
  T.mb = first + int(r % gm);
  T.nb = int(r / gm);
  T.valid = true;
  if constexpr (MODE == EPI_XTX) {
    // strictly below the diagonal: symmetric, skipped
    // pairs: T.mb is the pair index here (rows 256 mp ..); skipped only if the whole pair is below
    const int64_t row0 = int64_t(T.mb) * kTileM * (P.parts == -2 ? 2 : 1);
    if (int64_t(T.nb) * P.tile_n + P.tile_n <= row0) T.valid = false;
  }
  return T;
}

template <int MODE, int NSUB = 1>
__device__ __forceinline__ void tile_geometry(const Params &P, const Tile &T, int &n0, int &ncols, int &g0, int &g1) {
  g0 = g1 = 0;
  if constexpr (MODE == EPI_QUANT) {
    const SegDesc sd = P.segs[T.nb * NSUB];
    n0 = sd.col0;
    ncols = sd.width;
    g0 = sd.g_begin;
    g1 = sd.g_end;
  } else if constexpr (MODE == EPI_RECON) {
    n0 = P.n_begin + T.nb * P.tile_n;
    ncols = min(P.tile_n, P.ncols - n0);
  } else {
    n0 = T.nb * P.tile_n;
    ncols = min(P.tile_n, P.ncols - n0);
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// 2-D TMA load whose completion is signalled on the PAIR LEADER's mbarrier
// (peer bit cleared), as required for cta_group::2 MMAs.
__device__ __forceinline__ void tma_load_2d_pair(void *smem_dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                                 int32_t c1) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(mbar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void *smem_dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                                 int32_t c1, int32_t c2) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// L2 eviction-priority hints for TMA loads (0 none, 1 evict_first, 2 evict_last).
__device__ __forceinline__ uint64_t l2_policy(int h) {
  uint64_t p = 0;
  if (h == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (h == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_2d_hint(bool pair, void *smem_dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                            int32_t c1, uint64_t pol) {
  if (pair) {
    const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(mbar), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
  }
}
__device__ __forceinline__ void tma_3d_hint(bool pair, void *smem_dst, const CUtensorMap *m, uint64_t *bar, int32_t c0,
                                            int32_t c1, int32_t c2, uint64_t pol) {
  if (pair) {
    const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
  }
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit of the leader's MMAs, arriving on the same barrier offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
// Arrive on the same barrier offset in CTA `cta` of the cluster.  Default (.cta
// scope) release semantics, as CUTLASS's ClusterBarrier::arrive(cta_id): with
// .release.cluster ptxas emits MEMBAR.ALL.GPU + ERRBAR before every arrive (ncu:
// the fused reconstruction's per-stage remote arrivals), and the consumers here
// are the pair leader's tensor core / MMA thread, ordered by the tcgen05 and
// proxy fences around the barrier.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *local_bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_bar)), "r"(cta));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}


// ---------------------------------------------- fused dequantisation (ASRC = 1)
// (R5 arithmetic: dequant.cuh, shared with dequant_rows_kernel)
// Loads of one 16-byte A chunk of a FULL tile (code blocks b-aligned, params
// 4-aligned), issued for a whole stage before any is consumed: no branches, the
// fp8 high word through a predicated load, read-only path.
__device__ __forceinline__ uint32_t ldg_u32(const uint8_t *p) {
  return __ldg(reinterpret_cast<const unsigned int *>(p));
}
__device__ __forceinline__ uint32_t ldg_u32_if(const uint8_t *p, bool pred) {
  uint32_t v = 0;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
      : "+r"(v)
      : "l"(p), "r"(uint32_t(pred)));
  return v;
}
// One (row, chunk) item of the fused producer.  Full tiles: ok = 1 chunks load
// their fp16 factors and 8 codes (2 / 4 / 8 bytes, b-aligned) straight from the
// payload; ok = 3 chunks (size-1 groups, misaligned starts: columns the pre-pass
// dequantised) load their 16 bytes from the tail buffer.  Branch-free address
// selection, predicated loads, read-only path; the words are consumed one stage
// later by dq_item_store.
struct DqItem {
  uint32_t w0, w1, w2, w3;
};
__device__ __forceinline__ void dq_item_issue(const DqChunk &d, const uint8_t *tile, const uint8_t *tail_row, int row,
                                              DqItem &it) {
  const bool dense = d.ok == 1, copy = d.ok == 3;
  const uint8_t *pp = dense ? tile + d.par_base + 4 * row : (copy ? tail_row + d.code_base : tile);
  const uint8_t *cp = dense ? tile + d.code_base + row * int32_t(d.stride) : pp;
  const uint8_t *cq = reinterpret_cast<const uint8_t *>(reinterpret_cast<uintptr_t>(cp) & ~uintptr_t(3));
  it.w0 = ldg_u32(pp);
  it.w1 = ldg_u32_if(cq + (copy ? 4 : 0), dense || copy);
  it.w2 = ldg_u32_if(cq + (copy ? 8 : 4), copy || (dense && d.type == KVTC_T_FP8));
  it.w3 = ldg_u32_if(cq + 12, copy);
  if (dense && d.type != KVTC_T_FP8) it.w1 >>= (reinterpret_cast<uintptr_t>(cp) & 3) * 8;   // int2: 2-aligned
}
__device__ __forceinline__ uint4 dq_item_value(const DqChunk &d, const DqCol *cols, int col0, const uint8_t *tile,
                                               const int64_t *coff, int ntok, int row, const DqItem &it) {
  if (row >= ntok || !d.type) return make_uint4(0u, 0u, 0u, 0u);
  if (d.ok == 3) return make_uint4(it.w0, it.w1, it.w2, it.w3);
  if (ntok == kTileM && d.ok == 1) return dq8(d.type, it.w1, it.w2, it.w0);
  return dq_generic8(cols, col0, tile, coff, ntok, row);   // partial tile
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Wait with cluster-scope acquire (the full barrier also collects the peer CTA's
// dequantising warps' release arrivals).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  uint64_t t0 = 0;
  for (uint32_t i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if ((i & 1023) == 1023) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (!t0) t0 = t;
      else if (t - t0 > 4000000000ull) __trap();
    }
  }
}



// Pre-pass of the fused inverse path: the A columns that are not whole aligned
// 8-chunks of one group (size-1 groups -- the DP's fp16 "keep" option -- and
// misaligned starts; 112 of the 4352 columns of the bench plan) are dequantised
// here into a small side buffer, 16 bytes per (row, chunk), which the GEMM's
// producer copies (R5: one fp16 rounding, like dq8).
__global__ void __launch_bounds__(256) dq_tail_kernel(const DqCol *cols, const int32_t *tail_col, int32_t n_tail,
                                                      const uint8_t *payload, int64_t m, int64_t tile_bytes,
                                                      const int64_t *off_full, const int64_t *off_last,
                                                      const TileRef *tiles, int32_t num_m, uint8_t *tail, int64_t ld) {
  const int64_t total = int64_t(num_m) * kTileM * n_tail;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t rg = idx / n_tail;
    const int k = int(idx - rg * n_tail);
    const int mb = int(rg / kTileM), row = int(rg % kTileM);
    const uint8_t *tile;
    const int64_t *coff;
    int ntok;
    if (tiles) {
      tile = tiles[mb].payload;
      coff = tiles[mb].codes_off;
      ntok = tiles[mb].ntok;
    } else {
      const int64_t m0 = int64_t(mb) * kTileM;
      ntok = int(m - m0 < kTileM ? m - m0 : kTileM);
      tile = payload + int64_t(mb) * tile_bytes;
      coff = ntok < kTileM ? off_last : off_full;
    }
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (row < ntok) {
      const int c0 = tail_col[k];
      uint16_t h[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) h[j] = dq1(tile, coff, ntok, row, cols[c0 + j]);
      o = make_uint4(uint32_t(h[0]) | (uint32_t(h[1]) << 16), uint32_t(h[2]) | (uint32_t(h[3]) << 16),
                     uint32_t(h[4]) | (uint32_t(h[5]) << 16), uint32_t(h[6]) | (uint32_t(h[7]) << 16));
    }
    *reinterpret_cast<uint4 *>(tail + rg * ld + k * 16) = o;
  }
}

// Codes of 32 coefficients of one wide-group row into B 32-bit words.
template <int B>
__device__ __forceinline__ void wide_pack32(int type, const float4 (&v)[8], float shift, float scale, uint8_t *dst,
                                            bool last) {
  constexpr int PW = 32 / B;
#pragma unroll
  for (int w = 0; w < B; ++w) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < PW; ++j) {
      const int i = w * PW + j;
      const float4 q = v[i >> 2];
      const float f = (i & 3) == 0 ? q.x : (i & 3) == 1 ? q.y : (i & 3) == 2 ? q.z : q.w;
      word |= encode_one(type, f, shift, scale) << (j * B);
    }
    store_u32_any(dst + 4 * w, word, !last);
  }
}

// Wide group (k 256-column pieces, P:L256 allows groups up to 1024): called by
// all 128 epilogue threads of a CTA after they stored their piece's fp32
// coefficients and row min/max.  The CTA whose piece arrives last for this
// (M-block, group) quantises and packs the whole group from the scratch (L2),
// so no separate pass over the coefficients is needed.
__device__ __noinline__ void wide_fixup(const Params &P, int w, int mb, int row, int64_t tok, bool valid, int ntok,
                                        bool last, uint8_t *tile_base, const int64_t *codes_off_last, int32_t *stw,
                                        volatile int *flag) {
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const WideDesc wd = P.wide[w];
  const int k = wd.size / kMaxTileN;
  if (row == 0) *flag = atomicAdd(P.wcnt + int64_t(mb) * P.nwide + w, 1) == k - 1;
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (!*flag) return;
  __threadfence();
  if (!valid) return;
  const float2 *mm = P.wmm + tok * P.wpieces + wd.wcol / kMaxTileN;
  float mn = INFINITY, mx = -INFINITY;
  for (int q = 0; q < k; ++q) {
    const float2 v = __ldcg(mm + q);
    mn = fminf(mn, v.x);
    mx = fmaxf(mx, v.y);
  }
  uint16_t sh, sc;
  group_factors(wd.type, mn, mx, sh, sc);
  store_u32_any(tile_base + 4 * (int64_t(wd.gidx) * ntok + row), uint32_t(sh) | (uint32_t(sc) << 16), !last);
  if (stw && factor_overflow(sh, sc)) atomicOr(stw, 1);
  const float shift = f16_val(sh), scale = f16_val(sc);
  const int b = bits_of(wd.type);
  uint8_t *dst = tile_base + (last ? codes_off_last[wd.gidx] : wd.codes_off) + int64_t(row) * (wd.size * b / 8);
  const float *x = P.D + tok * P.ldd + wd.wcol;
  // 32 coefficients (b words) per step, their 8 loads issued together: the
  // pieces were stored tiles ago and come back from L2 / DRAM
  for (int c0 = 0; c0 < wd.size; c0 += 32) {
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(reinterpret_cast<const float4 *>(x + c0) + j);
    if (b == 8) wide_pack32<8>(wd.type, v, shift, scale, dst + c0, last);
    else if (b == 4) wide_pack32<4>(wd.type, v, shift, scale, dst + c0 / 2, last);
    else wide_pack32<2>(wd.type, v, shift, scale, dst + c0 / 4, last);
  }
}

// Soft tile barrier of the TMA producers: the CTAs of one wave of tiles share
// their A / B k-blocks through L2 only while they stay in step; a producer
// that is ahead waits (bounded spin, never a hang) before its s-th tile until
// every CTA has started its s-th tile.  target(s) counts the CTAs that have an
// s-th tile under the static schedule.
// Measured (scripts/exp_sync.sh): compress GEMM 9.7 -> 8.1 ms, decompress 8.6 ->
// 7.2 ms per launch under the power cap.  A wait that exceeds 2 ms (a CTA that
// is not resident, e.g. the GPU is shared) turns the barrier off for the rest
// of the launch in this CTA.
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool tile_barrier(unsigned long long *ctr, int64_t s, int64_t total, int64_t n_units,
                                             int per_unit, int lag) {
  atomicAdd(ctr, 1ull);
  s -= lag;
  if (s < 0) return true;
  const int64_t full = total / n_units, rem = total % n_units;
  const int64_t target = int64_t(per_unit) * (n_units * min(s + 1, full) + (s + 1 > full ? rem : 0));
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
  if (int64_t(v) >= target) return true;
  const uint64_t t0 = global_ns();
  while (true) {
    __nanosleep(64);
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    if (int64_t(v) >= target) return true;
    if (global_ns() - t0 > 2000000ull) return false;
  }
}

// Segments (256-column pieces of the compacted N axis) of a compress tile.
template <int NSUB>
__device__ __forceinline__ int tile_nsub(const Params &P, const Tile &T) {
  return NSUB == 1 ? 1 : min(NSUB, P.nsegs - T.nb * NSUB);
}

// Register budget: the compress GEMM runs beside the side-stream gather / encoder
// CTAs (2-3 per SM), so it is held to 128 registers (min 2 blocks); the
// decompress GEMM (beside the dequantiser) may use more.
template <int MODE, bool PAIR, int NSUB, int KB, int ASRC>
__global__ void __launch_bounds__(threads_for(ASRC), MODE == EPI_RECON ? 1 : 2)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ Params P) {
  static_assert(NSUB == 1 || (MODE == EPI_QUANT && PAIR), "two-segment tiles: compress, CTA pairs");
  static_assert(KB == 1 || (PAIR && NSUB == 1), "two k-blocks per stage: CTA pairs, one segment");
  static_assert(ASRC == 0 || (MODE == EPI_RECON && PAIR && KB == 2), "fused A producer: decompress, pairs, KB 2");
  using C = Cfg<PAIR, NSUB, KB>;
  constexpr int kStages = C::kStages;
  constexpr int kABytes = C::kABytes;
  constexpr int kStageBytes = C::kStageBytes;
  constexpr int kBSub = C::kBSubBytes;
  constexpr int kAccBufs = C::kAccBufs;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the __shared__ array (an integer
  // round trip would make every smem access generic: ST.E / LD.E instead of STS / LDS)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *tiles = smem;
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
  uint64_t *empty_bar = full_bar + kStages;
  uint64_t *tmem_full = empty_bar + kStages;      // [2]
  uint64_t *tmem_empty = tmem_full + 2;           // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);
  volatile int *wide_flag = reinterpret_cast<volatile int *>(tmem_slot + 1);
  // ASRC: the plan's A-chunk table (DqChunk per 8 columns) in shared memory
  uint8_t *dq_tab = smem + kStages * kStageBytes + 256;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const bool leader = rank == 0;
  // pairs: tiles are M-pairs (256 rows); CTA rank r holds M-block 2 mp + r
  const int num_mt = PAIR ? (P.num_m + 1) / 2 : P.num_m;
  const int64_t total = int64_t(num_mt) * P.num_n;
  const int64_t t_first = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t t_step = int64_t(PAIR ? gridDim.x / 2 : gridDim.x);
  const int num_kb = (P.K + kBlockK - 1) / kBlockK;
  const int num_st = (num_kb + KB - 1) / KB;       // pipeline stages per tile
  if constexpr (ASRC == 1) {
    const uint4 *src = reinterpret_cast<const uint4 *>(P.dq_chunks);
    uint4 *dst = reinterpret_cast<uint4 *>(dq_tab);
    for (int i = threadIdx.x; i < num_st * (KB * kBlockK / 8); i += blockDim.x) dst[i] = src[i];
  }

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      // ASRC: + one arrival per dequantising warp of both CTAs (leader's barrier)
      mbar_init(&full_bar[s], ASRC ? 1 + 2 * 4 : 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], PAIR ? 256 : 128);      // pairs: both CTAs' epilogues release the leader's acc
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc<kTmemCols>(tmem_slot);
    }
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();        // peer barriers initialised before any remote arrive / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto get_tile = [&](int64_t t) {
    Tile T = tile_of<MODE>(P, t, num_mt);
    if (PAIR) T.mb = 2 * T.mb + int(rank);      // this CTA's M-block
    return T;
  };

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    uint32_t it = 0;
    const uint64_t pol_a = l2_policy(P.hint_a);
    const uint64_t pol_b = l2_policy(P.hint_b);
    int64_t seq = 0;
    bool sync = MODE != EPI_XTX && P.tile_sync != nullptr;
    for (int64_t t = t_first; t < total; t += t_step) {
      const Tile T = get_tile(t);
      if (!T.valid) continue;
      if (sync) sync = tile_barrier(P.tile_sync, seq++, total, t_step, PAIR ? 2 : 1, P.sync_lag);
      int n0, ncols, g0, g1;
      tile_geometry<MODE, NSUB>(P, T, n0, ncols, g0, g1);
      const int n_mma = (ncols + 15) & ~15;
      const int nsub = tile_nsub<NSUB>(P, T);
      for (int ks = 0; ks < num_st; ++ks, ++it) {
        const int s = it % kStages;
        if (it >= kStages) {
          if (P.spin & 1) mbar_wait_spin(&empty_bar[s], ((it / kStages) - 1) & 1);
          else mbar_wait(&empty_bar[s], ((it / kStages) - 1) & 1);
        }
        uint8_t *a = tiles + s * kStageBytes;
        uint8_t *b = a + kABytes;
        const int32_t ka = ks * KB * kBlockK;
        if constexpr (NSUB == 2) {
          // A k-block + one B k-block per segment; both CTAs' bytes on the leader's barrier
          if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * (kABytes + nsub * kBSub));
          if (P.a_hd)
            tma_load_3d_pair(a, &tmA, &full_bar[s], ka % P.a_hd, int(P.a_row0) + T.mb * kTileM, ka / P.a_hd);
          else
            tma_load_2d_pair(a, &tmA, &full_bar[s], ka, T.mb * kTileM);
          for (int sb = 0; sb < nsub; ++sb) {
            const SegDesc sd = P.segs[T.nb * NSUB + sb];
            const int nm = (sd.width + 15) & ~15;
            tma_load_2d_pair(b + sb * kBSub, &tmB, &full_bar[s], ka, sd.col0 + int(rank) * (nm / 2));
          }
        } else if constexpr (KB == 2 && ASRC == 1) {
          // A comes from the dequantising warps: only the B k-blocks through TMA
          if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * C::kBBytes);
#pragma unroll
          for (int kk = 0; kk < KB; ++kk)
            tma_load_2d_pair(b + kk * kBSub, &tmB, &full_bar[s], ka + kk * kBlockK, n0 + int(rank) * (n_mma / 2));
        } else if constexpr (KB == 2) {
          // two k-blocks per stage: A blocks then B blocks; both CTAs' bytes on the leader's barrier
          if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * kStageBytes);
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const int32_t kak = ka + kk * kBlockK;
            uint8_t *ak = a + kk * C::kABlock;
            if (P.a_hd && P.a_layer_rows)
              tma_load_2d_pair(ak, &tmA, &full_bar[s], kak % P.a_hd,
                               int((kak / P.a_hd) * P.a_layer_rows + P.a_row0) + T.mb * kTileM);
            else if (P.a_hd)
              tma_load_3d_pair(ak, &tmA, &full_bar[s], kak % P.a_hd, int(P.a_row0) + T.mb * kTileM, kak / P.a_hd);
            else
              tma_load_2d_pair(ak, &tmA, &full_bar[s], kak, T.mb * kTileM);
            tma_load_2d_pair(b + kk * kBSub, &tmB, &full_bar[s], kak, n0 + int(rank) * (n_mma / 2));
          }
          if (P.l2_pref > 0 && ks + P.l2_pref < num_st) {
#pragma unroll
            for (int kk = 0; kk < KB; ++kk) {
              const int32_t kpf = (ks + P.l2_pref) * KB * kBlockK + kk * kBlockK;
              if (P.a_hd && P.a_layer_rows)
                tma_prefetch_l2_2d(&tmA, kpf % P.a_hd, int((kpf / P.a_hd) * P.a_layer_rows + P.a_row0) + T.mb * kTileM);
              else if (P.a_hd)
                tma_prefetch_l2_3d(&tmA, kpf % P.a_hd, int(P.a_row0) + T.mb * kTileM, kpf / P.a_hd);
              else
                tma_prefetch_l2_2d(&tmA, kpf, T.mb * kTileM);
              tma_prefetch_l2_2d(&tmB, kpf, n0 + int(rank) * (n_mma / 2));
            }
          }
        } else if constexpr (PAIR) {
          // both CTAs' bytes land on the leader's barrier
          if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * kStageBytes);
          if (P.a_hd && P.hint_a)
            tma_3d_hint(true, a, &tmA, &full_bar[s], ka % P.a_hd, int(P.a_row0) + T.mb * kTileM, ka / P.a_hd, pol_a);
          else if (P.a_hd && P.a_layer_rows)
            tma_load_2d_pair(a, &tmA, &full_bar[s], ka % P.a_hd,
                             int((ka / P.a_hd) * P.a_layer_rows + P.a_row0) + T.mb * kTileM);
          else if (P.a_hd)
            tma_load_3d_pair(a, &tmA, &full_bar[s], ka % P.a_hd, int(P.a_row0) + T.mb * kTileM, ka / P.a_hd);
          else if (P.hint_a)
            tma_2d_hint(true, a, &tmA, &full_bar[s], ka, T.mb * kTileM, pol_a);
          else
            tma_load_2d_pair(a, &tmA, &full_bar[s], ka, T.mb * kTileM);
          if (P.hint_b)
            tma_2d_hint(true, b, &tmB, &full_bar[s], ka, n0 + int(rank) * (n_mma / 2), pol_b);
          else
            tma_load_2d_pair(b, &tmB, &full_bar[s], ka, n0 + int(rank) * (n_mma / 2));
        } else {
          mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
          if (P.a_hd)
            tma_load_3d(a, &tmA, &full_bar[s], ka % P.a_hd, int(P.a_row0) + T.mb * kTileM, ka / P.a_hd);
          else
            tma_load_2d(a, &tmA, &full_bar[s], ka, T.mb * kTileM);
          tma_load_2d(b, &tmB, &full_bar[s], ka, n0);
          tma_load_2d(b + kBBoxRows * 128, &tmB, &full_bar[s], ka, n0 + kBBoxRows);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (one thread; the pair leader issues for both CTAs)
    uint32_t it = 0, acc_it = 0;
    for (int64_t t = t_first; t < total; t += t_step) {
      const Tile T = get_tile(t);
      if (!T.valid) continue;
      int n0, ncols, g0, g1;
      tile_geometry<MODE, NSUB>(P, T, n0, ncols, g0, g1);
      const int n_mma = (ncols + 15) & ~15;
      const uint32_t idesc = make_idesc_f16(P.fmt, PAIR ? 2 * kTileM : kTileM, n_mma);
      const uint32_t acc = acc_it % kAccBufs;
      if (acc_it >= kAccBufs) {
        if (P.spin & 2) mbar_wait_spin(&tmem_empty[acc], ((acc_it / kAccBufs) - 1) & 1);
        else mbar_wait(&tmem_empty[acc], ((acc_it / kAccBufs) - 1) & 1);
      }
      tc_fence_after();
      const uint32_t tacc = tmem_base + acc * kMaxTileN;
      const int nsub = tile_nsub<NSUB>(P, T);
      uint32_t idesc_sub[NSUB];
#pragma unroll
      for (int sb = 0; sb < NSUB; ++sb)
        idesc_sub[sb] = NSUB == 1 ? idesc
                                  : make_idesc_f16(P.fmt, 2 * kTileM,
                                                   sb < nsub ? (P.segs[T.nb * NSUB + sb].width + 15) & ~15 : 16);
      for (int ks = 0; ks < num_st; ++ks, ++it) {
        const int kb = ks;                         // KB == 1: stage == k-block
        const int s = it % kStages;
        if constexpr (ASRC == 1) mbar_wait_cluster(&full_bar[s], (it / kStages) & 1);
        else if (P.spin & 8) mbar_wait_spin(&full_bar[s], (it / kStages) & 1);
        else mbar_wait(&full_bar[s], (it / kStages) & 1);
        tc_fence_after();
        const uint64_t ad = make_sdesc_sw128(tiles + s * kStageBytes);
        const uint64_t bd = make_sdesc_sw128(tiles + s * kStageBytes + kABytes);
        if constexpr (KB == 2) {
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) {
            const uint64_t adk = make_sdesc_sw128(tiles + s * kStageBytes + kk * C::kABlock);
            const uint64_t bdk = make_sdesc_sw128(tiles + s * kStageBytes + kABytes + kk * kBSub);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k)
              umma_f16_pair(tacc, adk + 2 * k, bdk + 2 * k, idesc, (ks | kk | k) != 0);
          }
          umma_commit_pair(&empty_bar[s]);
        } else if constexpr (NSUB == 2) {
          // segment sb accumulates in TMEM columns [256 sb, 256 sb + 256)
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k)
            for (int sb = 0; sb < nsub; ++sb)
              umma_f16_pair(tmem_base + sb * kMaxTileN, ad + 2 * k,
                            make_sdesc_sw128(tiles + s * kStageBytes + kABytes + sb * kBSub) + 2 * k, idesc_sub[sb],
                            (kb | k) != 0);
          umma_commit_pair(&empty_bar[s]);
        } else if constexpr (PAIR) {
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k)
            umma_f16_pair(tacc, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          umma_commit_pair(&empty_bar[s]);
        } else {
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k) umma_f16(tacc, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty_bar[s]);
        }
      }
      if constexpr (PAIR) umma_commit_pair(&tmem_full[acc]);
      else umma_commit(&tmem_full[acc]);
      ++acc_it;
    }
  } else if (ASRC == 1 && warp >= 8) {
    // ---------------- dequantising A producer (D2 fused into K5).  Two
    // groups of four warps take alternate pipeline stages (two stages' loads in
    // flight); in a group, warp q covers rows 32 q .. 32 q + 31 of this CTA's A
    // half, two rows per step with lane = (row, 16-byte chunk) so a row's codes
    // are read as contiguous bytes.  All loads of a stage are issued before its
    // smem slot is awaited.
    constexpr int kCh = KB * kBlockK / 8;          // 16 chunks per stage and row
    const int grp = (warp - 8) / 4, q = (warp - 8) % 4;
    const int half = lane >> 4, ch = lane & 15;
    const int kk = ch / 8, c8 = ch % 8;
    const DqChunk *tab = reinterpret_cast<const DqChunk *>(dq_tab);
    const int64_t my_tiles = t_first < total ? (total - t_first + t_step - 1) / t_step : 0;
    int64_t ti = 0;
    int ks = grp;
    while (ks >= num_st && num_st > 0) {           // few stages per tile: the group starts on a later tile
      ks -= num_st;
      ++ti;
      while (ks >= num_st && num_st > 0) {
        ks -= num_st;
        ++ti;
      }
    }
    for (; ti < my_tiles && num_st > 0;) {
      const Tile T = get_tile(t_first + ti * t_step);
      const uint8_t *tile = P.dq_payload;
      const int64_t *coff = P.dq_off_full;
      int ntok = 0;
      int64_t row0 = 0;                             // first tail-buffer row of this tile
      if (P.tiles) {
        if (T.mb < P.num_m) {
          const TileRef &tr = P.tiles[T.mb];
          tile = tr.payload;
          coff = tr.codes_off;
          ntok = tr.ntok;
        }
        row0 = int64_t(T.mb) * kTileM;
      } else {
        row0 = int64_t(T.mb) * kTileM;
        ntok = int(P.m - row0 < kTileM ? (P.m > row0 ? P.m - row0 : 0) : kTileM);
        tile = P.dq_payload + int64_t(T.mb) * P.tile_bytes;
        coff = ntok < kTileM ? P.dq_off_last : P.dq_off_full;
      }
      for (; ks < num_st; ks += kDqGroups) {
        const uint32_t n = uint32_t(ti * num_st + ks);          // stage index of this CTA
        const DqChunk d = tab[ks * kCh + ch];
        DqItem items[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int row = 32 * q + 2 * i + half;
          const uint8_t *tail_row = P.dq_tail ? P.dq_tail + (row0 + row) * P.dq_tail_ld : tile;
          if ((P.dq_debug & 1) == 0 && (ntok == kTileM || (ntok > 0 && d.ok == 3)))
            dq_item_issue(d, tile, tail_row, row, items[i]);
          else
            items[i] = DqItem{0x3C003C00u, 0u, 0u, 0u};
        }
        const int s = int(n % kStages);
        if (n >= uint32_t(kStages)) mbar_wait_spin(&empty_bar[s], ((n / kStages) - 1) & 1);
        uint8_t *a = tiles + s * kStageBytes + kk * (kTileM * kBlockK * 2);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (P.dq_debug & 2) break;
          const int row = 32 * q + 2 * i + half;
          const uint4 o = dq_item_value(d, P.dq_cols, ks * KB * kBlockK + ch * 8, tile, coff, ntok, row, items[i]);
          *reinterpret_cast<uint4 *>(a + row * 128 + ((c8 ^ (row & 7)) << 4)) = o;
        }
        if (!(P.dq_debug & 4)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&full_bar[s]);
          else mbar_arrive_remote(&full_bar[s], 0);
        }
      }
      ks -= num_st;
      ++ti;
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue
    auto release_acc = [&](uint32_t a) {
      if (!PAIR || leader) mbar_arrive(&tmem_empty[a]);
      else mbar_arrive_remote(&tmem_empty[a], 0);
    };
    const int row = (warp & 3) * 32 + lane;                 // TMEM lane == tile row
    uint32_t acc_it = 0;
    for (int64_t t = t_first; t < total; t += t_step) {
      const Tile T = get_tile(t);
      if (!T.valid) continue;
      int n0, ncols, seg_g0, seg_g1;
      tile_geometry<MODE, NSUB>(P, T, n0, ncols, seg_g0, seg_g1);
      const int n_mma = (ncols + 15) & ~15;
      const int64_t m0 = int64_t(T.mb) * kTileM;
      const int64_t tok = m0 + row;
      // batched rows: the tile's table entry (the odd M-block of the last CTA pair
      // may lie past the table: no entry, no valid rows)
      const TileRef *tref =
          (MODE == EPI_QUANT || MODE == EPI_RECON) && P.tiles && T.mb < P.num_m ? P.tiles + T.mb : nullptr;
      const bool valid = tref ? row < tref->ntok : tok < P.m;
      const uint32_t acc = acc_it % kAccBufs;
      if (P.spin & 4) mbar_wait_spin(&tmem_full[acc], (acc_it / kAccBufs) & 1);
      else mbar_wait(&tmem_full[acc], (acc_it / kAccBufs) & 1);
      tc_fence_after();
      const uint32_t trow = tmem_base + acc * kMaxTileN + (uint32_t((warp & 3) * 32) << 16);

      if constexpr (MODE == EPI_F32 || MODE == EPI_XTX) {
        for (int c = 0; c < n_mma; c += 16) {
          float v[16];
          tmem_ld16(trow + c, v);
          if (valid && num_kb > 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = n0 + c + j;
              if (c + j < ncols) {
                float *dst = P.D + tok * P.ldd + col;
                if constexpr (MODE == EPI_F32) *dst = __fsub_rn(v[j], P.bias[col]);
                else *dst += v[j];
              }
            }
          }
        }
        tc_fence_before();
        release_acc(acc);
      } else if constexpr (MODE == EPI_QUANT) {
        // Straight from TMEM, group by group: pass 1 min/max, pass 2 encode + pack
        // (no shared-memory staging, so the next tile's MMAs overlap this epilogue).
        const int ntok = tref ? tref->ntok : int(P.m - m0 < kTileM ? (P.m > m0 ? P.m - m0 : 0) : kTileM);
        const bool last = ntok < kTileM;
        uint8_t *tile_base = tref ? tref->payload : P.payload + T.mb * P.tile_bytes;
        const int64_t *codes_off_last = tref ? tref->codes_off : P.codes_off_last;
        const int nsub = P.epi_skip ? 0 : tile_nsub<NSUB>(P, T);
        int wide_w[NSUB];                          // wide groups whose piece this tile stored
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb) wide_w[sb] = -1;
        for (int sb = 0; sb < nsub; ++sb) {
        const SegDesc sdq = P.segs[T.nb * NSUB + sb];
        const uint32_t trow_s = trow + (NSUB == 2 ? uint32_t(sb * kMaxTileN) : 0u);
        const float *bias = P.bias + sdq.col0;
        const int f32_col = sdq.f32_col;
        const int ncols_s = sdq.width;
        if (f32_col >= 0) {
          // piece of a wide group: fp32 D - mu V_c and its row min/max to the scratch
          float *dst = P.D + (valid ? tok : 0) * P.ldd + f32_col;
          float pmn = INFINITY, pmx = -INFINITY;
          for (int c = 0; c < ncols_s; c += 16) {
            float x[16];
            load_cols(trow_s, bias, c, 16, x);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              pmn = fminf(pmn, x[j]);
              pmx = fmaxf(pmx, x[j]);
            }
            if (valid) {
#pragma unroll
              for (int j = 0; j < 16; j += 4)
                *reinterpret_cast<float4 *>(dst + c + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
            }
          }
          if (valid) P.wmm[tok * P.wpieces + f32_col / kMaxTileN] = make_float2(pmn, pmx);
          wide_w[sb] = sdq.wide;
        }
        // sub-byte code block of one group (tokens of size * bits < 8 bits): OR-reduction over the warp
        auto emit_subbyte = [&](const GroupDesc &g, uint32_t bits_v) {
          const int nb = g.full_size * bits_of(g.type);
          const int bitpos = lane * nb;
          uint8_t *cb = tile_base + (last ? codes_off_last[g.gidx] : g.codes_off);
          const int64_t blk_len = (int64_t(ntok) * nb + 7) / 8;
          const int64_t warp_byte0 = int64_t((warp & 3) * 32) * nb / 8;
          for (int w = 0; w < nb; ++w) {
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
        };
        auto store_params = [&](const GroupDesc &g, uint16_t sh, uint16_t sc) {
          if (valid && g.part == 0) {
            store_u32_any(tile_base + 4 * (int64_t(g.gidx) * ntok + row), uint32_t(sh) | (uint32_t(sc) << 16), !last);
            int32_t *stw = tref ? tref->status : P.status;
            if (factor_overflow(sh, sc) && stw) atomicOr(stw, 1);
          }
        };
        for (int gi = sdq.g_begin; gi < sdq.g_end;) {
          const GroupDesc gd = P.groups[gi];
          if (gd.full_size == 1) {
            // a run of size-1 groups (the DP's fp16-exact "keep" option, Q1): up to 16
            // columns per TMEM load instead of two single-column round trips each
            int n = 1;
            while (n < 16 && gi + n < sdq.g_end && P.groups[gi + n].full_size == 1) ++n;
            float v[16];
            if (gd.col + 16 <= kMaxTileN) {
              tmem_ld16(trow_s + gd.col, v);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = j < n ? tmem_ld1(trow_s + gd.col + j) : 0.0f;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j >= n) break;
              const GroupDesc g = P.groups[gi + j];
              const float x = __fsub_rn(v[j], bias[g.col]);
              uint16_t sh, sc;
              group_factors(g.type, x, x, sh, sc);
              store_params(g, sh, sc);
              emit_subbyte(g, valid ? encode_one(g.type, x, f16_val(sh), f16_val(sc)) : 0u);
            }
            gi += n;
            continue;
          }
          if (gd.size % 16 == 0 && gd.size <= 64 && gd.size == gd.full_size) {
            // one TMEM pass: all columns in registers (one wait), min/max, encode
            const int nq = gd.size / 16;
            uint32_t r[64];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < nq) tmem_ld16_nw(trow_s + gd.col + 16 * q, r + 16 * q);
            tmem_wait_ld();
            float mn = INFINITY, mx = -INFINITY;
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              if (j < gd.size) {
                const float x = __fsub_rn(__uint_as_float(r[j]), bias[gd.col + j]);
                mn = fminf(mn, x);
                mx = fmaxf(mx, x);
              }
            }
            uint16_t sh, sc;
            group_factors(gd.type, mn, mx, sh, sc);
            store_params(gd, sh, sc);
            const int bq = bits_of(gd.type);
            uint8_t *cb = tile_base + (last ? codes_off_last[gd.gidx] : gd.codes_off);
            if (valid) {
              const float shift = f16_val(sh), scale = f16_val(sc);
              uint8_t *dst = cb + int64_t(row) * (gd.size * bq / 8);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (q < nq) {
                  float x[16];
#pragma unroll
                  for (int j = 0; j < 16; ++j) x[j] = __fsub_rn(__uint_as_float(r[16 * q + j]), bias[gd.col + 16 * q + j]);
                  write_codes16(dst + 2 * q * bq, x, gd.type, shift, scale, !last);
                }
              }
            }
            ++gi;
            continue;
          }
          // generic: two TMEM passes (groups and pieces wider than 64 columns)
          const int step = (gd.size % 16 == 0) ? 16 : 1;
          float mn = INFINITY, mx = -INFINITY;
          for (int c = 0; c < gd.size; c += step) {
            float x[16];
            load_cols(trow_s, bias, gd.col + c, step, x);
            for (int j = 0; j < step; ++j) {
              mn = fminf(mn, x[j]);
              mx = fmaxf(mx, x[j]);
            }
          }
          uint16_t sh, sc;
          group_factors(gd.type, mn, mx, sh, sc);
          const float shift = f16_val(sh), scale = f16_val(sc);
          store_params(gd, sh, sc);
          const int bq = bits_of(gd.type);
          const int tok_bits = gd.full_size * bq;
          uint8_t *cb = tile_base + (last ? codes_off_last[gd.gidx] : gd.codes_off);
          if ((tok_bits & 7) == 0) {
            uint8_t *dst = cb + int64_t(row) * (tok_bits / 8) + gd.part * (gd.size * bq / 8);
            for (int c = 0; c < gd.size; c += step) {
              float x[16];
              load_cols(trow_s, bias, gd.col + c, step, x);
              if (valid) write_codes_aligned(dst + (c * bq) / 8, x, step, gd.type, shift, scale, !last);
            }
          } else {
            float x[16];
            load_cols(trow_s, bias, gd.col, gd.size, x);
            uint32_t bits_v = 0;
            for (int c = 0; c < gd.size; ++c) bits_v |= (valid ? encode_one(gd.type, x[c], shift, scale) : 0u) << (c * bq);
            emit_subbyte(gd, bits_v);
          }
          ++gi;
        }
        }
        tc_fence_before();
        release_acc(acc);
        // wide groups: the last piece's CTA quantises the whole group (after the
        // accumulator is released, so the next tile's MMAs are not held up)
        if (ntok > 0 && !P.wide_defer) {
          int32_t *stw = tref ? tref->status : P.status;
#pragma unroll
          for (int sb = 0; sb < NSUB; ++sb)
            if (wide_w[sb] >= 0)
              wide_fixup(P, wide_w[sb], T.mb, row, tok, valid, ntok, last, tile_base, codes_off_last, stw, wide_flag);
        }
      } else if constexpr (MODE == EPI_RECON) {
        // tcgen05.ld is warp-collective: every lane loads, only valid rows store
        const int d = P.head_dim;
        const int hd = P.heads * d;
        const int layer = n0 / hd;
        const int head0 = (n0 % hd) / d;
        const int64_t ctok = tref ? tref->tok0 + row : P.tok_begin + tok;
        __nv_bfloat16 *rowp = nullptr;
        if (valid) {
          int64_t slot = ctok;
          const int lay = tref ? tref->layout : P.layout;
          const int pt = tref ? tref->page_tokens : P.page_tokens;
          const int32_t *bt = tref ? tref->block_table : P.block_table;
          if (lay == KVTC_LAYOUT_PAGED) slot = int64_t(bt[ctok / pt]) * pt + (ctok % pt);
          rowp = (tref ? tref->bases : P.layer_base)[layer] + slot * hd;
        }
        const float2 *cs = (P.cs && valid) ? P.cs + tok * (d / 2) : nullptr;
        const bool rot = P.cs != nullptr;
        for (int hh = 0; hh < ncols / d; ++hh) {
          const int f = n0 + hh * d;                         // first feature of the head
          __nv_bfloat16 *dst = valid ? rowp + (head0 + hh) * d : nullptr;
          if (P.pairing == 0 || !rot) {
            for (int c = 0; c < d / 2; c += 16) {
              float lo[16], hi[16];
              tmem_ld16(trow + hh * d + c, lo);
              tmem_ld16(trow + hh * d + d / 2 + c, hi);
              if (!valid) continue;
              if (num_kb == 0) {
#pragma unroll
                for (int j = 0; j < 16; ++j) lo[j] = hi[j] = 0.0f;
              }
              __align__(16) __nv_bfloat16 olo[16], ohi[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float x1 = __fadd_rn(lo[j], P.bias[f + c + j]);
                const float x2 = __fadd_rn(hi[j], P.bias[f + d / 2 + c + j]);
                float y1 = x1, y2 = x2;
                if (rot) {
                  const float2 tt = cs[c + j];
                  y1 = __fsub_rn(__fmul_rn(x1, tt.x), __fmul_rn(x2, tt.y));
                  y2 = __fadd_rn(__fmul_rn(x2, tt.x), __fmul_rn(x1, tt.y));
                }
                olo[j] = __float2bfloat16_rn(y1);
                ohi[j] = __float2bfloat16_rn(y2);
              }
              uint4 *a = reinterpret_cast<uint4 *>(dst + c);
              uint4 *b = reinterpret_cast<uint4 *>(dst + d / 2 + c);
              a[0] = reinterpret_cast<uint4 *>(olo)[0];
              a[1] = reinterpret_cast<uint4 *>(olo)[1];
              b[0] = reinterpret_cast<uint4 *>(ohi)[0];
              b[1] = reinterpret_cast<uint4 *>(ohi)[1];
            }
          } else {
            for (int c = 0; c < d; c += 16) {
              float v[16];
              tmem_ld16(trow + hh * d + c, v);
              if (!valid) continue;
              if (num_kb == 0) {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 0.0f;
              }
              __align__(16) __nv_bfloat16 o[16];
#pragma unroll
              for (int j = 0; j < 16; j += 2) {
                const float x1 = __fadd_rn(v[j], P.bias[f + c + j]);
                const float x2 = __fadd_rn(v[j + 1], P.bias[f + c + j + 1]);
                const float2 tt = cs[(c + j) / 2];
                o[j] = __float2bfloat16_rn(__fsub_rn(__fmul_rn(x1, tt.x), __fmul_rn(x2, tt.y)));
                o[j + 1] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(x2, tt.x), __fmul_rn(x1, tt.y)));
              }
              uint4 *a = reinterpret_cast<uint4 *>(dst + c);
              a[0] = reinterpret_cast<uint4 *>(o)[0];
              a[1] = reinterpret_cast<uint4 *>(o)[1];
            }
          }
        }
        tc_fence_before();
        release_acc(acc);
      }
      ++acc_it;
    }
  }
  tc_fence_before();
  if constexpr (PAIR) {
    __syncwarp();
    cluster_sync_all();                          // both CTAs done with the pair's TMEM and smem
    if (warp == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
  } else {
    __syncthreads();
    if (warp == 2) tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// One zeroed counter per launch, from a per-device ring of 4096 (launches in
// flight never share one).
static unsigned long long *next_sync_counter() {
  static std::mutex mu;
  static unsigned long long *ring[64] = {};
  static uint32_t next[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!ring[dev & 63] && cudaMalloc(&ring[dev & 63], 4096 * sizeof(unsigned long long)) != cudaSuccess) {
    set_error("tile-sync counters: cudaMalloc failed");
    return nullptr;
  }
  return ring[dev & 63] + (next[dev & 63]++ % 4096);
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int MODE, bool PAIR, int NSUB = 1, int KB = 1, int ASRC = 0>
static kvtc_status launch(const CUtensorMap *tmA, const CUtensorMap *tmB, const Params &p, dim3 grid, int cluster,
                          cudaStream_t st) {
  static bool configured = false;
  using C = Cfg<PAIR, NSUB, KB>;
  // ASRC: the A-chunk table lives after the barriers (256 B in), up to kDqTabMaxBytes
  constexpr int kSmemMax = ASRC ? C::kStages * C::kStageBytes + 1024 + 256 + kDqTabMaxBytes : C::kSmemBytes;
  int smem_bytes = C::kSmemBytes;
  if (ASRC) {
    const int num_st = int(ceil_div(ceil_div(p.K, kBlockK), KB));
    smem_bytes = std::max(smem_bytes, C::kStages * C::kStageBytes + 1024 + 256 + num_st * KB * kBlockK / 8 * 16);
    if (smem_bytes > kSmemMax) {
      set_error("fused reconstruction: %d plan columns exceed the shared-memory chunk table", p.K);
      return KVTC_E_INVALID;
    }
  }
  if (!configured) {
    KVTC_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE, PAIR, NSUB, KB, ASRC>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
    // the 228 KB configuration, shared with the side-stream kernels (internal.h)
    KVTC_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE, PAIR, NSUB, KB, ASRC>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout,
                                       int(cudaSharedmemCarveoutMaxShared)));
    configured = true;
  }
  if (grid.x == 0 || grid.y == 0) return KVTC_OK;
  Params pp = p;
  {
    static const char *names[4] = {"KVTC_GROUP_M_F32", "KVTC_GROUP_M_QUANT", "KVTC_GROUP_M_RECON", "KVTC_GROUP_M_XTX"};
    const char *e = getenv(names[MODE]);
    // defaults from interleaved A/B sweeps of the bench step with the tile barrier on
    // (scripts/sweep_env.py; 16 beat 4 and 8 on the compress GEMM by ~0.4 ms per step)
    static const int defaults[4] = {kGroupM, 16, 16, kGroupM};
    pp.group_m = e ? std::max(1, atoi(e)) : defaults[MODE];
    const char *ha = getenv("KVTC_HINT_A"), *hb = getenv("KVTC_HINT_B");
    if (ha) pp.hint_a = atoi(ha);
    if (hb) pp.hint_b = atoi(hb);
    // soft tile barrier (tile_barrier) for the codec GEMMs; KVTC_TILE_SYNC = bit mask
    // over modes overrides (0 = off)
    const char *dd = getenv("KVTC_DQ_DEBUG");
    pp.dq_debug = dd ? atoi(dd) : 0;
    const char *sw = getenv("KVTC_SPIN_WAITS");
    pp.spin = sw ? atoi(sw) : 0;
    static const char *pref_names[4] = {"KVTC_L2_PREF_F32", "KVTC_L2_PREF_QUANT", "KVTC_L2_PREF_RECON",
                                        "KVTC_L2_PREF_XTX"};
    const char *pf = getenv(pref_names[MODE]);
    pp.l2_pref = pf ? atoi(pf) : 0;
    const char *es = getenv("KVTC_EPI_SKIP");
    pp.epi_skip = es && es[0] == '1';
    const char *ts = getenv("KVTC_TILE_SYNC");
    const int sync_mask = ts ? atoi(ts) : ((1 << EPI_QUANT) | (1 << EPI_RECON));
    // lag 0: every tile starts together (KVTC_SYNC_LAG_<MODE> = k lets a producer
    // run k tiles ahead; lag 1 on the decompress GEMM doubled its DRAM reads in ncu
    // for no step-time gain)
    static const char *lag_names[4] = {"KVTC_SYNC_LAG_F32", "KVTC_SYNC_LAG_QUANT", "KVTC_SYNC_LAG_RECON",
                                       "KVTC_SYNC_LAG_XTX"};
    const char *lg = getenv(lag_names[MODE]);
    pp.sync_lag = lg ? std::max(0, atoi(lg)) : 0;
    if ((sync_mask >> MODE) & 1) {
      if (!(pp.tile_sync = next_sync_counter())) return KVTC_E_CUDA;
      KVTC_CUDA_TRY(cudaMemsetAsync(pp.tile_sync, 0, sizeof(unsigned long long), st));
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads_for(ASRC));
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KVTC_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_kernel<MODE, PAIR, NSUB, KB, ASRC>, *tmA, *tmB, pp));
  note_launch();
  return KVTC_OK;
}

// 128-column (two k-block) pipeline stages for the codec GEMMs: half the
// full/empty barrier round trips per MMA.  ncu: compress 7.06 -> 6.39 ms (cache
// read in place) and 6.62 -> 6.32 ms, decompress 6.91 -> 6.51 ms; tensor pipe
// 90-94 % busy.  KVTC_KB2 = bit mask over modes overrides (0 = 64-column stages).
static bool kb2_for(int mode) {
  const char *e = getenv("KVTC_KB2");
  const int mask = e ? atoi(e) : ((1 << EPI_QUANT) | (1 << EPI_RECON));
  return (mask >> mode) & 1;
}

// pairs: 2 CTAs per pair-tile, grid even, at most one CTA per SM
static unsigned pair_grid(int64_t pair_tiles) {
  return unsigned(2 * std::min<int64_t>(pair_tiles, num_sms() / 2));
}

kvtc_status launch_gemm_project_f32(const GemmCompressArgs &a, int32_t ncols, cudaStream_t st) {
  Params p = {};
  p.K = a.K;
  p.m = a.m;
  p.ncols = ncols;
  p.bias = a.bias;
  p.D = a.D;
  p.ldd = a.ldd;
  p.fmt = 1;
  p.tile_n = kMaxTileN;
  p.num_m = int32_t(ceil_div(a.m, kTileM));
  p.num_n = int32_t(ceil_div(ncols, kMaxTileN));
  return launch<EPI_F32, true>(a.tmA, a.tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2, st);
}

kvtc_status launch_gemm_project_quant(const GemmCompressArgs &a, cudaStream_t st) {
  Params p = {};
  p.K = a.K;
  p.m = a.m;
  p.bias = a.bias;
  p.payload = a.payload;
  p.segs = a.segs;
  p.groups = a.groups;
  p.G = a.G;
  p.tile_bytes = a.tile_bytes;
  p.codes_off_last = a.codes_off_last;
  p.fmt = 1;
  p.a_hd = a.a_hd;
  p.a_layer_rows = a.a_layer_rows;
  p.a_row0 = a.a_row0;
  p.num_m = int32_t(ceil_div(a.m, kTileM));
  p.nsegs = a.nsegs;
  p.D = a.D;
  p.ldd = a.ldd;
  p.tiles = a.tiles;
  p.status = a.status;
  if (a.nwide > 0) {
    // scratch layout (wide_scratch_bytes): fp32 pieces, row min/max, counters
    p.wide = a.wide;
    p.nwide = a.nwide;
    p.wpieces = int32_t(a.ldd / kMaxTileN);
    p.wmm = reinterpret_cast<float2 *>(a.D + a.m * a.ldd);
    p.wcnt = reinterpret_cast<int32_t *>(p.wmm + a.m * p.wpieces);
    KVTC_CUDA_TRY(cudaMemsetAsync(p.wcnt, 0, size_t(ceil_div(a.m, kTileM)) * a.nwide * 4, st));
    const char *wd = getenv("KVTC_WIDE_DEFER");
    p.wide_defer = wd && wd[0] == '1';
  }
  // KVTC_QUANT_NSUB=2: two segments per tile (Cfg<true, 2>, 25 % less L2 traffic);
  // measured slower (tensor pipe 58 % vs 88 %: the 512-column epilogue is not
  // overlapped), so one segment per tile with double-buffered TMEM is the default
  const char *e = getenv("KVTC_QUANT_NSUB");
  if (e && atoi(e) == 2) {
    p.num_n = (a.nsegs + 1) / 2;
    return launch<EPI_QUANT, true, 2>(a.tmA, a.tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2, st);
  }
  p.num_n = a.nsegs;
  if (kb2_for(EPI_QUANT))
    return launch<EPI_QUANT, true, 1, 2>(a.tmA, a.tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2,
                                         st);
  return launch<EPI_QUANT, true>(a.tmA, a.tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2, st);
}

kvtc_status launch_gemm_reconstruct(const GemmDecompressArgs &a, cudaStream_t st) {
  Params p = {};
  p.K = a.K;
  p.m = a.m;
  p.n_begin = a.n_begin;
  p.ncols = a.n_end;
  p.bias = a.mu;
  p.cs = a.cs;
  p.layers = a.layers;
  p.heads = a.heads;
  p.head_dim = a.head_dim;
  p.pairing = a.pairing;
  p.layout = a.layout;
  p.page_tokens = a.page_tokens;
  p.layer_base = a.layer_base;
  p.block_table = a.block_table;
  p.tok_begin = a.tok_begin;
  p.tiles = a.tiles;
  p.fmt = 0;
  p.tile_n = a.tile_n;
  p.num_m = int32_t(ceil_div(a.m, kTileM));
  p.num_n = int32_t(ceil_div(a.n_end - a.n_begin, a.tile_n));
  if (a.dqcols) {
    // fused inverse path: A dequantised from the payload by the producer warps
    p.dq_payload = a.payload;
    p.dq_off_full = a.codes_off_full;
    p.dq_off_last = a.codes_off_last;
    p.dq_cols = a.dqcols;
    p.dq_chunks = a.dqchunks;
    p.dq_tail = a.dq_tail;
    p.dq_tail_ld = int64_t(a.n_tail) * 16;
    if (a.n_tail > 0 && a.m > 0) {
      KVTC_CHECK_ARG(a.dq_tail && a.tail_cols, "fused reconstruction: tail buffer");
      const int64_t items = int64_t(p.num_m) * kTileM * a.n_tail;
      KVTC_MAX_CARVEOUT(dq_tail_kernel);
      dq_tail_kernel<<<unsigned(std::min<int64_t>(ceil_div(items, 256), 8 * num_sms())), 256, 0, st>>>(
          a.dqcols, a.tail_cols, a.n_tail, a.payload, a.m, a.tile_bytes, a.codes_off_full, a.codes_off_last, a.tiles,
          p.num_m, a.dq_tail, p.dq_tail_ld);
      KVTC_LAUNCH_CHECK();
    }
    p.tile_bytes = a.tile_bytes;
    return launch<EPI_RECON, true, 1, 2, 1>(a.tmB, a.tmB, p,
                                            dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2, st);
  }
  if (kb2_for(EPI_RECON))
    return launch<EPI_RECON, true, 1, 2>(a.tmA, a.tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2,
                                         st);
  return launch<EPI_RECON, true>(a.tmA, a.tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2, st);
}

kvtc_status launch_gemm_xtx(const CUtensorMap *tmA, const CUtensorMap *tmB, int32_t p_, int32_t nk, float *S,
                            cudaStream_t st) {
  Params p = {};
  p.K = nk;
  p.m = p_;
  p.ncols = p_;
  p.D = S;
  p.ldd = p_;
  p.fmt = 1;
  p.tile_n = kMaxTileN;
  p.num_m = int32_t(ceil_div(p_, kTileM));
  p.num_n = int32_t(ceil_div(p_, kMaxTileN));
  p.parts = -2;                                   // marks pair tiling for the symmetric skip
  return launch<EPI_XTX, true>(tmA, tmB, p, dim3(pair_grid(int64_t((p.num_m + 1) / 2) * p.num_n)), 2, st);
}

}  // namespace kvtc
