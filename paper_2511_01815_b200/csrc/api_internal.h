// api_internal.h — definitions of the opaque ABI handles and host helpers.
#pragma once

#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "internal.h"

// Calibrated transform of one stream: fp32 master on host and
// device, bf16 / fp16 GEMM operands derived by RNE (R2, R6).
struct kvtc_basis {
  kvtc_shape shape{};
  int32_t which = 0;
  int32_t p = 0, r = 0, r_pad = 0;
  std::vector<float> mu, V, sigma, invf;
  int32_t pairing = 0;
  bool has_rope = false;
  float *d_mu = nullptr;
  float *d_invf = nullptr;
  float *d_V = nullptr;               // [p x r] fp32 master
  __nv_bfloat16 *d_VcT = nullptr;     // [r x p] bf16
  __half *d_Vd = nullptr;             // [p x r_pad] fp16
  float *d_bias = nullptr;            // [r] mu V_c
  uint64_t fp = 0;
  ~kvtc_basis();
};

// Bit allocation of one stream compiled for the kernels.
struct kvtc_plan {
  int32_t r = 0;
  std::vector<kvtc::PlanGroup> groups;
  int32_t G = 0;
  int64_t bits = 0;
  int32_t r_eff = 0, r_nz = 0, r_nz_pad = 0;
  double expected_error = NAN;
  int64_t budget = -1;
  int64_t tile_bytes = 0;
  int32_t nsegs = 0;
  int32_t nwide = 0, wide_cols = 0;     // groups wider than a tile, their total columns
  kvtc::SegDesc *d_segs = nullptr;
  kvtc::WideDesc *d_wide = nullptr;
  kvtc::GroupDesc *d_gdesc = nullptr;
  kvtc::PlanGroup *d_pgroups = nullptr;
  int64_t *d_codes_off_full = nullptr;
  kvtc::DqCol *d_dqcols = nullptr;      // [r_nz rounded up to 128] decompress A-operand columns
  kvtc::DqChunk *d_dqchunks = nullptr;  // [the same / 8] 8-column chunks (fused producer table)
  int32_t dq_cols_n = 0;
  int32_t n_tail = 0;                   // ok = 3 chunks (dequantised by the pre-pass)
  int32_t *d_tail_cols = nullptr;
  std::map<int, int64_t *> codes_off_last;
  std::mutex mu;
  std::map<uint64_t, kvtc::Operands> ops;
  uint64_t fp = 0;
  ~kvtc_plan();
};

int64_t plan_tile_bytes(const kvtc_plan *pl, int64_t ntok);

namespace kvtc {
// Group sizes the compress / decompress kernels support for a type of `bits`
// bits: up to one 256-column tile with whole-byte tokens, or sub-byte tokens
// packed within one 32-bit word (the epilogue's warp OR-reduction); wider groups
// must be whole 256-column pieces.  {1, 16, 64, 256, 1024} qualify.
inline bool group_size_supported(int size, int bits) {
  if (size < 1) return false;
  if (size <= kMaxTileN) return (size * bits) % 8 == 0 || size * bits < 32;
  return size % kMaxTileN == 0;
}
uint64_t fnv1a(const void *data, size_t n, uint64_t h);
kvtc_status plan_compile(kvtc_plan *pl);
const int64_t *plan_codes_off_last(kvtc_plan *pl, int64_t ntok);
kvtc_status plan_operands(const kvtc_basis *b, kvtc_plan *pl, const Operands **out);
kvtc_status upload_bases(const kvtc_kv_view *v, void *dst_dev, cudaStream_t st);
kvtc_status check_view(const kvtc_kv_view *v);

// Carves aligned sub-buffers out of a caller workspace (or measures the need).
struct Bump {
  uint8_t *base;
  size_t cap, used = 0;
  explicit Bump(void *b = nullptr, size_t c = 0) : base(static_cast<uint8_t *>(b)), cap(c) {}
  template <typename T>
  T *take(size_t count, size_t align = 256) {
    used = (used + align - 1) / align * align;
    T *p = base ? reinterpret_cast<T *>(base + used) : nullptr;
    used += count * sizeof(T);
    return p;
  }
  bool ok() const { return base == nullptr || used <= cap; }
};
}  // namespace kvtc
