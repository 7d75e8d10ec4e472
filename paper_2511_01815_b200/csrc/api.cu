// api.cu — the C ABI of include/kvtc.h: handles, plan compilation, the
// compress / decompress orchestration and the container format.
// Host code only orchestrates; every step of the data path runs in the
// library's sm_100a kernels (gemm.cu, elementwise.cu, deflate.cu).
#include <cstdarg>
#include <cstring>
#include <mutex>

#include "api_internal.h"

namespace kvtc {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

namespace {
kvtc_status encode_fn(EncodeTiledFn *out) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    KVTC_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return KVTC_E_CUDA;
    }
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  *out = fn;
  return KVTC_OK;
}
}  // namespace

kvtc_status make_tmap_3d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, uint64_t d0, uint64_t d1,
                         uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box0, uint32_t box1) {
  EncodeTiledFn fn;
  kvtc_status s = encode_fn(&fn);
  if (s) return s;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, dt, 3, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3d) failed (%d)", int(r));
    return KVTC_E_CUDA;
  }
  return KVTC_OK;
}

kvtc_status make_tmap_2d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                         uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn fn;
  kvtc_status s = encode_fn(&fn);
  if (s) return s;
  if (outer == 0 || inner == 0) {
    set_error("empty tensor map");
    return KVTC_E_INVALID;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu row=%llu", int(r),
              (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_bytes);
    return KVTC_E_CUDA;
  }
  return KVTC_OK;
}

uint64_t fnv1a(const void *data, size_t n, uint64_t h) {
  const uint8_t *p = static_cast<const uint8_t *>(data);
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001B3ull;
  return h;
}

// ------------------------------------------------------------ small kernels
__global__ void basis_operands_kernel(const float *V, int p, int r, int r_pad, __nv_bfloat16 *VcT, __half *Vd) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= int64_t(p) * r) return;
  const int f = int(i / r), j = int(i % r);
  const float v = V[i];
  VcT[int64_t(j) * p + f] = __float2bfloat16_rn(v);
  Vd[int64_t(f) * r_pad + j] = __float2half_rn(v);
}
// bias_j = sum_f mu_f * bf16(V_fj) in fp64 (mu V_c, R2)
__global__ void basis_bias_kernel(const float *mu, const __nv_bfloat16 *VcT, int p, int r, float *bias) {
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int f = threadIdx.x; f < p; f += blockDim.x)
    acc += double(mu[f]) * double(__bfloat162float(VcT[int64_t(j) * p + f]));
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) bias[j] = float(red[0]);
}
__global__ void plan_operands_kernel(const int32_t *pc, int r_nz, int p, int r_pad_full, int r_nz_pad,
                                     const __nv_bfloat16 *VcT_full, const __half *Vd_full, const float *bias_full,
                                     __nv_bfloat16 *VcT, __half *Vd, float *bias) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= int64_t(p) * r_nz) return;
  const int j = int(i / p), f = int(i % p);
  const int src = pc[j];
  VcT[int64_t(j) * (p + kXPad) + f] = VcT_full[int64_t(src) * p + f];
  Vd[int64_t(f) * r_nz_pad + j] = Vd_full[int64_t(f) * r_pad_full + src];
  if (f == 0) bias[j] = bias_full[src];
}

}  // namespace kvtc

using namespace kvtc;

// =================================================================== misc
extern "C" int32_t kvtc_abi_version(void) { return KVTC_ABI_VERSION; }
extern "C" const char *kvtc_last_error(void) { return g_err; }
extern "C" kvtc_status kvtc_device_check(void) {
  int dev = 0;
  KVTC_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  KVTC_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0) {
    set_error("device %s is sm_%d%d; this library is built for sm_100a", prop.name, prop.major, prop.minor);
    return KVTC_E_UNSUPPORTED;
  }
  return KVTC_OK;
}

// =================================================================== basis
kvtc_basis::~kvtc_basis() {
  cudaFree(d_mu);
  cudaFree(d_invf);
  cudaFree(d_V);
  cudaFree(d_VcT);
  cudaFree(d_Vd);
  cudaFree(d_bias);
}

extern "C" kvtc_status kvtc_basis_create(const kvtc_shape *shape, kvtc_stream which, const kvtc_rope *rope,
                                         int32_t rank, const float *mu_host, const float *V_host,
                                         const float *sigma_host, kvtc_basis **out) {
  KVTC_CHECK_ARG(shape && out && mu_host && V_host, "null argument");
  KVTC_CHECK_ARG(shape->layers > 0 && shape->kv_heads > 0 && shape->head_dim > 0, "shape");
  KVTC_CHECK_ARG(shape->head_dim % 32 == 0, "head_dim must be a multiple of 32");
  const int64_t p = int64_t(shape->layers) * shape->kv_heads * shape->head_dim;
  KVTC_CHECK_ARG(rank >= 1 && rank <= p, "rank");
  KVTC_CHECK_ARG(which == KVTC_VALUES || rope != nullptr, "keys need a RoPE description");
  kvtc_status st = kvtc_device_check();
  if (st != KVTC_OK) return st;
  auto *b = new kvtc_basis();
  b->shape = *shape;
  b->which = which;
  b->p = int32_t(p);
  b->r = rank;
  b->r_pad = (rank + 7) & ~7;
  b->mu.assign(mu_host, mu_host + p);
  b->V.assign(V_host, V_host + p * rank);
  if (sigma_host) b->sigma.assign(sigma_host, sigma_host + rank);
  else b->sigma.assign(rank, NAN);
  b->has_rope = which == KVTC_KEYS && rope;
  if (b->has_rope) {
    b->invf.assign(rope->inv_freq_host, rope->inv_freq_host + shape->head_dim / 2);
    b->pairing = rope->pairing;
  }
  auto fail = [&](kvtc_status s) {
    delete b;
    return s;
  };
#define B_TRY(x)                          \
  do {                                    \
    cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) {              \
      set_error("%s", cudaGetErrorString(e_)); \
      return fail(KVTC_E_CUDA);           \
    }                                     \
  } while (0)
  B_TRY(cudaMalloc(&b->d_mu, p * 4));
  B_TRY(cudaMalloc(&b->d_V, p * rank * 4));
  B_TRY(cudaMalloc(&b->d_VcT, p * rank * 2));
  B_TRY(cudaMalloc(&b->d_Vd, p * b->r_pad * 2));
  B_TRY(cudaMalloc(&b->d_bias, rank * 4));
  B_TRY(cudaMemset(b->d_Vd, 0, p * b->r_pad * 2));
  if (b->has_rope) {
    B_TRY(cudaMalloc(&b->d_invf, b->invf.size() * 4));
    B_TRY(cudaMemcpy(b->d_invf, b->invf.data(), b->invf.size() * 4, cudaMemcpyHostToDevice));
  }
  B_TRY(cudaMemcpy(b->d_mu, mu_host, p * 4, cudaMemcpyHostToDevice));
  B_TRY(cudaMemcpy(b->d_V, V_host, p * rank * 4, cudaMemcpyHostToDevice));
  basis_operands_kernel<<<unsigned(ceil_div(p * rank, 256)), 256>>>(b->d_V, int(p), rank, b->r_pad, b->d_VcT, b->d_Vd);
  basis_bias_kernel<<<rank, 256>>>(b->d_mu, b->d_VcT, int(p), rank, b->d_bias);
  B_TRY(cudaGetLastError());
  B_TRY(cudaDeviceSynchronize());
#undef B_TRY
  uint64_t h = 0xCBF29CE484222325ull;
  h = fnv1a(shape, sizeof(*shape), h);
  h = fnv1a(&which, sizeof(which), h);
  h = fnv1a(b->mu.data(), b->mu.size() * 4, h);
  h = fnv1a(b->V.data(), b->V.size() * 4, h);
  // the RoPE description is part of the transform (keys are re-rotated with it)
  const int32_t rope_meta[2] = {b->has_rope ? 1 : 0, b->pairing};
  h = fnv1a(rope_meta, sizeof(rope_meta), h);
  if (b->has_rope) h = fnv1a(b->invf.data(), b->invf.size() * 4, h);
  b->fp = h;
  *out = b;
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_basis_destroy(kvtc_basis *b) {
  delete b;
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_basis_get(const kvtc_basis *b, int32_t *p, int32_t *rank, float *mu_host, float *V_host,
                                      float *sigma_host) {
  KVTC_CHECK_ARG(b, "null basis");
  if (p) *p = b->p;
  if (rank) *rank = b->r;
  if (mu_host) memcpy(mu_host, b->mu.data(), b->mu.size() * 4);
  if (V_host) memcpy(V_host, b->V.data(), b->V.size() * 4);
  if (sigma_host) memcpy(sigma_host, b->sigma.data(), b->sigma.size() * 4);
  return KVTC_OK;
}

// =================================================================== plan
kvtc_plan::~kvtc_plan() {
  cudaFree(d_segs);
  cudaFree(d_wide);
  cudaFree(d_gdesc);
  cudaFree(d_pgroups);
  cudaFree(d_codes_off_full);
  cudaFree(d_dqcols);
  cudaFree(d_dqchunks);
  cudaFree(d_tail_cols);
  for (auto &kv : codes_off_last) cudaFree(kv.second);
  for (auto &kv : ops) {
    cudaFree(kv.second.VcT);
    cudaFree(kv.second.Vd);
    cudaFree(kv.second.bias);
  }
}

int64_t plan_tile_bytes(const kvtc_plan *pl, int64_t ntok) {
  int64_t b = 4 * int64_t(pl->G) * ntok;
  for (const auto &g : pl->groups) b += (ntok * g.size * bits_of(g.type) + 7) / 8;
  return b;
}

namespace kvtc {
kvtc_status plan_compile(kvtc_plan *pl) {
  const int G = int(pl->groups.size());
  if (G > 65535) {
    set_error("plan has %d non-None groups (at most 65535)", G);
    return KVTC_E_INVALID;
  }
  pl->G = G;
  if (plan_tile_bytes(pl, kTileM) > (int64_t(1) << 31) - 1) {
    set_error("plan bits per token too large for 32-bit tile offsets");
    return KVTC_E_INVALID;
  }
  int col = 0;
  pl->bits = 0;
  for (auto &g : pl->groups) {
    g.col = col;
    col += g.size;
    pl->bits += int64_t(g.size) * bits_of(g.type) + 32;
  }
  pl->r_nz = col;
  pl->r_nz_pad = (col + 7) & ~7;
  pl->r_eff = G ? pl->groups.back().start + pl->groups.back().size : 0;
  pl->tile_bytes = plan_tile_bytes(pl, kTileM);
  std::vector<int64_t> off(G);
  int64_t o = 4 * int64_t(G) * kTileM;
  for (int g = 0; g < G; ++g) {
    off[g] = o;
    o += (int64_t(kTileM) * pl->groups[g].size * bits_of(pl->groups[g].type) + 7) / 8;
  }
  // segments: groups of <= 256 columns packed greedily into <= 256-column tiles;
  // wider groups (k * 256) become k pieces whose tiles store fp32 coefficients
  // and row min/max to a scratch; the last piece to finish quantises the group
  // in its epilogue (the row min/max spans the pieces).
  std::vector<SegDesc> segs;
  std::vector<GroupDesc> gd;
  std::vector<SegDesc> wide_segs;
  std::vector<WideDesc> wide;
  int wcol = 0;
  SegDesc cur{-1, 0, 0, 0, -1};
  auto close = [&]() {
    if (cur.col0 >= 0 && cur.g_end > cur.g_begin) segs.push_back(cur);
    cur = SegDesc{-1, 0, int32_t(gd.size()), int32_t(gd.size()), -1, -1};
  };
  close();
  for (int g = 0; g < G; ++g) {
    const PlanGroup &pg = pl->groups[g];
    if (pg.size <= kMaxTileN) {
      if (cur.col0 < 0 || cur.width + pg.size > kMaxTileN) {
        close();
        cur.col0 = pg.col;
      }
      gd.push_back(GroupDesc{pg.col - cur.col0, pg.size, pg.size, pg.type, g, 0, off[g]});
      cur.width = pg.col + pg.size - cur.col0;
      cur.g_end = int32_t(gd.size());
    } else {
      if (pg.size % kMaxTileN != 0) {
        set_error("group size %d unsupported (sizes > 256 must be multiples of 256)", pg.size);
        return KVTC_E_INVALID;
      }
      for (int q = 0; q < pg.size / kMaxTileN; ++q)
        wide_segs.push_back(SegDesc{pg.col + q * kMaxTileN, kMaxTileN, 0, 0, wcol + q * kMaxTileN, int32_t(wide.size())});
      wide.push_back(WideDesc{g, pg.size, pg.type, pg.col, wcol, 0, off[g]});
      wcol += pg.size;
    }
  }
  close();
  for (SegDesc &w : wide_segs) {
    w.g_begin = w.g_end = int32_t(gd.size());
    segs.push_back(w);
  }
  pl->nwide = int(wide.size());
  pl->wide_cols = wcol;
  if (!wide.empty()) {
    KVTC_CUDA_TRY(cudaMalloc(&pl->d_wide, wide.size() * sizeof(WideDesc)));
    KVTC_CUDA_TRY(cudaMemcpy(pl->d_wide, wide.data(), wide.size() * sizeof(WideDesc), cudaMemcpyHostToDevice));
  }
  pl->nsegs = int(segs.size());
  KVTC_CUDA_TRY(cudaMalloc(&pl->d_segs, std::max<size_t>(1, segs.size()) * sizeof(SegDesc)));
  KVTC_CUDA_TRY(cudaMalloc(&pl->d_gdesc, std::max<size_t>(1, gd.size()) * sizeof(GroupDesc)));
  KVTC_CUDA_TRY(cudaMalloc(&pl->d_pgroups, std::max(1, G) * sizeof(PlanGroup)));
  KVTC_CUDA_TRY(cudaMalloc(&pl->d_codes_off_full, std::max(1, G) * sizeof(int64_t)));
  if (!segs.empty()) KVTC_CUDA_TRY(cudaMemcpy(pl->d_segs, segs.data(), segs.size() * sizeof(SegDesc), cudaMemcpyHostToDevice));
  if (!gd.empty()) KVTC_CUDA_TRY(cudaMemcpy(pl->d_gdesc, gd.data(), gd.size() * sizeof(GroupDesc), cudaMemcpyHostToDevice));
  if (G) {
    KVTC_CUDA_TRY(cudaMemcpy(pl->d_pgroups, pl->groups.data(), G * sizeof(PlanGroup), cudaMemcpyHostToDevice));
    KVTC_CUDA_TRY(cudaMemcpy(pl->d_codes_off_full, off.data(), G * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  // decompress A-operand columns (fused dequantising producer of K5): one entry
  // per compacted column, padded with zero columns to whole 128-column stages
  {
    const int ncols = int(ceil_div(std::max(col, 1), 2 * kBlockK) * 2 * kBlockK);
    std::vector<DqCol> dq(ncols, DqCol{0, 0, 0, 0, 0, 0, 0});
    for (int g = 0; g < G; ++g) {
      const PlanGroup &pg = pl->groups[g];
      for (int j = 0; j < pg.size; ++j)
        dq[pg.col + j] = DqCol{uint16_t(g), uint8_t(pg.type), 0, uint16_t(j), uint16_t(pg.size), int32_t(off[g]), 0};
    }
    std::vector<DqChunk> ch(ncols / 8, DqChunk{0, 0, 0, 0, 0, -1});
    std::vector<int32_t> tail;
    for (int c = 0; c < ncols; c += 8) {
      const DqCol &d = dq[c];
      DqChunk &k = ch[c / 8];
      bool any = false;
      for (int q = 0; q < 8; ++q) any |= dq[c + q].type != 0;
      k.type = any ? uint8_t(d.type ? d.type : 0xFF) : 0;
      if (c + 8 <= col && d.type && d.j % 8 == 0 && d.j + 8 <= d.size) {
        dq[c].chunk = 1;
        const int b = bits_of(d.type);
        k.ok = 1;
        k.code_base = d.off_full + d.j * b / 8;
        k.par_base = 4 * d.gidx * kTileM;
        k.stride = uint16_t(d.size * b / 8);
      } else if (any) {
        k.ok = 3;                       // dequantised by the pre-pass into the tail buffer
        k.code_base = int32_t(tail.size()) * 16;
        tail.push_back(c);
        // 8 consecutive size-1 groups of one type with adjacent code blocks
        bool run = c + 8 <= col && d.type && d.size == 1;
        const int b = d.type ? bits_of(d.type) : 0;
        for (int q = 1; run && q < 8; ++q) {
          const DqCol &e = dq[c + q];
          run = e.type == d.type && e.size == 1 && e.gidx == d.gidx + q && e.off_full == d.off_full + q * 16 * b;
        }
        if (run) {
          k.run_code = d.off_full;
          k.par_base = 4 * d.gidx * kTileM;
          k.stride = uint16_t(16 * b);
        }
      }
    }
    pl->dq_cols_n = ncols;
    pl->n_tail = int32_t(tail.size());
    if (!tail.empty()) {
      KVTC_CUDA_TRY(cudaMalloc(&pl->d_tail_cols, tail.size() * sizeof(int32_t)));
      KVTC_CUDA_TRY(cudaMemcpy(pl->d_tail_cols, tail.data(), tail.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    KVTC_CUDA_TRY(cudaMalloc(&pl->d_dqcols, ncols * sizeof(DqCol)));
    KVTC_CUDA_TRY(cudaMemcpy(pl->d_dqcols, dq.data(), ncols * sizeof(DqCol), cudaMemcpyHostToDevice));
    KVTC_CUDA_TRY(cudaMalloc(&pl->d_dqchunks, ch.size() * sizeof(DqChunk)));
    KVTC_CUDA_TRY(cudaMemcpy(pl->d_dqchunks, ch.data(), ch.size() * sizeof(DqChunk), cudaMemcpyHostToDevice));
  }
  uint64_t h = 0xCBF29CE484222325ull;
  h = fnv1a(&pl->r, 4, h);
  for (auto &g : pl->groups) {
    h = fnv1a(&g.start, 4, h);
    h = fnv1a(&g.size, 4, h);
    h = fnv1a(&g.type, 4, h);
  }
  pl->fp = h;
  return KVTC_OK;
}

// codes_off_last for a partial tile of ntok tokens (cached per ntok)
const int64_t *plan_codes_off_last(kvtc_plan *pl, int64_t ntok) {
  if (ntok <= 0 || ntok >= kTileM) return pl->d_codes_off_full;
  std::lock_guard<std::mutex> lk(pl->mu);
  auto it = pl->codes_off_last.find(int(ntok));
  if (it != pl->codes_off_last.end()) return it->second;
  std::vector<int64_t> off(std::max(1, pl->G));
  int64_t o = 4 * int64_t(pl->G) * ntok;
  for (int g = 0; g < pl->G; ++g) {
    off[g] = o;
    o += (ntok * pl->groups[g].size * bits_of(pl->groups[g].type) + 7) / 8;
  }
  int64_t *d = nullptr;
  if (cudaMalloc(&d, off.size() * 8) != cudaSuccess) return nullptr;
  cudaMemcpy(d, off.data(), off.size() * 8, cudaMemcpyHostToDevice);
  pl->codes_off_last[int(ntok)] = d;
  return d;
}

kvtc_status plan_operands(const kvtc_basis *b, kvtc_plan *pl, const Operands **out) {
  if (pl->r != b->r && pl->r_eff > b->r) {
    set_error("plan (r=%d, r_eff=%d) does not fit basis rank %d", pl->r, pl->r_eff, b->r);
    return KVTC_E_MISMATCH;
  }
  std::lock_guard<std::mutex> lk(pl->mu);
  Operands &op = pl->ops[b->fp];
  if (!op.ready) {
    op.r_nz = pl->r_nz;
    op.r_nz_pad = pl->r_nz_pad;
    if (op.r_nz > 0) {
      std::vector<int32_t> pc;
      for (auto &g : pl->groups)
        for (int k = 0; k < g.size; ++k) pc.push_back(g.start + k);
      int32_t *d_pc = nullptr;
      KVTC_CUDA_TRY(cudaMalloc(&d_pc, pc.size() * 4));
      KVTC_CUDA_TRY(cudaMemcpy(d_pc, pc.data(), pc.size() * 4, cudaMemcpyHostToDevice));
      KVTC_CUDA_TRY(cudaMalloc(&op.VcT, int64_t(op.r_nz) * (b->p + kXPad) * 2));
      KVTC_CUDA_TRY(cudaMemset(op.VcT, 0, int64_t(op.r_nz) * (b->p + kXPad) * 2));
      KVTC_CUDA_TRY(cudaMalloc(&op.Vd, int64_t(b->p) * op.r_nz_pad * 2));
      KVTC_CUDA_TRY(cudaMalloc(&op.bias, op.r_nz * 4));
      KVTC_CUDA_TRY(cudaMemset(op.Vd, 0, int64_t(b->p) * op.r_nz_pad * 2));
      plan_operands_kernel<<<unsigned(ceil_div(int64_t(b->p) * op.r_nz, 256)), 256>>>(
          d_pc, op.r_nz, b->p, b->r_pad, op.r_nz_pad, b->d_VcT, b->d_Vd, b->d_bias, op.VcT, op.Vd, op.bias);
      KVTC_CUDA_TRY(cudaGetLastError());
      KVTC_CUDA_TRY(cudaDeviceSynchronize());
      cudaFree(d_pc);
      kvtc_status st = make_tmap_2d(&op.tm_VcT, op.VcT, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, b->p, op.r_nz,
                                    uint64_t(b->p + kXPad) * 2, kBlockK, kMaxTileN / 2);
      if (st != KVTC_OK) return st;
      st = make_tmap_2d(&op.tm_Vd, op.Vd, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, op.r_nz, b->p, uint64_t(op.r_nz_pad) * 2,
                        kBlockK, kMaxTileN / 2);
      if (st != KVTC_OK) return st;
    }
    op.ready = true;
  }
  *out = &op;
  return KVTC_OK;
}
}  // namespace kvtc

extern "C" kvtc_status kvtc_plan_create(int32_t r, int32_t ngroups, const int32_t *start_host,
                                        const int32_t *size_host, const int32_t *type_host, kvtc_plan **out) {
  KVTC_CHECK_ARG(out && r >= 0 && ngroups >= 0, "plan arguments");
  KVTC_CHECK_ARG(ngroups == 0 || (start_host && size_host && type_host), "null plan arrays");
  auto *pl = new kvtc_plan();
  pl->r = r;
  int prev_end = 0;
  for (int g = 0; g < ngroups; ++g) {
    const int s = start_host[g], z = size_host[g], t = type_host[g];
    if (z <= 0 || s < prev_end || s + z > r || t < KVTC_T_INT2 || t > KVTC_T_FP8 ||
        !group_size_supported(z, bits_of(t))) {
      delete pl;
      set_error("invalid: group %d (start %d size %d type %d)%s", g, s, z, t,
                z > 0 && t >= KVTC_T_INT2 && t <= KVTC_T_FP8 && !group_size_supported(z, bits_of(t))
                    ? ": unsupported group size (see kvtc_plan_create)" : "");
      return KVTC_E_INVALID;
    }
    pl->groups.push_back(PlanGroup{s, z, t, 0});
    prev_end = s + z;
  }
  pl->expected_error = NAN;
  pl->budget = -1;
  kvtc_status st = plan_compile(pl);
  if (st != KVTC_OK) {
    delete pl;
    return st;
  }
  *out = pl;
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_plan_destroy(kvtc_plan *p) {
  delete p;
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_plan_get(const kvtc_plan *p, int32_t *r, int32_t *ngroups, int32_t *start_host,
                                     int32_t *size_host, int32_t *type_host, int64_t *bits_per_token, int32_t *r_eff,
                                     double *expected_error, int64_t *budget) {
  KVTC_CHECK_ARG(p, "null plan");
  if (r) *r = p->r;
  if (ngroups) *ngroups = p->G;
  for (int g = 0; g < p->G; ++g) {
    if (start_host) start_host[g] = p->groups[g].start;
    if (size_host) size_host[g] = p->groups[g].size;
    if (type_host) type_host[g] = p->groups[g].type;
  }
  if (bits_per_token) *bits_per_token = p->bits;
  if (r_eff) *r_eff = p->r_eff;
  if (expected_error) *expected_error = p->expected_error;
  if (budget) *budget = p->budget;
  return KVTC_OK;
}

extern "C" size_t kvtc_payload_bytes(const kvtc_plan *plan, int64_t m) {
  if (!plan || m <= 0) return 0;
  return size_t((m / kTileM) * plan->tile_bytes + plan_tile_bytes(plan, m % kTileM));
}

// ============================================================ stage entry points
namespace kvtc {
kvtc_status upload_bases(const kvtc_kv_view *v, void *dst_dev, cudaStream_t st) {
  KVTC_CUDA_TRY(cudaMemcpyAsync(dst_dev, v->layer_base_host, sizeof(void *) * v->shape.layers, cudaMemcpyHostToDevice,
                                st));
  return KVTC_OK;
}
kvtc_status check_view(const kvtc_kv_view *v) {
  KVTC_CHECK_ARG(v && v->layer_base_host, "null view");
  KVTC_CHECK_ARG(v->shape.layers > 0 && v->shape.kv_heads > 0 && v->shape.head_dim % 32 == 0, "view shape");
  KVTC_CHECK_ARG(v->layout == KVTC_LAYOUT_CONTIGUOUS || (v->layout == KVTC_LAYOUT_PAGED && v->page_tokens > 0 &&
                                                         v->block_table),
                 "view layout");
  return KVTC_OK;
}
}  // namespace kvtc

extern "C" kvtc_status kvtc_stage_gather(const kvtc_kv_view *v, int64_t tok_begin, int64_t ntok, int32_t unrope,
                                         const kvtc_rope *rope, void *X, void *stream) {
  kvtc_status st = check_view(v);
  if (st) return st;
  KVTC_CHECK_ARG(tok_begin >= 0 && ntok >= 0 && tok_begin + ntok <= v->tokens, "token range");
  KVTC_CHECK_ARG(!unrope || (rope && rope->inv_freq_host), "unrope needs rope");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int half = v->shape.head_dim / 2;
  Bump need;
  need.take<void *>(v->shape.layers);
  need.take<float>(half);
  need.take<float2>(ntok * half);
  void *scratch = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&scratch, need.used, s));
  Bump ws(scratch, need.used);
  auto *bases = ws.take<__nv_bfloat16 *>(v->shape.layers);
  float *invf = ws.take<float>(half);
  float2 *cs = ws.take<float2>(ntok * half);
  if ((st = upload_bases(v, bases, s))) return st;
  if (unrope) {
    KVTC_CUDA_TRY(cudaMemcpyAsync(invf, rope->inv_freq_host, half * 4, cudaMemcpyHostToDevice, s));
    if ((st = launch_rope_table(invf, half, v->pos0 + tok_begin, ntok, cs, s))) return st;
  }
  st = launch_gather(*v, bases, tok_begin, ntok, unrope ? cs : nullptr, unrope ? rope->pairing : 0,
                     static_cast<__nv_bfloat16 *>(X), s);
  cudaFreeAsync(scratch, s);
  return st;
}
