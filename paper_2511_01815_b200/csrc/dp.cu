// dp.cu — the DP precision assignment of P:L1541-1603 on the GPU (K7, K8),
// bit-exact with the literal loop (oracle/dp.py, oracle/dp_literal.c).
//
// K7  error table: for every block end i, allowed size s <= i and type t,
//     Z = sum x^2 and Q_t = sum (x - x^_t)^2 over P[:, i-s:i] in fp64, with the
//     canonical order of reading Q9 (per row sequential over the block, then an
//     adjacent-pair tree over rows zero-padded to a power of two).  A CTA holds
//     32 rows x (max size + 64) columns of P in shared memory; lane = row, so the
//     first 5 tree levels are warp shuffles; kernel 2 finishes the tree over the
//     32-row chunks.  x^ follows Q2/Q3/Q5 in fp64 exactly as the oracle does
//     (explicit __d*_rn: no FMA contraction).
// K8  table recursion, one CTA: for each (i, size) pass of the pseudocode the
//     budget loop is the scan of reading Q7:
//         C[b] = first-min over types of E_t + best[i-s][b-cost_t]
//         S[b] = leftmost-argmin inclusive prefix scan of C
//         new[b] = old[b] if old[b] <= S[b] else S[b]
//     over even budgets only (every cost is even; odd columns equal the even
//     column below them, value and pointer — pinned in tests/test_oracle_dp.py).
// Backtracking from (r, B) runs on one thread.
#include <algorithm>
#include <vector>

#include "api_internal.h"

using namespace kvtc;

namespace {

constexpr int kRowsPerCta = 32;
constexpr int kITile = 64;
constexpr int kEThreads = 256;
constexpr int kMaxSizes = 8;

struct DPParams {
  const float *P;
  int64_t n;
  int32_t r;
  int32_t nsizes;
  int32_t sizes[kMaxSizes];
  int32_t maxsize;
  uint32_t type_mask;
};

__device__ __forceinline__ double qerr_intk(double x, double sh, double sc, double L) {
  double xh;
  if (sc == 0.0) {
    xh = __dadd_rn(__dmul_rn(0.0, sc), sh);
  } else {
    double y = __ddiv_rn(__dsub_rn(x, sh), sc);
    double c = rint(y);
    c = fmin(fmax(c, 0.0), L);
    xh = __dadd_rn(__dmul_rn(c, sc), sh);
  }
  const double e = __dsub_rn(x, xh);
  return __dmul_rn(e, e);
}
__device__ __forceinline__ double qerr_fp8(double x, double sh, double sc) {
  double xh;
  if (sc == 0.0) {
    xh = __dadd_rn(__dmul_rn(0.0, sc), sh);
  } else {
    const float y = __double2float_rn(__ddiv_rn(__dsub_rn(x, sh), sc));
    const double v = double(e4m3_to_f32(e4m3_from_f32(y)));
    xh = __dadd_rn(__dmul_rn(v, sc), sh);
  }
  const double e = __dsub_rn(x, xh);
  return __dmul_rn(e, e);
}

__device__ __forceinline__ double warp_tree(double v) {
  // adjacent-pair binary tree over the 32 lanes (= rows): (0+1), (2+3), ...
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// partial[chunk][i][si][4] = 32-row tree sums of (Z, Q_int2, Q_int4, Q_fp8)
__global__ void __launch_bounds__(kEThreads) etable_kernel(DPParams prm, double *partial) {
  extern __shared__ float sP[];   // [cols][32]
  const int64_t chunk = blockIdx.y;
  const int64_t row0 = chunk * kRowsPerCta;
  const int i0 = 1 + blockIdx.x * kITile;                        // first block end handled
  const int c_lo = max(0, i0 - prm.maxsize);                     // first column needed
  const int c_hi = min(prm.r, i0 + kITile - 1);                  // one past the last column
  const int ncol = c_hi - c_lo;
  for (int k = threadIdx.x; k < ncol * kRowsPerCta; k += kEThreads) {
    const int c = k / kRowsPerCta, rr = k % kRowsPerCta;
    const int64_t row = row0 + rr;
    sP[k] = row < prm.n ? prm.P[row * prm.r + c_lo + c] : 0.0f;
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool has2 = prm.type_mask & (1u << KVTC_T_INT2), has4 = prm.type_mask & (1u << KVTC_T_INT4),
             has8 = prm.type_mask & (1u << KVTC_T_FP8);
  const int nchunks_i = gridDim.y;
  (void)nchunks_i;
  for (int ii = warp; ii < kITile; ii += kEThreads / 32) {
    const int i = i0 + ii;
    if (i > prm.r) break;
    for (int si = 0; si < prm.nsizes; ++si) {
      const int s = prm.sizes[si];
      if (s > i) continue;
      const float *col = sP + (i - s - c_lo) * kRowsPerCta + lane;
      double z = 0.0, mn = double(col[0]), mx = mn;
      for (int c = 0; c < s; ++c) {
        const double x = double(col[c * kRowsPerCta]);
        z = __dadd_rn(z, __dmul_rn(x, x));
        mn = fmin(mn, x);
        mx = fmax(mx, x);
      }
      const double sh2 = f16_rne_f64(mn);
      const double sc2 = f16_rne_f64(__ddiv_rn(__dsub_rn(mx, mn), 3.0));
      const double sc4 = f16_rne_f64(__ddiv_rn(__dsub_rn(mx, mn), 15.0));
      const double sh8 = f16_rne_f64(__ddiv_rn(__dadd_rn(mx, mn), 2.0));
      const double sc8 = f16_rne_f64(__ddiv_rn(__ddiv_rn(__dsub_rn(mx, mn), 2.0), 448.0));
      double q2 = 0.0, q4 = 0.0, q8 = 0.0;
      for (int c = 0; c < s; ++c) {
        const double x = double(col[c * kRowsPerCta]);
        if (has2) q2 = __dadd_rn(q2, qerr_intk(x, sh2, sc2, 3.0));
        if (has4) q4 = __dadd_rn(q4, qerr_intk(x, sh2, sc4, 15.0));
        if (has8) q8 = __dadd_rn(q8, qerr_fp8(x, sh8, sc8));
      }
      z = warp_tree(z);
      q2 = warp_tree(q2);
      q4 = warp_tree(q4);
      q8 = warp_tree(q8);
      if (lane == 0) {
        double *o = partial + ((chunk * (prm.r + 1) + i) * prm.nsizes + si) * 4;
        o[0] = z;
        o[1] = q2;
        o[2] = q4;
        o[3] = q8;
      }
    }
  }
}

// Finish the tree over the 32-row chunks (zero-padded to a power of two; adding
// a padded zero is exact, so those additions are skipped), in place, then write
// E[i][si][t] = -Z + Q_t (None: -Z + Z = 0 exactly).
__global__ void etable_reduce_kernel(double *partial, int64_t nchunks, int64_t per, double *E) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;   // (i, si, q)
  if (e >= per) return;
  for (int64_t stride = 1; stride < nchunks; stride <<= 1)
    for (int64_t c = 0; c + stride < nchunks; c += 2 * stride)
      partial[c * per + e] = __dadd_rn(partial[c * per + e], partial[(c + stride) * per + e]);
}
__global__ void etable_final_kernel(const double *partial, int64_t nisz, double *E) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;   // (i, si)
  if (k >= nisz) return;
  const double z = partial[k * 4];
  E[k * 4 + 0] = 0.0;
  for (int q = 1; q < 4; ++q) E[k * 4 + q] = __dadd_rn(-z, partial[k * 4 + q]);
}

// ---------------------------------------------------------------- K8 scan
struct ScanItem {
  double v;
  uint32_t p;
};
__device__ __forceinline__ ScanItem leftmin(ScanItem a, ScanItem b) { return b.v < a.v ? b : a; }

constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads) dp_scan_kernel(const double *E, int32_t r, int32_t nsizes,
                                                               const int32_t *sizes, uint32_t type_mask, int64_t W,
                                                               double init, double *best, uint8_t *ptr) {
  __shared__ ScanItem agg[kScanThreads];
  __shared__ ScanItem wsum[32];
  const int t = threadIdx.x;
  const int64_t per = (W - 1 + kScanThreads - 1) / kScanThreads;
  const int64_t b_lo = 1 + t * per, b_hi = min(W, b_lo + per);     // this thread's even-budget slots [b_lo, b_hi)
  for (int64_t k = t; k < int64_t(r + 1) * W; k += kScanThreads) {
    best[k] = init;
    ptr[k] = 0;
  }
  __syncthreads();
  int hcost[kMaxSizes][4];
  for (int si = 0; si < nsizes; ++si)
    for (int ty = 0; ty < 4; ++ty) {
      const int bits = ty == 0 ? 0 : ty == 1 ? 2 : ty == 2 ? 4 : 8;
      hcost[si][ty] = ty == 0 ? 0 : (sizes[si] * bits + 32) / 2;
    }
  for (int i = 1; i <= r; ++i) {
    double *row = best + int64_t(i) * W;
    uint8_t *prow = ptr + int64_t(i) * W;
    for (int si = 0; si < nsizes; ++si) {
      const int s = sizes[si];
      if (s > i) continue;
      const double *prev = best + int64_t(i - s) * W;
      const double *Ei = E + (int64_t(i) * nsizes + si) * 4;
      double e[4];
      for (int ty = 0; ty < 4; ++ty) e[ty] = Ei[ty];
      // pass 1: this thread's aggregate of C over [b_lo, b_hi)
      ScanItem acc{INFINITY, 0};
      for (int64_t b = b_lo; b < b_hi; ++b) {
        ScanItem c{INFINITY, 0};
        for (int ty = 0; ty < 4; ++ty) {
          if (ty && !(type_mask & (1u << ty))) continue;
          const int h = hcost[si][ty];
          if (h > b) continue;
          const double v = __dadd_rn(e[ty], prev[b - h]);
          if (v < c.v) c = ScanItem{v, uint32_t(ty | (si << 2) | 0x80)};
        }
        acc = leftmin(acc, c);
      }
      // exclusive block scan of the aggregates (leftmost-argmin)
      agg[t] = acc;
      ScanItem x = acc;
      const int lane = t & 31, wid = t >> 5;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        ScanItem y{__shfl_up_sync(0xffffffffu, x.v, off), __shfl_up_sync(0xffffffffu, x.p, off)};
        if (lane >= off) x = leftmin(y, x);
      }
      if (lane == 31) wsum[wid] = x;
      __syncthreads();
      if (wid == 0) {
        ScanItem w = wsum[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          ScanItem y{__shfl_up_sync(0xffffffffu, w.v, off), __shfl_up_sync(0xffffffffu, w.p, off)};
          if (lane >= off) w = leftmin(y, w);
        }
        wsum[lane] = w;
      }
      __syncthreads();
      // carry-in = everything strictly left of this thread
      ScanItem carry{INFINITY, 0};
      if (wid > 0) carry = wsum[wid - 1];
      {
        ScanItem y{__shfl_up_sync(0xffffffffu, x.v, 1), __shfl_up_sync(0xffffffffu, x.p, 1)};
        if (lane > 0) carry = leftmin(carry, y);
      }
      // pass 2: recompute C, running scan, apply new[b] = old <= S ? old : S
      ScanItem S = carry;
      for (int64_t b = b_lo; b < b_hi; ++b) {
        ScanItem c{INFINITY, 0};
        for (int ty = 0; ty < 4; ++ty) {
          if (ty && !(type_mask & (1u << ty))) continue;
          const int h = hcost[si][ty];
          if (h > b) continue;
          const double v = __dadd_rn(e[ty], prev[b - h]);
          if (v < c.v) c = ScanItem{v, uint32_t(ty | (si << 2) | 0x80)};
        }
        S = leftmin(S, c);
        if (!(row[b] <= S.v)) {
          row[b] = S.v;
          prow[b] = uint8_t(S.p);
        }
      }
      __syncthreads();
    }
  }
}

// backtrack from (r, B/2): groups written in PC order; out[0] = ngroups
__global__ void dp_backtrack_kernel(const uint8_t *ptr, int32_t r, int64_t W, int64_t bhalf, const int32_t *sizes,
                                    int32_t *out, const double *best, double *err) {
  int i = r;
  int64_t b = bhalf;
  int ng = 0;
  *err = best[int64_t(r) * W + bhalf];
  while (i > 0) {
    const uint8_t p = ptr[int64_t(i) * W + b];
    if (!(p & 0x80)) break;
    const int ty = p & 3, si = (p >> 2) & 7;
    const int s = sizes[si];
    const int bits = ty == 0 ? 0 : ty == 1 ? 2 : ty == 2 ? 4 : 8;
    const int h = ty == 0 ? 0 : (s * bits + 32) / 2;
    out[1 + 3 * ng + 0] = i - s;
    out[1 + 3 * ng + 1] = s;
    out[1 + 3 * ng + 2] = ty;
    ++ng;
    i -= s;
    b -= h;
  }
  out[0] = ng;
}

struct DPRun {
  double *E = nullptr, *best = nullptr;
  uint8_t *ptr = nullptr;
  int64_t W = 0, B = 0;
};

kvtc_status dp_run(const float *P, int64_t n, int32_t r, int64_t B, const kvtc_dp_config *cfg, cudaStream_t st,
                   DPRun &run, std::vector<int32_t> &sizes_h) {
  KVTC_CHECK_ARG(P && n >= 1 && r >= 1 && B >= 0, "dp arguments");
  sizes_h.clear();
  if (cfg && cfg->nsizes > 0 && cfg->sizes_host) {
    for (int k = 0; k < cfg->nsizes; ++k) sizes_h.push_back(cfg->sizes_host[k]);
  } else {
    sizes_h = {1, 16, 64, 256, 1024};
  }
  KVTC_CHECK_ARG(int(sizes_h.size()) <= kMaxSizes, "too many group sizes");
  int maxsize = 0;
  const uint32_t mask = (cfg && cfg->type_mask) ? (cfg->type_mask | 1u) : 0xFu;
  for (int s : sizes_h) {
    KVTC_CHECK_ARG(s >= 1 && s <= 1024, "group sizes must be in [1, 1024]");
    for (int t = KVTC_T_INT2; t <= KVTC_T_FP8; ++t)
      KVTC_CHECK_ARG(!((mask >> t) & 1) || group_size_supported(s, bits_of(t)),
                     "group size unsupported by the codec kernels for an allowed type (see kvtc_plan_create)");
    maxsize = std::max(maxsize, s);
  }
  maxsize = std::min(maxsize, r);
  const int nsz = int(sizes_h.size());
  // ---- K7
  DPParams prm = {};
  prm.P = P;
  prm.n = n;
  prm.r = r;
  prm.nsizes = nsz;
  for (int k = 0; k < nsz; ++k) prm.sizes[k] = sizes_h[k];
  prm.maxsize = maxsize;
  prm.type_mask = mask;
  const int64_t nchunks = ceil_div(n, kRowsPerCta);
  const int64_t per = int64_t(r + 1) * nsz * 4;
  double *partial = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&partial, size_t(nchunks) * per * 8, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(partial, 0, size_t(nchunks) * per * 8, st));
  KVTC_CUDA_TRY(cudaMallocAsync(&run.E, size_t(per) * 8, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(run.E, 0, size_t(per) * 8, st));
  const size_t smem = size_t(maxsize + kITile) * kRowsPerCta * 4;
  KVTC_CUDA_TRY(cudaFuncSetAttribute(etable_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid(unsigned(ceil_div(r, kITile)), unsigned(nchunks));
  etable_kernel<<<grid, kEThreads, smem, st>>>(prm, partial);
  KVTC_LAUNCH_CHECK();
  etable_reduce_kernel<<<unsigned(ceil_div(per, 256)), 256, 0, st>>>(partial, nchunks, per, run.E);
  KVTC_LAUNCH_CHECK();
  etable_final_kernel<<<unsigned(ceil_div(per / 4, 256)), 256, 0, st>>>(partial, per / 4, run.E);
  KVTC_LAUNCH_CHECK();
  cudaFreeAsync(partial, st);
  run.B = B;
  run.W = B / 2 + 1;
  KVTC_CUDA_TRY(cudaMallocAsync(&run.best, size_t(r + 1) * run.W * 8, st));
  KVTC_CUDA_TRY(cudaMallocAsync(&run.ptr, size_t(r + 1) * run.W, st));
  return KVTC_OK;
}

// ||P||^2: per row sequential over all columns, tree over rows (zero-padded)
__global__ void init_rows_kernel(const float *P, int64_t n, int32_t r, int64_t pow2, double *rows) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= pow2) return;
  double s = 0.0;
  if (k < n)
    for (int c = 0; c < r; ++c) {
      const double x = double(P[k * r + c]);
      s = __dadd_rn(s, __dmul_rn(x, x));
    }
  rows[k] = s;
}
__global__ void tree_kernel(double *v, int64_t pow2) {
  // single block: adjacent-pair tree in place
  for (int64_t stride = 1; stride < pow2; stride <<= 1) {
    for (int64_t c = 2 * stride * threadIdx.x; c < pow2; c += 2 * stride * blockDim.x) v[c] = __dadd_rn(v[c], v[c + stride]);
    __syncthreads();
  }
}

kvtc_status dp_initial(const float *P, int64_t n, int32_t r, cudaStream_t st, double *init) {
  int64_t pow2 = 1;
  while (pow2 < n) pow2 *= 2;
  double *rows = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&rows, size_t(pow2) * 8, st));
  init_rows_kernel<<<unsigned(ceil_div(pow2, 256)), 256, 0, st>>>(P, n, r, pow2, rows);
  tree_kernel<<<1, 1024, 0, st>>>(rows, pow2);
  KVTC_LAUNCH_CHECK();
  KVTC_CUDA_TRY(cudaMemcpyAsync(init, rows, 8, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(rows);
  return KVTC_OK;
}

kvtc_status dp_full(const float *P, int64_t n, int32_t r, int64_t B, const kvtc_dp_config *cfg, cudaStream_t st,
                    DPRun &run, std::vector<int32_t> &sizes_h) {
  kvtc_status s = dp_run(P, n, r, B, cfg, st, run, sizes_h);
  if (s) return s;
  double init = 0;
  if ((s = dp_initial(P, n, r, st, &init))) return s;
  int32_t *d_sizes = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&d_sizes, sizes_h.size() * 4, st));
  KVTC_CUDA_TRY(cudaMemcpyAsync(d_sizes, sizes_h.data(), sizes_h.size() * 4, cudaMemcpyHostToDevice, st));
  const uint32_t mask = (cfg && cfg->type_mask) ? (cfg->type_mask | 1u) : 0xFu;
  dp_scan_kernel<<<1, kScanThreads, 0, st>>>(run.E, r, int32_t(sizes_h.size()), d_sizes, mask, run.W, init, run.best,
                                             run.ptr);
  KVTC_LAUNCH_CHECK();
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(d_sizes);
  return KVTC_OK;
}

void dp_free(DPRun &run) {
  cudaFree(run.E);
  cudaFree(run.best);
  cudaFree(run.ptr);
}

int64_t budget_from(const kvtc_dp_config *cfg, int32_t p_original) {
  const int fb = cfg->feature_bits > 0 ? cfg->feature_bits : 16;
  return int64_t(std::floor(double(fb) * double(p_original) / cfg->target_cr));
}

}  // namespace

extern "C" kvtc_status kvtc_dp_best_table(const float *P, int64_t n, int32_t r, int64_t budget,
                                          const kvtc_dp_config *cfg, double *best_even, void *stream) {
  KVTC_CHECK_ARG(best_even, "null table");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DPRun run;
  std::vector<int32_t> sizes;
  kvtc_status s = dp_full(P, n, r, budget, cfg, st, run, sizes);
  if (s == KVTC_OK)
    KVTC_CUDA_TRY(cudaMemcpyAsync(best_even, run.best, size_t(r + 1) * run.W * 8, cudaMemcpyDeviceToDevice, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  dp_free(run);
  return s;
}

namespace {
// Plan of budget column B (bits) from a finished DP run: backtrack (Q7) and compile.
kvtc_status backtrack_plan(const DPRun &run, int32_t r, int64_t B, const std::vector<int32_t> &sizes,
                           cudaStream_t st, kvtc_plan **out) {
  int32_t *d_out = nullptr;
  double *d_err = nullptr;
  int32_t *d_sizes = nullptr;
  KVTC_CUDA_TRY(cudaMalloc(&d_out, (1 + 3 * size_t(r)) * 4));
  KVTC_CUDA_TRY(cudaMalloc(&d_err, 8));
  KVTC_CUDA_TRY(cudaMalloc(&d_sizes, sizes.size() * 4));
  KVTC_CUDA_TRY(cudaMemcpy(d_sizes, sizes.data(), sizes.size() * 4, cudaMemcpyHostToDevice));
  dp_backtrack_kernel<<<1, 1, 0, st>>>(run.ptr, r, run.W, B / 2, d_sizes, d_out, run.best, d_err);
  KVTC_LAUNCH_CHECK();
  std::vector<int32_t> h(1 + 3 * size_t(r));
  double err = 0;
  KVTC_CUDA_TRY(cudaMemcpyAsync(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaMemcpyAsync(&err, d_err, 8, cudaMemcpyDeviceToHost, st));
  KVTC_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(d_out);
  cudaFree(d_err);
  cudaFree(d_sizes);
  const int ng = h[0];
  std::vector<int32_t> gs, gz, gt;
  for (int k = ng - 1; k >= 0; --k) {            // reverse: PC order
    if (h[1 + 3 * k + 2] == KVTC_T_NONE) continue;
    gs.push_back(h[1 + 3 * k]);
    gz.push_back(h[1 + 3 * k + 1]);
    gt.push_back(h[1 + 3 * k + 2]);
  }
  kvtc_plan *pl = nullptr;
  kvtc_status s = kvtc_plan_create(r, int32_t(gs.size()), gs.data(), gz.data(), gt.data(), &pl);
  if (s) return s;
  pl->expected_error = err;
  pl->budget = B;
  *out = pl;
  return KVTC_OK;
}
}  // namespace

extern "C" kvtc_status kvtc_allocate_bits_from_coeffs(const float *P, int64_t n, int32_t r, int32_t p_original,
                                                      const kvtc_dp_config *cfg, void *stream, kvtc_plan **out) {
  KVTC_CHECK_ARG(cfg && out && cfg->target_cr > 0 && p_original > 0, "allocate arguments");
  return kvtc_allocate_bits_from_coeffs_multi(P, n, r, p_original, cfg, &cfg->target_cr, 1, stream, out);
}

// One DP table at the largest budget serves every target CR: column b of the
// table does not depend on how many columns were computed, so the plan of budget
// B' is the backtrack from (r, B') (Q6/Q7; pinned against single-CR plans).
extern "C" kvtc_status kvtc_allocate_bits_from_coeffs_multi(const float *P, int64_t n, int32_t r, int32_t p_original,
                                                            const kvtc_dp_config *cfg, const double *crs_host,
                                                            int32_t ncr, void *stream, kvtc_plan **out) {
  KVTC_CHECK_ARG(cfg && out && crs_host && ncr > 0 && p_original > 0, "allocate arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t cap = cfg->dp_row_cap > 0 ? cfg->dp_row_cap : 32768;     // P:L1145, Q8
  n = std::min(n, cap);
  std::vector<int64_t> Bs(ncr);
  int64_t Bmax = 0;
  for (int i = 0; i < ncr; ++i) {
    KVTC_CHECK_ARG(crs_host[i] > 0, "target_cr must be > 0");
    kvtc_dp_config c = *cfg;
    c.target_cr = crs_host[i];
    Bs[i] = budget_from(&c, p_original);
    Bmax = std::max(Bmax, Bs[i]);
  }
  DPRun run;
  std::vector<int32_t> sizes;
  kvtc_status s = dp_full(P, n, r, Bmax, cfg, st, run, sizes);
  for (int i = 0; i < ncr && s == KVTC_OK; ++i) s = backtrack_plan(run, r, Bs[i], sizes, st, &out[i]);
  dp_free(run);
  return s;
}

extern "C" kvtc_status kvtc_allocate_bits(const kvtc_basis *b, const kvtc_kv_view *seqs, int32_t nseq,
                                          const int64_t *samples_host, int64_t n, const kvtc_dp_config *cfg,
                                          void *stream, kvtc_plan **out) {
  KVTC_CHECK_ARG(cfg, "allocate arguments");
  return kvtc_allocate_bits_multi(b, seqs, nseq, samples_host, n, cfg, &cfg->target_cr, 1, stream, out);
}

extern "C" kvtc_status kvtc_allocate_bits_multi(const kvtc_basis *b, const kvtc_kv_view *seqs, int32_t nseq,
                                                const int64_t *samples_host, int64_t n, const kvtc_dp_config *cfg,
                                                const double *crs_host, int32_t ncr, void *stream, kvtc_plan **out) {
  KVTC_CHECK_ARG(b && seqs && nseq > 0 && samples_host && n > 0 && cfg && out && crs_host && ncr > 0,
                 "allocate arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t cap = cfg->dp_row_cap > 0 ? cfg->dp_row_cap : 32768;
  const int64_t nd = std::min(n, cap);                       // first rows in sample order (Q8)
  kvtc_status s;
  // gather the DP rows (keys un-RoPE'd) and project them: P = X V_c - mu V_c
  std::vector<void *> bases_h(size_t(nseq) * b->shape.layers);
  for (int i = 0; i < nseq; ++i)
    for (int l = 0; l < b->shape.layers; ++l) bases_h[size_t(i) * b->shape.layers + l] = seqs[i].layer_base_host[l];
  __nv_bfloat16 **bases = nullptr;
  __nv_bfloat16 *X = nullptr;
  int64_t *rows = nullptr;
  float *P = nullptr;
  KVTC_CUDA_TRY(cudaMalloc(&bases, bases_h.size() * sizeof(void *)));
  KVTC_CUDA_TRY(cudaMemcpy(bases, bases_h.data(), bases_h.size() * sizeof(void *), cudaMemcpyHostToDevice));
  KVTC_CUDA_TRY(cudaMalloc(&X, size_t(nd) * b->p * 2));
  KVTC_CUDA_TRY(cudaMalloc(&rows, size_t(nd) * 16));
  KVTC_CUDA_TRY(cudaMalloc(&P, size_t(nd) * b->r * 4));
  KVTC_CUDA_TRY(cudaMemcpy(rows, samples_host, size_t(nd) * 16, cudaMemcpyHostToDevice));
  s = launch_gather_rows(seqs, nseq, bases, rows, nd, b->d_invf, b->has_rope ? 1 : 0, b->pairing, b->p, X, st);
  if (s == KVTC_OK) s = kvtc_stage_project(b, nullptr, X, nd, P, stream);
  if (s == KVTC_OK) s = kvtc_allocate_bits_from_coeffs_multi(P, nd, b->r, b->p, cfg, crs_host, ncr, stream, out);
  cudaStreamSynchronize(st);
  cudaFree(bases);
  cudaFree(X);
  cudaFree(rows);
  cudaFree(P);
  return s;
}
