// calib.cu — calibration (K6) of P:L222-229.
//
//   accumulate: rows (seq, token) gathered from the caches (keys un-RoPE'd, R1)
//               in chunks of kCalibChunk rows -> column sums in fp64 and
//               S += C_chunk^T C_chunk on the tcgen05 GEMM (EPI_XTX; bf16 x bf16
//               products are exact, accumulation fp32; only tiles on or above
//               the diagonal are computed).  These sums are what a multi-GPU
//               caller all-reduces (NCCL) before finalising.
//   finalize:   Sigma = S - n mu mu^T (full symmetric), top-r eigenpairs,
//               descending order, canonical sign (Q13), r = min(cap, n-1, p)
//               (Q12) -> kvtc_basis_create.  p <= 8192: exact fp64 syevdx.
//               Larger p: the paper's randomized SVD (Halko et al.; 8
//               power iterations) as subspace iteration on Sigma with
//               Householder re-orthonormalisation and a Rayleigh-Ritz step
//               (fp64 syevd of the small projected matrix).  cuBLAS / cuSOLVER
//               are calibration-time library steps (DESIGN.md §6 K6).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdlib>

#include "api_internal.h"

using namespace kvtc;

namespace {

constexpr int64_t kCalibChunk = 8192;

__global__ void transpose_bf16_kernel(const __nv_bfloat16 *X, int64_t rows, int64_t cols, __nv_bfloat16 *T) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int64_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? X[r * cols + c] : __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < rows) T[c * rows + r] = tile[threadIdx.x][k];
  }
}

__global__ void colsum_kernel(const __nv_bfloat16 *X, int64_t rows, int64_t cols, double *sum) {
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int64_t r = 0; r < rows; ++r) s += double(__bfloat162float(X[r * cols + c]));
  sum[c] += s;
}

// Sigma (fp64, full) from the accumulated upper-triangle S: Sigma_ij = S_min,max - n mu_i mu_j
__global__ void centre_kernel(const float *S, const double *sum, int64_t n, int64_t p, double *A) {
  const int64_t i = blockIdx.y, j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= p) return;
  const int64_t a = i < j ? i : j, b = i < j ? j : i;
  const double mi = sum[i] / double(n), mj = sum[j] / double(n);
  A[i * p + j] = double(S[a * p + b]) - double(n) * mi * mj;
}
__global__ void centre_kernel_f32(const float *S, const double *sum, int64_t n, int64_t p, float *A) {
  const int64_t i = blockIdx.y, j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= p) return;
  const int64_t a = i < j ? i : j, b = i < j ? j : i;
  const double mi = sum[i] / double(n), mj = sum[j] / double(n);
  A[i * p + j] = float(double(S[a * p + b]) - double(n) * mi * mj);
}

__global__ void gaussian_kernel(float *x, int64_t n, uint64_t seed) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  // counter-based: two splitmix64 draws -> Box-Muller
  auto mix = [](uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const uint64_t a = mix(seed ^ (uint64_t(i) * 2)), b = mix(seed ^ (uint64_t(i) * 2 + 1));
  const double u1 = (double(a >> 11) + 1.0) * (1.0 / 9007199254740992.0);
  const double u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
  x[i] = float(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}
__global__ void f32_to_f64_kernel(const float *a, double *b, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) b[i] = a[i];
}
__global__ void f64_to_f32_kernel(const double *a, float *b, int64_t n) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i < n) b[i] = float(a[i]);
}

// Randomized top-r eigenpairs of the symmetric p x p matrix A (fp32, device).
// Outputs (host): w[r] descending, V column-major p x r (fp64).
kvtc_status randomized_eig(float *A, int64_t p, int64_t r, int iters, cudaStream_t st, std::vector<double> &w,
                           std::vector<double> &V) {
  const int64_t k = std::min<int64_t>(p, r + 64);
  float *Y = nullptr, *Z = nullptr, *tau = nullptr, *Bk = nullptr, *U32 = nullptr, *Vd = nullptr;
  double *B64 = nullptr, *W64 = nullptr;
  int *info = nullptr;
  void *work = nullptr;
  cublasHandle_t cb = nullptr;
  cusolverDnHandle_t cs = nullptr;
  auto cleanup = [&]() {
    cudaFree(Y); cudaFree(Z); cudaFree(tau); cudaFree(Bk); cudaFree(U32); cudaFree(Vd);
    cudaFree(B64); cudaFree(W64); cudaFree(info); cudaFree(work);
    if (cb) cublasDestroy(cb);
    if (cs) cusolverDnDestroy(cs);
  };
#define R_TRY(x)                                           \
  do {                                                     \
    if (!(x)) {                                            \
      cleanup();                                           \
      set_error("randomized eig: %s failed", #x);          \
      return KVTC_E_CUDA;                                  \
    }                                                      \
  } while (0)
  R_TRY(cudaMalloc(&Y, size_t(p) * k * 4) == cudaSuccess);
  R_TRY(cudaMalloc(&Z, size_t(p) * k * 4) == cudaSuccess);
  R_TRY(cudaMalloc(&tau, size_t(k) * 4) == cudaSuccess);
  R_TRY(cudaMalloc(&Bk, size_t(k) * k * 4) == cudaSuccess);
  R_TRY(cudaMalloc(&B64, size_t(k) * k * 8) == cudaSuccess);
  R_TRY(cudaMalloc(&W64, size_t(k) * 8) == cudaSuccess);
  R_TRY(cudaMalloc(&info, 4) == cudaSuccess);
  R_TRY(cublasCreate(&cb) == CUBLAS_STATUS_SUCCESS);
  R_TRY(cublasSetStream(cb, st) == CUBLAS_STATUS_SUCCESS);
  R_TRY(cublasSetMathMode(cb, CUBLAS_PEDANTIC_MATH) == CUBLAS_STATUS_SUCCESS);
  R_TRY(cusolverDnCreate(&cs) == CUSOLVER_STATUS_SUCCESS);
  R_TRY(cusolverDnSetStream(cs, st) == CUSOLVER_STATUS_SUCCESS);
  int lw_qr = 0, lw_og = 0, lw_ev = 0;
  R_TRY(cusolverDnSgeqrf_bufferSize(cs, int(p), int(k), Y, int(p), &lw_qr) == CUSOLVER_STATUS_SUCCESS);
  R_TRY(cusolverDnSorgqr_bufferSize(cs, int(p), int(k), int(k), Y, int(p), tau, &lw_og) == CUSOLVER_STATUS_SUCCESS);
  R_TRY(cusolverDnDsyevd_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(k), B64, int(k), W64,
                                    &lw_ev) == CUSOLVER_STATUS_SUCCESS);
  const size_t wbytes = std::max<size_t>(size_t(std::max(lw_qr, lw_og)) * 4, size_t(lw_ev) * 8);
  R_TRY(cudaMalloc(&work, wbytes) == cudaSuccess);
  const float one = 1.f, zero = 0.f;
  gaussian_kernel<<<unsigned(ceil_div(p * k, 256)), 256, 0, st>>>(Z, p * k, 0x4B56544352534544ull);
  // Y = A * Omega
  R_TRY(cublasSgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, int(p), int(k), int(p), &one, A, int(p), Z, int(p), &zero, Y,
                    int(p)) == CUBLAS_STATUS_SUCCESS);
  auto orth = [&](float *M) {
    if (cusolverDnSgeqrf(cs, int(p), int(k), M, int(p), tau, static_cast<float *>(work), std::max(lw_qr, lw_og),
                         info) != CUSOLVER_STATUS_SUCCESS)
      return false;
    return cusolverDnSorgqr(cs, int(p), int(k), int(k), M, int(p), tau, static_cast<float *>(work),
                            std::max(lw_qr, lw_og), info) == CUSOLVER_STATUS_SUCCESS;
  };
  for (int it = 0; it < iters; ++it) {
    R_TRY(orth(Y));
    R_TRY(cublasSgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, int(p), int(k), int(p), &one, A, int(p), Y, int(p), &zero, Z,
                      int(p)) == CUBLAS_STATUS_SUCCESS);
    std::swap(Y, Z);
  }
  R_TRY(orth(Y));                                                   // Q
  R_TRY(cublasSgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, int(p), int(k), int(p), &one, A, int(p), Y, int(p), &zero, Z,
                    int(p)) == CUBLAS_STATUS_SUCCESS);              // A Q
  R_TRY(cublasSgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, int(k), int(k), int(p), &one, Y, int(p), Z, int(p), &zero, Bk,
                    int(k)) == CUBLAS_STATUS_SUCCESS);              // Q^T A Q
  f32_to_f64_kernel<<<unsigned(ceil_div(k * k, 256)), 256, 0, st>>>(Bk, B64, k * k);
  R_TRY(cusolverDnDsyevd(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(k), B64, int(k), W64,
                         static_cast<double *>(work), lw_ev, info) == CUSOLVER_STATUS_SUCCESS);
  // top r Ritz vectors: columns k-r .. k-1 of the eigenvector matrix (ascending)
  R_TRY(cudaMalloc(&U32, size_t(k) * r * 4) == cudaSuccess);
  f64_to_f32_kernel<<<unsigned(ceil_div(k * r, 256)), 256, 0, st>>>(B64 + size_t(k) * (k - r), U32, k * r);
  R_TRY(cudaMalloc(&Vd, size_t(p) * r * 4) == cudaSuccess);
  R_TRY(cublasSgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, int(p), int(r), int(k), &one, Y, int(p), U32, int(k), &zero, Vd,
                    int(p)) == CUBLAS_STATUS_SUCCESS);
  std::vector<double> wk(k);
  std::vector<float> vf(size_t(p) * r);
  int hinfo = 0;
  R_TRY(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, st) == cudaSuccess);
  R_TRY(cudaMemcpyAsync(wk.data(), W64, k * 8, cudaMemcpyDeviceToHost, st) == cudaSuccess);
  R_TRY(cudaMemcpyAsync(vf.data(), Vd, size_t(p) * r * 4, cudaMemcpyDeviceToHost, st) == cudaSuccess);
  R_TRY(cudaStreamSynchronize(st) == cudaSuccess);
  cleanup();
#undef R_TRY
  if (hinfo != 0) {
    set_error("randomized eig: syevd info %d", hinfo);
    return KVTC_E_NUMERIC;
  }
  // ascending -> the caller's convention (ascending, column-major): keep as is
  w.assign(wk.begin() + (k - r), wk.end());
  V.resize(vf.size());
  for (size_t i = 0; i < vf.size(); ++i) V[i] = vf[i];
  return KVTC_OK;
}

}  // namespace

extern "C" size_t kvtc_calibrate_workspace_bytes(const kvtc_shape *shape) {
  if (!shape) return 0;
  const int64_t p = int64_t(shape->layers) * shape->kv_heads * shape->head_dim;
  Bump b;
  b.take<__nv_bfloat16>(kCalibChunk * p);
  b.take<__nv_bfloat16>(kCalibChunk * p);
  b.take<int64_t>(2 * kCalibChunk);
  b.take<float>(shape->head_dim / 2);
  return b.used + 256;
}

extern "C" kvtc_status kvtc_calibrate_accumulate(const kvtc_kv_view *seqs, int32_t nseq, const int64_t *samples_host,
                                                 int64_t n, kvtc_stream which, const kvtc_rope *rope, double *sum_x,
                                                 float *xtx, void *workspace, size_t workspace_bytes, void *stream) {
  KVTC_CHECK_ARG(seqs && nseq > 0 && samples_host && n >= 0 && sum_x && xtx && workspace, "calibrate arguments");
  KVTC_CHECK_ARG(which == KVTC_VALUES || (rope && rope->inv_freq_host), "keys need rope");
  kvtc_status s;
  for (int i = 0; i < nseq; ++i) {
    if ((s = check_view(&seqs[i]))) return s;
    KVTC_CHECK_ARG(seqs[i].shape.layers == seqs[0].shape.layers && seqs[i].shape.kv_heads == seqs[0].shape.kv_heads &&
                       seqs[i].shape.head_dim == seqs[0].shape.head_dim,
                   "calibration sequences must share the shape");
  }
  for (int64_t r = 0; r < n; ++r)
    KVTC_CHECK_ARG(samples_host[2 * r] >= 0 && samples_host[2 * r] < nseq && samples_host[2 * r + 1] >= 0 &&
                       samples_host[2 * r + 1] < seqs[samples_host[2 * r]].tokens,
                   "sample out of range");
  const kvtc_shape &sh = seqs[0].shape;
  KVTC_CHECK_ARG(workspace_bytes >= kvtc_calibrate_workspace_bytes(&sh), "calibrate workspace");
  const int64_t p = int64_t(sh.layers) * sh.kv_heads * sh.head_dim;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Bump ws(workspace, workspace_bytes);
  auto *Xc = ws.take<__nv_bfloat16>(kCalibChunk * p);
  auto *Ct = ws.take<__nv_bfloat16>(kCalibChunk * p);
  auto *rows = ws.take<int64_t>(2 * kCalibChunk);
  float *invf = ws.take<float>(sh.head_dim / 2);
  // device array of layer bases for every sequence
  std::vector<void *> bases_h(size_t(nseq) * sh.layers);
  for (int i = 0; i < nseq; ++i)
    for (int l = 0; l < sh.layers; ++l) bases_h[size_t(i) * sh.layers + l] = seqs[i].layer_base_host[l];
  __nv_bfloat16 **bases = nullptr;
  KVTC_CUDA_TRY(cudaMallocAsync(&bases, bases_h.size() * sizeof(void *), st));
  KVTC_CUDA_TRY(cudaMemcpyAsync(bases, bases_h.data(), bases_h.size() * sizeof(void *), cudaMemcpyHostToDevice, st));
  const int unrope = which == KVTC_KEYS;
  if (unrope) KVTC_CUDA_TRY(cudaMemcpyAsync(invf, rope->inv_freq_host, sh.head_dim / 2 * 4, cudaMemcpyHostToDevice, st));
  for (int64_t r0 = 0; r0 < n; r0 += kCalibChunk) {
    const int64_t nk = std::min(kCalibChunk, n - r0);
    KVTC_CUDA_TRY(cudaMemcpyAsync(rows, samples_host + 2 * r0, nk * 16, cudaMemcpyHostToDevice, st));
    if ((s = launch_gather_rows(seqs, nseq, bases, rows, nk, invf, unrope, unrope ? rope->pairing : 0, p, Xc, st)))
      return s;
    colsum_kernel<<<unsigned(ceil_div(p, 256)), 256, 0, st>>>(Xc, nk, p, sum_x);
    // Ct [p x nk_pad]: rows padded to a multiple of 8 (16-byte TMA pitch), zeros past nk
    const int64_t nk_pad = (nk + 63) / 64 * 64;
    if (nk_pad != nk) KVTC_CUDA_TRY(cudaMemsetAsync(Xc + nk * p, 0, (nk_pad - nk) * p * 2, st));
    transpose_bf16_kernel<<<dim3(unsigned(ceil_div(p, 32)), unsigned(ceil_div(nk_pad, 32))), dim3(32, 8), 0, st>>>(
        Xc, nk_pad, p, Ct);
    KVTC_LAUNCH_CHECK();
    CUtensorMap tA, tB;
    if ((s = make_tmap_2d(&tA, Ct, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, nk_pad, p, nk_pad * 2, kBlockK, kTileM))) return s;
    if ((s = make_tmap_2d(&tB, Ct, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, nk_pad, p, nk_pad * 2, kBlockK, kMaxTileN / 2)))
      return s;
    if ((s = launch_gemm_xtx(&tA, &tB, int32_t(p), int32_t(nk_pad), xtx, st))) return s;
  }
  cudaFreeAsync(bases, st);
  return KVTC_OK;
}

extern "C" kvtc_status kvtc_calibrate_finalize(const kvtc_shape *shape, kvtc_stream which, const kvtc_rope *rope,
                                               const double *sum_x, const float *xtx, int64_t n, int32_t rank_cap,
                                               void *stream, kvtc_basis **out) {
  KVTC_CHECK_ARG(shape && sum_x && xtx && out && n >= 2 && rank_cap >= 1, "finalize arguments");
  const int64_t p = int64_t(shape->layers) * shape->kv_heads * shape->head_dim;
  const int64_t r = std::min<int64_t>(std::min<int64_t>(rank_cap, n - 1), p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // fp64 exact eigensolver where it is cheap; randomized SVD above (KVTC_CALIB_RSVD=1 forces it, for tests)
  const bool f64 = p <= 8192 && !getenv("KVTC_CALIB_RSVD");
  const size_t esz = f64 ? 8 : 4;
  void *A = nullptr, *W = nullptr;
  int *info = nullptr;
  KVTC_CUDA_TRY(cudaMalloc(&A, size_t(p) * p * esz));
  KVTC_CUDA_TRY(cudaMalloc(&W, size_t(p) * esz));
  KVTC_CUDA_TRY(cudaMalloc(&info, sizeof(int)));
  dim3 grid(unsigned(ceil_div(p, 256)), unsigned(p));
  if (f64) centre_kernel<<<grid, 256, 0, st>>>(xtx, sum_x, n, p, static_cast<double *>(A));
  else centre_kernel_f32<<<grid, 256, 0, st>>>(xtx, sum_x, n, p, static_cast<float *>(A));
  KVTC_LAUNCH_CHECK();
  std::vector<double> w(r), evec(size_t(p) * r), sumh(p);
  KVTC_CUDA_TRY(cudaMemcpy(sumh.data(), sum_x, p * 8, cudaMemcpyDeviceToHost));
  if (!f64) {
    // randomized SVD: 8 power iterations
    kvtc_status rs = randomized_eig(static_cast<float *>(A), p, r, 8, st, w, evec);
    cudaFree(A);
    cudaFree(W);
    cudaFree(info);
    if (rs) return rs;
  } else {
    cusolverDnHandle_t h = nullptr;
    cusolverDnParams_t prm = nullptr;
    auto cleanup = [&]() {
      if (prm) cusolverDnDestroyParams(prm);
      if (h) cusolverDnDestroy(h);
      cudaFree(A);
      cudaFree(W);
      cudaFree(info);
    };
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS || cusolverDnSetStream(h, st) != CUSOLVER_STATUS_SUCCESS ||
        cusolverDnCreateParams(&prm) != CUSOLVER_STATUS_SUCCESS) {
      cleanup();
      set_error("cusolver init failed");
      return KVTC_E_CUDA;
    }
    const cudaDataType dt = f64 ? CUDA_R_64F : CUDA_R_32F;
    int64_t meig = 0;
    size_t wd = 0, wh = 0;
    double vl = 0, vu = 0;
    float vlf = 0, vuf = 0;
    void *pvl = f64 ? static_cast<void *>(&vl) : static_cast<void *>(&vlf);
    void *pvu = f64 ? static_cast<void *>(&vu) : static_cast<void *>(&vuf);
    const int64_t il = p - r + 1, iu = p;
    cusolverStatus_t cs = cusolverDnXsyevdx_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                                       CUBLAS_FILL_MODE_LOWER, p, dt, A, p, pvl, pvu, il, iu, &meig, dt,
                                                       W, dt, &wd, &wh);
    if (cs != CUSOLVER_STATUS_SUCCESS) {
      cleanup();
      set_error("syevdx bufferSize failed (%d)", int(cs));
      return KVTC_E_CUDA;
    }
    void *dwork = nullptr;
    std::vector<uint8_t> hwork(std::max<size_t>(wh, 1));
    if (cudaMalloc(&dwork, std::max<size_t>(wd, 1)) != cudaSuccess) {
      cleanup();
      set_error("syevdx workspace (%zu bytes)", wd);
      return KVTC_E_NOMEM;
    }
    cs = cusolverDnXsyevdx(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, p, dt, A, p,
                           pvl, pvu, il, iu, &meig, dt, W, dt, dwork, wd, hwork.data(), wh, info);
    int hinfo = 0;
    cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(dwork);
    if (cs != CUSOLVER_STATUS_SUCCESS || hinfo != 0 || meig != r) {
      cleanup();
      set_error("syevdx failed (status %d, info %d, meig %lld)", int(cs), hinfo, (long long)meig);
      return KVTC_E_NUMERIC;
    }
    if (f64) {
      KVTC_CUDA_TRY(cudaMemcpy(w.data(), W, r * 8, cudaMemcpyDeviceToHost));
      KVTC_CUDA_TRY(cudaMemcpy(evec.data(), A, size_t(p) * r * 8, cudaMemcpyDeviceToHost));
    } else {
      std::vector<float> wf(r), ef(size_t(p) * r);
      KVTC_CUDA_TRY(cudaMemcpy(wf.data(), W, r * 4, cudaMemcpyDeviceToHost));
      KVTC_CUDA_TRY(cudaMemcpy(ef.data(), A, size_t(p) * r * 4, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < r; ++i) w[i] = wf[i];
      for (size_t i = 0; i < ef.size(); ++i) evec[i] = ef[i];
    }
    cleanup();

  }
  std::vector<float> Vh(size_t(p) * r), muh(p), sg(r);
  for (int64_t f = 0; f < p; ++f) muh[f] = float(sumh[f] / double(n));
  for (int64_t j = 0; j < r; ++j) {
    const int64_t src = r - 1 - j;                     // descending order
    const double *v = evec.data() + size_t(src) * p;
    int64_t arg = 0;
    for (int64_t f = 1; f < p; ++f)
      if (std::fabs(v[f]) > std::fabs(v[arg])) arg = f;
    const double sgn = v[arg] < 0 ? -1.0 : 1.0;       // canonical sign (Q13)
    for (int64_t f = 0; f < p; ++f) Vh[size_t(f) * r + j] = float(sgn * v[f]);
    sg[j] = float(std::sqrt(std::max(w[src], 0.0)));
  }
  return kvtc_basis_create(shape, which, rope, int32_t(r), muh.data(), Vh.data(), sg.data(), out);
}

extern "C" kvtc_status kvtc_calibrate(const kvtc_kv_view *seqs, int32_t nseq, const int64_t *samples_host, int64_t n,
                                      kvtc_stream which, const kvtc_rope *rope, int32_t rank_cap, void *stream,
                                      kvtc_basis **out) {
  KVTC_CHECK_ARG(seqs && nseq > 0, "calibrate arguments");
  const kvtc_shape sh = seqs[0].shape;
  const int64_t p = int64_t(sh.layers) * sh.kv_heads * sh.head_dim;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *sum = nullptr;
  float *xtx = nullptr;
  void *ws = nullptr;
  const size_t wsb = kvtc_calibrate_workspace_bytes(&sh);
  KVTC_CUDA_TRY(cudaMalloc(&sum, p * 8));
  KVTC_CUDA_TRY(cudaMalloc(&xtx, size_t(p) * p * 4));
  KVTC_CUDA_TRY(cudaMalloc(&ws, wsb));
  KVTC_CUDA_TRY(cudaMemsetAsync(sum, 0, p * 8, st));
  KVTC_CUDA_TRY(cudaMemsetAsync(xtx, 0, size_t(p) * p * 4, st));
  kvtc_status s = kvtc_calibrate_accumulate(seqs, nseq, samples_host, n, which, rope, sum, xtx, ws, wsb, stream);
  if (s == KVTC_OK) s = kvtc_calibrate_finalize(&sh, which, rope, sum, xtx, n, rank_cap, stream, out);
  cudaStreamSynchronize(st);
  cudaFree(sum);
  cudaFree(xtx);
  cudaFree(ws);
  return s;
}
