// integrity.cu — container checksums (the KVTC_E_CORRUPT contract).
//
// The paper's codec is lossless after quantisation ("This step is lossless",
// P:L263), so a decompressed cache must be either exactly what was compressed or
// an error.  DEFLATE without a checksum cannot promise that (a flipped bit inside
// a Huffman code can decode into another symbol of the same length), so the
// container carries three 64-bit checksums: one per stream payload
// (before DEFLATE; verified after inflate), one over the raw sink / window
// section, one over the header itself.
//
// Checksum of n bytes (little-endian 8-byte words w_i, the last one zero-padded):
//   H = mix(n ^ seed) + sum_i mix(w_i ^ (seed + (i + 1) * 0x9E3779B97F4A7C15))  (mod 2^64)
// mix = the SplitMix64 finaliser, a bijection on 64-bit words, so changing any
// single word changes exactly one term and therefore H, with certainty; several
// changed words collide with probability ~2^-64.  The sum is order-independent:
// thread blocks add their partial sums with atomics and the result is
// deterministic.
#include <cstring>

#include "internal.h"

namespace kvtc {

uint64_t host_hash(const void *data, size_t n, uint64_t seed) {
  const uint8_t *p = static_cast<const uint8_t *>(data);
  uint64_t h = mix64(uint64_t(n) ^ seed);
  const size_t nw = n / 8;
  for (size_t i = 0; i < nw; ++i) {
    uint64_t w;
    memcpy(&w, p + 8 * i, 8);
    h += hash_term(w, i, seed);
  }
  if (n % 8) {
    uint64_t w = 0;
    memcpy(&w, p + 8 * nw, n % 8);
    h += hash_term(w, nw, seed);
  }
  return h;
}

// Grid-stride (over blockIdx.x / gridDim.x) through 16-byte vectors of p (16-byte
// aligned); block 0 adds the length term and the ragged tail.
__device__ __forceinline__ void hash_range(const uint8_t *p, uint64_t n, uint64_t seed, unsigned long long *out) {
  const uint64_t nv = n / 16;
  const uint4 *v = reinterpret_cast<const uint4 *>(p);
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nv; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 q = __ldcs(v + i);
    acc += hash_term(uint64_t(q.x) | (uint64_t(q.y) << 32), 2 * i, seed);
    acc += hash_term(uint64_t(q.z) | (uint64_t(q.w) << 32), 2 * i + 1, seed);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    acc += mix64(n ^ seed);
    for (uint64_t b = nv * 16; b < n; b += 8) {
      uint64_t w = 0;
      for (uint64_t k = 0; k < 8 && b + k < n; ++k) w |= uint64_t(p[b + k]) << (8 * k);
      acc += hash_term(w, b / 8, seed);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ uint64_t part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < int(blockDim.x / 32); ++w) t += part[w];
    atomicAdd(out, static_cast<unsigned long long>(t));
  }
}

__global__ void __launch_bounds__(256) hash_kernel(const uint8_t *p, uint64_t n, uint64_t seed,
                                                   unsigned long long *out) {
  hash_range(p, n, seed, out);
}
__global__ void __launch_bounds__(256) hash_batch_kernel(const HashJob *jobs) {
  const HashJob j = jobs[blockIdx.y];
  hash_range(j.p, j.n, j.seed, reinterpret_cast<unsigned long long *>(j.out));
}
__global__ void hash_check_batch_kernel(const uint64_t *got, const uint64_t *expect, int32_t njobs, int32_t per,
                                        int32_t *status) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < njobs; j += gridDim.x * blockDim.x)
    if (got[j] != expect[j]) atomicOr(status + j / per, 1 << (j % per));
}

__global__ void hash_check_kernel(const uint64_t *got, uint64_t expect, int32_t bit, int32_t *status) {
  if (*got != expect) atomicOr(status, bit);
}

kvtc_status launch_hash(const void *p, uint64_t n, uint64_t seed, uint64_t *out, cudaStream_t st, int32_t max_ctas) {
  if (reinterpret_cast<uintptr_t>(p) & 15) {
    set_error("checksum input must be 16-byte aligned");
    return KVTC_E_INVALID;
  }
  const int64_t want = std::max<int64_t>(1, ceil_div(int64_t(n / 16), 256 * 4));
  const int64_t cap = max_ctas > 0 ? max_ctas : corun_ctas(8);
  KVTC_MAX_CARVEOUT(hash_kernel);               // may run beside a GEMM on the side stream
  hash_kernel<<<unsigned(std::min(want, cap)), 256, 0, st>>>(static_cast<const uint8_t *>(p), n, seed,
                                                             reinterpret_cast<unsigned long long *>(out));
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_hash_batch(const HashJob *jobs_dev, int32_t njobs, uint64_t max_n, cudaStream_t st,
                              int32_t max_ctas) {
  if (njobs <= 0) return KVTC_OK;
  const int64_t cap = std::max<int64_t>(1, (max_ctas > 0 ? max_ctas : corun_ctas(8)) / njobs);
  const int64_t want = std::max<int64_t>(1, ceil_div(int64_t(max_n / 16), 256 * 4));
  KVTC_MAX_CARVEOUT(hash_batch_kernel);
  hash_batch_kernel<<<dim3(unsigned(std::min(want, cap)), unsigned(njobs)), 256, 0, st>>>(jobs_dev);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_hash_check_batch(const uint64_t *got, const uint64_t *expect, int32_t njobs, int32_t per,
                                   int32_t *status, cudaStream_t st) {
  if (njobs <= 0) return KVTC_OK;
  hash_check_batch_kernel<<<unsigned(ceil_div(njobs, 256)), 256, 0, st>>>(got, expect, njobs, per, status);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_hash_check(const uint64_t *got, uint64_t expect, int32_t bit, int32_t *status, cudaStream_t st) {
  hash_check_kernel<<<1, 1, 0, st>>>(got, expect, bit, status);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

}  // namespace kvtc
