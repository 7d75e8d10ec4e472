// rans.cu — static-model interleaved rANS back-end of the lossless stage
// (the paper ablates ANS beside DEFLATE; reading
// Q24 of DESIGN.md §3 fixes the format, oracle/rans.py writes it out).
//
// The payload is tile-periodic (per 128-token tile the params,
// then each group's code block), so the byte statistics depend mostly on the
// offset inside the tile.  One order-0 table per CLASS (offset in tile >>
// span_log2, <= 64 classes), estimated on the whole payload and quantised to
// M = 2^12, costs ~16 KB per 100 MB section; chunks stay independent streams.
//
//   rans_hist_kernel    per-class byte counts (4 KiB blocks, smem histogram)
//   rans_norm_kernel    one block per class: quantise to M (the oracle's rule),
//                       encoder table (f | c << 16), decoder table per slot
//                       (sym | (f - 1) << 8 | (slot - c) << 20)
//   rans_encode_kernel  one warp per chunk, 32 interleaved states, steps from
//                       last to first, a step's renormalisation words placed by
//                       ballot + popc so the decoder reads them in order
//   rans_layout / copy  section header, tables, chunk table, streams
//   rans_decode_kernel  one warp per chunk, one table load per symbol, refills
//                       by ballot + popc; every read bounded by the section,
//                       final states must return to L (else corrupt)
#include <cub/block/block_scan.cuh>
#include <cstring>

#include "api_internal.h"

namespace kvtc {

namespace {
constexpr uint32_t kRansMagic = 0x4154564Bu;   // "KVTA"
constexpr uint32_t kRansVersion = 1;
constexpr int kScale = 12;
constexpr uint32_t kM = 1u << kScale;
constexpr uint32_t kL = 1u << 16;
constexpr int kLanes = 32;
constexpr int kWarpsPerCta = 4;
__host__ __device__ inline uint64_t umin64_(uint64_t a, uint64_t b) { return a < b ? a : b; }

struct RansHeader {
  uint32_t magic, version;
  uint64_t raw_bytes;
  uint32_t chunk_bytes, nchunks;
  uint64_t period;
  uint32_t span_log2, nclasses;
  uint64_t data_offset, section_bytes;
  uint64_t pad;
};
static_assert(sizeof(RansHeader) == 64, "rANS section header is 64 bytes");
struct RansChunk {
  uint64_t offset;   // from the data start, 16-byte aligned
  uint32_t bytes;    // stream bytes
  uint32_t kind;     // 0 rANS, 1 stored
};

struct Geometry {
  uint64_t n, period;
  uint32_t chunk, nchunks, sl, ncls;
  uint64_t tab_off, ctab_off, data_off;
};
__host__ __device__ inline int span_log2_of(uint64_t period) {
  const uint64_t t = (period + 63) / 64;
  const uint64_t target = t > 4096 ? t : 4096;
  int b = 12;
  while ((uint64_t(1) << b) < target) ++b;
  return b;
}
__host__ __device__ inline Geometry geometry(uint64_t n, int32_t chunk, int64_t tile_bytes) {
  Geometry g;
  g.n = n;
  const uint64_t n1 = n > 0 ? n : 1;
  g.period = tile_bytes > 0 ? (uint64_t(tile_bytes) < n1 ? uint64_t(tile_bytes) : n1) : n1;
  g.chunk = uint32_t(chunk);
  g.nchunks = uint32_t((n + chunk - 1) / chunk);
  g.sl = uint32_t(span_log2_of(g.period));
  g.ncls = uint32_t(((g.period - 1) >> g.sl) + 1);
  g.tab_off = sizeof(RansHeader);
  g.ctab_off = g.tab_off + ((uint64_t(g.ncls) * 256 * 2 + 15) & ~15ull);
  g.data_off = g.ctab_off + ((uint64_t(g.nchunks) * sizeof(RansChunk) + 15) & ~15ull);
  return g;
}
// per-chunk encoder slot: 32 states + up to one word per byte (+ padding)
__host__ __device__ inline uint64_t slot_words(uint32_t chunk) { return uint64_t(chunk) + 64; }
__host__ __device__ inline uint64_t slot_bytes(uint32_t chunk) { return ((4 * kLanes + 2 * slot_words(chunk)) + 15) & ~15ull; }

struct Work {               // carved from the caller's workspace
  uint32_t *counts;         // [ncls][256]
  uint32_t *enc;            // [ncls][256]  f | c << 16
  uint32_t *encr;           // [ncls][256]  ceil(2^32 / f)
  uint32_t *dec;            // [ncls][4096] decode entries
  uint16_t *freq;           // [ncls][256]  section copy
  uint8_t *slots;           // [nchunks][slot_bytes]
  uint32_t *clen, *ckind, *cwpos;   // per chunk: stream bytes, kind, first word index in the slot
};
Work carve(const Geometry &g, void *ws) {
  Bump b(ws, ~size_t(0));
  Work w;
  w.counts = b.take<uint32_t>(size_t(g.ncls) * 256);
  w.enc = b.take<uint32_t>(size_t(g.ncls) * 256);
  w.encr = b.take<uint32_t>(size_t(g.ncls) * 256);
  w.dec = b.take<uint32_t>(size_t(g.ncls) * kM);
  w.freq = b.take<uint16_t>(size_t(g.ncls) * 256);
  w.slots = b.take<uint8_t>(size_t(g.nchunks) * slot_bytes(g.chunk));
  w.clen = b.take<uint32_t>(g.nchunks + 1);
  w.ckind = b.take<uint32_t>(g.nchunks + 1);
  w.cwpos = b.take<uint32_t>(g.nchunks + 1);
  return w;
}
size_t work_bytes(const Geometry &g) {
  Bump b;
  b.take<uint32_t>(size_t(g.ncls) * 256);
  b.take<uint32_t>(size_t(g.ncls) * 256);
  b.take<uint32_t>(size_t(g.ncls) * 256);
  b.take<uint32_t>(size_t(g.ncls) * kM);
  b.take<uint16_t>(size_t(g.ncls) * 256);
  b.take<uint8_t>(size_t(g.nchunks) * slot_bytes(g.chunk));
  b.take<uint32_t>(g.nchunks + 1);
  b.take<uint32_t>(g.nchunks + 1);
  b.take<uint32_t>(g.nchunks + 1);
  return b.used + 256;
}

__device__ __forceinline__ uint32_t class_of(uint64_t i, uint64_t period, uint32_t sl) {
  return uint32_t((i % period) >> sl);
}

// ---------------------------------------------------------------- histograms
__global__ void __launch_bounds__(256) rans_hist_kernel(const uint8_t *in, uint64_t n, uint64_t period, uint32_t sl,
                                                        uint32_t *counts) {
  __shared__ uint32_t h[256];
  const uint64_t nblk = (n + 4095) / 4096;
  for (uint64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const uint64_t b0 = b * 4096, b1 = umin64_(n, b0 + 4096);
    const uint32_t c0 = class_of(b0, period, sl), c1 = class_of(b1 - 1, period, sl);
    const bool one = c0 == c1 && (b0 / period) == ((b1 - 1) / period);
    if (one) {
      h[threadIdx.x] = 0;
      __syncthreads();
      for (uint64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) atomicAdd(&h[in[i]], 1u);
      __syncthreads();
      if (h[threadIdx.x]) atomicAdd(&counts[size_t(c0) * 256 + threadIdx.x], h[threadIdx.x]);
      __syncthreads();
    } else {
      for (uint64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
        atomicAdd(&counts[size_t(class_of(i, period, sl)) * 256 + in[i]], 1u);
    }
  }
}

// ---------------------------------------------------------------- normalisation
// One block (256 threads) per class; the oracle's rule (oracle/rans.py normalize).
__global__ void __launch_bounds__(256) rans_norm_kernel(const uint32_t *counts, uint32_t *enc, uint32_t *encr,
                                                        uint32_t *dec, uint16_t *freq) {
  const int cls = blockIdx.x, s = threadIdx.x;
  __shared__ uint32_t f[256];
  __shared__ uint64_t tot;
  __shared__ uint32_t cum[257];
  const uint32_t h = counts[size_t(cls) * 256 + s];
  if (s == 0) tot = 0;
  __syncthreads();
  atomicAdd(reinterpret_cast<unsigned long long *>(&tot), (unsigned long long)h);
  __syncthreads();
  const uint64_t n = tot;
  const uint64_t q = n ? (uint64_t(h) * kM) / n : 0;
  f[s] = (n == 0 || h == 0) ? 0u : uint32_t(q > 0 ? q : 1);
  __syncthreads();
  if (s == 0 && n > 0) {
    int64_t sum = 0;
    for (int t = 0; t < 256; ++t) sum += f[t];
    int64_t d = int64_t(kM) - sum;
    if (d > 0) {
      int best = 0;
      uint32_t bh = counts[size_t(cls) * 256];
      for (int t = 1; t < 256; ++t) {
        const uint32_t v = counts[size_t(cls) * 256 + t];
        if (v > bh) {
          bh = v;
          best = t;
        }
      }
      f[best] += uint32_t(d);
    }
    while (d < 0) {
      int best = 0;
      for (int t = 1; t < 256; ++t)
        if (f[t] > f[best]) best = t;
      const int64_t take = -d < int64_t(f[best]) - 1 ? -d : int64_t(f[best]) - 1;
      f[best] -= uint32_t(take);
      d += take;
    }
    uint32_t c = 0;
    for (int t = 0; t < 256; ++t) {
      cum[t] = c;
      c += f[t];
    }
    cum[256] = c;
  }
  __syncthreads();
  freq[size_t(cls) * 256 + s] = uint16_t(f[s]);
  if (n == 0) return;
  enc[size_t(cls) * 256 + s] = f[s] | (cum[s] << 16);
  // ceil(2^32 / f): x / f = umulhi(x, rcp) or one less (f = 1: the quotient is x)
  encr[size_t(cls) * 256 + s] = f[s] > 1 ? uint32_t(((uint64_t(1) << 32) + f[s] - 1) / f[s]) : 0u;
  for (uint32_t k = 0; k < f[s]; ++k)
    dec[size_t(cls) * kM + cum[s] + k] = uint32_t(s) | ((f[s] - 1) << 8) | (k << 20);
}

// ---------------------------------------------------------------- encoder
__global__ void __launch_bounds__(kLanes * kWarpsPerCta) rans_encode_kernel(const uint8_t *in, Geometry g,
                                                                            const uint32_t *enc, const uint32_t *encr,
                                                                            uint8_t *slots, uint32_t *clen,
                                                                            uint32_t *ckind, uint32_t *cwpos) {
  constexpr int kBatch = 8;                       // steps whose table entries are loaded ahead
  const int lane = threadIdx.x % kLanes;
  const uint32_t c = blockIdx.x * kWarpsPerCta + threadIdx.x / kLanes;
  if (c >= g.nchunks) return;
  const uint64_t base = uint64_t(c) * g.chunk;
  const uint32_t nc = uint32_t(umin64_(g.chunk, g.n - base));
  const int steps = int((nc + kLanes - 1) / kLanes);
  uint8_t *slot = slots + uint64_t(c) * slot_bytes(g.chunk);
  uint16_t *words = reinterpret_cast<uint16_t *>(slot + 4 * kLanes);
  uint32_t wpos = uint32_t(slot_words(g.chunk));
  uint32_t x = kL;
  const uint32_t lt = (1u << lane) - 1;
  // offset of this lane's byte of the last step inside the period (decremented by 32 per step)
  int64_t off = int64_t((base + uint64_t(steps - 1) * kLanes + lane) % g.period);
  for (int k = steps - 1; k >= 0; k -= kBatch) {
    uint32_t e[kBatch], r[kBatch];
    int64_t o = off;
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {              // loads of kBatch steps in flight
      const int kk = k - u;
      const uint32_t j = uint32_t(kk) * kLanes + lane;
      e[u] = 1u;
      r[u] = 0u;
      if (kk >= 0 && j < nc) {
        const size_t t = size_t(uint32_t(o) >> g.sl) * 256 + in[base + j];
        e[u] = __ldg(enc + t);
        r[u] = __ldg(encr + t);
      }
      o -= kLanes;
      while (o < 0) o += int64_t(g.period);
    }
    off = o;
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int kk = k - u;
      if (kk < 0) break;
      const bool active = uint32_t(kk) * kLanes + lane < nc;
      const uint32_t f = e[u] & 0xFFFFu, cstart = e[u] >> 16;
      const bool emit = active && uint64_t(x) >= (uint64_t(f) << 20);   // f = M: never (2^32)
      const uint32_t bal = __ballot_sync(0xffffffffu, emit);
      const uint32_t cnt = __popc(bal);
      if (emit) {
        words[wpos - cnt + __popc(bal & lt)] = uint16_t(x & 0xFFFFu);
        x >>= 16;
      }
      wpos -= cnt;
      if (active) {
        uint32_t q = x;                             // f == 1
        if (f > 1) {
          q = __umulhi(x, r[u]);
          if (q * f > x) --q;
        }
        x = q * kM + (x - q * f) + cstart;          // (x / f) M + x mod f + c
      }
    }
  }
  reinterpret_cast<uint32_t *>(slot)[lane] = x;
  if (lane == 0) {
    const uint32_t bytes = 4 * kLanes + 2 * (uint32_t(slot_words(g.chunk)) - wpos);
    const bool stored = bytes >= nc;
    clen[c] = stored ? nc : bytes;
    ckind[c] = stored ? 1u : 0u;
    cwpos[c] = wpos;
  }
}

// ---------------------------------------------------------------- section assembly
__global__ void __launch_bounds__(1024) rans_layout_kernel(Geometry g, const uint32_t *clen, const uint32_t *ckind,
                                                           const uint16_t *freq, uint8_t *out_base,
                                                           const uint64_t *off_dev, uint64_t *section_len) {
  uint8_t *out = out_base + (off_dev ? *off_dev : 0);
  __shared__ typename cub::BlockScan<uint64_t, 1024>::TempStorage tmp;
  __shared__ uint64_t carry;
  RansChunk *tab = reinterpret_cast<RansChunk *>(out + g.ctab_off);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < g.nchunks; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const uint64_t sz = i < g.nchunks ? ((uint64_t(clen[i]) + 15) & ~15ull) : 0;
    uint64_t o, t;
    cub::BlockScan<uint64_t, 1024>(tmp).ExclusiveSum(sz, o, t);
    if (i < g.nchunks) tab[i] = RansChunk{carry + o, clen[i], ckind[i]};
    __syncthreads();
    if (threadIdx.x == 0) carry += t;
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < g.ncls * 256; i += blockDim.x)
    reinterpret_cast<uint16_t *>(out + g.tab_off)[i] = freq[i];
  if (threadIdx.x == 0) {
    RansHeader h{};
    h.magic = kRansMagic;
    h.version = kRansVersion;
    h.raw_bytes = g.n;
    h.chunk_bytes = g.chunk;
    h.nchunks = g.nchunks;
    h.period = g.period;
    h.span_log2 = g.sl;
    h.nclasses = g.ncls;
    h.data_offset = g.data_off;
    h.section_bytes = g.data_off + carry;
    *reinterpret_cast<RansHeader *>(out) = h;
    *section_len = h.section_bytes;
  }
}
__global__ void __launch_bounds__(256) rans_copy_kernel(Geometry g, const uint8_t *in, const uint8_t *slots,
                                                        const uint32_t *cwpos, uint8_t *out_base,
                                                        const uint64_t *off_dev) {
  uint8_t *out = out_base + (off_dev ? *off_dev : 0);
  const RansChunk *tab = reinterpret_cast<const RansChunk *>(out + g.ctab_off);
  for (uint32_t c = blockIdx.x; c < g.nchunks; c += gridDim.x) {
    const RansChunk e = tab[c];
    uint8_t *dst = out + g.data_off + e.offset;
    const uint32_t padded = (e.bytes + 15) & ~15u;
    if (e.kind == 1) {
      const uint8_t *src = in + uint64_t(c) * g.chunk;
      for (uint32_t i = threadIdx.x; i < padded; i += blockDim.x) dst[i] = i < e.bytes ? src[i] : 0;
    } else {
      // 16-bit units: the states (slot start) then the words (2-byte aligned in the slot)
      const uint16_t *slot = reinterpret_cast<const uint16_t *>(slots + uint64_t(c) * slot_bytes(g.chunk));
      const uint16_t *wsrc = slot + 2 * kLanes + cwpos[c];
      uint16_t *d16 = reinterpret_cast<uint16_t *>(dst);
      for (uint32_t i = threadIdx.x; i < padded / 2; i += blockDim.x)
        d16[i] = i < 2 * kLanes ? slot[i] : (2 * i < e.bytes ? wsrc[i - 2 * kLanes] : uint16_t(0));
    }
  }
}

// ---------------------------------------------------------------- decoder
__global__ void __launch_bounds__(kLanes * kWarpsPerCta) rans_decode_kernel(const uint8_t *sec, uint64_t sec_len,
                                                                            uint64_t n_out, const uint32_t *dec,
                                                                            uint8_t *out, int32_t *err) {
  const RansHeader h = *reinterpret_cast<const RansHeader *>(sec);
  const int lane = threadIdx.x % kLanes;
  const uint32_t c = blockIdx.x * kWarpsPerCta + threadIdx.x / kLanes;
  // the header must describe exactly the geometry of n_out bytes (else nothing is read)
  const Geometry g = geometry(n_out, int32_t(h.chunk_bytes ? h.chunk_bytes : 1), int64_t(h.period));
  if (h.magic != kRansMagic || h.version != kRansVersion || h.raw_bytes != n_out || h.chunk_bytes == 0 ||
      h.chunk_bytes > (1u << 20) || h.chunk_bytes % kLanes || h.nchunks != g.nchunks || h.period != g.period ||
      h.span_log2 != g.sl || h.nclasses != g.ncls || h.data_offset != g.data_off || h.section_bytes > sec_len ||
      h.section_bytes < h.data_offset) {
    if (c == 0 && lane == 0) atomicExch(err, -20);
    return;
  }
  if (c >= h.nchunks) return;
  const RansChunk *tab = reinterpret_cast<const RansChunk *>(sec + sizeof(RansHeader) +
                                                             ((uint64_t(h.nclasses) * 256 * 2 + 15) & ~15ull));
  const RansChunk e = tab[c];
  const uint64_t base = uint64_t(c) * h.chunk_bytes;
  const uint32_t nc = uint32_t(umin64_(h.chunk_bytes, n_out - base));
  if (e.kind > 1 || (e.offset & 15) || h.data_offset + e.offset + e.bytes > h.section_bytes ||
      (e.kind == 1 && e.bytes != nc) || (e.kind == 0 && (e.bytes < 4 * kLanes || (e.bytes & 1)))) {
    if (lane == 0) atomicExch(err, -21);
    return;
  }
  const uint8_t *stream = sec + h.data_offset + e.offset;
  if (e.kind == 1) {
    for (uint32_t i = lane; i < nc; i += kLanes) out[base + i] = stream[i];
    return;
  }
  uint32_t x = reinterpret_cast<const uint32_t *>(stream)[lane];
  const uint16_t *words = reinterpret_cast<const uint16_t *>(stream + 4 * kLanes);
  const uint32_t nwords = (e.bytes - 4 * kLanes) / 2;
  const uint32_t steps = (nc + kLanes - 1) / kLanes;
  const uint32_t lt = (1u << lane) - 1;
  uint32_t pos = 0;
  bool bad = false;
  uint64_t off = (base + lane) % h.period;
  // The next words live in registers, one per lane and block of 32 (win[b] = word
  // wbase + 32 b + lane): a refill is a shuffle, and the load of a block is issued
  // three window shifts before its words are read.  A step consumes <= 32 words, so
  // the words it reads are at window offsets < 64.
  auto wload = [&](uint32_t i) -> uint32_t { return i < nwords ? uint32_t(words[i]) : 0u; };
  uint32_t wbase = 0;
  uint32_t w0 = wload(lane), w1 = wload(32 + lane), w2 = wload(64 + lane), w3 = wload(96 + lane);
  for (uint32_t k = 0; k < steps; ++k) {
    const uint32_t j = k * kLanes + lane;
    const bool active = j < nc;
    if (active) {
      const uint32_t d = __ldg(dec + size_t(uint32_t(off >> h.span_log2)) * kM + (x & (kM - 1)));
      out[base + j] = uint8_t(d & 0xFF);
      x = (((d >> 8) & 0xFFFu) + 1) * (x >> kScale) + (d >> 20);
    }
    const bool need = active && x < kL;
    const uint32_t bal = __ballot_sync(0xffffffffu, need);
    const uint32_t rel = pos - wbase + __popc(bal & lt);          // < 64
    const uint32_t a = __shfl_sync(0xffffffffu, w0, rel & 31), b = __shfl_sync(0xffffffffu, w1, rel & 31);
    if (need) {
      if (pos + __popc(bal & lt) < nwords) x = (x << 16) | (rel < 32 ? a : b);
      else bad = true;
    }
    pos += __popc(bal);
    if (pos - wbase >= 32) {                                        // slide the window by one block
      w0 = w1;
      w1 = w2;
      w2 = w3;
      wbase += 32;
      w3 = wload(wbase + 96 + lane);
    }
    off += kLanes;
    while (off >= h.period) off -= h.period;
  }
  // every state must be back at L, every word consumed (else: corrupt stream)
  bad |= x != kL;
  if (__any_sync(0xffffffffu, bad) || pos != nwords) {
    if (lane == 0) atomicExch(err, -22);
  }
}

// Decoder tables from a section's frequency tables (one block per class).
__global__ void __launch_bounds__(256) rans_dec_tables_kernel(const uint8_t *sec, uint64_t sec_len, uint32_t *dec,
                                                              int32_t *err) {
  const RansHeader h = *reinterpret_cast<const RansHeader *>(sec);
  const int cls = blockIdx.x, s = threadIdx.x;
  if (uint32_t(cls) >= h.nclasses || h.nclasses > 64 || sizeof(RansHeader) + uint64_t(h.nclasses) * 512 > sec_len)
    return;                                        // a bad header is reported by the decoder
  const uint16_t *fr = reinterpret_cast<const uint16_t *>(sec + sizeof(RansHeader)) + size_t(cls) * 256;
  __shared__ uint32_t cum[257];
  const uint32_t f = fr[s];
  if (s == 0) {
    uint32_t c = 0;
    for (int t = 0; t < 256; ++t) {
      cum[t] = c;
      c += fr[t];
    }
    cum[256] = c;
  }
  __syncthreads();
  // a class is either empty or sums to M (else the section is corrupt); slots of an
  // empty class are never read by a valid stream, so they decode to symbol 0
  if (cum[256] != 0 && cum[256] != kM) {
    if (s == 0) atomicExch(err, -23);
    return;
  }
  if (cum[256] == 0) {
    for (uint32_t k = s; k < kM; k += 256) dec[size_t(cls) * kM + k] = 0;
    return;
  }
  for (uint32_t k = 0; k < f; ++k) dec[size_t(cls) * kM + cum[s] + k] = uint32_t(s) | ((f - 1) << 8) | (k << 20);
}
}  // namespace

// ================================================================== host side
size_t rans_section_bound(size_t n, int32_t chunk, int64_t tile_bytes) {
  const Geometry g = geometry(n, chunk, tile_bytes);
  return g.data_off + n + 16 * size_t(g.nchunks) + 16;
}
size_t rans_workspace(size_t n, int32_t chunk, int64_t tile_bytes) { return work_bytes(geometry(n, chunk, tile_bytes)); }

kvtc_status launch_rans_encode(const uint8_t *in, size_t n, int32_t chunk, int64_t tile_bytes, uint8_t *out,
                               const uint64_t *off_dev, uint64_t *section_len_dev, void *ws, size_t ws_bytes,
                               cudaStream_t st) {
  const Geometry g = geometry(n, chunk, tile_bytes);
  KVTC_CHECK_ARG(ws && ws_bytes >= work_bytes(g), "rANS workspace");
  Work w = carve(g, ws);
  KVTC_CUDA_TRY(cudaMemsetAsync(w.counts, 0, size_t(g.ncls) * 256 * 4, st));
  if (n) {
    rans_hist_kernel<<<unsigned(std::min<uint64_t>((n + 4095) / 4096, 4096)), 256, 0, st>>>(in, n, g.period, g.sl,
                                                                                           w.counts);
    KVTC_LAUNCH_CHECK();
  }
  rans_norm_kernel<<<g.ncls, 256, 0, st>>>(w.counts, w.enc, w.encr, w.dec, w.freq);
  KVTC_LAUNCH_CHECK();
  if (g.nchunks) {
    rans_encode_kernel<<<unsigned(ceil_div(g.nchunks, kWarpsPerCta)), kLanes * kWarpsPerCta, 0, st>>>(
        in, g, w.enc, w.encr, w.slots, w.clen, w.ckind, w.cwpos);
    KVTC_LAUNCH_CHECK();
  }
  rans_layout_kernel<<<1, 1024, 0, st>>>(g, w.clen, w.ckind, w.freq, out, off_dev, section_len_dev);
  KVTC_LAUNCH_CHECK();
  if (g.nchunks) {
    rans_copy_kernel<<<unsigned(std::min<uint32_t>(g.nchunks, 65535)), 256, 0, st>>>(g, in, w.slots, w.cwpos, out,
                                                                                    off_dev);
    KVTC_LAUNCH_CHECK();
  }
  return KVTC_OK;
}

// Host validation of a section header copy (len: bytes the section may occupy).
kvtc_status check_rans_header(const void *hdr_host, size_t len, size_t n_out, uint32_t *nchunks, uint32_t *nclasses) {
  RansHeader h;
  memcpy(&h, hdr_host, sizeof(h));
  const Geometry g = geometry(n_out, int32_t(h.chunk_bytes ? h.chunk_bytes : 1), int64_t(h.period));
  if (h.magic != kRansMagic || h.version != kRansVersion || h.raw_bytes != n_out || h.chunk_bytes == 0 ||
      h.chunk_bytes > (1u << 20) || h.nchunks != g.nchunks || h.span_log2 != g.sl || h.nclasses != g.ncls ||
      h.period != g.period || h.data_offset != g.data_off || h.section_bytes > len || h.section_bytes < h.data_offset) {
    set_error("corrupt rANS section header");
    return KVTC_E_CORRUPT;
  }
  *nchunks = h.nchunks;
  *nclasses = h.nclasses;
  return KVTC_OK;
}
size_t rans_decode_workspace(uint32_t nclasses) { return size_t(nclasses) * kM * 4 + 256; }

kvtc_status launch_rans_decode(const uint8_t *sec, uint64_t len, uint64_t n_out, uint32_t nchunks, uint32_t nclasses,
                               uint8_t *out, void *ws, int32_t *err, cudaStream_t st) {
  uint32_t *dec = static_cast<uint32_t *>(ws);
  rans_dec_tables_kernel<<<nclasses, 256, 0, st>>>(sec, len, dec, err);
  KVTC_LAUNCH_CHECK();
  if (nchunks) {
    rans_decode_kernel<<<unsigned(ceil_div(nchunks, kWarpsPerCta)), kLanes * kWarpsPerCta, 0, st>>>(sec, len, n_out,
                                                                                                  dec, out, err);
    KVTC_LAUNCH_CHECK();
  }
  return KVTC_OK;
}

}  // namespace kvtc
