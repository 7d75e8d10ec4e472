// deflate.cu — chunk-parallel DEFLATE (RFC 1951) encoder and decoders (K3/K4).
//
// Paper: the packed byte array is "further compressed using the DEFLATE
// algorithm" and runs on the GPU.  Reading Q15: 64 KiB chunks, each
// an independent raw DEFLATE stream that stock zlib inflates (wbits = -15).
//
// Encoder (one CTA of 128 threads per chunk, ~14 chunks resident per SM so the
// serial code construction of one chunk overlaps the parallel passes of the
// others): byte histogram (warp-private bins) -> symbols radix-sorted by
// (frequency, symbol) -> length-limited canonical Huffman code (<= 15 bits;
// in-place minimum-redundancy lengths + Kraft-sum repair) -> one dynamic block
// (literals + EOB only, no LZ77 matches in this version) -> thread j emits the
// bits of 1/128 of the chunk, two codes per accumulator step, at an offset from
// a block-wide exclusive scan.  Falls back to stored blocks when smaller.  The bit length of
// every segment goes to a u16 side index that lives in the section, NOT in the
// DEFLATE stream.
//
// Decoder, fast path (64 threads per chunk): thread 0 parses the block header
// (table-driven code-length decode), the block builds a two-level table (11-bit
// first level + 4-bit subtables for longer codes) in shared memory, then thread
// j decodes segment j from the prefix sum of the index — 64 independent serial
// decoders with 16-byte reads, two blocks of read-ahead and 16-byte stores.
// Decoder, generic path (kvtc_stage_inflate_raw): a complete sequential inflater
// (stored / fixed / dynamic blocks, LZ77 back-references) for foreign streams.
//
// Section layout: 64-byte header, chunk table [nchunks] x
// {u64 offset, u32 bytes, u32 kind}, segment index [nchunks][64] u16 (bit
// length of each 1/64 of the chunk's symbols; segment 0 starts right after the
// block header), then the chunk streams, each starting 16-byte aligned and zero-padded to
// a multiple of 16 bytes (the inflater reads 16-byte words).
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "internal.h"
#include "dequant.cuh"

namespace kvtc {

constexpr uint32_t kSectionMagic = 0x4454564Bu;  // "KVTD"
constexpr int kEncThreads = 128;  // two threads per index segment; ~14 chunks resident per SM
constexpr int kNSeg = 64;
constexpr uint32_t kSectionVersion = 3;
constexpr int kLitSyms = 257;                    // 0..255 literals + 256 end-of-block
constexpr int kMaxBits = 15;                     // RFC 1951 limit
// Code-length limit the encoder builds (runtime, <= kMaxBits).  A chunk whose
// codes all fit the inflater's 11-bit first-level table decodes without the
// subtable branch; KVTC_DEFLATE_MAXBITS=11 forces that for every chunk (A/B:
// inflate -15 % cycles, CR 19.08 -> 18.99 on the bench workload, so the default
// stays at the RFC limit).  Any limit >= 9 (257 symbols) is valid.
constexpr int kDefaultMaxBits = 15;

__host__ __device__ inline uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ inline uint32_t umin32(uint32_t a, uint32_t b) { return a < b ? a : b; }

struct SectionHeader {
  uint32_t magic, version;
  uint64_t raw_bytes;
  uint32_t chunk_bytes, nchunks;
  uint32_t seg_bytes, nseg;
  uint64_t data_offset;
  uint64_t section_bytes;
  uint64_t pad[2];
};
static_assert(sizeof(SectionHeader) == 64, "section header is 64 bytes");
struct ChunkEntry {
  uint64_t offset;     // from data start
  uint32_t bytes;      // stream bytes
  uint32_t kind;       // 0 = Huffman (indexed), 1 = stored
};

__host__ __device__ inline uint32_t stored_bytes(uint32_t n) {
  const uint32_t blocks = n == 0 ? 1 : (n + 32767) / 32768;
  return n + 5 * blocks;
}
__host__ __device__ inline uint64_t slot_stride(int32_t chunk) { return ((stored_bytes(chunk) + 64 + 15) / 16) * 16; }

size_t deflate_section_bound(size_t n, int32_t chunk) {
  const size_t nch = (n + chunk - 1) / chunk;
  return sizeof(SectionHeader) + nch * sizeof(ChunkEntry) + ((nch * kNSeg * 2 + 15) & ~size_t(15)) +
         nch * ((stored_bytes(chunk) + 15) & ~15u) + 16;
}
size_t deflate_workspace(size_t n, int32_t chunk) {
  const size_t nch = (n + chunk - 1) / chunk;
  return nch * slot_stride(chunk) + nch * 8 + nch * kNSeg * 2 + 256;
}

// ---------------------------------------------------------- Huffman lengths
// In-place minimum-redundancy code lengths for weights sorted ascending
// (A[i] becomes the code length of the i-th lightest symbol).
__device__ void min_redundancy_lengths(int *A, int n) {
  if (n == 0) return;
  if (n == 1) {
    A[0] = 1;
    return;
  }
  int root, leaf, next, avbl, used, dpth;
  A[0] += A[1];
  root = 0;
  leaf = 2;
  for (next = 1; next < n - 1; next++) {
    if (leaf >= n || A[root] < A[leaf]) {
      A[next] = A[root];
      A[root++] = next;
    } else {
      A[next] = A[leaf++];
    }
    if (leaf >= n || (root < next && A[root] < A[leaf])) {
      A[next] += A[root];
      A[root++] = next;
    } else {
      A[next] += A[leaf++];
    }
  }
  A[n - 2] = 0;
  for (next = n - 3; next >= 0; next--) A[next] = A[A[next]] + 1;
  avbl = 1;
  used = dpth = 0;
  root = n - 2;
  next = n - 1;
  while (avbl > 0) {
    while (root >= 0 && A[root] == dpth) {
      used++;
      root--;
    }
    while (avbl > used) {
      A[next--] = dpth;
      avbl--;
    }
    avbl = 2 * used;
    dpth++;
    used = 0;
  }
}


// Phase 1 of the in-place minimum-redundancy construction (Moffat-Katajainen,
// the first loop of min_redundancy_lengths) with the two queue fronts cached in
// registers and the next values prefetched, so each step is ALU work instead of
// a chain of dependent shared-memory loads.  A[0..n) = weights ascending (n >= 2);
// on return A[i] (i < n - 2) = parent of internal node i, A[n - 2] = 0 (the root).
__device__ void mk_merge(int *A, const int n) {
  constexpr int INF = 0x7FFFFFFF;
  A[0] += A[1];
  int root = 0, leaf = 2;
  // internal-node queue [root, next): r0 = A[root], r1 = A[root + 1] (when they exist)
  int r0 = A[0], r1 = INF;
  // leaf queue [leaf, n): l0..l3 = A[leaf .. leaf + 3]
  int l0 = leaf < n ? A[leaf] : INF, l1 = leaf + 1 < n ? A[leaf + 1] : INF, l2 = leaf + 2 < n ? A[leaf + 2] : INF,
      l3 = leaf + 3 < n ? A[leaf + 3] : INF;
  for (int next = 1; next < n - 1; ++next) {
    int w;
    // first child (the internal queue is never empty here)
    if (leaf >= n || r0 < l0) {
      w = r0;
      A[root] = next;
      ++root;
      r0 = r1;
      r1 = root + 1 < next ? A[root + 1] : INF;
    } else {
      w = l0;
      ++leaf;
      l0 = l1; l1 = l2; l2 = l3;
      l3 = leaf + 3 < n ? A[leaf + 3] : INF;
    }
    // second child
    if (leaf >= n || (root < next && r0 < l0)) {
      w += r0;
      A[root] = next;
      ++root;
      r0 = r1;
      r1 = root + 1 < next ? A[root + 1] : INF;
    } else {
      w += l0;
      ++leaf;
      l0 = l1; l1 = l2; l2 = l3;
      l3 = leaf + 3 < n ? A[leaf + 3] : INF;
    }
    A[next] = w;
    if (root == next) r0 = w;             // the new node is the internal queue's front ...
    else if (root + 1 == next) r1 = w;    // ... or right behind it
  }
  A[n - 2] = 0;
}

// Single-thread: code lengths (<= maxbits, complete prefix code) for nsym
// symbols with frequencies freq[]; sorted[] = symbols with freq > 0 sorted by
// (freq, symbol) ascending, count nz.  work: int[nsym].
__device__ void build_lengths(const uint32_t *freq, const int *sorted, int nz, int maxbits, uint8_t *len, int nsym,
                              int *work) {
  for (int s = 0; s < nsym; ++s) len[s] = 0;
  if (nz == 0) return;
  if (nz == 1) {
    len[sorted[0]] = 1;
    return;
  }
  for (int i = 0; i < nz; ++i) work[i] = int(freq[sorted[i]]);
  min_redundancy_lengths(work, nz);
  int num[33];
  for (int i = 0; i < 33; ++i) num[i] = 0;
  for (int i = 0; i < nz; ++i) num[work[i] > 32 ? 32 : work[i]]++;
  // enforce the maximum length while keeping the Kraft sum exactly 1
  for (int i = maxbits + 1; i <= 32; i++) {
    num[maxbits] += num[i];
    num[i] = 0;
  }
  uint32_t total = 0;
  for (int i = maxbits; i > 0; i--) total += uint32_t(num[i]) << (maxbits - i);
  while (total != (1u << maxbits)) {
    num[maxbits]--;
    for (int i = maxbits - 1; i > 0; i--)
      if (num[i]) {
        num[i]--;
        num[i + 1] += 2;
        break;
      }
    total--;
  }
  // most frequent symbols get the shortest codes
  int j = nz;
  for (int l = 1; l <= maxbits; ++l)
    for (int k = num[l]; k > 0; --k) len[sorted[--j]] = uint8_t(l);
}

// Canonical codes (RFC 1951 §3.2.2), returned bit-reversed for LSB-first output.
__device__ void canonical_codes(const uint8_t *len, int nsym, uint16_t *rev_code) {
  int bl_count[16] = {0};
  for (int s = 0; s < nsym; ++s) bl_count[len[s]]++;
  bl_count[0] = 0;
  int next_code[16];
  int code = 0;
  for (int b = 1; b <= 15; ++b) {
    code = (code + bl_count[b - 1]) << 1;
    next_code[b] = code;
  }
  for (int s = 0; s < nsym; ++s) {
    const int l = len[s];
    if (l) {
      const uint32_t c = uint32_t(next_code[l]++);
      rev_code[s] = uint16_t(__brev(c) >> (32 - l));
    } else {
      rev_code[s] = 0;
    }
  }
}

// Small LSB-first bit writer into shared memory (block header).
struct BitWriter {
  uint32_t *buf;
  uint32_t nbits;
  __device__ void put(uint32_t v, int n) {
    for (int i = 0; i < n; ++i, ++nbits) {
      if (((v >> i) & 1u)) buf[nbits >> 5] |= 1u << (nbits & 31);
    }
  }
};


constexpr int kSortItems = (kLitSyms + kEncThreads - 1) / kEncThreads;   // >= 257 sort keys
// three 64-bit words of 12-bit counters (one per code length 1..15), block-scanned
struct U3 {
  uint64_t a, b, c;
};
struct U3Sum {
  __device__ U3 operator()(const U3 &x, const U3 &y) const { return U3{x.a + y.a, x.b + y.b, x.c + y.c}; }
};
__device__ __forceinline__ uint64_t &u3_word(U3 &u, int i) { return i == 0 ? u.a : (i == 1 ? u.b : u.c); }
using EncSort = cub::BlockRadixSort<uint32_t, kEncThreads, kSortItems>;

struct EncShared {
  union {
    uint32_t whist[kEncThreads / 32][kLitSyms + 3];   // warp-private histograms
    typename EncSort::TempStorage sort;               // (freq, symbol) radix sort, after the merge
    uint32_t skeys[kEncThreads * kSortItems];       // sorted (freq << 9 | symbol) keys, after the sort
    struct {                                          // code construction, after nz / sorted are read
      int work[kLitSyms + 3], dep[kLitSyms + 3], par[kLitSyms + 3], ndep[kLitSyms + 3];
    } mk;
    uint32_t len4[32];   // after the header: literal code lengths, 8 nibbles per word, so the
                         // bit-count pass's lookups hit 32 words (bank-conflict free)
  } u;
  uint32_t hist[kLitSyms + 3];
  uint32_t clhist[19];
  int sorted[kLitSyms + 3];
  int num[33];
  int nz;
  uint8_t len[kLitSyms + 3];
  uint16_t rev[kLitSyms + 3];
  uint32_t sym[256];                                 // rev | len << 16 for literals
  uint8_t cllen[19];
  uint16_t clrev[19];
  uint16_t rle_sym[kLitSyms + 8];
  uint8_t rle_extra[kLitSyms + 8];
  uint32_t hdr[160];   // header bits (<= 5120)
  uint32_t hdr_bits;
  int next_code[16];
  uint32_t startmask[9];                             // run starts of the 258 code lengths
  int nrle;
  typename cub::BlockScan<U3, kEncThreads>::TempStorage scan3;
  uint32_t total_bits;
  uint32_t segst[kNSeg];
  int use_stored;
  typename cub::BlockScan<uint32_t, kEncThreads>::TempStorage scan;
};

// Single-thread code-length builder over shared arrays (see build_lengths).
__device__ void build_lengths_s(const uint32_t *freq, const int *sorted, int nz, int maxbits, uint8_t *len, int nsym,
                                int *work, int *num) {
  for (int s = 0; s < nsym; ++s) len[s] = 0;
  if (nz == 0) return;
  if (nz == 1) {
    len[sorted[0]] = 1;
    return;
  }
  for (int i = 0; i < nz; ++i) work[i] = int(freq[sorted[i]]);
  min_redundancy_lengths(work, nz);
  for (int i = 0; i < 33; ++i) num[i] = 0;
  for (int i = 0; i < nz; ++i) num[work[i] > 32 ? 32 : work[i]]++;
  for (int i = maxbits + 1; i <= 32; i++) {
    num[maxbits] += num[i];
    num[i] = 0;
  }
  uint32_t total = 0;
  for (int i = maxbits; i > 0; i--) total += uint32_t(num[i]) << (maxbits - i);
  while (total != (1u << maxbits)) {
    num[maxbits]--;
    for (int i = maxbits - 1; i > 0; i--)
      if (num[i]) {
        num[i]--;
        num[i + 1] += 2;
        break;
      }
    total--;
  }
  int j = nz;
  for (int l = 1; l <= maxbits; ++l)
    for (int k = num[l]; k > 0; --k) len[sorted[--j]] = uint8_t(l);
}

// LSB-first word writer into shared memory (block header).
struct WordWriter {
  uint32_t *buf;
  uint64_t acc;
  uint32_t nb, w;
  __device__ void put(uint32_t v, int n) {
    acc |= uint64_t(v & ((1u << n) - 1)) << nb;
    nb += n;
    if (nb >= 32) {
      buf[w++] = uint32_t(acc);
      acc >>= 32;
      nb -= 32;
    }
  }
  __device__ uint32_t finish() {
    if (nb) buf[w] = uint32_t(acc);
    return w * 32 + nb;
  }
};


// Number of code-length-code symbols the RLE (RFC 1951 §3.2.7) emits for a run of
// L equal lengths v (the rule of the former serial loop: zeros -> 18 (11..138)
// while >= 11, then one 17 (3..10), then single zeros; v != 0 -> v, then 16
// (3..6 repeats) while >= 3, then single v's).
__device__ __forceinline__ int rle_count(int v, int L) {
  if (v == 0) {
    const int n18 = L / 138 + ((L % 138) >= 11 ? 1 : 0);
    const int left = (L % 138) >= 11 ? 0 : L % 138;
    return n18 + (left >= 3 ? 1 : left);
  }
  const int rep = L - 1;
  const int n16 = rep / 6 + ((rep % 6) >= 3 ? 1 : 0);
  const int left = (rep % 6) >= 3 ? 0 : rep % 6;
  return 1 + n16 + left;
}
__device__ __forceinline__ int rle_emit(int v, int L, uint16_t *sym, uint8_t *extra) {
  int n = 0;
  if (v == 0) {
    int left = L;
    while (left >= 11) {
      const int r = min(left, 138);
      sym[n] = 18; extra[n++] = uint8_t(r - 11); left -= r;
    }
    if (left >= 3) {
      sym[n] = 17; extra[n++] = uint8_t(left - 3); left = 0;
    }
    while (left-- > 0) { sym[n] = 0; extra[n++] = 0; }
  } else {
    sym[n] = uint16_t(v); extra[n++] = 0;
    int left = L - 1;
    while (left >= 3) {
      const int r = min(left, 6);
      sym[n] = 16; extra[n++] = uint8_t(r - 3); left -= r;
    }
    while (left-- > 0) { sym[n] = uint16_t(v); extra[n++] = 0; }
  }
  return n;
}
__device__ __forceinline__ void hdr_put(uint32_t *hdr, uint32_t pos, uint32_t v, int n) {
  const uint64_t x = uint64_t(v & ((1u << n) - 1)) << (pos & 31);
  atomicOr(&hdr[pos >> 5], uint32_t(x));
  if ((pos & 31) + n > 32) atomicOr(&hdr[(pos >> 5) + 1], uint32_t(x >> 32));
}

// The chunk's Huffman code and dynamic block header, all 128 threads.  Only the
// minimum-redundancy length computation (O(nz), in-place two-queue merge) and the
// 19-symbol code-length code run on one thread; lengths -> symbols, canonical
// codes (ranks by block scan), the run-length coding of the code lengths and the
// header bits (scanned offsets, atomicOr) are parallel.  Bit-identical to the
// former single-thread construction.
__device__ __forceinline__ void build_header(EncShared &S, const int t, const int maxbits) {
  const int nz = S.nz;
  for (int s = t; s < kLitSyms + 3; s += kEncThreads) S.len[s] = 0;
  for (int j = t; j < nz; j += kEncThreads) S.u.mk.work[j] = int(S.hist[S.sorted[j]]);
  if (t < 33) S.num[t] = 0;
  if (t < 9) S.startmask[t] = 0;
  for (int d = t; d < kLitSyms + 3; d += kEncThreads) S.u.mk.ndep[d] = 0;
  __syncthreads();
  // minimum-redundancy code lengths (Moffat-Katajainen): the merge on one thread
  // (register-cached queue fronts), internal-node depths by pointer jumping, the
  // leaf-length counts from the per-depth internal-node counts -- the same
  // lengths as min_redundancy_lengths, of which only num[] is needed
  if (t == 0 && nz > 1) mk_merge(S.u.mk.work, nz);
  __syncthreads();
  const int n_int = nz - 1;                       // internal nodes 0 .. nz - 2, root nz - 2
  for (int i = t; i < n_int; i += kEncThreads) {
    S.u.mk.dep[i] = i == n_int - 1 ? 0 : 1;
    S.u.mk.par[i] = i == n_int - 1 ? i : S.u.mk.work[i];
  }
  __syncthreads();
  for (int round = 0; round < 9; ++round) {       // depth <= 256 < 2^9; stops once every node points at the root
    int nd[2], np[2];
    int open = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = t + k * kEncThreads;
      if (i < n_int) {
        nd[k] = S.u.mk.dep[i] + S.u.mk.dep[S.u.mk.par[i]];
        np[k] = S.u.mk.par[S.u.mk.par[i]];
        open |= np[k] != n_int - 1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = t + k * kEncThreads;
      if (i < n_int) {
        S.u.mk.dep[i] = nd[k];
        S.u.mk.par[i] = np[k];
      }
    }
    if (!__syncthreads_or(open)) break;
  }
  for (int i = t; i < n_int; i += kEncThreads) atomicAdd(&S.u.mk.ndep[S.u.mk.dep[i]], 1);
  __syncthreads();
  if (t == 0) {
    int *num = S.num;
    if (nz == 1) num[1] = 1;
    else {
      // depth d holds avbl(d) nodes, ndep[d] of them internal: the rest are leaves
      int avbl = 1;
      for (int d = 0; avbl > 0; ++d) {
        const int used = d < kLitSyms + 3 ? S.u.mk.ndep[d] : 0;
        num[d > 32 ? 32 : d] += avbl - used;
        avbl = 2 * used;
      }
    }
    // enforce the maximum length while keeping the Kraft sum exactly 1
    for (int i = maxbits + 1; i <= 32; i++) {
      num[maxbits] += num[i];
      num[i] = 0;
    }
    if (nz > 1) {
      uint32_t total = 0;
      for (int i = maxbits; i > 0; i--) total += uint32_t(num[i]) << (maxbits - i);
      while (total != (1u << maxbits)) {
        num[maxbits]--;
        for (int i = maxbits - 1; i > 0; i--)
          if (num[i]) {
            num[i]--;
            num[i + 1] += 2;
            break;
          }
        total--;
      }
    }
    int code = 0;
    S.next_code[0] = 0;
    for (int b = 1; b <= maxbits; ++b) {
      code = (code + (b > 1 ? num[b - 1] : 0)) << 1;
      S.next_code[b] = code;
    }
  }
  __syncthreads();
  // most frequent symbols get the shortest codes: sorted position j (ascending
  // frequency) has rank nz-1-j from the top
  for (int j = t; j < nz; j += kEncThreads) {
    const int r = nz - 1 - j;
    int l = 1, c = S.num[1];
    while (r >= c && l < maxbits) c += S.num[++l];
    S.len[S.sorted[j]] = uint8_t(l);
  }
  __syncthreads();
  // canonical codes: code(s) = next_code[l] + #{s' < s : len[s'] = l}; thread t owns
  // symbols 3t .. 3t+2, cross-thread ranks from one block scan of packed counters
  {
    U3 mine{0, 0, 0};
    uint8_t l3[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int s = 3 * t + k;
      l3[k] = s < kLitSyms ? S.len[s] : 0;
      if (l3[k]) u3_word(mine, (l3[k] - 1) / 5) += 1ull << (12 * ((l3[k] - 1) % 5));
    }
    U3 before;
    cub::BlockScan<U3, kEncThreads>(S.scan3).ExclusiveScan(mine, before, U3{0, 0, 0}, U3Sum());
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int s = 3 * t + k;
      if (s >= kLitSyms) continue;
      const int l = l3[k];
      if (!l) {
        S.rev[s] = 0;
        continue;
      }
      int r = int((u3_word(before, (l - 1) / 5) >> (12 * ((l - 1) % 5))) & 0xFFF);
      for (int q = 0; q < k; ++q) r += l3[q] == l;
      const uint32_t c = uint32_t(S.next_code[l] + r);
      S.rev[s] = uint16_t(__brev(c) >> (32 - l));
    }
  }
  // run-length coding of the 257 literal/length code lengths + 1 distance length (0)
  constexpr int nseq = kLitSyms + 1;
  auto val = [&](int i) -> int { return i < kLitSyms ? S.len[i] : 0; };
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i = 3 * t + k;
    if (i < nseq && (i == 0 || val(i) != val(i - 1))) atomicOr(&S.startmask[i >> 5], 1u << (i & 31));
  }
  if (t < 19) S.clhist[t] = 0;
  __syncthreads();
  int run_v[3], run_l[3], nrun = 0, my_syms = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i = 3 * t + k;
    if (i >= nseq || !((S.startmask[i >> 5] >> (i & 31)) & 1u)) continue;
    // next run start after i (or the end)
    int q = nseq;
    int w = (i + 1) >> 5;
    uint32_t mbits = (i + 1) < 32 * 9 ? (S.startmask[w] & (~0u << ((i + 1) & 31))) : 0u;
    while (true) {
      if (mbits) {
        q = min(nseq, 32 * w + __ffs(mbits) - 1);
        break;
      }
      if (++w >= 9) break;
      mbits = S.startmask[w];
    }
    run_v[nrun] = val(i);
    run_l[nrun] = q - i;
    my_syms += rle_count(run_v[nrun], run_l[nrun]);
    ++nrun;
  }
  uint32_t sym_off_u, nr;
  cub::BlockScan<uint32_t, kEncThreads>(S.scan).ExclusiveSum(uint32_t(my_syms), sym_off_u, nr);
  const int sym_off = int(sym_off_u);
  {
    int o = sym_off;
    for (int r = 0; r < nrun; ++r) o += rle_emit(run_v[r], run_l[r], S.rle_sym + o, S.rle_extra + o);
    for (int q = sym_off; q < o; ++q) atomicAdd(&S.clhist[S.rle_sym[q]], 1u);
  }
  __syncthreads();
  if (t == 0) {
    // code-length code (19 symbols, <= 7 bits); a complete code needs >= 2 used symbols
    int used = 0;
    for (int i = 0; i < 19; ++i) used += S.clhist[i] != 0;
    for (int i = 0; i < 19 && used < 2; ++i)
      if (!S.clhist[i]) { S.clhist[i] = 1; used++; }
    int csorted[19];
    int cnz = 0;
    for (int s = 0; s < 19; ++s)
      if (S.clhist[s]) {
        int k = cnz++;
        while (k > 0 && (S.clhist[csorted[k - 1]] > S.clhist[s])) { csorted[k] = csorted[k - 1]; --k; }
        csorted[k] = s;
      }
    build_lengths_s(S.clhist, csorted, cnz, 7, S.cllen, 19, S.u.mk.work, S.num);
    canonical_codes(S.cllen, 19, S.clrev);
    const int order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    int hclen = 19;
    while (hclen > 4 && S.cllen[order[hclen - 1]] == 0) hclen--;
    WordWriter bw{S.hdr, 0, 0, 0};
    bw.put(1, 1);            // BFINAL
    bw.put(2, 2);            // BTYPE = 10 (dynamic Huffman)
    bw.put(0, 5);            // HLIT  = 257 - 257
    bw.put(0, 5);            // HDIST = 1 - 1
    bw.put(hclen - 4, 4);    // HCLEN
    for (int i = 0; i < hclen; ++i) bw.put(S.cllen[order[i]], 3);
    S.hdr_bits = bw.finish();   // prefix; the code-length symbols follow
  }
  __syncthreads();
  // code-length symbols at scanned bit offsets
  {
    uint32_t my_bits = 0;
    for (int q = sym_off; q < sym_off + my_syms; ++q) {
      const int sm = S.rle_sym[q];
      my_bits += S.cllen[sm] + (sm == 16 ? 2 : sm == 17 ? 3 : sm == 18 ? 7 : 0);
    }
    uint32_t boff, btot;
    cub::BlockScan<uint32_t, kEncThreads>(S.scan).ExclusiveSum(my_bits, boff, btot);
    uint32_t pos = S.hdr_bits + boff;
    for (int q = sym_off; q < sym_off + my_syms; ++q) {
      const int sm = S.rle_sym[q];
      hdr_put(S.hdr, pos, S.clrev[sm], S.cllen[sm]);
      pos += S.cllen[sm];
      const int ne = sm == 16 ? 2 : sm == 17 ? 3 : sm == 18 ? 7 : 0;
      if (ne) {
        hdr_put(S.hdr, pos, S.rle_extra[q], ne);
        pos += ne;
      }
    }
    __syncthreads();
    if (t == 0) S.hdr_bits += btot;
  }
  (void)nr;
  __syncthreads();
}

__device__ __forceinline__ void encode_chunk(EncShared &S, const int c, const uint8_t *in, uint64_t n, int32_t chunk,
                                             uint8_t *slots, uint64_t stride, uint32_t *chunk_bytes,
                                             uint32_t *chunk_kind, uint16_t *index, const int maxbits) {
  const uint64_t base = uint64_t(c) * chunk;
  const uint32_t nc = uint32_t(umin64(chunk, n - base));
  const uint8_t *src = in + base;
  uint8_t *out = slots + uint64_t(c) * stride;
  const int t = threadIdx.x;
  const int warp = t / 32;
  const uint32_t piece = uint32_t(chunk) / kEncThreads;
  const uint32_t p0 = umin32(nc, t * piece), p1 = umin32(nc, (t + 1) * piece);

  for (int s = t; s < (kEncThreads / 32) * (kLitSyms + 3); s += kEncThreads) (&S.u.whist[0][0])[s] = 0;
  if (t < 19) S.clhist[t] = 0;
  for (int i = t; i < 160; i += kEncThreads) S.hdr[i] = 0;
  __syncthreads();
  // ---- histogram: 16-byte vector loads over the whole chunk, warp-private bins
  {
    const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const uint32_t nvec = aligned ? nc / 16 : 0;
    uint32_t *h = S.u.whist[warp];
    const uint4 *sv = reinterpret_cast<const uint4 *>(src);
    uint4 q = t < nvec ? __ldg(sv + t) : make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t v = t; v < nvec; v += kEncThreads) {       // next 16 bytes loaded while these are counted
      const uint4 qn = v + kEncThreads < nvec ? __ldg(sv + v + kEncThreads) : q;
      const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 16; ++k) atomicAdd(&h[(w4[k >> 2] >> (8 * (k & 3))) & 0xFF], 1u);
      q = qn;
    }
    for (uint32_t i = nvec * 16 + t; i < nc; i += kEncThreads) atomicAdd(&h[src[i]], 1u);
  }
  __syncthreads();
  for (int s = t; s < kLitSyms; s += kEncThreads) {
    uint32_t v = 0;
#pragma unroll
    for (int w = 0; w < kEncThreads / 32; ++w) v += S.u.whist[w][s];
    S.hist[s] = v;
  }
  __syncthreads();
  if (t == 0) S.hist[256] = 1;  // end-of-block
  __syncthreads();
  // symbols by (freq, symbol) ascending: one radix sort of unique 26-bit keys
  // (freq <= 2^16 + 1, symbol < 512); zero-frequency symbols sort first.
  {
    uint32_t keys[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const int sym = t * kSortItems + i;
      keys[i] = sym < kLitSyms ? (S.hist[sym] << 9) | uint32_t(sym) : 0x3FFFFFFu;
    }
    EncSort(S.u.sort).Sort(keys, 0, 26);
    __syncthreads();                               // the sort's storage is reused for the keys
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) S.u.skeys[t * kSortItems + i] = keys[i];
  }
  __syncthreads();
  for (int i = t; i < kLitSyms; i += kEncThreads)
    if ((S.u.skeys[i] >> 9) != 0 && (i == 0 || (S.u.skeys[i - 1] >> 9) == 0)) S.nz = kLitSyms - i;
  __syncthreads();
  for (int j = t; j < S.nz; j += kEncThreads) S.sorted[j] = int(S.u.skeys[kLitSyms - S.nz + j] & 511u);
  __syncthreads();
  build_header(S, t, maxbits);
  for (int i = t; i < 256; i += kEncThreads) S.sym[i] = uint32_t(S.rev[i]) | (uint32_t(S.len[i]) << 16);
  if (t < 32) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v |= uint32_t(S.len[8 * t + k]) << (4 * k);
    S.u.len4[t] = v;
  }
  __syncthreads();
  // ---- bit counts per piece, exclusive scan
  const bool vec = ((reinterpret_cast<uintptr_t>(src + p0) & 15) == 0) && ((p1 - p0) % 16 == 0);
  uint32_t mybits = 0;
  if (vec && p0 < p1) {
    // the next 16 bytes are loaded while the current ones are counted
    const uint4 *v = reinterpret_cast<const uint4 *>(src + p0);
    const uint32_t nv = (p1 - p0) / 16;
    uint4 q = __ldg(v);
    for (uint32_t j = 0; j < nv; ++j) {
      const uint4 qn = __ldg(v + (j + 1 < nv ? j + 1 : j));
      const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t b = (w4[k >> 2] >> (8 * (k & 3))) & 0xFF;
        mybits += (S.u.len4[b >> 3] >> ((b & 7) * 4)) & 15u;
      }
      q = qn;
    }
  } else if (!vec) {
    for (uint32_t i = p0; i < p1; ++i) mybits += S.sym[src[i]] >> 16;
  }
  if (t == 0) mybits += S.hdr_bits;
  if (p1 == nc && p0 < p1) mybits += S.len[256];  // EOB after the last byte
  if (nc == 0 && t == 0) mybits += S.len[256];
  uint32_t myoff, total;
  cub::BlockScan<uint32_t, kEncThreads>(S.scan).ExclusiveSum(mybits, myoff, total);
  if (t == 0) {
    const uint32_t huff = (total + 7) / 8;
    S.use_stored = huff >= stored_bytes(nc);
    S.total_bits = total;
  }
  __syncthreads();
  if (S.use_stored) {
    // stored blocks of <= 32 KiB: [BFINAL|00][pad] LEN NLEN data
    const uint32_t blocks = nc == 0 ? 1 : (nc + 32767) / 32768;
    for (uint32_t b = t; b < blocks; b += kEncThreads) {
      const uint32_t len = umin32(32768, nc - b * 32768);
      uint8_t *o = out + b * (32768 + 5);
      o[0] = (b + 1 == blocks) ? 1 : 0;
      o[1] = len & 0xFF; o[2] = len >> 8; o[3] = (~len) & 0xFF; o[4] = ((~len) >> 8) & 0xFF;
    }
    for (uint32_t i = t; i < nc; i += kEncThreads) out[(i / 32768) * (32768 + 5) + 5 + (i % 32768)] = src[i];
    if (t == 0) {
      chunk_bytes[c] = stored_bytes(nc);
      chunk_kind[c] = 1;
    }
    return;
  }
  // ---- segment index: bit length of each 1/64 of the chunk (<= 15 * 1024 bits)
  const uint32_t pieces_per_seg = kEncThreads / kNSeg;
  if (t % pieces_per_seg == 0) S.segst[t / pieces_per_seg] = myoff + (t == 0 ? S.hdr_bits : 0);
  __syncthreads();
  if (t < kNSeg) index[uint64_t(c) * kNSeg + t] = uint16_t((t + 1 < kNSeg ? S.segst[t + 1] : S.total_bits) - S.segst[t]);
  // ---- emission (the words a thread shares with its neighbours start zeroed)
  uint32_t *ow = reinterpret_cast<uint32_t *>(out);
  const uint32_t w_first = myoff >> 5, w_last = (myoff + mybits - 1) >> 5;
  if (mybits) {
    ow[w_first] = 0;
    ow[w_last] = 0;
  }
  __syncthreads();
  // Every completed word is stored plainly, the first one of a thread included
  // (its low bits, the previous thread's tail, are still zero there); after a
  // barrier each thread ORs its final partial word -- the only word a thread
  // shares with the next one -- atomically.  No branch per flush.
  uint64_t acc = 0;
  uint32_t nb = myoff & 31;
  uint32_t *wp = ow + w_first;
  if (mybits) {
    if (t == 0) {
      // the block header: whole words copied, the partial last word seeds the accumulator
      const uint32_t hw = S.hdr_bits >> 5;
      for (uint32_t i = 0; i < hw; ++i) ow[i] = S.hdr[i];
      wp = ow + hw;
      nb = S.hdr_bits & 31;
      acc = nb ? (S.hdr[hw] & ((1u << nb) - 1)) : 0;
    }
    auto flush = [&]() {
      *wp++ = uint32_t(acc);
      acc >>= 32;
      nb -= 32;
    };
    auto put = [&](uint32_t e) {
      acc |= uint64_t(e & 0xFFFF) << nb;
      nb += e >> 16;
      if (nb >= 32) flush();
    };
    // two codes (<= 15 bits each) per accumulator step: nb < 32 before, < 62 after
    auto put2 = [&](uint32_t e0, uint32_t e1) {
      const uint32_t l0 = e0 >> 16;
      acc |= uint64_t((e0 & 0xFFFF) | ((e1 & 0xFFFF) << l0)) << nb;
      nb += l0 + (e1 >> 16);
      if (nb >= 32) flush();
    };
    if (vec) {
      for (uint32_t i = p0; i < p1; i += 16) {
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(src + i));
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 16; k += 2)
          put2(S.sym[__byte_perm(w4[k >> 2], 0, 0x4440 | (k & 3))], S.sym[__byte_perm(w4[k >> 2], 0, 0x4440 | ((k + 1) & 3))]);
      }
    } else {
      for (uint32_t i = p0; i < p1; ++i) put(S.sym[src[i]]);
    }
    if (p1 == nc) put(uint32_t(S.rev[256]) | (uint32_t(S.len[256]) << 16));
  }
  __syncthreads();
  if (mybits && nb) atomicOr(wp, uint32_t(acc));
  if (t == 0) {
    chunk_bytes[c] = (S.total_bits + 7) / 8;
    chunk_kind[c] = 0;
  }
}

// Grid-stride over chunks: the full grid (one CTA per chunk, ~14 per SM) when the
// encoder has the GPU, or a bounded grid (a few CTAs per SM) when it runs beside
// a persistent GEMM on the side stream, so the GEMM CTA always fits.
__global__ void __launch_bounds__(kEncThreads, 14) deflate_encode_kernel(const uint8_t *in, uint64_t n, int32_t chunk,
                                                                        uint32_t c_begin, uint32_t c_end, uint8_t *slots,
                                                                        uint64_t stride, uint32_t *chunk_bytes,
                                                                        uint32_t *chunk_kind, uint16_t *index,
                                                                        int maxbits) {
  __shared__ EncShared S;
  for (uint32_t c = c_begin + blockIdx.x; c < c_end; c += gridDim.x) {
    encode_chunk(S, int(c), in, n, chunk, slots, stride, chunk_bytes, chunk_kind, index, maxbits);
    __syncthreads();
  }
}

// Section assembly: one block computes the chunk offsets and the header; then
// one block per chunk copies the stream and its index entry.
__global__ void __launch_bounds__(1024) section_layout_kernel(const uint32_t *chunk_bytes, const uint32_t *chunk_kind, uint32_t nch,
                                      uint64_t n, int32_t chunk, uint8_t *out_base, const uint64_t *off_dev,
                                      uint64_t *section_len) {
  uint8_t *out = out_base + (off_dev ? *off_dev : 0);
  __shared__ typename cub::BlockScan<uint64_t, 1024>::TempStorage tmp;
  __shared__ uint64_t carry;
  SectionHeader *h = reinterpret_cast<SectionHeader *>(out);
  ChunkEntry *tab = reinterpret_cast<ChunkEntry *>(out + sizeof(SectionHeader));
  const uint64_t data_off =
      sizeof(SectionHeader) + uint64_t(nch) * sizeof(ChunkEntry) + ((uint64_t(nch) * kNSeg * 2 + 15) & ~15ull);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < nch; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const uint64_t sz = i < nch ? ((uint64_t(chunk_bytes[i]) + 15) & ~15ull) : 0;
    uint64_t off, tot;
    cub::BlockScan<uint64_t, 1024>(tmp).ExclusiveSum(sz, off, tot);
    if (i < nch) {
      tab[i].offset = carry + off;
      tab[i].bytes = chunk_bytes[i];
      tab[i].kind = chunk_kind[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    SectionHeader hh = {};
    hh.magic = kSectionMagic;
    hh.version = kSectionVersion;
    hh.raw_bytes = n;
    hh.chunk_bytes = uint32_t(chunk);
    hh.nchunks = nch;
    hh.seg_bytes = uint32_t(chunk) / kNSeg;
    hh.nseg = kNSeg;
    hh.data_offset = data_off;
    hh.section_bytes = data_off + carry;
    *h = hh;
    *section_len = data_off + carry;
  }
}

// 16-byte vectors (slots, section data and stream offsets are 16-byte aligned);
// bytes past the stream's end inside its last vector are zeroed so the
// container bytes are a function of the input alone.
__global__ void __launch_bounds__(256) section_copy_kernel(const uint8_t *slots, uint64_t stride, const uint16_t *index,
                                                          uint32_t nch, uint8_t *out_base, const uint64_t *off_dev) {
  uint8_t *out = out_base + (off_dev ? *off_dev : 0);
  const uint32_t c = blockIdx.x;
  const SectionHeader *h = reinterpret_cast<const SectionHeader *>(out);
  const ChunkEntry e = reinterpret_cast<const ChunkEntry *>(out + sizeof(SectionHeader))[c];
  uint16_t *idx = reinterpret_cast<uint16_t *>(out + sizeof(SectionHeader) + uint64_t(nch) * sizeof(ChunkEntry));
  if (threadIdx.x < kNSeg) idx[uint64_t(c) * kNSeg + threadIdx.x] = e.kind == 0 ? index[uint64_t(c) * kNSeg + threadIdx.x] : 0;
  const uint4 *s = reinterpret_cast<const uint4 *>(slots + uint64_t(c) * stride);
  uint4 *d = reinterpret_cast<uint4 *>(out + h->data_offset + e.offset);
  const uint32_t nv = (e.bytes + 15) / 16;
  for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
    uint4 v = __ldcs(s + i);
    if (i == nv - 1 && (e.bytes & 15)) {
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
      const uint32_t keep = e.bytes & 15;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int lo = 4 * k;
        if (lo >= int(keep)) w[k] = 0;
        else if (lo + 4 > int(keep)) w[k] &= (1u << (8 * (keep - lo))) - 1;
      }
      v = make_uint4(w[0], w[1], w[2], w[3]);
    }
    d[i] = v;
  }
}

namespace {
struct DeflateWs {
  uint32_t nch;
  uint64_t stride;
  uint8_t *slots;
  uint32_t *cbytes, *ckind;
  uint16_t *index;
};
__host__ __device__ DeflateWs deflate_ws(size_t n, int32_t chunk, void *ws) {
  DeflateWs w;
  w.nch = uint32_t((n + chunk - 1) / chunk);
  w.stride = slot_stride(chunk);
  w.slots = static_cast<uint8_t *>(ws);
  w.cbytes = reinterpret_cast<uint32_t *>(w.slots + w.nch * w.stride);
  w.ckind = w.cbytes + w.nch;
  w.index = reinterpret_cast<uint16_t *>(w.ckind + w.nch);
  return w;
}
}  // namespace

int corun_ctas(int per_sm) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms * per_sm;
}

// Code-length limit of the encoder (kDefaultMaxBits; KVTC_DEFLATE_MAXBITS in [9, 15] for A/B runs).
static int deflate_max_bits() {
  static const int v = [] {
    const char *e = getenv("KVTC_DEFLATE_MAXBITS");
    const int b = e ? atoi(e) : kDefaultMaxBits;
    return b < 9 ? 9 : (b > kMaxBits ? kMaxBits : b);
  }();
  return v;
}

kvtc_status launch_deflate_encode(const uint8_t *in, size_t n, int32_t chunk, void *ws, size_t ws_bytes,
                                  int32_t max_ctas, cudaStream_t st, uint32_t c_begin, uint32_t c_end) {
  KVTC_CHECK_ARG(chunk == 16384 || chunk == 32768 || chunk == 65536, "chunk_bytes must be 16/32/64 KiB");
  KVTC_CHECK_ARG(ws_bytes >= deflate_workspace(n, chunk), "deflate workspace");
  const DeflateWs w = deflate_ws(n, chunk, ws);
  c_end = std::min(c_end, w.nch);
  if (c_begin >= c_end) return KVTC_OK;
  const uint32_t nc = c_end - c_begin;
  const uint32_t grid = max_ctas > 0 ? std::min<uint32_t>(nc, uint32_t(max_ctas)) : nc;
  KVTC_MAX_CARVEOUT(deflate_encode_kernel);
  deflate_encode_kernel<<<grid, kEncThreads, 0, st>>>(in, n, chunk, c_begin, c_end, w.slots, w.stride, w.cbytes,
                                                      w.ckind, w.index, deflate_max_bits());
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

// Batched codec: the chunks of many payloads in one launch (jobs[j].chunk0 ascending).
__global__ void __launch_bounds__(kEncThreads, 14) deflate_encode_batch_kernel(const EncodeJob *jobs, int32_t njobs,
                                                                              uint32_t total, int32_t chunk,
                                                                              int maxbits) {
  __shared__ EncShared S;
  const uint64_t stride = slot_stride(chunk);
  for (uint32_t b = blockIdx.x; b < total; b += gridDim.x) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (jobs[mid].chunk0 <= b) lo = mid;
      else hi = mid - 1;
    }
    const EncodeJob jb = jobs[lo];
    const DeflateWs w = deflate_ws(jb.n, chunk, jb.ws);
    encode_chunk(S, int(b - jb.chunk0), jb.in, jb.n, chunk, w.slots, stride, w.cbytes, w.ckind, w.index, maxbits);
    __syncthreads();
  }
}

kvtc_status launch_deflate_encode_batch(const EncodeJob *jobs_dev, int32_t njobs, uint32_t total_chunks,
                                        int32_t chunk, cudaStream_t st, int32_t max_ctas) {
  KVTC_CHECK_ARG(chunk == 16384 || chunk == 32768 || chunk == 65536, "chunk_bytes must be 16/32/64 KiB");
  if (njobs == 0 || total_chunks == 0) return KVTC_OK;
  KVTC_MAX_CARVEOUT(deflate_encode_batch_kernel);
  const uint32_t grid = max_ctas > 0 ? std::min<uint32_t>(total_chunks, uint32_t(max_ctas)) : total_chunks;
  deflate_encode_batch_kernel<<<grid, kEncThreads, 0, st>>>(jobs_dev, njobs, total_chunks, chunk, deflate_max_bits());
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_deflate_assemble(size_t n, int32_t chunk, const void *ws, uint8_t *out, const uint64_t *off_dev,
                                    uint64_t *section_len_dev, cudaStream_t st) {
  const DeflateWs w = deflate_ws(n, chunk, const_cast<void *>(ws));
  section_layout_kernel<<<1, 1024, 0, st>>>(w.cbytes, w.ckind, w.nch, n, chunk, out, off_dev, section_len_dev);
  KVTC_LAUNCH_CHECK();
  if (w.nch > 0) {
    section_copy_kernel<<<w.nch, 256, 0, st>>>(w.slots, w.stride, w.index, w.nch, out, off_dev);
    KVTC_LAUNCH_CHECK();
  }
  return KVTC_OK;
}

kvtc_status launch_deflate(const uint8_t *in, size_t n, int32_t chunk, uint8_t *out, const uint64_t *off_dev,
                           uint64_t *section_len_dev, void *ws, size_t ws_bytes, cudaStream_t st) {
  kvtc_status s = launch_deflate_encode(in, n, chunk, ws, ws_bytes, 0, st);
  if (s) return s;
  return launch_deflate_assemble(n, chunk, ws, out, off_dev, section_len_dev, st);
}

// ================================================================ decoders
struct BitReader {
  const uint8_t *p;
  uint64_t nbytes;
  uint64_t pos;   // bit position
  __device__ uint32_t bits(int n) {
    uint32_t v = 0;
    for (int i = 0; i < n; ++i, ++pos) {
      const uint64_t byte = pos >> 3;
      const uint32_t b = byte < nbytes ? (p[byte] >> (pos & 7)) & 1u : 0u;
      v |= b << i;
    }
    return v;
  }
};

// canonical decode tables (puff style): count[len], symbols sorted by (len, sym)
struct Huff {
  int16_t count[16];
  int16_t symbol[320];
};
__device__ int huff_build(Huff &h, const uint8_t *len, int n) {
  for (int l = 0; l < 16; ++l) h.count[l] = 0;
  for (int s = 0; s < n; ++s) h.count[len[s]]++;
  if (h.count[0] == n) return 0;
  int left = 1;
  for (int l = 1; l < 16; ++l) {
    left <<= 1;
    left -= h.count[l];
    if (left < 0) return -1;   // over-subscribed
  }
  int offs[16];
  offs[1] = 0;
  for (int l = 1; l < 15; ++l) offs[l + 1] = offs[l] + h.count[l];
  for (int s = 0; s < n; ++s)
    if (len[s]) h.symbol[offs[len[s]]++] = int16_t(s);
  return left;
}
__device__ int huff_decode(BitReader &br, const Huff &h) {
  int code = 0, first = 0, index = 0;
  for (int l = 1; l < 16; ++l) {
    code |= int(br.bits(1));
    const int count = h.count[l];
    if (code - count < first) return h.symbol[index + (code - first)];
    index += count;
    first += count;
    first <<= 1;
    code <<= 1;
  }
  return -10;
}

// Parse a dynamic block header; fills literal/length and distance lengths.
__device__ int parse_dynamic(BitReader &br, uint8_t *lens, int &nlen, int &ndist) {
  nlen = int(br.bits(5)) + 257;
  ndist = int(br.bits(5)) + 1;
  const int ncode = int(br.bits(4)) + 4;
  if (nlen > 286 || ndist > 30) return -3;
  const int order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
  uint8_t cl[19];
  for (int i = 0; i < 19; ++i) cl[i] = 0;
  for (int i = 0; i < ncode; ++i) cl[order[i]] = uint8_t(br.bits(3));
  Huff hc;
  if (huff_build(hc, cl, 19) != 0) return -4;
  int idx = 0;
  while (idx < nlen + ndist) {
    int sym = huff_decode(br, hc);
    if (sym < 0) return sym;
    if (sym < 16) {
      lens[idx++] = uint8_t(sym);
    } else {
      int rep = 0;
      uint8_t v = 0;
      if (sym == 16) {
        if (idx == 0) return -5;
        v = lens[idx - 1];
        rep = 3 + int(br.bits(2));
      } else if (sym == 17) {
        rep = 3 + int(br.bits(3));
      } else {
        rep = 11 + int(br.bits(7));
      }
      if (idx + rep > nlen + ndist) return -6;
      while (rep--) lens[idx++] = v;
    }
  }
  if (lens[256] == 0) return -9;
  return 0;
}

// ---- fast path: our indexed Huffman-literal chunks, 64 threads per chunk
// Bit reader over shared-memory words (header parsing).
struct SmemBits {
  const uint32_t *w;
  uint32_t pos;
  __device__ uint32_t get(int n) {   // n <= 25
    const uint32_t wi = pos >> 5;
    const uint64_t v = (uint64_t(w[wi]) | (uint64_t(w[wi + 1]) << 32)) >> (pos & 31);
    pos += n;
    return uint32_t(v) & ((1u << n) - 1);
  }
};
__device__ int huff_decode_s(SmemBits &br, const Huff &h) {
  int code = 0, first = 0, index = 0;
  for (int l = 1; l < 16; ++l) {
    code |= int(br.get(1));
    const int count = h.count[l];
    if (code - count < first) return h.symbol[index + (code - first)];
    index += count;
    first += count;
    first <<= 1;
    code <<= 1;
  }
  return -10;
}

constexpr int kHdrWords = 512;     // first 2 KiB of a chunk stream hold its block header
constexpr int kTabBits = 11;       // first-level decode table: codes <= 11 bits in one lookup
constexpr int kSubBits = 15 - kTabBits;
// Canonical codes longer than kTabBits fill a contiguous range at the end of the
// code space of measure <= 256 * 2^-12, i.e. at most 2^kTabBits / 16 + 1 distinct
// first-level prefixes.
constexpr int kSubTabs = (1 << kTabBits) / 16 + 1;
constexpr int kInfThreads = kNSeg; // one thread per segment, 2 warps per chunk
static_assert(kNSeg == 64, "the segment-start scan below assumes two warps");

constexpr int kRing = 4;           // per-lane ring of 16-byte stream blocks (cp.async read-ahead)
struct FastShared {
  union {                          // three phases of a chunk:
    uint32_t hdr[kHdrWords + 2];   //   header words (header parse by thread 0),
    struct {                       //   canonical codes + subtable prefixes (table build),
      uint16_t code[260];
      uint32_t premask[(1 << kTabBits) / 32], prebase[(1 << kTabBits) / 32];
    } tb;
    uint4 ring[kNSeg][kRing];      //   per-lane read-ahead blocks (segment decode), lane-contiguous
  };
  // entries: literal (sym << 8) | len; end-of-block kTeEob | len; no code kTeBad;
  // longer code (k << 8) | kTeLink: subtable k (first level only)
  uint16_t table[1 << kTabBits];
  uint16_t sub[kSubTabs << kSubBits];  // second level: the next kSubBits bits
  int cnt[16], next[16];
  uint32_t wsum[2][4];
  uint8_t lens[320];
  uint8_t cltab[128];              // code-length code: (sym << 3) | len, 7-bit lookup
  uint32_t segstart[kNSeg];
  uint32_t hdr_bits;
  int status;
  int fast;                        // every code <= kTabBits bits: no subtables
};
constexpr uint32_t kTeLink = 0x10, kTeBad = 0x20, kTeEob = 0x40;

struct InflateJobs {
  const uint8_t *sec[2];           // sections
  uint64_t sec_len[2];             // bytes the section may occupy (bounds every read)
  uint64_t n_out[2];
  uint32_t nch[2];
  uint8_t *out[2];
};

__constant__ uint8_t c_cl_order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// Canonical codes (RFC 1951 §3.2.2) bit-reversed for LSB-first lookup.
__device__ void reversed_codes(const uint8_t *len, int n, uint16_t *rev) {
  int cnt[16] = {0}, next[16];
  for (int s = 0; s < n; ++s) cnt[len[s]]++;
  cnt[0] = 0;
  int code = 0;
  for (int b = 1; b < 16; ++b) {
    code = (code + cnt[b - 1]) << 1;
    next[b] = code;
  }
  for (int s = 0; s < n; ++s)
    rev[s] = len[s] ? uint16_t(__brev(uint32_t(next[len[s]]++)) >> (32 - len[s])) : 0;
}

// Block header of one of our chunk streams (literals + EOB, one final dynamic
// block), parsed by one thread from the shared-memory copy of its first words.
__device__ int parse_header_fast(FastShared &S) {
  SmemBits br{S.hdr, 0};
  const uint32_t bfinal = br.get(1), btype = br.get(2);
  if (bfinal != 1 || btype != 2) return -1;
  const int nlen = int(br.get(5)) + 257;
  const int ndist = int(br.get(5)) + 1;
  const int ncode = int(br.get(4)) + 4;
  if (nlen != 257 || ndist > 30) return -7;            // our encoder: literals + EOB only
  uint8_t cl[19];
  for (int i = 0; i < 19; ++i) cl[i] = 0;
  for (int i = 0; i < ncode; ++i) cl[c_cl_order[i]] = uint8_t(br.get(3));
  {
    Huff hc;
    if (huff_build(hc, cl, 19) != 0) return -4;        // complete code-length code required
    uint16_t rv[19];
    reversed_codes(cl, 19, rv);
    for (int sym = 0; sym < 19; ++sym)
      if (cl[sym])
        for (uint32_t f = rv[sym]; f < 128; f += 1u << cl[sym]) S.cltab[f] = uint8_t((sym << 3) | cl[sym]);
  }
  int idx = 0;
  const int total = nlen + ndist;
  while (idx < total) {
    const uint32_t w = S.hdr[br.pos >> 5], w2 = S.hdr[(br.pos >> 5) + 1];
    const uint32_t peek = uint32_t(((uint64_t(w) | (uint64_t(w2) << 32)) >> (br.pos & 31)) & 127u);
    const uint8_t e = S.cltab[peek];
    br.pos += e & 7;
    const int sym = e >> 3;
    if (sym < 16) {
      S.lens[idx++] = uint8_t(sym);
      continue;
    }
    int rep;
    uint8_t v = 0;
    if (sym == 16) {
      if (idx == 0) return -5;
      v = S.lens[idx - 1];
      rep = 3 + int(br.get(2));
    } else if (sym == 17) {
      rep = 3 + int(br.get(3));
    } else {
      rep = 11 + int(br.get(7));
    }
    if (idx + rep > total) return -6;
    while (rep--) S.lens[idx++] = v;
    if (br.pos > 32u * kHdrWords) return -7;
  }
  if (br.pos > 32u * kHdrWords) return -7;
  if (S.lens[256] == 0) return -9;
  S.hdr_bits = br.pos;
  return 0;   // the literal/length code itself is checked and built in parallel (inflate_chunk)
}

// One lane's serial decoder over its segment.  Per pair of codes: the 32 bits at
// the bit position from two words kept in registers (lo, hi = stream words
// bp/32, bp/32 + 1) by one funnel shift (two codes of <= 15 bits fit), two table
// lookups, the output byte taken from the entry's high byte by a byte permute.
// The word after hi is loaded from the ring at the start of the pair, off the
// dependency chain, and shifted in when the pair crossed a word (<= 30 bits:
// at most one): one ring load and two table loads per pair (ncu: the shared-
// memory pipe, ~2.4 wavefronts per load from random bank conflicts, bounds this
// loop).  With every code <= kTabBits bits (kFast) there is no subtable branch and
// the ring advances once per 16 codes (16 x 11 + 96 bits stay inside 3 blocks),
// else once per 8 (8 x 15 + 96).
struct DecodeLane {
  const uint16_t *table, *sub;
  const uint32_t *ring;                    // this lane's 16 ring words
  const uint4 *blk;
  uint32_t nblk, issued, bp, bad;
  uint32_t lo, hi;                         // stream words bp/32 and bp/32 + 1 (after load_window)

  __device__ __forceinline__ void advance(uint4 *ring_slots) {   // blocks of bp .. bp+2 resident
    const uint32_t last = (bp >> 7) + kRing - 1;
    for (; issued <= last; ++issued) {
      if (issued < nblk)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ring_slots + (issued & (kRing - 1)))),
                     "l"(blk + issued)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
  }
  __device__ __forceinline__ void load_window() {
    const uint32_t w = bp >> 5;
    lo = ring[w & 15];
    hi = ring[(w + 1) & 15];
  }
  __device__ __forceinline__ uint32_t window() const {
    const uint32_t w = bp >> 5;
    return __funnelshift_r(ring[w & 15], ring[(w + 1) & 15], bp);
  }
  template <bool kFast>
  __device__ __forceinline__ uint32_t lookup(uint32_t bits) const {
    uint32_t te = table[bits & ((1u << kTabBits) - 1)];
    if (!kFast && (te & kTeLink)) te = sub[((te >> 8) << kSubBits) | ((bits >> kTabBits) & ((1u << kSubBits) - 1))];
    return te;
  }
  template <bool kFast>
  __device__ __forceinline__ uint32_t pair() {       // two codes -> bytes 0, 1
    const uint32_t w = bp >> 5;
    const uint32_t nxt = ring[(w + 2) & 15];
    const uint32_t bits = __funnelshift_r(lo, hi, bp);
    const uint32_t t0 = lookup<kFast>(bits);
    const uint32_t t1 = lookup<kFast>(bits >> (t0 & 15));
    bp += (t0 & 15) + (t1 & 15);
    bad |= t0 | t1;
    const bool adv = (bp >> 5) != w;
    lo = adv ? hi : lo;
    hi = adv ? nxt : hi;
    return __byte_perm(t0, t1, 0x0051);
  }
  template <bool kFast>
  __device__ __forceinline__ void run(uint8_t *o, uint32_t s0, uint32_t s1, bool vec_out, uint4 *ring_slots) {
    uint32_t i = s0;
    // 16 codes -> one 16-byte store (segments are 16-byte aligned)
    if (vec_out && i + 16 <= s1) {
      advance(ring_slots);
      load_window();
    }
    for (; vec_out && i + 16 <= s1; i += 16) {
      uint32_t w[4];
      if (kFast) advance(ring_slots);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!kFast) advance(ring_slots);
        const uint32_t p0 = pair<kFast>(), p1 = pair<kFast>();
        w[2 * h] = __byte_perm(p0, p1, 0x5410);
        const uint32_t p2 = pair<kFast>(), p3 = pair<kFast>();
        w[2 * h + 1] = __byte_perm(p2, p3, 0x5410);
      }
      *reinterpret_cast<uint4 *>(o + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (; i < s1; ++i) {
      if (((i - s0) & 7) == 0) advance(ring_slots);
      const uint32_t te = lookup<kFast>(window());
      bp += te & 15;
      bad |= te;
      o[i] = uint8_t(te >> 8);
    }
  }
};

// Chunk c of the section at `section` (raw size n_out, nch chunks) into out_base.
// Every read is bounded by sec_len (the section's extent in the container, known
// to the host): a damaged header, chunk table, index or stream sets *err (the
// caller reports KVTC_E_CORRUPT) and never reads outside the section.
__device__ __forceinline__ void inflate_chunk(FastShared &S, const uint8_t *section, uint64_t sec_len, uint64_t n_out,
                                              uint32_t nch, uint32_t c, uint8_t *out_base, int32_t *err) {
  const SectionHeader *hdr = reinterpret_cast<const SectionHeader *>(section);
  const int tid = threadIdx.x;
  const uint64_t data_off =
      sizeof(SectionHeader) + uint64_t(nch) * sizeof(ChunkEntry) + ((uint64_t(nch) * kNSeg * 2 + 15) & ~15ull);
  if (sec_len < data_off || hdr->magic != kSectionMagic || hdr->version != kSectionVersion ||
      hdr->raw_bytes != n_out || hdr->nchunks != nch || hdr->nseg != kNSeg ||
      hdr->seg_bytes * kNSeg != hdr->chunk_bytes || hdr->seg_bytes % 16 || hdr->data_offset != data_off ||
      hdr->section_bytes > sec_len || hdr->chunk_bytes == 0 ||
      uint64_t(nch) != (n_out + hdr->chunk_bytes - 1) / hdr->chunk_bytes) {
    if (tid == 0) atomicExch(err, -20);
    return;
  }
  const ChunkEntry e = reinterpret_cast<const ChunkEntry *>(section + sizeof(SectionHeader))[c];
  const uint64_t obase = uint64_t(c) * hdr->chunk_bytes;
  const uint32_t nc = uint32_t(umin64(hdr->chunk_bytes, hdr->raw_bytes - obase));
  if (e.kind > 1 || (e.offset & 15) || e.offset + ((uint64_t(e.bytes) + 15) & ~15ull) > hdr->section_bytes - data_off ||
      (e.kind == 1 && e.bytes < stored_bytes(nc))) {
    if (tid == 0) atomicExch(err, -21);
    return;
  }
  const uint16_t *index =
      reinterpret_cast<const uint16_t *>(section + sizeof(SectionHeader) + uint64_t(hdr->nchunks) * sizeof(ChunkEntry));
  const uint8_t *stream = section + data_off + e.offset;
  uint8_t *o = out_base + obase;
  if (e.kind == 1) {
    for (uint32_t i = tid; i < nc; i += kInfThreads) o[i] = stream[(i / 32768) * (32768 + 5) + 5 + (i % 32768)];
    return;
  }
  // header words -> shared memory (coalesced), parsed by thread 0 from there
  const uint32_t *words = reinterpret_cast<const uint32_t *>(stream);
  const uint32_t nw = umin32((e.bytes + 3) / 4, kHdrWords);
  for (uint32_t i = tid; i < kHdrWords + 2; i += kInfThreads) S.hdr[i] = i < nw ? __ldg(words + i) : 0u;
  // kTeBad marks "no code here" (len 0): a corrupt stream sets it in `bad`
  for (int i = tid; i < (1 << kTabBits); i += kInfThreads) S.table[i] = kTeBad;
  const uint32_t mylen = index[uint64_t(c) * kNSeg + tid];
  __syncthreads();
  if (tid == 0) {
    const int st = parse_header_fast(S);
    S.status = st;
    if (st) atomicExch(err, st);
  }
  __syncthreads();
  if (S.status) return;
  // ---- the literal/length code, all 64 threads (thread t owns symbols 5t .. 5t+4):
  // length counts, Kraft check (over-subscribed = corrupt), canonical codes by
  // rank within each length, first-level table, subtables for codes > 11 bits
  // indexed by the rank of their first-level prefix
  if (tid < 16) S.cnt[tid] = 0;
  if (tid < (1 << kTabBits) / 32) S.tb.premask[tid] = 0;
  __syncthreads();
  uint8_t l5[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int sym = 5 * tid + k;
    l5[k] = sym < 257 ? S.lens[sym] : 0;
    if (l5[k]) atomicAdd(&S.cnt[l5[k]], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int left = 1;                             // RFC 1951 §3.2.2 / zlib: over-subscribed codes are invalid
    int code = 0;
    for (int b = 1; b < 16; ++b) {
      left = (left << 1) - S.cnt[b];
      if (left < 0) {
        S.status = -4;
        atomicExch(err, -4);
        break;
      }
      code = (code + (b > 1 ? S.cnt[b - 1] : 0)) << 1;
      S.next[b] = code;
    }
    int longer = 0;
    for (int b = kTabBits + 1; b < 16; ++b) longer |= S.cnt[b];
    S.fast = longer == 0;
  }
  // ranks: per-thread length counts, exclusive prefix over the 64 threads (two
  // warps) with 16 x 9-bit... counters packed as 4 lengths per 32-bit word x 4 words
  {
    uint32_t pk[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (l5[k]) pk[l5[k] >> 2] += 1u << (8 * (l5[k] & 3));
    uint32_t ex[4];
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t v = pk[q];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += y;
      }
      ex[q] = v - pk[q];
      if (lane == 31) S.wsum[w][q] = v;
    }
    __syncthreads();
    if (S.status) return;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int sym = 5 * tid + k;
      const int l = l5[k];
      if (sym >= 257) break;
      if (!l) {
        S.tb.code[sym] = 0;
        continue;
      }
      int r = int((ex[l >> 2] >> (8 * (l & 3))) & 0xFF);
      if (w) r += int((S.wsum[0][l >> 2] >> (8 * (l & 3))) & 0xFF);
      for (int q = 0; q < k; ++q) r += l5[q] == l;
      S.tb.code[sym] = uint16_t(__brev(uint32_t(S.next[l] + r)) >> (32 - l));
    }
  }
  __syncthreads();
  if (!S.fast)
    for (int i = tid; i < (kSubTabs << kSubBits); i += kInfThreads) S.sub[i] = kTeBad;
  for (int sym = tid; sym < 257; sym += kInfThreads) {
    const int l = S.lens[sym];
    if (l == 0) continue;
    const uint16_t ent = uint16_t(sym < 256 ? (sym << 8) | l : kTeEob | l);
    if (l <= kTabBits) {
      for (uint32_t f = S.tb.code[sym]; f < (1u << kTabBits); f += (1u << l)) S.table[f] = ent;
    } else {
      const uint32_t pre = S.tb.code[sym] & ((1u << kTabBits) - 1);
      atomicOr(&S.tb.premask[pre >> 5], 1u << (pre & 31));
    }
  }
  __syncthreads();
  {
    // subtable index of a prefix = its rank among the marked prefixes
    if (tid < 32) {
      const uint32_t a = __popc(S.tb.premask[2 * tid]), b = __popc(S.tb.premask[2 * tid + 1]);
      uint32_t v = a + b;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
        if (tid >= d) v += y;
      }
      S.tb.prebase[2 * tid] = v - a - b;
      S.tb.prebase[2 * tid + 1] = v - b;
    }
    __syncthreads();
    for (int sym = tid; sym < 257; sym += kInfThreads) {
      const int l = S.lens[sym];
      if (l <= kTabBits) continue;
      const uint32_t pre = S.tb.code[sym] & ((1u << kTabBits) - 1);
      const uint32_t k = S.tb.prebase[pre >> 5] + __popc(S.tb.premask[pre >> 5] & ((1u << (pre & 31)) - 1));
      if (k >= uint32_t(kSubTabs)) {
        S.status = -8;
        atomicExch(err, -8);
        continue;
      }
      S.table[pre] = uint16_t((k << 8) | kTeLink);
      uint16_t *st = S.sub + (k << kSubBits);
      const uint16_t ent = uint16_t(sym < 256 ? (sym << 8) | l : kTeEob | l);
      for (uint32_t f = S.tb.code[sym] >> kTabBits; f < (1u << kSubBits); f += (1u << (l - kTabBits))) st[f] = ent;
    }
  }
  // segment start = header bits + exclusive prefix of the segment lengths
  {
    uint32_t v = mylen;
    const int lane = tid & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += y;
    }
    S.segstart[tid] = v;                     // inclusive within the warp
  }
  __syncthreads();
  if (S.status) return;
  const uint32_t seg = hdr->seg_bytes;
  const uint32_t s0 = tid * seg, s1 = umin32(nc, (tid + 1) * seg);
  if (s0 >= s1) return;
  uint64_t pos = S.hdr_bits + S.segstart[tid] - mylen + (tid >= 32 ? S.segstart[31] : 0);
  // Read-ahead through shared memory: each lane streams its own segment, so
  // loads cannot be coalesced; 16-byte cp.async copies fill a per-lane ring of 4
  // blocks (16 words, lane-contiguous) in the background.
  const uint4 *blk = reinterpret_cast<const uint4 *>(stream);
  const uint32_t nblk = (e.bytes + 15) / 16;
  DecodeLane L{S.table, S.sub, reinterpret_cast<const uint32_t *>(&S.ring[tid][0]), blk, nblk, uint32_t(pos >> 7),
               uint32_t(pos), 0u};
  const bool vec_out = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
  if (S.fast) L.run<true>(o, s0, s1, vec_out, &S.ring[tid][0]);
  else L.run<false>(o, s0, s1, vec_out, &S.ring[tid][0]);
  uint32_t bad = L.bad;
  if (s1 == nc) {                            // the chunk's last segment ends with the end-of-block code
    L.advance(&S.ring[tid][0]);
    const uint32_t te = L.lookup<false>(L.window());
    if ((te & (kTeBad | kTeEob)) != kTeEob) bad |= kTeBad;
    L.bp += te & 15;
  }
  // each segment must end exactly where the side index says, inside the stream
  if (uint64_t(L.bp) != pos + mylen || uint64_t(L.bp) > uint64_t(e.bytes) * 8) bad |= kTeBad;
  if (bad & (kTeBad | kTeEob)) atomicExch(err, -7);
  asm volatile("cp.async.wait_all;" ::: "memory");   // no copy may land in the next chunk's header
}

// Grid-stride over the chunks of both jobs (full grid alone; bounded grid
// beside a persistent GEMM, see deflate_encode_kernel).
__global__ void __launch_bounds__(kInfThreads, 16) inflate_fast_kernel(InflateJobs J, int32_t *err) {
  __shared__ FastShared S;
  const uint32_t total = J.nch[0] + J.nch[1];
  for (uint32_t b = blockIdx.x; b < total; b += gridDim.x) {
    const int job = b < J.nch[0] ? 0 : 1;
    const uint32_t c = job == 0 ? b : b - J.nch[0];
    inflate_chunk(S, J.sec[job], J.sec_len[job], J.n_out[job], J.nch[job], c, J.out[job], err);
    __syncthreads();
  }
}

// ---- fused inverse front end: inflate -> unpack -> dequantise, one launch.
// Work items: the chunks of both sections (inflate, as inflate_fast_kernel), then
// per stream, tile and 32-chunk block the four 32-row blocks of D^ (dequant_block,
// 2 warps).  A
// block of D^ needs every chunk overlapping its 128-token tile; each inflated
// chunk bumps its tiles' arrival counters (release), and a CTA that finishes a
// chunk takes the next dequant block as soon as its tile is complete (acquire),
// so the payload is dequantised while still in L2 and the dequantisation fills
// the SM slots the latency-bound inflater leaves idle.  Deadlock-free: a CTA only
// waits for a tile once every chunk item has been handed out (to running CTAs,
// which never wait); before that, a CTA whose claimed block is not ready yet
// inflates chunks meanwhile.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t tile_chunks(const InflateDqStream &s, uint32_t cb_shift, uint32_t t) {
  const uint64_t b0 = uint64_t(t) * uint64_t(s.dq.tile_bytes);
  const uint64_t b1 = umin64(s.n_out, b0 + uint64_t(s.dq.tile_bytes));
  return uint32_t(((b1 - 1) >> cb_shift) - (b0 >> cb_shift) + 1);
}
// dequant item q of the launch = (stream, tile, 32-chunk block): its 4 row blocks
__device__ __forceinline__ bool dq_item_ready(const InflateDqArgs &A, uint32_t q) {
  const int sv = q < A.s[0].ndq ? 0 : 1;
  const InflateDqStream &s = A.s[sv];
  const uint32_t t = (sv ? q - A.s[0].ndq : q) / s.nbx;
  return ld_acquire_u32(s.tile_done + t) >= tile_chunks(s, A.cb_shift, t);
}

__global__ void __launch_bounds__(kInfThreads, 16) inflate_dequant_kernel(InflateDqArgs A) {
  __shared__ FastShared S;
  __shared__ int s_kind;
  __shared__ uint32_t s_arg;
  const uint32_t nch = A.s[0].nch + A.s[1].nch, ndq = A.s[0].ndq + A.s[1].ndq;
  int64_t pending = -1;                                  // thread 0: a claimed, not yet ready block
  for (;;) {
    if (threadIdx.x == 0) {
      int kind = 0;
      uint32_t arg = 0;
      for (;;) {
        if (pending >= 0) {
          if (dq_item_ready(A, uint32_t(pending))) {
            kind = 2;
            arg = uint32_t(pending);
            pending = -1;
            break;
          }
          const uint32_t c = atomicAdd(&A.ctr[0], 1u);
          if (c < nch) {
            kind = 1;
            arg = c;
            break;
          }
          __nanosleep(200);
          continue;
        }
        const uint32_t qp = *reinterpret_cast<volatile uint32_t *>(&A.ctr[1]);
        if (qp < ndq && dq_item_ready(A, qp)) {
          const uint32_t q = atomicAdd(&A.ctr[1], 1u);
          if (q < ndq) {
            pending = q;
            continue;
          }
        }
        const uint32_t c = atomicAdd(&A.ctr[0], 1u);
        if (c < nch) {
          kind = 1;
          arg = c;
          break;
        }
        const uint32_t q = atomicAdd(&A.ctr[1], 1u);
        if (q < ndq) {
          pending = q;
          continue;
        }
        break;                                           // nothing left
      }
      s_kind = kind;
      s_arg = arg;
    }
    __syncthreads();
    const int kind = s_kind;
    const uint32_t arg = s_arg;
    if (kind == 0) break;
    if (kind == 1) {
      const int sv = arg < A.s[0].nch ? 0 : 1;
      const InflateDqStream &s = A.s[sv];
      const uint32_t c = sv ? arg - A.s[0].nch : arg;
      inflate_chunk(S, s.sec, s.sec_len, s.n_out, s.nch, c, s.out, A.err);
      __syncthreads();
      if (threadIdx.x == 0 && s.ndq) {                   // publish the chunk to its tiles
        __threadfence();
        const uint64_t b0 = uint64_t(c) << A.cb_shift, b1 = umin64(s.n_out, b0 + (uint64_t(1) << A.cb_shift));
        const uint64_t tb = uint64_t(s.dq.tile_bytes);
        for (uint64_t t = b0 / tb; t <= (b1 - 1) / tb; ++t) atomicAdd(s.tile_done + t, 1u);
      }
    } else {
      const int sv = arg < A.s[0].ndq ? 0 : 1;
      const InflateDqStream &s = A.s[sv];
      const uint32_t q = sv ? arg - A.s[0].ndq : arg;
      const uint32_t t = q / s.nbx, bx = q - t * s.nbx;
      const int64_t nby = (s.dq.m + 31) / 32;
      for (int64_t by = int64_t(t) * (kTileM / 32); by < nby && by < int64_t(t + 1) * (kTileM / 32); ++by)
        dequant_block<kInfThreads / 32>(s.dq, by, bx, threadIdx.x & 31, threadIdx.x >> 5);
    }
    __syncthreads();
  }
}

kvtc_status launch_inflate_dequant(const InflateDqArgs &a, cudaStream_t st) {
  const uint32_t items = a.s[0].nch + a.s[1].nch + a.s[0].ndq + a.s[1].ndq;
  if (!items) return KVTC_OK;
  static int max_grid = 0;
  if (!max_grid) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    KVTC_MAX_CARVEOUT(inflate_dequant_kernel);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, inflate_dequant_kernel, kInfThreads, 0);
    max_grid = std::max(1, sms * std::max(per, 1));
  }
  const uint32_t grid = std::min<uint32_t>(items, uint32_t(max_grid));
  inflate_dequant_kernel<<<grid, kInfThreads, 0, st>>>(a);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

// Batched codec: any number of sections; jobs[j].chunk0 = first global chunk of
// job j (ascending), a binary search maps a chunk to its job.
__global__ void __launch_bounds__(kInfThreads, 16) inflate_batch_kernel(const InflateJob *jobs, int32_t njobs,
                                                                   uint32_t total, int32_t *err) {
  __shared__ FastShared S;
  for (uint32_t b = blockIdx.x; b < total; b += gridDim.x) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (jobs[mid].chunk0 <= b) lo = mid;
      else hi = mid - 1;
    }
    const InflateJob jb = jobs[lo];
    inflate_chunk(S, jb.section, jb.sec_len, jb.n_out, jb.nch, b - jb.chunk0, jb.out, jb.err ? jb.err : err);
    __syncthreads();
  }
}

kvtc_status launch_inflate_batch(const InflateJob *jobs_dev, int32_t njobs, uint32_t total_chunks, int32_t *err,
                                 cudaStream_t st) {
  if (njobs == 0 || total_chunks == 0) return KVTC_OK;
  KVTC_MAX_CARVEOUT(inflate_batch_kernel);
  inflate_batch_kernel<<<total_chunks, kInfThreads, 0, st>>>(jobs_dev, njobs, total_chunks, err);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_inflate_sections(const uint8_t *sec0, uint64_t len0, uint64_t n0, uint32_t nch0, uint8_t *out0,
                                    const uint8_t *sec1, uint64_t len1, uint64_t n1, uint32_t nch1, uint8_t *out1,
                                    int32_t *err, cudaStream_t st, int32_t max_ctas) {
  InflateJobs J;
  J.sec[0] = sec0;
  J.sec[1] = sec1;
  J.sec_len[0] = len0;
  J.sec_len[1] = len1;
  J.n_out[0] = n0;
  J.n_out[1] = n1;
  J.nch[0] = nch0;
  J.nch[1] = nch1;
  J.out[0] = out0;
  J.out[1] = out1;
  if (nch0 + nch1 == 0) return KVTC_OK;
  const uint32_t grid = max_ctas > 0 ? std::min<uint32_t>(nch0 + nch1, uint32_t(max_ctas)) : nch0 + nch1;
  KVTC_MAX_CARVEOUT(inflate_fast_kernel);
  inflate_fast_kernel<<<grid, kInfThreads, 0, st>>>(J, err);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

kvtc_status launch_inflate_section(const uint8_t *sec, uint64_t len, uint64_t n_out, uint32_t nchunks, uint8_t *out,
                                   int32_t *err, cudaStream_t st, int32_t max_ctas) {
  return launch_inflate_sections(sec, len, n_out, nchunks, out, nullptr, 0, 0, 0, nullptr, err, st, max_ctas);
}

// Validates a section header (host copy) against the expected payload size.
kvtc_status check_section_header(const void *hdr_host, size_t len, size_t n_out, uint32_t *nchunks) {
  const SectionHeader *h = static_cast<const SectionHeader *>(hdr_host);
  if (h->magic != kSectionMagic || h->version != kSectionVersion || h->section_bytes > len || h->raw_bytes != n_out ||
      h->nseg != kNSeg || h->chunk_bytes == 0 || h->nchunks != (n_out + h->chunk_bytes - 1) / h->chunk_bytes) {
    set_error("corrupt entropy section header");
    return KVTC_E_CORRUPT;
  }
  *nchunks = h->nchunks;
  return KVTC_OK;
}

// ---- generic sequential inflater (one thread per stream)
__constant__ uint16_t c_lbase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                     31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dbase[30] = {1,   2,   3,   4,   5,   7,    9,    13,   17,   25,   33,   49,   65,    97,    129,
                                     193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

__global__ void inflate_raw_kernel(const uint8_t *in, const int64_t *in_off, const int64_t *in_len, int32_t nstreams,
                                   uint8_t *out, const int64_t *out_off, const int64_t *out_len, int32_t *status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nstreams) return;
  BitReader br{in + in_off[i], uint64_t(in_len[i]), 0};
  uint8_t *o = out + out_off[i];
  const uint64_t cap = uint64_t(out_len[i]);
  uint64_t w = 0;
  Huff lit, dist;
  uint8_t lens[320];
  int last = 0, st = 0;
  do {
    last = int(br.bits(1));
    const int type = int(br.bits(2));
    if (type == 0) {
      br.pos = (br.pos + 7) & ~7ull;
      const uint32_t len = br.bits(16), nlen = br.bits(16);
      if ((len ^ 0xFFFFu) != nlen) { st = -2; break; }
      if ((br.pos >> 3) + len > br.nbytes || w + len > cap) { st = -2; break; }
      for (uint32_t k = 0; k < len; ++k) o[w++] = br.p[(br.pos >> 3) + k];
      br.pos += 8ull * len;
      continue;
    }
    int nlen = 288, ndist = 30;
    if (type == 1) {
      for (int s = 0; s < 144; ++s) lens[s] = 8;
      for (int s = 144; s < 256; ++s) lens[s] = 9;
      for (int s = 256; s < 280; ++s) lens[s] = 7;
      for (int s = 280; s < 288; ++s) lens[s] = 8;
      for (int s = 0; s < 30; ++s) lens[288 + s] = 5;
      huff_build(lit, lens, 288);
      huff_build(dist, lens + 288, 30);
    } else if (type == 2) {
      st = parse_dynamic(br, lens, nlen, ndist);
      if (st) break;
      if (huff_build(lit, lens, nlen) < 0 || huff_build(dist, lens + nlen, ndist) < 0) { st = -4; break; }
    } else {
      st = -1;
      break;
    }
    for (;;) {
      int sym = huff_decode(br, lit);
      if (sym < 0) { st = sym; break; }
      if (sym < 256) {
        if (w >= cap) { st = -8; break; }
        o[w++] = uint8_t(sym);
      } else if (sym == 256) {
        break;
      } else {
        sym -= 257;
        if (sym >= 29) { st = -10; break; }
        const uint32_t len = c_lbase[sym] + br.bits(c_lext[sym]);
        const int ds = huff_decode(br, dist);
        if (ds < 0 || ds >= 30) { st = -11; break; }
        const uint32_t dd = c_dbase[ds] + br.bits(c_dext[ds]);
        if (dd > w || w + len > cap) { st = -12; break; }
        for (uint32_t k = 0; k < len; ++k, ++w) o[w] = o[w - dd];
      }
    }
    if (st) break;
    if (br.pos > 8 * br.nbytes) { st = -13; break; }
  } while (!last);
  if (!st && w != cap) st = -14;
  status[i] = st;
}

kvtc_status launch_inflate_raw(const uint8_t *in, const int64_t *in_off, const int64_t *in_len, int32_t n,
                               uint8_t *out, const int64_t *out_off, const int64_t *out_len, int32_t *status,
                               cudaStream_t st) {
  if (n == 0) return KVTC_OK;
  inflate_raw_kernel<<<unsigned(ceil_div(n, 32)), 32, 0, st>>>(in, in_off, in_len, n, out, out_off, out_len, status);
  KVTC_LAUNCH_CHECK();
  return KVTC_OK;
}

}  // namespace kvtc
