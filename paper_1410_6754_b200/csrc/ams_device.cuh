// Device-side building blocks shared by the level and final-sort kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ams_b200.h"

namespace ams {

// Level kernel geometry: a tile is kThreads x kItems consecutive keys of one
// segment (PE); a chunk is up to kChunkTiles consecutive tiles of one
// segment, processed by one CTA of the histogram kernel.
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = AMS_TILE / kThreads;  // 16
constexpr int kTile = AMS_TILE;              // 4096
constexpr int kChunkTiles = 16;
constexpr int kChunk = kTile * kChunkTiles;  // keys per histogram / scatter CTA
static_assert(kItems * kThreads == kTile, "tile geometry");

// Tree classifier blob (one per group) in global memory: header, sorted
// splitter keys and positions, and a key-range LUT whose cells hold
// (first splitter index | splitter count << 16).
constexpr int kLutExtraBits = 6;  // LUT cells per splitter = 2^6 (2^5: 1.129 -> 1.161 ms for config 2's histograms)
constexpr int kMaxSpl = AMS_MAX_BUCKETS;  // room for nb-1 <= 4095 splitters
constexpr int kMaxLutBits = 13;
constexpr int kMaxCells = 1 << kMaxLutBits;
constexpr size_t kBlobKeys = 64;
constexpr size_t kBlobPos = kBlobKeys + sizeof(uint64_t) * kMaxSpl;
constexpr size_t kBlobLut = kBlobPos + sizeof(uint32_t) * kMaxSpl;
constexpr size_t kBlobStride = 128 * 1024;
static_assert(kBlobLut + 4 * (size_t)(kMaxCells + 1) <= kBlobStride, "blob layout");

struct ClsHeader {
  uint64_t lo, hi;   // first / last splitter key
  uint32_t nspl;     // number of splitters = buckets - 1
  uint32_t shift;    // LUT cell of key k: (k - lo) >> shift, clamped
  uint32_t ncells;   // LUT entries
  uint32_t max_inside;  // most splitters in one LUT cell (> 8: duplicate-heavy splitters)
};

// Digit classifier (final-sort partitions): digit = (k-lo) * nb / (range+1)
// via a 64-bit multiply-high by mult ~ 2^64 nb / (range+1), so all nb
// digits cover the key range evenly; mult == 0 means range < nb and the
// digit is k - lo itself (one key value per digit).
struct DigitCls {
  uint64_t lo, hi;
  uint64_t mult;
  uint32_t nb;
  uint32_t pad;
  // Cell-relative map for the cell sort (k_final_ranges): cell c starts at or
  // after lo + c * q; sub = ((key - that) >> sh) * m32 >> 32 (m32 == 0: none).
  uint64_t q;
  uint32_t m32, sh;
};

// Multiplier of the scaled digit above.  Any value keeps digits monotone in
// the key (what correctness needs); double precision only affects balance.
__host__ __device__ inline uint64_t digit_mult(uint64_t range, uint32_t nb) {
  if (range < (uint64_t)nb) return 0;
  const double m = (double)nb * 18446744073709551616.0 / ((double)range + 1.0);
  return m >= 18446744073709549568.0 ? 0xFFFFFFFFFFFFF800ULL : (uint64_t)m;
}

// Final-sort overflow record: a cell too large for the shared-memory sort.
struct OverflowRec {
  uint64_t off, count, lo, hi;
  uint64_t out;  // output index of the cell (== off except for fixed-capacity cells)
};

__host__ __device__ inline int bit_length64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return x ? 64 - __clzll((long long)x) : 0;
#else
  return x ? 64 - __builtin_clzll(x) : 0;
#endif
}

// LUT of ~64 cells per splitter: most keys see a cell with no splitter or
// one, so classification is one LUT load plus at most one compare.
__host__ __device__ inline int lut_bits_for(int nspl) {
  int lg = bit_length64((uint64_t)nspl);  // ~ceil(log2(nspl+1))
  int b = lg + kLutExtraBits;
  return b < 4 ? 4 : (b > kMaxLutBits ? kMaxLutBits : b);
}

// ---- order-preserving key maps -------------------------------------------
template <int KIND>
__device__ __forceinline__ uint64_t to_ordered(uint64_t x) {
  if (KIND == AMS_KEY_I64) return x ^ 0x8000000000000000ULL;
  if (KIND == AMS_KEY_F64) return (x >> 63) ? ~x : (x | 0x8000000000000000ULL);
  return x;
}
template <int KIND>
__device__ __forceinline__ uint64_t from_ordered(uint64_t x) {
  if (KIND == AMS_KEY_I64) return x ^ 0x8000000000000000ULL;
  if (KIND == AMS_KEY_F64) return (x >> 63) ? (x & 0x7fffffffffffffffULL) : ~x;
  return x;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint64_t ldg_stream(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// ---- tree classifier in shared memory ------------------------------------
// Shared-memory loads by 32-bit shared address (a generic pointer kept in a
// struct compiles to generic LD.E; these stay LDS).
// The "memory" clobber keeps them after the __syncthreads() that publishes
// the tree (the compiler may otherwise hoist them above the barrier).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}

struct TreeView {
  ClsHeader h;
  uint32_t skeys, spos, lut;  // shared addresses

  // Bucket of (key, pos) = number of splitters strictly below it under the
  // (key, position) order — bisect_left on tie-broken elements
  // (ams.py:201-211).  Splitters before the key's LUT cell
  // are all below it, those after all above; the few inside the cell
  // (sorted) are compared one by one.
  // hint: a likely answer (the thread's previous bucket); checked only in
  // the rare many-splitter cells, where consecutive keys of duplicate-heavy
  // inputs keep landing in the same bucket.
  __device__ __forceinline__ uint32_t classify(uint64_t key, uint32_t pos,
                                               uint32_t hint = 0xFFFFFFFFu) const {
    if (h.nspl == 0) return 0;
    uint64_t c = (key - h.lo) >> h.shift;
    c = key < h.lo ? 0 : (c >= h.ncells ? h.ncells - 1 : c);
    const uint32_t rec = lds_u32(lut + 4 * (uint32_t)c);
    uint32_t b = rec & 0xFFFFu;
    const uint32_t inside = rec >> 16;
    if (inside == 0) return b;
    // Usually one splitter shares the cell: one compare; more are rare.
    const uint64_t sk = lds_u64(skeys + 8 * b);
    if (!(sk < key || (sk == key && lds_u32(spos + 4 * b) < pos))) return b;
    const uint32_t end = b + inside;
    if (inside <= 8) {
      for (++b; b < end; ++b) {
        const uint64_t sk2 = lds_u64(skeys + 8 * b);
        if (!(sk2 < key || (sk2 == key && lds_u32(spos + 4 * b) < pos))) break;
      }
      return b;
    }
    // Many splitters in one cell (duplicate-heavy keys: runs of equal
    // splitter keys told apart by position): the hint if it brackets
    // (key, pos), else the lower bound by (key, pos).
    if (hint > b && hint <= end) {
      const uint64_t pk = lds_u64(skeys + 8 * (hint - 1));
      const bool above_prev = pk < key || (pk == key && lds_u32(spos + 4 * (hint - 1)) < pos);
      bool below_next = true;
      if (hint < end) {
        const uint64_t nk = lds_u64(skeys + 8 * hint);
        below_next = !(nk < key || (nk == key && lds_u32(spos + 4 * hint) < pos));
      }
      if (above_prev && below_next) return hint;
    }
    uint32_t lo = b + 1, hi = end;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint64_t sk2 = lds_u64(skeys + 8 * mid);
      if (sk2 < key || (sk2 == key && lds_u32(spos + 4 * mid) < pos)) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
};

// Shared-memory bytes a tree view needs.
__host__ __device__ inline size_t tree_smem_bytes(int nspl_cap, int cells_cap) {
  size_t b = 64 + (size_t)nspl_cap * 12 + (size_t)cells_cap * 4;
  return (b + 15) & ~(size_t)15;
}

// Cooperatively copy blob -> smem and return the view.
__device__ inline TreeView load_tree(const uint8_t* blob, uint8_t* smem, int nspl_cap) {
  TreeView v;
  const ClsHeader* gh = reinterpret_cast<const ClsHeader*>(blob);
  v.h = *gh;
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem + 64);
  uint32_t* sp = reinterpret_cast<uint32_t*>(smem + 64 + (size_t)nspl_cap * 8);
  uint32_t* lu = reinterpret_cast<uint32_t*>(smem + 64 + (size_t)nspl_cap * 12);
  const uint64_t* gk = reinterpret_cast<const uint64_t*>(blob + kBlobKeys);
  const uint32_t* gp = reinterpret_cast<const uint32_t*>(blob + kBlobPos);
  const uint32_t* gl = reinterpret_cast<const uint32_t*>(blob + kBlobLut);
  for (uint32_t i = threadIdx.x; i < v.h.nspl; i += blockDim.x) { sk[i] = gk[i]; sp[i] = gp[i]; }
  if (v.h.nspl)
    for (uint32_t i = threadIdx.x; i < v.h.ncells; i += blockDim.x) lu[i] = gl[i];
  v.skeys = (uint32_t)__cvta_generic_to_shared(sk);
  v.spos = (uint32_t)__cvta_generic_to_shared(sp);
  v.lut = (uint32_t)__cvta_generic_to_shared(lu);
  return v;
}

struct DigitView {
  DigitCls c;
  __device__ __forceinline__ uint32_t classify(uint64_t key, uint32_t) const {
    if (key <= c.lo) return 0;
    const uint64_t x = key - c.lo;
    const uint64_t d = c.mult ? __umul64hi(x, c.mult) : x;
    return d >= c.nb ? c.nb - 1 : (uint32_t)d;
  }
};

// ---- block-wide exclusive scans in shared memory ----------------------------
// Each warp owns a contiguous range of the array and walks it 32 entries at
// a time (consecutive lanes -> consecutive words: no bank conflicts), with
// shuffle scans inside each 32-entry block.  `scratch` needs NT/32 + 1 words.
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Exclusive scan of the per-warp totals in scratch[0..NW); returns the total.
template <int NT>
__device__ __forceinline__ uint32_t scan_warp_totals(uint32_t* scratch) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = lane < NW ? scratch[lane] : 0;
    const uint32_t s = warp_incl_scan(v);
    if (lane < NW) scratch[lane] = s - v;
    if (lane == NW - 1) scratch[NW] = s;
  }
  __syncthreads();
  return scratch[NW];
}

// The same with ONE barrier: every warp's last lane has stored its inclusive
// total in scratch[w]; returns the sum of the totals of the warps below this
// one (a few broadcast loads instead of a second barrier).  scratch must not
// be rewritten before every thread has passed a later barrier.
template <int NT>
__device__ __forceinline__ uint32_t warp_base_direct(const uint32_t* scratch) {
  constexpr int NW = NT / 32;
  const int w = threadIdx.x >> 5;
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) s += ww < w ? scratch[ww] : 0u;
  return s;
}

// VAL(i) = value of entry i (u32 array or packed u16 pairs).
template <int NT>
__device__ inline uint32_t block_excl_scan(uint32_t* a, int n, uint32_t* scratch) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (((n + NW - 1) / NW) + 31) & ~31;
  const int beg = w * per;
  const int end = beg + per < n ? beg + per : n;
  uint32_t sum = 0;
  for (int i = beg + lane; i < end; i += 32) sum += a[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) scratch[w] = sum;
  const uint32_t total = scan_warp_totals<NT>(scratch);
  uint32_t carry = scratch[w];
  for (int i0 = beg; i0 < end; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t v = i < end ? a[i] : 0;
    const uint32_t inc = warp_incl_scan(v);
    if (i < end) a[i] = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncthreads();
  return total;
}

// Packed 16-bit counters (two per word, low half first), scanned in place.
template <int NT>
__device__ inline void block_excl_scan_u16(uint32_t* wv, int nwords, uint32_t* scratch) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (((nwords + NW - 1) / NW) + 31) & ~31;
  const int beg = w * per;
  const int end = beg + per < nwords ? beg + per : nwords;
  uint32_t sum = 0;
  for (int i = beg + lane; i < end; i += 32) { const uint32_t v = wv[i]; sum += (v & 0xFFFFu) + (v >> 16); }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) scratch[w] = sum;
  scan_warp_totals<NT>(scratch);
  uint32_t carry = scratch[w];
  for (int i0 = beg; i0 < end; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t v = i < end ? wv[i] : 0;
    const uint32_t pair = (v & 0xFFFFu) + (v >> 16);
    const uint32_t inc = warp_incl_scan(pair);
    if (i < end) {
      const uint32_t lo = carry + inc - pair;
      wv[i] = lo | ((lo + (v & 0xFFFFu)) << 16);
    }
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncthreads();
}


// ---- helpers shared by the kernel translation units -------------------------
// Unstable scatters (k_scatter_u, k_scatter_fixed): 16 warps x 8 keys per tile, 2 CTAs per SM.
constexpr int kThreadsU = 512;
constexpr int kItemsU = kTile / kThreadsU;
constexpr int kWarpsU = kThreadsU / 32;
// Sub-buckets of the cell sort: two per key of cell capacity.
constexpr int kCellSubBuckets = 2 * AMS_SMEM_SORT_CAP;
// ... and of the fixed-capacity cells (their refined digit, k_bucket_ranges).
constexpr int kFxSubBuckets = 2 * AMS_FX_CAP;  // (one per key of capacity: 1.345 -> 1.467 ms)

__device__ __forceinline__ int upper_bound_u64(const uint64_t* a, int n, uint64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

constexpr uint32_t kInvalid = 0xFFFFFFFFu;

// Ranking modes of the scatter.
constexpr int kClsTree = 0, kClsDigit = 1, kClsIds = 2;
constexpr int kClsTreeTags = 3;  // tree, tie-break by the carried origin tag (the values)
constexpr int kClsIds16 = 4;     // 16-bit bucket ids stored by the histogram pass (> 256 buckets)
constexpr int kRankWarp = 0;     // stable, one bucket-counter array per warp
constexpr int kRankSerial = 1;   // stable, one shared array, warps take turns
constexpr int kRankAtomic = 2;   // unstable (keys only, order inside a run is free)

// Stable rank of this lane's item among the warp's items in the same bucket
// (lower lanes first), plus the per-warp bucket counter update.  Peers are
// found with one ballot per bucket-id bit (and one for validity unless the
// whole warp is valid): __match_any_sync costs ~57 SM-cycles per warp on
// B200 (tools/microbench.cu).  NBITS is a compile-time width so the vote
// chain unrolls to ~3 instructions per bit.
template <int NBITS>
__device__ __forceinline__ uint32_t warp_stable_rank(uint32_t b, int lane, uint32_t lt,
                                                     uint32_t* whw, bool all_valid) {
  const bool valid = b != kInvalid;
  uint32_t peers = 0xffffffffu;
  if (!all_valid) {
    const uint32_t v = __ballot_sync(0xffffffffu, valid);
    peers = valid ? v : ~v;
  }
#pragma unroll
  for (int bit = 0; bit < NBITS; ++bit) {
    const uint32_t x = (b >> bit) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, x);
    peers &= ~(bal ^ (0u - x));  // lanes whose bit equals mine
  }
  uint32_t cnt = 0;
  if (valid) cnt = whw[b];
  __syncwarp();
  if (valid && lane == __ffs(peers) - 1) whw[b] = cnt + __popc(peers);
  __syncwarp();
  return cnt + __popc(peers & lt);
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---- 1-D bulk copies (TMA engine) with an mbarrier -------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
// Arm `bar` for `bytes` and copy them global -> shared (16-byte aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sdst);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes)
               : "memory");
  if (bytes)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(d), "l"(gsrc), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}

}  // namespace ams

#define AMS_KIND_DISPATCH(kind, K, ...)          \
  switch (kind) {                                \
    case AMS_KEY_I64: { constexpr int K = AMS_KEY_I64; __VA_ARGS__; } break; \
    case AMS_KEY_F64: { constexpr int K = AMS_KEY_F64; __VA_ARGS__; } break; \
    default: { constexpr int K = AMS_KEY_U64; __VA_ARGS__; } break;          \
  }

