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

// Tree classifier blob (one per group) in global memory.
constexpr int kMaxSpl = AMS_MAX_BUCKETS;  // room for nb-1 <= 4095 splitters
constexpr int kMaxLutBits = 12;
constexpr int kMaxCells = 1 << kMaxLutBits;
constexpr size_t kBlobKeys = 64;
constexpr size_t kBlobPos = kBlobKeys + sizeof(uint64_t) * kMaxSpl;
constexpr size_t kBlobLut = kBlobPos + sizeof(uint32_t) * kMaxSpl;
constexpr size_t kBlobStride = 64 * 1024;
static_assert(kBlobLut + 2 * (kMaxCells + 1) <= kBlobStride, "blob layout");

struct ClsHeader {
  uint64_t lo, hi;   // first / last splitter key
  uint32_t nspl;     // number of splitters = buckets - 1
  uint32_t shift;    // LUT cell of key k: (k - lo) >> shift
  uint32_t ncells;   // LUT has ncells + 1 entries
  uint32_t pad;
};

// Digit classifier (final-sort partitions): bucket = clamp((k-lo)>>shift).
struct DigitCls {
  uint64_t lo, hi;
  uint32_t shift;
  uint32_t nb;
};

// Final-sort overflow record: a cell too large for the shared-memory sort.
struct OverflowRec {
  uint64_t off, count, lo, hi;
};

__host__ __device__ inline int bit_length64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return x ? 64 - __clzll((long long)x) : 0;
#else
  return x ? 64 - __builtin_clzll(x) : 0;
#endif
}

__host__ __device__ inline int lut_bits_for(int nspl) {
  int lg = bit_length64((uint64_t)nspl);  // ~ceil(log2(nspl+1))
  int b = lg + 3;
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
struct TreeView {
  ClsHeader h;
  const uint64_t* skeys;
  const uint32_t* spos;
  const uint16_t* lut;

  // Bucket of (key, pos) = number of splitters strictly below it under the
  // (key, position) order — bisect_left on tie-broken elements
  // (ams.py:201-211).  The LUT narrows the search to the
  // splitters whose key shares the element's cell.
  __device__ __forceinline__ uint32_t classify(uint64_t key, uint32_t pos) const {
    if (h.nspl == 0 || key < h.lo) return 0;
    if (key > h.hi) return h.nspl;
    const uint32_t cell = (uint32_t)((key - h.lo) >> h.shift);
    uint32_t l = lut[cell], r = lut[cell + 1];
    while (l < r) {
      const uint32_t m = (l + r) >> 1;
      const uint64_t sk = skeys[m];
      const bool lt = sk < key || (sk == key && spos[m] < pos);
      l = lt ? m + 1 : l;
      r = lt ? r : m;
    }
    return l;
  }
};

// Shared-memory bytes a tree view needs.
__host__ __device__ inline size_t tree_smem_bytes(int nspl_cap, int cells_cap) {
  size_t b = 64 + (size_t)nspl_cap * 12 + (size_t)(cells_cap + 1) * 2;
  return (b + 15) & ~(size_t)15;
}

// Cooperatively copy blob -> smem and return the view.
__device__ inline TreeView load_tree(const uint8_t* blob, uint8_t* smem, int nspl_cap) {
  TreeView v;
  const ClsHeader* gh = reinterpret_cast<const ClsHeader*>(blob);
  v.h = *gh;
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem + 64);
  uint32_t* sp = reinterpret_cast<uint32_t*>(smem + 64 + (size_t)nspl_cap * 8);
  uint16_t* lu = reinterpret_cast<uint16_t*>(smem + 64 + (size_t)nspl_cap * 12);
  const uint64_t* gk = reinterpret_cast<const uint64_t*>(blob + kBlobKeys);
  const uint32_t* gp = reinterpret_cast<const uint32_t*>(blob + kBlobPos);
  const uint16_t* gl = reinterpret_cast<const uint16_t*>(blob + kBlobLut);
  for (uint32_t i = threadIdx.x; i < v.h.nspl; i += blockDim.x) { sk[i] = gk[i]; sp[i] = gp[i]; }
  if (v.h.nspl)
    for (uint32_t i = threadIdx.x; i <= v.h.ncells; i += blockDim.x) lu[i] = gl[i];
  v.skeys = sk; v.spos = sp; v.lut = lu;
  return v;
}

struct DigitView {
  DigitCls c;
  __device__ __forceinline__ uint32_t classify(uint64_t key, uint32_t) const {
    if (key <= c.lo) return 0;
    const uint64_t d = (key - c.lo) >> c.shift;
    return d >= c.nb ? c.nb - 1 : (uint32_t)d;
  }
};

// ---- block-wide exclusive scan of a shared u32 array (n <= 64K) ----------
// Returns the total; `scratch` needs NT/32 + 1 words.
template <int NT>
__device__ inline uint32_t block_excl_scan(uint32_t* a, int n, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per = (n + NT - 1) / NT;
  const int beg = threadIdx.x * per;
  const int end = beg + per < n ? beg + per : n;
  uint32_t sum = 0;
  for (int i = beg; i < end; ++i) sum += a[i];
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t v = lane < NT / 32 ? scratch[lane] : 0;
    uint32_t s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) scratch[lane] = s - v;
    if (lane == NT / 32 - 1) scratch[NT / 32] = s;
  }
  __syncthreads();
  uint32_t run = scratch[w] + x - sum;
  for (int i = beg; i < end; ++i) { uint32_t t = a[i]; a[i] = run; run += t; }
  const uint32_t total = scratch[NT / 32];
  __syncthreads();
  return total;
}

}  // namespace ams
