// Final local sort (sorted(), ams.py:310-312): fixed-capacity digit partition
// and the CTA-local shared-memory sorts (K8, K9).
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ams_device.cuh"
#include "launch.h"

namespace ams {

namespace {
// Geometry of the fixed-capacity partition: 2048-key tiles, 256 threads, 4
// CTAs per SM (4096-key tiles on 512 threads at 2 CTAs per SM: 1.202 ->
// 1.154 ms at config 2 — fewer warps per barrier, more CTAs to interleave;
// 1024-key tiles: 1.36 ms, profiles/r02t_ab_fixed_tile.txt).
constexpr int kFTile = 2048;
constexpr int kFItems = 8;
constexpr int kFThreads = kFTile / kFItems;
constexpr int kFWarps = kFThreads / 32;
constexpr int kFCtas = 2 * 4096 / kFTile;
static_assert(kTile % kFTile == 0, "chunks are whole tiles of both kinds");

// Fixed-capacity digit partition (keys only, the final sort of a bucket-major
// last level): segments are the last level's buckets, each split into nb_s
// digit cells of capacity AMS_FX_CAP in `dst` (cell ci at dst[ci * AMS_FX_CAP]).
// No histogram pass: every (tile, digit) run reserves its room with one
// global atomic on the cell's fill counter, so a cell's keys land in any
// order (only membership matters: F7).  A cell that would exceed its
// capacity flags its segment; the host re-partitions such segments exactly
// from `src`, which this kernel does not modify.
template <int KIND>
__global__ void __launch_bounds__(kFThreads, kFCtas)
    k_scatter_fixed(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, SegMeta m,
                    const DigitCls* __restrict__ dcls, const uint32_t* __restrict__ cell0,
                    uint32_t* __restrict__ fill, uint32_t* __restrict__ seg_ovf) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ uint32_t s_scan[kFWarps + 1];
  __shared__ uint32_t s_clip;
  __shared__ __align__(8) uint64_t s_bar[2];
  constexpr int kBuf = kFTile + 2;
  uint64_t* buf0 = reinterpret_cast<uint64_t*>(smem);
  const int tid = threadIdx.x;
  const uint64_t c = blockIdx.x;
  if (tid == 0) {
    s_seg = upper_bound_u64(m.chunk_prefix, m.nseg + 1, c) - 1;
    s_clip = 0;
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int s = s_seg;
  const DigitCls dc = dcls[s];
  const int nb = (int)dc.nb;
  const uint64_t dlo = dc.lo;
  const uint32_t dsh = dc.sh, dm = dc.m32, dmax = dc.nb - 1;
  const int per = (nb + kFThreads - 1) / kFThreads | 1;
  const int nbp = per * kFThreads;
  int64_t* adj = reinterpret_cast<int64_t*>(buf0 + 2 * kBuf);  // this tile: dst index - slot
  uint32_t* cnt = reinterpret_cast<uint32_t*>(adj + nbp);       // counts, then tile starts
  int32_t* lim = reinterpret_cast<int32_t*>(cnt + nbp);         // writable keys of the run
  uint16_t* bkt = reinterpret_cast<uint16_t*>(lim + nbp);
  const uint64_t seg_off = m.off[s];
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)m.chunk;
  const uint64_t last = min(first + (uint64_t)m.chunk, m.len[s]);
  const int ntiles = (int)((last - first + kFTile - 1) / kFTile);
  const uint64_t cbase = cell0[s];
  // Tile t = keys [base, base + tc); the copy starts at the 16-byte boundary
  // base - h and is rounded up to whole 16-byte units (the source is the
  // last level's work buffer, padded by two keys), so key e of the tile sits
  // at buf[e + h].
  auto issue = [&](int t) {
    const uint64_t base = seg_off + first + (uint64_t)t * kFTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kFTile, last - first - (uint64_t)t * kFTile);
    const uint32_t h = (uint32_t)(base & 1);
    bulk_load(buf0 + (t & 1) * kBuf, src + (base - h), ((tc + h + 1) & ~1u) * 8, &s_bar[t & 1]);
  };
  if (tid == 0) issue(0);
  for (int b = tid; b < nbp; b += kFThreads) cnt[b] = 0;
  const int w = tid >> 5, lane = tid & 31;
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    uint64_t* buf = buf0 + (t & 1) * kBuf;
    const uint64_t base = seg_off + first + (uint64_t)t * kFTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kFTile, last - first - (uint64_t)t * kFTile);
    const uint32_t h = (uint32_t)(base & 1);
    if (tid == 0 && t + 1 < ntiles) {
      fence_proxy_async();
      issue(t + 1);
    }
    mbar_wait(&s_bar[t & 1], (uint32_t)(t >> 1) & 1u);
    const uint64_t* tb = buf + h;
    uint64_t kr[kFItems];
    uint32_t pk[kFItems];
    auto classify_all = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int i = 0; i < kFItems; ++i) {
        const uint32_t e = w * (kFItems * 32) + i * 32 + lane;
        pk[i] = kInvalid;
        if (FULL || e < tc) {
          const uint64_t key = to_ordered<KIND>(tb[e]);
          const uint64_t x = key - dlo;
          const uint32_t b = dm ? min(__umulhi((uint32_t)(x >> dsh), dm), dmax) : (uint32_t)x;
          kr[i] = key;
          if (FULL && dm == 0) {  // counting cells (few values): one atomic per uniform warp
            const uint32_t b0 = __shfl_sync(0xffffffffu, b, 0);
            if (__all_sync(0xffffffffu, b == b0)) {
              uint32_t base0 = 0;
              if (lane == 0) base0 = atomicAdd(&cnt[b0], 32u);
              pk[i] = (b0 << 16) | (__shfl_sync(0xffffffffu, base0, 0) + lane);
              continue;
            }
          }
          pk[i] = (b << 16) | atomicAdd(&cnt[b], 1u);
        }
      }
    };
    if (tc == (uint32_t)kFTile) classify_all(std::true_type{});
    else classify_all(std::false_type{});
    __syncthreads();
    if (dm == 0) {
      // One key value per cell: only the counts matter (no capacity bound).
      for (int b = tid; b < nbp; b += kFThreads) {
        const uint32_t v = cnt[b];
        if (v) atomicAdd(&fill[cbase + b], v);
        cnt[b] = 0;
      }
      __syncthreads();
      continue;
    }
    {
      const int b0 = tid * per;
      uint32_t sum = 0;
      for (int j = 0; j < per; ++j) sum += cnt[b0 + j];
      const uint32_t inc = warp_incl_scan(sum);
      if (lane == 31) s_scan[w] = inc;
      uint32_t start = warp_base_direct<kFThreads>(s_scan) + inc - sum;
      for (int j = 0; j < per; ++j) {
        const int b = b0 + j;
        const uint32_t v = cnt[b];
        cnt[b] = start;
        if (v) {
          // Reserve this run's room in cell (s, b).
          const uint32_t at = atomicAdd(&fill[cbase + b], v);
          adj[b] = (int64_t)((cbase + b) * (uint64_t)AMS_FX_CAP + at) - (int64_t)start;
          const int32_t room = (int32_t)AMS_FX_CAP - (int32_t)at;
          lim[b] = (int32_t)start + room;  // slots below lim are written
          if ((uint32_t)max(room, 0) < v) {
            s_clip = 1;
            seg_ovf[s] = 1;
          }
        }
        start += v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kFItems; ++i) {
      if (pk[i] != kInvalid) {
        const uint32_t b = pk[i] >> 16;
        const uint32_t slot = cnt[b] + (pk[i] & 0xFFFFu);
        buf[slot] = kr[i];
        bkt[slot] = (uint16_t)b;
      }
    }
    __syncthreads();
    if (!s_clip) {
      for (uint32_t j = tid; j < tc; j += kFThreads) dst[adj[bkt[j]] + j] = buf[j];
    } else {
      for (uint32_t j = tid; j < tc; j += kFThreads) {
        const uint32_t b = bkt[j];
        if ((int32_t)j < lim[b]) dst[adj[b] + j] = buf[j];
      }
    }
    for (int j = 0; j < per; ++j) cnt[tid * per + j] = 0;
    // This thread's generic-proxy writes into the tile buffer (the in-place
    // permutation) must be ordered before the bulk copy (async proxy) that
    // refills the buffer two tiles on: every writer fences, then the barrier.
    fence_proxy_async();
    __syncthreads();
  }
}

// -------------------------------------------------------------------- K9
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortCap = AMS_SMEM_SORT_CAP;
constexpr int kSortItems = kSortCap / kSortThreads;  // per-warp iterations
constexpr int kRadix = 256;

__device__ __forceinline__ void block_minmax(uint64_t& mn, uint64_t& mx, uint64_t* s2) {
  // s2: 2*kSortWarps scratch
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, (uint64_t)__shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, (uint64_t)__shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s2[w] = mn; s2[kSortWarps + w] = mx; }
  __syncthreads();
  mn = s2[0]; mx = s2[kSortWarps];
  for (int i = 1; i < kSortWarps; ++i) { mn = min(mn, s2[i]); mx = max(mx, s2[kSortWarps + i]); }
  __syncthreads();
}

__device__ __forceinline__ void cell_of(const CellSource& cs, uint64_t cid, uint64_t& off,
                                        uint64_t& count, uint64_t& oo) {
  if (cs.mode == 0) {
    off = cs.cell_base[cid];
    count = cs.cell_cnt[cid];
    oo = off;
  } else if (cs.mode == 1) {
    off = cs.seg_off[cid];
    count = cs.seg_len[cid];
    oo = off;
  } else if (cs.mode == 2) {
    if (cs.nrecs && cid >= *cs.nrecs) { off = 0; count = 0; oo = 0; return; }
    off = cs.recs[cid].off;
    count = cs.recs[cid].count;
    oo = cs.recs[cid].out;
  } else {  // fixed-capacity cells: source slot cid, output base from k_fixed_cells
    off = cid * (uint64_t)AMS_FX_CAP;
    count = cs.cell_cnt[cid];
    oo = cs.cell_base[cid];
  }
}

// Cells too big for shared memory: copy when they hold one key value,
// otherwise record them (with their exact key range) for another
// partition round.  Returns true when the cell was handled here.
template <int KIND_OUT, bool VALS>
__device__ bool big_cell(const uint64_t* __restrict__ src, const uint64_t* __restrict__ src_vals,
                         uint64_t* __restrict__ out, uint64_t* __restrict__ out_vals, uint64_t off,
                         uint64_t oo, uint64_t count, OverflowRec* ovf, unsigned int* ovf_count,
                         uint64_t* s_mm) {
  if (count <= (uint64_t)kSortCap) return false;
  uint64_t mn = ~0ULL, mx = 0;
  for (uint64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const uint64_t k = src[off + i];
    mn = min(mn, k); mx = max(mx, k);
  }
  block_minmax(mn, mx, s_mm);
  if (mn == mx) {
    const uint64_t ko = from_ordered<KIND_OUT>(mn);
    for (uint64_t i = threadIdx.x; i < count; i += blockDim.x) {
      out[oo + i] = ko;
      if constexpr (VALS) out_vals[oo + i] = src_vals[off + i];
    }
  } else if (threadIdx.x == 0) {
    const unsigned int slot = atomicAdd(ovf_count, 1u);
    OverflowRec r; r.off = off; r.count = count; r.lo = mn; r.hi = mx; r.out = oo;
    ovf[slot] = r;
  }
  return true;
}

// Fallback for cells whose keys cluster (a sub-bucket of the counting sort
// got too big): LSD radix sort over the bits that vary inside the cell
// (key - min), 8 bits per pass, each pass a stable counting sort with
// warp ranks — stable end to end.
template <int KIND_OUT, bool VALS>
__global__ void __launch_bounds__(kSortThreads, 1)
    k_smem_sort_lsd(const uint64_t* __restrict__ src, const uint64_t* __restrict__ src_vals,
                    uint64_t* __restrict__ out, uint64_t* __restrict__ out_vals, CellSource cs) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t s_mm[2 * kSortWarps];
  __shared__ uint32_t s_scan[kSortWarps + 1];
  uint64_t* kA = reinterpret_cast<uint64_t*>(smem);
  uint64_t* kB = kA + kSortCap;
  uint16_t* iA = reinterpret_cast<uint16_t*>(kB + kSortCap);
  uint16_t* iB = iA + kSortCap;
  uint32_t* wh = reinterpret_cast<uint32_t*>(iB + kSortCap);  // [kSortWarps][kRadix]
  uint32_t* btot = wh + kSortWarps * kRadix;

  uint64_t off, count, oo;
  cell_of(cs, blockIdx.x, off, count, oo);
  if (count == 0 || count > (uint64_t)kSortCap) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t n = (uint32_t)count;
  uint64_t mn = ~0ULL, mx = 0;
  for (uint32_t i = threadIdx.x; i < n; i += kSortThreads) {
    const uint64_t k = src[off + i];
    kA[i] = k;
    iA[i] = (uint16_t)i;
    mn = min(mn, k); mx = max(mx, k);
  }
  block_minmax(mn, mx, s_mm);
  if (mn != mx) {
    const int bits = bit_length64(mx - mn);
    const int passes = (bits + 7) / 8;
    const uint32_t lt = lanemask_lt();
    const uint32_t chunk = ((n + kSortWarps - 1) / kSortWarps + 31) & ~31u;
    uint32_t* whw = wh + w * kRadix;
    for (int p = 0; p < passes; ++p) {
      const int sh = 8 * p;
      for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) wh[i] = 0;
      __syncthreads();
      uint32_t pk[kSortItems];
#pragma unroll
      for (int it = 0; it < kSortItems; ++it) {
        const uint32_t e = w * chunk + it * 32 + lane;
        const bool valid = (it * 32 < (int)chunk) && e < n;
        const uint32_t d = valid ? (uint32_t)(((kA[e] - mn) >> sh) & 255) : kInvalid;
        const uint32_t r = warp_stable_rank<8>(d, lane, lt, whw, false);
        pk[it] = valid ? ((d << 16) | r) : kInvalid;
      }
      __syncthreads();
      for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        uint32_t acc = 0;
#pragma unroll
        for (int ww = 0; ww < kSortWarps; ++ww) {
          const uint32_t v = wh[ww * kRadix + d];
          wh[ww * kRadix + d] = acc;
          acc += v;
        }
        btot[d] = acc;
      }
      __syncthreads();
      block_excl_scan<kSortThreads>(btot, kRadix, s_scan);
#pragma unroll
      for (int it = 0; it < kSortItems; ++it) {
        if (pk[it] != kInvalid) {
          const uint32_t e = w * chunk + it * 32 + lane;
          const uint32_t d = pk[it] >> 16;
          const uint32_t slot = btot[d] + whw[d] + (pk[it] & 0xFFFFu);
          kB[slot] = kA[e];
          iB[slot] = iA[e];
        }
      }
      __syncthreads();
      uint64_t* tk = kA; kA = kB; kB = tk;
      uint16_t* ti = iA; iA = iB; iB = ti;
    }
  }
  for (uint32_t i = threadIdx.x; i < n; i += kSortThreads) {
    out[oo + i] = from_ordered<KIND_OUT>(kA[i]);
    if constexpr (VALS) out_vals[oo + i] = src_vals[off + iA[i]];
  }
}

// One CTA per cell (<= kSortCap keys), keys held in registers:
//  1. one shared atomic per key counts it into one of kSubK sub-buckets (16-
//     bit counters packed in pairs); the atomic's return value is the key's
//     rank inside its sub-bucket, so placement needs no second pass.
//     Digit cells of the final partition use the partition digit refined by
//     kSubK: sub = mulhi(key - lo, mult * kSubK) - digit * kSubK, exact since
//     floor(floor(x*m*K / 2^64) / K) = floor(x*m / 2^64) — no min/max pass.
//     Other cells (and digit cells whose keys cluster) scale (key - min) to
//     2n sub-buckets by the cell's own min/max;
//  2. register-blocked exclusive scan of the counters (thread t owns words
//     [16t, 16t + 16); conflict-free 128-bit accesses), fused with the scan of how many
//     multi-key sub-buckets each thread will queue;
//  3. keys go to slot start(sub-bucket) + rank; the key of rank 1 queues its
//     sub-bucket (one entry per sub-bucket holding >= 2 keys);
//  4. thread per queued sub-bucket: 2 or 3 keys by a compare-exchange
//     network; larger ones (rare) are re-queued and insertion-sorted, in
//     place; ties by input index with values (stable), any order of equal
//     keys without;
//  5. coalesced (16-byte) copy to the output.
// When the range is narrower than 2n each sub-bucket is one key value, so
// keys alone skip step 4.  Cells whose keys cluster (a sub-bucket above
// kRankMax that still needs ordering) go to the LSD fallback list.
constexpr int kRankMax = 64;
constexpr int kSortCtas = 3;  // resident CTAs per SM (register budget)
constexpr int kSubK = kCellSubBuckets;                   // sub-buckets of the refined digit
constexpr int kScanWords = kSubK / 2 / kSortThreads;  // counter words per thread (2 sub-buckets each)
static_assert(kScanWords % 4 == 0, "scan loads 4 words at a time");
constexpr int kScanChunks = kScanWords / 4;  // uint4 chunks per thread (4 at 256 threads, 2 at 512)
static_assert(kScanChunks == 2 || kScanChunks == 4, "swizzle covers 2 or 4 chunks per thread");
constexpr int kLgChunks = kScanChunks == 4 ? 2 : 1;
constexpr int kQueueCap = kSortCap / 2;               // sub-buckets with >= 2 keys

// Counter layout: thread t of the scan owns logical words [16t, 16t + 16) as
// four uint4 chunks (256 threads; [8t, 8t + 8) as two at 512); chunk c is
// stored at chunk c ^ rot(t) of its block, so the 8 threads of one 128-bit
// shared-memory phase hit 32 distinct banks.  Logical word w lives at
// sw_word(w); the u16 counter of sub-bucket s at sw16(s).
__device__ __forceinline__ uint32_t sw_word(uint32_t w) {
  return w ^ (((w >> 5) & (uint32_t)(kScanChunks - 1)) << 2);
}
__device__ __forceinline__ uint32_t sw16(uint32_t s) {
  return s ^ (((s >> 6) & (uint32_t)(kScanChunks - 1)) << 3);
}

template <bool VALS>
__device__ __forceinline__ bool slot_after(uint64_t ka, uint16_t ia, uint64_t kb, uint16_t ib) {
  if constexpr (VALS) return ka > kb || (ka == kb && ia > ib);
  else return ka > kb;
}

template <bool VALS>
__device__ __forceinline__ void cmp_swap(uint64_t& ka, uint16_t& ia, uint64_t& kb, uint16_t& ib) {
  if (slot_after<VALS>(ka, ia, kb, ib)) {
    const uint64_t t = ka; ka = kb; kb = t;
    if constexpr (VALS) { const uint16_t u = ia; ia = ib; ib = u; }
  }
}

template <bool VALS>
__device__ __forceinline__ void insertion_sort(uint64_t* kB, uint16_t* iB, uint32_t b0, uint32_t b1) {
  for (uint32_t a = b0 + 1; a < b1; ++a) {
    const uint64_t ka = kB[a];
    uint16_t ia = 0;
    if constexpr (VALS) ia = iB[a];
    uint32_t d = a;
    while (d > b0) {
      uint16_t ib = 0;
      if constexpr (VALS) ib = iB[d - 1];
      if (!slot_after<VALS>(kB[d - 1], ib, ka, ia)) break;
      kB[d] = kB[d - 1];
      if constexpr (VALS) iB[d] = ib;
      --d;
    }
    kB[d] = ka;
    if constexpr (VALS) iB[d] = ia;
  }
}

template <int KIND_OUT, bool VALS>
__global__ void __launch_bounds__(kSortThreads, kSortCtas)
    k_smem_sort(const uint64_t* __restrict__ src, const uint64_t* __restrict__ src_vals,
                uint64_t* __restrict__ out, uint64_t* __restrict__ out_vals, CellSource cs,
                OverflowRec* __restrict__ ovf, unsigned int* __restrict__ ovf_count,
                OverflowRec* __restrict__ fb, unsigned int* __restrict__ fb_count) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t s_mm[2 * kSortWarps];
  __shared__ uint32_t s_scan[kSortWarps + 1];
  __shared__ uint32_t s_max[kSortWarps];
  __shared__ uint32_t s_q2;
  uint64_t* kB = reinterpret_cast<uint64_t*>(smem);
  uint32_t* cw = reinterpret_cast<uint32_t*>(kB + kSortCap);   // [kSubK / 2] words of u16 pairs
  const uint16_t* c16 = reinterpret_cast<const uint16_t*>(cw);
  uint16_t* qB = reinterpret_cast<uint16_t*>(cw + kSubK / 2);   // queued sub-buckets
  uint16_t* iB = qB + kQueueCap;                                // input index of slot j (VALS)

  uint64_t off, count, oo;
  cell_of(cs, blockIdx.x, off, count, oo);
  if (count == 0) return;
  if (cs.mode == 3) {
    // Fixed-capacity cells of a bucket whose digits are key values (m == 0)
    // were only counted: the cell is `count` copies of lo + digit.
    const uint32_t seg = cs.cell_seg[blockIdx.x];
    const DigitCls& d = cs.dcls[seg];
    if (d.m32 == 0) {
      const uint64_t ko = from_ordered<KIND_OUT>(d.lo + (blockIdx.x - cs.cell0[seg]));
      for (uint64_t i = threadIdx.x; i < count; i += blockDim.x) out[oo + i] = ko;
      return;
    }
  }
  if (big_cell<KIND_OUT, VALS>(src, src_vals, out, out_vals, off, oo, count, ovf, ovf_count, s_mm))
    return;
  const uint32_t n = (uint32_t)count;
  const uint32_t tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  // Digit cells of the first partition round: cell c of a segment holds the
  // keys with floor((key - lo) * mult / 2^64) == c, i.e. key - lo in
  // [c * 2^64 / mult, (c + 1) * 2^64 / mult).  With q = floor((2^64 - 1) /
  // mult), key - (lo + c * q) is >= 0 and below q + 2c + 2 (cell nb - 1 also
  // takes the clamped keys: the clamp below keeps its map monotone), so
  // sub = ((key - cell_lo) >> sh) * m32 >> 32 spreads the cell over kSubK
  // sub-buckets with one 32-bit multiply and no min/max pass.
  // Fixed-capacity cells (mode 3, k_bucket_ranges): cell c of a bucket holds
  // the keys with umulhi(x32, m) == c, x32 = (key - lo) >> sh, so
  // sub = umulhi(x32, m * kSubK) - c * kSubK is in [0, kSubK) exactly
  // (floor(floor(y * K) / K) = floor(y)); q holds m * kSubK (0: no refine).
  uint64_t lo = 0;
  uint32_t m32 = 0, sh = 0, sub0 = 0;
  int attempt = 1;
  if (cs.mode == 0 && cs.dcls) {
    const uint32_t seg = blockIdx.x / cs.cells_per_seg;
    const DigitCls& d = cs.dcls[seg];
    if (d.m32 != 0) {
      attempt = 0;
      lo = d.lo + (uint64_t)(blockIdx.x - seg * cs.cells_per_seg) * d.q;
      m32 = d.m32;
      sh = d.sh;
    }
  } else if (cs.mode == 3) {
    const uint32_t seg = cs.cell_seg[blockIdx.x];
    const DigitCls& d = cs.dcls[seg];
    if (d.q != 0) {
      attempt = 0;
      lo = d.lo;
      m32 = (uint32_t)d.q;
      sh = d.sh;
      sub0 = (blockIdx.x - cs.cell0[seg]) * (uint32_t)kFxSubBuckets;
    }
  }
  uint64_t kr[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    const uint32_t i = it * kSortThreads + tid;
    kr[it] = i < n ? ldg_stream(src + off + i) : ~0ULL;
  }
  uint4* const cw4 = reinterpret_cast<uint4*>(cw) + tid * (kScanWords / 4);
  // chunk c of this thread is stored at c ^ rot: the 8 threads of one
  // 128-bit shared-memory phase then cover 32 distinct banks.
  const uint32_t rot = (tid >> (3 - kLgChunks)) & (uint32_t)(kScanChunks - 1);
  uint32_t pk[kSortItems];
  uint32_t all, qpos;
  uint64_t hi_key = 0;
  bool exact = false;
  for (;; ++attempt) {
#pragma unroll
    for (int c = 0; c < kScanWords / 4; ++c) cw4[c ^ rot] = make_uint4(0, 0, 0, 0);
    if (attempt == 1) {
      uint64_t mn = ~0ULL, mx = 0;
#pragma unroll
      for (int it = 0; it < kSortItems; ++it) {
        mn = min(mn, kr[it]);
        if (it * kSortThreads + tid < n) mx = max(mx, kr[it]);
      }
      block_minmax(mn, mx, s_mm);  // its barriers also publish the zeroed counters
      if (mn == mx) {
        const uint64_t ko = from_ordered<KIND_OUT>(mn);
        for (uint32_t i = tid; i < n; i += kSortThreads) {
          out[oo + i] = ko;
          if constexpr (VALS) out_vals[oo + i] = src_vals[off + i];
        }
        return;
      }
      const uint64_t range = mx - mn;
      const uint32_t nsub = min(2 * n, (uint32_t)kSubK);
      exact = range < (uint64_t)nsub;  // one key value per sub-bucket
      // Sub-bucket = ((k - mn) >> sh) * m32 >> 32 in [0, nsub), monotone.
      lo = mn;
      hi_key = mx;
      sh = (uint32_t)max(0, bit_length64(range) - 32);
      // floor(2n * 2^32 / w32) - 1 <= the exact quotient: sub stays below 2n.
      m32 = exact ? 0
                  : (uint32_t)((float)nsub * 4294967296.0f / (float)((range >> sh) + 1)) - 1u;
      sub0 = 0;
    } else {
      __syncthreads();
    }
    // 1. count; the atomic's old value is the rank inside the sub-bucket.
    uint32_t nq = 0;  // sub-buckets this thread will queue (its keys of rank 1)
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
      pk[it] = 0xFFFFFFFFu;
      if (it * kSortThreads + tid < n) {
        const uint64_t x = kr[it] - lo;
        const uint32_t s =
            exact ? (uint32_t)x : min(__umulhi((uint32_t)(x >> sh), m32) - sub0, (uint32_t)kSubK - 1);
        const uint32_t sh = (s & 1) * 16;
        const uint32_t rk = (atomicAdd(&cw[sw_word(s >> 1)], 1u << sh) >> sh) & 0xFFFFu;
        pk[it] = (s << 16) | rk;
        nq += rk == 1;
      }
    }
    __syncthreads();
    // 2. scan.  Packed (keys | queue entries << 16): both prefixes stay < 2^16;
    // the per-word sums of the two u16 halves cannot carry (total <= n).
    uint32_t tw = 0, big = 0;
#pragma unroll
    for (int c = 0; c < kScanWords / 4; ++c) {
      const uint4 v = cw4[c ^ rot];
      tw += v.x + v.y + v.z + v.w;
      big = max(max(big, max(v.x, v.y)), max(v.z, v.w));
      big = max(max(big, max(v.x << 16, v.y << 16)), max(v.z << 16, v.w << 16));
    }
    big >>= 16;  // max over the high halves and the (shifted) low halves
    const uint32_t tot = (tw & 0xFFFFu) + (tw >> 16);
    const uint32_t mine = tot | (nq << 16);
    const uint32_t inc = warp_incl_scan(mine);
#pragma unroll
    for (int o = 16; o; o >>= 1) big = max(big, __shfl_xor_sync(0xffffffffu, big, o));
    if (lane == 31) s_scan[wid] = inc;
    if (lane == 0) s_max[wid] = big;
    all = scan_warp_totals<kSortThreads>(s_scan);
    const uint32_t pre = s_scan[wid] + inc - mine;
    big = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) big = max(big, s_max[w]);
    if (big > (uint32_t)kRankMax && (VALS || !exact)) {
      if (attempt == 0) continue;  // keys cluster inside the digit cell: use its min/max
      if (tid == 0) {
        const unsigned int slot = atomicAdd(fb_count, 1u);
        OverflowRec r; r.off = off; r.count = count; r.lo = lo; r.hi = hi_key; r.out = oo;
        fb[slot] = r;
      }
      return;
    }
    // Exclusive starts, two per word: (run, run + lo) + run * 0x10001.
    uint32_t run = (pre & 0xFFFFu) * 0x10001u;
#pragma unroll
    for (int c = 0; c < kScanWords / 4; ++c) {
      uint4 v = cw4[c ^ rot];
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t st = run + (w[q] << 16);
        run += ((w[q] * 0x10001u) >> 16) * 0x10001u;
        w[q] = st;
      }
      cw4[c ^ rot] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    qpos = pre >> 16;
    break;
  }
  __syncthreads();
  // 3. place: slot = start(sub-bucket) + rank.
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    if (pk[it] != 0xFFFFFFFFu) {
      const uint32_t s = pk[it] >> 16, rk = pk[it] & 0xFFFFu;
      const uint32_t slot = c16[sw16(s)] + rk;
      kB[slot] = kr[it];
      if constexpr (VALS) iB[slot] = (uint16_t)(it * kSortThreads + tid);
      if (rk == 1) qB[qpos++] = (uint16_t)s;
    }
  }
  if (tid == 0) s_q2 = 0;
  __syncthreads();
  // 4. order the multi-key sub-buckets in place.  c16[s] = start of
  // sub-bucket s; past the last counter the starts are n.
  if (VALS || !exact) {
    const uint32_t nqueue = all >> 16;
    uint16_t* q2 = qB + nqueue;  // larger sub-buckets, re-queued behind
    for (uint32_t q = tid; q < nqueue; q += kSortThreads) {
      const uint32_t s = qB[q];
      const uint32_t b0 = c16[sw16(s)];
      const uint32_t b1 = s + 1 < (uint32_t)kSubK ? c16[sw16(s + 1)] : n;
      if (b1 - b0 > 3) {
        q2[atomicAdd(&s_q2, 1u)] = (uint16_t)s;
        continue;
      }
      const bool three = b1 - b0 == 3;
      uint64_t k0 = kB[b0], k1 = kB[b0 + 1], k2 = three ? kB[b0 + 2] : ~0ULL;
      uint16_t i0 = 0, i1 = 0, i2 = 0xFFFFu;
      if constexpr (VALS) {
        i0 = iB[b0]; i1 = iB[b0 + 1];
        if (three) i2 = iB[b0 + 2];
      }
      cmp_swap<VALS>(k0, i0, k1, i1);
      cmp_swap<VALS>(k1, i1, k2, i2);
      cmp_swap<VALS>(k0, i0, k1, i1);
      kB[b0] = k0; kB[b0 + 1] = k1;
      if (three) kB[b0 + 2] = k2;
      if constexpr (VALS) {
        iB[b0] = i0; iB[b0 + 1] = i1;
        if (three) iB[b0 + 2] = i2;
      }
    }
    __syncthreads();
    const uint32_t n2 = s_q2;
    for (uint32_t q = tid; q < n2; q += kSortThreads) {
      const uint32_t s = q2[q];
      insertion_sort<VALS>(kB, iB, c16[sw16(s)], s + 1 < (uint32_t)kSubK ? c16[sw16(s + 1)] : n);
    }
    __syncthreads();
  }
  // 5. write-out, 16-byte stores when the output allows.
  const uint32_t a = (uint32_t)(oo & 1);
  if (((reinterpret_cast<uintptr_t>(out) & 15) == 0) && n > 2) {
    if (a && tid == 0) out[oo] = from_ordered<KIND_OUT>(kB[0]);
    const uint32_t np = (n - a) >> 1;
    uint4* o4 = reinterpret_cast<uint4*>(out + oo + a);
    for (uint32_t j = tid; j < np; j += kSortThreads) {
      const uint64_t k0 = from_ordered<KIND_OUT>(kB[a + 2 * j]);
      const uint64_t k1 = from_ordered<KIND_OUT>(kB[a + 2 * j + 1]);
      o4[j] = make_uint4((uint32_t)k0, (uint32_t)(k0 >> 32), (uint32_t)k1, (uint32_t)(k1 >> 32));
    }
    if (((n - a) & 1) && tid == 0) out[oo + n - 1] = from_ordered<KIND_OUT>(kB[n - 1]);
  } else {
    for (uint32_t j = tid; j < n; j += kSortThreads) out[oo + j] = from_ordered<KIND_OUT>(kB[j]);
  }
  if constexpr (VALS) {
    for (uint32_t j = tid; j < n; j += kSortThreads) out_vals[oo + j] = src_vals[off + iB[j]];
  }
}

// Keys-only sort of the fixed-capacity digit cells (mode 3), the hot final
// step of a bucket-major last level.  Same counting sort as k_smem_sort,
// specialised: the cell's refined digit is always available (no min/max
// attempt), counters are whole 32-bit words (no packed halves), the item
// loop runs over the cell's used items only (uniform bound), and equal keys
// need no tie order.
//   1. sub = umulhi((key - lo) >> sh, m * K) - digit * K in [0, K); one
//      shared atomic per key gives its rank in the sub-bucket;
//   2. block scan of the K counters (thread t owns words [32t, 32t + 32),
//      uint4 chunk c stored at c ^ (t & 7): conflict-free) fused with the
//      count of sub-buckets holding >= 2 keys;
//   3. place; the key of rank 1 queues its sub-bucket;
//   4. a thread per queued sub-bucket sorts it in place (2-3 keys by a
//      network, more by insertion; above kRankMax the cell goes to the LSD
//      fallback list);
//   5. 16-byte stores to the output.
// Cells without a refined digit (m * K >= 2^32) go to the LSD list; cells
// of counting-only buckets (m == 0) are one key value: filled directly.
constexpr int kFxItems = 16;  // 8 keys per thread on twice the threads measured no better
constexpr int kFxCap = AMS_FX_CAP;
constexpr int kFxSubK = kFxSubBuckets;
constexpr int kFxQueueCap = kFxCap / 2;
constexpr int kFxThreads = kFxCap / kFxItems;
constexpr int kFxCtas = 4 * 256 / kFxThreads;
// Counters: pairs of 16-bit halves in 32-bit words.
constexpr int kFxWords = kFxSubK / kFxThreads / 2;  // counter words per scan thread
static_assert(kFxWords == 16 || kFxWords == 8, "fixed-cell counter layout");
constexpr int kFxChunks = kFxWords / 4;
__device__ __forceinline__ uint32_t fx_sw(uint32_t w) {
  // word w belongs to scan thread w / kFxWords, whose chunk c sits at c ^ rot(thread)
  return w ^ (((w >> 5) & (uint32_t)(kFxChunks - 1)) << 2);
}

// Start of sub-bucket s after the scan.
__device__ __forceinline__ uint32_t fx_start(const uint16_t* c16, uint32_t s) {
  return c16[2 * fx_sw(s >> 1) + (s & 1)];
}

template <int KIND_OUT>
__global__ void __launch_bounds__(kFxThreads, kFxCtas)
    k_cell_sort_fixed(const uint64_t* __restrict__ src, uint64_t* __restrict__ out, CellSource cs,
                      OverflowRec* __restrict__ fb, unsigned int* __restrict__ fb_count) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_scan[kFxThreads / 32 + 1];
  __shared__ uint32_t s_big[kFxThreads / 32];
  uint64_t* kB = reinterpret_cast<uint64_t*>(smem);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(kB + kFxCap);
  uint16_t* q = reinterpret_cast<uint16_t*>(cnt + kFxWords * kFxThreads);
  const uint16_t* c16 = reinterpret_cast<const uint16_t*>(cnt);
  const uint32_t cid = blockIdx.x;
  const uint32_t n = cs.cell_cnt[cid];
  if (n == 0) return;
  const uint64_t off = (uint64_t)cid * kFxCap, oo = cs.cell_base[cid];
  const uint32_t seg = cs.cell_seg[cid];
  const DigitCls& d = cs.dcls[seg];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t digit = cid - cs.cell0[seg];
  if (d.m32 == 0) {  // counting-only bucket: one key value per cell
    const uint64_t ko = from_ordered<KIND_OUT>(d.lo + digit);
    for (uint32_t i = tid; i < n; i += kFxThreads) out[oo + i] = ko;
    return;
  }
  // No refined digit (m * K >= 2^32, dense keys): then sh == 0 and the cell
  // is the keys with key - lo in [ceil(digit 2^32 / m), ceil((digit+1) 2^32 / m)),
  // at most K values wide — one sub-bucket per key value (exact: no fix-ups).
  bool exact = false;
  uint64_t lo = d.lo;
  if (d.q == 0) {
    const uint64_t m = d.m32;
    const uint64_t x0 = (((uint64_t)digit << 32) + m - 1) / m;
    const uint64_t x1 = (((uint64_t)(digit + 1) << 32) + m - 1) / m;
    if (d.sh != 0 || x1 - x0 > (uint64_t)kFxSubK) {
      if (tid == 0) {
        OverflowRec r; r.off = off; r.count = n; r.lo = 0; r.hi = 0; r.out = oo;
        fb[atomicAdd(fb_count, 1u)] = r;
      }
      return;
    }
    exact = true;
    lo += x0;
  }
  const uint32_t sh = d.sh, mk = (uint32_t)d.q, sub0 = digit * (uint32_t)kFxSubK;
  uint4* const cw4 = reinterpret_cast<uint4*>(cnt) + tid * (kFxWords / 4);
  // chunk c of thread t sits at c ^ rot(t), rot(t) = ((first word of t) >> 5) & (chunks - 1)
  const uint32_t rot = ((tid * (uint32_t)kFxWords) >> 5) & (uint32_t)(kFxChunks - 1);
#pragma unroll
  for (int c = 0; c < kFxWords / 4; ++c) cw4[c ^ rot] = make_uint4(0, 0, 0, 0);
  const uint32_t nit = (n + kFxThreads - 1) / kFxThreads;  // uniform
  uint64_t kr[kFxItems];
  uint32_t pk[kFxItems];
#pragma unroll
  for (int it = 0; it < kFxItems; ++it) {
    const uint32_t i = it * kFxThreads + tid;
    kr[it] = (it < (int)nit && i < n) ? ldg_stream(src + off + i) : 0;
  }
  __syncthreads();  // counters zeroed
  uint32_t nq = 0;
#pragma unroll
  for (int it = 0; it < kFxItems; ++it) {
    if (it < (int)nit) {
      pk[it] = 0xFFFFFFFFu;
      if (it * kFxThreads + tid < n) {
        const uint32_t sb = exact ? (uint32_t)(kr[it] - lo) : __umulhi((uint32_t)((kr[it] - lo) >> sh), mk) - sub0;
        const uint32_t hs = (sb & 1) * 16;
        const uint32_t rk = (atomicAdd(&cnt[fx_sw(sb >> 1)], 1u << hs) >> hs) & 0xFFFFu;
        pk[it] = (sb << 12) | rk;
        nq += rk == 1;
      }
    }
  }
  __syncthreads();
  // Scan: 32 counters per thread, plus the queue count and the largest sub-bucket.
  uint32_t tw = 0, big = 0;
#pragma unroll
  for (int c = 0; c < kFxWords / 4; ++c) {
    const uint4 v = cw4[c ^ rot];
    tw += v.x + v.y + v.z + v.w;
    big = max(big, max(max(v.x, v.y), max(v.z, v.w)));
    big = max(big, max(max(v.x << 16, v.y << 16), max(v.z << 16, v.w << 16)));
  }
  big >>= 16;
  tw = (tw & 0xFFFFu) + (tw >> 16);  // halves cannot carry: total <= n
  const uint32_t mine = tw | (nq << 16);  // both prefixes < 2^16
  const uint32_t inc = warp_incl_scan(mine);
#pragma unroll
  for (int o = 16; o; o >>= 1) big = max(big, __shfl_xor_sync(0xffffffffu, big, o));
  if (lane == 31) s_scan[wid] = inc;
  if (lane == 0) s_big[wid] = big;
  scan_warp_totals<kFxThreads>(s_scan);  // (the one-barrier form measured slower here: 1.343 -> 1.443 ms)
  const uint32_t pre = s_scan[wid] + inc - mine;
  big = 0;
#pragma unroll
  for (int w = 0; w < kFxThreads / 32; ++w) big = max(big, s_big[w]);
  if (!exact && big > (uint32_t)kRankMax) {  // clustered keys: LSD fallback
    if (tid == 0) {
      OverflowRec r; r.off = off; r.count = n; r.lo = 0; r.hi = 0; r.out = oo;
      fb[atomicAdd(fb_count, 1u)] = r;
    }
    return;
  }
  uint32_t run = pre & 0xFFFFu;
#pragma unroll
  for (int c = 0; c < kFxWords / 4; ++c) {
    uint4 w4 = cw4[c ^ rot];
    uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const uint32_t t = wv[qq];
      wv[qq] = run | ((run + (t & 0xFFFFu)) << 16);  // (start of low half, start of high half)
      run += (t & 0xFFFFu) + (t >> 16);
    }
    cw4[c ^ rot] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  uint32_t qpos = pre >> 16;
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kFxItems; ++it) {
    if (it < (int)nit && pk[it] != 0xFFFFFFFFu) {
      const uint32_t sb = pk[it] >> 12, rk = pk[it] & 0xFFFu;
      kB[fx_start(c16, sb) + rk] = kr[it];
      if (rk == 1) q[qpos++] = (uint16_t)sb;
    }
  }
  __syncthreads();
  const uint32_t nqueue = exact ? 0 : s_scan[kFxThreads / 32] >> 16;  // exact: one value per sub-bucket
  for (uint32_t i = tid; i < nqueue; i += kFxThreads) {
    const uint32_t sb = q[i];
    const uint32_t b0 = fx_start(c16, sb);
    const uint32_t b1 = sb + 1 < (uint32_t)kFxSubK ? fx_start(c16, sb + 1) : n;
    if (b1 - b0 <= 3) {
      uint64_t k0 = kB[b0], k1 = kB[b0 + 1];
      if (b1 - b0 == 3) {
        uint64_t k2 = kB[b0 + 2];
        if (k0 > k1) { const uint64_t t = k0; k0 = k1; k1 = t; }
        if (k1 > k2) { const uint64_t t = k1; k1 = k2; k2 = t; }
        if (k0 > k1) { const uint64_t t = k0; k0 = k1; k1 = t; }
        kB[b0 + 2] = k2;
      } else if (k0 > k1) {
        const uint64_t t = k0; k0 = k1; k1 = t;
      }
      kB[b0] = k0;
      kB[b0 + 1] = k1;
    } else {
      for (uint32_t a = b0 + 1; a < b1; ++a) {
        const uint64_t ka = kB[a];
        uint32_t e = a;
        while (e > b0 && kB[e - 1] > ka) { kB[e] = kB[e - 1]; --e; }
        kB[e] = ka;
      }
    }
  }
  __syncthreads();
  const uint32_t a = (uint32_t)(oo & 1);
  if (a && tid == 0) out[oo] = from_ordered<KIND_OUT>(kB[0]);
  const uint32_t np = (n - a) >> 1;
  uint4* o4 = reinterpret_cast<uint4*>(out + oo + a);
  for (uint32_t j = tid; j < np; j += kFxThreads) {
    const uint64_t k0 = from_ordered<KIND_OUT>(kB[a + 2 * j]);
    const uint64_t k1 = from_ordered<KIND_OUT>(kB[a + 2 * j + 1]);
    o4[j] = make_uint4((uint32_t)k0, (uint32_t)(k0 >> 32), (uint32_t)k1, (uint32_t)(k1 >> 32));
  }
  if (((n - a) & 1) && tid == 0) out[oo + n - 1] = from_ordered<KIND_OUT>(kB[n - 1]);
}

}  // namespace

size_t smem_sort_bytes(bool vals) {
  return (size_t)kSortCap * 12 + 2 * (size_t)kQueueCap + (vals ? 2 * (size_t)kSortCap : 0);
}

size_t smem_sort_lsd_bytes() {
  return (size_t)kSortCap * (8 + 8 + 2 + 2) + (size_t)4 * kSortWarps * kRadix + 4 * kRadix;
}

cudaError_t launch_smem_sort(cudaStream_t st, const void* src, const void* src_vals, void* out,
                             void* out_vals, int kind_out, const CellSource& cs, uint64_t ncells,
                             OverflowRec* ovf, unsigned int* ovf_count, OverflowRec* fb,
                             unsigned int* fb_count) {
  if (ncells == 0) return cudaSuccess;
  if (cs.mode == 3 && !src_vals && (out != nullptr) &&
      ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
    const size_t smem = (size_t)kFxCap * 8 + (size_t)kFxWords * kFxThreads * 4 + 2 * (size_t)kFxQueueCap;
    cudaError_t e = cudaSuccess;
    AMS_KIND_DISPATCH(kind_out, K, {
      auto fn = k_cell_sort_fixed<K>;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      fn<<<(unsigned)ncells, kFxThreads, smem, st>>>(static_cast<const uint64_t*>(src),
                                                     static_cast<uint64_t*>(out), cs, fb, fb_count);
    });
    return cudaGetLastError();
  }
  const size_t smem = smem_sort_bytes(src_vals != nullptr);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  const uint64_t* sv = static_cast<const uint64_t*>(src_vals);
  uint64_t* o = static_cast<uint64_t*>(out);
  uint64_t* ov = static_cast<uint64_t*>(out_vals);
  cudaError_t e = cudaSuccess;
#define AMS_SORT_GO(K, V)                                                                   \
  {                                                                                         \
    auto fn = k_smem_sort<K, V>;                                                            \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    if (e != cudaSuccess) return e;                                                         \
    fn<<<(unsigned)ncells, kSortThreads, smem, st>>>(s, sv, o, ov, cs, ovf, ovf_count, fb,   \
                                                     fb_count);                             \
  }
  if (sv) {
    AMS_KIND_DISPATCH(kind_out, K, AMS_SORT_GO(K, true))
  } else {
    AMS_KIND_DISPATCH(kind_out, K, AMS_SORT_GO(K, false))
  }
#undef AMS_SORT_GO
  return cudaGetLastError();
}

cudaError_t launch_smem_sort_lsd(cudaStream_t st, const void* src, const void* src_vals, void* out,
                                 void* out_vals, int kind_out, const CellSource& cs,
                                 uint64_t ncells) {
  if (ncells == 0) return cudaSuccess;
  const size_t smem = smem_sort_lsd_bytes();
  const uint64_t* s = static_cast<const uint64_t*>(src);
  const uint64_t* sv = static_cast<const uint64_t*>(src_vals);
  uint64_t* o = static_cast<uint64_t*>(out);
  uint64_t* ov = static_cast<uint64_t*>(out_vals);
  cudaError_t e = cudaSuccess;
#define AMS_SORT_GO(K, V)                                                                 \
  {                                                                                       \
    auto fn = k_smem_sort_lsd<K, V>;                                                      \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                       \
    fn<<<(unsigned)ncells, kSortThreads, smem, st>>>(s, sv, o, ov, cs);                   \
  }
  if (sv) {
    AMS_KIND_DISPATCH(kind_out, K, AMS_SORT_GO(K, true))
  } else {
    AMS_KIND_DISPATCH(kind_out, K, AMS_SORT_GO(K, false))
  }
#undef AMS_SORT_GO
  return cudaGetLastError();
}

size_t scatter_fixed_smem_bytes(int nb) {
  const int per = (nb + kFThreads - 1) / kFThreads | 1;
  const size_t nbp = (size_t)per * kFThreads;
  return 2 * 8 * (size_t)(kFTile + 2) + 16 * nbp + 2 * (size_t)kFTile;
}

cudaError_t launch_scatter_fixed(cudaStream_t st, const void* src, int kind, void* dst,
                                 const SegMeta& m, uint64_t nchunks, int max_nb,
                                 const DigitCls* dcls, const uint32_t* cell0, uint32_t* fill,
                                 uint32_t* seg_ovf) {
  if (nchunks == 0) return cudaSuccess;
  const size_t smem = scatter_fixed_smem_bytes(max_nb);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  uint64_t* d = static_cast<uint64_t*>(dst);
  cudaError_t e = cudaSuccess;
  (void)kind;  // the last level's output holds order-mapped u64 keys
  auto fn = k_scatter_fixed<AMS_KEY_U64>;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<(unsigned)nchunks, kFThreads, smem, st>>>(s, d, m, dcls, cell0, fill, seg_ovf);
  return cudaGetLastError();
}

}  // namespace ams
