// sm_100a kernels of the AMS-sort hot path.
//
//   K1 k_gather_sample   sample elements at host-drawn positions
//                        (draw_sample, ams.py:157-175)
//   K2 k_sample_rank     work-inefficient rank-by-counting of the group
//      k_build_cls       sample, splitters at ranks (i*S)//nb, key LUT
//                        (select_splitters ams.py:178-198, fastsort.py:57-130)
//   K3 k_hist            classification + chunk/segment histograms
//                        (partition_buckets ams.py:201-211, allreduce 236-237)
//   K4 k_chunk_scan,     offsets of every (group, source PE, bucket) cell
//      k_cell_base,      (deliver_simple prefix sums delivery.py:138-180)
//      k_digit_base, k_child_bounds (key range of every next-level group)
//   K6 k_scatter         stable bucket-contiguous scatter (pieces ams.py:
//                        240-248, exchange order simnet.py:324-325)
//   K7 k_final_ranges    key range of every final PE
//   K9 k_smem_sort       CTA-local stable sort in shared memory (sorted(),
//                        ams.py:310-312)
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ams_device.cuh"
#include "launch.h"

// Sub-buckets of the cell sort per key of capacity (A/B knob).
#ifndef AMS_SUBK_MULT
#define AMS_SUBK_MULT 2
#endif

namespace ams {

namespace {

__device__ __forceinline__ int upper_bound_u64(const uint64_t* a, int n, uint64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

constexpr uint32_t kInvalid = 0xFFFFFFFFu;

// -------------------------------------------------------------------- K1
template <int KIND>
__global__ void k_gather_sample(const uint64_t* __restrict__ src, const uint64_t* __restrict__ idx,
                                const uint64_t* __restrict__ gpos, uint64_t n,
                                uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_pos,
                                const uint64_t* __restrict__ tags) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out_keys[i] = to_ordered<KIND>(src[idx[i]]);
  out_pos[i] = tags ? (uint32_t)tags[idx[i]] : (uint32_t)gpos[i];
}

// Deterministic delivery relayout: work item w copies up to kCopyItem keys
// of one range (ranges pre-split on the host).
constexpr uint64_t kCopyItem = 8192;
__global__ void k_copy_ranges(const uint64_t* __restrict__ items, const uint64_t* __restrict__ src,
                              uint64_t* __restrict__ dst, const uint64_t* __restrict__ src_vals,
                              uint64_t* __restrict__ dst_vals) {
  const uint64_t s0 = items[3 * blockIdx.x], d0 = items[3 * blockIdx.x + 1], len = items[3 * blockIdx.x + 2];
  for (uint64_t i = threadIdx.x; i < len; i += blockDim.x) {
    dst[d0 + i] = src[s0 + i];
    if (src_vals) dst_vals[d0 + i] = src_vals[s0 + i];
  }
}

// Small transfers between device memory and mapped pinned host memory
// (16-byte units while both sides allow, then bytes).
__global__ void k_copy_bytes(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t bytes) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  size_t head = 0;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const size_t n16 = bytes / 16;
    for (size_t i = tid; i < n16; i += nt)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    head = n16 * 16;
  }
  for (size_t i = head + tid; i < bytes; i += nt) dst[i] = src[i];
}

__global__ void k_iota(uint64_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = i;
}

__global__ void k_gather_vals(const uint64_t* __restrict__ vals, const uint64_t* __restrict__ idx,
                              uint64_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = vals[idx[i]];
}

// -------------------------------------------------------------------- K2
// rank_i = #{j : (k_j, p_j) < (k_i, p_i)} over the group's sample (the
// all-gather + rank-by-counting of fastsort.py:57-108).  A CTA ranks 64
// elements: warp w owns elements (w & 1) * 32 + lane and counts over the
// w >> 1 quarter of the sample, 32 sample elements at a time broadcast
// with __shfl_sync; the four partial counts meet in shared memory.
constexpr int kRankElems = 64, kRankSplit = 4;
__global__ void __launch_bounds__(256) k_sample_rank(const uint64_t* __restrict__ keys,
                                                     const uint32_t* __restrict__ pos,
                                                     const uint64_t* __restrict__ soff,
                                                     uint64_t* __restrict__ sorted_keys,
                                                     uint32_t* __restrict__ sorted_pos) {
  __shared__ uint32_t part[kRankSplit][kRankElems];
  const int g = blockIdx.y;
  const uint64_t s0 = soff[g], S = soff[g + 1] - s0;
  const uint64_t first = (uint64_t)blockIdx.x * kRankElems;
  if (first >= S) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = (w & 1) * 32 + lane, quarter = w >> 1;
  const uint64_t i = first + slot;
  const bool mine = i < S;
  const uint64_t ki = mine ? keys[s0 + i] : ~0ULL;
  const uint32_t pi = mine ? pos[s0 + i] : 0xFFFFFFFFu;
  const uint64_t per = ((S + kRankSplit - 1) / kRankSplit + 31) & ~31ULL;
  const uint64_t j0 = quarter * per, j1 = min(S, j0 + per);
  uint32_t cnt = 0;
  for (uint64_t c = j0; c < j1; c += 32) {
    const bool ok = c + lane < j1;
    const uint64_t kl = ok ? keys[s0 + c + lane] : ~0ULL;
    const uint32_t pl = ok ? pos[s0 + c + lane] : 0xFFFFFFFFu;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) {
      const uint64_t kj = __shfl_sync(0xffffffffu, kl, t);
      const uint32_t pj = __shfl_sync(0xffffffffu, pl, t);
      cnt += (kj < ki) | ((kj == ki) & (pj < pi));
    }
  }
  part[quarter][slot] = cnt;
  __syncthreads();
  if (threadIdx.x < kRankElems) {
    const uint64_t e = first + threadIdx.x;
    if (e < S) {
      uint32_t rank = 0;
#pragma unroll
      for (int q = 0; q < kRankSplit; ++q) rank += part[q][threadIdx.x];
      sorted_keys[s0 + rank] = keys[s0 + e];
      sorted_pos[s0 + rank] = pos[s0 + e];
    }
  }
}

__device__ __forceinline__ uint32_t lower_bound_smem(const uint64_t* a, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One CTA per group: splitter i (0-based) = sorted sample at rank
// ((i+1)*S)//nb (ams.py:190), then the cell LUT.
__global__ void __launch_bounds__(1024) k_build_cls(const uint64_t* __restrict__ sorted_keys,
                                                    const uint32_t* __restrict__ sorted_pos,
                                                    const uint64_t* __restrict__ soff,
                                                    const int32_t* __restrict__ nbs,
                                                    uint8_t* __restrict__ blobs) {
  __shared__ uint64_t sk[kMaxSpl];
  const int g = blockIdx.x;
  const uint64_t s0 = soff[g], S = soff[g + 1] - s0;
  const uint32_t nb = (uint32_t)nbs[g], nspl = nb - 1;
  uint8_t* blob = blobs + (size_t)g * kBlobStride;
  ClsHeader* h = reinterpret_cast<ClsHeader*>(blob);
  uint64_t* bk = reinterpret_cast<uint64_t*>(blob + kBlobKeys);
  uint32_t* bp = reinterpret_cast<uint32_t*>(blob + kBlobPos);
  uint32_t* lut = reinterpret_cast<uint32_t*>(blob + kBlobLut);
  for (uint32_t i = threadIdx.x; i < nspl; i += blockDim.x) {
    const uint64_t r = ((uint64_t)(i + 1) * S) / nb;
    const uint64_t k = sorted_keys[s0 + r];
    sk[i] = k;
    bk[i] = k;
    bp[i] = sorted_pos[s0 + r];
  }
  __syncthreads();
  if (nspl == 0) {
    if (threadIdx.x == 0) { h->lo = 0; h->hi = 0; h->nspl = 0; h->shift = 0; h->ncells = 0; h->max_inside = 0; }
    return;
  }
  const uint64_t lo = sk[0], hi = sk[nspl - 1];
  const int bits = lut_bits_for((int)nspl);
  const int bl = bit_length64(hi - lo);
  const uint32_t shift = bl > bits ? (uint32_t)(bl - bits) : 0u;
  const uint32_t ncells = (uint32_t)((hi - lo) >> shift) + 1;
  // Cell c covers keys [lo + c<<shift, lo + (c+1)<<shift); its record is
  // (#splitters below the cell) | (#splitters inside it) << 16.
  __shared__ uint32_t s_inside;
  if (threadIdx.x == 0) s_inside = 0;
  __syncthreads();
  uint32_t my_inside = 0;
  for (uint32_t c = threadIdx.x; c < ncells; c += blockDim.x) {
    const uint32_t first = lower_bound_smem(sk, nspl, lo + ((uint64_t)c << shift));
    const uint32_t next = c + 1 < ncells ? lower_bound_smem(sk, nspl, lo + ((uint64_t)(c + 1) << shift))
                                         : nspl;
    lut[c] = first | ((next - first) << 16);
    my_inside = max(my_inside, next - first);
  }
  atomicMax(&s_inside, my_inside);
  __syncthreads();
  if (threadIdx.x == 0) {
    h->lo = lo; h->hi = hi; h->nspl = nspl; h->shift = shift; h->ncells = ncells;
    h->max_inside = s_inside;
  }
}

// -------------------------------------------------------------------- K3
// One CTA per chunk (<= kChunkTiles tiles of one segment): classify every
// key, count buckets in shared memory with run-aggregated atomics (a run of
// same-bucket items of one thread costs one atomic — sorted and
// duplicate-heavy inputs stay cheap), then write the chunk histogram and
// add it to the segment histogram.
// IDS: also store every key's bucket (< 256) as a byte at its buffer index,
// so the level's scatter does not classify again.
// IDS: 0 = none, 1 = bucket bytes (<= 256 buckets), 2 = 16-bit bucket ids.
// DUP (tree classifiers): the launch is a pair; DUP = 1 does the groups
// whose LUT has no cell with more than 8 splitters, DUP = 2 the others
// (duplicate-heavy keys), trying the thread's previous bucket first in
// the binary search.  Each CTA of the other variant exits at once.
template <int KIND, bool DIGIT, bool MINMAX, int IDS, bool TAGS = false, int DUP = 1>
__global__ void __launch_bounds__(kThreads) k_hist(const uint64_t* __restrict__ src, SegMeta m,
                                                   const uint8_t* __restrict__ blobs,
                                                   const DigitCls* __restrict__ dcls, int nspl_cap,
                                                   int nb_stride, uint32_t* __restrict__ chunk_tot,
                                                   uint32_t* __restrict__ seg_hist,
                                                   unsigned long long* __restrict__ minmax,
                                                   uint8_t* __restrict__ ids) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ unsigned long long s_min[kWarps], s_max[kWarps];
  const uint64_t c = blockIdx.x;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);
  uint8_t* clsmem = smem + (((size_t)4 * nb_stride + 15) & ~(size_t)15);
  if (threadIdx.x == 0) s_seg = upper_bound_u64(m.chunk_prefix, m.nseg + 1, c) - 1;
  for (int b = threadIdx.x; b < nb_stride; b += kThreads) hist[b] = 0;
  __syncthreads();
  const int s = s_seg;
  const uint64_t seg_off = m.off[s], seg_len = m.len[s];
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)kChunk;
  const uint64_t last = min(first + (uint64_t)kChunk, seg_len);
  const int cls = m.cls[s];
  TreeView tv;
  DigitView dv;
  int64_t posbase = 0;
  if constexpr (DIGIT) {
    dv.c = dcls[cls];
  } else {
    if ((DUP == 2) != (reinterpret_cast<const ClsHeader*>(blobs + (size_t)cls * kBlobStride)->max_inside > 8))
      return;  // the other variant of the pair classifies this group
    tv = load_tree(blobs + (size_t)cls * kBlobStride, clsmem, nspl_cap);
    posbase = m.posbase[cls];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  unsigned long long mn = ~0ULL, mx = 0;
  // hint (DUP == 2): this thread's last bucket of the previous tile, tried
  // first in the many-splitter LUT cells; fixed for the tile, so the items'
  // classifications stay independent.
  uint32_t hint = kInvalid;
  auto tile = [&](const uint64_t t0, const uint32_t tcount, auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    const uint64_t base = seg_off + t0;
    uint64_t keys[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t e = i * kThreads + threadIdx.x;
      keys[i] = (FULL || e < tcount) ? to_ordered<KIND>(ldg_stream(src + base + e)) : 0;
    }
    // Run-aggregated shared atomics: consecutive items of a thread that
    // share a bucket (sorted / duplicate-heavy inputs) cost one atomic.
    uint32_t cur = kInvalid, cnt = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t e = i * kThreads + threadIdx.x;
      if (FULL || e < tcount) {
        uint32_t b;
        if constexpr (DIGIT) b = dv.classify(keys[i], 0);
        else if constexpr (TAGS) b = tv.classify(keys[i], (uint32_t)m.tags[base + e], hint);
        else b = tv.classify(keys[i], (uint32_t)((int64_t)base + posbase) + e, hint);
        if constexpr (IDS == 1) ids[base + e] = (uint8_t)b;
        if constexpr (IDS == 2) reinterpret_cast<uint16_t*>(ids)[base + e] = (uint16_t)b;
        if constexpr (MINMAX) { mn = min(mn, (unsigned long long)keys[i]); mx = max(mx, (unsigned long long)keys[i]); }
        if (b != cur) {
          if (cnt) atomicAdd(&hist[cur], cnt);
          cur = b;
          cnt = 0;
        }
        ++cnt;
      }
    }
    if (cnt) atomicAdd(&hist[cur], cnt);
    if constexpr (DUP == 2) hint = cur;
  };
  for (uint64_t t0 = first; t0 < last; t0 += kTile) {
    const uint32_t tcount = (uint32_t)min((uint64_t)kTile, last - t0);
    if (tcount == (uint32_t)kTile) tile(t0, tcount, std::true_type{});
    else tile(t0, tcount, std::false_type{});
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb_stride; b += kThreads) {
    const uint32_t v = hist[b];
    chunk_tot[c * nb_stride + b] = v;
    if (v) atomicAdd(&seg_hist[(uint64_t)s * nb_stride + b], v);
  }
  if constexpr (MINMAX) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) { s_min[threadIdx.x >> 5] = mn; s_max[threadIdx.x >> 5] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kWarps; ++w) { mn = min(mn, s_min[w]); mx = max(mx, s_max[w]); }
      atomicMin(&minmax[0], mn);
      atomicMax(&minmax[1], mx);
    }
  }
}

// -------------------------------------------------------------------- K4
// Exclusive scan of the chunk histograms along each segment's chunks.
__global__ void k_chunk_scan(uint32_t* __restrict__ chunk_tot, SegMeta m, int nb_stride) {
  const int s = blockIdx.x;
  const uint64_t c0 = m.chunk_prefix[s], c1 = m.chunk_prefix[s + 1];
  for (int b = threadIdx.x; b < nb_stride; b += blockDim.x) {
    uint32_t run = 0;
    uint64_t c = c0;
    for (; c + 8 <= c1; c += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = chunk_tot[(c + u) * nb_stride + b];
#pragma unroll
      for (int u = 0; u < 8; ++u) { chunk_tot[(c + u) * nb_stride + b] = run; run += v[u]; }
    }
    for (; c < c1; ++c) {
      const uint32_t v = chunk_tot[c * nb_stride + b];
      chunk_tot[c * nb_stride + b] = run;
      run += v;
    }
  }
}

// Output offset of every (source segment j, bucket b) cell of a group in
// the simple-delivery order (g(b), j, b) (SURVEY §8 layout contract step 5).
__global__ void __launch_bounds__(256) k_cell_base(const uint32_t* __restrict__ seg_hist, int nb_stride,
                                                   GroupMeta gm, int r, uint64_t* __restrict__ pieces,
                                                   uint64_t* __restrict__ cell_base) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* mtot = reinterpret_cast<uint64_t*>(smem);  // r entries
  const int g = blockIdx.x;
  const int first = gm.first[g], P = gm.nseg[g];
  const uint64_t* bnd = gm.bnd + (size_t)g * (r + 1);
  for (int idx = threadIdx.x; idx < P * r; idx += blockDim.x) {
    const int j = idx / r, gg = idx % r;
    const uint32_t* hrow = seg_hist + (uint64_t)(first + j) * nb_stride;
    uint64_t sum = 0;
    for (uint64_t b = bnd[gg]; b < bnd[gg + 1]; ++b) sum += hrow[b];
    pieces[(uint64_t)(first + j) * r + gg] = sum;
  }
  __syncthreads();
  for (int gg = threadIdx.x; gg < r; gg += blockDim.x) {
    uint64_t run = 0;
    for (int j = 0; j < P; ++j) {
      uint64_t* p = pieces + (uint64_t)(first + j) * r + gg;
      const uint64_t v = *p;
      *p = run;
      run += v;
    }
    mtot[gg] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int gg = 0; gg < r; ++gg) { const uint64_t t = mtot[gg]; mtot[gg] = acc; acc += t; }
  }
  __syncthreads();
  const uint64_t start = gm.dst_start[g];
  for (int idx = threadIdx.x; idx < P * r; idx += blockDim.x) {
    const int j = idx / r, gg = idx % r;
    const uint32_t* hrow = seg_hist + (uint64_t)(first + j) * nb_stride;
    uint64_t* crow = cell_base + (uint64_t)(first + j) * nb_stride;
    uint64_t base = start + mtot[gg] + pieces[(uint64_t)(first + j) * r + gg];
    for (uint64_t b = bnd[gg]; b < bnd[gg + 1]; ++b) { crow[b] = base; base += hrow[b]; }
  }
}

// Bucket-major variant for a keys-only last level (only PE membership
// matters there, F7): cell (j, b) of group g starts at dst_start + sum of
// the group's earlier buckets + bucket b of earlier segments, so every
// bucket is contiguous and the children (consecutive bucket ranges) keep
// the same extents as in the (g(b), j, b) order.  One CTA per group.
__global__ void __launch_bounds__(256) k_cell_base_bm(const uint32_t* __restrict__ seg_hist, int nb_stride,
                                                      GroupMeta gm, uint64_t* __restrict__ cell_base) {
  __shared__ uint64_t tot[AMS_MAX_BUCKETS];
  const int g = blockIdx.x;
  const int first = gm.first[g], P = gm.nseg[g];
  const int nb = nb_stride;  // buckets beyond a group's count are empty columns
  // Column sums (bucket totals of the group).
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    uint64_t sum = 0;
    for (int j = 0; j < P; ++j) sum += seg_hist[(uint64_t)(first + j) * nb_stride + b];
    tot[b] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = gm.dst_start[g];
    for (int b = 0; b < nb; ++b) { const uint64_t t = tot[b]; tot[b] = acc; acc += t; }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    uint64_t run = tot[b];
    for (int j = 0; j < P; ++j) {
      cell_base[(uint64_t)(first + j) * nb_stride + b] = run;
      run += seg_hist[(uint64_t)(first + j) * nb_stride + b];
    }
  }
}

// Digit partition: cell (s, d) starts at off[s] + sum of earlier digits.
__global__ void k_digit_base(const uint32_t* __restrict__ seg_hist, int nb_stride, SegMeta m,
                             uint64_t* __restrict__ cell_base) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m.nseg) return;
  uint64_t base = m.off[s];
  for (int d = 0; d < nb_stride; ++d) {
    cell_base[(uint64_t)s * nb_stride + d] = base;
    base += seg_hist[(uint64_t)s * nb_stride + d];
  }
}

// Key bounds of every child group: child t of group g holds buckets
// [B_t, B_{t+1}) of g, so its keys lie between splitter B_t - 1 and
// splitter B_{t+1} - 1 (the parent's bounds at the open ends).
__global__ void k_child_bounds(const uint8_t* __restrict__ blobs, GroupMeta gm, int ngroups, int r,
                               const uint64_t* __restrict__ parent, uint64_t* __restrict__ child) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ngroups * r) return;
  const int g = idx / r, t = idx % r;
  const uint8_t* blob = blobs + (size_t)g * kBlobStride;
  const ClsHeader* h = reinterpret_cast<const ClsHeader*>(blob);
  const uint64_t* bk = reinterpret_cast<const uint64_t*>(blob + kBlobKeys);
  const uint64_t nb = (uint64_t)h->nspl + 1;
  const uint64_t* bnd = gm.bnd + (size_t)g * (r + 1);
  const uint64_t b0 = bnd[t], b1 = bnd[t + 1];
  uint64_t lo = parent[2 * g], hi = parent[2 * g + 1];
  if (b0 > 0) lo = max(lo, bk[b0 - 1]);
  if (b1 < nb) hi = min(hi, bk[b1 - 1]);
  if (hi < lo) hi = lo;  // empty child
  child[2 * idx] = lo;
  child[2 * idx + 1] = hi;
}

// -------------------------------------------------------------------- K6
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

// One CTA per chunk (the histogram kernel's chunks): the running output
// offset of every bucket starts at cell base + the chunk's exclusive prefix.
// Per tile: cp.async stages the keys in shared memory, every key is
// classified and ranked from there, the tile is permuted bucket-major in
// place (keys pass through registers only for that step, so the kernel fits
// 4 CTAs per SM) and written as coalesced runs; the running offsets
// advance.  With a stable mode the order inside a bucket is the input order
// — the stable (cell, position) order the reference's concatenations produce.
// CLS: kClsTree (splitter tree in shared memory), kClsDigit (final digit),
// kClsIds (bucket bytes stored by the level's histogram pass).
// PEERS (multi-GPU level 1): bucket b's runs go to the buffer at address
// bucket_dst[b] (values: bucket_vdst[b]) — this GPU's own or a peer GPU's,
// mapped over NVLink — at the cell bases' indices; dst / dst_vals are unused.
template <int KIND, int CLS, bool VALS, int MODE, bool PEERS = false>
__global__ void __launch_bounds__(kThreads, VALS ? 2 : 4)
    k_scatter(const uint64_t* __restrict__ src, const uint64_t* __restrict__ src_vals,
              uint64_t* __restrict__ dst, uint64_t* __restrict__ dst_vals, SegMeta m,
              const uint8_t* __restrict__ blobs, const DigitCls* __restrict__ dcls, int nspl_cap,
              int nb_stride, const uint32_t* __restrict__ chunk_tot,
              const uint64_t* __restrict__ cell_base, const uint8_t* __restrict__ ids,
              const uint64_t* __restrict__ bucket_dst = nullptr,
              const uint64_t* __restrict__ bucket_vdst = nullptr) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ uint32_t s_scan[kWarps + 1];
  constexpr int kHists = MODE == kRankWarp ? kWarps : 1;
  uint64_t* keys_s = reinterpret_cast<uint64_t*>(smem);
  uint64_t* vals_s = keys_s + kTile;
  // Per-bucket output bases of the tile (dst index - slot); the serial mode
  // (> kSerialAbove buckets) has no room for them and adds run - start per key.
  constexpr bool kAdj = MODE != kRankSerial;
  int64_t* run = reinterpret_cast<int64_t*>(smem + (VALS ? 16 : 8) * (size_t)kTile);
  int64_t* adj = run + nb_stride;
  uint32_t* wh = reinterpret_cast<uint32_t*>(adj + (kAdj ? nb_stride : 0));
  uint32_t* btot = wh + (size_t)kHists * nb_stride;
  uint16_t* bkt_s = reinterpret_cast<uint16_t*>(btot + nb_stride);
  uint8_t* clsmem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(bkt_s + kTile) + 15) & ~static_cast<uintptr_t>(15));

  const uint64_t c = blockIdx.x;
  if (threadIdx.x == 0) s_seg = upper_bound_u64(m.chunk_prefix, m.nseg + 1, c) - 1;
  __syncthreads();
  const int s = s_seg;
  const uint64_t seg_off = m.off[s];
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)kChunk;
  const uint64_t last = min(first + (uint64_t)kChunk, m.len[s]);
  const int cls = m.cls[s];
  {
    const uint32_t* ct = chunk_tot + c * nb_stride;
    const uint64_t* cb = cell_base + (uint64_t)s * nb_stride;
    for (int b = threadIdx.x; b < nb_stride; b += kThreads) run[b] = (int64_t)(cb[b] + ct[b]);
  }
  TreeView tv;
  DigitView dv;
  int64_t posbase = 0;
  if constexpr (CLS == kClsDigit) {
    dv.c = dcls[cls];
  } else if constexpr (CLS == kClsTree || CLS == kClsTreeTags) {
    tv = load_tree(blobs + (size_t)cls * kBlobStride, clsmem, nspl_cap);
    posbase = m.posbase[cls];
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const int nbits = bit_length64((uint64_t)(nb_stride - 1));
  // Unstable mode: a chunk whose first and last key share a bucket (sorted /
  // duplicate-heavy input) ranks warps of one bucket with one atomic.
  bool runs = false;
  if constexpr (MODE == kRankAtomic && (CLS == kClsIds || CLS == kClsIds16)) {
    if (last > first) {
      const uint64_t i0 = seg_off + first, i1 = seg_off + last - 1;
      runs = CLS == kClsIds ? ids[i0] == ids[i1]
                            : reinterpret_cast<const uint16_t*>(ids)[i0] ==
                                  reinterpret_cast<const uint16_t*>(ids)[i1];
    }
  }
  uint32_t* whw = wh + (MODE == kRankWarp ? (size_t)w * nb_stride : 0);
  for (uint64_t t0 = first; t0 < last; t0 += kTile) {
    const uint32_t tcount = (uint32_t)min((uint64_t)kTile, last - t0);
    const uint64_t base = seg_off + t0;
    for (uint32_t j = threadIdx.x; j < tcount; j += kThreads) {
      cp_async8(keys_s + j, src + base + j);
      if constexpr (VALS) cp_async8(vals_s + j, src_vals + base + j);
    }
    for (int i = threadIdx.x; i < kHists * nb_stride; i += kThreads) wh[i] = 0;
    cp_async_wait_all();
    __syncthreads();  // tile staged, counters zeroed, tree loaded
    uint32_t pk[kItems];
    auto classify_all = [&](auto full_tag, auto runs_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      constexpr bool RUNS = decltype(runs_tag)::value;
      [[maybe_unused]] const uint32_t pos0 = (uint32_t)((int64_t)base + posbase);
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const uint32_t e = w * (kItems * 32) + i * 32 + lane;
        uint32_t b = kInvalid;
        if (FULL || e < tcount) {
          if constexpr (CLS == kClsIds) {
            b = ids[base + e];
          } else if constexpr (CLS == kClsIds16) {
            b = reinterpret_cast<const uint16_t*>(ids)[base + e];
          } else {
            const uint64_t key = to_ordered<KIND>(keys_s[e]);
            if constexpr (CLS == kClsDigit) b = dv.classify(key, 0);
            else if constexpr (CLS == kClsTreeTags) b = tv.classify(key, (uint32_t)vals_s[e]);
            else b = tv.classify(key, pos0 + e);
          }
        }
        pk[i] = b;
        if constexpr (MODE == kRankAtomic) {
          // A warp whose 32 keys share one bucket (sorted / duplicate-heavy
          // input) takes one atomic instead of 32 colliding ones.
          if constexpr (RUNS) {
            const uint32_t b0 = __shfl_sync(0xffffffffu, b, 0);
            if (__all_sync(0xffffffffu, b == b0) && b0 != kInvalid) {
              uint32_t base0 = 0;
              if (lane == 0) base0 = atomicAdd(&whw[b0], 32u);
              pk[i] = (b0 << 16) | (__shfl_sync(0xffffffffu, base0, 0) + lane);
            } else if (FULL || b != kInvalid) {
              pk[i] = (b << 16) | atomicAdd(&whw[b], 1u);
            }
          } else {
            if (FULL || b != kInvalid) pk[i] = (b << 16) | atomicAdd(&whw[b], 1u);
          }
        }
      }
    };
    if (tcount == (uint32_t)kTile) {
      if (runs) classify_all(std::true_type{}, std::true_type{});
      else classify_all(std::true_type{}, std::false_type{});
    } else {
      classify_all(std::false_type{}, std::false_type{});
    }
    if constexpr (MODE != kRankAtomic) {
      const bool full = tcount == (uint32_t)kTile;
      auto rank_all = [&](auto nbits_tag) {
        constexpr int NB = decltype(nbits_tag)::value;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
          const uint32_t b = pk[i];
          const uint32_t r = warp_stable_rank<NB>(b, lane, lt, whw, full);
          if (b != kInvalid) pk[i] = (b << 16) | r;
        }
      };
      for (int turn = 0; turn < (MODE == kRankSerial ? kWarps : 1); ++turn) {
        if (MODE == kRankWarp || w == turn) {
          if (nbits <= 7) rank_all(std::integral_constant<int, 7>{});
          else if (nbits <= 9) rank_all(std::integral_constant<int, 9>{});
          else rank_all(std::integral_constant<int, 12>{});
        }
        if (MODE == kRankSerial) __syncthreads();
      }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb_stride; b += kThreads) {
      uint32_t acc = 0;
#pragma unroll
      for (int ww = 0; ww < kHists; ++ww) {
        const uint32_t v = wh[(size_t)ww * nb_stride + b];
        wh[(size_t)ww * nb_stride + b] = acc;
        acc += v;
      }
      btot[b] = acc;
    }
    __syncthreads();
    block_excl_scan<kThreads>(btot, nb_stride, s_scan);
    // Permute the staged tile bucket-major in place.
    {
      uint64_t kr[kItems];
      uint64_t vr[VALS ? kItems : 1];
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const uint32_t e = w * (kItems * 32) + i * 32 + lane;
        kr[i] = keys_s[e];
        if constexpr (VALS) vr[i] = vals_s[e];
      }
      // Output base of every bucket run of this tile; advance the running offsets.
      if constexpr (kAdj) {
        for (int b = threadIdx.x; b < nb_stride; b += kThreads) {
          const uint32_t st = btot[b];
          const int64_t r = run[b];
          adj[b] = r - (int64_t)st;
          run[b] = r + (int64_t)((b + 1 < nb_stride ? btot[b + 1] : tcount) - st);
        }
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (pk[i] != kInvalid) {
          const uint32_t b = pk[i] >> 16;
          const uint32_t slot = btot[b] + whw[b] + (pk[i] & 0xFFFFu);
          keys_s[slot] = to_ordered<KIND>(kr[i]);
          bkt_s[slot] = (uint16_t)b;
          if constexpr (VALS) vals_s[slot] = vr[i];
        }
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tcount; j += kThreads) {
      const uint32_t b = bkt_s[j];
      const int64_t d = (kAdj ? adj[b] : run[b] - (int64_t)btot[b]) + (int64_t)j;
      if constexpr (PEERS) {
        reinterpret_cast<uint64_t*>(__ldg(bucket_dst + b))[d] = keys_s[j];
        if constexpr (VALS) reinterpret_cast<uint64_t*>(__ldg(bucket_vdst + b))[d] = vals_s[j];
      } else {
        dst[d] = keys_s[j];
        if constexpr (VALS) dst_vals[d] = vals_s[j];
      }
    }
    __syncthreads();
    if constexpr (!kAdj) {
      for (int b = threadIdx.x; b < nb_stride; b += kThreads)
        run[b] += (int64_t)((b + 1 < nb_stride ? btot[b + 1] : tcount) - btot[b]);
    }
  }
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

// Unstable scatter (keys only): the last level without values and the final
// digit partition, where any order inside a (tile, bucket) run gives the same
// result (F7).  Same chunk geometry and offsets as k_scatter.  Per tile:
// the 16-byte-aligned body arrives by one bulk copy into one of two shared
// buffers (the next tile's copy overlaps this tile's work); every key is
// classified and takes a rank from one shared atomic; a register-blocked
// scan turns the counts into tile starts and per-bucket output bases; the
// tile is permuted bucket-major in place and written as coalesced runs.
constexpr int kThreadsU = 512;                 // 16 warps x 8 keys per tile: 2 CTAs per SM
constexpr int kItemsU = kTile / kThreadsU;
constexpr int kWarpsU = kThreadsU / 32;

template <int KIND, int CLS>
__global__ void __launch_bounds__(kThreadsU, 2)
    k_scatter_u(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, SegMeta m,
                const uint8_t* __restrict__ blobs, const DigitCls* __restrict__ dcls, int nspl_cap,
                int nb, const uint32_t* __restrict__ chunk_tot,
                const uint64_t* __restrict__ cell_base, const uint8_t* __restrict__ ids) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ uint32_t s_scan[kWarpsU + 1];
  __shared__ __align__(8) uint64_t s_bar[2];
  constexpr int kBuf = kTile + 2;  // room for the odd head key
  uint64_t* buf0 = reinterpret_cast<uint64_t*>(smem);
  const int per = (nb + kThreadsU - 1) / kThreadsU | 1;  // buckets per scan thread (odd: no conflicts)
  const int nbp = per * kThreadsU;
  int64_t* run = reinterpret_cast<int64_t*>(buf0 + 2 * kBuf);  // running output offset
  int64_t* adj = run + nbp;                                     // this tile: dst index - slot
  uint32_t* cnt = reinterpret_cast<uint32_t*>(adj + nbp);       // counts, then tile starts
  uint16_t* bkt = reinterpret_cast<uint16_t*>(cnt + nbp);
  uint8_t* clsmem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(bkt + kTile) + 15) & ~static_cast<uintptr_t>(15));

  const uint64_t c = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_seg = upper_bound_u64(m.chunk_prefix, m.nseg + 1, c) - 1;
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int s = s_seg;
  const uint64_t seg_off = m.off[s];
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)kChunk;
  const uint64_t last = min(first + (uint64_t)kChunk, m.len[s]);
  const int ntiles = (int)((last - first + kTile - 1) / kTile);
  // Tile t = keys [base, base + tc); the copy covers whole 16-byte units
  // from the boundary base - h, so key e of the tile sits at buf[e + h]; when
  // tc + h is odd the last key is outside the copy and thread 0 adds it.
  auto issue = [&](int t) {
    const uint64_t base = seg_off + first + (uint64_t)t * kTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kTile, last - first - (uint64_t)t * kTile);
    const uint32_t h = (uint32_t)(base & 1);
    bulk_load(buf0 + (t & 1) * kBuf, src + (base - h), ((tc + h) & ~1u) * 8, &s_bar[t & 1]);
  };
  if (tid == 0) issue(0);
  {
    const uint32_t* ct = chunk_tot + c * nb;
    const uint64_t* cb = cell_base + (uint64_t)s * nb;
    for (int b = tid; b < nb; b += kThreadsU) run[b] = (int64_t)(cb[b] + ct[b]);
    for (int b = tid; b < nbp; b += kThreadsU) cnt[b] = 0;
  }
  TreeView tv;
  DigitView dv;
  int64_t posbase = 0;
  const int cls = m.cls[s];
  if constexpr (CLS == kClsDigit) dv.c = dcls[cls];
  else if constexpr (CLS == kClsTree) {
    tv = load_tree(blobs + (size_t)cls * kBlobStride, clsmem, nspl_cap);
    posbase = m.posbase[cls];
  }
  const int w = tid >> 5, lane = tid & 31;
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    uint64_t* buf = buf0 + (t & 1) * kBuf;
    const uint64_t base = seg_off + first + (uint64_t)t * kTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kTile, last - first - (uint64_t)t * kTile);
    const uint32_t h = (uint32_t)(base & 1);
    if (tid == 0 && t + 1 < ntiles) {
      fence_proxy_async();
      issue(t + 1);
    }
    mbar_wait(&s_bar[t & 1], (uint32_t)(t >> 1) & 1u);
    if ((tc + h) & 1) {  // the last key is outside the 16-byte copy
      if (tid == 0) buf[tc - 1 + h] = src[base + tc - 1];
      __syncthreads();
    }
    const uint64_t* tb = buf + h;
    uint64_t kr[kItemsU];
    uint32_t pk[kItemsU];
    const uint32_t pos0 = (uint32_t)((int64_t)base + posbase);
    auto classify_all = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int i = 0; i < kItemsU; ++i) {
        const uint32_t e = w * (kItemsU * 32) + i * 32 + lane;
        pk[i] = kInvalid;
        if (FULL || e < tc) {
          const uint64_t key = to_ordered<KIND>(tb[e]);
          uint32_t b;
          if constexpr (CLS == kClsIds) b = ids[base + e];
          else if constexpr (CLS == kClsDigit) b = dv.classify(key, 0);
          else b = tv.classify(key, pos0 + e);
          kr[i] = key;
          pk[i] = (b << 16) | atomicAdd(&cnt[b], 1u);
        }
      }
    };
    if (tc == (uint32_t)kTile) classify_all(std::true_type{});
    else classify_all(std::false_type{});
    __syncthreads();
    // Scan: thread t owns buckets [t*per, t*per + per).
    {
      const int b0 = tid * per;
      uint32_t sum = 0;
      for (int j = 0; j < per; ++j) sum += cnt[b0 + j];
      const uint32_t inc = warp_incl_scan(sum);
      if (lane == 31) s_scan[w] = inc;
      scan_warp_totals<kThreadsU>(s_scan);
      uint32_t start = s_scan[w] + inc - sum;
      for (int j = 0; j < per; ++j) {
        const int b = b0 + j;
        const uint32_t v = cnt[b];
        cnt[b] = start;
        if (b < nb) {
          const int64_t r = run[b];
          adj[b] = r - (int64_t)start;
          run[b] = r + v;
        }
        start += v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItemsU; ++i) {
      if (pk[i] != kInvalid) {
        const uint32_t b = pk[i] >> 16;
        const uint32_t slot = cnt[b] + (pk[i] & 0xFFFFu);
        buf[slot] = kr[i];
        bkt[slot] = (uint16_t)b;
      }
    }
    __syncthreads();
    for (uint32_t j = tid; j < tc; j += kThreadsU) dst[adj[bkt[j]] + j] = buf[j];
    for (int j = 0; j < per; ++j) cnt[tid * per + j] = 0;
    // This thread's generic-proxy writes into the tile buffer (the in-place
    // permutation) must be ordered before the bulk copy (async proxy) that
    // refills the buffer two tiles on: every writer fences, then the barrier.
    fence_proxy_async();
    __syncthreads();
  }
}

// Fixed-capacity digit partition (keys only, the final sort of a bucket-major
// last level): segments are the last level's buckets, each split into nb_s
// digit cells of capacity kSortCap in `dst` (cell ci at dst[ci * kSortCap]).
// No histogram pass: every (tile, digit) run reserves its room with one
// global atomic on the cell's fill counter, so a cell's keys land in any
// order (only membership matters: F7).  A cell that would exceed its
// capacity flags its segment; the host re-partitions such segments exactly
// from `src`, which this kernel does not modify.
template <int KIND>
__global__ void __launch_bounds__(kThreadsU, 2)
    k_scatter_fixed(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, SegMeta m,
                    const DigitCls* __restrict__ dcls, const uint32_t* __restrict__ cell0,
                    uint32_t* __restrict__ fill, uint32_t* __restrict__ seg_ovf) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ uint32_t s_scan[kWarpsU + 1];
  __shared__ uint32_t s_clip;
  __shared__ __align__(8) uint64_t s_bar[2];
  constexpr int kBuf = kTile + 2;
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
  const int per = (nb + kThreadsU - 1) / kThreadsU | 1;
  const int nbp = per * kThreadsU;
  int64_t* adj = reinterpret_cast<int64_t*>(buf0 + 2 * kBuf);  // this tile: dst index - slot
  uint32_t* cnt = reinterpret_cast<uint32_t*>(adj + nbp);       // counts, then tile starts
  int32_t* lim = reinterpret_cast<int32_t*>(cnt + nbp);         // writable keys of the run
  uint16_t* bkt = reinterpret_cast<uint16_t*>(lim + nbp);
  const uint64_t seg_off = m.off[s];
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)kChunk;
  const uint64_t last = min(first + (uint64_t)kChunk, m.len[s]);
  const int ntiles = (int)((last - first + kTile - 1) / kTile);
  const uint64_t cbase = cell0[s];
  // Tile t = keys [base, base + tc); the copy starts at the 16-byte boundary
  // base - h and is rounded up to whole 16-byte units (the source is the
  // last level's work buffer, padded by two keys), so key e of the tile sits
  // at buf[e + h].
  auto issue = [&](int t) {
    const uint64_t base = seg_off + first + (uint64_t)t * kTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kTile, last - first - (uint64_t)t * kTile);
    const uint32_t h = (uint32_t)(base & 1);
    bulk_load(buf0 + (t & 1) * kBuf, src + (base - h), ((tc + h + 1) & ~1u) * 8, &s_bar[t & 1]);
  };
  if (tid == 0) issue(0);
  for (int b = tid; b < nbp; b += kThreadsU) cnt[b] = 0;
  const int w = tid >> 5, lane = tid & 31;
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    uint64_t* buf = buf0 + (t & 1) * kBuf;
    const uint64_t base = seg_off + first + (uint64_t)t * kTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kTile, last - first - (uint64_t)t * kTile);
    const uint32_t h = (uint32_t)(base & 1);
    if (tid == 0 && t + 1 < ntiles) {
      fence_proxy_async();
      issue(t + 1);
    }
    mbar_wait(&s_bar[t & 1], (uint32_t)(t >> 1) & 1u);
    const uint64_t* tb = buf + h;
    uint64_t kr[kItemsU];
    uint32_t pk[kItemsU];
    auto classify_all = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int i = 0; i < kItemsU; ++i) {
        const uint32_t e = w * (kItemsU * 32) + i * 32 + lane;
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
    if (tc == (uint32_t)kTile) classify_all(std::true_type{});
    else classify_all(std::false_type{});
    __syncthreads();
    if (dm == 0) {
      // One key value per cell: only the counts matter (no capacity bound).
      for (int b = tid; b < nbp; b += kThreadsU) {
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
      scan_warp_totals<kThreadsU>(s_scan);
      uint32_t start = s_scan[w] + inc - sum;
      for (int j = 0; j < per; ++j) {
        const int b = b0 + j;
        const uint32_t v = cnt[b];
        cnt[b] = start;
        if (v) {
          // Reserve this run's room in cell (s, b).
          const uint32_t at = atomicAdd(&fill[cbase + b], v);
          adj[b] = (int64_t)((cbase + b) * (uint64_t)AMS_SMEM_SORT_CAP + at) - (int64_t)start;
          const int32_t room = (int32_t)AMS_SMEM_SORT_CAP - (int32_t)at;
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
    for (int i = 0; i < kItemsU; ++i) {
      if (pk[i] != kInvalid) {
        const uint32_t b = pk[i] >> 16;
        const uint32_t slot = cnt[b] + (pk[i] & 0xFFFFu);
        buf[slot] = kr[i];
        bkt[slot] = (uint16_t)b;
      }
    }
    __syncthreads();
    if (!s_clip) {
      for (uint32_t j = tid; j < tc; j += kThreadsU) dst[adj[bkt[j]] + j] = buf[j];
    } else {
      for (uint32_t j = tid; j < tc; j += kThreadsU) {
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

// Output base of every fixed-capacity cell: one warp per segment scans its
// cells' fill counts (segments flagged as overflowed get empty cells: the
// host partitions them again).  Also records each cell's segment.
__global__ void k_fixed_cells(const uint32_t* __restrict__ fill, const uint32_t* __restrict__ cell0,
                              const uint64_t* __restrict__ seg_off, const uint32_t* __restrict__ seg_ovf,
                              int nseg, uint64_t* __restrict__ out_base, uint32_t* __restrict__ cnt,
                              uint32_t* __restrict__ cell_seg) {
  const int s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= nseg) return;
  const uint32_t c0 = cell0[s], c1 = cell0[s + 1];
  const bool ovf = seg_ovf[s] != 0;
  uint64_t run = seg_off[s];
  for (uint32_t ci0 = c0; ci0 < c1; ci0 += 32) {
    const uint32_t ci = ci0 + lane;
    const uint32_t v = (ci < c1 && !ovf) ? fill[ci] : 0;
    const uint32_t inc = warp_incl_scan(v);
    if (ci < c1) {
      out_base[ci] = run + inc - v;
      cnt[ci] = v;
      cell_seg[ci] = (uint32_t)s;
    }
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// Digit classifier of every bucket segment of a bucket-major last level:
// bucket b of group g holds keys between splitter b-1 and splitter b (the
// group's bounds at the open ends); nb digits each (per segment).
__global__ void k_bucket_ranges(const uint8_t* __restrict__ blobs, const uint64_t* __restrict__ gbounds,
                                const int32_t* __restrict__ seg_gb, int nseg, DigitCls* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int g = seg_gb[3 * s], b = seg_gb[3 * s + 1];
  const uint8_t* blob = blobs + (size_t)g * kBlobStride;
  const ClsHeader* h = reinterpret_cast<const ClsHeader*>(blob);
  const uint64_t* bk = reinterpret_cast<const uint64_t*>(blob + kBlobKeys);
  uint64_t lo = gbounds[2 * g], hi = gbounds[2 * g + 1];
  if (b > 0) lo = max(lo, bk[b - 1]);
  if ((uint32_t)b < h->nspl) hi = min(hi, bk[b]);
  if (hi < lo) hi = lo;
  // 32-bit digit: x32 = (key - lo) >> sh, digit = umulhi(x32, m) with
  // m = floor(nb * 2^32 / (R + 1)), R = range >> sh: monotone and below nb;
  // m == 0: range < nb, the digit is key - lo itself (every cell holds one
  // key value: the partition only counts, the cell sort fills).
  DigitCls d;
  d.lo = lo;
  d.hi = hi;
  d.nb = (uint32_t)seg_gb[3 * s + 2];
  d.mult = 0;
  d.pad = 0;
  // R < 2^26 keeps m >= 64 nb (the floor of m costs < 1/64 of a cell) and
  // m * 2 * cap below 2^32 for nb <= 2048.
  const uint64_t range = hi - lo;
  d.sh = (uint32_t)max(0, bit_length64(range) - 26);
  const uint64_t R = range >> d.sh;
  d.m32 = R + 1 <= (uint64_t)d.nb ? 0u : (uint32_t)(((uint64_t)d.nb << 32) / (R + 1));
  const uint64_t mk = (uint64_t)d.m32 * (uint64_t)(AMS_SUBK_MULT * AMS_SMEM_SORT_CAP);
  d.q = mk < (1ull << 32) ? mk : 0;  // sub-bucket multiplier of the cell sort
  out[s] = d;
}

// -------------------------------------------------------------------- K7
__global__ void k_gather_bounds(const uint64_t* __restrict__ bounds, const int32_t* __restrict__ sel,
                                int n, uint64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[2 * i] = bounds[2 * sel[i]];
  out[2 * i + 1] = bounds[2 * sel[i] + 1];
}

constexpr int kCellSubBuckets = AMS_SUBK_MULT * AMS_SMEM_SORT_CAP;  // sub-buckets of a digit cell (= kSubK)

__global__ void k_final_ranges(const uint64_t* __restrict__ bounds, int nseg, int nb,
                               DigitCls* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const uint64_t lo = bounds[2 * s], hi = bounds[2 * s + 1];
  DigitCls d;
  d.lo = lo;
  d.hi = hi;
  d.nb = (uint32_t)nb;
  d.mult = digit_mult(hi - lo, d.nb);
  d.pad = 0;
  d.q = 0;
  d.m32 = 0;
  d.sh = 0;
  if (d.mult != 0) {
    // key - lo of cell c lies in [c * 2^64 / mult, (c + 1) * 2^64 / mult):
    // with q = floor((2^64 - 1) / mult), key - (lo + c * q) is in [0, w).
    d.q = (~0ULL) / d.mult;
    const uint64_t w = d.q + 2ull * d.nb + 2;
    d.sh = (uint32_t)max(0, bit_length64(w) - 32);
    const uint64_t w32 = ((w - 1) >> d.sh) + 1;
    if (w32 > (uint64_t)kCellSubBuckets) d.m32 = (uint32_t)(((uint64_t)kCellSubBuckets << 32) / w32);
  }
  out[s] = d;
}

// -------------------------------------------------------------------- K9
#ifndef AMS_SORT_THREADS
#define AMS_SORT_THREADS 256
#endif
constexpr int kSortThreads = AMS_SORT_THREADS;
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
    off = cid * (uint64_t)AMS_SMEM_SORT_CAP;
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
#ifndef AMS_SORT_CTAS
#define AMS_SORT_CTAS 3
#endif
constexpr int kSortCtas = AMS_SORT_CTAS;  // resident CTAs per SM (register budget)
#ifndef AMS_NIT_BREAK
#define AMS_NIT_BREAK 0
#endif
constexpr bool kNitBreak = AMS_NIT_BREAK;
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
      sub0 = (blockIdx.x - cs.cell0[seg]) * (uint32_t)kSubK;
    }
  }
  const int nit = (int)((n + kSortThreads - 1) / kSortThreads);  // items in use per thread
  uint64_t kr[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    if (kNitBreak && it >= nit) break;
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
        if (kNitBreak && it >= nit) break;
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
      if (kNitBreak && it >= nit) break;
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
    if (kNitBreak && it >= nit) break;
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
#ifndef AMS_FX_U16
#define AMS_FX_U16 1
#endif
constexpr int kFxThreads = 256;
constexpr int kFxItems = kSortCap / kFxThreads;   // 16
constexpr int kFxCtas = AMS_FX_U16 ? 4 : 3;
// Counters: 32-bit words, or (AMS_FX_U16) pairs of 16-bit halves.
constexpr int kFxWords = kSubK / kFxThreads / (AMS_FX_U16 ? 2 : 1);  // counter words per scan thread
static_assert(kFxWords == 32 || kFxWords == 16, "fixed-cell counter layout");
constexpr int kFxChunks = kFxWords / 4;
__device__ __forceinline__ uint32_t fx_sw(uint32_t w) {
  // word w belongs to scan thread w / kFxWords, whose chunk c sits at c ^ rot(thread)
  return w ^ (((w >> 5) & (uint32_t)(kFxChunks - 1)) << 2);
}

// Start of sub-bucket s after the scan.
__device__ __forceinline__ uint32_t fx_start(const uint32_t* cnt, const uint16_t* c16, uint32_t s) {
  if constexpr (AMS_FX_U16) return c16[2 * fx_sw(s >> 1) + (s & 1)];
  else return cnt[fx_sw(s)];
}

template <int KIND_OUT>
__global__ void __launch_bounds__(kFxThreads, kFxCtas)
    k_cell_sort_fixed(const uint64_t* __restrict__ src, uint64_t* __restrict__ out, CellSource cs,
                      OverflowRec* __restrict__ fb, unsigned int* __restrict__ fb_count) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_scan[kFxThreads / 32 + 1];
  __shared__ uint32_t s_big[kFxThreads / 32];
  uint64_t* kB = reinterpret_cast<uint64_t*>(smem);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(kB + kSortCap);
  uint16_t* q = reinterpret_cast<uint16_t*>(cnt + kFxWords * kFxThreads);
  const uint16_t* c16 = reinterpret_cast<const uint16_t*>(cnt);
  const uint32_t cid = blockIdx.x;
  const uint32_t n = cs.cell_cnt[cid];
  if (n == 0) return;
  const uint64_t off = (uint64_t)cid * kSortCap, oo = cs.cell_base[cid];
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
    if (d.sh != 0 || x1 - x0 > (uint64_t)kSubK) {
      if (tid == 0) {
        OverflowRec r; r.off = off; r.count = n; r.lo = 0; r.hi = 0; r.out = oo;
        fb[atomicAdd(fb_count, 1u)] = r;
      }
      return;
    }
    exact = true;
    lo += x0;
  }
  const uint32_t sh = d.sh, mk = (uint32_t)d.q, sub0 = digit * (uint32_t)kSubK;
  uint4* const cw4 = reinterpret_cast<uint4*>(cnt) + tid * (kFxWords / 4);
  const uint32_t rot = (kFxChunks == 8 ? tid : tid >> 1) & (uint32_t)(kFxChunks - 1);
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
        uint32_t rk;
        if constexpr (AMS_FX_U16) {
          const uint32_t hs = (sb & 1) * 16;
          rk = (atomicAdd(&cnt[fx_sw(sb >> 1)], 1u << hs) >> hs) & 0xFFFFu;
        } else {
          rk = atomicAdd(&cnt[fx_sw(sb)], 1u);
        }
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
    if constexpr (AMS_FX_U16)
      big = max(big, max(max(v.x << 16, v.y << 16), max(v.z << 16, v.w << 16)));
  }
  if constexpr (AMS_FX_U16) {
    big >>= 16;
    tw = (tw & 0xFFFFu) + (tw >> 16);  // halves cannot carry: total <= n
  }
  const uint32_t mine = tw | (nq << 16);  // both prefixes < 2^16
  const uint32_t inc = warp_incl_scan(mine);
#pragma unroll
  for (int o = 16; o; o >>= 1) big = max(big, __shfl_xor_sync(0xffffffffu, big, o));
  if (lane == 31) s_scan[wid] = inc;
  if (lane == 0) s_big[wid] = big;
  scan_warp_totals<kFxThreads>(s_scan);
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
      if constexpr (AMS_FX_U16) {  // (start of low half, start of high half)
        wv[qq] = run | ((run + (t & 0xFFFFu)) << 16);
        run += (t & 0xFFFFu) + (t >> 16);
      } else {
        wv[qq] = run;
        run += t;
      }
    }
    cw4[c ^ rot] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  uint32_t qpos = pre >> 16;
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kFxItems; ++it) {
    if (it < (int)nit && pk[it] != 0xFFFFFFFFu) {
      const uint32_t sb = pk[it] >> 12, rk = pk[it] & 0xFFFu;
      kB[fx_start(cnt, c16, sb) + rk] = kr[it];
      if (rk == 1) q[qpos++] = (uint16_t)sb;
    }
  }
  __syncthreads();
  const uint32_t nqueue = exact ? 0 : s_scan[kFxThreads / 32] >> 16;  // exact: one value per sub-bucket
  for (uint32_t i = tid; i < nqueue; i += kFxThreads) {
    const uint32_t sb = q[i];
    const uint32_t b0 = fx_start(cnt, c16, sb);
    const uint32_t b1 = sb + 1 < (uint32_t)kSubK ? fx_start(cnt, c16, sb + 1) : n;
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

template <int FROM, int TO>
__global__ void k_map_keys(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = from_ordered<TO>(to_ordered<FROM>(src[i]));
}

}  // namespace

// ======================================================================
// Launchers
// ======================================================================

#define AMS_KIND_DISPATCH(kind, K, ...)          \
  switch (kind) {                                \
    case AMS_KEY_I64: { constexpr int K = AMS_KEY_I64; __VA_ARGS__; } break; \
    case AMS_KEY_F64: { constexpr int K = AMS_KEY_F64; __VA_ARGS__; } break; \
    default: { constexpr int K = AMS_KEY_U64; __VA_ARGS__; } break;          \
  }

cudaError_t launch_gather_sample(cudaStream_t st, const void* src, int kind, const uint64_t* idx,
                                 const uint64_t* gpos, uint64_t n, uint64_t* out_keys,
                                 uint32_t* out_pos, const uint64_t* tags) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  AMS_KIND_DISPATCH(kind, K, k_gather_sample<K><<<blocks, 256, 0, st>>>(
      static_cast<const uint64_t*>(src), idx, gpos, n, out_keys, out_pos, tags));
  return cudaGetLastError();
}

cudaError_t launch_copy_ranges(cudaStream_t st, const uint64_t* items, int nitems, const void* src,
                               void* dst, const void* src_vals, void* dst_vals, uint64_t) {
  if (nitems == 0) return cudaSuccess;
  k_copy_ranges<<<(unsigned)nitems, 256, 0, st>>>(items, static_cast<const uint64_t*>(src),
                                                  static_cast<uint64_t*>(dst),
                                                  static_cast<const uint64_t*>(src_vals),
                                                  static_cast<uint64_t*>(dst_vals));
  return cudaGetLastError();
}

cudaError_t launch_copy_bytes(cudaStream_t st, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<size_t>((bytes + 4095) / 4096, 64);
  k_copy_bytes<<<blocks, 256, 0, st>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
  return cudaGetLastError();
}

cudaError_t launch_iota(cudaStream_t st, void* dst, uint64_t n) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  k_iota<<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(dst), n);
  return cudaGetLastError();
}

cudaError_t launch_gather_vals(cudaStream_t st, const void* vals, const void* idx, void* out, uint64_t n) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  k_gather_vals<<<blocks, 256, 0, st>>>(static_cast<const uint64_t*>(vals),
                                        static_cast<const uint64_t*>(idx), static_cast<uint64_t*>(out), n);
  return cudaGetLastError();
}

cudaError_t launch_sample_rank(cudaStream_t st, int ngroups, uint64_t max_s, const uint64_t* keys,
                               const uint32_t* pos, const uint64_t* soff, uint64_t* sorted_keys,
                               uint32_t* sorted_pos) {
  if (ngroups == 0 || max_s == 0) return cudaSuccess;
  dim3 grid((unsigned)((max_s + kRankElems - 1) / kRankElems), (unsigned)ngroups);
  k_sample_rank<<<grid, 256, 0, st>>>(keys, pos, soff, sorted_keys, sorted_pos);
  return cudaGetLastError();
}

cudaError_t launch_build_cls(cudaStream_t st, int ngroups, const uint64_t* sorted_keys,
                             const uint32_t* sorted_pos, const uint64_t* soff, const int32_t* nbs,
                             uint8_t* blobs) {
  if (ngroups == 0) return cudaSuccess;
  k_build_cls<<<ngroups, 1024, 0, st>>>(sorted_keys, sorted_pos, soff, nbs, blobs);
  return cudaGetLastError();
}

size_t hist_smem_bytes(int nb_stride, int nspl_cap, int cells_cap, bool digit) {
  return (((size_t)4 * nb_stride + 15) & ~(size_t)15) +
         (digit ? 0 : tree_smem_bytes(nspl_cap, cells_cap));
}

cudaError_t launch_hist(cudaStream_t st, const void* src, int kind, bool digit, const SegMeta& m,
                        uint64_t nchunks, const uint8_t* blobs, const DigitCls* dcls, int nspl_cap,
                        int cells_cap, int nb_stride, uint32_t* chunk_tot, uint32_t* seg_hist,
                        unsigned long long* minmax, uint8_t* ids, int id_bytes) {
  if (nchunks == 0) return cudaSuccess;
  const size_t smem = hist_smem_bytes(nb_stride, nspl_cap, cells_cap, digit);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  cudaError_t e = cudaSuccess;
  if (digit) {
    auto fn = k_hist<AMS_KEY_U64, true, false, 0>;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<(unsigned)nchunks, kThreads, smem, st>>>(s, m, blobs, dcls, nspl_cap, nb_stride,
                                                   chunk_tot, seg_hist, minmax, nullptr);
  } else if (m.tags) {
    // Origin-tag tie-breaks (deterministic delivery, levels >= 2): keys are order-mapped u64.
#define AMS_HIST_TAGS(D)                                                                          \
  {                                                                                               \
    auto fn = !ids ? k_hist<AMS_KEY_U64, false, false, 0, true, D>                                \
              : id_bytes == 2 ? k_hist<AMS_KEY_U64, false, false, 2, true, D>                     \
                              : k_hist<AMS_KEY_U64, false, false, 1, true, D>;                    \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    if (e != cudaSuccess) return e;                                                               \
    fn<<<(unsigned)nchunks, kThreads, smem, st>>>(s, m, blobs, dcls, nspl_cap, nb_stride, chunk_tot, \
                                                   seg_hist, minmax, ids);                        \
  }
    AMS_HIST_TAGS(1)
    AMS_HIST_TAGS(2)
#undef AMS_HIST_TAGS
  } else {
#define AMS_HIST_TREE(K, D)                                                                       \
  {                                                                                               \
    auto fn = minmax ? (!ids ? k_hist<K, false, true, 0, false, D>                                \
                       : id_bytes == 2 ? k_hist<K, false, true, 2, false, D>                      \
                                       : k_hist<K, false, true, 1, false, D>)                     \
                     : (!ids ? k_hist<K, false, false, 0, false, D>                               \
                       : id_bytes == 2 ? k_hist<K, false, false, 2, false, D>                     \
                                       : k_hist<K, false, false, 1, false, D>);                   \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    if (e != cudaSuccess) return e;                                                               \
    fn<<<(unsigned)nchunks, kThreads, smem, st>>>(s, m, blobs, dcls, nspl_cap, nb_stride,         \
                                                   chunk_tot, seg_hist, minmax, ids);             \
  }
    AMS_KIND_DISPATCH(kind, K, { AMS_HIST_TREE(K, 1) AMS_HIST_TREE(K, 2) });
#undef AMS_HIST_TREE
  }
  return cudaGetLastError();
}

cudaError_t launch_chunk_scan(cudaStream_t st, uint32_t* chunk_tot, const SegMeta& m, int nb_stride) {
  if (m.nseg == 0) return cudaSuccess;
  const int threads = nb_stride < 1024 ? ((nb_stride + 31) / 32) * 32 : 1024;
  k_chunk_scan<<<m.nseg, threads, 0, st>>>(chunk_tot, m, nb_stride);
  return cudaGetLastError();
}

cudaError_t launch_cell_base(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                             const GroupMeta& gm, int ngroups, int r, uint64_t* pieces,
                             uint64_t* cell_base) {
  if (ngroups == 0) return cudaSuccess;
  const size_t smem = sizeof(uint64_t) * (size_t)r;
  k_cell_base<<<ngroups, 256, smem, st>>>(seg_hist, nb_stride, gm, r, pieces, cell_base);
  return cudaGetLastError();
}

cudaError_t launch_cell_base_bm(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                                const GroupMeta& gm, int ngroups, uint64_t* cell_base) {
  if (ngroups == 0) return cudaSuccess;
  k_cell_base_bm<<<ngroups, 256, 0, st>>>(seg_hist, nb_stride, gm, cell_base);
  return cudaGetLastError();
}

cudaError_t launch_digit_base(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                              const SegMeta& m, uint64_t* cell_base) {
  if (m.nseg == 0) return cudaSuccess;
  k_digit_base<<<(m.nseg + 127) / 128, 128, 0, st>>>(seg_hist, nb_stride, m, cell_base);
  return cudaGetLastError();
}

cudaError_t launch_child_bounds(cudaStream_t st, const uint8_t* blobs, const GroupMeta& gm,
                                int ngroups, int r, const uint64_t* parent, uint64_t* child) {
  const int n = ngroups * r;
  if (n == 0) return cudaSuccess;
  k_child_bounds<<<(n + 127) / 128, 128, 0, st>>>(blobs, gm, ngroups, r, parent, child);
  return cudaGetLastError();
}

constexpr int kSerialAbove = 1024;  // buckets beyond which warps share one counter array

int scatter_mode(int nb_stride, bool stable) {
  if (!stable) return kRankAtomic;
  return nb_stride > kSerialAbove ? kRankSerial : kRankWarp;
}

size_t scatter_smem_bytes(int nb_stride, int nspl_cap, int cells_cap, bool digit, bool vals,
                          bool stable) {
  const int mode = scatter_mode(nb_stride, stable);
  size_t b = (vals ? 16 : 8) * (size_t)kTile;                         // keys (+vals)
  b += 8 * (size_t)nb_stride;                                         // running offsets
  b += 4 * (size_t)(mode == kRankWarp ? kWarps : 1) * nb_stride;      // bucket counters
  b += 4 * (size_t)nb_stride;                                         // tile bucket starts
  if (mode != kRankSerial) b += 8 * (size_t)nb_stride;                // tile output bases
  b += 2 * (size_t)kTile;                                             // bucket ids
  b = (b + 15) & ~(size_t)15;
  if (!digit) b += tree_smem_bytes(nspl_cap, cells_cap) + 16;
  return b;
}

size_t scatter_u_smem_bytes(int nb, int nspl_cap, int cells_cap, bool digit) {
  const int per = (nb + kThreadsU - 1) / kThreadsU | 1;
  const size_t nbp = (size_t)per * kThreadsU;
  size_t b = 2 * 8 * (size_t)(kTile + 2) + 16 * nbp + 4 * nbp + 2 * (size_t)kTile;
  b = (b + 15) & ~(size_t)15;
  if (!digit) b += tree_smem_bytes(nspl_cap, cells_cap) + 16;
  return b;
}

#ifndef AMS_SCATTER_U_IDS
#define AMS_SCATTER_U_IDS 0
#endif
constexpr bool kScatterUIds = AMS_SCATTER_U_IDS;

cudaError_t launch_scatter_u(cudaStream_t st, const void* src, int kind, bool digit, void* dst,
                             const SegMeta& m, uint64_t nchunks, const uint8_t* blobs,
                             const DigitCls* dcls, int nspl_cap, int cells_cap, int nb_stride,
                             const uint32_t* chunk_tot, const uint64_t* cell_base,
                             const uint8_t* ids) {
  if (nchunks == 0) return cudaSuccess;
  const size_t smem = scatter_u_smem_bytes(nb_stride, nspl_cap, cells_cap, digit || ids);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  uint64_t* d = static_cast<uint64_t*>(dst);
  cudaError_t e = cudaSuccess;
#define AMS_SCATTER_U_GO(K, CL)                                                               \
  {                                                                                           \
    auto fn = k_scatter_u<K, CL>;                                                             \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    if (e != cudaSuccess) return e;                                                           \
    fn<<<(unsigned)nchunks, kThreadsU, smem, st>>>(s, d, m, blobs, dcls, nspl_cap, nb_stride, \
                                                    chunk_tot, cell_base, ids);               \
  }
  if (digit) AMS_SCATTER_U_GO(AMS_KEY_U64, kClsDigit)
  else if (ids) AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_U_GO(K, kClsIds))
  else AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_U_GO(K, kClsTree))
#undef AMS_SCATTER_U_GO
  return cudaGetLastError();
}

cudaError_t launch_scatter(cudaStream_t st, const void* src, const void* src_vals, int kind,
                           bool digit, bool stable, void* dst, void* dst_vals, const SegMeta& m,
                           uint64_t nchunks, const uint8_t* blobs, const DigitCls* dcls,
                           int nspl_cap, int cells_cap, int nb_stride, const uint32_t* chunk_tot,
                           const uint64_t* cell_base, const uint8_t* ids, int id_bytes) {
  if (nchunks == 0) return cudaSuccess;
  const bool vals = src_vals != nullptr;
#ifndef AMS_NO_SCATTER_U
  // The lean unstable kernel pays off with the cheap digit classifier (the
  // final partition); the tree classifier keeps the 4-CTA kernel below.
  if (!stable && !vals && (digit || (ids && id_bytes == 1 && kScatterUIds)))
    return launch_scatter_u(st, src, kind, digit, dst, m, nchunks, blobs, dcls, nspl_cap,
                            cells_cap, nb_stride, chunk_tot, cell_base, digit ? nullptr : ids);
#endif
  const int mode = scatter_mode(nb_stride, stable);
  // Bucket bytes from the histogram pass replace the tree (and its shared memory).
  const size_t smem = scatter_smem_bytes(nb_stride, nspl_cap, cells_cap, digit || ids, vals, stable);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  const uint64_t* sv = static_cast<const uint64_t*>(src_vals);
  uint64_t* d = static_cast<uint64_t*>(dst);
  uint64_t* dv = static_cast<uint64_t*>(dst_vals);
  cudaError_t e = cudaSuccess;
#define AMS_SCATTER_GO(K, CL, V)                                                              \
  {                                                                                           \
    auto fn = mode == kRankWarp ? k_scatter<K, CL, V, kRankWarp>                              \
              : mode == kRankSerial ? k_scatter<K, CL, V, kRankSerial>                        \
                                    : k_scatter<K, CL, V, kRankAtomic>;                       \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    if (e != cudaSuccess) return e;                                                           \
    fn<<<(unsigned)nchunks, kThreads, smem, st>>>(s, sv, d, dv, m, blobs, dcls, nspl_cap,     \
                                                   nb_stride, chunk_tot, cell_base, ids,      \
                                                   nullptr, nullptr);                          \
  }
  if (digit) {
    if (vals) AMS_SCATTER_GO(AMS_KEY_U64, kClsDigit, true) else AMS_SCATTER_GO(AMS_KEY_U64, kClsDigit, false)
  } else if (m.tags && !ids) {
    if (!vals || mode == kRankAtomic) return cudaErrorInvalidValue;  // tags travel as the values
    AMS_SCATTER_GO(AMS_KEY_U64, kClsTreeTags, true)
  } else if (ids && id_bytes == 2) {
    if (vals) {
      AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_GO(K, kClsIds16, true))
    } else {
      AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_GO(K, kClsIds16, false))
    }
  } else if (ids) {
    if (vals) {
      AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_GO(K, kClsIds, true))
    } else {
      AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_GO(K, kClsIds, false))
    }
  } else if (vals) {
    AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_GO(K, kClsTree, true))
  } else {
    AMS_KIND_DISPATCH(kind, K, AMS_SCATTER_GO(K, kClsTree, false))
  }
#undef AMS_SCATTER_GO
  return cudaGetLastError();
}

cudaError_t launch_scatter_peers(cudaStream_t st, const void* src, const void* src_vals, int kind,
                                 const SegMeta& m, uint64_t nchunks, int nb_stride,
                                 const uint32_t* chunk_tot, const uint64_t* cell_base, const uint8_t* ids,
                                 int id_bytes, const uint64_t* bucket_dst, const uint64_t* bucket_vdst) {
  if (nchunks == 0) return cudaSuccess;
  if (!ids || nb_stride > kSerialAbove) return cudaErrorInvalidValue;  // stable warp ranks from stored ids
  const bool vals = src_vals != nullptr;
  const size_t smem = scatter_smem_bytes(nb_stride, 0, 0, true, vals, true);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  const uint64_t* sv = static_cast<const uint64_t*>(src_vals);
  cudaError_t e = cudaSuccess;
#define AMS_PEERS_GO(K, CL, V)                                                                      \
  {                                                                                                 \
    auto fn = k_scatter<K, CL, V, kRankWarp, true>;                                                 \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);           \
    if (e != cudaSuccess) return e;                                                                 \
    fn<<<(unsigned)nchunks, kThreads, smem, st>>>(s, sv, nullptr, nullptr, m, nullptr, nullptr, 0,  \
                                                   nb_stride, chunk_tot, cell_base, ids, bucket_dst, \
                                                   bucket_vdst);                                    \
  }
  if (id_bytes == 2) {
    if (vals) { AMS_KIND_DISPATCH(kind, K, AMS_PEERS_GO(K, kClsIds16, true)) }
    else { AMS_KIND_DISPATCH(kind, K, AMS_PEERS_GO(K, kClsIds16, false)) }
  } else {
    if (vals) { AMS_KIND_DISPATCH(kind, K, AMS_PEERS_GO(K, kClsIds, true)) }
    else { AMS_KIND_DISPATCH(kind, K, AMS_PEERS_GO(K, kClsIds, false)) }
  }
#undef AMS_PEERS_GO
  return cudaGetLastError();
}

cudaError_t launch_gather_bounds(cudaStream_t st, const uint64_t* bounds, const int32_t* sel, int n,
                                 uint64_t* out) {
  if (n == 0) return cudaSuccess;
  k_gather_bounds<<<(n + 127) / 128, 128, 0, st>>>(bounds, sel, n, out);
  return cudaGetLastError();
}

cudaError_t launch_final_ranges(cudaStream_t st, const uint64_t* bounds, int nseg, int nb,
                                DigitCls* out) {
  if (nseg == 0) return cudaSuccess;
  k_final_ranges<<<(nseg + 127) / 128, 128, 0, st>>>(bounds, nseg, nb, out);
  return cudaGetLastError();
}

// keys, 2x u16 sub-bucket counters (+ value index): two CTAs per SM.
size_t smem_sort_bytes(bool vals) {
  return (size_t)kSortCap * 12 + 2 * (size_t)kQueueCap + (vals ? 2 * (size_t)kSortCap : 0);
}

size_t smem_sort_lsd_bytes() {
  return (size_t)kSortCap * (8 + 8 + 2 + 2) + (size_t)4 * kSortWarps * kRadix + 4 * kRadix;
}

#ifndef AMS_FX_SORT
#define AMS_FX_SORT 1
#endif

cudaError_t launch_smem_sort(cudaStream_t st, const void* src, const void* src_vals, void* out,
                             void* out_vals, int kind_out, const CellSource& cs, uint64_t ncells,
                             OverflowRec* ovf, unsigned int* ovf_count, OverflowRec* fb,
                             unsigned int* fb_count) {
  if (ncells == 0) return cudaSuccess;
  if (AMS_FX_SORT && cs.mode == 3 && !src_vals && (out != nullptr) &&
      ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
    const size_t smem = (size_t)kSortCap * 8 + (size_t)kFxWords * kFxThreads * 4 + 2 * (size_t)kQueueCap;
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
  const int per = (nb + kThreadsU - 1) / kThreadsU | 1;
  const size_t nbp = (size_t)per * kThreadsU;
  return 2 * 8 * (size_t)(kTile + 2) + 16 * nbp + 2 * (size_t)kTile;
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
  fn<<<(unsigned)nchunks, kThreadsU, smem, st>>>(s, d, m, dcls, cell0, fill, seg_ovf);
  return cudaGetLastError();
}

cudaError_t launch_fixed_cells(cudaStream_t st, const uint32_t* fill, const uint32_t* cell0,
                               const uint64_t* seg_off, const uint32_t* seg_ovf, int nseg,
                               uint64_t* out_base, uint32_t* cnt, uint32_t* cell_seg) {
  if (nseg == 0) return cudaSuccess;
  k_fixed_cells<<<(nseg + 7) / 8, 256, 0, st>>>(fill, cell0, seg_off, seg_ovf, nseg, out_base, cnt,
                                                 cell_seg);
  return cudaGetLastError();
}

cudaError_t launch_bucket_ranges(cudaStream_t st, const uint8_t* blobs, const uint64_t* gbounds,
                                 const int32_t* seg_gb, int nseg, DigitCls* out) {
  if (nseg == 0) return cudaSuccess;
  k_bucket_ranges<<<(nseg + 127) / 128, 128, 0, st>>>(blobs, gbounds, seg_gb, nseg, out);
  return cudaGetLastError();
}

cudaError_t launch_map_keys(cudaStream_t st, const void* src, void* dst, uint64_t n, int from,
                            int to) {
  if (n == 0) return cudaSuccess;
  const uint64_t* s = static_cast<const uint64_t*>(src);
  uint64_t* d = static_cast<uint64_t*>(dst);
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
#define AMS_MAP_GO(F)                                                              \
  switch (to) {                                                                    \
    case AMS_KEY_I64: k_map_keys<F, AMS_KEY_I64><<<blocks, 256, 0, st>>>(s, d, n); break; \
    case AMS_KEY_F64: k_map_keys<F, AMS_KEY_F64><<<blocks, 256, 0, st>>>(s, d, n); break; \
    default: k_map_keys<F, AMS_KEY_U64><<<blocks, 256, 0, st>>>(s, d, n); break;          \
  }
  switch (from) {
    case AMS_KEY_I64: AMS_MAP_GO(AMS_KEY_I64) break;
    case AMS_KEY_F64: AMS_MAP_GO(AMS_KEY_F64) break;
    default: AMS_MAP_GO(AMS_KEY_U64) break;
  }
#undef AMS_MAP_GO
  return cudaGetLastError();
}

}  // namespace ams
