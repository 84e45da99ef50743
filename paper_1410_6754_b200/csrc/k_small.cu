// Small kernels of the level loop: sample gather (K1), sample ranking and
// classifier build (K2), offset scans (K4), relayout copies, key-range tables.
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ams_device.cuh"
#include "launch.h"

namespace ams {

namespace {
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

// Fast-mode sample: member m contributes take[m] elements
// (draw_sample's quota split, ams.py:166-171); element i of a member comes
// from stratum [i * size / take, (i + 1) * size / take) at a hashed offset,
// so positions are distinct and ascending and every element of the member
// is equally likely.  One thread per sample element; sample_off[m] = first
// output slot of member m (ascending; sample_off[nmem] = total).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
template <int KIND>
__global__ void k_draw_gather(const uint64_t* __restrict__ src, const uint64_t* __restrict__ sample_off,
                              const uint64_t* __restrict__ mem_off, const uint64_t* __restrict__ mem_len,
                              const uint64_t* __restrict__ mem_gpos, int nmem, uint64_t seed,
                              uint64_t* __restrict__ out_keys, uint32_t* __restrict__ out_pos,
                              const uint64_t* __restrict__ tags) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= sample_off[nmem]) return;
  const int m = upper_bound_u64(sample_off, nmem + 1, t) - 1;
  const uint64_t i = t - sample_off[m], take = sample_off[m + 1] - sample_off[m], size = mem_len[m];
  // strata by 128-bit products: size < 2^32 and take <= size
  const uint64_t lo = (uint64_t)(((unsigned __int128)i * size) / take);
  const uint64_t hi = (uint64_t)(((unsigned __int128)(i + 1) * size) / take);
  const uint64_t pos = lo + splitmix64(seed ^ splitmix64(((uint64_t)m << 40) ^ i)) % (hi - lo);
  const uint64_t idx = mem_off[m] + pos;
  out_keys[t] = to_ordered<KIND>(src[idx]);
  out_pos[t] = tags ? (uint32_t)tags[idx] : (uint32_t)(mem_gpos[m] + pos);
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

__global__ void k_iota(uint64_t* __restrict__ dst, uint64_t n, uint64_t start) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = start + i;
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

// Large samples (config 5 with one level: 256 PEs x 4096 buckets draw ~53 K
// sample elements, and counting over all pairs is S^2 = 2.8 G compares):
// the same rank-by-counting, with the counting done by binary search.
//   k_sample_block_sort  each CTA sorts kSortBlock elements by (key, pos)
//                        (bitonic network in shared memory) into tmp;
//   k_sample_merge_rank  rank of an element = its index in its own block +
//                        its lower bound in every other sorted block.
// (key, pos) pairs are unique inside a group, so ranks are a permutation.
constexpr int kSortBlock = 1024;
__global__ void __launch_bounds__(kSortBlock / 2)
    k_sample_block_sort(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ pos,
                        const uint64_t* __restrict__ soff, uint64_t* __restrict__ tk,
                        uint32_t* __restrict__ tp) {
  __shared__ uint64_t sk[kSortBlock];
  __shared__ uint32_t sp[kSortBlock];
  const int g = blockIdx.y;
  const uint64_t s0 = soff[g], S = soff[g + 1] - s0;
  const uint64_t first = (uint64_t)blockIdx.x * kSortBlock;
  if (first >= S) return;
  for (int i = threadIdx.x; i < kSortBlock; i += blockDim.x) {
    const bool ok = first + i < S;
    sk[i] = ok ? keys[s0 + first + i] : ~0ULL;
    sp[i] = ok ? pos[s0 + first + i] : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int k = 2; k <= kSortBlock; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int t = threadIdx.x;
      const int a = ((t & ~(j - 1)) << 1) | (t & (j - 1));  // lower index of the pair
      const int b = a | j;
      const bool up = (a & k) == 0;
      const uint64_t ka = sk[a], kb = sk[b];
      const uint32_t pa = sp[a], pb = sp[b];
      const bool a_after = ka > kb || (ka == kb && pa > pb);
      if (a_after == up) { sk[a] = kb; sk[b] = ka; sp[a] = pb; sp[b] = pa; }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kSortBlock; i += blockDim.x) {
    if (first + i < S) { tk[s0 + first + i] = sk[i]; tp[s0 + first + i] = sp[i]; }
  }
}

__global__ void __launch_bounds__(256)
    k_sample_merge_rank(const uint64_t* __restrict__ tk, const uint32_t* __restrict__ tp,
                        const uint64_t* __restrict__ soff, uint64_t* __restrict__ sorted_keys,
                        uint32_t* __restrict__ sorted_pos) {
  const int g = blockIdx.y;
  const uint64_t s0 = soff[g], S = soff[g + 1] - s0;
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S) return;
  const uint64_t k = tk[s0 + e];
  const uint32_t p = tp[s0 + e];
  const uint64_t mine = e / kSortBlock, nblk = (S + kSortBlock - 1) / kSortBlock;
  uint64_t rank = e % kSortBlock;
  for (uint64_t bj = 0; bj < nblk; ++bj) {
    if (bj == mine) continue;
    const uint64_t b0 = s0 + bj * kSortBlock;
    uint32_t lo = 0, hi = (uint32_t)min((uint64_t)kSortBlock, S - bj * kSortBlock);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint64_t km = tk[b0 + mid];
      if (km < k || (km == k && tp[b0 + mid] < p)) lo = mid + 1; else hi = mid;
    }
    rank += lo;
  }
  sorted_keys[s0 + rank] = k;
  sorted_pos[s0 + rank] = p;
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
// the simple-delivery order (g(b), j, b) (SURVEY §8 layout contract step 5),
// in three grid-wide steps (a level of 256 PEs x 4096 buckets is 1 M cells:
// one CTA per group would be bound by one SM's load bandwidth):
//   k_piece_sums   one CTA per segment: piece (j, t) = its keys for subgroup t;
//   k_piece_scan   one warp per (group, t): exclusive scan of the pieces over
//                  the group's segments + the subgroup total;
//   k_cell_rows    one CTA per segment: subgroup starts (scan of the totals)
//                  + piece offset + earlier buckets of the piece.
__global__ void __launch_bounds__(128) k_piece_sums(const uint32_t* __restrict__ seg_hist, int nb_stride,
                                                    GroupMeta gm, const int32_t* __restrict__ seg_group,
                                                    int r, uint64_t* __restrict__ pieces) {
  const int s = blockIdx.x, g = seg_group[s];
  const uint64_t* bnd = gm.bnd + (size_t)g * (r + 1);
  const uint32_t* hrow = seg_hist + (uint64_t)s * nb_stride;
  for (int t = threadIdx.x; t < r; t += blockDim.x) {
    uint64_t sum = 0;
    for (uint64_t b = bnd[t]; b < bnd[t + 1]; ++b) sum += hrow[b];
    pieces[(uint64_t)s * r + t] = sum;
  }
}

constexpr int kScanWarps = 8;
__global__ void __launch_bounds__(32 * kScanWarps)
    k_piece_scan(GroupMeta gm, int ngroups, int r, const uint64_t* __restrict__ pieces,
                 uint64_t* __restrict__ piece_off, uint64_t* __restrict__ sub_tot) {
  const int col = blockIdx.x * kScanWarps + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (col >= ngroups * r) return;
  const int g = col / r, t = col % r;
  const int first = gm.first[g], P = gm.nseg[g];
  uint64_t run = 0;
  for (int j0 = 0; j0 < P; j0 += 128) {
    uint64_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + 32 * u + lane;
      v[u] = j < P ? pieces[(uint64_t)(first + j) * r + t] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + 32 * u + lane;
      uint64_t x = v[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (j < P) piece_off[(uint64_t)(first + j) * r + t] = run + x - v[u];
      run += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  if (lane == 0) sub_tot[col] = run;
}

__global__ void __launch_bounds__(128) k_cell_rows(const uint32_t* __restrict__ seg_hist, int nb_stride,
                                                   GroupMeta gm, const int32_t* __restrict__ seg_group,
                                                   int r, const uint64_t* __restrict__ piece_off,
                                                   const uint64_t* __restrict__ sub_tot,
                                                   uint64_t* __restrict__ cell_base) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* sub0 = reinterpret_cast<uint64_t*>(smem);  // r subgroup starts
  __shared__ uint64_t s_w[4];
  const int s = blockIdx.x, g = seg_group[s];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // Exclusive scan of the group's subgroup totals, 128 at a time.
  uint64_t carry = 0;
  for (int t0 = 0; t0 < r; t0 += 128) {
    const int t = t0 + threadIdx.x;
    const uint64_t v = t < r ? sub_tot[(size_t)g * r + t] : 0;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    uint64_t before = carry;
    for (int ww = 0; ww < w; ++ww) before += s_w[ww];
    if (t < r) sub0[t] = before + x - v;
    carry += s_w[0] + s_w[1] + s_w[2] + s_w[3];
    __syncthreads();
  }
  const uint64_t* bnd = gm.bnd + (size_t)g * (r + 1);
  const uint32_t* hrow = seg_hist + (uint64_t)s * nb_stride;
  uint64_t* crow = cell_base + (uint64_t)s * nb_stride;
  const uint64_t start = gm.dst_start[g];
  for (int t = threadIdx.x; t < r; t += blockDim.x) {
    uint64_t base = start + sub0[t] + piece_off[(uint64_t)s * r + t];
    for (uint64_t b = bnd[t]; b < bnd[t + 1]; ++b) { crow[b] = base; base += hrow[b]; }
  }
}

// Bucket-major variant for a keys-only last level (only PE membership
// matters there, F7): cell (j, b) of group g starts at dst_start + sum of
// the group's earlier buckets + bucket b of earlier segments, so every
// bucket is contiguous and the children (consecutive bucket ranges) keep
// the same extents as in the (g(b), j, b) order.  k_bucket_totals sums
// every bucket over the group's segments; k_cell_base_bm (a CTA per 256
// buckets of a group) adds the buckets before its own and walks the segments.
__global__ void __launch_bounds__(256) k_bucket_totals(const uint32_t* __restrict__ seg_hist, int nb_stride,
                                                       GroupMeta gm, uint64_t* __restrict__ tot) {
  const int g = blockIdx.y, b = blockIdx.x * 256 + threadIdx.x;
  if (b >= nb_stride) return;
  const int first = gm.first[g], P = gm.nseg[g];
  uint64_t sum = 0;
#pragma unroll 8
  for (int j = 0; j < P; ++j) sum += seg_hist[(uint64_t)(first + j) * nb_stride + b];
  tot[(size_t)g * nb_stride + b] = sum;
}

__global__ void __launch_bounds__(256) k_cell_base_bm(const uint32_t* __restrict__ seg_hist, int nb_stride,
                                                      GroupMeta gm, const uint64_t* __restrict__ tot,
                                                      uint64_t* __restrict__ cell_base) {
  __shared__ uint64_t s_w[8], s_b[8];
  const int g = blockIdx.y, b0 = blockIdx.x * 256, b = b0 + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t* trow = tot + (size_t)g * nb_stride;
  // Buckets before this CTA's first, then an exclusive scan of its own 256.
  uint64_t before = 0;
  for (int i = threadIdx.x; i < b0; i += 256) before += trow[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
  const uint64_t v = b < nb_stride ? trow[b] : 0;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  if (lane == 0) s_b[w] = before;
  __syncthreads();
  uint64_t run = gm.dst_start[g] + x - v;
#pragma unroll
  for (int ww = 0; ww < 8; ++ww) run += s_b[ww] + (ww < w ? s_w[ww] : 0);
  if (b >= nb_stride) return;
  const int first = gm.first[g], P = gm.nseg[g];
  for (int j0 = 0; j0 < P; j0 += 8) {
    uint32_t h[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      h[u] = j0 + u < P ? seg_hist[(uint64_t)(first + j0 + u) * nb_stride + b] : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j0 + u < P) cell_base[(uint64_t)(first + j0 + u) * nb_stride + b] = run;
      run += h[u];
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
  const uint64_t mk = (uint64_t)d.m32 * (uint64_t)(kFxSubBuckets);
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

template <int FROM, int TO>
__global__ void k_map_keys(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = from_ordered<TO>(to_ordered<FROM>(src[i]));
}

}  // namespace

cudaError_t launch_draw_gather(cudaStream_t st, const void* src, int kind, const uint64_t* sample_off,
                               const uint64_t* mem_off, const uint64_t* mem_len, const uint64_t* mem_gpos,
                               int nmem, uint64_t total, uint64_t seed, uint64_t* out_keys,
                               uint32_t* out_pos, const uint64_t* tags) {
  if (total == 0 || nmem == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  AMS_KIND_DISPATCH(kind, K, k_draw_gather<K><<<blocks, 256, 0, st>>>(
      static_cast<const uint64_t*>(src), sample_off, mem_off, mem_len, mem_gpos, nmem, seed, out_keys,
      out_pos, tags));
  return cudaGetLastError();
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

cudaError_t launch_iota(cudaStream_t st, void* dst, uint64_t n, uint64_t start) {
  if (n == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  k_iota<<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(dst), n, start);
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
                               uint32_t* sorted_pos, uint64_t* tmp_keys, uint32_t* tmp_pos) {
  if (ngroups == 0 || max_s == 0) return cudaSuccess;
  if (max_s > kSampleRankPairsMax && tmp_keys && tmp_pos) {
    const dim3 ga((unsigned)((max_s + kSortBlock - 1) / kSortBlock), (unsigned)ngroups);
    k_sample_block_sort<<<ga, kSortBlock / 2, 0, st>>>(keys, pos, soff, tmp_keys, tmp_pos);
    const dim3 gb((unsigned)((max_s + 255) / 256), (unsigned)ngroups);
    k_sample_merge_rank<<<gb, 256, 0, st>>>(tmp_keys, tmp_pos, soff, sorted_keys, sorted_pos);
    return cudaGetLastError();
  }
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

cudaError_t launch_chunk_scan(cudaStream_t st, uint32_t* chunk_tot, const SegMeta& m, int nb_stride) {
  if (m.nseg == 0) return cudaSuccess;
  const int threads = nb_stride < 1024 ? ((nb_stride + 31) / 32) * 32 : 1024;
  k_chunk_scan<<<m.nseg, threads, 0, st>>>(chunk_tot, m, nb_stride);
  return cudaGetLastError();
}

cudaError_t launch_cell_base(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                             const GroupMeta& gm, int ngroups, int nseg, const int32_t* seg_group, int r,
                             uint64_t* pieces, uint64_t* cell_base) {
  if (ngroups == 0 || nseg == 0) return cudaSuccess;
  // pieces: [nseg * r] raw sums, [nseg * r] scanned offsets, [ngroups * r] subgroup totals.
  uint64_t* piece_off = pieces + (size_t)nseg * r;
  uint64_t* sub_tot = piece_off + (size_t)nseg * r;
  k_piece_sums<<<nseg, 128, 0, st>>>(seg_hist, nb_stride, gm, seg_group, r, pieces);
  k_piece_scan<<<(ngroups * r + kScanWarps - 1) / kScanWarps, 32 * kScanWarps, 0, st>>>(
      gm, ngroups, r, pieces, piece_off, sub_tot);
  k_cell_rows<<<nseg, 128, sizeof(uint64_t) * (size_t)r, st>>>(seg_hist, nb_stride, gm, seg_group, r,
                                                                piece_off, sub_tot, cell_base);
  return cudaGetLastError();
}

cudaError_t launch_cell_base_bm(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                                const GroupMeta& gm, int ngroups, uint64_t* tot, uint64_t* cell_base) {
  if (ngroups == 0) return cudaSuccess;
  const dim3 grid((unsigned)((nb_stride + 255) / 256), (unsigned)ngroups);
  k_bucket_totals<<<grid, 256, 0, st>>>(seg_hist, nb_stride, gm, tot);
  k_cell_base_bm<<<grid, 256, 0, st>>>(seg_hist, nb_stride, gm, tot, cell_base);
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
