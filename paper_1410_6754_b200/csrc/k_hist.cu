// K3: classification + chunk/segment histograms (partition_buckets
// ams.py:201-211, allreduce 236-237).
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ams_device.cuh"
#include "launch.h"

namespace ams {

namespace {
// The plain-atomic variants without the min/max fold fit 48 registers
// without spills: 5 CTAs per SM with 8 keys in flight per thread beat 4 CTAs
// with 16 there.  The other variants keep the compiler's allocation (forcing
// 48 registers on them spills, and the duplicate-heavy variant then faulted
// on sm_100a: profiles/r02m_hist_bounds.md).
template <int KIND, bool DIGIT, bool MINMAX, bool TAGS, int DUP>
constexpr int hist_min_ctas() {
  return (!DIGIT && !MINMAX && !TAGS && DUP == 1 && KIND != AMS_KEY_I64) ? 5 : 0;  // 0: no bound
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
__global__ void __launch_bounds__(kThreads, hist_min_ctas<KIND, DIGIT, MINMAX, TAGS, DUP>()) k_hist(const uint64_t* __restrict__ src, SegMeta m,
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
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)m.chunk;
  const uint64_t last = min(first + (uint64_t)m.chunk, seg_len);
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
  // Chunks whose first and last key share a bucket (sorted / duplicate-heavy
  // input: most of the chunk is one bucket, and one atomic per key would
  // serialise 32-way on that counter) aggregate runs; the others (keys
  // spread over the buckets) take one atomic per key — no run bookkeeping.
  bool runs = true;
  if constexpr (!DIGIT && !TAGS && DUP == 1) {
    if (last > first) {
      const uint32_t pb = (uint32_t)((int64_t)seg_off + posbase);
      const uint32_t b0 = tv.classify(to_ordered<KIND>(src[seg_off + first]), pb + (uint32_t)first);
      const uint32_t b1 = tv.classify(to_ordered<KIND>(src[seg_off + last - 1]), pb + (uint32_t)(last - 1));
      runs = b0 == b1;
    }
  }
  // keys a thread loads before classifying them: 8 at 5 CTAs/SM, else all 16
  constexpr int kPlainBatch = hist_min_ctas<KIND, DIGIT, MINMAX, TAGS, DUP>() != 0 ? 8 : kItems;
  auto tile_plain = [&](const uint64_t t0) {  // full tiles only
    const uint64_t base = seg_off + t0;
#pragma unroll
    for (int h = 0; h < kItems / kPlainBatch; ++h) {
      uint64_t keys[kPlainBatch];
#pragma unroll
      for (int i = 0; i < kPlainBatch; ++i)
        keys[i] = to_ordered<KIND>(ldg_stream(src + base + (h * kPlainBatch + i) * kThreads + threadIdx.x));
#pragma unroll
      for (int i = 0; i < kPlainBatch; ++i) {
        const uint32_t e = (h * kPlainBatch + i) * kThreads + threadIdx.x;
        const uint32_t b = tv.classify(keys[i], (uint32_t)((int64_t)base + posbase) + e, hint);
        if constexpr (IDS == 1) ids[base + e] = (uint8_t)b;
        if constexpr (IDS == 2) reinterpret_cast<uint16_t*>(ids)[base + e] = (uint16_t)b;
        if constexpr (MINMAX) { mn = min(mn, (unsigned long long)keys[i]); mx = max(mx, (unsigned long long)keys[i]); }
        atomicAdd(&hist[b], 1u);
      }
    }
  };
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
    if (tcount == (uint32_t)kTile) {
      if constexpr (!DIGIT && !TAGS && DUP == 1) {
        if (!runs) { tile_plain(t0); continue; }
      }
      tile(t0, tcount, std::true_type{});
    } else {
      tile(t0, tcount, std::false_type{});
    }
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

}  // namespace

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

}  // namespace ams
