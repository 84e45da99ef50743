// K6: level scatters (pieces ams.py:240-248, exchange order simnet.py:324-325).
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "ams_device.cuh"
#include "launch.h"

namespace ams {

namespace {
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
// 256 threads x 16 keys per 4096-key tile, 4 CTAs per SM (512 threads x 8 keys
// at 2 or 3 CTAs per SM: 1.47 -> 1.75-1.92 ms, profiles/r02v_ab_scatter_threads.txt).
constexpr int kSThreads = 256;
constexpr int kSWarps = kSThreads / 32;
constexpr int kSItems = kTile / kSThreads;
constexpr int kSCtas = 4;  // resident CTAs per SM without values
template <int KIND, int CLS, bool VALS, int MODE, bool PEERS = false>
__global__ void __launch_bounds__(kSThreads, VALS ? kSCtas / 2 : kSCtas)
    k_scatter(const uint64_t* __restrict__ src, const uint64_t* __restrict__ src_vals,
              uint64_t* __restrict__ dst, uint64_t* __restrict__ dst_vals, SegMeta m,
              const uint8_t* __restrict__ blobs, const DigitCls* __restrict__ dcls, int nspl_cap,
              int nb_stride, const uint32_t* __restrict__ chunk_tot,
              const uint64_t* __restrict__ cell_base, const uint8_t* __restrict__ ids,
              const uint64_t* __restrict__ bucket_dst = nullptr,
              const uint64_t* __restrict__ bucket_vdst = nullptr) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ uint32_t s_scan[kSWarps + 1];
  constexpr int kHists = MODE == kRankWarp ? kSWarps : 1;
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
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)m.chunk;
  const uint64_t last = min(first + (uint64_t)m.chunk, m.len[s]);
  const int cls = m.cls[s];
  {
    const uint32_t* ct = chunk_tot + c * nb_stride;
    const uint64_t* cb = cell_base + (uint64_t)s * nb_stride;
    for (int b = threadIdx.x; b < nb_stride; b += kSThreads) run[b] = (int64_t)(cb[b] + ct[b]);
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
    // (16-byte copies, two keys each, measured worse here: 1.475 -> 1.503 ms)
    for (uint32_t j = threadIdx.x; j < tcount; j += kSThreads) {
      cp_async8(keys_s + j, src + base + j);
      if constexpr (VALS) cp_async8(vals_s + j, src_vals + base + j);
    }
    for (int i = threadIdx.x; i < kHists * nb_stride; i += kSThreads) wh[i] = 0;
    cp_async_wait_all();
    __syncthreads();  // tile staged, counters zeroed, tree loaded
    uint32_t pk[kSItems];
    auto classify_all = [&](auto full_tag, auto runs_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      constexpr bool RUNS = decltype(runs_tag)::value;
      [[maybe_unused]] const uint32_t pos0 = (uint32_t)((int64_t)base + posbase);
#pragma unroll
      for (int i = 0; i < kSItems; ++i) {
        const uint32_t e = w * (kSItems * 32) + i * 32 + lane;
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
        for (int i = 0; i < kSItems; ++i) {
          const uint32_t b = pk[i];
          const uint32_t r = warp_stable_rank<NB>(b, lane, lt, whw, full);
          if (b != kInvalid) pk[i] = (b << 16) | r;
        }
      };
      for (int turn = 0; turn < (MODE == kRankSerial ? kSWarps : 1); ++turn) {
        if (MODE == kRankWarp || w == turn) {
          if (nbits <= 7) rank_all(std::integral_constant<int, 7>{});
          else if (nbits <= 9) rank_all(std::integral_constant<int, 9>{});
          else rank_all(std::integral_constant<int, 12>{});
        }
        if (MODE == kRankSerial) __syncthreads();
      }
    }
    __syncthreads();
    // Bucket totals -> tile starts (exclusive scan) -> output bases.  Up to
    // kSThreads buckets: one bucket per thread, the scan in registers with
    // one barrier (1.472 -> 1.413 ms at config 2's level 1); more buckets:
    // the shared-memory scan.
    const bool fast_scan = kAdj && nb_stride <= kSThreads;
    uint64_t kr[kSItems];
    uint64_t vr[VALS ? kSItems : 1];
    if (fast_scan) {
      const int b = threadIdx.x;
      uint32_t acc = 0;
      if (b < nb_stride) {
#pragma unroll
        for (int ww = 0; ww < kHists; ++ww) {
          const uint32_t v = wh[(size_t)ww * nb_stride + b];
          wh[(size_t)ww * nb_stride + b] = acc;
          acc += v;
        }
      }
      const uint32_t inc = warp_incl_scan(acc);
      if (lane == 31) s_scan[w] = inc;
#pragma unroll
      for (int i = 0; i < kSItems; ++i) {
        const uint32_t e = w * (kSItems * 32) + i * 32 + lane;
        kr[i] = keys_s[e];
        if constexpr (VALS) vr[i] = vals_s[e];
      }
      __syncthreads();
      uint32_t st = inc - acc;
      for (int ww = 0; ww < w; ++ww) st += s_scan[ww];
      if (b < nb_stride) {
        btot[b] = st;
        if constexpr (kAdj) {
          const int64_t r = run[b];
          adj[b] = r - (int64_t)st;
          run[b] = r + (int64_t)acc;
        }
      }
    } else {
      for (int b = threadIdx.x; b < nb_stride; b += kSThreads) {
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
      block_excl_scan<kSThreads>(btot, nb_stride, s_scan);
#pragma unroll
      for (int i = 0; i < kSItems; ++i) {
        const uint32_t e = w * (kSItems * 32) + i * 32 + lane;
        kr[i] = keys_s[e];
        if constexpr (VALS) vr[i] = vals_s[e];
      }
      // Output base of every bucket run of this tile; advance the running offsets.
      if constexpr (kAdj) {
        for (int b = threadIdx.x; b < nb_stride; b += kSThreads) {
          const uint32_t st = btot[b];
          const int64_t r = run[b];
          adj[b] = r - (int64_t)st;
          run[b] = r + (int64_t)((b + 1 < nb_stride ? btot[b + 1] : tcount) - st);
        }
      }
    }
    // Permute the staged tile bucket-major in place.
    {
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kSItems; ++i) {
        if (pk[i] != kInvalid) {
          const uint32_t b = pk[i] >> 16;
          // (one counter array: its scanned base is zero — no load)
          const uint32_t slot = btot[b] + (kHists > 1 ? whw[b] : 0u) + (pk[i] & 0xFFFFu);
          keys_s[slot] = to_ordered<KIND>(kr[i]);
          bkt_s[slot] = (uint16_t)b;
          if constexpr (VALS) vals_s[slot] = vr[i];
        }
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tcount; j += kSThreads) {
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
      for (int b = threadIdx.x; b < nb_stride; b += kSThreads)
        run[b] += (int64_t)((b + 1 < nb_stride ? btot[b + 1] : tcount) - btot[b]);
    }
  }
}

// Unstable scatter (keys only): the last level without values and the final
// digit partition, where any order inside a (tile, bucket) run gives the same
// result (F7).  Same chunk geometry and offsets as k_scatter.  Per tile:
// the 16-byte-aligned body arrives by one bulk copy into one of two shared
// buffers (the next tile's copy overlaps this tile's work); every key is
// classified and takes a rank from one shared atomic; a register-blocked
// scan turns the counts into tile starts and per-bucket output bases; the
// tile is permuted bucket-major in place and written as coalesced runs.

// 2048-key tiles on 256 threads, 4 CTAs per SM (with stored bucket ids:
// 1.104 -> 1.070 ms for config 2's last level against the cp.async kernel
// above; on 4096-key tiles / 512 threads it loses, 1.21 ms).
constexpr int kUTile = 2048;          // tile of the lean unstable scatter
constexpr int kLeanMaxBuckets = 1024;  // more buckets: the cp.async kernel's atomic mode
constexpr int kUItems = 8;
constexpr int kUThreads = kUTile / kUItems;
constexpr int kUWarps = kUThreads / 32;
constexpr int kUCtas = 2 * 4096 / kUTile;
static_assert(kTile % kUTile == 0, "chunks are whole tiles of both kinds");

template <int KIND, int CLS>
__global__ void __launch_bounds__(kUThreads, kUCtas)
    k_scatter_u(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, SegMeta m,
                const uint8_t* __restrict__ blobs, const DigitCls* __restrict__ dcls, int nspl_cap,
                int nb, const uint32_t* __restrict__ chunk_tot,
                const uint64_t* __restrict__ cell_base, const uint8_t* __restrict__ ids) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_seg;
  __shared__ uint32_t s_scan[kUWarps + 1];
  __shared__ __align__(8) uint64_t s_bar[2];
  constexpr int kBuf = kUTile + 2;  // room for the odd head key
  uint64_t* buf0 = reinterpret_cast<uint64_t*>(smem);
  const int per = (nb + kUThreads - 1) / kUThreads | 1;  // buckets per scan thread (odd: no conflicts)
  const int nbp = per * kUThreads;
  int64_t* run = reinterpret_cast<int64_t*>(buf0 + 2 * kBuf);  // running output offset
  int64_t* adj = run + nbp;                                     // this tile: dst index - slot
  uint32_t* cnt = reinterpret_cast<uint32_t*>(adj + nbp);       // counts, then tile starts
  uint16_t* bkt = reinterpret_cast<uint16_t*>(cnt + nbp);
  uint8_t* clsmem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(bkt + kUTile) + 15) & ~static_cast<uintptr_t>(15));

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
  const uint64_t first = (c - m.chunk_prefix[s]) * (uint64_t)m.chunk;
  const uint64_t last = min(first + (uint64_t)m.chunk, m.len[s]);
  const int ntiles = (int)((last - first + kUTile - 1) / kUTile);
  // Tile t = keys [base, base + tc); the copy covers whole 16-byte units
  // from the boundary base - h, so key e of the tile sits at buf[e + h]; when
  // tc + h is odd the last key is outside the copy and thread 0 adds it.
  auto issue = [&](int t) {
    const uint64_t base = seg_off + first + (uint64_t)t * kUTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kUTile, last - first - (uint64_t)t * kUTile);
    const uint32_t h = (uint32_t)(base & 1);
    bulk_load(buf0 + (t & 1) * kBuf, src + (base - h), ((tc + h) & ~1u) * 8, &s_bar[t & 1]);
  };
  if (tid == 0) issue(0);
  {
    const uint32_t* ct = chunk_tot + c * nb;
    const uint64_t* cb = cell_base + (uint64_t)s * nb;
    for (int b = tid; b < nb; b += kUThreads) run[b] = (int64_t)(cb[b] + ct[b]);
    for (int b = tid; b < nbp; b += kUThreads) cnt[b] = 0;
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
    const uint64_t base = seg_off + first + (uint64_t)t * kUTile;
    const uint32_t tc = (uint32_t)min((uint64_t)kUTile, last - first - (uint64_t)t * kUTile);
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
    uint64_t kr[kUItems];
    uint32_t pk[kUItems];
    const uint32_t pos0 = (uint32_t)((int64_t)base + posbase);
    auto classify_all = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int i = 0; i < kUItems; ++i) {
        const uint32_t e = w * (kUItems * 32) + i * 32 + lane;
        pk[i] = kInvalid;
        if (FULL || e < tc) {
          const uint64_t key = to_ordered<KIND>(tb[e]);
          uint32_t b;
          if constexpr (CLS == kClsIds) b = ids[base + e];
          else if constexpr (CLS == kClsIds16) b = reinterpret_cast<const uint16_t*>(ids)[base + e];
          else if constexpr (CLS == kClsDigit) b = dv.classify(key, 0);
          else b = tv.classify(key, pos0 + e);
          kr[i] = key;
          pk[i] = (b << 16) | atomicAdd(&cnt[b], 1u);
        }
      }
    };
    if (tc == (uint32_t)kUTile) classify_all(std::true_type{});
    else classify_all(std::false_type{});
    __syncthreads();
    // Scan: thread t owns buckets [t*per, t*per + per).
    {
      const int b0 = tid * per;
      uint32_t sum = 0;
      for (int j = 0; j < per; ++j) sum += cnt[b0 + j];
      const uint32_t inc = warp_incl_scan(sum);
      if (lane == 31) s_scan[w] = inc;
      uint32_t start = warp_base_direct<kUThreads>(s_scan) + inc - sum;
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
    for (int i = 0; i < kUItems; ++i) {
      if (pk[i] != kInvalid) {
        const uint32_t b = pk[i] >> 16;
        const uint32_t slot = cnt[b] + (pk[i] & 0xFFFFu);
        buf[slot] = kr[i];
        bkt[slot] = (uint16_t)b;
      }
    }
    __syncthreads();
    for (uint32_t j = tid; j < tc; j += kUThreads) dst[adj[bkt[j]] + j] = buf[j];
    for (int j = 0; j < per; ++j) cnt[tid * per + j] = 0;
    // This thread's generic-proxy writes into the tile buffer (the in-place
    // permutation) must be ordered before the bulk copy (async proxy) that
    // refills the buffer two tiles on: every writer fences, then the barrier.
    fence_proxy_async();
    __syncthreads();
  }
}

}  // namespace

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
  b += 4 * (size_t)(mode == kRankWarp ? kSWarps : 1) * nb_stride;      // bucket counters
  b += 4 * (size_t)nb_stride;                                         // tile bucket starts
  if (mode != kRankSerial) b += 8 * (size_t)nb_stride;                // tile output bases
  b += 2 * (size_t)kTile;                                             // bucket ids
  b = (b + 15) & ~(size_t)15;
  if (!digit) b += tree_smem_bytes(nspl_cap, cells_cap) + 16;
  return b;
}

size_t scatter_u_smem_bytes(int nb, int nspl_cap, int cells_cap, bool digit) {
  const int per = (nb + kUThreads - 1) / kUThreads | 1;
  const size_t nbp = (size_t)per * kUThreads;
  size_t b = 2 * 8 * (size_t)(kUTile + 2) + 16 * nbp + 4 * nbp + 2 * (size_t)kUTile;
  b = (b + 15) & ~(size_t)15;
  if (!digit) b += tree_smem_bytes(nspl_cap, cells_cap) + 16;
  return b;
}

// The lean unstable kernel serves the exact digit rounds of the final sort
// (keys only) and, with stored bucket bytes, the keys-only last level.
cudaError_t launch_scatter_u(cudaStream_t st, const void* src, int kind, void* dst, const SegMeta& m,
                             uint64_t nchunks, const DigitCls* dcls, int nb_stride,
                             const uint32_t* chunk_tot, const uint64_t* cell_base, const uint8_t* ids,
                             int id_bytes) {
  if (nchunks == 0) return cudaSuccess;
  const size_t smem = scatter_u_smem_bytes(nb_stride, 0, 0, true);
  const uint64_t* s = static_cast<const uint64_t*>(src);
  uint64_t* d = static_cast<uint64_t*>(dst);
  cudaError_t e = cudaSuccess;
  if (!ids) {
    auto fn = k_scatter_u<AMS_KEY_U64, kClsDigit>;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<(unsigned)nchunks, kUThreads, smem, st>>>(s, d, m, nullptr, dcls, 0, nb_stride, chunk_tot, cell_base,
                                                    nullptr);
  } else {
#define AMS_U_GO(K, CL)                                                                          \
  {                                                                                              \
    auto fn = k_scatter_u<K, CL>;                                                                \
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    if (e != cudaSuccess) return e;                                                              \
    fn<<<(unsigned)nchunks, kUThreads, smem, st>>>(s, d, m, nullptr, nullptr, 0, nb_stride, chunk_tot, \
                                                    cell_base, ids);                             \
  }
    if (id_bytes == 2) AMS_KIND_DISPATCH(kind, K, AMS_U_GO(K, kClsIds16))
    else AMS_KIND_DISPATCH(kind, K, AMS_U_GO(K, kClsIds))
#undef AMS_U_GO
  }
  return cudaGetLastError();
}

cudaError_t launch_scatter(cudaStream_t st, const void* src, const void* src_vals, int kind,
                           bool digit, bool stable, void* dst, void* dst_vals, const SegMeta& m,
                           uint64_t nchunks, const uint8_t* blobs, const DigitCls* dcls,
                           int nspl_cap, int cells_cap, int nb_stride, const uint32_t* chunk_tot,
                           const uint64_t* cell_base, const uint8_t* ids, int id_bytes) {
  if (nchunks == 0) return cudaSuccess;
  const bool vals = src_vals != nullptr;
  if (!stable && !vals && (digit || (ids && nb_stride <= kLeanMaxBuckets)))
    return launch_scatter_u(st, src, kind, dst, m, nchunks, dcls, nb_stride, chunk_tot, cell_base,
                            digit ? nullptr : ids, id_bytes);
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
    fn<<<(unsigned)nchunks, kSThreads, smem, st>>>(s, sv, d, dv, m, blobs, dcls, nspl_cap,     \
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
    fn<<<(unsigned)nchunks, kSThreads, smem, st>>>(s, sv, nullptr, nullptr, m, nullptr, nullptr, 0,  \
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

}  // namespace ams
