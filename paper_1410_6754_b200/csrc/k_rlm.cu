// RLM-sort (rlm.py:86-132): exact multisequence selection on the device.
//
// multiselect_many (multiselect.py:45-137) finds the element of global rank
// t across the members' sorted sequences by randomized quickselect with
// vector collectives; its result is unique (element identities are unique),
// so the device computes it directly: a bisection over the key domain, then
// one over the origin tags of the elements holding that key, each step one
// block-wide sum of per-member binary searches.
#include <cstdint>
#include <cuda_runtime.h>

#include "ams_device.cuh"
#include "launch.h"

namespace ams {

namespace {

constexpr int kSelThreads = 256;

__device__ __forceinline__ uint64_t block_sum(uint64_t v, uint64_t* s_part) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // s_part of the previous call is consumed
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  uint64_t t = 0;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) t += s_part[w];
  return t;
}

// Elements of a[0, n) that are <= x (a ascending).
__device__ __forceinline__ uint64_t count_le(const uint64_t* a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ uint64_t count_lt(const uint64_t* a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One CTA per query (group, target rank t, 1 <= t <= group size): member j
// of the group holds keys[pe_off[first + j], pe_off[first + j + 1]) sorted
// by (key, tag).  Writes cuts[q.out + j] = the member's elements among the
// t smallest of the group (splits[pe] of SelectionResult,
// multiselect.py:24-36) and split_key[query] = the key of the rank-t element.
__global__ void __launch_bounds__(kSelThreads)
    k_rlm_select(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ tags,
                 const uint64_t* __restrict__ pe_off, const RlmQuery* __restrict__ qs,
                 uint64_t max_tag, uint64_t* __restrict__ cuts, uint64_t* __restrict__ split_key) {
  __shared__ uint64_t s_part[kSelThreads / 32];
  const RlmQuery q = qs[blockIdx.x];
  const int tid = threadIdx.x;
  // 1. smallest key K with #(key <= K) >= t.
  uint64_t lo = 0, hi = ~0ULL;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    uint64_t c = 0;
    for (int j = tid; j < q.npe; j += kSelThreads) {
      const uint64_t o = pe_off[q.first + j];
      c += count_le(keys + o, pe_off[q.first + j + 1] - o, mid);
    }
    if (block_sum(c, s_part) >= q.target) hi = mid; else lo = mid + 1;
  }
  const uint64_t K = lo;
  // 2. elements below K, and the rank still needed among the holders of K.
  uint64_t below = 0;
  for (int j = tid; j < q.npe; j += kSelThreads) {
    const uint64_t o = pe_off[q.first + j];
    below += count_lt(keys + o, pe_off[q.first + j + 1] - o, K);
  }
  const uint64_t need = q.target - block_sum(below, s_part);
  // 3. smallest tag T with #(key == K, tag <= T) >= need (tags ascend inside
  // a member's run of equal keys).
  uint64_t tlo = 0, thi = max_tag;
  while (tlo < thi) {
    const uint64_t mid = tlo + ((thi - tlo) >> 1);
    uint64_t c = 0;
    for (int j = tid; j < q.npe; j += kSelThreads) {
      const uint64_t o = pe_off[q.first + j], n = pe_off[q.first + j + 1] - o;
      const uint64_t a = count_lt(keys + o, n, K), b = count_le(keys + o, n, K);
      c += count_le(tags + o + a, b - a, mid);
    }
    if (block_sum(c, s_part) >= need) thi = mid; else tlo = mid + 1;
  }
  for (int j = tid; j < q.npe; j += kSelThreads) {
    const uint64_t o = pe_off[q.first + j], n = pe_off[q.first + j + 1] - o;
    const uint64_t a = count_lt(keys + o, n, K), b = count_le(keys + o, n, K);
    cuts[q.out + j] = a + count_le(tags + o + a, b - a, tlo);
  }
  if (tid == 0) split_key[blockIdx.x] = K;
}

}  // namespace

cudaError_t launch_rlm_select(cudaStream_t st, const uint64_t* keys, const uint64_t* tags,
                              const uint64_t* pe_off, const RlmQuery* qs, int nq, uint64_t max_tag,
                              uint64_t* cuts, uint64_t* split_key) {
  if (nq == 0) return cudaSuccess;
  k_rlm_select<<<nq, kSelThreads, 0, st>>>(keys, tags, pe_off, qs, max_tag, cuts, split_key);
  return cudaGetLastError();
}

}  // namespace ams
