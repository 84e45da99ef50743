// Device context and staging helpers shared by the C-ABI translation units
// (capi.cu: AMS-sort; capi_rlm.cu: RLM-sort).  Helpers live in an anonymous
// namespace: every translation unit gets its own copy.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "ams_host.h"
#include "launch.h"

namespace ams {
namespace {

#define AMS_CK(call)                                                                   \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return set_error(AMS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Makes `dev` current for one C-ABI call and restores the caller's device
// on return (a sort on cuda:1 must not leave a thread on cuda:1).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define AMS_ON_DEVICE(dev)  \
  DeviceGuard _ams_dg(dev); \
  AMS_CK(_ams_dg.err)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) {
      cudaError_t e = cudaFree(p);
      if (e != cudaSuccess) return e;
      p = nullptr;
      cap = 0;
    }
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Pinned host memory mapped into the device address space.  Small host <->
// device transfers of the sort go through it with a copy kernel, not the
// copy engines: a host pipeline's multi-GiB H2D / D2H of other batches
// occupy those, and a small cudaMemcpy queued behind one would stall the
// sort for the whole transfer.
struct HostBuf {
  void* p = nullptr;   // host address
  void* dp = nullptr;  // device address of the same bytes
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = dp = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 4096);
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    e = cudaHostGetDevicePointer(&dp, p, 0);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = dp = nullptr;
    cap = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Device -> mapped host copy on `st` (no copy engine); the caller syncs.
cudaError_t to_host(HostBuf& h, const void* dsrc, size_t bytes, cudaStream_t st) {
  cudaError_t e = h.ensure(bytes);
  if (e != cudaSuccess) return e;
  return launch_copy_bytes(st, h.dp, dsrc, bytes);
}

// Packs small host arrays, uploads them with one async copy from pinned
// memory, and keeps the device copy until the next upload on this stage.
struct Stage {
  std::vector<uint8_t> pack;
  HostBuf h;
  DevBuf d;
  cudaEvent_t ev = nullptr;
  bool pending = false;

  void reset() { pack.clear(); }
  template <class T>
  size_t put(const T* src, size_t n) {
    size_t off = (pack.size() + 15) & ~(size_t)15;
    pack.resize(off + sizeof(T) * n);
    if (n) std::memcpy(pack.data() + off, src, sizeof(T) * n);
    return off;
  }
  template <class T>
  size_t put(const std::vector<T>& v) { return put(v.data(), v.size()); }
  cudaError_t upload(cudaStream_t st) {
    cudaError_t e;
    if (!ev) {
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    if (pending) {
      e = cudaEventSynchronize(ev);
      if (e != cudaSuccess) return e;
      pending = false;
    }
    const size_t bytes = std::max<size_t>(pack.size(), 16);
    if ((e = h.ensure(bytes)) != cudaSuccess) return e;
    if ((e = d.ensure(bytes)) != cudaSuccess) return e;
    std::memcpy(h.p, pack.data(), pack.size());
    if ((e = launch_copy_bytes(st, d.p, h.dp, pack.size())) != cudaSuccess) return e;
    if ((e = cudaEventRecord(ev, st)) != cudaSuccess) return e;
    pending = true;
    return cudaSuccess;
  }
  template <class T> const T* dev(size_t off) const {
    return reinterpret_cast<const T*>(static_cast<const uint8_t*>(d.p) + off);
  }
  void release() {
    h.release();
    d.release();
    if (ev) cudaEventDestroy(ev);
    ev = nullptr;
  }
};

}  // namespace
}  // namespace ams

using namespace ams;

constexpr uint64_t kCopyItemKeys = 8192;  // keys per relayout work item (k_copy_ranges CTA)

struct ams_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  Stage st_sample, st_split, st_level, st_scatter, st_final;
  // splitters / classifiers of the current level
  DevBuf blobs, sorted_keys, sorted_pos, sample_idx, rank_tmp_keys, rank_tmp_pos;
  std::vector<int32_t> group_nb;
  int nspl_cap = 0, cells_cap = 0;
  // level state (classify -> scatter)
  int nseg = 0, ngroups = 0, nb_stride = 0;
  uint64_t nchunks = 0, level_elems = 0;
  std::vector<int32_t> group_first, group_nseg;
  SegMeta meta{};
  DevBuf chunk_tot, seg_hist, cell_base, pieces, minmax;
  bool level_stable = true;
  DevBuf ids;  // per-key bucket ids of the current level (bytes, or u16 above 256 buckets)
  bool level_ids = false;
  int level_id_bytes = 1;
  // key bounds [lo, hi] of the current level's groups (ping-pong)
  DevBuf bounds[2];
  int bcur = 0;
  HostBuf h_hist;
  // final sort
  DevBuf dcls, ovf, ovf_count, fb, fb_count;
  // bucket-major final sort (fixed-capacity cells)
  DevBuf fx_scratch, fx_fill, fx_ovf, fx_base, fx_cnt, fx_seg;
  Stage st_fixed;
  uint64_t fixed_segments = 0, fixed_overflow_segments = 0;
  bool bm_final = true;  // keys-only runs: bucket-major last level + fixed-capacity final sort
  bool host_trace = false;  // AMS_HOST_TRACE=1: host-side step times of ams_sort_run on stderr
  int fixed_fill_pct = 88;  // mean fill of the fixed-capacity cells (percent)
  // multi-GPU: buffers peers map (CUDA IPC) and the peers' buffers mapped here
  DevBuf peer_buf[8];
  std::vector<std::pair<std::string, void*>> peer_open;  // (handle bytes, mapped address)
  Stage st_peers;
  // deterministic delivery: origin tags (tie-breaks) and relayout work items
  const uint64_t* level_tags = nullptr;
  DevBuf tags0;
  Stage st_copy;
  HostBuf h_small, h_big;
  uint64_t overflow_cells = 0, fallback_cells = 0;
  // one-call driver (ams_sort_run): workspace and the last run's level records
  DevBuf work[2], work_v[2], s_keys, s_pos;
  struct LevelRec {
    int r = 0, G = 0, P = 0, nb_stride = 0;
    std::vector<int32_t> group_first, group_npe, nb;
    std::vector<uint64_t> sizes_before, drawn, boundaries, loads, max_load, new_sizes, stats;
    std::vector<uint32_t> hist;
    std::vector<uint32_t> holders;  // per PE: splitters drawn from it (record_holders)
    bool has_stats = false;
  };
  std::vector<LevelRec> run_levels;
  std::vector<std::vector<uint32_t>> hist_pool;  // histogram buffers of dropped runs, reused
  std::vector<uint64_t> run_final_sizes;
  // records of the last kRunHistory runs (run id, levels), newest last
  static constexpr size_t kRunHistory = 8;
  uint64_t run_id = 0;
  std::vector<std::pair<uint64_t, std::vector<LevelRec>>> run_history;
  // RLM-sort (capi_rlm.cu): extra work buffers, selection staging and the
  // last run's level records
  DevBuf rlm_buf[3], rlm_cuts, rlm_skey;
  Stage st_rlm;
  struct RlmLevel {
    int r = 0;
    std::vector<int32_t> group_first, group_npe;
    std::vector<uint64_t> sizes_before, cuts, new_sizes, stats;  // cuts [P][r+1], stats [G][4]
  };
  std::vector<RlmLevel> rlm_levels;
  // optional per-category kernel timing (CUDA events on the launching stream)
  bool timing = false;
  struct Timed { int cat; cudaEvent_t a, b; double bytes; };
  struct Span { int cat; float t0, t1; };
  std::vector<Span> timeline;  // resolved launches, ms from the first of each resolve batch
  std::vector<Timed> pending;
  std::vector<cudaEvent_t> free_events;
  double cat_ms[AMS_NUM_KCAT] = {};
  double cat_bytes[AMS_NUM_KCAT] = {};
  uint64_t cat_launches[AMS_NUM_KCAT] = {};
};


namespace ams {
// Stable sort by key of every segment [off, off + len) of (src, src_vals)
// into (out, out_vals) (capi.cu: shared-memory sorts for segments that fit,
// digit partition rounds by the given key bounds [lo, hi] for the others;
// src and tmp are clobbered).
int sort_segments_lohi(ams_ctx* c, void* src, void* src_vals, void* tmp, void* tmp_vals, void* out,
                       void* out_vals, int key_kind, int nseg, const uint64_t* h_seg_off,
                       const uint64_t* h_seg_len, const std::vector<uint64_t>& lo,
                       const std::vector<uint64_t>& hi);
}  // namespace ams
