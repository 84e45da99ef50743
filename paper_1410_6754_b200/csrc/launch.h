// Host-callable kernel launchers (kernels.cu) and the small device-side
// metadata structs they take by value.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ams_device.cuh"

namespace ams {

// Segments (PEs) of one launch; arrays are device pointers.
struct SegMeta {
  const uint64_t* off;           // [nseg] start index in the source buffer
  const uint64_t* len;           // [nseg]
  const int32_t* cls;            // [nseg] classifier index
  const uint64_t* chunk_prefix;  // [nseg+1] first global chunk of each segment
  const int64_t* posbase;        // [ncls] tie-break position = index + posbase
  int nseg;
  const uint64_t* tags;          // origin tags (deterministic delivery, levels >= 2): tie-break by tag
  uint32_t chunk;                // keys per chunk (a multiple of kTile, <= kChunk): one CTA's share
};

// Groups of one level (contiguous runs of segments).
struct GroupMeta {
  const int32_t* first;       // [ngroups] first segment
  const int32_t* nseg;        // [ngroups] member count
  const uint64_t* bnd;        // [ngroups][r+1] plan boundaries
  const uint64_t* dst_start;  // [ngroups] output start of the group
};

// Work list of the shared-memory sort: mode 0 = cells of a digit
// partition (cell id = seg * nb + digit), mode 1 = explicit segments,
// mode 2 = records (fallback list on the device), mode 3 = fixed-capacity
// digit cells.
struct CellSource {
  int mode;
  uint32_t cells_per_seg;  // mode 0: cells of one segment (cell id = seg * cells_per_seg + digit)
  const uint64_t* cell_base;
  const uint32_t* cell_cnt;
  const DigitCls* dcls;
  const uint64_t* seg_off;
  const uint64_t* seg_len;
  const OverflowRec* recs;
  const unsigned int* nrecs;  // mode 2: record count on the device (may be null)
  // mode 3 = fixed-capacity cells (k_scatter_fixed): cell ci at src[ci * cap],
  // count cell_cnt[ci], output at cell_base[ci]; digit classifier of its
  // segment cell_seg[ci], whose first cell is cell0[seg].
  const uint32_t* cell_seg;
  const uint32_t* cell0;
};

// tags != NULL: the sample's tie-break value is its origin tag (tags[idx]),
// else its group position gpos.
cudaError_t launch_gather_sample(cudaStream_t st, const void* src, int kind, const uint64_t* idx,
                                 const uint64_t* gpos, uint64_t n, uint64_t* out_keys,
                                 uint32_t* out_pos, const uint64_t* tags);
// Fast-mode sample drawn and gathered on the device (k_draw_gather).
cudaError_t launch_draw_gather(cudaStream_t st, const void* src, int kind, const uint64_t* sample_off,
                               const uint64_t* mem_off, const uint64_t* mem_len, const uint64_t* mem_gpos,
                               int nmem, uint64_t total, uint64_t seed, uint64_t* out_keys,
                               uint32_t* out_pos, const uint64_t* tags);
// Copy ranges {src, dst, len} of keys (and values) — the deterministic
// delivery's relayout.
cudaError_t launch_copy_ranges(cudaStream_t st, const uint64_t* ranges, int nranges, const void* src,
                               void* dst, const void* src_vals, void* dst_vals, uint64_t total);
cudaError_t launch_iota(cudaStream_t st, void* dst, uint64_t n, uint64_t start = 0);
// Byte copy by a kernel (mapped host memory <-> device without the copy engines).
cudaError_t launch_copy_bytes(cudaStream_t st, void* dst, const void* src, size_t bytes);
// out[i] = vals[idx[i]]
cudaError_t launch_gather_vals(cudaStream_t st, const void* vals, const void* idx, void* out, uint64_t n);
// Samples above kSampleRankPairsMax elements per group (1024: config 1's 4096
// elements rank in ~15 instead of 33 us) take the block-sort +
// merge-rank kernels (tmp_keys / tmp_pos: scratch of the sample's size).
constexpr uint64_t kSampleRankPairsMax = 1024;
cudaError_t launch_sample_rank(cudaStream_t st, int ngroups, uint64_t max_s, const uint64_t* keys,
                               const uint32_t* pos, const uint64_t* soff, uint64_t* sorted_keys,
                               uint32_t* sorted_pos, uint64_t* tmp_keys = nullptr,
                               uint32_t* tmp_pos = nullptr);
cudaError_t launch_build_cls(cudaStream_t st, int ngroups, const uint64_t* sorted_keys,
                             const uint32_t* sorted_pos, const uint64_t* soff, const int32_t* nbs,
                             uint8_t* blobs);
size_t hist_smem_bytes(int nb_stride, int nspl_cap, int cells_cap, bool digit);
cudaError_t launch_hist(cudaStream_t st, const void* src, int kind, bool digit, const SegMeta& m,
                        uint64_t nchunks, const uint8_t* blobs, const DigitCls* dcls, int nspl_cap,
                        int cells_cap, int nb_stride, uint32_t* chunk_tot, uint32_t* seg_hist,
                        unsigned long long* minmax, uint8_t* ids, int id_bytes = 1);
cudaError_t launch_chunk_scan(cudaStream_t st, uint32_t* chunk_tot, const SegMeta& m, int nb_stride);
// seg_group: [nseg] group of every segment; pieces: scratch of
// (2 * nseg + ngroups) * r entries.  Three launches.
cudaError_t launch_cell_base(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                             const GroupMeta& gm, int ngroups, int nseg, const int32_t* seg_group, int r,
                             uint64_t* pieces, uint64_t* cell_base);
// Bucket-major cell bases (keys-only last level): buckets contiguous per
// group.  tot: scratch of ngroups * nb_stride entries.  Two launches.
cudaError_t launch_cell_base_bm(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                                const GroupMeta& gm, int ngroups, uint64_t* tot, uint64_t* cell_base);
cudaError_t launch_digit_base(cudaStream_t st, const uint32_t* seg_hist, int nb_stride,
                              const SegMeta& m, uint64_t* cell_base);
size_t scatter_smem_bytes(int nb_stride, int nspl_cap, int cells_cap, bool digit, bool vals,
                          bool stable);
// stable=false lets items of one tile land in any order inside their
// bucket run (keys-only last level / final partition: only membership matters).
cudaError_t launch_scatter(cudaStream_t st, const void* src, const void* src_vals, int kind,
                           bool digit, bool stable, void* dst, void* dst_vals, const SegMeta& m,
                           uint64_t nchunks, const uint8_t* blobs, const DigitCls* dcls,
                           int nspl_cap, int cells_cap, int nb_stride, const uint32_t* chunk_tot,
                           const uint64_t* cell_base, const uint8_t* ids, int id_bytes = 1);
// Stable level scatter from stored bucket ids whose bucket b lands in the
// buffer at device address bucket_dst[b] (values bucket_vdst[b]) at index
// cell_base[seg][b] + rank: the multi-GPU level 1 (peer buffers over NVLink).
cudaError_t launch_scatter_peers(cudaStream_t st, const void* src, const void* src_vals, int kind,
                                 const SegMeta& m, uint64_t nchunks, int nb_stride,
                                 const uint32_t* chunk_tot, const uint64_t* cell_base, const uint8_t* ids,
                                 int id_bytes, const uint64_t* bucket_dst, const uint64_t* bucket_vdst);
// Child-group key bounds [2*(g*r+t)] from parent bounds [2*g] and the plan.
cudaError_t launch_child_bounds(cudaStream_t st, const uint8_t* blobs, const GroupMeta& gm,
                                int ngroups, int r, const uint64_t* parent, uint64_t* child);
cudaError_t launch_gather_bounds(cudaStream_t st, const uint64_t* bounds, const int32_t* sel, int n,
                                 uint64_t* out);
cudaError_t launch_final_ranges(cudaStream_t st, const uint64_t* bounds, int nseg, int nb,
                                DigitCls* out);
// Counting + insertion sort of every cell; cells above the shared-memory
// capacity go to `ovf` (or are copied when constant), clustered cells to `fb`.
cudaError_t launch_smem_sort(cudaStream_t st, const void* src, const void* src_vals, void* out,
                             void* out_vals, int kind_out, const CellSource& cs, uint64_t ncells,
                             OverflowRec* ovf, unsigned int* ovf_count, OverflowRec* fb,
                             unsigned int* fb_count);
// LSD radix fallback for the `fb` records.
cudaError_t launch_smem_sort_lsd(cudaStream_t st, const void* src, const void* src_vals, void* out,
                                 void* out_vals, int kind_out, const CellSource& cs,
                                 uint64_t ncells);
// Fixed-capacity digit partition of bucket segments (keys only): cells of
// AMS_SMEM_SORT_CAP slots in dst, fill counts in `fill`, overflow flags per
// segment in seg_ovf (see k_scatter_fixed).
cudaError_t launch_scatter_fixed(cudaStream_t st, const void* src, int kind, void* dst,
                                 const SegMeta& m, uint64_t nchunks, int max_nb,
                                 const DigitCls* dcls, const uint32_t* cell0, uint32_t* fill,
                                 uint32_t* seg_ovf);
cudaError_t launch_fixed_cells(cudaStream_t st, const uint32_t* fill, const uint32_t* cell0,
                               const uint64_t* seg_off, const uint32_t* seg_ovf, int nseg,
                               uint64_t* out_base, uint32_t* cnt, uint32_t* cell_seg);
// seg_gb[3*s] = (group, bucket, digits) of every bucket segment.
cudaError_t launch_bucket_ranges(cudaStream_t st, const uint8_t* blobs, const uint64_t* gbounds,
                                 const int32_t* seg_gb, int nseg, DigitCls* out);
cudaError_t launch_map_keys(cudaStream_t st, const void* src, void* dst, uint64_t n, int from,
                            int to);

// RLM-sort selection (k_rlm.cu): one query = the element of rank `target`
// (1-based) among the members [first, first + npe) of a group; the members'
// cut positions go to cuts[out .. out + npe).
struct RlmQuery {
  int32_t first, npe;
  uint64_t target;
  uint64_t out;
};
cudaError_t launch_rlm_select(cudaStream_t st, const uint64_t* keys, const uint64_t* tags,
                              const uint64_t* pe_off, const RlmQuery* qs, int nq, uint64_t max_tag,
                              uint64_t* cuts, uint64_t* split_key);

}  // namespace ams
