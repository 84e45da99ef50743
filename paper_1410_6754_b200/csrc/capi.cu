// C ABI of the AMS-sort hot path: device context, metadata staging and the
// level / final-sort entry points declared in include/ams_b200.h.
#include <algorithm>
#include <unordered_map>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "ams_host.h"
#include "launch.h"

namespace ams {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace ams

#include "ctx.h"

namespace {

cudaEvent_t take_event(ams_ctx* c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one launch with events when timing is on; `bytes` is the
// launch's algorithmic traffic (what bench.py divides by the time).
struct KTimer {
  ams_ctx* c;
  int cat;
  double bytes;
  cudaEvent_t a = nullptr;
  KTimer(ams_ctx* c_, int cat_, double bytes_) : c(c_), cat(cat_), bytes(bytes_) {
    if (c->timing) {
      a = take_event(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~KTimer() {
    c->cat_launches[cat] += 1;
    if (a) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, c->stream);
      c->pending.push_back({cat, a, b, bytes});
    } else {
      c->cat_bytes[cat] += bytes;
    }
  }
};

void resolve_timing(ams_ctx* c) {
  const cudaEvent_t origin = c->pending.empty() ? nullptr : c->pending.front().a;
  for (auto& t : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(t.b);
    cudaEventElapsedTime(&ms, t.a, t.b);
    c->cat_ms[t.cat] += ms;
    c->cat_bytes[t.cat] += t.bytes;
    if (c->timeline.size() < (1u << 16)) {
      float t0 = 0.f, t1 = 0.f;
      cudaEventElapsedTime(&t0, origin, t.a);
      cudaEventElapsedTime(&t1, origin, t.b);
      c->timeline.push_back({t.cat, t0, t1});
    }
  }
  for (auto& t : c->pending) {
    c->free_events.push_back(t.a);
    c->free_events.push_back(t.b);
  }
  c->pending.clear();
}

// Chunk prefix of a segment list (a chunk = kChunk keys of one segment,
// one CTA of the histogram and scatter kernels).
void chunk_layout(const uint64_t* len, int nseg, uint64_t chunk, std::vector<uint64_t>& chunk_prefix) {
  chunk_prefix.assign(nseg + 1, 0);
  for (int s = 0; s < nseg; ++s)
    chunk_prefix[s + 1] = chunk_prefix[s] + (len[s] + chunk - 1) / chunk;
}

// Keys per chunk: kChunk for inputs that fill the GPU several times over,
// fewer (whole tiles) for small inputs so that about kFillCtas CTAs exist
// (config 1 at 2^20 keys has 16 chunks of kChunk: a tenth of the SMs); with
// many buckets a chunk stays >= 4 keys per bucket (its histogram row is
// nb_stride words of scan work).
constexpr uint64_t kFillCtas = 148 * 8;
uint32_t pick_chunk(const uint64_t* len, int nseg, int nb_stride, uint64_t max_chunk) {
  uint64_t total = 0;
  for (int s = 0; s < nseg; ++s) total += len[s];
  uint64_t c = (total / kFillCtas + kTile - 1) / kTile * kTile;
  c = std::max<uint64_t>(c, (uint64_t)kTile);
  c = std::max<uint64_t>(c, std::min<uint64_t>(max_chunk, 4 * (uint64_t)std::max(nb_stride, 1) / kTile * kTile));
  return (uint32_t)std::min<uint64_t>(c, max_chunk);
}

// Upload a segment table; returns the device-side SegMeta.
cudaError_t upload_segments(Stage& st, cudaStream_t stream, const uint64_t* off,
                            const uint64_t* len, const int32_t* cls, int nseg,
                            const int64_t* posbase, int ncls, SegMeta* m, uint64_t* nchunks,
                            int nb_stride, uint64_t max_chunk = kChunk) {
  std::vector<uint64_t> cp;
  m->chunk = pick_chunk(len, nseg, nb_stride, max_chunk);
  chunk_layout(len, nseg, m->chunk, cp);
  st.reset();
  const size_t o_off = st.put(off, nseg), o_len = st.put(len, nseg), o_cls = st.put(cls, nseg);
  const size_t o_cp = st.put(cp);
  const size_t o_pb = posbase ? st.put(posbase, ncls) : 0;
  cudaError_t e = st.upload(stream);
  if (e != cudaSuccess) return e;
  m->off = st.dev<uint64_t>(o_off);
  m->len = st.dev<uint64_t>(o_len);
  m->cls = st.dev<int32_t>(o_cls);
  m->chunk_prefix = st.dev<uint64_t>(o_cp);
  m->posbase = posbase ? st.dev<int64_t>(o_pb) : nullptr;
  m->nseg = nseg;
  m->tags = nullptr;
  *nchunks = cp[nseg];
  return cudaSuccess;
}

// Histogram pass (classify -> chunk and segment histograms) then the chunk
// scan, for a segment table whose classifiers are ready.
int run_histogram(ams_ctx* c, const void* src, int kind, bool digit, const SegMeta& m,
                  uint64_t nchunks, int nb_stride, const DigitCls* dcls,
                  unsigned long long* minmax, uint64_t nelems, uint8_t* ids, int id_bytes = 1) {
  AMS_CK(c->chunk_tot.ensure(sizeof(uint32_t) * std::max<uint64_t>(nchunks, 1) * nb_stride));
  AMS_CK(c->seg_hist.ensure(sizeof(uint32_t) * (size_t)std::max(m.nseg, 1) * nb_stride));
  AMS_CK(cudaMemsetAsync(c->seg_hist.p, 0, sizeof(uint32_t) * (size_t)m.nseg * nb_stride, c->stream));
  {
    KTimer kt(c, digit ? AMS_KCAT_FHIST : AMS_KCAT_HIST, 8.0 * nelems);
    AMS_CK(launch_hist(c->stream, src, kind, digit, m, nchunks, c->blobs.as<uint8_t>(), dcls,
                       c->nspl_cap, c->cells_cap, nb_stride, c->chunk_tot.as<uint32_t>(),
                       c->seg_hist.as<uint32_t>(), minmax, ids, id_bytes));
  }
  {
    KTimer kt(c, AMS_KCAT_CHUNKSCAN, 8.0 * nchunks * nb_stride);
    AMS_CK(launch_chunk_scan(c->stream, c->chunk_tot.as<uint32_t>(), m, nb_stride));
  }
  c->launches += 2;
  return AMS_OK;
}

int level_scatter_impl(ams_ctx_t* c, const void* src, const void* src_vals, int key_kind,
                       void* dst, void* dst_vals, int r, const uint64_t* h_boundaries,
                       const uint64_t* h_group_dst_start, int child_first, int child_count,
                       bool bucket_major);
int level_sample_impl(ams_ctx_t* c, const void* src, int key_kind, uint64_t count,
                      const uint64_t* h_idx, const uint64_t* h_gpos, uint64_t* d_out_keys,
                      uint32_t* d_out_pos, const uint64_t* tags);

}  // namespace

extern "C" {

const char* ams_last_error(void) { return g_last_error.c_str(); }
int ams_version(void) { return 1; }

int ams_ctx_create(int device, void* stream, ams_ctx_t** out) {
  if (!out) return set_error(AMS_EINVAL, "null output pointer");
  int ndev = 0;
  AMS_CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return set_error(AMS_EINVAL, "device " + std::to_string(device) + " out of range");
  AMS_ON_DEVICE(device);
  ams_ctx* c = new ams_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  if (const char* e = std::getenv("AMS_HOST_TRACE")) c->host_trace = std::atoi(e) != 0;
  *out = c;
  return AMS_OK;
}

int ams_ctx_destroy(ams_ctx_t* c) {
  if (!c) return AMS_OK;
  DeviceGuard dg(c->device);
  cudaStreamSynchronize(c->stream);
  resolve_timing(c);
  for (cudaEvent_t e : c->free_events) cudaEventDestroy(e);
  for (Stage* s : {&c->st_sample, &c->st_split, &c->st_level, &c->st_scatter, &c->st_final, &c->st_fixed,
                   &c->st_copy, &c->st_rlm})
    s->release();
  for (DevBuf* b : {&c->blobs, &c->sorted_keys, &c->sorted_pos, &c->sample_idx, &c->bounds[0], &c->bounds[1],
                    &c->chunk_tot, &c->seg_hist, &c->cell_base, &c->pieces, &c->minmax, &c->dcls,
                    &c->ovf, &c->ovf_count, &c->fb, &c->fb_count,
                    &c->ids, &c->work[0], &c->work[1], &c->work_v[0], &c->work_v[1], &c->s_keys,
                    &c->s_pos, &c->fx_scratch, &c->fx_fill, &c->fx_ovf, &c->fx_base, &c->fx_cnt,
                    &c->fx_seg, &c->tags0, &c->rank_tmp_keys, &c->rank_tmp_pos, &c->rlm_buf[0],
                    &c->rlm_buf[1], &c->rlm_buf[2], &c->rlm_cuts, &c->rlm_skey})
    b->release();
  for (auto& po : c->peer_open) cudaIpcCloseMemHandle(po.second);
  for (DevBuf& b : c->peer_buf) b.release();
  c->st_peers.release();
  c->h_hist.release();
  c->h_small.release();
  c->h_big.release();
  delete c;
  return AMS_OK;
}

int ams_ctx_set_stream(ams_ctx_t* c, void* stream) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  c->stream = static_cast<cudaStream_t>(stream);
  return AMS_OK;
}

uint64_t ams_ctx_launches(const ams_ctx_t* c) { return c ? c->launches : 0; }

int ams_ctx_set_timing(ams_ctx_t* c, int enable) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  c->timing = enable != 0;
  return AMS_OK;
}

int ams_ctx_kernel_stats(ams_ctx_t* c, double* ms, double* bytes, uint64_t* launches, int ncat) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  AMS_ON_DEVICE(c->device);
  resolve_timing(c);
  for (int i = 0; i < ncat && i < AMS_NUM_KCAT; ++i) {
    if (ms) ms[i] = c->cat_ms[i];
    if (bytes) bytes[i] = c->cat_bytes[i];
    if (launches) launches[i] = c->cat_launches[i];
  }
  return AMS_OK;
}

int ams_ctx_timeline(ams_ctx_t* c, int* cat, float* t0, float* t1, int cap, int* count) {
  if (!c || !count) return set_error(AMS_EINVAL, "null argument");
  AMS_ON_DEVICE(c->device);
  resolve_timing(c);
  const int n = (int)std::min<size_t>(c->timeline.size(), (size_t)std::max(cap, 0));
  for (int i = 0; i < n; ++i) {
    if (cat) cat[i] = c->timeline[i].cat;
    if (t0) t0[i] = c->timeline[i].t0;
    if (t1) t1[i] = c->timeline[i].t1;
  }
  *count = (int)c->timeline.size();
  c->timeline.clear();
  return AMS_OK;
}

int ams_ctx_reset_stats(ams_ctx_t* c) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  AMS_ON_DEVICE(c->device);
  resolve_timing(c);
  for (int i = 0; i < AMS_NUM_KCAT; ++i) { c->cat_ms[i] = 0; c->cat_bytes[i] = 0; c->cat_launches[i] = 0; }
  c->timeline.clear();
  return AMS_OK;
}

int ams_ctx_sync(ams_ctx_t* c) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  AMS_ON_DEVICE(c->device);
  AMS_CK(cudaStreamSynchronize(c->stream));
  return AMS_OK;
}

int ams_level_sample(ams_ctx_t* c, const void* src, int key_kind, uint64_t count,
                     const uint64_t* h_idx, const uint64_t* h_gpos, uint64_t* d_out_keys,
                     uint32_t* d_out_pos) {
  return level_sample_impl(c, src, key_kind, count, h_idx, h_gpos, d_out_keys, d_out_pos, nullptr);
}

}  // extern "C"

namespace {

// tags != NULL: the sample's tie-break value is its origin tag.
int level_sample_impl(ams_ctx_t* c, const void* src, int key_kind, uint64_t count,
                      const uint64_t* h_idx, const uint64_t* h_gpos, uint64_t* d_out_keys,
                      uint32_t* d_out_pos, const uint64_t* tags) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (count == 0) return AMS_OK;
  if (!src || !h_idx || !h_gpos || !d_out_keys || !d_out_pos)
    return set_error(AMS_EINVAL, "null argument");
  AMS_ON_DEVICE(c->device);
  Stage& st = c->st_sample;
  st.reset();
  const size_t oi = st.put(h_idx, count), og = st.put(h_gpos, count);
  AMS_CK(st.upload(c->stream));
  {
    KTimer kt(c, AMS_KCAT_SAMPLE, 12.0 * count);
    AMS_CK(launch_gather_sample(c->stream, src, key_kind, st.dev<uint64_t>(oi),
                                st.dev<uint64_t>(og), count, d_out_keys, d_out_pos, tags));
  }
  c->launches += 1;
  return AMS_OK;
}

}  // namespace

extern "C" {

int ams_level_splitters(ams_ctx_t* c, int ngroups, const uint64_t* d_sample_keys,
                        const uint32_t* d_sample_pos, const uint64_t* h_soff, const int32_t* h_nb) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (ngroups < 1 || !h_soff || !h_nb) return set_error(AMS_EINVAL, "bad group list");
  AMS_ON_DEVICE(c->device);
  uint64_t max_s = 0;
  int max_nb = 1, cells_cap = 1;
  for (int g = 0; g < ngroups; ++g) {
    const uint64_t S = h_soff[g + 1] - h_soff[g];
    const int nb = h_nb[g];
    if (h_soff[g + 1] < h_soff[g]) return set_error(AMS_EINVAL, "sample offsets not ascending");
    if (nb < 1 || nb > AMS_MAX_BUCKETS)
      return set_error(AMS_EINVAL, "bucket count " + std::to_string(nb) + " outside 1.." +
                                       std::to_string(AMS_MAX_BUCKETS));
    if (S < (uint64_t)(nb - 1))  // ams.py:186-187
      return set_error(AMS_EINVAL, "sample of " + std::to_string(S) + " too small for " +
                                       std::to_string(nb) + " buckets");
    max_s = std::max(max_s, S);
    max_nb = std::max(max_nb, nb);
    if (nb > 1) cells_cap = std::max(cells_cap, 1 << lut_bits_for(nb - 1));
  }
  const uint64_t total = h_soff[ngroups];
  if (total > 0 && (!d_sample_keys || !d_sample_pos)) return set_error(AMS_EINVAL, "null sample");
  Stage& st = c->st_split;
  st.reset();
  const size_t os = st.put(h_soff, ngroups + 1), on = st.put(h_nb, ngroups);
  AMS_CK(st.upload(c->stream));
  AMS_CK(c->blobs.ensure(kBlobStride * (size_t)ngroups));
  AMS_CK(c->sorted_keys.ensure(sizeof(uint64_t) * std::max<uint64_t>(total, 1)));
  AMS_CK(c->sorted_pos.ensure(sizeof(uint32_t) * std::max<uint64_t>(total, 1)));
  {
    KTimer kt(c, AMS_KCAT_RANK, 24.0 * total);
    uint64_t* tk = nullptr;
    uint32_t* tp = nullptr;
    if (max_s > kSampleRankPairsMax) {
      AMS_CK(c->rank_tmp_keys.ensure(sizeof(uint64_t) * total));
      AMS_CK(c->rank_tmp_pos.ensure(sizeof(uint32_t) * total));
      tk = c->rank_tmp_keys.as<uint64_t>();
      tp = c->rank_tmp_pos.as<uint32_t>();
    }
    AMS_CK(launch_sample_rank(c->stream, ngroups, max_s, d_sample_keys, d_sample_pos,
                              st.dev<uint64_t>(os), c->sorted_keys.as<uint64_t>(),
                              c->sorted_pos.as<uint32_t>(), tk, tp));
  }
  {
    KTimer kt(c, AMS_KCAT_CLS, 12.0 * total);
    AMS_CK(launch_build_cls(c->stream, ngroups, c->sorted_keys.as<uint64_t>(),
                            c->sorted_pos.as<uint32_t>(), st.dev<uint64_t>(os),
                            st.dev<int32_t>(on), c->blobs.as<uint8_t>()));
  }
  c->launches += (max_s ? 1 : 0) + 1;
  c->group_nb.assign(h_nb, h_nb + ngroups);
  c->ngroups = ngroups;
  c->nspl_cap = max_nb - 1;
  c->cells_cap = cells_cap;
  return AMS_OK;
}

int ams_read_splitters(ams_ctx_t* c, int group, uint64_t* keys, uint32_t* pos, int* nspl) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (group < 0 || group >= c->ngroups) return set_error(AMS_EINVAL, "group out of range");
  AMS_ON_DEVICE(c->device);
  ClsHeader h;
  const uint8_t* blob = c->blobs.as<uint8_t>() + (size_t)group * kBlobStride;
  AMS_CK(cudaMemcpyAsync(&h, blob, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  AMS_CK(cudaStreamSynchronize(c->stream));
  if (nspl) *nspl = (int)h.nspl;
  if (h.nspl) {
    if (keys) AMS_CK(cudaMemcpy(keys, blob + kBlobKeys, 8 * (size_t)h.nspl, cudaMemcpyDeviceToHost));
    if (pos) AMS_CK(cudaMemcpy(pos, blob + kBlobPos, 4 * (size_t)h.nspl, cudaMemcpyDeviceToHost));
  }
  return AMS_OK;
}

int ams_level_classify(ams_ctx_t* c, const void* src, int key_kind, int nseg,
                       const uint64_t* h_seg_off, const uint64_t* h_seg_len,
                       const int32_t* h_seg_group, int ngroups, const int64_t* h_group_posbase,
                       int nb_stride, int track_minmax, int stable, uint32_t* h_seg_hist_out) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (nseg < 1 || !h_seg_off || !h_seg_len || !h_seg_group || !h_group_posbase)
    return set_error(AMS_EINVAL, "bad segment list");
  if (ngroups != c->ngroups)
    return set_error(AMS_EINVAL, "group count differs from the last ams_level_splitters call");
  int max_nb = 1;
  for (int g = 0; g < ngroups; ++g) max_nb = std::max(max_nb, c->group_nb[g]);
  if (nb_stride < max_nb) return set_error(AMS_EINVAL, "nb_stride smaller than the bucket count");
  AMS_ON_DEVICE(c->device);
  // Groups are contiguous runs of segments.
  c->group_first.assign(ngroups, -1);
  c->group_nseg.assign(ngroups, 0);
  for (int s = 0; s < nseg; ++s) {
    const int g = h_seg_group[s];
    if (g < 0 || g >= ngroups) return set_error(AMS_EINVAL, "segment group out of range");
    if (s > 0 && g < h_seg_group[s - 1]) return set_error(AMS_EINVAL, "segments not group-major");
    if (c->group_first[g] < 0) c->group_first[g] = s;
    c->group_nseg[g] += 1;
  }
  for (int g = 0; g < ngroups; ++g) {
    if (c->group_nseg[g] == 0) return set_error(AMS_EINVAL, "group without segments");
    uint64_t n_g = 0;
    for (int j = 0; j < c->group_nseg[g]; ++j) n_g += h_seg_len[c->group_first[g] + j];
    if (n_g >= 0xFFFFFFFFull) return set_error(AMS_EINVAL, "group too large for 32-bit positions");
  }
  AMS_CK(upload_segments(c->st_level, c->stream, h_seg_off, h_seg_len, h_seg_group, nseg,
                         h_group_posbase, ngroups, &c->meta, &c->nchunks, nb_stride));
  c->meta.tags = c->level_tags;  // origin tags of this level's buffer (deterministic, levels >= 2)
  c->nseg = nseg;
  c->nb_stride = nb_stride;
  unsigned long long* mm = nullptr;
  if (track_minmax) {
    AMS_CK(c->minmax.ensure(16));
    // {min, max} = {~0, 0}: two byte fills, no host round trip.
    AMS_CK(cudaMemsetAsync(c->minmax.p, 0xFF, 8, c->stream));
    AMS_CK(cudaMemsetAsync(static_cast<uint8_t*>(c->minmax.p) + 8, 0, 8, c->stream));
    mm = c->minmax.as<unsigned long long>();
  }
  uint64_t nel = 0;
  for (int s = 0; s < nseg; ++s) nel += h_seg_len[s];
  c->level_elems = nel;
  c->level_stable = stable != 0;
  // The histogram pass also stores each key's bucket at its buffer index (a
  // byte up to 256 buckets, else 16 bits); the scatter reads it instead of
  // classifying again.
  uint8_t* ids = nullptr;
  int id_bytes = nb_stride <= 256 ? 1 : 2;  // u16 ids up to AMS_MAX_BUCKETS buckets
  {
    uint64_t span = 0;
    for (int s = 0; s < nseg; ++s) span = std::max(span, h_seg_off[s] + h_seg_len[s]);
    AMS_CK(c->ids.ensure((size_t)id_bytes * std::max<uint64_t>(span, 1)));
    ids = c->ids.as<uint8_t>();
  }
  c->level_ids = ids != nullptr;
  c->level_id_bytes = id_bytes;
  int rc = run_histogram(c, src, key_kind, false, c->meta, c->nchunks, nb_stride, nullptr, mm,
                         nel, ids, id_bytes);
  if (rc) return rc;
  if (track_minmax) {
    // The whole input is one group at the first level: its bounds are the
    // global key range.
    AMS_CK(c->bounds[0].ensure(16 * (size_t)ngroups));
    AMS_CK(launch_copy_bytes(c->stream, c->bounds[0].p, c->minmax.p, 16));
    c->bcur = 0;
  } else if (!c->bounds[c->bcur].p || c->bounds[c->bcur].cap < 16 * (size_t)ngroups) {
    return set_error(AMS_EINVAL, "no key bounds for these groups (first level needs track_minmax)");
  }
  const size_t hb = sizeof(uint32_t) * (size_t)nseg * nb_stride;
  AMS_CK(to_host(c->h_hist, c->seg_hist.p, hb, c->stream));
  AMS_CK(cudaStreamSynchronize(c->stream));
  if (h_seg_hist_out) std::memcpy(h_seg_hist_out, c->h_hist.p, hb);
  return AMS_OK;
}

int ams_level_scatter(ams_ctx_t* c, const void* src, const void* src_vals, int key_kind,
                      void* dst, void* dst_vals, int r, const uint64_t* h_boundaries,
                      const uint64_t* h_group_dst_start, int child_first, int child_count) {
  return level_scatter_impl(c, src, src_vals, key_kind, dst, dst_vals, r, h_boundaries,
                            h_group_dst_start, child_first, child_count, false);
}

}  // extern "C"

namespace {

// bucket_major (keys-only last level of ams_sort_run): cells in (g, b, j)
// order instead of (g(b), j, b) — same children extents, buckets contiguous.
int level_scatter_impl(ams_ctx_t* c, const void* src, const void* src_vals, int key_kind,
                       void* dst, void* dst_vals, int r, const uint64_t* h_boundaries,
                       const uint64_t* h_group_dst_start, int child_first, int child_count,
                       bool bucket_major) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (c->nseg == 0) return set_error(AMS_EINVAL, "ams_level_classify must run first");
  if (r < 1 || !h_boundaries || !h_group_dst_start) return set_error(AMS_EINVAL, "bad plan");
  if ((src_vals == nullptr) != (dst_vals == nullptr))
    return set_error(AMS_EINVAL, "values must be given for both source and destination");
  const int G = c->ngroups;
  if (child_first < 0 || child_count < 0 || child_first + child_count > G * r)
    return set_error(AMS_EINVAL, "child group range outside the level's children");
  AMS_ON_DEVICE(c->device);
  for (int g = 0; g < G; ++g) {
    const uint64_t* b = h_boundaries + (size_t)g * (r + 1);
    if (b[0] != 0 || b[r] != (uint64_t)c->group_nb[g])
      return set_error(AMS_EINVAL, "plan boundaries do not cover the buckets");
    for (int i = 0; i < r; ++i)
      if (b[i + 1] < b[i]) return set_error(AMS_EINVAL, "plan boundaries not ascending");
  }
  Stage& st = c->st_scatter;
  st.reset();
  const size_t of = st.put(c->group_first), on = st.put(c->group_nseg);
  const size_t ob = st.put(h_boundaries, (size_t)G * (r + 1));
  const size_t od = st.put(h_group_dst_start, G);
  AMS_CK(st.upload(c->stream));
  GroupMeta gm;
  gm.first = st.dev<int32_t>(of);
  gm.nseg = st.dev<int32_t>(on);
  gm.bnd = st.dev<uint64_t>(ob);
  gm.dst_start = st.dev<uint64_t>(od);
  const bool bm = bucket_major && !c->level_stable && !src_vals;
  AMS_CK(c->pieces.ensure(sizeof(uint64_t) * std::max((size_t)(2 * c->nseg + G) * r,
                                                      (size_t)G * c->nb_stride)));
  AMS_CK(c->cell_base.ensure(sizeof(uint64_t) * (size_t)c->nseg * c->nb_stride));
  {
    KTimer kt(c, AMS_KCAT_CELLBASE, 12.0 * c->nseg * c->nb_stride);
    if (bm)
      AMS_CK(launch_cell_base_bm(c->stream, c->seg_hist.as<uint32_t>(), c->nb_stride, gm, G,
                                 c->pieces.as<uint64_t>(), c->cell_base.as<uint64_t>()));
    else
      AMS_CK(launch_cell_base(c->stream, c->seg_hist.as<uint32_t>(), c->nb_stride, gm, G, c->nseg,
                              c->meta.cls, r, c->pieces.as<uint64_t>(), c->cell_base.as<uint64_t>()));
    c->launches += bm ? 1 : 2;
  }
  {
    KTimer kt(c, c->level_stable ? AMS_KCAT_SCATTER : AMS_KCAT_SCATTER_U,
              (src_vals ? 32.0 : 16.0) * c->level_elems);
    AMS_CK(launch_scatter(c->stream, src, src_vals, key_kind, false, c->level_stable, dst,
                          dst_vals, c->meta, c->nchunks, c->blobs.as<uint8_t>(), nullptr,
                          c->nspl_cap, c->cells_cap, c->nb_stride, c->chunk_tot.as<uint32_t>(),
                          c->cell_base.as<uint64_t>(), c->level_ids ? c->ids.as<uint8_t>() : nullptr,
                          c->level_id_bytes));
  }
  // Key bounds of the next level's groups (this rank's children).
  const int nxt = 1 - c->bcur;
  AMS_CK(c->bounds[nxt].ensure(16 * (size_t)std::max(G * r, 1)));
  {
    KTimer kt(c, AMS_KCAT_RANGES, 0.0);
    AMS_CK(launch_child_bounds(c->stream, c->blobs.as<uint8_t>(), gm, G, r,
                               c->bounds[c->bcur].as<uint64_t>(), c->bounds[nxt].as<uint64_t>()));
  }
  if (child_first > 0 && child_count > 0)
    AMS_CK(launch_copy_bytes(c->stream, c->bounds[nxt].p, c->bounds[nxt].as<uint64_t>() + 2 * child_first,
                             16 * (size_t)child_count));
  c->bcur = nxt;
  c->launches += 3;
  return AMS_OK;
}

}  // namespace

extern "C" {

int ams_peer_buffer(ams_ctx_t* c, int slot, uint64_t bytes, void** dptr, void* ipc_handle, int* grown) {
  if (!c || !dptr || !ipc_handle) return set_error(AMS_EINVAL, "null argument");
  if (slot < 0 || slot >= 8) return set_error(AMS_EINVAL, "peer buffer slot outside 0..7");
  AMS_ON_DEVICE(c->device);
  DevBuf& b = c->peer_buf[slot];
  const bool grow = bytes > b.cap || !b.p;
  if (grow) AMS_CK(b.ensure(std::max<uint64_t>(bytes, 256)));
  cudaIpcMemHandle_t h;
  AMS_CK(cudaIpcGetMemHandle(&h, b.p));
  std::memcpy(ipc_handle, &h, sizeof h);
  *dptr = b.p;
  if (grown) *grown = grow ? 1 : 0;
  return AMS_OK;
}

int ams_peer_open(ams_ctx_t* c, const void* ipc_handle, void** dptr) {
  if (!c || !ipc_handle || !dptr) return set_error(AMS_EINVAL, "null argument");
  AMS_ON_DEVICE(c->device);
  const std::string key(static_cast<const char*>(ipc_handle), sizeof(cudaIpcMemHandle_t));
  for (const auto& po : c->peer_open)
    if (po.first == key) { *dptr = po.second; return AMS_OK; }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof h);
  void* p = nullptr;
  AMS_CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  c->peer_open.emplace_back(key, p);
  *dptr = p;
  return AMS_OK;
}

int ams_peer_close_all(ams_ctx_t* c) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  AMS_ON_DEVICE(c->device);
  AMS_CK(cudaStreamSynchronize(c->stream));
  for (auto& po : c->peer_open) AMS_CK(cudaIpcCloseMemHandle(po.second));
  c->peer_open.clear();
  return AMS_OK;
}

int ams_level_scatter_peers(ams_ctx_t* c, const void* src, const void* src_vals, int key_kind, int ndst,
                            void* const* dst, void* const* dst_vals, const int32_t* bucket_dst,
                            const uint64_t* cell_base, int r, const uint64_t* h_boundaries, int child_first,
                            int child_count) {
  if (!c || !src || !dst || !bucket_dst || !cell_base || !h_boundaries) return set_error(AMS_EINVAL, "null argument");
  if (c->nseg == 0) return set_error(AMS_EINVAL, "ams_level_classify must run first");
  if (c->ngroups != 1) return set_error(AMS_EINVAL, "the peer scatter takes a single-group level");
  if ((src_vals == nullptr) != (dst_vals == nullptr))
    return set_error(AMS_EINVAL, "values must be given for both source and destination");
  if (!c->level_stable || !c->level_ids) return set_error(AMS_EINVAL, "the peer scatter is stable, from stored ids");
  if (r < 1 || child_first < 0 || child_count < 0 || child_first + child_count > r)
    return set_error(AMS_EINVAL, "child group range outside the level's children");
  AMS_ON_DEVICE(c->device);
  const int nb = c->nb_stride;
  std::vector<uint64_t> bd(nb), bvd(nb, 0);
  for (int b = 0; b < nb; ++b) {
    const int d = bucket_dst[b];
    if (d < 0 || d >= ndst) return set_error(AMS_EINVAL, "bucket destination out of range");
    bd[b] = reinterpret_cast<uint64_t>(dst[d]);
    if (src_vals) bvd[b] = reinterpret_cast<uint64_t>(dst_vals[d]);
  }
  Stage& st = c->st_peers;
  st.reset();
  const size_t oc = st.put(cell_base, (size_t)c->nseg * nb), ob = st.put(bd), ov = st.put(bvd);
  const size_t oq = st.put(h_boundaries, (size_t)r + 1);
  const int32_t zero = 0, one = 1;
  const size_t of = st.put(&zero, 1), on = st.put(&one, 1), os = st.put(&cell_base[0], 1);
  AMS_CK(st.upload(c->stream));
  {
    KTimer kt(c, AMS_KCAT_SCATTER, (src_vals ? 32.0 : 16.0) * c->level_elems);
    AMS_CK(launch_scatter_peers(c->stream, src, src_vals, key_kind, c->meta, c->nchunks, nb,
                                c->chunk_tot.as<uint32_t>(), st.dev<uint64_t>(oc), c->ids.as<uint8_t>(),
                                c->level_id_bytes, st.dev<uint64_t>(ob), src_vals ? st.dev<uint64_t>(ov) : nullptr));
  }
  // Key bounds of this rank's children (the later levels' groups).
  GroupMeta gm;
  gm.first = st.dev<int32_t>(of);
  gm.nseg = st.dev<int32_t>(on);
  gm.bnd = st.dev<uint64_t>(oq);
  gm.dst_start = st.dev<uint64_t>(os);
  const int nxt = 1 - c->bcur;
  AMS_CK(c->bounds[nxt].ensure(16 * (size_t)std::max(r, 1)));
  AMS_CK(launch_child_bounds(c->stream, c->blobs.as<uint8_t>(), gm, 1, r, c->bounds[c->bcur].as<uint64_t>(),
                             c->bounds[nxt].as<uint64_t>()));
  if (child_first > 0 && child_count > 0)
    AMS_CK(launch_copy_bytes(c->stream, c->bounds[nxt].p, c->bounds[nxt].as<uint64_t>() + 2 * child_first,
                             16 * (size_t)child_count));
  c->bcur = nxt;
  c->launches += 2;
  return AMS_OK;
}

int ams_copy_ranges(ams_ctx_t* c, const uint64_t* h_ranges, int nranges, const void* src, void* dst,
                    const void* src_vals, void* dst_vals) {
  if (!c || nranges < 0 || (nranges && (!h_ranges || !src || !dst))) return set_error(AMS_EINVAL, "null argument");
  if ((src_vals == nullptr) != (dst_vals == nullptr))
    return set_error(AMS_EINVAL, "values must be given for both source and destination");
  if (nranges == 0) return AMS_OK;
  AMS_ON_DEVICE(c->device);
  // One work item (CTA) per kCopyItemKeys keys of a range.
  std::vector<uint64_t> items;
  uint64_t total = 0;
  for (int q = 0; q < nranges; ++q) {
    const uint64_t s0 = h_ranges[3 * q], d0 = h_ranges[3 * q + 1], len = h_ranges[3 * q + 2];
    total += len;
    for (uint64_t o = 0; o < len; o += kCopyItemKeys) {
      items.push_back(s0 + o);
      items.push_back(d0 + o);
      items.push_back(std::min<uint64_t>(kCopyItemKeys, len - o));
    }
  }
  if (items.empty()) return AMS_OK;
  Stage& sc = c->st_copy;
  sc.reset();
  const size_t oi = sc.put(items);
  AMS_CK(sc.upload(c->stream));
  KTimer kt(c, AMS_KCAT_SCATTER, (src_vals ? 32.0 : 16.0) * (double)total);
  AMS_CK(launch_copy_ranges(c->stream, sc.dev<uint64_t>(oi), (int)(items.size() / 3), src, dst, src_vals,
                            dst_vals, total));
  c->launches += 1;
  return AMS_OK;
}

int ams_fill_iota(ams_ctx_t* c, void* dst, uint64_t n, uint64_t start) {
  if (!c || (n && !dst)) return set_error(AMS_EINVAL, "null argument");
  AMS_ON_DEVICE(c->device);
  AMS_CK(launch_iota(c->stream, dst, n, start));
  c->launches += n ? 1 : 0;
  return AMS_OK;
}

int ams_get_minmax(ams_ctx_t* c, uint64_t out[2]) {
  if (!c || !out) return set_error(AMS_EINVAL, "null argument");
  if (!c->minmax.p) return set_error(AMS_EINVAL, "no min/max recorded");
  AMS_ON_DEVICE(c->device);
  AMS_CK(to_host(c->h_small, c->minmax.p, 16, c->stream));
  AMS_CK(cudaStreamSynchronize(c->stream));
  std::memcpy(out, c->h_small.p, 16);
  return AMS_OK;
}

int ams_set_minmax(ams_ctx_t* c, const uint64_t in[2]) {
  if (!c || !in) return set_error(AMS_EINVAL, "null argument");
  AMS_ON_DEVICE(c->device);
  AMS_CK(c->minmax.ensure(16));
  AMS_CK(c->h_small.ensure(64));
  AMS_CK(cudaStreamSynchronize(c->stream));
  std::memcpy(c->h_small.p, in, 16);
  AMS_CK(launch_copy_bytes(c->stream, c->minmax.p, c->h_small.dp, 16));
  AMS_CK(c->bounds[c->bcur].ensure(16));
  AMS_CK(launch_copy_bytes(c->stream, c->bounds[c->bcur].p, c->minmax.p, 16));
  return AMS_OK;
}

namespace {

// Counting sort of a cell list into `out`, then the LSD fallback for the
// cells whose keys cluster.  Syncs once to learn the fallback count.
// Cells of the clustered-key fallback list (k_smem_sort_lsd) launched
// speculatively when the caller defers the host read of the list's length.
constexpr unsigned int kSpecFallback = 256;

// slot >= 0 defers the read of the fallback count: the call uses fallback
// list `slot` (records at fb + slot * fb_stride, count at fb_count[slot]),
// launches the LSD kernel for the first kSpecFallback records with the count
// read on the device, and the caller finishes with finish_fallback() after
// its own synchronisation — no host round trip here.
int sort_cells(ams_ctx* c, const void* src, const void* src_vals, void* out, void* out_vals,
               int key_kind, const CellSource& cs, uint64_t ncells, uint64_t nelems, int slot = -1,
               uint64_t fb_stride = 0) {
  const bool vals = src_vals != nullptr;
  const bool defer = slot >= 0;
  unsigned int* cnt = c->fb_count.as<unsigned int>() + (defer ? slot : 0);
  OverflowRec* recs = c->fb.as<OverflowRec>() + (defer ? (size_t)slot * fb_stride : 0);
  AMS_CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned int), c->stream));
  {
    KTimer kt(c, AMS_KCAT_SMEMSORT, (vals ? 32.0 : 16.0) * nelems);
    AMS_CK(launch_smem_sort(c->stream, src, src_vals, out, out_vals, key_kind, cs, ncells,
                            c->ovf.as<OverflowRec>(), c->ovf_count.as<unsigned int>(), recs, cnt));
  }
  c->launches += 1;
  CellSource fc{};
  fc.mode = 2;
  fc.recs = recs;
  if (defer) {
    fc.nrecs = cnt;
    KTimer kt(c, AMS_KCAT_SMEMSORT, 0.0);
    AMS_CK(launch_smem_sort_lsd(c->stream, src, src_vals, out, out_vals, key_kind, fc,
                                std::min<uint64_t>(ncells, kSpecFallback)));
    c->launches += 1;
    return AMS_OK;
  }
  unsigned int nfb = 0;
  AMS_CK(to_host(c->h_small, cnt, sizeof nfb, c->stream));
  AMS_CK(cudaStreamSynchronize(c->stream));
  std::memcpy(&nfb, c->h_small.p, sizeof nfb);
  c->fallback_cells += nfb;
  if (nfb) {
    KTimer kt(c, AMS_KCAT_SMEMSORT, 0.0);
    AMS_CK(launch_smem_sort_lsd(c->stream, src, src_vals, out, out_vals, key_kind, fc, nfb));
    c->launches += 1;
  }
  return AMS_OK;
}

// After a deferred sort_cells and the caller's synchronisation: `nfb` is
// the list's length (read by the caller); records past the speculative
// launch are sorted now.
int finish_fallback(ams_ctx* c, const void* src, void* out, int key_kind, int slot, uint64_t fb_stride,
                    unsigned int nfb) {
  c->fallback_cells += nfb;
  if (nfb <= kSpecFallback) return AMS_OK;
  CellSource fc{};
  fc.mode = 2;
  fc.recs = c->fb.as<OverflowRec>() + (size_t)slot * fb_stride + kSpecFallback;
  KTimer kt(c, AMS_KCAT_SMEMSORT, 0.0);
  AMS_CK(launch_smem_sort_lsd(c->stream, src, nullptr, out, nullptr, key_kind, fc, nfb - kSpecFallback));
  c->launches += 1;
  return AMS_OK;
}

// Exact digit-partition rounds over segments that exceed shared memory:
// histogram + stable scatter cur -> oth, then per-cell sorts into `out`;
// cells still too big go round again with their exact key range.  Key
// bounds of the first round come from the last level's bounds (`sel` =
// final segment index of every entry) or, without `sel`, from lo/hi.
int partition_rounds(ams_ctx* c, void* src, void* src_vals, void* tmp, void* tmp_vals, void* out,
                     void* out_vals, int key_kind, std::vector<uint64_t>& b_off,
                     std::vector<uint64_t>& b_len, std::vector<uint64_t>& b_lo,
                     std::vector<uint64_t>& b_hi, const std::vector<int32_t>* sel) {
  const bool vals = src_vals != nullptr;
  constexpr uint64_t kTargetCell = AMS_SMEM_SORT_CAP * 78 / 100;
  uint64_t max_big = 0;
  for (uint64_t v : b_len) max_big = std::max(max_big, v);
  Stage& st = c->st_final;
  void* cur = src;
  void* cur_v = src_vals;
  void* oth = tmp;
  void* oth_v = tmp_vals;
  bool first_round = sel != nullptr;
  int rounds = 0;
  while (!b_off.empty()) {
    // Every round splits each non-constant cell into >= 2 non-empty cells,
    // so the key ranges shrink; 64-bit keys cannot need more than 64.
    if (++rounds > 64) return set_error(AMS_EINTERNAL, "final partition did not converge");
    const int nb_seg = (int)b_off.size();
    const int nbs = (int)std::min<uint64_t>(AMS_MAX_BUCKETS / 2,
                                            std::max<uint64_t>(2, (max_big + kTargetCell - 1) / kTargetCell));
    std::vector<int32_t> idx(nb_seg);
    for (int i = 0; i < nb_seg; ++i) idx[i] = i;
    SegMeta m;
    uint64_t nchunks;
    AMS_CK(c->dcls.ensure(sizeof(DigitCls) * (size_t)nb_seg));
    AMS_CK(c->pieces.ensure(16 * (size_t)nb_seg));
    Stage& sf = c->st_split;  // free after the levels: reuse for the range table
    sf.reset();
    size_t ob;
    if (first_round) {
      // Bounds of the final segments that need a partition (segment order).
      ob = sf.put(*sel);
    } else {
      std::vector<uint64_t> lohi(2 * (size_t)nb_seg);
      for (int i = 0; i < nb_seg; ++i) { lohi[2 * i] = b_lo[i]; lohi[2 * i + 1] = b_hi[i]; }
      ob = sf.put(lohi);
    }
    AMS_CK(sf.upload(c->stream));
    const uint64_t* bounds;
    if (first_round) {
      AMS_CK(launch_gather_bounds(c->stream, c->bounds[c->bcur].as<uint64_t>(),
                                  sf.dev<int32_t>(ob), nb_seg, c->pieces.as<uint64_t>()));
      bounds = c->pieces.as<uint64_t>();
    } else {
      bounds = sf.dev<uint64_t>(ob);
    }
    {
      KTimer kt(c, AMS_KCAT_RANGES, 0.0);
      AMS_CK(launch_final_ranges(c->stream, bounds, nb_seg, nbs, c->dcls.as<DigitCls>()));
    }
    AMS_CK(upload_segments(st, c->stream, b_off.data(), b_len.data(), idx.data(), nb_seg, nullptr,
                           0, &m, &nchunks, nbs));
    uint64_t nel = 0;
    for (uint64_t v : b_len) nel += v;
    int rc = run_histogram(c, cur, AMS_KEY_U64, true, m, nchunks, nbs, c->dcls.as<DigitCls>(),
                           nullptr, nel, nullptr);
    if (rc) return rc;
    AMS_CK(c->cell_base.ensure(sizeof(uint64_t) * (size_t)nb_seg * nbs));
    {
      KTimer kt(c, AMS_KCAT_CELLBASE, 12.0 * nb_seg * nbs);
      AMS_CK(launch_digit_base(c->stream, c->seg_hist.as<uint32_t>(), nbs, m,
                               c->cell_base.as<uint64_t>()));
    }
    {
      KTimer kt(c, AMS_KCAT_FSCATTER, (vals ? 32.0 : 16.0) * nel);
      AMS_CK(launch_scatter(c->stream, cur, cur_v, AMS_KEY_U64, true, /*stable=*/vals, oth, oth_v,
                            m, nchunks, c->blobs.as<uint8_t>(), c->dcls.as<DigitCls>(), 0, 0, nbs,
                            c->chunk_tot.as<uint32_t>(), c->cell_base.as<uint64_t>(), nullptr));
    }
    c->launches += 5;
    AMS_CK(cudaMemsetAsync(c->ovf_count.p, 0, sizeof(unsigned int), c->stream));
    CellSource cs{};
    cs.mode = 0;
    cs.cell_base = c->cell_base.as<uint64_t>();
    cs.cell_cnt = c->seg_hist.as<uint32_t>();
    cs.dcls = c->dcls.as<DigitCls>();
    cs.cells_per_seg = (uint32_t)nbs;
    rc = sort_cells(c, oth, oth_v, out, out_vals, key_kind, cs, (uint64_t)nb_seg * nbs, nel);
    if (rc) return rc;
    // Cells that still exceed shared memory go round again (sort_cells synced).
    unsigned int novf = 0;
    AMS_CK(to_host(c->h_small, c->ovf_count.p, sizeof novf, c->stream));
    AMS_CK(cudaStreamSynchronize(c->stream));
    std::memcpy(&novf, c->h_small.p, sizeof novf);
    b_off.clear(); b_len.clear(); b_lo.clear(); b_hi.clear();
    max_big = 0;
    c->overflow_cells += novf;
    if (novf) {
      std::vector<OverflowRec> recs(novf);
      AMS_CK(to_host(c->h_big, c->ovf.p, sizeof(OverflowRec) * novf, c->stream));
      AMS_CK(cudaStreamSynchronize(c->stream));
      std::memcpy(recs.data(), c->h_big.p, sizeof(OverflowRec) * novf);
      std::sort(recs.begin(), recs.end(),
                [](const OverflowRec& a, const OverflowRec& b) { return a.off < b.off; });
      for (const OverflowRec& r : recs) {
        b_off.push_back(r.off);
        b_len.push_back(r.count);
        b_lo.push_back(r.lo);  // exact min/max of the cell
        b_hi.push_back(r.hi);
        max_big = std::max(max_big, r.count);
      }
    }
    first_round = false;
    std::swap(cur, oth);
    std::swap(cur_v, oth_v);
  }
  return AMS_OK;
}

// Final sort after a bucket-major keys-only last level: every non-empty
// bucket (g, b) of the last level is a segment at bk_off with bk_len keys.
// Buckets that fit in shared memory are sorted straight into `out`; the
// others are split into fixed-capacity digit cells in scratch
// (k_scatter_fixed: no histogram pass), whose sorts write `out`.  Buckets
// whose cells overflowed go through the exact partition rounds from `src`.
int final_sort_bm(ams_ctx* c, void* src, void* tmp, void* out, int key_kind,
                  const std::vector<uint64_t>& bk_off, const std::vector<uint64_t>& bk_len,
                  const std::vector<int32_t>& bk_g, const std::vector<int32_t>& bk_b,
                  const uint64_t* d_group_bounds) {
  constexpr uint64_t kCap = AMS_FX_CAP;
  // Cells average fixed_fill_pct of capacity: with keys uniform inside a
  // bucket a cell's count is ~ N(target, sqrt(target)), far below capacity.
  const uint64_t kTarget = kCap * (uint64_t)c->fixed_fill_pct / 100;
  constexpr uint64_t kMaxDigits = AMS_MAX_BUCKETS / 2;
  std::vector<uint64_t> s_off, s_len, f_off, f_len;
  std::vector<int32_t> f_gb;
  std::vector<uint32_t> cell0{0};
  uint64_t total = 0, small_n = 0, fixed_n = 0;
  int max_nb = 2;
  for (size_t i = 0; i < bk_off.size(); ++i) {
    const uint64_t len = bk_len[i];
    total += len;
    if (len == 0) continue;
    if (len <= kCap) {
      s_off.push_back(bk_off[i]);
      s_len.push_back(len);
      small_n += len;
      continue;
    }
    const uint64_t d = std::min<uint64_t>(kMaxDigits, std::max<uint64_t>(2, (len + kTarget - 1) / kTarget));
    f_off.push_back(bk_off[i]);
    f_len.push_back(len);
    f_gb.push_back(bk_g[i]);
    f_gb.push_back(bk_b[i]);
    f_gb.push_back((int32_t)d);
    cell0.push_back(cell0.back() + (uint32_t)d);
    max_nb = std::max(max_nb, (int)d);
    fixed_n += len;
  }
  const int nseg = (int)f_off.size();
  const uint64_t ncells = cell0.back();
  const uint64_t rec_cap = std::max<uint64_t>(total / (kCap / 2), ncells) + 64;
  AMS_CK(c->ovf.ensure(sizeof(OverflowRec) * rec_cap));
  AMS_CK(c->fb.ensure(sizeof(OverflowRec) * 2 * rec_cap));  // two fallback lists (deferred reads)
  AMS_CK(c->ovf_count.ensure(sizeof(unsigned int)));
  AMS_CK(c->fb_count.ensure(sizeof(unsigned int)));
  AMS_CK(c->h_small.ensure(4096));
  AMS_CK(cudaMemsetAsync(c->ovf_count.p, 0, sizeof(unsigned int), c->stream));
  if (!s_off.empty()) {
    Stage& ss = c->st_sample;  // free after the levels
    ss.reset();
    const size_t oo = ss.put(s_off), ol = ss.put(s_len);
    AMS_CK(ss.upload(c->stream));
    CellSource cs{};
    cs.mode = 1;
    cs.seg_off = ss.dev<uint64_t>(oo);
    cs.seg_len = ss.dev<uint64_t>(ol);
    int rc = sort_cells(c, src, nullptr, out, nullptr, key_kind, cs, s_off.size(), small_n, 0, rec_cap);
    if (rc) return rc;
  }
  // The fallback counts of both cell sorts are read with the overflow flags
  // below: one host synchronisation for the whole final sort.
  auto read_counts = [&](unsigned int nfb[2]) -> int {
    AMS_CK(to_host(c->h_small, c->fb_count.p, 2 * sizeof(unsigned int), c->stream));
    AMS_CK(cudaStreamSynchronize(c->stream));
    std::memcpy(nfb, c->h_small.p, 2 * sizeof(unsigned int));
    return AMS_OK;
  };
  if (nseg == 0) {
    if (s_off.empty()) return AMS_OK;
    unsigned int nfb[2];
    int rc = read_counts(nfb);
    return rc ? rc : finish_fallback(c, src, out, key_kind, 0, rec_cap, nfb[0]);
  }
  c->fixed_segments += (uint64_t)nseg;
  Stage& sx = c->st_fixed;
  sx.reset();
  const size_t o_gb = sx.put(f_gb), o_c0 = sx.put(cell0), o_off = sx.put(f_off);
  AMS_CK(sx.upload(c->stream));
  std::vector<int32_t> idx(nseg);
  for (int i = 0; i < nseg; ++i) idx[i] = i;
  SegMeta m;
  uint64_t nchunks;
  // (the fixed partition likes half-size chunks: 1.153 -> 1.131 ms at config 2)
  AMS_CK(upload_segments(c->st_final, c->stream, f_off.data(), f_len.data(), idx.data(), nseg, nullptr,
                         0, &m, &nchunks, 1, kChunk / 2));
  AMS_CK(c->dcls.ensure(sizeof(DigitCls) * (size_t)nseg));
  AMS_CK(c->fx_fill.ensure(4 * (size_t)ncells));
  AMS_CK(c->fx_ovf.ensure(4 * (size_t)nseg));
  AMS_CK(c->fx_base.ensure(8 * (size_t)ncells));
  AMS_CK(c->fx_cnt.ensure(4 * (size_t)ncells));
  AMS_CK(c->fx_seg.ensure(4 * (size_t)ncells));
  AMS_CK(c->fx_scratch.ensure(8 * kCap * (size_t)ncells));
  AMS_CK(cudaMemsetAsync(c->fx_fill.p, 0, 4 * (size_t)ncells, c->stream));
  AMS_CK(cudaMemsetAsync(c->fx_ovf.p, 0, 4 * (size_t)nseg, c->stream));
  {
    KTimer kt(c, AMS_KCAT_RANGES, 0.0);
    AMS_CK(launch_bucket_ranges(c->stream, c->blobs.as<uint8_t>(), d_group_bounds, sx.dev<int32_t>(o_gb),
                                nseg, c->dcls.as<DigitCls>()));
  }
  {
    KTimer kt(c, AMS_KCAT_FSCATTER, 16.0 * fixed_n);
    AMS_CK(launch_scatter_fixed(c->stream, src, AMS_KEY_U64, c->fx_scratch.p, m, nchunks, max_nb,
                                c->dcls.as<DigitCls>(), sx.dev<uint32_t>(o_c0), c->fx_fill.as<uint32_t>(),
                                c->fx_ovf.as<uint32_t>()));
  }
  {
    KTimer kt(c, AMS_KCAT_CELLBASE, 16.0 * ncells);
    AMS_CK(launch_fixed_cells(c->stream, c->fx_fill.as<uint32_t>(), sx.dev<uint32_t>(o_c0),
                              sx.dev<uint64_t>(o_off), c->fx_ovf.as<uint32_t>(), nseg,
                              c->fx_base.as<uint64_t>(), c->fx_cnt.as<uint32_t>(), c->fx_seg.as<uint32_t>()));
  }
  c->launches += 3;
  CellSource cs{};
  cs.mode = 3;
  cs.cell_base = c->fx_base.as<uint64_t>();
  cs.cell_cnt = c->fx_cnt.as<uint32_t>();
  cs.dcls = c->dcls.as<DigitCls>();
  cs.cell_seg = c->fx_seg.as<uint32_t>();
  cs.cell0 = sx.dev<uint32_t>(o_c0);
  int rc = sort_cells(c, c->fx_scratch.p, nullptr, out, nullptr, key_kind, cs, ncells, fixed_n, 1, rec_cap);
  if (rc) return rc;
  // Overflowed buckets: exact partition rounds from src.
  std::vector<uint32_t> flags(nseg);
  AMS_CK(to_host(c->h_big, c->fx_ovf.p, 4 * (size_t)nseg, c->stream));
  unsigned int nfb[2] = {0, 0};
  if ((rc = read_counts(nfb))) return rc;
  std::memcpy(flags.data(), c->h_big.p, 4 * (size_t)nseg);
  if (!s_off.empty() && (rc = finish_fallback(c, src, out, key_kind, 0, rec_cap, nfb[0]))) return rc;
  if ((rc = finish_fallback(c, c->fx_scratch.p, out, key_kind, 1, rec_cap, nfb[1]))) return rc;
  std::vector<uint64_t> o_off2, o_len2, o_lo, o_hi;
  std::vector<DigitCls> dc;
  for (int i = 0; i < nseg; ++i) {
    if (!flags[i]) continue;
    if (dc.empty()) {
      dc.resize(nseg);
      AMS_CK(to_host(c->h_big, c->dcls.p, sizeof(DigitCls) * (size_t)nseg, c->stream));
      AMS_CK(cudaStreamSynchronize(c->stream));
      std::memcpy(dc.data(), c->h_big.p, sizeof(DigitCls) * (size_t)nseg);
    }
    o_off2.push_back(f_off[i]);
    o_len2.push_back(f_len[i]);
    o_lo.push_back(dc[i].lo);
    o_hi.push_back(dc[i].hi);
  }
  c->fixed_overflow_segments += o_off2.size();
  if (!o_off2.empty())
    return partition_rounds(c, src, nullptr, tmp, nullptr, out, nullptr, key_kind, o_off2, o_len2, o_lo,
                            o_hi, nullptr);
  return AMS_OK;
}

// Final sort with explicit per-segment key bounds [lo, hi] (no last-level
// bounds needed): small segments straight into `out`, the rest through
// the exact partition rounds.
int final_sort_lohi(ams_ctx* c, void* src, void* src_vals, void* tmp, void* tmp_vals, void* out,
                    void* out_vals, int key_kind, int nseg, const uint64_t* h_seg_off,
                    const uint64_t* h_seg_len, const std::vector<uint64_t>& lo,
                    const std::vector<uint64_t>& hi) {
  std::vector<uint64_t> s_off, s_len, b_off, b_len, b_lo, b_hi;
  uint64_t total = 0, small_n = 0;
  for (int s = 0; s < nseg; ++s) {
    total += h_seg_len[s];
    if (h_seg_len[s] == 0) continue;
    if (h_seg_len[s] <= (uint64_t)AMS_SMEM_SORT_CAP) {
      s_off.push_back(h_seg_off[s]);
      s_len.push_back(h_seg_len[s]);
      small_n += h_seg_len[s];
    } else {
      b_off.push_back(h_seg_off[s]);
      b_len.push_back(h_seg_len[s]);
      b_lo.push_back(lo[s]);
      b_hi.push_back(hi[s]);
    }
  }
  const uint64_t rec_cap = total / (AMS_SMEM_SORT_CAP / 2) + 64;
  AMS_CK(c->ovf.ensure(sizeof(OverflowRec) * rec_cap));
  AMS_CK(c->fb.ensure(sizeof(OverflowRec) * rec_cap));
  AMS_CK(c->ovf_count.ensure(sizeof(unsigned int)));
  AMS_CK(c->fb_count.ensure(sizeof(unsigned int)));
  AMS_CK(c->h_small.ensure(4096));
  AMS_CK(cudaMemsetAsync(c->ovf_count.p, 0, sizeof(unsigned int), c->stream));
  if (!s_off.empty()) {
    Stage& ss = c->st_sample;
    ss.reset();
    const size_t oo = ss.put(s_off), ol = ss.put(s_len);
    AMS_CK(ss.upload(c->stream));
    CellSource cs{};
    cs.mode = 1;
    cs.seg_off = ss.dev<uint64_t>(oo);
    cs.seg_len = ss.dev<uint64_t>(ol);
    int rc = sort_cells(c, src, src_vals, out, out_vals, key_kind, cs, s_off.size(), small_n);
    if (rc) return rc;
  }
  if (!b_off.empty())
    return partition_rounds(c, src, src_vals, tmp, tmp_vals, out, out_vals, key_kind, b_off, b_len, b_lo,
                            b_hi, nullptr);
  return AMS_OK;
}

}  // namespace

}  // extern "C"

namespace ams {
int sort_segments_lohi(ams_ctx* c, void* src, void* src_vals, void* tmp, void* tmp_vals, void* out,
                       void* out_vals, int key_kind, int nseg, const uint64_t* h_seg_off,
                       const uint64_t* h_seg_len, const std::vector<uint64_t>& lo,
                       const std::vector<uint64_t>& hi) {
  return final_sort_lohi(c, src, src_vals, tmp, tmp_vals, out, out_vals, key_kind, nseg, h_seg_off,
                         h_seg_len, lo, hi);
}
}  // namespace ams

extern "C" {

int ams_final_sort(ams_ctx_t* c, void* src, void* src_vals, void* tmp, void* tmp_vals, void* out,
                   void* out_vals, int key_kind, int nseg, const uint64_t* h_seg_off,
                   const uint64_t* h_seg_len) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (nseg < 0 || (nseg > 0 && (!h_seg_off || !h_seg_len))) return set_error(AMS_EINVAL, "bad segments");
  const bool vals = src_vals != nullptr;
  if (vals && (!tmp_vals || !out_vals)) return set_error(AMS_EINVAL, "missing value buffers");
  AMS_ON_DEVICE(c->device);
  std::vector<uint64_t> s_off, s_len, b_off, b_len, b_lo, b_hi;
  std::vector<int32_t> b_seg;
  uint64_t total = 0, small_n = 0;
  for (int s = 0; s < nseg; ++s) {
    total += h_seg_len[s];
    if (h_seg_len[s] == 0) continue;
    if (h_seg_len[s] <= (uint64_t)AMS_SMEM_SORT_CAP) {
      s_off.push_back(h_seg_off[s]);
      s_len.push_back(h_seg_len[s]);
      small_n += h_seg_len[s];
    } else {
      b_off.push_back(h_seg_off[s]);
      b_len.push_back(h_seg_len[s]);
      b_seg.push_back(s);
    }
  }
  if (!b_off.empty() && c->bounds[c->bcur].cap < 16 * (size_t)nseg)
    return set_error(AMS_EINVAL, "final segments need the key bounds of the last level");
  const uint64_t rec_cap = total / (AMS_SMEM_SORT_CAP / 2) + 64;
  AMS_CK(c->ovf.ensure(sizeof(OverflowRec) * rec_cap));
  AMS_CK(c->fb.ensure(sizeof(OverflowRec) * rec_cap));
  AMS_CK(c->ovf_count.ensure(sizeof(unsigned int)));
  AMS_CK(c->fb_count.ensure(sizeof(unsigned int)));
  AMS_CK(c->h_small.ensure(4096));
  AMS_CK(cudaMemsetAsync(c->ovf_count.p, 0, sizeof(unsigned int), c->stream));
  // 1. Segments that fit in shared memory: sort straight into `out`.
  if (!s_off.empty()) {
    Stage& ss = c->st_sample;  // free after the levels
    ss.reset();
    const size_t oo = ss.put(s_off), ol = ss.put(s_len);
    AMS_CK(ss.upload(c->stream));
    CellSource cs{};
    cs.mode = 1;
    cs.seg_off = ss.dev<uint64_t>(oo);
    cs.seg_len = ss.dev<uint64_t>(ol);
    int rc = sort_cells(c, src, src_vals, out, out_vals, key_kind, cs, s_off.size(), small_n);
    if (rc) return rc;
  }
  // 2. Large segments: digit partition src -> tmp, then per-cell sorts;
  //    cells still above shared memory go round again (tmp -> src -> ...).
  if (!b_off.empty()) {
    int rc = partition_rounds(c, src, src_vals, tmp, tmp_vals, out, out_vals, key_kind, b_off, b_len,
                              b_lo, b_hi, &b_seg);
    if (rc) return rc;
  }
  return AMS_OK;
}

int ams_level_scatter_ex(ams_ctx_t* c, const void* src, const void* src_vals, int key_kind,
                         void* dst, void* dst_vals, int r, const uint64_t* h_boundaries,
                         const uint64_t* h_group_dst_start, int child_first, int child_count,
                         int flags) {
  return level_scatter_impl(c, src, src_vals, key_kind, dst, dst_vals, r, h_boundaries,
                            h_group_dst_start, child_first, child_count,
                            (flags & AMS_SCATTER_BUCKET_MAJOR) != 0);
}

int ams_final_sort_buckets(ams_ctx_t* c, void* src, void* tmp, void* out, int key_kind, int nbk,
                           const uint64_t* bk_off, const uint64_t* bk_len, const int32_t* bk_group,
                           const int32_t* bk_bucket) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  if (nbk < 0 || (nbk > 0 && (!bk_off || !bk_len || !bk_group || !bk_bucket)))
    return set_error(AMS_EINVAL, "bad bucket list");
  if (nbk > 0 && c->bounds[1 - c->bcur].cap == 0)
    return set_error(AMS_EINVAL, "no key bounds of the last level's groups");
  AMS_ON_DEVICE(c->device);
  std::vector<uint64_t> bo(bk_off, bk_off + nbk), bl(bk_len, bk_len + nbk);
  std::vector<int32_t> bg(bk_group, bk_group + nbk), bb(bk_bucket, bk_bucket + nbk);
  return final_sort_bm(c, src, tmp, out, key_kind, bo, bl, bg, bb, c->bounds[1 - c->bcur].as<uint64_t>());
}

int ams_final_sort_fixed_stats(ams_ctx_t* c, uint64_t out[2]) {
  if (!c || !out) return set_error(AMS_EINVAL, "null argument");
  out[0] = c->fixed_segments;
  out[1] = c->fixed_overflow_segments;
  return AMS_OK;
}

int ams_final_sort_stats(ams_ctx_t* c, uint64_t out[2]) {
  if (!c || !out) return set_error(AMS_EINVAL, "null argument");
  out[0] = c->overflow_cells;
  out[1] = c->fallback_cells;
  return AMS_OK;
}

int ams_map_keys(ams_ctx_t* c, const void* src, void* dst, uint64_t n, int from_kind, int to_kind) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  AMS_ON_DEVICE(c->device);
  KTimer kt(c, AMS_KCAT_MAP, 16.0 * n);
  AMS_CK(launch_map_keys(c->stream, src, dst, n, from_kind, to_kind));
  c->launches += n ? 1 : 0;
  return AMS_OK;
}


// ---------------------------------------------------------------------------
// One-call driver: ams_sort (ams.py:271-313) with scheme "simple" on one GPU,
// the level loop of paper_1410_6754_b200/engine.py in C++ (no Python between
// the level steps).
namespace {
// Host-side step timer of ams_sort_run (AMS_HOST_TRACE=1).
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  std::string line;
  explicit HostTrace(bool on_) : on(on_) { t0 = last = std::chrono::steady_clock::now(); }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s=%.0f", what,
                  std::chrono::duration<double, std::micro>(now - last).count());
    line += buf;
    last = now;
  }
  ~HostTrace() {
    if (!on) return;
    std::fprintf(stderr, "ams_sort_run host us:%s total=%.0f\n", line.c_str(),
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
};
}  // namespace

// Per PE, how many of its level's splitters were drawn from it (host
// bookkeeping for the ledger; one D2H of the sample tags and of every
// group's splitter tags).
static int splitter_holders(ams_ctx_t* c, int G, uint64_t S, const uint64_t* soff,
                            const uint64_t* idx, const uint64_t* offs, int p,
                            std::vector<uint32_t>* out) {
  std::vector<uint32_t> spos(S);
  AMS_CK(cudaMemcpyAsync(spos.data(), c->s_pos.p, 4 * S, cudaMemcpyDeviceToHost, c->stream));
  AMS_CK(cudaStreamSynchronize(c->stream));
  out->assign(p, 0);
  std::vector<uint32_t> pos(AMS_MAX_BUCKETS);
  for (int g = 0; g < G; ++g) {
    int nspl = 0;
    int rc = ams_read_splitters(c, g, nullptr, pos.data(), &nspl);
    if (rc) return rc;
    std::unordered_map<uint32_t, int> pe_of;
    pe_of.reserve(2 * (soff[g + 1] - soff[g]));
    for (uint64_t i = soff[g]; i < soff[g + 1]; ++i)
      pe_of[spos[i]] = (int)(std::upper_bound(offs, offs + p + 1, idx[i]) - offs) - 1;
    for (int j = 0; j < nspl; ++j) {
      auto it = pe_of.find(pos[j]);
      if (it == pe_of.end()) return set_error(AMS_EINTERNAL, "splitter not found in the sample");
      (*out)[it->second] += 1;
    }
  }
  return AMS_OK;
}

int ams_sort_run(ams_ctx_t* c, const ams_params_t* prm, int p, const uint64_t* pe_sizes,
                 const void* keys, const void* vals, void* out, void* out_vals,
                 uint64_t* out_pe_sizes, ams_level_report_t* reports) {
  if (!c || !prm) return set_error(AMS_EINVAL, "null argument");
  const int k = prm->levels;
  if (k < 1 || k > AMS_MAX_LEVELS) return set_error(AMS_EINVAL, "levels outside 1..AMS_MAX_LEVELS");
  // Continuation (multi-GPU: the levels below level_base ran as the
  // exchange between the GPUs): this call's PEs start as g0 equal groups.
  const int lv0 = prm->level_base;
  const int g0 = prm->init_groups > 0 ? prm->init_groups : 1;
  const int pe_base = prm->pe_base;
  if (lv0 < 0 || lv0 > k || pe_base < 0) return set_error(AMS_EINVAL, "bad continuation parameters");
  if (lv0 == 0 && (g0 != 1 || pe_base != 0))
    return set_error(AMS_EINVAL, "init_groups / pe_base need level_base > 0");
  if (lv0 > 0 && !(prm->oversampling > 0))
    return set_error(AMS_EINVAL, "a continuation needs the sort's oversampling factor");
  uint64_t prod = (uint64_t)g0;
  for (int lv = 0; lv < k; ++lv) {  // AmsParams validation (ams.py:45-52, 61-65)
    if (prm->group_counts[lv] < 1) return set_error(AMS_EINVAL, "group counts must be positive");
    if (lv >= lv0) prod *= (uint64_t)prm->group_counts[lv];
  }
  if (prm->overpartition < 1) return set_error(AMS_EINVAL, "overpartitioning factor must be at least 1");
  if (!(prm->imbalance > 0)) return set_error(AMS_EINVAL, "imbalance budget must be positive");
  if (p < 1 || prod != (uint64_t)p)
    return set_error(AMS_EINVAL, "group counts do not telescope " + std::to_string(p) + " PEs");
  if (!pe_sizes || !prm->stream_id) return set_error(AMS_EINVAL, "null argument");
  if (prm->key_kind < AMS_KEY_U64 || prm->key_kind > AMS_KEY_F64)
    return set_error(AMS_EINVAL, "unknown key kind");
  uint64_t n = 0;
  for (int i = 0; i < p; ++i) n += pe_sizes[i];
  if (n && (!keys || !out)) return set_error(AMS_EINVAL, "null key buffer");
  if (prm->scheme < AMS_SCHEME_SIMPLE || prm->scheme > AMS_SCHEME_RANDOMIZED)
    return set_error(AMS_EINVAL, "unknown delivery scheme");
  if (prm->sample_mode != AMS_SAMPLE_PARITY && prm->sample_mode != AMS_SAMPLE_DEVICE)
    return set_error(AMS_EINVAL, "unknown sample mode");
  if (prm->sample_mode == AMS_SAMPLE_DEVICE && prm->record_holders)
    return set_error(AMS_EINVAL, "splitter holders need the parity sample mode");
  // A continuation under a non-simple scheme takes the input's origin tags
  // as `vals` (not user payloads).
  const bool tags_in = lv0 > 0 && prm->scheme != AMS_SCHEME_SIMPLE && n > 0;
  if (tags_in && !vals) return set_error(AMS_EINVAL, "the continuation needs the origin tags as vals");
  const bool user_vals = vals != nullptr && !tags_in;
  if (user_vals && !out_vals) return set_error(AMS_EINVAL, "values need an output buffer");
  // Deterministic delivery (delivery.py:188-306) can put a later source's
  // piece into an earlier member, so group-buffer order stops being origin
  // order: origin tags travel as the values and break key ties
  // from level 2 on (and order the final sort); user values are gathered by
  // tag at the end.
  // (The permuted scheme's receivers also concatenate by source id while
  // the enumeration follows the permutation: same treatment.)
  const bool det = prm->scheme != AMS_SCHEME_SIMPLE && n > 0;
  const bool with_vals = user_vals || det;
  AMS_ON_DEVICE(c->device);
  // ams.py:278-280 and AmsParams.per_level_imbalance (ams.py:58-59).
  const double a = prm->oversampling > 0 ? prm->oversampling
                                         : 1.6 * std::log10((double)std::max<uint64_t>(n, 10));
  const double eps_l = std::pow(1.0 + prm->imbalance, 1.0 / k) - 1.0;
  const int b = prm->overpartition;
  // Workspace (two ping-pong buffers) and one-element stand-ins for n == 0.
  // +2 keys: the fixed-capacity partition (k_scatter_fixed) copies whole
  // 16-byte units past a segment end.
  const size_t wb = 8 * ((size_t)std::max<uint64_t>(n, 1) + 2);
  for (int i = 0; i < 2; ++i) {
    AMS_CK(c->work[i].ensure(wb));
    if (with_vals) AMS_CK(c->work_v[i].ensure(wb));
  }
  if (det) {
    AMS_CK(c->tags0.ensure(wb));  // origin tags, later relayout scratch
    if (!tags_in) {
      AMS_CK(launch_iota(c->stream, c->tags0.p, n));
      c->launches += 1;
    }
  }
  const void* src = n ? keys : c->work[1].p;
  const void* src_v = tags_in ? vals : det ? c->tags0.p : (with_vals ? (n ? vals : c->work_v[1].p) : nullptr);
  void* dst_out = n ? out : c->work[1].p;
  void* dst_out_v = with_vals ? (n && !det ? out_vals : c->work_v[1].p) : nullptr;
  // A continuation's input went through a level scatter: order-mapped u64.
  int src_kind = lv0 > 0 ? AMS_KEY_U64 : prm->key_kind;
  std::vector<uint64_t> sizes(pe_sizes, pe_sizes + p);
  std::vector<int32_t> gf, gn;
  for (int g = 0; g < g0; ++g) { gf.push_back(g * (p / g0)); gn.push_back(p / g0); }
  c->run_levels.assign(k, ams_ctx::LevelRec{});
  HostTrace tr(c->host_trace);
  tr.mark("setup");
  int rc;
  bool used_bm = false;
  for (int lv = lv0; lv < k; ++lv) {
    const int r = prm->group_counts[lv];
    const int G = (int)gf.size();
    std::vector<uint64_t> offs(p + 1, 0);
    for (int i = 0; i < p; ++i) offs[i + 1] = offs[i] + sizes[i];
    // ams.py:224-225 per group.
    std::vector<uint64_t> targets(G), br(G);
    for (int g = 0; g < G; ++g) {
      uint64_t n_g = 0;
      for (int i = 0; i < gn[g]; ++i) n_g += sizes[gf[g] + i];
      br[g] = std::min<uint64_t>((uint64_t)b * r, n_g + 1);
      const uint64_t x = br[g];
      targets[g] = std::min<uint64_t>(n_g, std::max<uint64_t>(x - 1, (uint64_t)std::ceil(a * (double)x)));
    }
    const bool dev_sample = prm->sample_mode == AMS_SAMPLE_DEVICE;
    uint64_t cap = 0;
    for (uint64_t t : targets) cap += t;
    std::vector<uint64_t> idx(std::max<uint64_t>(cap, 1)), gpos(std::max<uint64_t>(cap, 1)), drawn(G);
    // Fast mode: only the quota split on the host (ams.py:166-171); the
    // positions are drawn by the gather kernel.
    std::vector<uint64_t> smp_off, mem_gpos;
    if (dev_sample) {
      smp_off.assign((size_t)p + 1, 0);
      mem_gpos.assign(p, 0);
      uint64_t w = 0;
      for (int g = 0; g < G; ++g) {
        const int first = gf[g], P = gn[g];
        const uint64_t base = targets[g] / P, extra = targets[g] % P;
        uint64_t gp = 0, dr = 0;
        for (int i = 0; i < P; ++i) {
          const uint64_t take = std::min<uint64_t>(base + ((uint64_t)i < extra ? 1 : 0), sizes[first + i]);
          smp_off[first + i] = w;
          mem_gpos[first + i] = gp;
          w += take;
          dr += take;
          gp += sizes[first + i];
        }
        drawn[g] = dr;
      }
      smp_off[p] = w;
      rc = AMS_OK;
    } else {
      if (pe_base == 0) {
        rc = ams_draw_sample_positions(prm->master_seed, prm->stream_id, lv, G, gf.data(), gn.data(),
                                       targets.data(), sizes.data(), offs.data(), cap, idx.data(),
                                       gpos.data(), drawn.data());
      } else {
        // The streams are named by global PE ids (ams.py:168-174): shifted tables.
        std::vector<uint64_t> gsz((size_t)pe_base + p, 0), gof((size_t)pe_base + p, 0);
        std::copy(sizes.begin(), sizes.end(), gsz.begin() + pe_base);
        std::copy(offs.begin(), offs.begin() + p, gof.begin() + pe_base);
        std::vector<int32_t> gfn(gf);
        for (int32_t& f : gfn) f += pe_base;
        rc = ams_draw_sample_positions(prm->master_seed, prm->stream_id, lv, G, gfn.data(), gn.data(),
                                       targets.data(), gsz.data(), gof.data(), cap, idx.data(),
                                       gpos.data(), drawn.data());
      }
      if (rc) return rc;
    }
    if (rc) return rc;
    tr.mark("draw");
    std::vector<int32_t> nb(G);
    std::vector<uint64_t> soff(G + 1, 0);
    int nb_stride = 1;
    for (int g = 0; g < G; ++g) {
      nb[g] = (int)std::min<uint64_t>(br[g], drawn[g] + 1);  // ams.py:228
      if (nb[g] > AMS_MAX_BUCKETS)
        return set_error(AMS_EINVAL, std::to_string(nb[g]) + " buckets exceed the supported " +
                                         std::to_string(AMS_MAX_BUCKETS));
      nb_stride = std::max(nb_stride, nb[g]);
      soff[g + 1] = soff[g] + drawn[g];
    }
    const uint64_t S = soff[G];
    AMS_CK(c->s_keys.ensure(8 * (size_t)std::max<uint64_t>(S, 1)));
    AMS_CK(c->s_pos.ensure(4 * (size_t)std::max<uint64_t>(S, 1)));
    const uint64_t* tie_tags = det && lv > 0 ? static_cast<const uint64_t*>(src_v) : nullptr;
    // (lv counts from the whole sort's first level: a continuation's input
    // already went through a non-simple delivery.)
    if (dev_sample) {
      if (S) {
        Stage& st = c->st_sample;
        st.reset();
        const size_t o_so = st.put(smp_off), o_mo = st.put(offs.data(), (size_t)p), o_ml = st.put(sizes),
                     o_mg = st.put(mem_gpos);
        AMS_CK(st.upload(c->stream));
        // one stream per (seed, stream id, level): blake2b of its name
        const std::string name = std::to_string(prm->master_seed) + "\x1f" + prm->stream_id + "/L" +
                                 std::to_string(lv) + "/device-sample";
        uint8_t dg[16];
        blake2b_128(reinterpret_cast<const uint8_t*>(name.data()), name.size(), dg);
        uint64_t seed64;
        std::memcpy(&seed64, dg, 8);
        KTimer kt(c, AMS_KCAT_SAMPLE, 12.0 * S);
        AMS_CK(launch_draw_gather(c->stream, src, src_kind, st.dev<uint64_t>(o_so), st.dev<uint64_t>(o_mo),
                                  st.dev<uint64_t>(o_ml), st.dev<uint64_t>(o_mg), p, S, seed64,
                                  c->s_keys.as<uint64_t>(), c->s_pos.as<uint32_t>(), tie_tags));
        c->launches += 1;
      }
    } else if ((rc = level_sample_impl(c, src, src_kind, S, idx.data(), gpos.data(),
                                       c->s_keys.as<uint64_t>(), c->s_pos.as<uint32_t>(), tie_tags))) {
      return rc;
    }
    if ((rc = ams_level_splitters(c, G, c->s_keys.as<uint64_t>(), c->s_pos.as<uint32_t>(),
                                  soff.data(), nb.data())))
      return rc;
    std::vector<uint32_t> holders;
    if (prm->record_holders && S) {
      // Member each splitter was drawn from (the holder that contributes it
      // to extract_by_ranks, fastsort.py:111-130): splitters carry the
      // sample element's unique position (or origin tag) value.
      if ((rc = splitter_holders(c, G, S, soff.data(), idx.data(), offs.data(), p, &holders)))
        return rc;
    }
    std::vector<int32_t> seg_group(p);
    std::vector<int64_t> posbase(G);
    for (int g = 0; g < G; ++g) {
      for (int i = 0; i < gn[g]; ++i) seg_group[gf[g] + i] = g;
      posbase[g] = -(int64_t)offs[gf[g]];
    }
    const bool last = lv == k - 1;
    ams_ctx::LevelRec& rec = c->run_levels[lv];
    rec.r = r; rec.G = G; rec.P = p; rec.nb_stride = nb_stride;
    rec.group_first = gf; rec.group_npe = gn; rec.nb = nb;
    rec.sizes_before = sizes; rec.drawn = drawn;
    rec.holders = std::move(holders);
    // Fully overwritten by the classify step; a buffer recycled from the
    // oldest kept run avoids 4 MB of page faults and zeroing per level at
    // 256 PEs x 4096 buckets.
    if (!c->hist_pool.empty()) {
      rec.hist = std::move(c->hist_pool.back());
      c->hist_pool.pop_back();
    }
    rec.hist.resize((size_t)p * nb_stride);
    c->level_tags = tie_tags;
    tr.mark("sample");
    rc = ams_level_classify(c, src, src_kind, p, offs.data(), sizes.data(), seg_group.data(), G,
                            posbase.data(), nb_stride, lv == 0, !(last && !with_vals), rec.hist.data());
    c->level_tags = nullptr;
    if (rc) return rc;
    tr.mark("classify+sync");
    rec.boundaries.assign((size_t)G * (r + 1), 0);
    rec.loads.assign((size_t)G * r, 0);
    rec.max_load.assign(G, 0);
    rec.new_sizes.assign(p, 0);
    rec.has_stats = prm->with_stats != 0;
    rec.stats.assign(rec.has_stats ? (size_t)G * 4 : 0, 0);
    if ((rc = ams_plan_level(G, gn.data(), nb.data(), r, rec.hist.data(), nb_stride,
                             rec.boundaries.data(), rec.loads.data(), rec.max_load.data(),
                             rec.new_sizes.data(), rec.has_stats ? rec.stats.data() : nullptr)))
      return rc;
    std::vector<uint64_t> dst_start(G);
    for (int g = 0; g < G; ++g) dst_start[g] = offs[gf[g]];
    void* dst = c->work[lv % 2].p;
    void* dst_v = with_vals ? c->work_v[lv % 2].p : nullptr;
    const bool bm = last && !with_vals && c->bm_final;
    // Deterministic delivery where subgroups have several members: member
    // assignment per group (host), the simple layout into scratch, then the
    // slices copied to the members' arrays in receive order.
    const bool relayout = det && gn[0] / r > 1;
    // Randomized delivery chunks large pieces into several messages even
    // with one member per subgroup: its planner also supplies those stats.
    const bool plan_slices = relayout || (prm->scheme == AMS_SCHEME_RANDOMIZED && rec.has_stats && n > 0);
    std::vector<uint64_t> items;
    if (plan_slices) {
      std::vector<uint64_t> pieces, slices;
      for (int g = 0; g < G; ++g) {
        const int P = gn[g];
        pieces.assign((size_t)P * r, 0);
        for (int j = 0; j < P; ++j)
          for (int t = 0; t < r; ++t)
            for (uint64_t bb = rec.boundaries[(size_t)g * (r + 1) + t];
                 bb < rec.boundaries[(size_t)g * (r + 1) + t + 1]; ++bb)
              pieces[(size_t)j * r + t] += rec.hist[(size_t)(gf[g] + j) * nb_stride + bb];
        const int cap = P * (2 * r + 2) + 16;
        slices.assign(3 * (size_t)cap, 0);
        int ns = 0;
        uint64_t* st4 = rec.has_stats ? rec.stats.data() + 4 * (size_t)g : nullptr;
        const std::string ls = std::string(prm->stream_id) + "/L" + std::to_string(lv) + "-g" +
                               std::to_string(gf[g] + pe_base);
        if (prm->scheme == AMS_SCHEME_PERMUTED)
          rc = ams_deliver_permuted(P, r, prm->master_seed, ls.c_str(), pieces.data(),
                                    rec.new_sizes.data() + gf[g], slices.data(), cap, &ns, st4);
        else if (prm->scheme == AMS_SCHEME_RANDOMIZED)
          rc = ams_deliver_randomized(P, r, prm->master_seed, ls.c_str(), pieces.data(),
                                      rec.new_sizes.data() + gf[g], slices.data(), cap, &ns, st4);
        else
          rc = ams_deliver_deterministic(P, r, gf[g] + pe_base, pieces.data(), rec.new_sizes.data() + gf[g],
                                         slices.data(), cap, &ns, st4);
        if (rc) return rc;
        for (int q = 0; relayout && q < ns; ++q) {
          const uint64_t s0 = dst_start[g] + slices[3 * q], d0 = dst_start[g] + slices[3 * q + 1];
          for (uint64_t o = 0; o < slices[3 * q + 2]; o += kCopyItemKeys) {
            items.push_back(s0 + o);
            items.push_back(d0 + o);
            items.push_back(std::min<uint64_t>(kCopyItemKeys, slices[3 * q + 2] - o));
          }
        }
      }
    }
    void* sdst = dst;
    void* sdst_v = dst_v;
    if (relayout) {  // scratch for the simple layout: the free work buffer / the output
      sdst = lv == 0 ? c->work[1].p : dst_out;
      sdst_v = lv == 0 ? c->work_v[1].p : c->tags0.p;  // tags0: free once level 1 is done
    }
    tr.mark("plan");
    if ((rc = level_scatter_impl(c, src, src_v, src_kind, sdst, sdst_v, r, rec.boundaries.data(),
                                 dst_start.data(), 0, G * r, bm)))
      return rc;
    tr.mark("scatter");
    if (relayout) {
      Stage& sc = c->st_copy;
      sc.reset();
      const size_t oi = sc.put(items);
      AMS_CK(sc.upload(c->stream));
      KTimer kt(c, AMS_KCAT_SCATTER, 32.0 * (double)n);
      AMS_CK(launch_copy_ranges(c->stream, sc.dev<uint64_t>(oi), (int)(items.size() / 3), sdst, dst,
                                sdst_v, dst_v, n));
      c->launches += 1;
    }
    used_bm = bm;
    // Level report (ams.py:258-268, 294-308).
    if (reports) {
      ams_level_report_t& rp = reports[lv];
      std::memset(&rp, 0, sizeof rp);
      rp.level = lv + 1;
      rp.r = r;
      rp.max_load = *std::max_element(rec.new_sizes.begin(), rec.new_sizes.end());
      rp.min_load = *std::min_element(rec.new_sizes.begin(), rec.new_sizes.end());
      rp.sample_size = *std::max_element(drawn.begin(), drawn.end());
      rp.plan_load = *std::max_element(rec.max_load.begin(), rec.max_load.end());
      for (int g = 0; g < G; ++g) {
        uint64_t n_g = 0;
        for (int i = 0; i < gn[g]; ++i) n_g += sizes[gf[g] + i];
        const uint64_t budget = (uint64_t)std::ceil((1.0 + eps_l) * (double)n_g / r);
        rp.over_budget += rec.max_load[g] > budget;
        if (rec.has_stats) {
          rp.max_words = std::max(rp.max_words, rec.stats[4 * g + 0]);
          rp.max_msgs = std::max(rp.max_msgs, rec.stats[4 * g + 1]);
          rp.max_sent_msgs = std::max(rp.max_sent_msgs, rec.stats[4 * g + 2]);
          rp.max_recv_msgs = std::max(rp.max_recv_msgs, rec.stats[4 * g + 3]);
        }
      }
    }
    src = dst;
    src_v = dst_v;
    src_kind = AMS_KEY_U64;
    sizes = rec.new_sizes;
    std::vector<int32_t> nf, nn;
    for (int g = 0; g < G; ++g) {
      const int step = gn[g] / r;
      for (int t = 0; t < r; ++t) { nf.push_back(gf[g] + t * step); nn.push_back(step); }
    }
    gf.swap(nf);
    gn.swap(nn);
  }
  // Final local sort (ams.py:310-312).
  std::vector<uint64_t> offs(p + 1, 0);
  for (int i = 0; i < p; ++i) offs[i + 1] = offs[i] + sizes[i];
  void* tmp = c->work[k % 2].p;
  void* tmp_v = with_vals ? c->work_v[k % 2].p : nullptr;
  tr.mark("levels-end");
  if (used_bm) {
    // Buckets of the bucket-major last level, in output order.
    const ams_ctx::LevelRec& L = c->run_levels[k - 1];
    std::vector<uint64_t> bo, bl;
    std::vector<int32_t> bg, bb;
    uint64_t at = 0;
    std::vector<uint64_t> tot;
    for (int g = 0; g < L.G; ++g) {
      // Bucket totals of the group: member rows outermost (each row is
      // contiguous; 256 PEs x 4096 buckets is 4 MB of histogram).
      tot.assign((size_t)L.nb[g], 0);
      for (int j = 0; j < L.group_npe[g]; ++j) {
        const uint32_t* row = L.hist.data() + (size_t)(L.group_first[g] + j) * L.nb_stride;
        for (int b = 0; b < L.nb[g]; ++b) tot[b] += row[b];
      }
      for (int b = 0; b < L.nb[g]; ++b) {
        bo.push_back(at);
        bl.push_back(tot[b]);
        bg.push_back(g);
        bb.push_back(b);
        at += tot[b];
      }
    }
    if ((rc = final_sort_bm(c, const_cast<void*>(src), tmp, dst_out, prm->key_kind, bo, bl, bg, bb,
                            c->bounds[1 - c->bcur].as<uint64_t>())))
      return rc;
  } else if (det && !user_vals) {
    // Keys only: equal keys are indistinguishable, so a key sort suffices.
    if ((rc = ams_final_sort(c, const_cast<void*>(src), nullptr, tmp, nullptr, dst_out, nullptr,
                             prm->key_kind, p, offs.data(), sizes.data())))
      return rc;
  } else if (det) {
    // Final order (key, origin): each PE by tag, then stably by key; the
    // user's values are gathered by the sorted tags.
    void* K = const_cast<void*>(src);
    void* T = const_cast<void*>(src_v);
    void* W = c->work[k % 2].p;
    void* X = c->tags0.p;
    std::vector<uint64_t> lo(p, 0), hi(p, n - 1);
    if ((rc = final_sort_lohi(c, T, K, out, out_vals, X, W, AMS_KEY_U64, p, offs.data(), sizes.data(),
                              lo, hi)))
      return rc;
    if ((rc = ams_final_sort(c, W, X, K, T, dst_out, c->work_v[k % 2].p, prm->key_kind, p, offs.data(),
                             sizes.data())))
      return rc;
    AMS_CK(launch_gather_vals(c->stream, vals, c->work_v[k % 2].p, out_vals, n));
    c->launches += 1;
  } else if ((rc = ams_final_sort(c, const_cast<void*>(src), const_cast<void*>(src_v), tmp, tmp_v, dst_out,
                                  dst_out_v, prm->key_kind, p, offs.data(), sizes.data()))) {
    return rc;
  }
  tr.mark("final");
  c->run_id += 1;
  c->run_history.emplace_back(c->run_id, std::move(c->run_levels));
  c->run_levels.clear();
  if (c->run_history.size() > ams_ctx::kRunHistory) {
    for (auto& lr : c->run_history.front().second)
      if (c->hist_pool.size() < 2 * AMS_MAX_LEVELS) c->hist_pool.push_back(std::move(lr.hist));
    c->run_history.erase(c->run_history.begin());
  }
  c->run_final_sizes = sizes;
  if (out_pe_sizes) std::memcpy(out_pe_sizes, sizes.data(), sizeof(uint64_t) * p);
  return AMS_OK;
}

uint64_t ams_run_id(const ams_ctx_t* c) { return c ? c->run_id : 0; }

}  // extern "C"

namespace {
// Records of run `id` (0 = the last run); null when no longer kept.
const std::vector<ams_ctx::LevelRec>* run_records(const ams_ctx* c, uint64_t id) {
  if (id == 0) return c->run_history.empty() ? nullptr : &c->run_history.back().second;
  for (const auto& h : c->run_history)
    if (h.first == id) return &h.second;
  return nullptr;
}
}  // namespace

extern "C" {

int ams_run_level_dims(ams_ctx_t* c, int level, int* r, int* ngroups, int* npe, int* nb_stride,
                       int* has_stats) {
  return ams_run_level_dims_at(c, 0, level, r, ngroups, npe, nb_stride, has_stats);
}

int ams_run_level(ams_ctx_t* c, int level, int32_t* group_first, int32_t* group_npe,
                  uint64_t* sizes_before, uint64_t* drawn, int32_t* nb, uint32_t* seg_hist,
                  uint64_t* boundaries, uint64_t* loads, uint64_t* max_load, uint64_t* new_sizes,
                  uint64_t* stats) {
  return ams_run_level_at(c, 0, level, group_first, group_npe, sizes_before, drawn, nb, seg_hist,
                          boundaries, loads, max_load, new_sizes, stats);
}

int ams_run_level_dims_at(ams_ctx_t* c, uint64_t run, int level, int* r, int* ngroups, int* npe,
                          int* nb_stride, int* has_stats) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  const std::vector<ams_ctx::LevelRec>* rl = run_records(c, run);
  if (!rl) return set_error(AMS_EINVAL, "records of that run are no longer kept");
  if (level < 0 || level >= (int)rl->size()) return set_error(AMS_EINVAL, "no such level");
  const ams_ctx::LevelRec& L = (*rl)[level];
  if (r) *r = L.r;
  if (ngroups) *ngroups = L.G;
  if (npe) *npe = L.P;
  if (nb_stride) *nb_stride = L.nb_stride;
  if (has_stats) *has_stats = L.has_stats;
  return AMS_OK;
}

int ams_run_level_at(ams_ctx_t* c, uint64_t run, int level, int32_t* group_first, int32_t* group_npe,
                     uint64_t* sizes_before, uint64_t* drawn, int32_t* nb, uint32_t* seg_hist,
                     uint64_t* boundaries, uint64_t* loads, uint64_t* max_load, uint64_t* new_sizes,
                     uint64_t* stats) {
  if (!c) return set_error(AMS_EINVAL, "null context");
  const std::vector<ams_ctx::LevelRec>* rl = run_records(c, run);
  if (!rl) return set_error(AMS_EINVAL, "records of that run are no longer kept");
  if (level < 0 || level >= (int)rl->size()) return set_error(AMS_EINVAL, "no such level");
  const ams_ctx::LevelRec& L = (*rl)[level];
  auto cp = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(v[0]) * v.size());
  };
  cp(group_first, L.group_first); cp(group_npe, L.group_npe); cp(sizes_before, L.sizes_before);
  cp(drawn, L.drawn); cp(nb, L.nb); cp(seg_hist, L.hist); cp(boundaries, L.boundaries);
  cp(loads, L.loads); cp(max_load, L.max_load); cp(new_sizes, L.new_sizes); cp(stats, L.stats);
  return AMS_OK;
}

int ams_run_level_holders_at(ams_ctx_t* c, uint64_t run, int level, uint32_t* holders) {
  if (!c || !holders) return set_error(AMS_EINVAL, "null argument");
  const std::vector<ams_ctx::LevelRec>* rl = run_records(c, run);
  if (!rl) return set_error(AMS_EINVAL, "records of that run are no longer kept");
  if (level < 0 || level >= (int)rl->size()) return set_error(AMS_EINVAL, "no such level");
  const ams_ctx::LevelRec& L = (*rl)[level];
  if (L.holders.empty()) {
    std::memset(holders, 0, 4 * (size_t)L.P);  // no sample (n == 0) or not recorded
    bool any = false;
    for (uint64_t d : L.drawn) any = any || d;
    if (any) return set_error(AMS_EINVAL, "splitter holders were not recorded (record_holders)");
    return AMS_OK;
  }
  std::memcpy(holders, L.holders.data(), 4 * L.holders.size());
  return AMS_OK;
}

}  // extern "C"
